#!/bin/bash
# bench.py at several stream counts (no CPU baseline / e2e), one line each
for s in ${STREAMS:-1 2 3 4}; do
  timeout 300 python bench.py --steps ${STEPS:-30} --warmup ${WARMUP:-10} --no-cpu --no-e2e --streams $s ${EXTRA} 2>/dev/null \
   | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('streams', $s, 'value %.0f' % d['value'], 'ms/step %.3f' % d['ms_per_step'], 'launches', d['gpu_launches'], {k: round(v, 3) for k, v in d['roofline']['kernel_ms'].items()})"
done
