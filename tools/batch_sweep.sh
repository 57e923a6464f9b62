#!/bin/bash
# bench.py over (batch, streams) pairs, one line each (no CPU baseline / e2e)
for bs in ${PAIRS:-256:6 512:3 512:4 1024:2 1024:3}; do
  b=${bs%%:*}; s=${bs##*:}
  timeout 300 python bench.py --steps ${STEPS:-100} --warmup ${WARMUP:-10} --no-cpu --no-e2e --batch $b --streams $s ${EXTRA} 2>/dev/null \
   | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('batch', $b, 'streams', $s, 'value %.0f' % d['value'], 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['roofline']['kernel_ms'].items()})"
done
