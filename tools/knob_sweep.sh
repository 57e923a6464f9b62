#!/bin/bash
# bench.py over (streams, seq_bits, warm_bits)
for st in ${STREAMS:-3}; do for sb in ${SEQ:-1024 2048 4096}; do for ov in ${OV:-0 1024 2048}; do
  timeout 300 python bench.py --steps ${STEPS:-40} --warmup 10 --no-cpu --no-e2e --streams $st --seq-bits $sb --warm-bits $ov 2>/dev/null \
   | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('streams', $st, 'seq', $sb, 'ov', $ov, 'value %.0f' % d['value'], 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['roofline']['kernel_ms'].items()})"
done; done; done
