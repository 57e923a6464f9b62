#!/bin/bash
# bench.py over (streams, seq_bits, overlap_bits)
for st in ${STREAMS:-3}; do for sb in ${SEQ:-1024 2048 4096}; do for ov in ${OV:-512 1024}; do
  timeout 300 python bench.py --steps ${STEPS:-40} --warmup 10 --no-cpu --no-e2e --streams $st --seq-bits $sb --overlap-bits $ov 2>/dev/null \
   | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('streams', $st, 'seq', $sb, 'ov', $ov, 'value %.0f' % d['value'], 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['roofline']['kernel_ms'].items()})"
done; done; done
