#!/bin/bash
# e2e (host-staged) images/s across staging options, one line each
for opt in ${OPTS:-"--gather-ctas 8" "--gather-ctas 16" "--gather-ctas 32" "--staging copy"}; do
  timeout 300 python bench.py --steps ${STEPS:-100} --warmup 10 --no-cpu $opt 2>/dev/null \
   | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$opt', 'value %.0f' % d['value'], 'e2e %.0f' % d['e2e']['value'])"
done
