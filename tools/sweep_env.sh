#!/bin/bash
# A/B of one environment knob on the bench step: tools/sweep_env.sh VAR "v1 v2 ..." [bench args]
# prints value, ms_per_step, factorize_ms, solve_ms per setting (run on the GPU box).
VAR=$1; VALS=$2; shift 2
for v in $VALS; do
  if [ "$v" = "unset" ]; then unset $VAR; else export $VAR=$v; fi
  python bench.py --no-cpu-baseline --no-accuracy --no-clocks "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$VAR=$v', d['config']['workload'], 'step', d['ms_per_step'], 'fact', d['factorize_ms'], 'solve', d['solve_ms'], 'e2e', d['e2e']['ms_per_step'])"
done
