#!/bin/bash
# C2 bench step under alternating environment settings: run_env.sh "VAR=a" "VAR=b" ...
for i in 1 2; do
  for e in "$@"; do
    echo -n "$e "; env $e python bench.py --steps 2000 --no-cpu-baseline --no-query --no-configs --no-stages --e2e-steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
  done
done
