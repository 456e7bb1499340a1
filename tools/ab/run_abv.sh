#!/bin/bash
# A/B of several libtgcu builds on one box (C2 bench step): tools/ab/libtgcu_<name>.so for each name given
for i in 1 2; do
  for v in "$@"; do
    cp tools/ab/libtgcu_$v.so paper_2402_14415_b200/libtgcu.so
    echo -n "$v "; python bench.py --steps 2000 --no-cpu-baseline --no-query --no-configs --no-stages --e2e-steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
  done
done
