#!/bin/bash
# Same-box A/B of several libtgcu builds (tools/ab/libtgcu_NAME.so, gitignored):
#   bash tools/ab/run_abn.sh NAME1 NAME2 ...   (C2 bench step time, 3 rounds, alternating)
for i in 1 2 3; do
  for v in "$@"; do
    cp tools/ab/libtgcu_$v.so paper_2402_14415_b200/libtgcu.so
    echo -n "$v "; python bench.py --steps 2000 --no-cpu-baseline --no-query --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
  done
done
