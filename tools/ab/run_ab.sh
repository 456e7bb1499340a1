#!/bin/bash
# Put the two builds at tools/ab/libtgcu_old.so and tools/ab/libtgcu_new.so first (gitignored);
# the script overwrites paper_2402_14415_b200/libtgcu.so on the box it runs on.
# A/B of two libtgcu builds on one box: bench step time, alternating.
for i in 1 2 3; do
  for v in old new; do
    cp tools/ab/libtgcu_$v.so paper_2402_14415_b200/libtgcu.so
    echo -n "$v "; python bench.py --steps 2000 --no-cpu-baseline --no-query --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))"
  done
done
for v in old new; do
  cp tools/ab/libtgcu_$v.so paper_2402_14415_b200/libtgcu.so
  echo -n "$v "; python tools/bench_configs.py c3 c5 --steps 20 2>/dev/null | python -c "import json,sys; print([ (json.loads(l)['config'], round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin if l.startswith('{')])"
done
