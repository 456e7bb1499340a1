#!/bin/bash
# One GPU call: the round's ncu evidence (run under gpurun from the repo root).
#   bash tools/profile_all.sh TAG [all|query-rays]
# Each target first runs once without ncu (must exit 0), then:
#   - launch list of 2 C2 bench steps (gpu__time_duration per kernel)
#   - --set full of the fused brick kernel (C2), the sorted o2 query kernel
#     (512^3, 2^26 points) and the radiance kernel with gradients
set -e
TAG=${1:-final}
OUT=gpurun_out
ONLY=${2:-all}
if [ "$ONLY" = all ]; then
python bench.py --steps 2 --warmup 3 --no-query --no-cpu-baseline --no-configs > $OUT/pa_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-query --no-cpu-baseline --no-configs > $OUT/pa_ncu_bench.log 2>&1
python tools/prof_train.py --steps 4 > $OUT/pa_train.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_brick_step -s 3 -c 1 -o $OUT/brick_$TAG -f \
    python tools/prof_train.py --steps 4 > $OUT/pa_ncu_train.log 2>&1
fi
python tools/prof_query.py --order 2 --reps 1 > $OUT/pa_query.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_eval_brick<.int.3, .int.2, .bool.0, .int.3, .int.0>" -c 1 -o $OUT/query_o2_$TAG -f \
    python tools/prof_query.py --order 2 --reps 1 > $OUT/pa_ncu_query.log 2>&1
python tools/prof_query.py --order 1 --reps 1 > $OUT/pa_query1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_eval_brick<.int.3, .int.1, .bool.0, .int.3, .int.0>" -c 1 -o $OUT/query_o1_$TAG -f \
    python tools/prof_query.py --order 1 --reps 1 > $OUT/pa_ncu_query1.log 2>&1
python tools/prof_radiance.py --no-margins > $OUT/pa_rays.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_rays<.int.2, .int.2, .bool.1>" \
    -c 1 -o $OUT/rays_$TAG -f python tools/prof_radiance.py --no-margins > $OUT/pa_ncu_rays.log 2>&1
echo profile_all done
