#!/bin/bash
# C4 query leg under several environment settings (one process each):
#   bash tools/qvar_env.sh "TGCU_UNSCATTER_MB=0" "TGCU_UNSCATTER_MB=48" ...
for i in 1 2; do
  for e in "$@"; do
    echo -n "$e "
    env $e python -c "
import json, bench
q = bench.query_leg(0, 6549.1, reps=10, cpu=False)
print(json.dumps({k: (round(v['ms'], 3), round(v['frac'], 3)) for k, v in q.items() if isinstance(v, dict) and 'ms' in v}), round(q.get('sort_ms', 0), 3))
"
  done
done
