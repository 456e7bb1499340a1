"""Time the C4 query leg against an alternative libtgcu build (A/B variants).

    python tools/qvar_run.py path/to/libtgcu.so
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2402_14415_b200 as tg  # noqa: E402

tg.LIB_PATH = os.path.abspath(sys.argv[1])
import bench  # noqa: E402

q = bench.query_leg(0, 6549.1, reps=10)
print(os.path.basename(sys.argv[1]), json.dumps({k: (round(v["ms"], 3), round(v["frac"], 3)) for k, v in q.items()
                                                 if isinstance(v, dict)}))
