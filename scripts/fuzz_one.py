"""One case of tests/test_gpu_fuzz.py by seed, with overrides (repro aid):
    python scripts/fuzz_one.py SEED [host|dev] [key=value ...]     e.g. fmt=0 d=3208 L=2 nq=5 sizes=2,5,3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import test_gpu_fuzz as F  # noqa: E402

c = F.draw_case(int(sys.argv[1]))
for a in sys.argv[2:]:
    if a in ("host", "dev"):
        c["host"] = a == "host"
    else:
        k, v = a.split("=")
        c[k] = [int(x) for x in v.split(",")] if k == "sizes" else int(v)
print(c, flush=True)
print("pairs", F.run_case(c), "ok")
