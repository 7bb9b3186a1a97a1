"""Time the MPM extras (C3 step, C4 iteration) from bench.py; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

out = {"binned": os.environ.get("SG_NO_BIN") != "1"}
for name, fn in (("c3", bench.measure_c3), ("c4", bench.measure_c4)):
    try:
        out[name] = fn()
    except Exception as e:
        out[name] = {"error": repr(e)[:300]}
print(json.dumps(out))
