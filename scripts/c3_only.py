"""C3 steps/s and per-kernel launch times (both particle layouts) from bench.measure_c3; one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.measure_c3()
print(json.dumps({v: {"steps_per_s": r[v]["steps_per_s"],
                      "us": {n: round(e["avg_launch_us"], 1) for n, e in r[v]["kernels"].items()}}
                  for v in ("in_place", "bin_order")}))
