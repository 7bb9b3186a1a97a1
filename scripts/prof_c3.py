"""Short C3 driver for ncu: a few MPM steps (1M particles, 128^3)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
print(bench.measure_c3(steps=n, warmup=1))
