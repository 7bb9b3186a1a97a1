"""Probe (one GPU): where the time of a host-synchronous C5 step goes
(device events per step, host time of the enqueue and of the sync)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402


class A:
    pass


args = A()
args.c5_particles = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
args.warmup, args.steps = 3, 10
sg.jit_set_mode(2)
sim = bench.c5_sim(args, 0, 1, 0)
for _ in range(3):
    sim.step(fused=True)
torch.cuda.synchronize()
stream = torch.cuda.current_stream()
rows = []
for _ in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(stream)
    st = sim.step(fused=True)
    b.record(stream)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rows.append({"enqueue_ms": (t1 - t0) * 1e3, "sync_ms": (t2 - t1) * 1e3, "device_ms": a.elapsed_time(b),
                 "launches": [s["launches"] for s in st], "plan_us": [s.get("plan_us") for s in st]})
print(json.dumps(rows))
