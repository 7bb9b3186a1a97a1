"""Short C5 driver for ncu: one GPU, 16M particles, n fused steps."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
args = argparse.Namespace(c5_particles=16_000_000, steps=n, warmup=1)
sim = bench.c5_sim(args, 0, 1, 0)
for _ in range(n):
    sim.step(fused=True)
torch.cuda.synchronize()
print("ok", sim.ranks[0].n())
