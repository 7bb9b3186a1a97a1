"""Probe (one GPU): C5 step time and particle count over many host-synchronous
steps (the step cost must stay flat; the count is conserved)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2012_08141_b200 import sg
class A: pass
args = A(); args.c5_particles = 16_000_000; args.warmup = 3; args.steps = 10
sg.jit_set_mode(2)
sim = bench.c5_sim(args, 0, 1, 0)
me = sim.ranks[0]
for _ in range(3): sim.step(fused=True)
torch.cuda.synchronize()
out = {"no_sync": [], "sync_each": [], "item_each": []}
t0 = time.perf_counter()
for _ in range(10): sim.step(fused=True)
torch.cuda.synchronize(); out["no_sync"].append((time.perf_counter() - t0) * 100)
for _ in range(10):
    t0 = time.perf_counter(); st = sim.step(fused=True); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    out["sync_each"].append((round((t1-t0)*1e3,2), round((t2-t1)*1e3,2), st[0]["launches"], st[0].get("plan_cache_hits"), st[0].get("aux_kernels")))
for _ in range(40):
    t0 = time.perf_counter(); st = sim.step(fused=True); t1 = time.perf_counter(); _ = int(me.count[0].item()); t2 = time.perf_counter()
    out["item_each"].append((round((t1-t0)*1e3,2), round((t2-t1)*1e3,2), _))
print(json.dumps(out))
