"""Host cost of one C2 solve flush (enqueue + sg_flush, no sync) vs its device time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402

L, lv, coords, calls, result = bench.c2_setup(50)
g = sg.Grid(L.desc())
dc = torch.as_tensor(coords).cuda()
for _ in range(5):
    bench.enqueue_calls(g, calls, dc)
    g.flush("all")
torch.cuda.synchronize()
N = 50
host = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N):
    t0 = time.perf_counter()
    bench.enqueue_calls(g, calls, dc)
    t1 = time.perf_counter()
    g.flush("all")
    t2 = time.perf_counter()
    host.append((t1 - t0, t2 - t1))
e1.record()
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) / N
enq = sum(h[0] for h in host) / N * 1e6
fl = sum(h[1] for h in host) / N * 1e6
print(f"per solve: device {dev*1e3:.1f} us, host enqueue {enq:.1f} us, host flush {fl:.1f} us (55 launches)")
