"""Short C2 driver for ncu: a few solves through the C-ABI (all passes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
L, lv, coords, calls, result = bench.c2_setup(50)
g = sg.Grid(L.desc())
dc = torch.as_tensor(coords).cuda()
for _ in range(n):
    bench.enqueue_calls(g, calls, dc)
    g.flush("all")
torch.cuda.synchronize()
print("ok", float(g.field(L.fields["s"])))
