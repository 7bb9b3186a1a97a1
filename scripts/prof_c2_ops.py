"""Per-op device time of one C2 solve (library events around each launch, direct launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402

L, lv, coords, calls, result = bench.c2_setup(50)
g = sg.Grid(L.desc())
dc = torch.as_tensor(coords).cuda()
names = {100 + v: k for k, v in sg.OPS.items()}
names.update({0: "activate", 1: "listgen", 2: "clear_list", 3: "struct_for", 4: "range_for", 5: "serial", 6: "deactivate"})
for rep in range(4):
    bench.enqueue_calls(g, calls, dc)
    if rep == 3:
        sg.set_profiling(g, True)
        sg.profile_read(g)
    g.flush("all")
    torch.cuda.synchronize()
res = sg.profile_read(g)
for k, (ms, n) in sorted(res.items()):
    print(f"{names.get(k, k)!s:14s} n={n:3d} avg={ms / n * 1e3:8.2f} us total={ms * 1e3:8.1f} us")

