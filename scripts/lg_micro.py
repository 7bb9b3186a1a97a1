"""Per-listgen device time inside a CUDA graph: a window of k explicit listgens
of the C4 grid tree's bitmasked level (no passes, so none is removed), k = 1, 41."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402

L, lv, lg = W.c4_layout(64)
g = sg.Grid(L.desc())
coords = W.c4_particles(100_000)["x"]
blocks = sorted({(int(x * 64) // 4 * 4, int(y * 64) // 4 * 4, int(z * 64) // 4 * 4) for x, y, z in coords.T})
dc = torch.as_tensor(blocks, dtype=torch.int32).cuda()
g.activate(L.fields["px"], dc)
g.flush("all")
g.sync()
res = {}
for k in (1, 41):
    for _ in range(3):
        for _ in range(k):
            g.listgen(lv[1])
        g.flush("none")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        for _ in range(k):
            g.listgen(lv[1])
        g.flush("none")
    e1.record()
    torch.cuda.synchronize()
    res[k] = e0.elapsed_time(e1) / 20
print(f"blocks {len(blocks)}; flush with 1 listgen pair {res[1]*1e3:.1f} us; per listgen pair in a graph {(res[41]-res[1])/40*1e3:.2f} us")
