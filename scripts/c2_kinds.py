"""Per-launch-kind device time of one C2 solve (library events around each
launch group, direct launches): where the non-JACOBI part of the step goes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402

sg.jit_set_mode(2)
L, lv, coords, calls, result = bench.c2_setup(50)
dc = torch.as_tensor(coords).cuda()
g = sg.Grid(L.desc())
for _ in range(5):
    bench.enqueue_calls(g, calls, dc)
    g.flush("all")
torch.cuda.synchronize()
sg.set_profiling(g, True)
sg.profile_read(g)
for _ in range(5):
    bench.enqueue_calls(g, calls, dc)
    g.flush("all")
prof = sg.profile_read(g)
print(json.dumps({str(k): {"us_per_launch": t / max(c, 1) * 1e3, "launches_per_step": c / 5} for k, (t, c) in sorted(prof.items())}))
