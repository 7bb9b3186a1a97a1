"""C2 solve timed as bench.py times its headline (device events around each
flush, steps pipelined, L2 flushed before each) with passes "all" (one launch
per sweep, graph-replayed) and "all+chain" (the sweeps as one flag-chained
launch, or two sweeps per launch with SG_T2=1; kernels_flow.cu); one JSON line."""
import json
import os
import sys

# the chain pass runs the flag-chained kernel (SG_FLOW=1) unless SG_T2=1 picks
# the two-sweep kernel
if os.environ.get("SG_T2") != "1":
    os.environ.setdefault("SG_FLOW", "1")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
out = {}
L, lv, coords, calls, result = bench.c2_setup(50)
dc = torch.as_tensor(coords).cuda()
l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
for passes in ("all", "all+chain", "all"):
    g = sg.Grid(L.desc())
    for _ in range(5):
        bench.enqueue_calls(g, calls, dc)
        g.flush(passes)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        l2.zero_()
        a.record(stream)
        bench.enqueue_calls(g, calls, dc)
        st = g.flush(passes)
        b.record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    out[passes if passes not in out else passes + "_again"] = {
        "solves_per_s": 1000.0 / ms, "ms_per_step": ms, "launches": st["launches"],
        "chained": st.get("launches_chained"), "s": float(g.field(L.fields["s"]))}
    g.close()
print(json.dumps(out))
