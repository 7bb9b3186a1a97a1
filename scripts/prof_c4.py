"""One C4 forward+backward iteration (T substeps, default 8) for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prog = W.c4_program(n_grid=64, n_particles=100_000, T=T)
g = sg.Grid(prog["desc"])
for it in range(iters):
    sg.replay(g, prog, device="cuda")
    g.sync()
print("loss", float(g.field(prog["layout"].fields["loss"]).reshape(-1)[0]))
