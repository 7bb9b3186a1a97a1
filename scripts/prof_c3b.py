"""Short C3 driver for ncu: bin-order layout (1M particles, 128^3), n steps."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workloads as W  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prog = W.c3_program(n_grid=128, n_particles=1_000_000, steps=n, bin_order=True)
g = sg.Grid(prog["desc"])
sg.replay(g, prog, device="cuda")
g.sync()
print("ok")
