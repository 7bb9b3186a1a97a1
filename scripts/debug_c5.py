"""Diagnostics for the sharded MPM path (GPU): mismatch statistics vs the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_2012_08141_b200 import parallel, sg  # noqa: E402

NG, PTR, N = 128, 4, 30000
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = W.c5_particles(N, NG, length=100, width=16, seed=3, shear=40.0)
L, lv = W.c5_layout(NG, PTR)
prm = W.mpm_params(NG)
calls = []
for _ in range(steps):
    calls += W.c3_step_calls(L, lv, N, prm) + [W.flush()]
prog = W.program(L, calls, arrays=p)
o = oracle.run_program(prog)
g, st = sg.run_program(prog)
m_o, mag = o.field(L.fields["m"], with_mag=True)
m_g = g.field(L.fields["m"]).astype(np.float64)
d = np.abs(m_g - m_o)
print("plain GPU vs oracle: bad", (d > 1e-4 * np.maximum(np.abs(m_o), mag)).sum(), "max", d.max())
for world in (1, 2):
    sim = parallel.SlabMPM(NG, PTR, p, world, list(range(world)), parallel.LocalTransport(), prm,
                           lambda r: torch.device("cuda", 0), halo_cap=1024, mig_cap=8192)
    for _ in range(steps):
        sim.step()
    m_s = sim.gather_field("m").astype(np.float64)
    d = np.abs(m_s - m_o)
    bad = d > 1e-4 * np.maximum(np.abs(m_o), mag)
    print("world", world, "bad", bad.sum(), "max", d.max(), "sum_s", m_s.sum(), "sum_o", m_o.sum(), "sum_g", m_g.sum())
    idx = np.argwhere(bad)[:5]
    for c in idx:
        c = tuple(c)
        print("   ", c, m_s[c], m_o[c], m_g[c])
    for st in sim.ranks.values():
        print("   rank", st.rank, "n", st.n(), "halo counts", [int(st.bufs["halo"][k][0]) for k in ("sendL", "sendR", "recvL", "recvR")])
