"""Parity margins on the GPU: for each case, the worst |g - o| / max(|o|, M)
over every compared element (the tolerance the case would need).  Diagnostic
for choosing handoff points; not a test.  python scripts/parity_margins.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402


def margin(got, want, mag):
    got = np.asarray(got, dtype=np.float64)
    den = np.maximum(np.abs(want), mag)
    r = np.where(den > 0, np.abs(got - want) / np.where(den > 0, den, 1), np.where(got != want, np.inf, 0))
    return float(r.max()) if r.size else 0.0


def grid_margins(g, o, prog, arrays=True):
    L = prog["layout"]
    out = {}
    for name, fid in L.fields.items():
        want, mag = o.field(fid, with_mag=True)
        out[name] = margin(g.field(fid), want, mag)
    if arrays:
        for i, name in enumerate(prog.get("arrays", {})):
            want, mag = o.array(i, with_mag=True)
            out["a:" + name] = margin(g.tensors[name].cpu().numpy(), want, mag)
    return out


def run(prog, passes=None):
    g = sg.Grid(prog["desc"])
    sg.replay(g, prog, passes=passes, device="cuda")
    g.sync()
    return g


def report(name, d):
    worst = max(d.values()) if d else 0
    print(f"{name:40s} worst {worst:.2e}  " + " ".join(f"{k}={v:.1e}" for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:6]),
          flush=True)


def main():
    import test_gpu_c4 as C4
    for ng, n, seed in ((32, 4000, 11), (64, 100_000, 12)):
        prog, L, lg = C4.one_substep_program(ng, n, seed)
        o = oracle.run_program(prog)
        g = run(prog)
        d = grid_margins(g, o, prog, arrays=False)
        names = list(prog["arrays"])
        for i in range(12, 16):
            want, mag = o.array(i, with_mag=True)
            d[names[i]] = margin(g.tensors[names[i]].cpu().numpy(), want, mag)
        report(f"C4 one backward substep {ng}^3 {n}", d)
    for cycles in (1, 2):
        prog = W.mg_program(n=64, levels=3, block=8, cycles=cycles, radius_frac=0.3)
        report(f"MG 64^2 {cycles} cycles", grid_margins(run(prog), oracle.run_program(prog), prog))
    prog = W.mg_program(n=512, cycles=1)
    report("MG 512^2 1 cycle", grid_margins(run(prog), oracle.run_program(prog), prog))
    for it in (1, 2):
        prog = W.mgpcg_program(n=64, levels=3, block=8, iters=it, radius_frac=0.3)
        report(f"MGPCG 64^2 {it} it", grid_margins(run(prog), oracle.run_program(prog), prog))
    prog = W.c3_program(n_grid=32, n_particles=3000, steps=3, flush_every=3, seed=6, v_scale=0.5)
    report("C3 32^3 3 steps", grid_margins(run(prog), oracle.run_program(prog), prog))


if __name__ == "__main__":
    main()
