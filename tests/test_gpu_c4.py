"""GPU parity of the C4 differentiable-MPM path (-m gpu).

* one backward substep, both sides fed the same seeded state and adjoint seed:
  grid-adjoint tree masks exact, grid adjoints and particle adjoints within
  1e-5 of the oracle's shadow magnitude M (readings R15, R32), at a small size
  and at the full 64^3 / 100K-particle size;
* a whole small forward + backward window (T = 4, all passes): the loss within
  1e-5, and every forward and backward substep of the window by single-step
  handoff (reading R17): the oracle's own state (and adjoint) entering the
  substep is loaded on both sides, one substep runs, everything within 1e-5 of M;
* full size (T = 64): the gradient is finite and its directional derivative
  along the initial velocity matches f32 central differences of the GPU loss.
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2012_08141_b200 import sg  # noqa: E402
from test_gpu_parity import as_set  # noqa: E402


def gpu_run(prog, passes=None):
    g = sg.Grid(prog["desc"])
    stats = sg.replay(g, prog, passes=passes, device="cuda")
    g.sync()
    return g, g.tensors, stats


def close(got, want, mag, tol, what, floor=0.0):
    """|got - want| <= tol * max(|want|, M, floor * max|want|): the floor covers
    entries whose true value is ~0 (e.g. d mean(x) / d v_y) where f32 roundoff
    of the O(scale) terms they are combined from exceeds their own M."""
    got = np.asarray(got, dtype=np.float64)
    bound = tol * np.maximum(np.maximum(np.abs(want), mag), floor * np.abs(want).max())
    bad = np.abs(got - want) > bound
    assert not bad.any(), (f"{what}: {bad.sum()}/{bad.size} off, worst abs {np.abs(got - want)[bad].max():.3e}, "
                           f"rel-to-M {(np.abs(got - want) / np.maximum(mag, 1e-300)).max():.3e}")


def one_substep_program(n_grid, n, seed, dt=2e-4):
    """Backward of one substep from the seeded initial state with a random
    adjoint seed of state 1 (no ADJ_INIT): identical inputs on both sides."""
    L, lv, lg = W.c4_layout(n_grid)
    prm = W.mpm_params(n_grid, dt=dt)
    arrays = W.c4_arrays(n, 1, n_grid, seed=seed)
    rng = np.random.default_rng(seed + 1)
    for k in ("x", "v", "C", "J"):
        arrays[f"adjA_{k}"] = rng.standard_normal(arrays[f"adjA_{k}"].shape).astype(np.float32)
    calls = W.c4_backward_calls(L, lv, lg, n, 1, prm)[1:]
    calls.append(W.flush())
    return W.program(L, calls, arrays=arrays, name="C4-1"), L, lg


def check_one_substep(prog, L, lg, tol=1e-5):
    o = oracle.run_program(prog)
    g, arrs, st = gpu_run(prog)
    for s in lg:
        if L.rows[s][0] in (W.BITMASKED, W.POINTER):
            assert as_set(g.mask(s)) == as_set(o.mask(s)), f"adjoint tree mask {s}"
    for name in ("gpx", "gpy", "gpz", "gm"):
        fid = L.fields[name]
        want, mag = o.field(fid, with_mag=True)
        close(g.field(fid), want, mag, tol, f"grid adjoint {name}")
    names = list(prog["arrays"])
    for i in range(12, 16):   # adjoint buffer B = d F / d state 0
        want, mag = o.array(i, with_mag=True)
        close(arrs[names[i]].cpu().numpy(), want, mag, tol, f"particle adjoint {names[i]}")
    return st


@pytest.mark.parametrize("binned", [True, False])
def test_c4_one_backward_substep_small(binned, monkeypatch):
    # binned kernels (default) and the per-particle kernels (SG_NO_BIN=1)
    if not binned:
        monkeypatch.setenv("SG_NO_BIN", "1")
    prog, L, lg = one_substep_program(32, 4000, seed=11)
    check_one_substep(prog, L, lg)


def test_c4_one_backward_substep_full_size():
    prog, L, lg = one_substep_program(64, 100_000, seed=12)
    check_one_substep(prog, L, lg)


def handoff_backward_program(n_grid, state, adj, prm):
    """One backward substep (recompute P2G, G2P_ADJ, P2G_ADJ) entering from a
    given particle state s and adjoint of state s+1 (both f32 on both sides)."""
    L, lv, lg = W.c4_layout(n_grid)
    n = state["x"].shape[1]
    arrays = W.c4_arrays(n, 1, n_grid)
    for k in ("x", "v", "C", "J"):
        arrays[f"{k}0"] = np.ascontiguousarray(state[k], dtype=np.float32)
        arrays[f"adjA_{k}"] = np.ascontiguousarray(adj[k], dtype=np.float32)
    calls = W.c4_backward_calls(L, lv, lg, n, 1, prm)[1:] + [W.flush()]
    return W.program(L, calls, arrays=arrays, name="C4-handoff"), L, lg


def handoff_forward_program(n_grid, state, prm):
    """One forward substep (DEACTIVATE, grad clears, P2G, GRID_OP, G2P) from a
    given particle state."""
    L, lv, lg = W.c4_layout(n_grid)
    n = state["x"].shape[1]
    arrays = W.c4_arrays(n, 1, n_grid)
    for k in ("x", "v", "C", "J"):
        arrays[f"{k}0"] = np.ascontiguousarray(state[k], dtype=np.float32)
    calls = W.c4_forward_calls(L, lv, lg, n, 1, prm)[:-2] + [W.flush()]
    return W.program(L, calls, arrays=arrays, name="C4-fwd-handoff"), L


@pytest.mark.parametrize("passes", [0, "all"])
def test_c4_small_window(passes):
    T, ng, n = 4, 32, 4000
    prog = W.c4_program(n_grid=ng, n_particles=n, T=T, seed=13, passes="all")
    prm = prog["params"]
    o = oracle.run_program(prog)
    g, arrs, st = gpu_run(prog, passes)
    L = prog["layout"]
    loss = float(g.field(L.fields["loss"]).reshape(-1)[0])
    want, mag = o.field(L.fields["loss"], with_mag=True)
    close(loss, want, mag, 1e-5, "loss")
    if passes == "all":
        assert st[0]["dead_removed"] == 8 * T
    names = list(prog["arrays"])
    keys = ("x", "v", "C", "J")

    def ostate(oo, s):
        return {k: oo.array(4 * s + i) for i, k in enumerate(keys)}

    # forward substeps s -> s+1 from the oracle's state s
    for s in range(T):
        p1, L1 = handoff_forward_program(ng, ostate(o, s), prm)
        o1 = oracle.run_program(p1)
        g1, a1, _ = gpu_run(p1, passes)
        n1 = list(p1["arrays"])
        for i in range(4, 8):
            want, mag = o1.array(i, with_mag=True)
            close(a1[n1[i]].cpu().numpy(), want, mag, 1e-5, f"forward substep {s}: {n1[i]}")
        for name in ("px", "py", "pz", "m"):
            want, mag = o1.field(L1.fields[name], with_mag=True)
            close(g1.field(L1.fields[name]), want, mag, 1e-5, f"forward substep {s}: grid {name}")
    # backward substeps: the oracle's adjoint of state s+1 (after ADJ_INIT and the
    # backward substeps T-1 .. s+1 of the eager program) and its state s
    n_fwd = len(W.c4_forward_calls(L, *W.c4_layout(ng)[1:], n, T, prm))
    A = [4 * (T + 1) + k for k in range(4)]
    B = [4 * (T + 1) + 4 + k for k in range(4)]
    for j, s in enumerate(reversed(range(T))):
        op = oracle.run_program(prog, upto=n_fwd + 1 + 5 * j)
        src = A if j % 2 == 0 else B
        adj = {k: op.array(src[i]) for i, k in enumerate(keys)}
        p1, L1, lg1 = handoff_backward_program(ng, ostate(o, s), adj, prm)
        check_one_substep(p1, L1, lg1)
    del names


def test_c4_full_size_gradient_properties():
    T, n = 64, 100_000
    prog = W.c4_program(n_grid=64, n_particles=n, T=T, seed=0)
    g, arrs, st = gpu_run(prog)
    L = prog["layout"]
    names = list(prog["arrays"])
    grads = [arrs[names[i]].double().cpu().numpy() for i in prog["result_arrays"]]
    assert all(np.isfinite(a).all() for a in grads)
    # momentum: the summed x-gradient w.r.t. v0_x is T dt (f32 params) up to f32 drift
    dt32 = float(np.float32(prog["params"]["dt"]))
    assert grads[1][0].sum() == pytest.approx(T * dt32, rel=2e-3)
    # directional derivative along a random v0 perturbation vs f32 central differences
    # (d_x has mean 1 so the loss change, ~T dt h, sits well above the f32 loss resolution)
    d = np.random.default_rng(3).standard_normal((3, n)).astype(np.float32)
    d[0] += 1.0
    v0 = prog["arrays"]["v0"]
    h = 0.05
    Lf, lv, lg = W.c4_layout(64)

    def loss_at(v):
        arrays = dict(prog["arrays"])
        arrays["v0"] = v.astype(np.float32)
        calls = W.c4_forward_calls(Lf, lv, lg, n, T, prog["params"]) + [W.flush()]
        gg, _, _ = gpu_run(W.program(Lf, calls, arrays=arrays))
        return float(gg.field(Lf.fields["loss"]).reshape(-1)[0])

    fd = (loss_at(v0 + h * d) - loss_at(v0 - h * d)) / (2 * h)
    ad = float((grads[1] * d).sum())
    assert ad == pytest.approx(fd, rel=2e-2, abs=2e-6)
