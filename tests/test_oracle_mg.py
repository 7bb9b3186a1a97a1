"""Pins for the multigrid ops.

* the oracle's V-cycles equal a dense numpy V-cycle written here from the
  textbook (red-black Gauss-Seidel, residual restriction by summation,
  piecewise-constant prolongation, A = -Laplacian with zero Dirichlet values
  outside the active region) -- brute force on a 64^2 instance, f64;
* restriction and prolongation are adjoint: <R u, v> = w <u, P v>;
* the residual norm decreases from cycle to cycle.
"""
import numpy as np
import pytest

import workloads as W
from oracle import Oracle, run_program

N, LEVELS, BLOCK, RADIUS = 64, 3, 8, 0.3


def run_exact(prog):
    o = Oracle(prog["desc"])
    o.set_exact(True)
    for c in prog["calls"]:
        o.call(c)
    return o


# ---- dense textbook reference (independent of the oracle) -----------------
def lap_apply(z, m):
    zz = np.pad(z * m, 1)
    nb = zz[2:, 1:-1] + zz[:-2, 1:-1] + zz[1:-1, 2:] + zz[1:-1, :-2]
    return (4.0 * z - nb) * m


def rb_half_sweep(z, r, m, parity):
    n = z.shape[0]
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    zz = np.pad(z * m, 1)
    nb = zz[2:, 1:-1] + zz[:-2, 1:-1] + zz[1:-1, 2:] + zz[1:-1, :-2]
    sel = (((ii + jj) & 1) == parity) & (m > 0)
    out = z.copy()
    out[sel] = ((r + nb) / 4.0)[sel]
    return out


def coarse_mask(m, block):
    n = m.shape[0] // 2
    mc = m.reshape(n, 2, n, 2).max(axis=(1, 3))
    b = min(block, n)
    nb = n // b
    return np.kron(mc.reshape(nb, b, nb, b).max(axis=(1, 3)), np.ones((b, b)))


def dense_vcycle(z, r, masks, l, nu=2, bottom=8, w=0.5):
    m = masks[l]
    if l == len(masks) - 1:
        for _ in range(bottom):
            z = rb_half_sweep(rb_half_sweep(z, r, m, 0), r, m, 1)
        return z
    for _ in range(nu):
        z = rb_half_sweep(rb_half_sweep(z, r, m, 0), r, m, 1)
    res = (r - lap_apply(z, m)) * m
    n = z.shape[0] // 2
    rc = res.reshape(n, 2, n, 2).sum(axis=(1, 3)) * w * masks[l + 1]
    zc = dense_vcycle(np.zeros((n, n)), rc, masks, l + 1, nu, bottom, w)
    z = z + np.kron(zc, np.ones((2, 2))) * m
    for _ in range(nu):
        z = rb_half_sweep(rb_half_sweep(z, r, m, 1), r, m, 0)
    return z


def dense_masks():
    m0 = np.zeros((N, N))
    for x, y in W.mg_region(N, BLOCK, RADIUS):
        m0[x:x + BLOCK, y:y + BLOCK] = 1.0
    masks = [m0]
    for _ in range(LEVELS - 1):
        masks.append(coarse_mask(masks[-1], BLOCK))
    return masks


@pytest.mark.parametrize("cycles", [1, 3])
def test_mg_vcycles_match_dense_textbook(cycles):
    prog = W.mg_program(n=N, levels=LEVELS, block=BLOCK, cycles=cycles, radius_frac=RADIUS)
    o = run_exact(prog)
    L = prog["layout"]
    masks = dense_masks()
    z = np.zeros((N, N))
    r = masks[0].copy()
    for _ in range(cycles):
        z = dense_vcycle(z, r, masks, 0)
    np.testing.assert_allclose(o.field(L.fields["z0"]), z, rtol=1e-12, atol=1e-12)
    res = ((r - lap_apply(z, masks[0])) ** 2).sum()
    assert float(np.asarray(o.field(L.fields["res"])).reshape(-1)[0]) == pytest.approx(res, rel=1e-12)
    # coarse levels are active exactly where restriction wrote (block granularity)
    for l in range(1, LEVELS):
        leaf = prog["levels"][l][-1]
        act = o.mask(prog["levels"][l][0])
        n = N >> l
        b = min(BLOCK, n)
        want = {(x // b, y // b) for x, y in zip(*np.nonzero(masks[l]))}
        assert {tuple(c) for c in np.asarray(act).reshape(-1, 2)} == want, l
        del leaf


def test_restriction_and_prolongation_are_adjoint():
    """<R u, v> = w <u, P v> with R u[C] = w sum_{c -> C} u[c] (RESTRICT with z = 0)
    and P v[c] = v[c // 2] (PROLONG into a zero field)."""
    L, lv = W.mg_layout(N, 2, BLOCK)
    f = L.fields
    coords = W.mg_region(N, BLOCK, RADIUS)
    rng = np.random.default_rng(1)
    w = 0.5
    o = Oracle(L.desc())
    o.set_exact(True)
    o.call(W.activate(f["z0"], coords))
    u = rng.standard_normal((N, N))
    o.load_field(f["r0"], u)
    o.call(W.struct_for("RESTRICT", lv[0][-1], [f["r1"], f["r0"], f["z0"]], [w], [True]))
    Ru = o.field(f["r1"])
    v = rng.standard_normal((N // 2, N // 2))
    o.load_field(f["z1"], v)
    o.call(W.struct_for("PROLONG", lv[0][-1], [f["z0"], f["z1"]]))
    Pv = o.field(f["z0"])
    m0 = dense_masks()[0]
    m1 = coarse_mask(m0, BLOCK)
    lhs = (Ru * v * m1).sum()
    rhs = w * (u * m0 * Pv).sum()
    assert lhs == pytest.approx(rhs, rel=1e-12)
    assert abs(lhs) > 1e-3


def test_mg_residual_decreases():
    res = []
    for cycles in (1, 2, 4, 8):
        prog = W.mg_program(n=N, levels=LEVELS, block=BLOCK, cycles=cycles, radius_frac=RADIUS)
        o = run_program(prog)
        res.append(float(np.asarray(o.field(prog["layout"].fields["res"])).reshape(-1)[0]))
    assert res[0] > res[1] > res[2] > res[3]
    assert res[3] < 0.25 * res[0]
