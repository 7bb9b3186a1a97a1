"""Pins for the C4 (differentiable MPM) oracle ops.

The adjoint ops (G2P_ADJ with the grid-op adjoint folded in, P2G_ADJ) and the
loss are pinned against central finite differences of the oracle's own forward
pass in exact (f64) mode -- the gradient is a property of the forward map, so a
dropped term, a wrong sign or a transposed operand anywhere in the hand-written
adjoints fails one of the directional-derivative checks below (SURVEY.md s4:
"the full gradient matches f64 central differences on a tiny instance").
PAPER.md:174 (two-scale AD: kernels plus their gradients).
"""
import numpy as np
import pytest

import workloads as W
from oracle import Oracle

pytestmark = pytest.mark.filterwarnings("ignore")

N_GRID, N, T = 16, 100, 4


def make(dt=1e-3, seed=3, **kw):
    L, lv, lg = W.c4_layout(N_GRID)
    prm = W.mpm_params(N_GRID, dt=dt)
    arrays = W.c4_arrays(N, T, N_GRID, side=6, center=(0.5, 0.5, 0.5), seed=seed, **kw)
    return L, lv, lg, prm, arrays


def run(L, arrays, calls, over=None, exact=True):
    o = Oracle(L.desc())
    o.set_exact(exact)
    for a in arrays.values():
        o.register_array(a)
    for i, data in (over or {}).items():
        o.load_array(i, data)
    for c in calls:
        o.call(c)
    return o


def seeds(arrays, seed=7):
    """Random adjoint seed r over the final state (x_T, v_T, C_T, J_T)."""
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(np.shape(arrays[f"{k}0"])) for k in ("x", "v", "C", "J")]


def functional(L, lv, lg, prm, arrays, over, r):
    """F = <r, state_T>: a linear readout of every component of the final
    state, so the pins reach the v, C and J adjoint paths (the mean-x loss is
    blind to C and J at first order: the B-spline first moment vanishes and
    internal forces cancel)."""
    o = run(L, arrays, W.c4_forward_calls(L, lv, lg, N, T, prm), over)
    return sum(float((o.array(4 * T + k) * r[k]).sum()) for k in range(4))


@pytest.fixture(scope="module")
def c4():
    L, lv, lg, prm, arrays = make()
    r = seeds(arrays)
    back = W.c4_backward_calls(L, lv, lg, N, T, prm)
    assert back[0]["op"] == "ADJ_INIT"
    A = [4 * (T + 1) + k for k in range(4)]
    o = run(L, arrays, W.c4_forward_calls(L, lv, lg, N, T, prm))
    for k in range(4):
        o.load_array(A[k], r[k])
    for c in back[1:]:
        o.call(c)
    grads = [o.array(i) for i in W.c4_result_arrays(T)]
    base = [np.asarray(arrays[k], dtype=np.float64) for k in ("x0", "v0", "C0", "J0")]
    return L, lv, lg, prm, arrays, grads, base, o, r


@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_c4_gradient_matches_central_differences(c4, which):
    """<dF/dp, d> == (F(p + h d) - F(p - h d)) / 2h for a random direction d
    over every particle's x0 / v0 / C0 / J0 (f64 throughout)."""
    L, lv, lg, prm, arrays, grads, base, _, r = c4
    rng = np.random.default_rng(100 + which)
    d = rng.standard_normal(base[which].shape)
    h = 1e-6
    fp = functional(L, lv, lg, prm, arrays, {which: base[which] + h * d}, r)
    fm = functional(L, lv, lg, prm, arrays, {which: base[which] - h * d}, r)
    fd = (fp - fm) / (2 * h)
    ad = float((grads[which] * d).sum())
    assert abs(fd) > 1e-3, "direction with no effect: the pin would be vacuous"
    assert ad == pytest.approx(fd, rel=1e-6)


def test_c4_gradient_single_particle_components(c4):
    """Per-entry central differences for a few (array, component, particle);
    the step balances truncation (x enters through the B-spline, curvature
    ~ inv_dx^2) against f64 cancellation in F (|F| ~ 1e2; C-gradients are small)."""
    L, lv, lg, prm, arrays, grads, base, _, r = c4
    hs = {0: 1e-6, 1: 1e-6, 2: 1e-4, 3: 1e-5}
    for which, comp, i in [(0, 0, 7), (0, 1, 31), (0, 2, 64), (1, 0, 5), (1, 1, 9), (2, 4, 11), (2, 0, 42), (3, 0, 77)]:
        e = np.zeros_like(base[which])
        e[comp, i] = 1.0
        h = hs[which]
        fp = functional(L, lv, lg, prm, arrays, {which: base[which] + h * e}, r)
        fm = functional(L, lv, lg, prm, arrays, {which: base[which] - h * e}, r)
        fd = (fp - fm) / (2 * h)
        assert abs(fd) > 1e-4
        assert grads[which][comp, i] == pytest.approx(fd, rel=1e-5), (which, comp, i)


def test_c4_mean_loss_pipeline_matches_central_differences():
    """The bench pipeline (LOSS_MEAN + ADJ_INIT): dL/dv0 against central
    differences of the loss field."""
    L, lv, lg, prm, arrays = make()
    calls = W.c4_forward_calls(L, lv, lg, N, T, prm) + W.c4_backward_calls(L, lv, lg, N, T, prm)
    o = run(L, arrays, calls)
    gv = o.array(W.c4_result_arrays(T)[1])
    base = np.asarray(arrays["v0"], dtype=np.float64)
    d = np.random.default_rng(5).standard_normal(base.shape)
    h = 1e-6

    def loss(v):
        oo = run(L, arrays, W.c4_forward_calls(L, lv, lg, N, T, prm), {1: v})
        return float(np.asarray(oo.field(L.fields["loss"])).reshape(-1)[0])

    fd = (loss(base + h * d) - loss(base - h * d)) / (2 * h)
    assert float((gv * d).sum()) == pytest.approx(fd, rel=1e-6)


def test_c4_loss_is_mean_position(c4):
    """LOSS_MEAN: loss = mean over particles of x_T[comp] (closed form)."""
    L, lv, lg, prm, arrays, grads, base, o, r = c4
    xT = o.array(4 * T)
    assert float(np.asarray(o.field(L.fields["loss"])).reshape(-1)[0]) == pytest.approx(
        xT[0].sum() * float(np.float32(1.0 / N)), rel=1e-14)   # task params are f32 (1/n rounded)


def test_c4_zero_steps_gradient_is_closed_form():
    """T = 0: loss = mean x0[comp], so dL/dx0 = e_comp / n and the rest is 0."""
    L, lv, lg = W.c4_layout(N_GRID)
    prm = W.mpm_params(N_GRID)
    arrays = W.c4_arrays(N, 0, N_GRID, side=6, center=(0.5, 0.5, 0.5))
    calls = W.c4_forward_calls(L, lv, lg, N, 0, prm, comp=1) + W.c4_backward_calls(L, lv, lg, N, 0, prm, comp=1)
    o = run(L, arrays, calls)
    gx, gv, gC, gJ = [o.array(i) for i in W.c4_result_arrays(0)]
    want = np.zeros_like(gx)
    want[1] = float(np.float32(1.0 / N))
    np.testing.assert_allclose(gx, want, rtol=0, atol=1e-15)
    assert not gv.any() and not gC.any() and not gJ.any()


def test_c4_out_of_place_g2p_matches_in_place():
    """G2P writing state s+1 to separate arrays is the C3 in-place G2P."""
    L, lv, lg, prm, arrays = make(dt=1e-3)
    o = run(L, arrays, W.c4_forward_calls(L, lv, lg, N, 1, prm), exact=False)
    L3, lv3 = W.c3_layout(N_GRID)
    parts = {k: arrays[f"{k}0"] for k in ("x", "v", "C", "J")}
    p3 = W.program(L3, W.c3_step_calls(L3, lv3, N, prm), arrays=parts)
    from oracle import run_program
    o3 = run_program(p3)
    for k in range(4):
        np.testing.assert_array_equal(o.array(4 + k), o3.array(k))


def test_c4_free_fall_velocity_gradient():
    """Pure free fall with E = 0 and C = 0, v = const: one step moves every
    particle by dt * (v - dt g e_y) (grid velocity is the particle velocity
    minus gravity), so the summed d mean(x_T) / d v0_x is T dt."""
    L, lv, lg = W.c4_layout(N_GRID)
    prm = W.mpm_params(N_GRID, dt=1e-3, E=0.0)
    arrays = W.c4_arrays(N, 2, N_GRID, side=6, center=(0.5, 0.5, 0.5), C_scale=0.0, J_jitter=0.0, v_scale=0.0)
    calls = W.c4_forward_calls(L, lv, lg, N, 2, prm) + W.c4_backward_calls(L, lv, lg, N, 2, prm)
    o = run(L, arrays, calls)
    gx, gv, gC, gJ = [o.array(i) for i in W.c4_result_arrays(2)]
    # uniform translation: total x-momentum per unit v is conserved by the
    # transfers, so the summed gradient is exact even where individual entries mix
    dt32, inv_n32 = float(np.float32(prm["dt"])), float(np.float32(1.0 / N))   # f32 task params
    assert gv[0].sum() == pytest.approx(2 * dt32 * inv_n32 * N, rel=1e-12)
    assert gx[0].sum() == pytest.approx(inv_n32 * N, rel=1e-12)
    assert not gv[1:].any() or np.abs(gv[1:]).max() < 1e-14
