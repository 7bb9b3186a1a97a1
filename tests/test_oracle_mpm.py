"""Pins of the oracle's MLS-MPM ops (-m "not gpu").

What fixes them (MLS-MPM, hu2018moving, the method PAPER.md:444 builds on):
* the quadratic B-spline weights are a partition of unity and reproduce linear
  functions: sum_i w_ip = 1 and sum_i w_ip (x_i - x_p) = 0, so P2G conserves
  mass exactly and momentum = sum_p m_p v_p (the affine/stress terms vanish in
  the sum) -- closed forms;
* free fall from rest for one step gives v = -dt g e_y, C = 0, J = 1 --
  special case;
* a uniform translation is transported unchanged (g = 0) -- special case.
"""
import numpy as np

import oracle
import workloads as W


def p2g_only(n_particles=3000, seed=1, v_scale=1.0, J_jitter=0.05, C_scale=2.0):
    L, lv = W.c3_layout(32)
    prm = W.mpm_params(32)
    arrays = W.mpm_particles(n_particles, 0.2, 0.7, seed, v_scale, J_jitter)
    rng = np.random.default_rng(seed + 7)
    arrays["C"] = (rng.uniform(-1, 1, size=(9, n_particles)) * C_scale).astype(np.float32)
    f = L.fields
    calls = [W.range_for("P2G", n_particles, [f["vx"], f["vy"], f["vz"], f["m"]], [0, 1, 2, 3],
                         [prm["dt"], prm["inv_dx"], prm["p_mass"], prm["p_vol"], prm["E"]], [True] * 4)]
    prog = W.program(L, calls, arrays=arrays)
    return prog, oracle.run_program(prog), prm


def test_p2g_conserves_mass_and_momentum():
    prog, o, prm = p2g_only()
    L = prog["layout"]
    f = L.fields
    n = prog["arrays"]["x"].shape[1]
    m = o.field(f["m"])
    np.testing.assert_allclose(m.sum(), n * prm["p_mass"], rtol=1e-6)
    v = prog["arrays"]["v"].astype(np.float64)
    for a, name in enumerate(("vx", "vy", "vz")):
        mom, mag = o.field(f[name], with_mag=True)
        want = prm["p_mass"] * v[a].sum()
        assert abs(mom.sum() - want) <= 1e-5 * mag.sum(), name


def test_p2g_activates_exactly_the_stencil_blocks():
    prog, o, prm = p2g_only(500)
    x = prog["arrays"]["x"]
    X = (x * np.float32(prm["inv_dx"])).astype(np.float32)
    base = np.floor((X - np.float32(0.5)).astype(np.float32)).astype(np.int64)
    blocks = set()
    for p in range(x.shape[1]):
        for off in np.ndindex(3, 3, 3):
            blocks.add(tuple((base[:, p] + np.array(off)) // 4))
    L, lv = W.c3_layout(32)
    got = set(map(tuple, o.mask(lv[1]).tolist()))
    assert got == blocks


def test_free_fall_one_step():
    prog = W.c3_program(n_grid=32, n_particles=2000, steps=1, seed=3)
    o = oracle.run_program(prog)
    prm = W.mpm_params(32)
    v, C, J, x = o.array(1), o.array(2), o.array(3), o.array(0)
    np.testing.assert_allclose(v[1], -prm["dt"] * prm["gravity"], rtol=1e-6)
    np.testing.assert_allclose(v[0], 0, atol=1e-12)
    assert np.abs(C).max() < 1e-8
    np.testing.assert_allclose(J, 1.0, rtol=1e-7)
    x0 = prog["arrays"]["x"].astype(np.float64)
    np.testing.assert_allclose(x[1], x0[1] - prm["dt"] ** 2 * prm["gravity"], atol=1e-7)


def test_uniform_translation():
    prog = W.c3_program(n_grid=32, n_particles=2000, steps=2, seed=4, gravity=0.0)
    u = np.array([0.3, -0.2, 0.1], dtype=np.float32)
    prog["arrays"]["v"][:] = u[:, None]
    o = oracle.run_program(prog)
    v = o.array(1)
    for a in range(3):
        np.testing.assert_allclose(v[a], u[a], rtol=1e-5)
    assert np.abs(o.array(2)).max() < 1e-4
    assert prog["calls"][0]["call"] == "clear"
    assert o.tasks_eager_folded == 16      # 8 lowered tasks per step (reading R19 analog for C3)


# ---------------------------------------------------------------------------
# Closed-form pins of the forward MLS-MPM terms (hu2018moving, the transfer
# scheme PAPER.md:444 cites; reading R28).  They fix what the conservation pins
# above are blind to: the APIC scale 4/dx^2 in G2P, the affine term p_mass*C and
# the stress -dt*4*E*p_vol*(J-1)/dx^2 in P2G, and the J update.
#
# Facts used (quadratic B-spline, nodes x_i = i*dx):
#   sum_i w_ip = 1,  sum_i w_ip (x_i - x_p) = 0,
#   D_p = sum_i w_ip (x_i - x_p)(x_i - x_p)^T = dx^2/4 * I.
# Hence for an affine grid velocity u(x) = A x + b, G2P gives
#   v_p = A x_p + b,  C_p = (4/dx^2) sum_i w_ip u_i (x_i - x_p)^T = A,
#   J' = J (1 + dt tr A),  x' = x + dt v_p;
# and P2G of one particle gives the grid first moment
#   sum_i p_i (x_i - x_p)^T = aff * D_p = aff * dx^2/4,
#   aff = p_mass*C - dt*4*E*p_vol*(J-1)/dx^2 * I,
# with sum_i p_i = p_mass v and sum_i m_i = p_mass.
# ---------------------------------------------------------------------------
def _region_coords(lo, hi):
    r = np.arange(lo, hi)
    return np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)


def _g2p_affine(A, b, n_particles=40, seed=11, n_grid=32, dt=1e-3, J0=None):
    L, lv = W.c3_layout(n_grid)
    f = L.fields
    inv_dx = float(n_grid)
    dx = 1.0 / n_grid
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.35, 0.65, size=(3, n_particles)).astype(np.float32)
    J = (rng.uniform(0.8, 1.2, size=(1, n_particles)) if J0 is None else np.full((1, n_particles), J0)).astype(np.float32)
    arrays = {"x": x, "v": np.zeros((3, n_particles), np.float32), "C": np.zeros((9, n_particles), np.float32), "J": J}
    o = oracle.Oracle(L.desc())
    o.set_exact(True)
    for name in ("x", "v", "C", "J"):
        o.register_array(arrays[name])
    o.activate(f["vx"], _region_coords(8, 24))
    idx = np.stack(np.meshgrid(*(np.arange(n_grid),) * 3, indexing="ij"), 0).astype(np.float64) * dx
    for r, name in enumerate(("vx", "vy", "vz")):
        u = b[r] + sum(A[r][d] * idx[d] for d in range(3))
        o.load_field(f[name], u)
    o.range_for_task("G2P", n_particles, [f["vx"], f["vy"], f["vz"]], [0, 1, 2, 3], [dt, inv_dx])
    return o, x.astype(np.float64), J.astype(np.float64)


def _f32(v):
    """Task params cross the ABI as f32 (sg_task.params): expected values use the rounded ones."""
    return float(np.float32(v))


def test_g2p_recovers_affine_velocity_field():
    rng = np.random.default_rng(5)
    A = rng.uniform(-2, 2, size=(3, 3))
    b = rng.uniform(-1, 1, size=3)
    dt = _f32(1e-3)
    o, x0, J0 = _g2p_affine(A, b, dt=dt)
    v, C, J, x = o.array(1), o.array(2), o.array(3), o.array(0)
    want_v = A @ x0 + b[:, None]
    np.testing.assert_allclose(v, want_v, rtol=0, atol=1e-12)
    # C stored row-major: C[3r+d] = dv_r / dx_d
    np.testing.assert_allclose(C, np.repeat(A.reshape(9, 1), x0.shape[1], 1), rtol=0, atol=1e-10)
    np.testing.assert_allclose(J, J0 * (1.0 + dt * np.trace(A)), rtol=1e-13)
    np.testing.assert_allclose(x, x0 + dt * want_v, rtol=0, atol=1e-13)


def test_g2p_uniform_expansion_updates_J():
    # u = alpha * x  =>  C = alpha I, J' = J (1 + 3 alpha dt)
    alpha, dt = 0.7, _f32(2e-3)
    o, x0, J0 = _g2p_affine(alpha * np.eye(3), np.zeros(3), dt=dt, J0=0.9)
    np.testing.assert_allclose(o.array(3), J0 * (1.0 + 3.0 * alpha * dt), rtol=1e-13)
    np.testing.assert_allclose(o.array(1), alpha * x0, atol=1e-12)


def _p2g_single(xp, vp, Cp, Jp, prm, n_grid=32):
    L, lv = W.c3_layout(n_grid)
    f = L.fields
    o = oracle.Oracle(L.desc())
    o.set_exact(True)
    o.register_array(np.asarray(xp, np.float32).reshape(3, 1))
    o.register_array(np.asarray(vp, np.float32).reshape(3, 1))
    o.register_array(np.asarray(Cp, np.float32).reshape(9, 1))
    o.register_array(np.asarray([Jp], np.float32).reshape(1, 1))
    o.range_for_task("P2G", 1, [f["vx"], f["vy"], f["vz"], f["m"]], [0, 1, 2, 3],
                     [prm["dt"], prm["inv_dx"], prm["p_mass"], prm["p_vol"], prm["E"]], 0b1111)
    return o, L


def test_p2g_first_moment_is_affine_times_inertia():
    n_grid = 32
    prm = {k: _f32(v) for k, v in W.mpm_params(n_grid, dt=1e-3, E=400.0).items()}
    dx = 1.0 / n_grid
    rng = np.random.default_rng(17)
    idx = np.stack(np.meshgrid(*(np.arange(n_grid),) * 3, indexing="ij"), 0).astype(np.float64) * dx
    for trial in range(6):
        xp = rng.uniform(0.3, 0.7, size=3).astype(np.float32)
        vp = rng.uniform(-1, 1, size=3).astype(np.float32)
        Cp = rng.uniform(-3, 3, size=9).astype(np.float32)
        Jp = np.float32(rng.uniform(0.7, 1.3))
        o, L = _p2g_single(xp, vp, Cp, Jp, prm)
        f = L.fields
        x64 = xp.astype(np.float64)
        m = o.field(f["m"])
        p = np.stack([o.field(f[n]) for n in ("vx", "vy", "vz")], 0)
        np.testing.assert_allclose(m.sum(), prm["p_mass"], rtol=1e-13)
        np.testing.assert_allclose(p.reshape(3, -1).sum(1), prm["p_mass"] * vp.astype(np.float64), rtol=1e-12,
                                   atol=1e-20)
        # inertia D_p = dx^2/4 I (from the mass distribution)
        dpos = idx - x64[:, None, None, None]
        D = np.einsum("xyz,axyz,bxyz->ab", m, dpos, dpos) / prm["p_mass"]
        np.testing.assert_allclose(D, dx * dx / 4 * np.eye(3), rtol=0, atol=1e-15)
        stress = -prm["dt"] * 4.0 * prm["E"] * prm["p_vol"] * (float(Jp) - 1.0) / (dx * dx)
        aff = prm["p_mass"] * Cp.astype(np.float64).reshape(3, 3) + stress * np.eye(3)
        first = np.einsum("rxyz,dxyz->rd", p, dpos)
        np.testing.assert_allclose(first, aff * dx * dx / 4, rtol=1e-10, atol=1e-22)
        # the stress alone is visible: with C = 0 the moment is diagonal and equals stress * dx^2/4
        assert abs(stress) > 1e-3 * abs(aff).max() or abs(float(Jp) - 1.0) < 1e-3


def test_grid_op_gravity_and_walls():
    # GRID_OP (mpm3d grid update, reading R28): u = p/m - dt g e_y, then a
    # component pointing into a wall within `bound` cells is zeroed.
    n_grid = 32
    prm = {k: _f32(v) for k, v in W.mpm_params(n_grid, dt=1e-3).items()}
    L, lv = W.c3_layout(n_grid)
    f = L.fields
    o = oracle.Oracle(L.desc())
    o.set_exact(True)
    nodes = np.array([[1, 10, 10], [30, 10, 10], [10, 1, 10], [10, 10, 30], [10, 10, 10], [1, 1, 1]], np.int32)
    o.activate(f["m"], nodes)
    m = np.zeros((n_grid,) * 3)
    p = np.zeros((3,) + (n_grid,) * 3)
    mom = {(1, 10, 10): (-2.0, 1.0, 0.5), (30, 10, 10): (2.0, -1.0, 0.5), (10, 1, 10): (0.5, -3.0, 0.5),
           (10, 10, 30): (0.5, 1.0, -0.5), (10, 10, 10): (-1.0, -1.0, -1.0), (1, 1, 1): (1.0, 1.0, 1.0)}
    for c, q in mom.items():
        m[c] = 2.0
        for r in range(3):
            p[(r,) + c] = q[r]
    o.load_field(f["m"], m)
    for r, n in enumerate(("vx", "vy", "vz")):
        o.load_field(f[n], p[r])
    o.call(W.struct_for("GRID_OP", lv[-1], [f["vx"], f["vy"], f["vz"], f["m"]],
                        [prm["dt"], prm["gravity"], prm["bound"], prm["n_grid"]]))
    g = prm["dt"] * prm["gravity"]
    want = {(1, 10, 10): (0.0, 0.5 - g, 0.25),          # x < bound moving -x: zeroed
            (30, 10, 10): (0.0, -0.5 - g, 0.25),        # x > n - bound moving +x: zeroed
            (10, 1, 10): (0.25, 0.0, 0.25),             # y < bound moving -y (after gravity): zeroed
            (10, 10, 30): (0.25, 0.5 - g, -0.25),       # z > n - bound moving -z: kept
            (10, 10, 10): (-0.5, -0.5 - g, -0.5),       # interior: p/m - dt g e_y
            (1, 1, 1): (0.5, 0.5 - g, 0.5)}             # at the walls but moving away: kept
    for c, u in want.items():
        got = [o.field(f[n])[c] for n in ("vx", "vy", "vz")]
        np.testing.assert_allclose(got, u, rtol=1e-14, atol=1e-15, err_msg=str(c))


def test_bin_order_program_equals_in_place_on_the_oracle():
    """The oracle's PERMUTE / bin-order G2P take the identity permutation: the
    two-state-set program equals the in-place one value for value."""
    a = W.c3_program(n_grid=32, n_particles=1500, steps=3, seed=2, v_scale=1.0, J_jitter=0.02, lo=0.2, hi=0.7)
    b = W.c3_program(n_grid=32, n_particles=1500, steps=3, seed=2, v_scale=1.0, J_jitter=0.02, lo=0.2, hi=0.7,
                     bin_order=True)
    oa, ob = oracle.run_program(a), oracle.run_program(b)
    for i in range(4):
        np.testing.assert_array_equal(ob.array(b["result_set"][i]), oa.array(i))
    np.testing.assert_array_equal(ob.array(b["result_set"][4])[0], np.arange(1500))
