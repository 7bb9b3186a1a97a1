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
