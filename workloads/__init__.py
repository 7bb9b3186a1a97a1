"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module is the ONLY code both sides see.  It holds no arithmetic of the
method: it builds layout descriptors (the SNode tree as plain integer rows),
seeded coordinate / particle buffers, and *programs* -- ordered lists of user
calls (activate / struct_for / range_for / serial / clear / listgen / flush)
written as plain dicts.  Each side replays a program through its own API:
``paper_2012_08141_b200.sg.run_program`` (C-ABI) and ``oracle.run_program``
(CPU oracle).  Op names are strings; each side maps them to its own ids.

Config recipes follow SURVEY.md s8.0 and DESIGN.md "Input recipe".
"""
from __future__ import annotations

import numpy as np

# ----------------------------------------------------------------------------
# Layout descriptor rows: [kind, parent, ndim, e0, e1, e2, dtype]
# (Fig. 2 caption `ti.root.pointer(ti.i, 4).dense(ti.i, 2).place(x)`;
#  PAPER.md:187 "Commonly used SNodes include dense, bitmasked, pointer")
# ----------------------------------------------------------------------------
ROOT, DENSE, BITMASKED, POINTER, PLACE = 0, 1, 2, 3, 4
F32, I32 = 0, 1
KIND = {"root": ROOT, "dense": DENSE, "bitmasked": BITMASKED, "pointer": POINTER}
DTYPE = {"f32": F32, "i32": I32}


class Layout:
    """Builds the descriptor table.  Field ids are the order of place rows."""

    def __init__(self):
        self.rows = [[ROOT, -1, 0, 1, 1, 1, 0]]
        self.fields = {}      # name -> field id
        self.field_snode = {}  # name -> place snode id
        self.leaf = {}        # name -> leaf level snode id (parent of place)
        self.field_dtype = {}
        self.field_ndim = {}

    def chain(self, levels, fields, ndim=None):
        """levels: [(kind, extents tuple)], root-to-leaf; fields: [(name, dtype)].
        Returns the list of level snode ids."""
        parent = 0
        ids = []
        for kind, ext in levels:
            ext = tuple(int(e) for e in ext)
            nd = len(ext) if ndim is None else ndim
            e = list(ext) + [1] * (3 - len(ext))
            self.rows.append([KIND[kind], parent, nd, e[0], e[1], e[2], 0])
            parent = len(self.rows) - 1
            ids.append(parent)
        nd = self.rows[parent][2] if ids else 0
        for name, dt in fields:
            self.rows.append([PLACE, parent, nd, 1, 1, 1, DTYPE[dt]])
            self.fields[name] = len(self.fields)
            self.field_snode[name] = len(self.rows) - 1
            self.leaf[name] = parent
            self.field_dtype[name] = dt
            self.field_ndim[name] = nd
        return ids

    def scalar(self, name, dtype="f32"):
        return self.chain([], [(name, dtype)])

    def desc(self):
        return np.asarray(self.rows, dtype=np.int32)

    def shape(self, name):
        """Full-resolution bounding shape of a field (product of ancestor extents)."""
        s = [1, 1, 1]
        node = self.rows[self.field_snode[name]][1]
        while node > 0:
            r = self.rows[node]
            for a in range(3):
                s[a] *= r[3 + a]
            node = r[1]
        return tuple(s[: self.field_ndim[name]])


def program(layout, calls, arrays=None, name=""):
    return {"name": name, "layout": layout, "desc": layout.desc(),
            "arrays": arrays or {}, "calls": calls}


# ---- call constructors (plain data) -----------------------------------------
def activate(field, coords):
    return {"call": "activate", "field": field, "coords": np.ascontiguousarray(coords, dtype=np.int32)}


def struct_for(op, snode, fields, params=(), activating=()):
    return {"call": "struct_for", "op": op, "snode": int(snode), "fields": list(fields),
            "params": [float(p) for p in params], "activating": list(activating)}


def range_for(op, n, fields=(), arrays=(), params=(), activating=()):
    return {"call": "range_for", "op": op, "n": int(n), "fields": list(fields), "arrays": list(arrays),
            "params": [float(p) for p in params], "activating": list(activating)}


def serial(op, fields, params=()):
    return {"call": "serial", "op": op, "fields": list(fields), "params": [float(p) for p in params]}


def clear_values(field):
    return {"call": "clear", "mode": "values", "target": field}


def deactivate(snode):
    return {"call": "clear", "mode": "deactivate", "target": int(snode)}


def listgen(snode):
    return {"call": "listgen", "snode": int(snode)}


def flush(passes="all", observed=None):
    return {"call": "flush", "passes": passes, "observed": observed}


# ----------------------------------------------------------------------------
# C1: 2D 64x64, pointer(16x16) -> bitmasked(4x4) leaf.  Disk r=24 (1,804 cells).
# ----------------------------------------------------------------------------
def c1_layout(dtype="f32"):
    L = Layout()
    lv = L.chain([("pointer", (16, 16)), ("bitmasked", (4, 4))], [("x", dtype), ("y", dtype)])
    L.scalar("s", dtype)
    return L, lv


def c1_disk_coords(n=64, r=24.0):
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    m = (i + 0.5 - n / 2) ** 2 + (j + 0.5 - n / 2) ** 2 < r * r
    return np.stack([i[m], j[m]], axis=1).astype(np.int32)


def c1_random_coords(seed=0, p_ptr=0.5, p_bit=0.5):
    rng = np.random.default_rng(seed)
    ptr = rng.random((16, 16)) < p_ptr
    bits = rng.random((64, 64)) < p_bit
    i, j = np.meshgrid(np.arange(64), np.arange(64), indexing="ij")
    m = bits & ptr[i // 4, j // 4]
    return np.stack([i[m], j[m]], axis=1).astype(np.int32)


def c1_step_calls(L, lv, coords):
    """Reading 19: activate, fill x=1, stencil y<-x, clear s, reduce s+=y."""
    f = L.fields
    leaf = lv[-1]
    return [activate(f["x"], coords),
            struct_for("FILL", leaf, [f["x"]], [1.0]),
            struct_for("STENCIL", leaf, [f["y"], f["x"]]),
            serial("CLEAR_SCALAR", [f["s"]]),
            struct_for("REDUCE_SUM", leaf, [f["s"], f["y"]])]


def c1_program(steps=1, disk=True, dtype="f32", passes="all", seed=0):
    L, lv = c1_layout(dtype)
    coords = c1_disk_coords() if disk else c1_random_coords(seed)
    calls = []
    for _ in range(steps):
        calls += c1_step_calls(L, lv, coords)
        calls.append(flush(passes))
    return program(L, calls, name="C1")


# ----------------------------------------------------------------------------
# C2: 3D 256^3, pointer(8^3)[32^3] -> bitmasked(4^3)[8^3] -> dense(8^3).
# Block-ball: leaf blocks whose nearest point lies within R voxels of the centre.
# ----------------------------------------------------------------------------
def c2_layout(ptr=8, bm=4, dn=8):
    L = Layout()
    lv = L.chain([("pointer", (ptr,) * 3), ("bitmasked", (bm,) * 3), ("dense", (dn,) * 3)],
                 [("x0", "f32"), ("x1", "f32"), ("b", "f32")])
    L.scalar("s", "f32")
    return L, lv


def block_ball_coords(n_blocks_axis, block, radius):
    """One cell coordinate (the block origin) per active leaf block."""
    b = np.arange(n_blocks_axis)
    bx, by, bz = np.meshgrid(b, b, b, indexing="ij")
    c = n_blocks_axis * block / 2.0
    near = lambda q: np.clip(c, q * block, q * block + block)
    d2 = (near(bx) - c) ** 2 + (near(by) - c) ** 2 + (near(bz) - c) ** 2
    m = d2 < radius * radius
    return (np.stack([bx[m], by[m], bz[m]], axis=1) * block).astype(np.int32)


def c2_solve_calls(L, lv, coords, iters=50, reduce_result=True):
    f = L.fields
    leaf = lv[-1]
    calls = [activate(f["b"], coords),
             struct_for("FILL", leaf, [f["b"]], [1.0]),
             struct_for("FILL", leaf, [f["x0"]], [0.0])]
    src, dst = f["x0"], f["x1"]
    for _ in range(iters):
        calls.append(struct_for("JACOBI", leaf, [dst, src, f["b"]]))
        src, dst = dst, src
    if reduce_result:
        calls += [serial("CLEAR_SCALAR", [f["s"]]),
                  struct_for("REDUCE_SUM", leaf, [f["s"], src])]
    return calls, src


def c2_program(iters=50, radius=68.0, ptr=8, passes="all", solves=1):
    L, lv = c2_layout(ptr=ptr)
    nb = ptr * 4
    coords = block_ball_coords(nb, 8, radius * ptr / 8)
    calls = []
    for _ in range(solves):
        c, _ = c2_solve_calls(L, lv, coords, iters)
        calls += c + [flush(passes)]
    return program(L, calls, name="C2")


def c2_small_program(iters=6, passes="all"):
    """Oracle-sized C2 variant: 64^3 bound (pointer 2^3), ball R=20 -> spans several
    containers, ragged block set."""
    L, lv = c2_layout(ptr=2)
    coords = block_ball_coords(8, 8, 20.0)
    c, _ = c2_solve_calls(L, lv, coords, iters)
    return program(L, c + [flush(passes)], name="C2-small")


# ----------------------------------------------------------------------------
# C3: 3D sparse MLS-MPM (mpm3d-like), 128^3 grid, 1M particles.
# pointer(n/16)^3 [16^3 cells each] -> bitmasked(4^3) [4^3] -> dense(4^3).
# ----------------------------------------------------------------------------
def c3_layout(n_grid=128):
    L = Layout()
    lv = L.chain([("pointer", (n_grid // 16,) * 3), ("bitmasked", (4,) * 3), ("dense", (4,) * 3)],
                 [("vx", "f32"), ("vy", "f32"), ("vz", "f32"), ("m", "f32")])
    return L, lv


def mpm_params(n_grid=128, dt=None, E=400.0, gravity=9.8, bound=3):
    """mpm3d-style constants (reading R28).  dt defaults to 1e-4 up to a 128^3
    grid and shrinks with dx above it (reading R42): the sound speed
    sqrt(E / rho) = 20 makes the CFL number 20 dt / dx, 0.26 at 128^3 with
    1e-4 but 1.02 at 512^3 -- C5 blew up after ~15 steps (particles left the
    domain into the per-particle overflow path, the step went 3 -> 290 ms)."""
    if dt is None:
        dt = 1e-4 * min(1.0, 128.0 / n_grid)
    dx = 1.0 / n_grid
    p_vol = (dx * 0.5) ** 3
    p_rho = 1.0
    return {"dt": dt, "inv_dx": float(n_grid), "p_mass": p_vol * p_rho, "p_vol": p_vol, "E": E,
            "gravity": gravity, "bound": float(bound), "n_grid": float(n_grid)}


def mpm_particles(n, lo=0.15, hi=0.55, seed=0, v_scale=0.0, J_jitter=0.0):
    """SoA float32 arrays: x (3,n), v (3,n), C (9,n), J (1,n)."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(lo, hi, size=(3, n)).astype(np.float32)
    v = (rng.uniform(-1, 1, size=(3, n)) * v_scale).astype(np.float32)
    C = np.zeros((9, n), dtype=np.float32)
    J = (1.0 + rng.uniform(-1, 1, size=(1, n)) * J_jitter).astype(np.float32)
    return {"x": x, "v": v, "C": C, "J": J}


def c3_step_calls(L, lv, n, prm, src=(0, 1, 2, 3), dst=None, ids=None):
    """One MPM substep.  dst=None: G2P in place on the state arrays `src`.
    dst given: G2P out of place from `src` into `dst` in bin order (a
    permutation of the particles, include/sg.h), and PERMUTE moves the id array
    ids[0] -> ids[1] the same way."""
    f = L.fields
    grid_f = [f["vx"], f["vy"], f["vz"], f["m"]]
    src = list(src)
    calls = [deactivate(lv[0]),
             range_for("P2G", n, grid_f, src,
                       [prm["dt"], prm["inv_dx"], prm["p_mass"], prm["p_vol"], prm["E"]], [True] * 4),
             struct_for("GRID_OP", lv[-1], grid_f, [prm["dt"], prm["gravity"], prm["bound"], prm["n_grid"]])]
    if dst is None:
        calls.append(range_for("G2P", n, grid_f, src, [prm["dt"], prm["inv_dx"]]))
    else:
        calls.append(range_for("G2P", n, grid_f, src + list(dst), [prm["dt"], prm["inv_dx"], 1.0]))
        calls.append(range_for("PERMUTE", n, [f["m"]], [src[0], ids[0], ids[1]], [0.0, prm["inv_dx"]]))
    return calls


def c3_program(n_grid=128, n_particles=1_000_000, steps=1, flush_every=1, seed=0, v_scale=0.0, J_jitter=0.0,
               lo=0.15, hi=0.55, passes="all", bin_order=False, **prm_kw):
    """bin_order: two particle state sets A (arrays 0-3, ids 4) and B (5-8,
    ids 9); step s runs G2P out of place A -> B (s even) or B -> A (s odd) in
    bin order, ids permuted along (reading R38)."""
    L, lv = c3_layout(n_grid)
    prm = mpm_params(n_grid, **prm_kw)
    arrays = mpm_particles(n_particles, lo, hi, seed, v_scale, J_jitter)
    if bin_order:
        arrays["id"] = np.arange(n_particles, dtype=np.float32)[None]
        for k in ("x", "v", "C", "J", "id"):
            arrays[k + "B"] = np.zeros_like(arrays[k])
    calls = []
    for s in range(steps):
        if bin_order:
            a, b = ((0, 1, 2, 3), (5, 6, 7, 8)) if s % 2 == 0 else ((5, 6, 7, 8), (0, 1, 2, 3))
            ids = (4, 9) if s % 2 == 0 else (9, 4)
            calls += c3_step_calls(L, lv, n_particles, prm, a, b, ids)
        else:
            calls += c3_step_calls(L, lv, n_particles, prm)
        if (s + 1) % flush_every == 0 or s == steps - 1:
            calls.append(flush(passes))
    prog = program(L, calls, arrays=arrays, name="C3")
    prog["bin_order"] = bin_order
    prog["result_set"] = None if not bin_order else ((0, 1, 2, 3, 4) if steps % 2 == 0 else (5, 6, 7, 8, 9))
    return prog


# ----------------------------------------------------------------------------
# C4: differentiable MPM (diffmpm-like; "global
# fields as checkpoints", PAPER.md:375-377 gradient clears).  Forward T
# substeps keep every particle state (the checkpoints); the backward pass
# recomputes each substep's grid (P2G) and runs the hand-written adjoints
# G2P_ADJ (grid-op adjoint folded in) and P2G_ADJ, scattering grid adjoints
# into a second tree of the same shape (activating).
# ----------------------------------------------------------------------------
def c4_layout(n_grid=64):
    L = Layout()
    lv = L.chain([("pointer", (n_grid // 16,) * 3), ("bitmasked", (4,) * 3), ("dense", (4,) * 3)],
                 [("px", "f32"), ("py", "f32"), ("pz", "f32"), ("m", "f32")])
    lg = L.chain([("pointer", (n_grid // 16,) * 3), ("bitmasked", (4,) * 3), ("dense", (4,) * 3)],
                 [("gpx", "f32"), ("gpy", "f32"), ("gpz", "f32"), ("gm", "f32")])
    L.scalar("loss")
    return L, lv, lg


def c4_particles(n, n_grid=64, side=23, center=(0.5, 0.4, 0.5), seed=0, v_scale=0.5, C_scale=1.0, J_jitter=0.02):
    """A cube of `side` cells (about 8 particles per cell at n = 100K) with a
    random initial velocity, affine C and J, so every adjoint term is nonzero."""
    rng = np.random.default_rng(seed)
    half = side / (2.0 * n_grid)
    c = np.asarray(center, dtype=np.float64)[:, None]
    x = (c - half + rng.random((3, n)) * 2 * half).astype(np.float32)
    v = (rng.uniform(-1, 1, (3, n)) * v_scale).astype(np.float32)
    C = (rng.uniform(-1, 1, (9, n)) * C_scale).astype(np.float32)
    J = (1.0 + rng.uniform(-1, 1, (1, n)) * J_jitter).astype(np.float32)
    return {"x": x, "v": v, "C": C, "J": J}


def c4_arrays(n, T, n_grid=64, **kw):
    """Array table: state s = ids 4s..4s+3 (x, v, C, J) for s = 0..T, then two
    adjoint buffers A = 4(T+1)+0..3 and B = 4(T+1)+4..7 (same shapes)."""
    p0 = c4_particles(n, n_grid, **kw)
    arrays = {}
    for s in range(T + 1):
        for k in ("x", "v", "C", "J"):
            arrays[f"{k}{s}"] = p0[k] if s == 0 else np.zeros_like(p0[k])
    for b in ("A", "B"):
        for k in ("x", "v", "C", "J"):
            arrays[f"adj{b}_{k}"] = np.zeros_like(p0[k])
    return arrays


def c4_forward_calls(L, lv, lg, n, T, prm, comp=0, grad_clears=True):
    f = L.fields
    grid_f = [f["px"], f["py"], f["pz"], f["m"]]
    grad_f = [f["gpx"], f["gpy"], f["gpz"], f["gm"]]
    calls = []
    for s in range(T):
        st, nx = [4 * s + k for k in range(4)], [4 * (s + 1) + k for k in range(4)]
        calls.append(deactivate(lv[0]))
        if grad_clears:   # diffmpm's clear_grid also zeroes the grads: dead stores
            calls += [clear_values(g) for g in grad_f]
        calls.append(range_for("P2G", n, grid_f, st,
                               [prm["dt"], prm["inv_dx"], prm["p_mass"], prm["p_vol"], prm["E"]], [True] * 4))
        calls.append(struct_for("GRID_OP", lv[-1], grid_f, [prm["dt"], prm["gravity"], prm["bound"], prm["n_grid"]]))
        calls.append(range_for("G2P", n, grid_f, st + nx, [prm["dt"], prm["inv_dx"]]))
    calls.append(serial("CLEAR_SCALAR", [f["loss"]]))
    calls.append(range_for("LOSS_MEAN", n, [f["loss"]], [4 * T], [comp, 1.0 / n]))
    return calls


def c4_backward_calls(L, lv, lg, n, T, prm, comp=0):
    f = L.fields
    grid_f = [f["px"], f["py"], f["pz"], f["m"]]
    grad_f = [f["gpx"], f["gpy"], f["gpz"], f["gm"]]
    A = [4 * (T + 1) + k for k in range(4)]
    B = [4 * (T + 1) + 4 + k for k in range(4)]
    calls = [range_for("ADJ_INIT", n, [], A, [comp, 1.0 / n])]
    for j, s in enumerate(reversed(range(T))):
        adj1, adj0 = (A, B) if j % 2 == 0 else (B, A)
        st = [4 * s + k for k in range(4)]
        calls.append(deactivate(lv[0]))
        calls.append(range_for("P2G", n, grid_f, st,
                               [prm["dt"], prm["inv_dx"], prm["p_mass"], prm["p_vol"], prm["E"]], [True] * 4))
        calls.append(deactivate(lg[0]))
        calls.append(range_for("G2P_ADJ", n, grid_f + grad_f, [st[0], st[3]] + adj1 + [adj0[0], adj0[3]],
                               [prm["dt"], prm["inv_dx"], prm["gravity"], prm["bound"], prm["n_grid"]],
                               [False] * 4 + [True] * 4))
        calls.append(range_for("P2G_ADJ", n, grad_f, st + adj0,
                               [prm["dt"], prm["inv_dx"], prm["p_mass"], prm["p_vol"], prm["E"]]))
    return calls


def c4_result_arrays(T):
    """Array ids holding d loss / d (x0, v0, C0, J0) after the backward pass."""
    A = [4 * (T + 1) + k for k in range(4)]
    B = [4 * (T + 1) + 4 + k for k in range(4)]
    return B if T % 2 == 1 else A


def c4_program(n_grid=64, n_particles=100_000, T=64, seed=0, passes="all", comp=0, grad_clears=True,
               observed=None, dt=2e-4, **kw):
    L, lv, lg = c4_layout(n_grid)
    prm = mpm_params(n_grid, dt=dt)
    arrays = c4_arrays(n_particles, T, n_grid, seed=seed, **kw)
    calls = c4_forward_calls(L, lv, lg, n_particles, T, prm, comp, grad_clears)
    calls += c4_backward_calls(L, lv, lg, n_particles, T, prm, comp)
    calls.append(flush(passes, observed))
    prog = program(L, calls, arrays=arrays, name="C4")
    prog["params"] = prm
    prog["T"] = T
    prog["result_arrays"] = c4_result_arrays(T)
    return prog


# ----------------------------------------------------------------------------
# MG: multigrid V-cycle Poisson solver in the style of the paper's
# MGPCG benchmark (512^2 domain, sparsely populated region,
# four levels, each a two-level sparse grid; hu2019taichi's MGPCG): red-black
# Gauss-Seidel smoothing, residual restriction with activate-on-write on the
# coarse level (demoted after the first cycle), prolongation.
# ----------------------------------------------------------------------------
MG_BOTTOM = 32   # red-black sweeps on the coarsest level (reading R36)


def mg_layout(n=512, levels=4, block=16, cg=False):
    """Level l is a two-level sparse grid pointer(n/block) -> dense(block >> l)
    ("for each level we use a two-level sparse grid"): a coarse
    block is exactly the image of one fine block, so the coarse active region
    that restriction activates (block granularity) is exactly the image of the
    fine region (reading R36)."""
    L = Layout()
    lv = []
    for l in range(levels):
        nl = n >> l
        b = max(1, block >> l)
        fields = [(f"z{l}", "f32"), (f"r{l}", "f32")]
        if cg and l == 0:
            fields += [("x", "f32"), ("p", "f32"), ("Ap", "f32")]
        ids = L.chain([("pointer", (nl // b,) * 2), ("dense", (b,) * 2)], fields)
        lv.append(ids)
    L.scalar("res")
    if cg:
        for name in ("zTr_old", "zTr_new", "pAp", "rTr"):
            L.scalar(name)
    return L, lv


def mg_region(n=512, block=16, radius_frac=0.3125, center=(0.5, 0.5)):
    """Block origins (pointer-cell coords) of the finest level's active region:
    blocks whose nearest point lies inside a disk of radius radius_frac * n."""
    nb = n // block
    cx, cy = center[0] * n, center[1] * n
    R = radius_frac * n
    out = []
    for i in range(nb):
        for j in range(nb):
            x0, y0 = i * block, j * block
            dx = max(x0 - cx, 0.0, cx - (x0 + block))
            dy = max(y0 - cy, 0.0, cy - (y0 + block))
            if dx * dx + dy * dy < R * R:
                out.append((x0, y0))
    return np.asarray(out, dtype=np.int32)


def mg_vcycle_calls(L, lv, levels=4, nu=2, bottom=MG_BOTTOM, weight=1.0):
    f = L.fields
    z = [f[f"z{l}"] for l in range(levels)]
    r = [f[f"r{l}"] for l in range(levels)]
    leaf = [ids[-1] for ids in lv]
    calls = []

    def smooth(l, order=(0, 1)):
        return [struct_for("SMOOTH_RB", leaf[l], [z[l], r[l]], [p]) for p in order]

    for l in range(levels - 1):
        for _ in range(nu):
            calls += smooth(l)
        calls += [clear_values(r[l + 1]), clear_values(z[l + 1])]
        calls.append(struct_for("RESTRICT", leaf[l], [r[l + 1], r[l], z[l]], [weight], [True]))
    # bottom: (red, black) sweeps then (black, red) sweeps -- a symmetric smoother,
    # so the V-cycle is a symmetric preconditioner for MGPCG
    for _ in range(bottom // 2):
        calls += smooth(levels - 1)
    for _ in range(bottom - bottom // 2):
        calls += smooth(levels - 1, (1, 0))
    for l in reversed(range(levels - 1)):
        calls.append(struct_for("PROLONG", leaf[l], [z[l], z[l + 1]]))
        for _ in range(nu):
            calls += smooth(l, (1, 0))
    return calls


def mg_weight(dim=2):
    """Restriction weight 4 / 2^dim (= 1 in 2-D): the re-discretized coarse
    operator (the h^2 scaling of the coarse grid, 4, times the average over the
    2^dim children).  Reading R36."""
    return 4.0 / (1 << dim)


def mg_solve_calls(L, lv, coords, cycles=10, levels=4, nu=2, bottom=MG_BOTTOM, dim=2, with_residual=True):
    """Activate the finest level, r0 = 1 (the right-hand side), z0 = 0, then
    `cycles` V-cycles; finally res = ||r0 - A z0||^2."""
    f = L.fields
    calls = [activate(f["z0"], coords), struct_for("FILL", lv[0][-1], [f["r0"]], [1.0]),
             struct_for("FILL", lv[0][-1], [f["z0"]], [0.0])]
    for _ in range(cycles):
        calls += mg_vcycle_calls(L, lv, levels, nu, bottom, weight=mg_weight(dim))
    if with_residual:
        calls += [serial("CLEAR_SCALAR", [f["res"]]),
                  struct_for("RESID_NORM2", lv[0][-1], [f["res"], f["r0"], f["z0"]])]
    return calls


def mgpcg_calls(L, lv, coords, iters=10, levels=4, nu=2, bottom=MG_BOTTOM, dim=2):
    """Conjugate gradients preconditioned by one V-cycle (MGPCG, PAPER.md:438-441
    after hu2019taichi): solve A x = b (b = 1 on the active region).  The
    V-cycle works on (z0, r0), so r0 doubles as the CG residual.  STENCIL gives
    -A p, so pAp = -<p, STENCIL p> and r -= alpha A p becomes r += alpha (-A p)."""
    f = L.fields
    leaf0 = lv[0][-1]
    w = mg_weight(dim)

    def precondition():
        return [struct_for("FILL", leaf0, [f["z0"]], [0.0])] + mg_vcycle_calls(L, lv, levels, nu, bottom, weight=w)

    calls = [activate(f["z0"], coords), struct_for("FILL", leaf0, [f["r0"]], [1.0]),
             struct_for("FILL", leaf0, [f["x"]], [0.0])]
    calls += precondition()
    calls += [struct_for("ADD_CONST", leaf0, [f["p"], f["z0"]], [0.0]),
              serial("CLEAR_SCALAR", [f["zTr_old"]]), struct_for("DOT", leaf0, [f["zTr_old"], f["z0"], f["r0"]], [1.0])]
    for _ in range(iters):
        calls += [struct_for("STENCIL", leaf0, [f["Ap"], f["p"]]),
                  serial("CLEAR_SCALAR", [f["pAp"]]), struct_for("DOT", leaf0, [f["pAp"], f["p"], f["Ap"]], [-1.0]),
                  struct_for("AXPY_RATIO", leaf0, [f["x"], f["p"], f["zTr_old"], f["pAp"]], [1.0]),
                  struct_for("AXPY_RATIO", leaf0, [f["r0"], f["Ap"], f["zTr_old"], f["pAp"]], [1.0]),
                  serial("CLEAR_SCALAR", [f["rTr"]]), struct_for("DOT", leaf0, [f["rTr"], f["r0"], f["r0"]], [1.0])]
        calls += precondition()
        calls += [serial("CLEAR_SCALAR", [f["zTr_new"]]),
                  struct_for("DOT", leaf0, [f["zTr_new"], f["z0"], f["r0"]], [1.0]),
                  struct_for("XPAY_RATIO", leaf0, [f["p"], f["z0"], f["zTr_new"], f["zTr_old"]]),
                  serial("COPY_SCALAR", [f["zTr_old"], f["zTr_new"]])]
    return calls


def mgpcg_program(n=512, levels=4, block=16, iters=10, nu=2, bottom=MG_BOTTOM, radius_frac=0.3125, passes="all"):
    L, lv = mg_layout(n, levels, block, cg=True)
    coords = mg_region(n, block, radius_frac)
    calls = mgpcg_calls(L, lv, coords, iters, levels, nu, bottom)
    calls.append(flush(passes))
    prog = program(L, calls, name="MGPCG")
    prog["levels"] = lv
    return prog


def mg_program(n=512, levels=4, block=16, cycles=10, nu=2, bottom=MG_BOTTOM, radius_frac=0.3125, passes="all"):
    L, lv = mg_layout(n, levels, block)
    coords = mg_region(n, block, radius_frac)
    calls = mg_solve_calls(L, lv, coords, cycles, levels, nu, bottom)
    calls.append(flush(passes))
    prog = program(L, calls, name="MG")
    prog["levels"] = lv
    return prog


# ----------------------------------------------------------------------------
# C5: large sparse MPM, 512^3 bound, x-slab sharded.
# pointer(P^3) [n/P cells each] -> bitmasked((n/P/4)^3) -> dense(4^3).
# ----------------------------------------------------------------------------
def c5_layout(n_grid=512, ptr_cells=16):
    L = Layout()
    bm = n_grid // ptr_cells // 4
    lv = L.chain([("pointer", (ptr_cells,) * 3), ("bitmasked", (bm,) * 3), ("dense", (4,) * 3)],
                 [("vx", "f32"), ("vy", "f32"), ("vz", "f32"), ("m", "f32")])
    return L, lv


def c5_particles(n, n_grid=512, length=460, width=66, seed=0, shear=2.0):
    """An x-spanning bar of length x width x width cells, uniform, with an x-velocity
    shear v_x = shear * (y - y_c) / width so particles cross slab faces."""
    rng = np.random.default_rng(seed)
    dx = 1.0 / n_grid
    c = n_grid / 2.0
    lo = np.array([c - length / 2.0, c - width / 2.0, c - width / 2.0]) * dx
    ext = np.array([length, width, width]) * dx
    x = (lo[:, None] + rng.random((3, n)) * ext[:, None]).astype(np.float32)
    v = np.zeros((3, n), dtype=np.float32)
    v[0] = (shear * (x[1] - 0.5) / (width * dx)).astype(np.float32)
    return {"x": x, "v": v, "C": np.zeros((9, n), dtype=np.float32), "J": np.ones((1, n), dtype=np.float32)}


def c5_slab_counts(n, n_grid=512, ptr_cells=16, length=460):
    """Particles per pointer x-slab of the bar: proportional to the slab's
    overlap with the bar, largest remainders first (sums to n)."""
    dx_slab = n_grid / ptr_cells
    lo, hi = n_grid / 2.0 - length / 2.0, n_grid / 2.0 + length / 2.0
    ov = np.array([max(0.0, min(hi, (j + 1) * dx_slab) - max(lo, j * dx_slab)) for j in range(ptr_cells)])
    exact = n * ov / ov.sum()
    cnt = np.floor(exact).astype(np.int64)
    rem = n - cnt.sum()
    cnt[np.argsort(-(exact - cnt), kind="stable")[:rem]] += 1
    return cnt


def c5_slab_particles(n, j, n_grid=512, ptr_cells=16, length=460, width=66, seed=0, shear=2.0):
    """The particles of pointer x-slab j of the C5 bar (uniform in the slab's
    part of the bar, x-velocity shear), generated from seed (seed, j) alone:
    any rank can build its own slabs and every world size sees the same
    particle set.  ids are global (prefix of the slab counts)."""
    cnt = c5_slab_counts(n, n_grid, ptr_cells, length)
    rng = np.random.default_rng([seed, j])
    dx = 1.0 / n_grid
    c = n_grid / 2.0
    x0 = max(c - length / 2.0, j * n_grid / ptr_cells)
    x1 = min(c + length / 2.0, (j + 1) * n_grid / ptr_cells)
    k = int(cnt[j])
    x = np.empty((3, k), dtype=np.float32)
    x[0] = (x0 + rng.random(k) * (x1 - x0)) * dx
    x[1:] = ((c - width / 2.0) + rng.random((2, k)) * width) * dx
    # keep the cell inside the slab under f32 rounding (ownership by floor(x * n))
    top = np.float32((x1 * dx))
    x[0] = np.minimum(x[0], np.nextafter(top, np.float32(0)))
    v = np.zeros((3, k), dtype=np.float32)
    v[0] = (shear * (x[1] - 0.5) / (width * dx)).astype(np.float32)
    ids = (np.int64(cnt[:j].sum()) + np.arange(k)).astype(np.int32)[None]
    return {"x": x, "v": v, "C": np.zeros((9, k), dtype=np.float32), "J": np.ones((1, k), dtype=np.float32),
            "id": ids}


def c5_rank_particles(n, rank, world, n_grid=512, ptr_cells=16, **kw):
    """Rank `rank`'s particles under the x-slab partition (its pointer slabs)."""
    per = ptr_cells // world
    parts = [c5_slab_particles(n, j, n_grid, ptr_cells, **kw) for j in range(rank * per, (rank + 1) * per)]
    return {k: np.concatenate([p[k] for p in parts], axis=1) for k in parts[0]}


def c5_program(n_grid=512, ptr_cells=16, n_particles=16_000_000, steps=1, seed=0, **kw):
    """The unpartitioned C5 problem as a plain program (oracle / 1-GPU reference)."""
    L, lv = c5_layout(n_grid, ptr_cells)
    prm = mpm_params(n_grid)
    arrays = c5_particles(n_particles, n_grid, seed=seed, **kw)
    calls = []
    for _ in range(steps):
        calls += c3_step_calls(L, lv, n_particles, prm)
        calls.append(flush())
    return program(L, calls, arrays=arrays, name="C5")


# ----------------------------------------------------------------------------
# Random integer programs (SPEC.md:386/454 fuzzer idea: seeded layouts of
# depth <= 4, a handful of kernels, integer fields for exact comparison).
# ----------------------------------------------------------------------------
def fuzz_layout(rng):
    nd = int(rng.integers(1, 4))
    depth = int(rng.integers(1, 5))
    kinds = []
    for k in range(depth):
        last = k == depth - 1
        choices = ["dense", "bitmasked"] if last else ["dense", "bitmasked", "pointer"]
        kinds.append(choices[int(rng.integers(0, len(choices)))])
    # per-axis total resolution: <=64 (1D), <=16 (2D), <=8 (3D)
    max_log = {1: 6, 2: 4, 3: 3}[nd]
    logs = np.zeros((depth, nd), dtype=int)
    for a in range(nd):
        budget = int(rng.integers(1, max_log + 1))
        for _ in range(budget):
            logs[int(rng.integers(0, depth)), a] += 1
    if logs[-1].min() == 0:  # leaf extent >= 2 on every axis so DOWNSAMPLE has a coarse twin
        for a in range(nd):
            if logs[-1, a] == 0:
                logs[-1, a] = 1
    levels = [(kinds[k], tuple(int(2 ** logs[k, a]) for a in range(nd))) for k in range(depth)]
    coarse = levels[:-1] + [(levels[-1][0], tuple(e // 2 for e in levels[-1][1]))]
    L = Layout()
    main = L.chain(levels, [("a", "i32"), ("b", "i32"), ("c", "i32")])
    half = L.chain(coarse, [("h", "i32")])
    L.scalar("s", "i32")
    return L, main, half


def fuzz_program(seed, n_ops=None, passes="all"):
    rng = np.random.default_rng(seed)
    L, main, half = fuzz_layout(rng)
    f = L.fields
    shape = L.shape("a")
    nd = len(shape)
    leaf, hleaf = main[-1], half[-1]
    sparse_main = [s for s in main if L.rows[s][0] in (BITMASKED, POINTER)]
    calls = []

    def rand_cells(k):
        return np.stack([rng.integers(0, shape[a], size=k) for a in range(nd)], axis=1).astype(np.int32)

    calls.append(activate(f["a"], rand_cells(int(rng.integers(1, 6)))))
    n_ops = int(rng.integers(3, 9)) if n_ops is None else n_ops
    fl = ["a", "b", "c"]
    for _ in range(n_ops):
        r = int(rng.integers(0, 16))
        if r >= 14:  # repeat the previous struct-for (demotion / listgen-removal / fusion bait)
            prev = [c for c in calls if c["call"] == "struct_for"]
            if prev:
                calls.append(dict(prev[-1]))
                continue
            r = 1
        x, y, z = (fl[i] for i in rng.permutation(3))
        act = [bool(rng.integers(0, 2))]
        k = float(rng.integers(-3, 4))
        if r == 0:
            calls.append(activate(f[x], rand_cells(int(rng.integers(1, 4)))))
        elif r == 1:
            calls.append(struct_for("FILL", leaf, [f[x]], [k], act))
        elif r == 2:
            calls.append(struct_for("INC", leaf, [f[x]], [k], act))
        elif r == 3:
            calls.append(struct_for("ADD_CONST", leaf, [f[x], f[y]], [k], act))
        elif r == 4:
            calls.append(struct_for("AXPY", leaf, [f[x], f[y], f[z]], [k], act))
        elif r == 5:
            calls.append(struct_for("STENCIL", leaf, [f[x], f[y]], [], act))
        elif r == 6:
            calls.append(struct_for("JITTER", leaf, [f[x]], [], act))
        elif r == 7:
            calls.append(struct_for("DOWNSAMPLE", leaf, [f["h"], f[x]], [k, float(rng.integers(0, 3))], [True]))
        elif r == 8:
            calls += [serial("CLEAR_SCALAR", [f["s"]]), struct_for("REDUCE_SUM", leaf, [f["s"], f[x]])]
        elif r == 9:
            calls.append(clear_values(f[x]))
        elif r == 10 and sparse_main:
            calls.append(deactivate(sparse_main[int(rng.integers(0, len(sparse_main)))]))
        elif r == 11:
            calls.append(struct_for("INC", hleaf, [f["h"]], [k], act))
        elif r == 12:
            calls.append(flush(passes))
        else:
            calls.append(struct_for("FILL", leaf, [f[x]], [k], act))
    calls.append(flush(passes))
    return program(L, calls, name=f"fuzz{seed}")
