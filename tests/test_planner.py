"""Host planner tests (-m "not gpu"): plan-only grids, no device.

T2 pins: the paper's printed task counts and facts (PAPER.md:316-323 6->3,
:487-505 microbenchmarks, :346/:361 demotion), adapted to our lowering
(SURVEY.md Appendix A).  T3 soundness on the CPU: the planner's schedule
(what survives, in which order, with which activating flags) is replayed on
the CPU oracle and must leave exactly the state of the eager oracle run, for
every pass subset, on the integer fuzz corpus.  (The GPU executes the same
schedule with fused kernels; tests/test_gpu_parity.py checks that.)
"""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W
from paper_2012_08141_b200 import sg


def plan_counts(prog, passes="all", faithful=False):
    g = sg.Grid(prog["desc"], plan_only=True, faithful=faithful)
    stats, plans = [], []
    sg.replay(g, prog, passes=passes, on_flush=lambda gr, st: (stats.append(st), plans.append(gr.last_plan())))
    return stats, plans


def types_of(plan):
    return [sg.TASK_TYPES[t] for t in plan[:, 1]]


# ---------------------------------------------------------------------------
# Paper-printed counts
# ---------------------------------------------------------------------------
def fig6_program(n_kernels=2):
    L = W.Layout()
    lv = L.chain([("pointer", (4,)), ("dense", (2,))], [("x", "i32")])
    calls = [W.activate(0, np.array([[1], [5]], dtype=np.int32)), W.flush()]
    calls += [W.struct_for("INC", lv[-1], [0], [1.0]) for _ in range(n_kernels)] + [W.flush()]
    return W.program(L, calls)


def test_fig6_three_tasks_per_kernel_and_6_to_3():
    # PAPER.md:316 "there are 3 tasks per such a small kernel"
    # "we reduce the number of generated tasks from 6 to 3".
    st, plans = plan_counts(fig6_program(1), passes=0, faithful=True)
    assert st[1]["tasks_lowered"] == 3
    st, plans = plan_counts(fig6_program(2), passes=0, faithful=True)
    assert st[1]["tasks_lowered"] == 6 and st[1]["launches"] == 6
    # Without DSE our clear-list version sits between the two listgens, so
    # nothing is removable (reading R3: the paper's 3 keeps a clear-list task)
    st, plans = plan_counts(fig6_program(2), passes="listgen+fusion+demotion", faithful=True)
    assert st[1]["launches"] == 6
    # With DSE our clear-list is dead (listgen completely overwrites List, reading R3): 6 -> 2
    st, plans = plan_counts(fig6_program(2), passes="all", faithful=True)
    assert st[1]["launches"] == 2
    assert types_of(plans[1]) == ["listgen", "struct_for", "struct_for"]
    assert len(set(plans[1][:, 0])) == 2                      # two INCs in one group
    # folded lowering: 4 -> 2
    st, _ = plan_counts(fig6_program(2), passes="all")
    assert (st[1]["tasks_lowered"], st[1]["launches"]) == (4, 2)


def dense1d(n=1024, fields=("x",), dtype="i32"):
    L = W.Layout()
    lv = L.chain([("dense", (n,))], [(f, dtype) for f in fields])
    return L, lv


def test_fill_array_10_to_1():
    # PAPER.md:491 "only 1 task is launched in these cases instead of 10"
    L, lv = dense1d()
    calls = [W.struct_for("FILL", lv[-1], [0], [7.0]) for _ in range(10)] + [W.flush()]
    st, plans = plan_counts(W.program(L, calls))
    assert st[0]["tasks_lowered"] == 10 and st[0]["launches"] == 1
    st, _ = plan_counts(W.program(L, calls), passes=0)
    assert st[0]["launches"] == 10


def test_chain_copy_fuses():
    # PAPER.md:487 "y[i] = x[i] + 1 and z[i] = y[i] + 4 ... They are fused"
    L, lv = dense1d(fields=("x", "y", "z"))
    calls = [W.struct_for("ADD_CONST", lv[-1], [1, 0], [1.0]), W.struct_for("ADD_CONST", lv[-1], [2, 1], [4.0]),
             W.flush()]
    st, plans = plan_counts(W.program(L, calls))
    assert st[0]["launches"] == 1 and st[0]["tasks_fused"] == 1


def test_increments_fuse_to_one():
    # PAPER.md:489 increments: 10 inc() kernels -> one fused task; on a 2-level sparse field
    L = W.Layout()
    lv = L.chain([("pointer", (8,)), ("dense", (4,))], [("x", "i32")])
    calls = [W.activate(0, np.array([[0], [9]], dtype=np.int32)), W.flush()]
    calls += [W.struct_for("INC", lv[-1], [0], [1.0]) for _ in range(10)] + [W.flush()]
    st, plans = plan_counts(W.program(L, calls))
    assert st[1]["tasks_lowered"] == 20
    assert types_of(plans[1]) == ["listgen"] + ["struct_for"] * 10
    assert st[1]["launches"] == 2 and st[1]["listgens_removed"] == 9


def autodiff_program(iters=10, observed=None):
    L = W.Layout()
    lv = L.chain([("dense", (256,))], [("x", "f32"), ("grad", "f32")])
    L.scalar("loss", "f32")
    f = L.fields
    calls = []
    for _ in range(iters):
        calls += [W.serial("CLEAR_SCALAR", [f["loss"]]),
                  W.struct_for("REDUCE_SUM", lv[-1], [f["loss"], f["x"]]),
                  W.struct_for("INC", lv[-1], [f["grad"]], [1.0])]
    calls.append(W.flush(observed=observed))
    return W.program(L, calls)


def test_autodiff_dse_keeps_last_forward():
    # "the forward tasks computing the loss function should be
    # eliminated except for the last one, so the number of launched tasks reduces by roughly a half"
    st, plans = plan_counts(autodiff_program())
    eager = st[0]["tasks_lowered"]
    assert eager == 30
    assert st[0]["launches"] <= 0.6 * eager
    p = plans[0]
    reduces = [r for r in p if r[1] == 3 and r[2] % 3 == 1]
    assert len(reduces) == 1 and reduces[0][2] == 28           # the last forward reduction survives
    # no DSE: nothing removed
    st2, _ = plan_counts(autodiff_program(), passes="listgen+demotion+fusion")
    assert st2[0]["dead_removed"] == 0


def multires_program(n=8, demote=True):
    L = W.Layout()
    xl = L.chain([("pointer", (4, 4)), ("dense", (4, 4))], [("x", "f32")])
    yl = L.chain([("pointer", (4, 4)), ("dense", (2, 2))], [("y", "f32")])
    f = L.fields
    rng = np.random.default_rng(1)
    cells = np.stack([rng.integers(0, 16, 12), rng.integers(0, 16, 12)], 1).astype(np.int32)
    calls = [W.activate(f["x"], cells), W.struct_for("FILL", xl[-1], [f["x"]], [1.0]), W.flush()]
    for _ in range(n):
        calls += [W.struct_for("DOWNSAMPLE", xl[-1], [f["y"], f["x"]], [0.25, 0.0], [True]),
                  W.struct_for("INC", yl[-1], [f["y"]], [1.0])]
    calls.append(W.flush())
    return W.program(L, calls), yl


def test_downsample_demotion():
    # PAPER.md:346-361 / Fig. 9 caption: with x unchanged, repeated
    # y[i//2] += x[i]*0.25 keeps y's mask, so y's list generation is not repeated.
    prog, yl = multires_program(8)
    st, plans = plan_counts(prog, passes="listgen+demotion")
    p = plans[1]
    y_listgens = [r for r in p if r[1] == 1 and r[3] == yl[0]]
    one, plans1 = plan_counts(multires_program(1)[0], passes="listgen+demotion")
    y_listgens_1 = [r for r in plans1[1] if r[1] == 1 and r[3] == yl[0]]
    assert len(y_listgens) == len(y_listgens_1) == 1
    ds = [r for r in p if r[1] == 3 and r[2] % 2 == 0]
    assert len(ds) == 8 and ds[0][4] == 1 and all(r[4] == 0 for r in ds[1:])   # runs 2..8 non-activating
    # without demotion every run re-generates y's list
    st0, plans0 = plan_counts(prog, passes="listgen")
    assert len([r for r in plans0[1] if r[1] == 1 and r[3] == yl[0]]) == 8


def test_deep_hierarchy_no_fusion_fewer_listgens():
    # PAPER.md:505 "The tasks are not fusible but we can still get some
    # performance boost by eliminating list generation tasks."
    L = W.Layout()
    lv = L.chain([("pointer", (4,)), ("pointer", (4,)), ("bitmasked", (4,)), ("dense", (4,))], [("x", "i32")])
    calls = [W.activate(0, np.array([[3], [70], [200]], dtype=np.int32)), W.flush()]
    calls += [W.struct_for("JITTER", lv[-1], [0]) for _ in range(5)] + [W.flush()]
    st, _ = plan_counts(W.program(L, calls))
    st0, _ = plan_counts(W.program(L, calls), passes=0)
    assert st[1]["tasks_fused"] == 0
    assert st[1]["listgen_launched"] < st0[1]["listgen_launched"]
    assert (st0[1]["listgen_launched"], st[1]["listgen_launched"]) == (15, 3)


def test_c1_c2_launch_counts():
    # SURVEY.md Appendix A (readings R3, R5, R19): C1 8 -> 5 per step, faithful 11
    st, _ = plan_counts(W.c1_program(steps=3))
    assert all((s["tasks_lowered"], s["launches"]) == (8, 5) for s in st)
    assert st[1]["plan_cache_hits"] == 1
    st, _ = plan_counts(W.c1_program(steps=1), faithful=True)
    assert (st[0]["tasks_lowered"], st[0]["launches"]) == (11, 5)
    # C2: 50-iteration solve + final reduction: 161 eager -> 55
    st, plans = plan_counts(W.c2_program())
    assert (st[0]["tasks_lowered"], st[0]["launches"]) == (161, 55)
    st0, _ = plan_counts(W.c2_program(), passes=0)
    assert st0[0]["launches"] == 161


def test_chain_pass_beyond_paper():
    # SG_PASS_CHAIN (beyond PAPER.md:367-368): the 50 dependent
    # JACOBI sweeps become phases of one cooperative launch; the independent
    # scalar clear is hoisted in front of the chain.
    st, plans = plan_counts(W.c2_program(), passes="all+chain")
    assert st[0]["launches"] == 5 and st[0]["tasks_chained"] == 50
    assert types_of(plans[0])[:4] == ["activate", "listgen", "listgen", "serial"]
    assert len(set(plans[0][4:, 0])) == 1           # one group holds every struct-for
    # without the flag nothing changes
    st2, _ = plan_counts(W.c2_program(), passes="all")
    assert st2[0]["launches"] == 55 and st2[0]["tasks_chained"] == 0


@pytest.mark.parametrize("seed", range(60))
def test_chain_schedule_soundness_on_oracle(seed):
    prog = W.fuzz_program(seed)
    ref = oracle.run_program(prog)
    o = replay_plan_on_oracle(prog, 15 | 16)
    L = prog["layout"]
    for name, fid in L.fields.items():
        assert np.array_equal(o.field(fid), ref.field(fid)), (seed, name)


# ---------------------------------------------------------------------------
# C4 (differentiable MPM): the forward gradient clears are dead stores
# ("clear_all_gradients ... a typical source of dead stores");
# an unobserved loss is dead too (the autodiff example).
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("T", [1, 2, 4])
def test_c4_dse_removes_forward_gradient_clears(T):
    prog = W.c4_program(n_grid=16, n_particles=100, T=T)
    st, plans = plan_counts(prog)
    s = st[0]
    # eager lowering: forward substep = deactivate (+2 listgens), 4 grad
    # clears (+2 listgens each), P2G, GRID_OP (+2 listgens), G2P = 19; backward substep =
    # deactivate grid (+2), P2G, deactivate grad (+2), G2P_ADJ, P2G_ADJ = 10; +3 loss/seed
    assert s["tasks_lowered"] == 29 * T + 3
    # dead per substep: the 4 forward grad clears, and 4 listgens that only fed
    # DEACTIVATEs -- a whole-tree DEACTIVATE on these small trees is a pool reset
    # with no list input (reading R33)
    assert s["dead_removed"] == 8 * T
    assert s["launches"] == 11 * T + 3
    rf_groups = {int(r[0]) for r in plans[0] if sg.TASK_TYPES[r[1]] == "range_for"}
    # P2G, G2P per forward substep; P2G, G2P_ADJ, P2G_ADJ per backward substep;
    # LOSS_MEAN, ADJ_INIT -- the MPM transfers have their own (binned) kernels and run unfused
    assert len(rf_groups) == 5 * T + 2
    assert sum(sg.TASK_TYPES[r[1]] == "range_for" for r in plans[0]) == 5 * T + 2
    st_dse, _ = plan_counts(prog, passes="dse")
    assert st_dse[0]["dead_removed"] == 18 * T        # clears plus their listgens, reset inputs
    # an unobserved loss (observed = no fields) is dead as well
    L = prog["layout"]
    prog2 = W.c4_program(n_grid=16, n_particles=100, T=T, observed=[])
    st2, _ = plan_counts(prog2)
    assert st2[0]["dead_removed"] == 8 * T + 2


def test_mg_demotion_and_listgen_removal():
    # SURVEY N1, PAPER.md:438-441 (MGPCG: restriction/smoothing/prolongation listgens
    # 351,440 -> 343) and PAPER.md:346-361 (demotion of the [i//2] restriction).
    prog = W.mg_program(n=512, cycles=10)
    st, _ = plan_counts(prog)
    s = st[0]
    assert s["demotions"] == 3 * 9            # RESTRICT into the 3 coarse levels, cycles 2..10
    assert s["listgen_launched"] == 7         # 4 levels' lists once, coarse ones after cycle 1
    assert s["tasks_fused"] == 31             # the two coarse clears per level, FILL r0 + FILL z0
    st0, _ = plan_counts(prog, passes=0)
    # eager: per cycle 2 x (4 pre + 4 post) + 64 bottom half sweeps, 3 restrictions, 3
    # prolongations (a listgen + a body each), 6 clears, + setup / residual
    assert st0[0]["launches"] == s["tasks_lowered"] == 2008
    assert s["launches"] == 981
    nodem, _ = plan_counts(prog, passes=15 & ~2)
    assert nodem[0]["demotions"] == 0 and nodem[0]["listgen_launched"] == 34
    assert nodem[0]["launches"] > s["launches"]


def test_mgpcg_counts():
    # MGPCG: listgens 657 -> 7; demotion alone accounts for 37 -> 7
    # (the paper: 6.7x from demotion); the per-iteration residual monitor (rTr) is
    # overwritten before it is observed except in the last iteration: DSE
    prog = W.mgpcg_program(n=512, iters=10)
    s = plan_counts(prog)[0][0]
    assert (s["tasks_lowered"], s["launches"], s["listgen_launched"]) == (2412, 1127, 7)
    assert s["dead_removed"] == 2 * 9 and s["demotions"] == 30
    nodem = plan_counts(prog, passes=15 & ~2)[0][0]
    assert nodem["listgen_launched"] == 37


@pytest.mark.parametrize("passes", [0, 1, 3, 15])
def test_mgpcg_schedule_soundness_on_oracle(passes):
    prog = W.mgpcg_program(n=64, levels=3, block=8, iters=3, radius_frac=0.3)
    ref = oracle.run_program(prog)
    o = replay_plan_on_oracle(prog, passes)
    for name, fid in prog["layout"].fields.items():
        assert np.array_equal(o.field(fid), ref.field(fid)), (passes, name)


@pytest.mark.parametrize("passes", [0, 1, 3, 15])
def test_mg_schedule_soundness_on_oracle(passes):
    prog = W.mg_program(n=64, levels=3, block=8, cycles=2, radius_frac=0.3)
    ref = oracle.run_program(prog)
    o = replay_plan_on_oracle(prog, passes)
    for name, fid in prog["layout"].fields.items():
        assert np.array_equal(o.field(fid), ref.field(fid)), (passes, name)


def test_deactivate_reset_rule():
    # R33: whole-tree DEACTIVATE of a small tree runs as a pool reset (no lists);
    # a deeper level, or a tree whose dense volume exceeds 64 MiB, keeps the list-based kernel
    st, plans = plan_counts(W.c3_program(n_grid=32, n_particles=100, steps=1))
    assert types_of(plans[0]) == ["deactivate", "range_for", "listgen", "listgen", "struct_for", "range_for"]
    st5, plans5 = plan_counts(W.c5_program(n_grid=512, n_particles=100, steps=1))
    assert types_of(plans5[0])[:3] == ["listgen", "listgen", "deactivate"]


@pytest.mark.parametrize("passes", [0, 1, 4, 8, 15, 31])
def test_c4_schedule_soundness_on_oracle(passes):
    prog = W.c4_program(n_grid=16, n_particles=60, T=2, side=6, center=(0.5, 0.5, 0.5))
    ref = oracle.run_program(prog)
    o = replay_plan_on_oracle(prog, passes)
    for i in range(len(prog["arrays"])):
        assert np.array_equal(o.array(i), ref.array(i)), (passes, i)
    L = prog["layout"]
    assert np.array_equal(o.field(L.fields["loss"]), ref.field(L.fields["loss"]))


def test_plan_is_topological_and_deterministic():
    p1 = plan_counts(W.c2_program())[1][0]
    p2 = plan_counts(W.c2_program())[1][0]
    assert np.array_equal(p1, p2)


# ---------------------------------------------------------------------------
# T3 on the CPU: replay the planner's schedule on the oracle
# ---------------------------------------------------------------------------
def replay_plan_on_oracle(prog, passes):
    """Eager oracle vs oracle executing the planner's schedule window by window."""
    g = sg.Grid(prog["desc"], plan_only=True)
    o = oracle.Oracle(prog["desc"])
    for arr in prog.get("arrays", {}).values():
        o.register_array(arr)
    window = []
    for c in prog["calls"]:
        if c["call"] != "flush":
            k = c["call"]
            if k == "activate":
                g.activate(c["field"], c["coords"])
            elif k == "struct_for":
                g.struct_for(c["op"], c["snode"], c["fields"], c.get("params", []), c.get("activating", []))
            elif k == "serial":
                g.serial(c["op"], c["fields"], c.get("params", []))
            elif k == "range_for":
                g.range_for(c["op"], c["n"], c["fields"], c["arrays"], c.get("params", []), c.get("activating", []))
            elif k == "clear":
                g.clear(c["target"], sg.CLEAR_VALUES if c["mode"] == "values" else sg.DEACTIVATE)
            elif k == "listgen":
                g.listgen(c["snode"])
            window.append(c)
            continue
        g.flush(passes)
        for grp, ttype, call, snode, act, _ in g.last_plan():
            c = window[call]
            t = sg.TASK_TYPES[ttype]
            if t == "activate":
                o.activate(c["field"], c["coords"])
            elif t == "listgen":
                o.listgen(int(snode))
            elif t == "clear_list":
                o.clear_list(int(snode))
            elif t == "deactivate":
                o.deactivate_task(int(snode))
            elif t == "serial":
                if c["call"] == "serial":
                    o.serial_task(c["op"], c["fields"], c.get("params", []))
                else:
                    o.serial_task("CLEAR_SCALAR", [c["target"]])
            elif t == "range_for":
                o.range_for_task(c["op"], c["n"], c["fields"], c["arrays"], c.get("params", []), int(act))
            elif t == "struct_for":
                if c["call"] == "clear":
                    o.struct_for_task("FILL", int(snode), [c["target"]], [0.0], 0)
                else:
                    o.struct_for_task(c["op"], int(snode), c["fields"], c.get("params", []), int(act))
        window = []
    return o


PASS_SUBSETS = [0, 1, 2, 4, 8, 1 | 2, 1 | 4, 15]


@pytest.mark.parametrize("seed", range(120))
def test_schedule_soundness_on_oracle(seed):
    prog = W.fuzz_program(seed)
    ref = oracle.run_program(prog)
    L = prog["layout"]
    for passes in PASS_SUBSETS:
        try:
            o = replay_plan_on_oracle(prog, passes)
        except oracle.OracleError as e:
            raise AssertionError(f"seed {seed} passes {passes}: {e}")
        for name, fid in L.fields.items():
            assert np.array_equal(o.field(fid), ref.field(fid)), (seed, passes, name)
        for s in range(1, len(L.rows)):
            if L.rows[s][0] in (W.BITMASKED, W.POINTER):
                assert np.array_equal(o.mask(s), ref.mask(s)), (seed, passes, s)


def test_all_passes_never_more_launches_than_any_subset():
    # SPEC.md:457 acceptance 10
    for seed in range(40):
        prog = W.fuzz_program(seed)
        counts = {}
        for passes in PASS_SUBSETS:
            st, _ = plan_counts(prog, passes=passes)
            counts[passes] = sum(s["launches"] for s in st)
        assert counts[15] <= min(counts.values()), (seed, counts)
        assert all(counts[p] <= counts[0] for p in counts)


def test_layout_errors_match_spec():
    bad = [
        [[0, -1, 0, 1, 1, 1, 0], [3, 0, 1, 3, 1, 1, 0], [4, 1, 1, 1, 1, 1, 0]],
        [[0, -1, 0, 1, 1, 1, 0], [1, 0, 1, 4, 1, 1, 0], [4, 1, 1, 1, 1, 1, 0], [1, 2, 1, 2, 1, 1, 0]],
        [[0, -1, 0, 1, 1, 1, 0], [1, 0, 2, 4, 4, 1, 0], [1, 1, 1, 2, 1, 1, 0], [4, 2, 1, 1, 1, 1, 0]],
        [[0, -1, 0, 1, 1, 1, 0], [3, 0, 1, 4, 1, 1, 0], [4, 1, 1, 1, 1, 1, 0]],   # pointer leaf
    ]
    for d in bad:
        with pytest.raises(sg.SgError) as e:
            sg.Grid(np.array(d, dtype=np.int32), plan_only=True)
        assert e.value.kind == "LAYOUT"


def test_bad_task_rejected():
    L, lv = W.c1_layout()
    g = sg.Grid(L.desc(), plan_only=True)
    with pytest.raises(sg.SgError):
        g.struct_for("STENCIL", lv[-1], [0, 0])          # in-place stencil would race
    with pytest.raises(sg.SgError):
        g.struct_for("FILL", lv[0], [0], [1.0])          # not the leaf level
    with pytest.raises(sg.SgError):
        g.struct_for("NOPE" if False else 99, lv[-1], [0])


def test_library_exports_every_declared_symbol():
    import re
    import ctypes
    hdr = open(sg.LIB_PATH.replace("paper_2012_08141_b200/libsg.so", "include/sg.h")).read()
    declared = set(re.findall(r"\b(sg_[a-z_]+)\s*\(", hdr)) - {"sg_alloc_fn", "sg_free_fn"}
    lib = ctypes.CDLL(sg.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(sg.EXPORTS)


def test_stats_struct_matches_header():
    import ctypes
    """The ctypes sg_stats mirror has the header's fields, in order, with the
    header's types (a drifted mirror would corrupt memory on every flush)."""
    import re
    hdr = open(sg.LIB_PATH.replace("paper_2012_08141_b200/libsg.so", "include/sg.h")).read()
    body = hdr[: hdr.index("} sg_stats;")]
    body = body[body.rindex("typedef struct {"):]
    fields = re.findall(r"^\s*(int64_t|double|int32_t)\s+(\w+);", body, re.M)
    ctype = {"int64_t": ctypes.c_int64, "double": ctypes.c_double, "int32_t": ctypes.c_int32}
    assert [(n, ctype[t]) for t, n in fields] == [(n, t) for n, t in sg.Stats._fields_]
