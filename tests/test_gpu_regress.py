"""GPU regressions (-m gpu): the paper-faithful lowering on the device and
CUDA-graph relaunch with changed task parameters."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2012_08141_b200 import sg  # noqa: E402
from test_gpu_parity import compare  # noqa: E402


@pytest.mark.parametrize("passes", [0, "listgen+demotion+fusion", "all"])
@pytest.mark.parametrize("which", ["c1", "c1_i32", "c2_small", "fuzz"])
def test_faithful_lowering_runs_clear_list(passes, which):
    """sg_opts.lowering = 1 ("3 tasks": clear-list + listgen per
    sparse level): k_clear_list runs on the device and results still equal the
    oracle's eager replay.  Without DSE the clear-lists survive; with DSE they
    are dead (our listgen completely overwrites the list, reading R3)."""
    progs = {"c1": lambda: [W.c1_program(steps=2)], "c1_i32": lambda: [W.c1_program(steps=2, dtype="i32")],
             "c2_small": lambda: [W.c2_small_program(iters=3)],
             "fuzz": lambda: [W.fuzz_program(s) for s in range(12)]}[which]()
    for prog in progs:
        g, st = sg.run_program(prog, passes=passes, faithful=True, debug=True)
        o = oracle.run_program(prog)
        compare(g, o, prog)
        cl = sum(s["clear_list_launched"] for s in st)
        lowered = sum(s["tasks_lowered"] for s in st)
        if which != "fuzz":
            if passes == "all":
                assert cl == 0
            else:
                assert cl > 0
        if which == "c1" and passes == 0:
            assert st[0]["tasks_lowered"] == 11 and st[0]["launches"] == 11
        assert lowered >= sum(s["launches"] for s in st)
        g.close()


def test_graph_relaunch_sees_new_params():
    """A cached plan is captured as a CUDA graph on its 2nd flush and relaunched
    as-is from the 3rd on; task params are baked into the captured op tables,
    so a flush with different params must not replay stale ones."""
    L, lv = W.c2_layout(ptr=2)
    f = L.fields
    coords = torch.as_tensor(W.block_ball_coords(8, 8, 20.0), device="cuda")
    g = sg.Grid(L.desc())
    vals = [1.0, 2.0, 3.0, 4.0, 5.0, 5.0, -7.5]
    for k, v in enumerate(vals):
        g.activate(f["b"], coords)
        g.struct_for("FILL", lv[-1], [f["b"]], [v])
        g.struct_for("INC", lv[-1], [f["b"]], [0.25 * k])
        st = g.flush("all")
        g.sync()
        b = g.field(f["b"])
        nz = b[b != 0]
        assert nz.size > 0 and np.all(nz == np.float32(v + 0.25 * k)), (k, v, np.unique(nz)[:4], st)
