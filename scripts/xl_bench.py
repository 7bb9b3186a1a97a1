"""Roofline variants sized far above L2:

  JAC-XL  1024^3, pointer(32^3) -> bitmasked(4^3) -> dense(8^3), block-ball R=288,
          one JACOBI struct-for per launch (12 B algorithmic per active cell).
  LG-XL   2048^3, pointer(64^3) -> bitmasked(32^3) leaf, 25% of pointer cells,
          10% of their bits; one cell-level listgen of the leaf (reads the mask
          words of every listed container + 4 B per parent entry, writes 4 B per
          active cell + the count).

Prints one JSON line per variant: achieved algorithmic GB/s per launch (CUDA
events on the grid's stream around each launch, sg_profile_read) vs the HBM peak.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_2012_08141_b200 import sg  # noqa: E402


def jac_xl(iters=10, radius=288.0):
    L, lv = W.c2_layout(ptr=32)
    f = L.fields
    coords = W.block_ball_coords(128, 8, radius)
    g = sg.Grid(L.desc())
    dc = torch.as_tensor(coords).cuda()
    calls, _ = W.c2_solve_calls(L, lv, coords, iters=0, reduce_result=False)
    bench.enqueue_calls(g, calls, dc)
    g.flush("all")
    g.sync()
    flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    src, dst = f["x0"], f["x1"]

    def solve(k):
        # k iterations in one flush window (one listgen pair; the first JACOBI
        # after the listgen also builds the block table)
        nonlocal src, dst
        flush_buf.zero_()
        for _ in range(k):
            g.struct_for("JACOBI", lv[-1], [dst, src, f["b"]])
            src, dst = dst, src
        g.flush("all")
        return sg.profile_read(g).get(100 + sg.OPS["JACOBI"], (0.0, 0))

    solve(2)
    sg.set_profiling(g, True)
    t1, _ = solve(1)
    tk, nk = solve(iters + 1)
    # steady-state launches: (k+1 iterations) - (1 iteration), the latter carrying the table build
    ms, n = tk - t1, iters
    nbytes = len(coords) * 512 * 12
    peak, kind = bench.hbm_peak()
    ach = nbytes / (ms / n / 1e3) / 1e9
    return {"variant": "JAC-XL", "blocks": len(coords), "cells": len(coords) * 512, "bytes_per_launch": nbytes,
            "avg_launch_us": ms / n * 1e3, "achieved_GBps": ach, "peak_GBps": peak, "peak_source": kind,
            "frac": ach / peak, "launches": n}


def sf_xl(iters=10, radius=288.0, jit=False, interpreter=False, group="jacobi_reduce"):
    """SF-XL: the generic fused megakernel (k_struct_for op table) at JAC-XL
    size: JACOBI fused with the residual-style reduction s += x1 (PAPER.md:440
    "fuse the Jacobi smoothing and reduction kernels"), one launch per
    iteration.  Algorithmic bytes: 12 B per active cell (read x0, b; write x1;
    the reduction reads x1 from the thread's registers)."""
    prev = sg.jit_info()["mode"]
    if not jit:
        sg.jit_set_mode(0)
    if (interpreter or jit) and group == "jacobi_reduce":   # not the dedicated k_jacobi8<RED>
        os.environ["SG_NO_JAC8"] = "1"
    L, lv = W.c2_layout(ptr=32)
    f = L.fields
    coords = W.block_ball_coords(128, 8, radius)
    g = sg.Grid(L.desc())
    dc = torch.as_tensor(coords).cuda()
    calls, _ = W.c2_solve_calls(L, lv, coords, iters=0, reduce_result=False)
    bench.enqueue_calls(g, calls, dc)
    g.flush("all")
    g.sync()
    flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    src, dst = f["x0"], f["x1"]

    def solve(k):
        # s accumulates every sweep's sum (no clear in between: each reduction
        # is read by the next one, so DSE keeps all of them and every sweep is
        # one fused JACOBI+REDUCE_SUM launch)
        nonlocal src, dst
        flush_buf.zero_()
        g.serial("CLEAR_SCALAR", [f["s"]])
        for _ in range(k):
            if group == "jacobi_reduce":
                g.struct_for("JACOBI", lv[-1], [dst, src, f["b"]])
                g.struct_for("REDUCE_SUM", lv[-1], [f["s"], dst])
            else:   # MGPCG's A p and p.Ap (no dedicated kernel: interpreter or JIT)
                g.struct_for("STENCIL", lv[-1], [dst, src])
                g.struct_for("DOT", lv[-1], [f["s"], src, dst], [-1.0])
            src, dst = dst, src
        st = g.flush("all")
        return sg.profile_read(g).get(100 + sg.OPS["JACOBI" if group == "jacobi_reduce" else "STENCIL"], (0.0, 0)), st

    solve(2)
    solve(1)
    solve(iters + 1)   # every group content of the timed flushes compiled (JIT) and warm
    solve(1)
    sg.set_profiling(g, True)
    (t1, _), _ = solve(1)
    (tk, nk), st = solve(iters + 1)
    if not jit:
        sg.jit_set_mode(prev)
    os.environ.pop("SG_NO_JAC8", None)
    ms, n = tk - t1, iters
    # 12 B per cell (x0, b read, x1 written) for JACOBI+REDUCE; 8 B (p read,
    # Ap written; the dot reads both from registers) for STENCIL+DOT
    nbytes = len(coords) * 512 * (12 if group == "jacobi_reduce" else 8)
    peak, kind = bench.hbm_peak()
    ach = nbytes / (ms / n / 1e3) / 1e9
    assert st["tasks_fused"] == iters + 1, st
    gname = "JACOBI+REDUCE_SUM" if group == "jacobi_reduce" else "STENCIL+DOT"
    kern = ("NVRTC-specialized streaming kernel (stream8_body, constant op table)" if jit
            else "k_stream8 (streaming kernel, runtime op table)" if interpreter or group != "jacobi_reduce"
            else "k_jacobi8<RED> (dedicated)") + f" running the fused {gname} group"
    return {"variant": "SF-XL", "kernel": kern, "blocks": len(coords),
            "cells": len(coords) * 512, "bytes_per_launch": nbytes, "avg_launch_us": ms / n * 1e3,
            "achieved_GBps": ach, "peak_GBps": peak, "peak_source": kind, "frac": ach / peak, "launches": n,
            "tasks_fused": st["tasks_fused"]}


def sf_xl_jit(**kw):
    """SF-XL with the group's NVRTC-specialized kernel (JIT
    synchronous, so every timed launch runs it) beside the interpreter's."""
    prev = sg.jit_info()["mode"]
    sg.jit_set_mode(2)
    try:
        r = sf_xl(jit=True, **kw)
    finally:
        sg.jit_set_mode(prev)
    r["variant"] = "SF-XL (JIT-specialized)"
    r["jit"] = sg.jit_info()
    return r


def lg_xl(reps=15, p_ptr=0.25, p_bit=0.10, seed=0):
    L = W.Layout()
    lv = L.chain([("pointer", (64,) * 3), ("bitmasked", (32,) * 3)], [("m", "f32")])
    gen = torch.Generator(device="cuda").manual_seed(seed)
    n_ptr = 64 ** 3
    ptr_on = torch.randperm(n_ptr, device="cuda", generator=gen)[: int(n_ptr * p_ptr)]
    n_act = ptr_on.numel()
    g = sg.Grid(L.desc(), pool_capacity=n_act, list_capacity=int(n_act * 32768 * p_bit * 1.05) + 1024)
    # 10% of the bits of each active container, activated in chunks
    cells_per = int(32768 * p_bit)
    total = 0
    chunk = 4096
    for s in range(0, n_act, chunk):
        pc = ptr_on[s:s + chunk]
        px, py, pz = pc // 4096, (pc // 64) % 64, pc % 64
        loc = torch.randint(0, 32768, (pc.numel(), cells_per), device="cuda", generator=gen)
        lx, ly, lz = loc // 1024, (loc // 32) % 32, loc % 32
        co = torch.stack([(px[:, None] * 32 + lx), (py[:, None] * 32 + ly), (pz[:, None] * 32 + lz)], -1)
        co = co.reshape(-1, 3).to(torch.int32).contiguous()
        g.activate(0, co)
        g.flush("all")
        total += co.shape[0]
    g.sync()
    flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    # per-launch device time: the library's CUDA events around the listgen
    # kernel itself on the grid's stream (sg_set_profiling), L2 flushed before
    # each repetition; the median is reported -- single launches vary
    times = []
    if os.environ.get("SG_PROFILE_FROM_HERE"):
        torch.cuda.profiler.start()   # ncu --profile-from-start off: skip the setup launches
    sg.set_profiling(g, True)
    key = 200 + lv[-1]
    for _ in range(reps):
        flush_buf.zero_()
        sg.profile_read(g)            # drains (and clears) earlier events
        g.listgen(lv[-1])
        g.flush("all")
        ms1, n1 = sg.profile_read(g).get(key, (0.0, 0))
        assert n1 == 1, (ms1, n1)
        times.append(ms1)
    sg.set_profiling(g, False)
    g.sync()
    times.sort()
    ms, n = times[len(times) // 2] * reps, reps
    import ctypes
    cnt = ctypes.c_int64()
    sg._check(sg._lib.sg_export_list(g.h, lv[-1], None, 0, ctypes.byref(cnt)))
    n_out = cnt.value
    nbytes = n_act * 4 + n_act * 32768 // 8 + n_out * 4 + 4
    peak, kind = bench.hbm_peak()
    ach = nbytes / (ms / n / 1e3) / 1e9
    return {"variant": "LG-XL", "containers": n_act, "active_cells": n_out, "activate_requests": total,
            "bytes_per_launch": nbytes, "avg_launch_us": ms / n * 1e3, "achieved_GBps": ach, "peak_GBps": peak,
            "peak_source": kind, "frac": ach / peak, "launches": n,
            "min_us": times[0] * 1e3, "max_us": times[-1] * 1e3}


def act_xl(p_ptr=0.25, p_bit=0.10, seed=0):
    """ACT-XL: the LG-XL activation (214.7M random cell coordinates, 25% of the
    64^3 pointer cells, 10% of each 32^3 container) as ONE sg_activate launch,
    first touch into a fresh grid (pointer CAS + pool pops + atomicOr), then the
    same buffer again (every bit already set: the read-before-atomic path).
    Device time of the k_activate launch from the library's events."""
    L = W.Layout()
    lv = L.chain([("pointer", (64,) * 3), ("bitmasked", (32,) * 3)], [("m", "f32")])
    gen = torch.Generator(device="cuda").manual_seed(seed)
    n_ptr = 64 ** 3
    ptr_on = torch.randperm(n_ptr, device="cuda", generator=gen)[: int(n_ptr * p_ptr)]
    n_act = ptr_on.numel()
    cells_per = int(32768 * p_bit)
    px, py, pz = ptr_on // 4096, (ptr_on // 64) % 64, ptr_on % 64
    loc = torch.randint(0, 32768, (n_act, cells_per), device="cuda", generator=gen)
    co = torch.stack([px[:, None] * 32 + loc // 1024, py[:, None] * 32 + (loc // 32) % 32,
                      pz[:, None] * 32 + loc % 32], -1).reshape(-1, 3).to(torch.int32).contiguous()
    del loc
    # 10 mask-word lines and the pointer slot per request at most; order of the
    # requests is random (no two lanes of a warp share a container, typically)
    g = sg.Grid(L.desc(), pool_capacity=n_act, list_capacity=int(n_act * cells_per * 1.05) + 1024)
    # one request first: the pools are allocated and zeroed by the first flush,
    # outside the timed launches
    g.activate(0, co[:1].clone())
    g.flush(0)
    g.sync()
    sg.set_profiling(g, True)
    out = {"variant": "ACT-XL", "requests": int(co.shape[0]), "containers": n_act}
    for name in ("first_touch", "again"):
        sg.profile_read(g)
        g.activate(0, co)
        g.flush(0)
        ms, n = sg.profile_read(g).get(0, (0.0, 0))
        assert n == 1, (ms, n)
        out[name] = {"us": ms * 1e3, "requests_per_s": co.shape[0] / (ms / 1e3),
                     "coord_GBps": co.numel() * 4 / (ms / 1e3) / 1e9}
    import ctypes
    cnt = ctypes.c_int64()
    g.listgen(lv[-1])
    g.flush("all")
    sg._check(sg._lib.sg_export_list(g.h, lv[-1], None, 0, ctypes.byref(cnt)))
    out["active_cells"] = cnt.value
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["jac", "lg"]
    if "jac" in which:
        print(json.dumps(jac_xl()), flush=True)
    if "lg" in which:
        print(json.dumps(lg_xl()), flush=True)
    if "act" in which:
        print(json.dumps(act_xl()), flush=True)
    if "sf" in which:
        print(json.dumps(sf_xl()), flush=True)
    if "sfjit" in which:
        print(json.dumps(sf_xl_jit()), flush=True)
    if "sfint" in which:
        print(json.dumps(sf_xl(interpreter=True)), flush=True)
    if "cg" in which:
        print(json.dumps(sf_xl(group="axpy_dot")), flush=True)
        print(json.dumps(sf_xl_jit(group="axpy_dot")), flush=True)
