"""The library's peer transport across PROCESSES (-m gpu): two ranks, one per
process, both on cuda:0 (the only GPU a test run has), connected through
sg_dist_peer_info / sg_dist_connect (CUDA IPC of each rank's exchange arena,
blobs exchanged over gloo).  Each rank runs the whole sharded C5-shape step as
ONE flush (device-side signal / wait between the phases, include/sg.h); the
gathered particles and the stitched grid mass must equal the unpartitioned
oracle's single step within 1e-5 of the shadow magnitude (same bar as the
virtual-rank handoff tests in test_gpu_parallel.py).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

NG, PTR, N = 128, 4, 30000


def _particles():
    import workloads as W
    return W.c5_particles(N, NG, length=100, width=16, seed=3, shear=40.0)


def _worker(rank, world, port, q, steps):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        import workloads as W
        from paper_2012_08141_b200 import parallel
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        prm = W.mpm_params(NG)
        sim = parallel.SlabMPM(NG, PTR, _particles(), world, [rank], prm, lambda r: torch.device("cuda", 0),
                               halo_cap=1024, mig_cap=8192, connect="ipc")
        st = sim.ranks[rank]
        stats = []
        for _ in range(steps):
            stats.append(sim.step(fused=True))
        st.grid.sync()
        n = st.n()
        parts = {k: getattr(st, k)[:, :n].cpu().numpy() for k in ("x", "v", "C", "J", "id")}
        m = st.grid.field(sim.L.fields["m"])
        lo, hi = sim.part.lo[rank], sim.part.hi[rank]
        q.put((rank, {"transport": st.transport, "parts": parts, "m": m[lo:hi], "lo": lo, "hi": hi,
                      "flushes_per_step": len(stats[-1])}))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure to the parent
        q.put((rank, {"error": repr(e)}))
        raise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, steps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, steps)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert "error" not in res[r], res[r]["error"]
    for p in procs:
        assert p.exitcode == 0
    return res


def test_ipc_peer_transport_two_processes_one_step():
    import oracle
    import workloads as W
    res = _run(2, 1)
    assert [res[r]["transport"] for r in range(2)] == ["peer", "peer"]
    assert all(res[r]["flushes_per_step"] == 1 for r in range(2))
    parts = {k: np.concatenate([res[r]["parts"][k] for r in range(2)], axis=1) for k in ("x", "v", "C", "J", "id")}
    order = np.argsort(parts["id"][0])
    parts = {k: v[:, order] for k, v in parts.items()}
    assert (parts["id"][0] == np.arange(N)).all()      # nobody lost or duplicated
    L, lv = W.c5_layout(NG, PTR)
    prm = W.mpm_params(NG)
    p0 = _particles()
    prog = W.program(L, W.c3_step_calls(L, lv, N, prm) + [W.flush()], arrays=p0)
    o = oracle.run_program(prog)
    for i, k in enumerate(("x", "v", "C", "J")):
        want, mag = o.array(i, with_mag=True)
        err = np.abs(parts[k].astype(np.float64) - want)
        bad = err > 1e-5 * np.maximum(np.abs(want), mag)
        assert not bad.any(), f"{k}: {bad.sum()} off"
    m_want, m_mag = o.field(L.fields["m"], with_mag=True)
    m_got = np.zeros_like(m_want)
    for r in range(2):
        m_got[res[r]["lo"]:res[r]["hi"]] = res[r]["m"]
    bad = np.abs(m_got - m_want) > 1e-5 * np.maximum(np.abs(m_want), m_mag)
    assert not bad.any(), f"m: {bad.sum()} off"


def test_ipc_peer_transport_two_processes_three_steps():
    """Three fused steps: the exchange buffers are reused without
    double-buffering (dist.cu) -- nothing lost, mass conserved."""
    import workloads as W
    res = _run(2, 3)
    ids = np.concatenate([res[r]["parts"]["id"][0] for r in range(2)])
    assert np.array_equal(np.sort(ids), np.arange(N))
    prm = W.mpm_params(NG)
    mass = sum(res[r]["m"].astype(np.float64).sum() for r in range(2))
    np.testing.assert_allclose(mass, N * prm["p_mass"], rtol=1e-5)
