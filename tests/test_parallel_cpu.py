"""Host-side logic of the x-slab partitioner on CPU (-m "not gpu").

* SlabPartition arithmetic: ownership, ghost / boundary layers, exchange pairs;
  the ghost layers cover exactly the P2G/G2P stencil overhang of owned
  particles (base in [lo-1, hi-1], base+2 <= hi+1).
* the library data plane's host side (sg_dist_init on plan-only grids): every
  rank's plan of a C5 step carries the same exchange sequence, each kind's
  signal before its wait -- in-process groups (world 1..8, phase-split or one
  fused flush per step) and one rank per process over gloo, world size 2.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2012_08141_b200.parallel import SlabPartition


def test_partition_layers_cover_stencils():
    p = SlabPartition(512, 16, 8)
    assert p.lo == [64 * r for r in range(8)] and p.hi[-1] == 512
    for r in range(8):
        (gl0, gl1), (gr0, gr1) = p.ghost_layers(r)
        (bl0, bl1), (br0, br1) = p.boundary_layers(r)
        # every node an owned particle touches: base-1 .. base+2 with base in [lo-1, hi-1]
        nodes = np.arange(p.lo[r] - 1, p.hi[r] + 2)
        outside = nodes[(nodes < p.lo[r]) | (nodes >= p.hi[r])]
        assert all((gl0 <= n < gl1) or (gr0 <= n < gr1) for n in outside)
        # my boundary layer is exactly my neighbour's ghost layer
        left, right = p.neighbours(r)
        if left is not None:
            assert (bl0, bl1) == p.ghost_layers(left)[1]
        if right is not None:
            assert (br0, br1) == p.ghost_layers(right)[0]
    cells = np.arange(512)
    assert (p.owner(cells) == cells // 64).all()
    assert p.migration_bounds(0) == (-1e9, 64.0) and p.migration_bounds(7) == (448.0, 1e9)
    assert p.neighbours(0) == (None, 1) and p.neighbours(7) == (6, None)


def test_partition_rejects_uneven_split():
    with pytest.raises(ValueError):
        SlabPartition(512, 16, 3)


EXCHANGE_OPS = {40: "signal", 41: "wait"}


def exchange_sequence(grid):
    """[(signal|wait), ...] of the last flush's plan, in launch order (the
    sg_last_plan op column), and the plan's launch count."""
    plan = grid.last_plan()
    seq = [EXCHANGE_OPS[int(r[5])] for r in plan if int(r[1]) == 5 and int(r[5]) in EXCHANGE_OPS]
    return seq, len({int(r[0]) for r in plan})


def plan_c5_step(world, ranks, fused, uid=None):
    """Plan (no device) one sharded C5 step for `ranks` of `world`; returns
    {rank: [per-flush exchange sequences]}."""
    import workloads as W
    from paper_2012_08141_b200 import parallel
    prm = W.mpm_params(512)
    sim = parallel.SlabMPM(512, 16, None, world, ranks, prm, None, halo_cap=64, mig_cap=256, n_total=16_000_000,
                           plan_only=True, nccl_uid=uid, connect="nccl" if uid else None)
    out = {}
    for r, st in sim.ranks.items():
        flushes = []
        for ph in sim.phases(st):
            ph()
            if not fused:
                st.grid.flush("all")
                flushes.append(exchange_sequence(st.grid)[0])
        if fused:
            st.grid.flush("all")
            flushes.append(exchange_sequence(st.grid)[0])
        out[r] = flushes
    return sim, out


def check_sequences(seqs, world):
    """Every rank enqueues the same exchanges in the same order, each kind's
    signal before its wait (the SPMD condition under which device-side waits
    cannot deadlock, include/sg.h)."""
    flat = {r: [x for f in fl for x in f] for r, fl in seqs.items()}
    ref = flat[min(flat)]
    assert ref == ["signal", "wait"] * 3 if world > 1 else ref == []
    for r, f in flat.items():
        assert f == ref, (r, f)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("fused", [False, True])
def test_exchange_plan_in_process_group(world, fused):
    sim, seqs = plan_c5_step(world, list(range(world)), fused)
    check_sequences(seqs, world)
    for st in sim.ranks.values():
        assert st.transport == ("peer" if world > 1 else "peer")
        ids = set(st.send.values()) | set(st.recv.values())
        assert len(ids) == 12 and all(i >= 5 for i in ids)   # after the 5 particle arrays


def _plan_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)        # the id every rank receives (plumbing)
    sim, seqs = plan_c5_step(world, [rank], fused=True, uid=uid[0])
    seq = seqs[rank][0]
    st = sim.ranks[rank]
    everyone = [None] * world
    dist.all_gather_object(everyone, (seq, st.transport))
    q.put((rank, everyone))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_exchange_plans_agree_gloo_world2():
    """One rank per process (gloo, world 2), each planning its own fused C5
    step through the library (plan-only grids, sg_dist_init with a broadcast
    id): both ranks' plans carry the same exchange sequence."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        seqs = [s for s, _ in res[r]]
        assert seqs[0] == seqs[1] == ["signal", "wait"] * 3
        assert [t for _, t in res[r]] == ["nccl", "nccl"]


def test_send_buffer_writes_stay_between_their_exchanges():
    """Peer transport: a send buffer is the neighbour's receive buffer, so the
    count reset, the pack and the migration writes must not move across an
    exchange in the optimized plan (a count reset hoisted before the previous
    WAIT would zero a buffer the neighbour is still appending from)."""
    sim, _ = plan_c5_step(4, list(range(4)), fused=True)
    for st in sim.ranks.values():
        plan = st.grid.last_plan()
        calls = sorted({int(r[2]): int(r[5]) for r in plan}.items())   # program order: call index -> op
        checked = 0
        for pos, r in enumerate(plan):
            op, call = int(r[5]), int(r[2])
            if op not in (11, 23, 25, 43):  # ARRAY_COUNT, HALO_PACK, G2P_MIGRATE, MIGRATE_COMPACT
                continue
            for x in (40, 41):
                in_plan = sum(1 for q in plan[:pos] if int(q[5]) == x)
                in_prog = sum(1 for c, o in calls if c < call and o == x)
                assert in_plan == in_prog, (st.rank, call, op, x, in_plan, in_prog)
            checked += 1
        assert checked >= 4
