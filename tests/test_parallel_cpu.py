"""Host-side logic of the x-slab partitioner on CPU (-m "not gpu").

* SlabPartition arithmetic: ownership, ghost / boundary layers, exchange pairs;
  the ghost layers cover exactly the P2G/G2P stencil overhang of owned
  particles (base in [lo-1, hi-1], base+2 <= hi+1).
* DistTransport over torch.distributed with the gloo backend, world size 2:
  the send buffers of each side arrive in the neighbour's receive buffers
  (the same code path runs NCCL over NVLink on the GPU box).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2012_08141_b200.parallel import DistTransport, SlabPartition


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
    pairs = p.exchange_pairs()
    assert len(pairs) == 2 * 7 and (0, 1, "R") in pairs and (1, 0, "L") in pairs


def test_partition_rejects_uneven_split():
    with pytest.raises(ValueError):
        SlabPartition(512, 16, 3)


class _FakeRank:
    def __init__(self, r, words):
        self.bufs = {"halo": {}}
        for name in ("sendL", "sendR", "recvL", "recvR"):
            t = torch.zeros(words, dtype=torch.int32)
            if name.startswith("send"):
                t[0] = 3 + r          # record count
                t[4:] = 1000 * r + (1 if name == "sendR" else 2)
            self.bufs["halo"][name] = t


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = SlabPartition(64, 4, world)
    st = _FakeRank(rank, 16)
    DistTransport().exchange({rank: st}, p.exchange_pairs(), "halo")
    got = {k: st.bufs["halo"][k].tolist() for k in ("recvL", "recvR")}
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_dist_transport_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # rank 0 receives rank 1's left send in its right buffer, and vice versa
    assert res[0]["recvR"][0] == 4 and res[0]["recvR"][4] == 1002
    assert res[1]["recvL"][0] == 3 and res[1]["recvL"][4] == 1
    assert res[0]["recvL"] == [0] * 16 and res[1]["recvR"] == [0] * 16   # no neighbour there
