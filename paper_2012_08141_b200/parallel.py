"""x-slab partitioner for sparse MLS-MPM across GPUs.

Rank g of G owns the pointer-cell x-slab [g*Px/G, (g+1)*Px/G) of the grid and
the particles whose cell x lies in it.  Every step:

  1. DEACTIVATE, P2G (activating) of the owned particles: contributions reach
     one leaf-block layer beyond each face (the ghost layers);
     HALO_PACK of the two ghost layers.
  2. exchange #1 (halo reduce): ghost layers go to their owners, which
     HALO_UNPACK them with add (activating); GRID_OP; HALO_PACK of the two
     boundary layers.
  3. exchange #2 (halo fill): boundary layers overwrite the neighbours' ghost
     layers (HALO_UNPACK set); G2P_MIGRATE: G2P fused with the stable in-place
     compaction of the particles that stay, leavers packed per side.
  4. exchange #3 (migration): MIGRATE_APPEND of the received particles.

All of it runs in libsg kernels enqueued through the C-ABI; the only
device-to-device traffic is the three exchanges, each a fixed-capacity buffer
per side whose first word is the device-side record count (no host sync).
Transports: `DistTransport` (torch.distributed P2P: NCCL over NVLink on GPUs,
gloo on CPU) and `LocalTransport` (several virtual ranks in one process on one
GPU, buffers copied device-to-device -- what the single-GPU tests drive).
"""
from __future__ import annotations

import numpy as np

from . import sg

PREC_WORDS = 17   # particle record: x3 v3 C9 J1 id1 (exchange_ops.cuh)


class SlabPartition:
    """Pure arithmetic of the decomposition (tested on CPU)."""

    def __init__(self, n_grid, ptr_cells_x, world, block=4):
        if ptr_cells_x % world:
            raise ValueError(f"{ptr_cells_x} pointer slabs do not split over {world} ranks")
        self.n_grid, self.world, self.block = n_grid, world, block
        per = ptr_cells_x // world
        cells_per_ptr = n_grid // ptr_cells_x
        self.lo = [r * per * cells_per_ptr for r in range(world)]
        self.hi = [(r + 1) * per * cells_per_ptr for r in range(world)]

    def owner(self, cell_x):
        cell_x = np.asarray(cell_x)
        w = self.hi[0] - self.lo[0]
        return np.clip(cell_x // w, 0, self.world - 1)

    def neighbours(self, r):
        return (r - 1 if r > 0 else None, r + 1 if r < self.world - 1 else None)

    # [lo, hi) in cells of the block layers (block origin x must fall inside)
    def ghost_layers(self, r):
        B = self.block
        return (self.lo[r] - B, self.lo[r]), (self.hi[r], self.hi[r] + B)

    def boundary_layers(self, r):
        B = self.block
        return (self.lo[r], self.lo[r] + B), (self.hi[r] - B, self.hi[r])

    def exchange_pairs(self):
        """(src, dst, side) for one exchange: side 'L' = src's left buffer."""
        out = []
        for r in range(self.world):
            left, right = self.neighbours(r)
            if left is not None:
                out.append((r, left, "L"))
            if right is not None:
                out.append((r, right, "R"))
        return out


class LocalTransport:
    """Virtual ranks in one process: each send buffer is copied into the
    matching receive buffer of the destination rank (device to device)."""

    def exchange(self, ranks, pairs, kind):
        for src, dst, side in pairs:
            send = ranks[src].bufs[kind]["send" + side]
            recv = ranks[dst].bufs[kind]["recv" + ("R" if side == "L" else "L")]
            recv.copy_(send, non_blocking=True)


class DistTransport:
    """One rank per process: batched P2P over torch.distributed (NCCL on GPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, ranks, pairs, kind):
        dist = self.dist
        (me,) = ranks.keys()
        st = ranks[me]
        ops = []
        for src, dst, side in pairs:
            if src == me:
                ops.append(dist.P2POp(dist.isend, st.bufs[kind]["send" + side], dst, self.group))
            if dst == me:
                ops.append(dist.P2POp(dist.irecv, st.bufs[kind]["recv" + ("R" if side == "L" else "L")], src,
                                      self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()


class RankState:
    """One rank: its grid, particle arrays with a device count, exchange buffers."""

    def __init__(self, rank, part, desc, fields, grid_leaf, ptr_level, particles, capacity, halo_cap, mig_cap,
                 device, stream=None):
        import torch
        self.rank, self.part = rank, part
        self.grid = sg.Grid(desc, device=device.index or 0, stream=stream)
        self.fields = fields
        self.leaf, self.ptr_level = grid_leaf, ptr_level
        n = particles["x"].shape[1]
        self.capacity = capacity
        dev = device

        def arr(ncomp, dtype=torch.float32):
            return torch.zeros((ncomp, capacity), dtype=dtype, device=dev)

        self.x, self.v, self.C, self.J = arr(3), arr(3), arr(9), arr(1)
        self.id = arr(1, torch.int32)
        self.count = torch.zeros(4, dtype=torch.int32, device=dev)
        self.x[:, :n] = torch.as_tensor(particles["x"], device=dev)
        self.v[:, :n] = torch.as_tensor(particles["v"], device=dev)
        self.C[:, :n] = torch.as_tensor(particles["C"], device=dev)
        self.J[:, :n] = torch.as_tensor(particles["J"], device=dev)
        self.id[:, :n] = torch.as_tensor(particles["id"], device=dev)
        self.count[0] = n
        g = self.grid
        self.a = [g.register_array(t, t.shape[0]) for t in (self.x, self.v, self.C, self.J, self.id)]
        for a in self.a:
            sg.set_array_count(g, a, self.count)
        # exchange buffers: int32 tensors, word 0 = record count, records from word 4
        blk_words = 4 + 4 * 64
        self.halo_rec = blk_words
        self.bufs = {"halo": {}, "part": {}}
        self.buf_ids = {"halo": {}, "part": {}}
        for kind, cap_words in (("halo", halo_cap * blk_words), ("part", mig_cap * PREC_WORDS)):
            for name in ("sendL", "sendR", "recvL", "recvR"):
                t = torch.zeros(4 + cap_words, dtype=torch.int32, device=dev)
                self.bufs[kind][name] = t
                i = g.register_array(t[4:], 1)
                sg.set_array_count(g, i, t[:1])
                self.buf_ids[kind][name] = i
        self.halo_cap = halo_cap

    def n(self):
        return int(self.count[0].item())


class SlabMPM:
    """C5-style sharded MPM over G ranks (virtual or real)."""

    def __init__(self, n_grid, ptr_cells, particles, world, ranks_here, transport, prm, device_of,
                 capacity_factor=1.5, halo_cap=2048, mig_cap=16384, streams=None):
        import workloads as W
        self.world = world
        self.prm = prm
        self.part = SlabPartition(n_grid, ptr_cells, world)
        L, lv = W.c5_layout(n_grid, ptr_cells)
        self.L, self.lv = L, lv
        f = L.fields
        self.gf = [f["vx"], f["vy"], f["vz"], f["m"]]
        ids = np.arange(particles["x"].shape[1], dtype=np.int32)
        cells = np.floor(particles["x"][0].astype(np.float32) * np.float32(prm["inv_dx"])).astype(np.int64)
        own = self.part.owner(cells)
        n_total = particles["x"].shape[1]
        cap = int(capacity_factor * n_total / world) + mig_cap
        self.ranks = {}
        for r in ranks_here:
            sel = own == r
            p = {k: np.ascontiguousarray(v[:, sel]) for k, v in particles.items()}
            p["id"] = ids[sel][None]
            self.ranks[r] = RankState(r, self.part, L.desc(), self.gf, lv[-1], lv[0], p, cap, halo_cap, mig_cap,
                                      device_of(r), None if streams is None else streams[r])
        self.transport = transport
        self.pairs = self.part.exchange_pairs()

    # --- enqueue helpers -----------------------------------------------------
    def _pack(self, st, layers):
        """Reset the send counts and pack the given (left, right) layers."""
        g = st.grid
        nbs = self.part.neighbours(st.rank)
        ids = st.buf_ids["halo"]
        for side, nb, rng in (("L", nbs[0], layers[0]), ("R", nbs[1], layers[1])):
            if nb is None:
                continue
            g.task(sg.TASK_SERIAL, "ARRAY_COUNT", arrays=[ids["send" + side]], params=[0.0])
            g.task(sg.TASK_STRUCT_FOR, "HALO_PACK", st.leaf, self.gf, [ids["send" + side]],
                   [float(rng[0]), float(rng[1]), float(st.halo_cap)])

    def _unpack(self, st, mode):
        g = st.grid
        nbs = self.part.neighbours(st.rank)
        ids = st.buf_ids["halo"]
        for side, nb in (("L", nbs[0]), ("R", nbs[1])):
            if nb is not None:
                g.task(sg.TASK_RANGE_FOR, "HALO_UNPACK", -1, self.gf, [ids["recv" + side]], [float(mode)],
                       [True] * 4, n=0)

    # --- one MPM step on every local rank -------------------------------------
    def step(self):
        prm = self.prm
        stats = []
        # phase 1: P2G with ghost contributions, pack ghost layers
        for st in self.ranks.values():
            g = st.grid
            g.clear(st.ptr_level, sg.DEACTIVATE)
            g.range_for("P2G", -1, self.gf, st.a[:4],
                        [prm["dt"], prm["inv_dx"], prm["p_mass"], prm["p_vol"], prm["E"]], [True] * 4)
            self._pack(st, self.part.ghost_layers(st.rank))
            stats.append(g.flush("all"))
        self.transport.exchange(self.ranks, self.pairs, "halo")          # halo reduce
        # phase 2: add received ghost contributions, grid update, pack boundary layers
        for st in self.ranks.values():
            g = st.grid
            self._unpack(st, 0)
            g.struct_for("GRID_OP", st.leaf, self.gf, [prm["dt"], prm["gravity"], prm["bound"], prm["n_grid"]])
            self._pack(st, self.part.boundary_layers(st.rank))
            stats.append(g.flush("all"))
        self.transport.exchange(self.ranks, self.pairs, "halo")          # halo fill
        # phase 3: overwrite ghost layers, G2P + compaction + migration packing
        for st in self.ranks.values():
            g = st.grid
            self._unpack(st, 1)
            pid = st.buf_ids["part"]
            for side in ("L", "R"):
                g.task(sg.TASK_SERIAL, "ARRAY_COUNT", arrays=[pid["send" + side]], params=[0.0])
            lo, hi = self.part.lo[st.rank], self.part.hi[st.rank]
            lo_f = -1e9 if st.rank == 0 else float(lo)
            hi_f = 1e9 if st.rank == self.world - 1 else float(hi)
            g.task(sg.TASK_RANGE_FOR, "G2P_MIGRATE", -1, self.gf, st.a + [pid["sendL"], pid["sendR"]],
                   [prm["dt"], prm["inv_dx"], lo_f, hi_f], n=-1)
            stats.append(g.flush("all"))
        if self.world > 1:
            self.transport.exchange(self.ranks, self.pairs, "part")      # migration
            for st in self.ranks.values():
                pid = st.buf_ids["part"]
                st.grid.task(sg.TASK_RANGE_FOR, "MIGRATE_APPEND", -1, [], st.a + [pid["recvL"], pid["recvR"]],
                             n=0)
                stats.append(st.grid.flush("all"))
        return stats

    # --- inspection (tests) --------------------------------------------------
    def gather_particles(self):
        """All particles sorted by id: dict of (ncomp, N) numpy arrays."""
        parts = {k: [] for k in ("x", "v", "C", "J", "id")}
        for st in self.ranks.values():
            st.grid.sync()
            n = st.n()
            for k in parts:
                parts[k].append(getattr(st, k)[:, :n].cpu().numpy())
        out = {k: np.concatenate(v, axis=1) for k, v in parts.items()}
        order = np.argsort(out["id"][0])
        return {k: v[:, order] for k, v in out.items()}

    def gather_field(self, name):
        """Owned slabs of every rank stitched into one dense array."""
        fid = self.L.fields[name]
        out = None
        for st in self.ranks.values():
            d = st.grid.field(fid)
            if out is None:
                out = np.zeros_like(d)
            lo, hi = self.part.lo[st.rank], self.part.hi[st.rank]
            out[lo:hi] = d[lo:hi]
        return out
