"""x-slab partitioner for sparse MLS-MPM across GPUs.

Rank g of G owns the pointer-cell x-slab [g*Px/G, (g+1)*Px/G) of the grid and
the particles whose cell x lies in it.  Every step, in libsg tasks only:

  1. DEACTIVATE, P2G (activating) of the owned particles: contributions reach
     one leaf-block layer beyond each face (the ghost layers);
     HALO_PACK of the two ghost layers into the halo-reduce send buffers;
     DIST_SIGNAL(halo reduce).
  2. DIST_WAIT(halo reduce); HALO_UNPACK add (activating) of what the
     neighbours packed; GRID_OP; HALO_PACK of the two boundary layers;
     DIST_SIGNAL(halo fill).
  3. DIST_WAIT(halo fill); HALO_UNPACK store into the ghost layers;
     G2P into the rank's second particle state set in the binned kernels'
     order (bin-order storage: the next step's particle reads are sequential),
     PERMUTE of the ids, MIGRATE_COMPACT: leavers packed into the migration
     send buffers and their slots refilled from the tail; DIST_SIGNAL(migration).
  4. DIST_WAIT(migration); MIGRATE_APPEND of the received particles.

The library moves the bytes (sg_dist_init, include/sg.h): on the peer
transport the send buffers ARE the neighbours' receive buffers (NVLink peer
memory, or the same allocation for virtual ranks), so packing kernels store
straight into the neighbour and only device flags synchronize; on the NCCL
transport DIST_WAIT is an ncclSend/ncclRecv pair per neighbour.  This module
holds only the partition arithmetic and the task sequence.
"""
from __future__ import annotations

import numpy as np

from . import sg

PREC_WORDS = 17   # particle record: x3 v3 C9 J1 id1 (exchange_ops.cuh)
HALO, FILL, PART = 0, 1, 2   # exchange kinds (sg_dist_init)


class SlabPartition:
    """Pure arithmetic of the decomposition (tested on CPU)."""

    def __init__(self, n_grid, ptr_cells_x, world, block=4):
        if ptr_cells_x % world:
            raise ValueError(f"{ptr_cells_x} pointer slabs do not split over {world} ranks")
        self.n_grid, self.world, self.block = n_grid, world, block
        self.ptr_cells_x = ptr_cells_x
        per = ptr_cells_x // world
        cells_per_ptr = n_grid // ptr_cells_x
        self.lo = [r * per * cells_per_ptr for r in range(world)]
        self.hi = [(r + 1) * per * cells_per_ptr for r in range(world)]
        self.ptr_slabs = [list(range(r * per, (r + 1) * per)) for r in range(world)]

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

    def migration_bounds(self, r):
        """Cell-x bounds of G2P_MIGRATE: particles whose cell x leaves [lo, hi)
        go left / right (open-ended at the outer ranks)."""
        lo = -1e9 if r == 0 else float(self.lo[r])
        hi = 1e9 if r == self.world - 1 else float(self.hi[r])
        return lo, hi


def halo_record_words(n_fields=4, block_cells=64):
    return 4 + n_fields * block_cells


class RankState:
    """One rank: its grid (with the library's exchange buffers), particle
    arrays with a device count."""

    def __init__(self, rank, part, desc, fields, grid_leaf, ptr_level, particles, capacity, halo_cap, mig_cap,
                 device, stream=None, plan_only=False):
        self.rank, self.part = rank, part
        self.halo_cap, self.mig_cap = halo_cap, mig_cap
        self.grid = sg.Grid(desc, device=0 if plan_only else (device.index or 0), stream=stream,
                            plan_only=plan_only,
                            dist_halo_words=4 + halo_cap * halo_record_words(),
                            dist_part_words=4 + mig_cap * PREC_WORDS)
        self.fields = fields
        self.leaf, self.ptr_level = grid_leaf, ptr_level
        self.capacity = capacity
        self.plan_only = plan_only
        g = self.grid
        if plan_only:
            self.aset = [[g.register_array_plan(capacity, nc) for nc in (3, 3, 9, 1, 1)] for _ in range(2)]
            self.cur = 0
            return
        import torch
        n = particles["x"].shape[1]
        if n > capacity:
            raise ValueError(f"rank {rank}: {n} particles exceed the capacity {capacity}")
        dev = device

        def arr(ncomp, dtype=torch.float32):
            return torch.zeros((ncomp, capacity), dtype=dtype, device=dev)

        # two particle state sets: G2P writes the new state of set `cur` into the
        # other one in the binned kernels' order (bin-order storage, reading
        # R38); both share one device count
        self.count = torch.zeros(4, dtype=torch.int32, device=dev)
        self.sets, self.aset = [], []
        for k in range(2):
            st = {"x": arr(3), "v": arr(3), "C": arr(9), "J": arr(1), "id": arr(1, torch.int32)}
            if k == 0:
                for name in ("x", "v", "C", "J", "id"):
                    st[name][:, :n] = torch.as_tensor(np.ascontiguousarray(particles[name]), device=dev)
            ids = [g.register_array(t, t.shape[0]) for t in (st["x"], st["v"], st["C"], st["J"], st["id"])]
            for a in ids:
                sg.set_array_count(g, a, self.count)
            self.sets.append(st)
            self.aset.append(ids)
        self.count[0] = n
        self.cur = 0

    # the current particle state (set `cur`)
    @property
    def a(self):
        return self.aset[self.cur]

    @property
    def a_next(self):
        return self.aset[1 - self.cur]

    def __getattr__(self, name):
        if name in ("x", "v", "C", "J", "id"):
            return self.__dict__["sets"][self.__dict__["cur"]][name]
        raise AttributeError(name)

    def connect(self, world, nccl_uid=None):
        sg.dist_init(self.grid, self.rank, world, nccl_uid)

    def connect_ipc(self, world, group=None):
        """One rank per process without NCCL: exchange the connection blobs over
        torch.distributed (any backend) and map the neighbours' arenas."""
        import torch.distributed as dist
        sg.dist_init(self.grid, self.rank, world, None)
        blobs = [None] * world
        dist.all_gather_object(blobs, sg.dist_peer_info(self.grid), group=group)
        sg.dist_connect(self.grid, blobs)

    def ids(self):
        info = sg.dist_info(self.grid)
        self.transport = info["transport"]
        self.send, self.recv = info["send"], info["recv"]

    def n(self):
        return int(self.count[0].item())


class SlabMPM:
    """C5-style sharded MPM over G ranks.

    ranks_here: the ranks this process drives (all of them for virtual ranks on
    one GPU, [rank] for one rank per process).  connect: "local" (every rank in
    this process: an in-process group), "nccl" (nccl_uid = the 128-byte id
    every rank received; the library picks peer memory or NCCL send/recv), or
    "ipc" (one rank per process, connection blobs exchanged over the default
    torch.distributed group, peer memory through CUDA IPC).
    particles: the global particle dict (filtered by owner here) or a callable
    rank -> that rank's particles (dict with an "id" row)."""

    def __init__(self, n_grid, ptr_cells, particles, world, ranks_here, prm, device_of,
                 capacity_factor=1.5, halo_cap=2048, mig_cap=16384, streams=None, nccl_uid=None,
                 n_total=None, plan_only=False, connect=None):
        import workloads as W
        self.world = world
        self.prm = prm
        self.part = SlabPartition(n_grid, ptr_cells, world)
        L, lv = W.c5_layout(n_grid, ptr_cells)
        self.L, self.lv = L, lv
        f = L.fields
        self.gf = [f["vx"], f["vy"], f["vz"], f["m"]]
        local = {}
        if plan_only:
            local = {r: None for r in ranks_here}
            n_total = n_total or 0
        elif callable(particles):
            for r in ranks_here:
                local[r] = particles(r)
            if n_total is None:
                raise ValueError("n_total is needed with per-rank particle generators")
        else:
            n_total = particles["x"].shape[1]
            ids = np.arange(n_total, dtype=np.int32)
            cells = np.floor(particles["x"][0].astype(np.float32) * np.float32(prm["inv_dx"])).astype(np.int64)
            own = self.part.owner(cells)
            for r in ranks_here:
                sel = own == r
                p = {k: np.ascontiguousarray(v[:, sel]) for k, v in particles.items() if k != "id"}
                p["id"] = ids[sel][None]
                local[r] = p
        cap = int(capacity_factor * n_total / world) + mig_cap
        self.ranks = {}
        for r in ranks_here:
            self.ranks[r] = RankState(r, self.part, L.desc(), self.gf, lv[-1], lv[0], local[r], cap, halo_cap,
                                      mig_cap, None if plan_only else device_of(r),
                                      None if streams is None else streams[r], plan_only)
        # the library connects the neighbours (in-process group: ranks in order)
        if connect is None:
            connect = "nccl" if nccl_uid is not None else ("local" if len(self.ranks) == world else "ipc")
        self.connect_mode = connect
        for r in sorted(self.ranks):
            if connect == "ipc":
                self.ranks[r].connect_ipc(world)
            else:
                self.ranks[r].connect(world, nccl_uid if connect == "nccl" else None)
        for st in self.ranks.values():
            st.ids()

    # --- enqueue helpers -----------------------------------------------------
    def _xchg_arrays(self, st, kind):
        return [st.send[(kind, 0)], st.send[(kind, 1)], st.recv[(kind, 0)], st.recv[(kind, 1)]]

    def _pack(self, st, kind, layers):
        """Reset the send counts and pack the given (left, right) layers."""
        g = st.grid
        nbs = self.part.neighbours(st.rank)
        for side, nb, rng in ((0, nbs[0], layers[0]), (1, nbs[1], layers[1])):
            if nb is None:
                continue
            g.task(sg.TASK_SERIAL, "ARRAY_COUNT", arrays=[st.send[(kind, side)]], params=[0.0])
            g.task(sg.TASK_STRUCT_FOR, "HALO_PACK", st.leaf, self.gf, [st.send[(kind, side)]],
                   [float(rng[0]), float(rng[1]), float(st.halo_cap)])

    def _unpack(self, st, kind, mode):
        g = st.grid
        nbs = self.part.neighbours(st.rank)
        for side, nb in ((0, nbs[0]), (1, nbs[1])):
            if nb is not None:
                g.task(sg.TASK_RANGE_FOR, "HALO_UNPACK", -1, self.gf, [st.recv[(kind, side)]], [float(mode)],
                       [True] * 4, n=0)

    def _signal(self, st, kind):
        if self.world > 1:
            st.grid.task(sg.TASK_SERIAL, "DIST_SIGNAL", arrays=self._xchg_arrays(st, kind), params=[float(kind)])

    def _wait(self, st, kind):
        if self.world > 1:
            st.grid.task(sg.TASK_SERIAL, "DIST_WAIT", arrays=self._xchg_arrays(st, kind), params=[float(kind)])

    def phases(self, st):
        """The step as 4 enqueue functions; an exchange's SIGNAL ends a phase and
        its WAIT starts the next (virtual ranks flush between them)."""
        prm = self.prm

        def p1():
            g = st.grid
            g.clear(st.ptr_level, sg.DEACTIVATE)
            g.range_for("P2G", -1, self.gf, st.a[:4],
                        [prm["dt"], prm["inv_dx"], prm["p_mass"], prm["p_vol"], prm["E"]], [True] * 4)
            self._pack(st, HALO, self.part.ghost_layers(st.rank))
            self._signal(st, HALO)

        def p2():
            g = st.grid
            self._wait(st, HALO)
            self._unpack(st, HALO, 0)
            g.struct_for("GRID_OP", st.leaf, self.gf, [prm["dt"], prm["gravity"], prm["bound"], prm["n_grid"]])
            self._pack(st, FILL, self.part.boundary_layers(st.rank))
            self._signal(st, FILL)

        def p3():
            g = st.grid
            self._wait(st, FILL)
            self._unpack(st, FILL, 1)
            for side in (0, 1):
                g.task(sg.TASK_SERIAL, "ARRAY_COUNT", arrays=[st.send[(PART, side)]], params=[0.0])
            lo_f, hi_f = self.part.migration_bounds(st.rank)
            a, b = st.a, st.a_next
            # G2P into the other state set in bin order, ids along, then the
            # particles that left the slab are packed and their slots refilled
            g.task(sg.TASK_RANGE_FOR, "G2P", -1, self.gf, a[:4] + b[:4], [prm["dt"], prm["inv_dx"], 1.0], n=-1)
            g.task(sg.TASK_RANGE_FOR, "PERMUTE", -1, [self.gf[3]], [a[0], a[4], b[4]], [0.0, prm["inv_dx"]], n=-1)
            g.task(sg.TASK_RANGE_FOR, "MIGRATE_COMPACT", -1, [],
                   b + [st.send[(PART, 0)], st.send[(PART, 1)]], [0.0, prm["inv_dx"], lo_f, hi_f], n=-1)
            self._signal(st, PART)

        def p4():
            if self.world > 1:
                self._wait(st, PART)
                st.grid.task(sg.TASK_RANGE_FOR, "MIGRATE_APPEND", -1, [],
                             st.a_next + [st.recv[(PART, 0)], st.recv[(PART, 1)]], n=0)

        return [p1, p2, p3, p4]

    # --- one MPM step on every local rank -------------------------------------
    def step(self, fused=None):
        """fused: one flush per step per rank (one rank per process: every
        exchange is device-side, the whole step is one plan / one CUDA graph);
        default for a single local rank.  Otherwise (virtual ranks sharing a
        stream) each phase is flushed on every rank before the next starts."""
        if fused is None:
            fused = len(self.ranks) == 1
        stats = []
        if fused:
            for st in self.ranks.values():
                for ph in self.phases(st):
                    ph()
                stats.append(st.grid.flush("all"))
        else:
            per_rank = {r: self.phases(st) for r, st in self.ranks.items()}
            for k in range(4):
                if k == 3 and self.world == 1:
                    break
                for r, st in self.ranks.items():
                    per_rank[r][k]()
                    stats.append(st.grid.flush("all"))
        for st in self.ranks.values():
            st.cur = 1 - st.cur   # the new state lives in the other set
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
