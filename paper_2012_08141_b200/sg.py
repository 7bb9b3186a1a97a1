"""Thin ctypes binding of libsg (include/sg.h).  Argument marshalling only:
every step of the hot path runs in the CUDA kernels behind the C-ABI.

PyTorch supplies device memory (caching-allocator callbacks), the stream and,
for multi-GPU runs, process groups.  If libsg.so is missing this module raises
at import: there is no CPU fallback.
"""
from __future__ import annotations

import atexit
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SG_LIB_PATH: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("SG_LIB_PATH") or os.path.join(_HERE, "libsg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsg.so not built at {LIB_PATH}: run __graft_entry__.build() (no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)

# --- enums mirrored from include/sg.h -----------------------------------------
ROOT, DENSE, BITMASKED, POINTER, PLACE = 0, 1, 2, 3, 4
F32, I32 = 0, 1
TASK_STRUCT_FOR, TASK_RANGE_FOR, TASK_SERIAL = 0, 1, 2
OPS = {"FILL": 1, "ADD_CONST": 2, "INC": 3, "AXPY": 4, "STENCIL": 5, "JACOBI": 6, "REDUCE_SUM": 7,
       "DOWNSAMPLE": 8, "JITTER": 9, "CLEAR_SCALAR": 10, "ARRAY_COUNT": 11, "P2G": 20, "GRID_OP": 21, "G2P": 22,
       "HALO_PACK": 23, "HALO_UNPACK": 24, "G2P_MIGRATE": 25, "MIGRATE_APPEND": 26,
       "LOSS_MEAN": 27, "ADJ_INIT": 28, "G2P_ADJ": 29, "P2G_ADJ": 30,
       "SMOOTH_RB": 31, "RESTRICT": 32, "PROLONG": 33, "RESID_NORM2": 34,
       "DOT": 35, "AXPY_RATIO": 36, "XPAY_RATIO": 37, "COPY_SCALAR": 38,
       "DIST_SIGNAL": 40, "DIST_WAIT": 41, "PERMUTE": 42, "MIGRATE_COMPACT": 43}
CLEAR_VALUES, DEACTIVATE = 0, 1
PASS_LISTGEN_REMOVAL, PASS_ACT_DEMOTION, PASS_FUSION, PASS_DSE = 1, 2, 4, 8
PASS_ALL = 15
PASS_CHAIN = 16
PASS_NAMES = {"none": 0, "all": 15, "listgen": 1, "demotion": 2, "fusion": 4, "dse": 8, "chain": 16}
ERRORS = {0: "OK", -1: "ARG", -2: "LAYOUT", -3: "RANGE", -4: "CUDA", -5: "NCCL", -6: "DEMOTION_TRAP",
          -7: "OVERFLOW", -8: "POOL_EXHAUSTED", -9: "LIST_OVERFLOW", -10: "STATE", -11: "TIMEOUT"}
TASK_TYPES = ["activate", "listgen", "clear_list", "struct_for", "range_for", "serial", "deactivate"]


class SnodeDesc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("parent", ctypes.c_int32), ("ndim", ctypes.c_int32),
                ("extent", ctypes.c_int32 * 3), ("dtype", ctypes.c_int32)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("debug", ctypes.c_int32), ("plan_only", ctypes.c_int32),
                ("lowering", ctypes.c_int32), ("stream", ctypes.c_void_p), ("alloc", ALLOC_FN),
                ("free", FREE_FN), ("alloc_ctx", ctypes.c_void_p), ("pool_capacity", ctypes.c_int64),
                ("list_capacity", ctypes.c_int64), ("dist_halo_words", ctypes.c_int64),
                ("dist_part_words", ctypes.c_int64)]


class Task(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("op", ctypes.c_int32), ("snode", ctypes.c_int32),
                ("pad_", ctypes.c_int32), ("range_n", ctypes.c_int64), ("fields", ctypes.c_int32 * 8),
                ("arrays", ctypes.c_int32 * 8), ("activating", ctypes.c_uint32), ("params", ctypes.c_float * 8)]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "tasks_lowered", "launches", "listgen_launched", "clear_list_launched", "listgens_removed",
        "demotions", "tasks_fused", "dead_removed", "plan_cache_hits", "plan_cache_misses")] + [
        ("plan_us", ctypes.c_double), ("tasks_chained", ctypes.c_int64), ("launches_chained", ctypes.c_int64),
        ("aux_kernels", ctypes.c_int64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_P = ctypes.POINTER
_vp = ctypes.c_void_p
_lib.sg_create.argtypes = [_P(SnodeDesc), ctypes.c_int32, _P(Opts), _P(_vp)]
_lib.sg_destroy.argtypes = [_vp]
_lib.sg_register_array.argtypes = [_vp, _vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _P(ctypes.c_int32)]
_lib.sg_activate.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.c_int64]
_lib.sg_listgen.argtypes = [_vp, ctypes.c_int32]
_lib.sg_struct_for.argtypes = [_vp, _P(Task)]
_lib.sg_clear.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32]
_lib.sg_flush.argtypes = [_vp, ctypes.c_uint32, _P(ctypes.c_int32), ctypes.c_int32, _P(Stats)]
_lib.sg_sync.argtypes = [_vp]
_lib.sg_export_mask.argtypes = [_vp, ctypes.c_int32, _P(ctypes.c_int32), ctypes.c_int64, _P(ctypes.c_int64)]
_lib.sg_export_list.argtypes = [_vp, ctypes.c_int32, _P(ctypes.c_int32), ctypes.c_int64, _P(ctypes.c_int64)]
_lib.sg_read_field.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.c_int64]
_lib.sg_load_field.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.c_int64]
_lib.sg_last_plan.argtypes = [_vp, _P(ctypes.c_int32), ctypes.c_int64, _P(ctypes.c_int64)]
_lib.sg_device_info.argtypes = [_vp, _P(ctypes.c_int64), ctypes.c_int32]
_lib.sg_last_error.restype = ctypes.c_char_p
for _n in ("sg_create", "sg_destroy", "sg_register_array", "sg_activate", "sg_listgen", "sg_struct_for", "sg_clear",
           "sg_flush", "sg_sync", "sg_export_mask", "sg_export_list", "sg_read_field", "sg_load_field",
           "sg_last_plan", "sg_device_info"):
    getattr(_lib, _n).restype = ctypes.c_int32

EXPORTS = ["sg_create", "sg_destroy", "sg_register_array", "sg_activate", "sg_listgen", "sg_struct_for", "sg_clear",
           "sg_flush", "sg_sync", "sg_export_mask", "sg_export_list", "sg_read_field", "sg_load_field",
           "sg_last_plan", "sg_device_info", "sg_last_error"]


class SgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"sg {ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


def _check(rc):
    if rc != 0:
        raise SgError(rc, _lib.sg_last_error().decode())


def passes_mask(p):
    if isinstance(p, int):
        return p
    if isinstance(p, str):
        m = 0
        for part in p.split("+"):
            m |= PASS_NAMES[part]
        return m
    raise ValueError(p)


_torch_alloc_keep = []


def _torch_allocators(device):
    import torch

    @ALLOC_FN
    def _alloc(ctx, nbytes, stream):
        # the grid's own device, not the caller's current one (lazy allocations
        # inside sg_flush of a grid on another device)
        return torch.cuda.caching_allocator_alloc(int(nbytes), device, stream)

    @FREE_FN
    def _free(ctx, ptr, stream):
        torch.cuda.caching_allocator_delete(ptr)

    _torch_alloc_keep.append((_alloc, _free))
    return _alloc, _free


class Grid:
    """One sparse grid behind the C-ABI."""

    def __init__(self, desc, device=0, stream=None, plan_only=False, debug=False, faithful=False,
                 pool_capacity=0, list_capacity=0, torch_alloc=True, dist_halo_words=0, dist_part_words=0):
        d = np.ascontiguousarray(desc, dtype=np.int32)
        self.desc = d
        rows = (SnodeDesc * len(d))()
        for i, r in enumerate(d):
            rows[i].kind, rows[i].parent, rows[i].ndim = int(r[0]), int(r[1]), int(r[2])
            for a in range(3):
                rows[i].extent[a] = int(r[3 + a])
            rows[i].dtype = int(r[6])
        o = Opts()
        o.device = device
        o.debug = int(debug)
        o.plan_only = int(plan_only)
        o.lowering = int(faithful)
        o.pool_capacity = pool_capacity
        o.list_capacity = list_capacity
        o.dist_halo_words = dist_halo_words
        o.dist_part_words = dist_part_words
        self._keep = []         # borrowed device buffers kept alive until the flush ran
        self._keep_prev = []
        if not plan_only:
            import torch
            if stream is None:
                stream = torch.cuda.current_stream(device).cuda_stream
            o.stream = stream
            if torch_alloc:
                a, f = _torch_allocators(device)
                o.alloc, o.free = a, f
        self.plan_only = plan_only
        h = _vp()
        _check(_lib.sg_create(rows, len(d), ctypes.byref(o), ctypes.byref(h)))
        self.h = h
        self._derive()

    def _derive(self):
        d = self.desc
        self.places = [i for i in range(len(d)) if d[i][0] == PLACE]
        self.parent = d[:, 1].tolist()

    def close(self):
        if getattr(self, "h", None):
            _lib.sg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- enqueue ---
    def register_array(self, tensor, ncomp):
        i = ctypes.c_int32()
        n = tensor.numel() // ncomp
        dt = I32 if str(tensor.dtype) == "torch.int32" else F32
        self._keep.append(tensor)
        _check(_lib.sg_register_array(self.h, _vp(tensor.data_ptr()), n, dt, ncomp, ctypes.byref(i)))
        return i.value

    def register_array_plan(self, n, ncomp):
        """Plan-only grids: an array id without memory (planner tests)."""
        i = ctypes.c_int32()
        _check(_lib.sg_register_array(self.h, None, n, F32, ncomp, ctypes.byref(i)))
        return i.value

    def activate(self, field, coords):
        """coords: int32 (n, ndim) on the device (torch tensor), or numpy for plan-only grids."""
        if hasattr(coords, "data_ptr"):
            ptr, n = coords.data_ptr(), coords.shape[0]
        else:
            ptr, n = coords.ctypes.data, coords.shape[0]
        self._keep.append(coords)
        _check(_lib.sg_activate(self.h, field, _vp(ptr), n))

    def listgen(self, snode):
        _check(_lib.sg_listgen(self.h, snode))

    def task(self, kind, op, snode=-1, fields=(), arrays=(), params=(), activating=(), n=0):
        # marshalled descriptors are memoized: repeated launches (solver loops)
        # cost one ctypes call
        key = (kind, op, snode, tuple(fields), tuple(arrays), tuple(params), tuple(activating), n)
        cache = self.__dict__.setdefault("_task_cache", {})
        t = cache.get(key)
        if t is not None:
            _check(_lib.sg_struct_for(self.h, ctypes.byref(t)))
            return
        t = Task()
        t.kind = kind
        t.op = OPS[op] if isinstance(op, str) else op
        t.snode = snode
        t.range_n = n
        for i in range(8):
            t.fields[i] = fields[i] if i < len(fields) else -1
            t.arrays[i] = arrays[i] if i < len(arrays) else -1
            t.params[i] = params[i] if i < len(params) else 0.0
        t.activating = sum(1 << i for i, a in enumerate(activating) if a)
        if len(cache) < 65536:
            cache[key] = t
        _check(_lib.sg_struct_for(self.h, ctypes.byref(t)))

    def struct_for(self, op, snode, fields, params=(), activating=()):
        self.task(TASK_STRUCT_FOR, op, snode, fields, (), params, activating)

    def range_for(self, op, n, fields=(), arrays=(), params=(), activating=()):
        self.task(TASK_RANGE_FOR, op, -1, fields, arrays, params, activating, n)

    def serial(self, op, fields, params=()):
        self.task(TASK_SERIAL, op, -1, fields, (), params)

    def clear(self, target, mode):
        _check(_lib.sg_clear(self.h, target, mode))

    def flush(self, passes="all", observed=None):
        st = Stats()
        if observed is None:
            _check(_lib.sg_flush(self.h, passes_mask(passes), None, -1, ctypes.byref(st)))
        else:
            ob = (ctypes.c_int32 * max(1, len(observed)))(*observed)
            _check(_lib.sg_flush(self.h, passes_mask(passes), ob, len(observed), ctypes.byref(st)))
        # buffers of the previous window can go once this flush is ordered after them
        self._keep_prev = self._keep
        self._keep = []
        return st.as_dict()

    def sync(self):
        _check(_lib.sg_sync(self.h))
        self._keep_prev = []

    # --- exports ---
    def _ndim(self, snode):
        return int(self.desc[snode][2])

    def mask(self, snode):
        n = ctypes.c_int64()
        _check(_lib.sg_export_mask(self.h, snode, None, 0, ctypes.byref(n)))
        nd = self._ndim(snode)
        out = np.zeros((max(n.value, 1), nd), dtype=np.int32)
        _check(_lib.sg_export_mask(self.h, snode, out.ctypes.data_as(_P(ctypes.c_int32)), n.value, ctypes.byref(n)))
        return out[: n.value]

    def list(self, snode):
        n = ctypes.c_int64()
        _check(_lib.sg_export_list(self.h, snode, None, 0, ctypes.byref(n)))
        nd = self._ndim(snode)
        out = np.zeros((max(n.value, 1), nd), dtype=np.int32)
        _check(_lib.sg_export_list(self.h, snode, out.ctypes.data_as(_P(ctypes.c_int32)), n.value, ctypes.byref(n)))
        return out[: n.value]

    def field_shape(self, f):
        row = self.places[f]
        nd = int(self.desc[row][2])
        s = [1, 1, 1]
        x = self.parent[row]
        while x > 0:
            for a in range(3):
                s[a] *= int(self.desc[x][3 + a])
            x = self.parent[x]
        return tuple(s[:nd])

    def field_dtype(self, f):
        return np.int32 if int(self.desc[self.places[f]][6]) == I32 else np.float32

    def field(self, f):
        shape = self.field_shape(f)
        out = np.zeros(shape if shape else (), dtype=self.field_dtype(f))
        _check(_lib.sg_read_field(self.h, f, _vp(out.ctypes.data), out.nbytes))
        return out

    def load_field(self, f, dense):
        a = np.ascontiguousarray(dense, dtype=self.field_dtype(f))
        _check(_lib.sg_load_field(self.h, f, _vp(a.ctypes.data), a.nbytes))

    def last_plan(self):
        n = ctypes.c_int64()
        _check(_lib.sg_last_plan(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros((max(n.value, 1), 6), dtype=np.int32)
        _check(_lib.sg_last_plan(self.h, out.ctypes.data_as(_P(ctypes.c_int32)), n.value, ctypes.byref(n)))
        return out[: n.value]

    def device_info(self):
        out = (ctypes.c_int64 * 64)()
        _check(_lib.sg_device_info(self.h, out, 64))
        return list(out)


def replay(grid, prog, passes=None, device="cuda", upto=None, on_flush=None):
    """Replay a workloads program through the C-ABI.  `passes` overrides every
    flush's pass set when given.  Returns the list of per-flush stats."""
    import torch
    stats = []
    grid.tensors = {}
    for name, arr in prog.get("arrays", {}).items():
        if grid.plan_only:
            continue
        t = torch.as_tensor(arr).to(device).contiguous()
        grid.tensors[name] = t
        grid.register_array(t, arr.shape[0])
    calls = prog["calls"] if upto is None else prog["calls"][:upto]
    for c in calls:
        k = c["call"]
        if k == "activate":
            co = c["coords"]
            if not grid.plan_only:
                co = torch.as_tensor(co).to(device).contiguous()
            grid.activate(c["field"], co)
        elif k == "struct_for":
            grid.struct_for(c["op"], c["snode"], c["fields"], c.get("params", []), c.get("activating", []))
        elif k == "range_for":
            grid.range_for(c["op"], c["n"], c["fields"], c.get("arrays", []), c.get("params", []),
                           c.get("activating", []))
        elif k == "serial":
            grid.serial(c["op"], c["fields"], c.get("params", []))
        elif k == "clear":
            grid.clear(c["target"], CLEAR_VALUES if c["mode"] == "values" else DEACTIVATE)
        elif k == "listgen":
            grid.listgen(c["snode"])
        elif k == "flush":
            st = grid.flush(c["passes"] if passes is None else passes, c.get("observed"))
            stats.append(st)
            if on_flush:
                on_flush(grid, st)
    return stats


def run_program(prog, passes=None, device=0, plan_only=False, **kw):
    g = Grid(prog["desc"], device=device, plan_only=plan_only, **kw)
    st = replay(g, prog, passes=passes, device=f"cuda:{device}" if not plan_only else None)
    if not plan_only:
        g.sync()
    return g, st


_lib.sg_set_profiling.argtypes = [_vp, ctypes.c_int32]
_lib.sg_set_profiling.restype = ctypes.c_int32
_lib.sg_profile_read.argtypes = [_vp, _P(ctypes.c_double), _P(ctypes.c_int64), ctypes.c_int32]
_lib.sg_profile_read.restype = ctypes.c_int32
_lib.sg_set_array_count.argtypes = [_vp, ctypes.c_int32, _vp]
_lib.sg_set_array_count.restype = ctypes.c_int32
EXPORTS += ["sg_set_profiling", "sg_profile_read", "sg_set_array_count"]

_lib.sg_struct_for_batch.argtypes = [_vp, _vp, ctypes.c_int32]
_lib.sg_struct_for_batch.restype = ctypes.c_int32
_lib.sg_read_scalar_async.argtypes = [_vp, ctypes.c_int32, _vp]
_lib.sg_read_scalar_async.restype = ctypes.c_int32
EXPORTS += ["sg_struct_for_batch", "sg_read_scalar_async"]


class Batch:
    """A marshalled task list submitted with one library call (sg_struct_for_batch):
    for loops that re-enqueue the same tasks every step."""

    def __init__(self, tasks):
        self.n = len(tasks)
        self.arr = (Task * max(1, self.n))(*tasks)


def make_batch(grid, calls):
    """Marshal workloads-style task calls (struct_for / range_for / serial) into a Batch."""
    tasks = []
    for c in calls:
        k = c["call"]
        kind = {"struct_for": TASK_STRUCT_FOR, "range_for": TASK_RANGE_FOR, "serial": TASK_SERIAL}[k]
        t = Task()
        t.kind = kind
        t.op = OPS[c["op"]]
        t.snode = c.get("snode", -1) if k == "struct_for" else -1
        t.range_n = c.get("n", 0) if k == "range_for" else 0
        fields, arrays, params = c.get("fields", []), c.get("arrays", []), c.get("params", [])
        for i in range(8):
            t.fields[i] = fields[i] if i < len(fields) else -1
            t.arrays[i] = arrays[i] if i < len(arrays) else -1
            t.params[i] = params[i] if i < len(params) else 0.0
        t.activating = sum(1 << i for i, a in enumerate(c.get("activating", [])) if a)
        tasks.append(t)
    return Batch(tasks)


def submit(grid, batch):
    _check(_lib.sg_struct_for_batch(grid.h, ctypes.cast(batch.arr, _vp), batch.n))


def read_scalar_async(grid, field, pinned):
    """Enqueue the D2H copy of a 0-D field into a pinned torch tensor (4 bytes)."""
    _check(_lib.sg_read_scalar_async(grid.h, field, _vp(pinned.data_ptr())))


def set_array_count(grid, array_id, count_tensor):
    """Attach a device int32 count (a torch tensor element) to a registered array."""
    grid._keep.append(count_tensor)
    _check(_lib.sg_set_array_count(grid.h, array_id, _vp(count_tensor.data_ptr())))

PROFILE_KINDS = 400


def set_profiling(grid, on=True):
    _check(_lib.sg_set_profiling(grid.h, int(on)))


def profile_read(grid):
    """{kind: (total_ms, launches)}; kinds 0..6 task types, 100+op struct-for ops,
    200+snode listgens, 300+op range-for ops."""
    ms = (ctypes.c_double * PROFILE_KINDS)()
    cnt = (ctypes.c_int64 * PROFILE_KINDS)()
    _check(_lib.sg_profile_read(grid.h, ms, cnt, PROFILE_KINDS))
    return {k: (ms[k], cnt[k]) for k in range(PROFILE_KINDS) if cnt[k]}


# --- multi-GPU data plane (include/sg.h sg_dist_init) ---------------------------
_lib.sg_dist_init.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32]
_lib.sg_dist_init.restype = ctypes.c_int32
_lib.sg_dist_info.argtypes = [_vp, _P(ctypes.c_int32), ctypes.c_int32]
_lib.sg_dist_info.restype = ctypes.c_int32
_lib.sg_nccl_unique_id.argtypes = [_vp]
_lib.sg_nccl_unique_id.restype = ctypes.c_int32
_lib.sg_dist_peer_info.argtypes = [_vp, _vp]
_lib.sg_dist_peer_info.restype = ctypes.c_int32
_lib.sg_dist_connect.argtypes = [_vp, _vp]
_lib.sg_dist_connect.restype = ctypes.c_int32
EXPORTS += ["sg_dist_init", "sg_dist_info", "sg_nccl_unique_id", "sg_dist_peer_info", "sg_dist_connect"]
TRANSPORTS = {0: "none", 1: "peer", 2: "nccl"}
DIST_KINDS = {"halo_reduce": 0, "halo_fill": 1, "part": 2}


def nccl_unique_id():
    """128 bytes (ncclGetUniqueId) for rank 0 to broadcast to the other ranks."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.sg_nccl_unique_id(buf))
    return buf.raw


def dist_init(grid, rank, world, nccl_uid=None, axis=0):
    """sg_dist_init: nccl_uid (bytes) for one rank per process, None for an
    in-process group of virtual ranks (call for ranks 0..world-1 in order)."""
    if nccl_uid is None:
        _check(_lib.sg_dist_init(grid.h, rank, world, None, axis))
    else:
        buf = ctypes.create_string_buffer(bytes(nccl_uid), 128)
        _check(_lib.sg_dist_init(grid.h, rank, world, buf, axis))


def dist_peer_info(grid):
    """256-byte connection blob of this rank (after dist_init with nccl_uid=None)."""
    buf = ctypes.create_string_buffer(256)
    _check(_lib.sg_dist_peer_info(grid.h, buf))
    return buf.raw


def dist_connect(grid, blobs):
    """Map the neighbours' exchange arenas from every rank's blob (rank order)."""
    data = b"".join(bytes(b) for b in blobs)
    buf = ctypes.create_string_buffer(data, len(data))
    _check(_lib.sg_dist_connect(grid.h, buf))


def dist_info(grid):
    """{'transport', 'rank', 'world', 'axis', 'send': {(kind, side): id}, 'recv': {...}}"""
    out = (ctypes.c_int32 * 16)()
    _check(_lib.sg_dist_info(grid.h, out, 16))
    v = list(out)
    return {"transport": TRANSPORTS.get(v[0], v[0]), "rank": v[1], "world": v[2], "axis": v[3],
            "send": {(k, s): v[4 + 2 * k + s] for k in range(3) for s in range(2)},
            "recv": {(k, s): v[10 + 2 * k + s] for k in range(3) for s in range(2)}}


_lib.sg_jit_info.argtypes = [_P(ctypes.c_int64), ctypes.c_int32]
_lib.sg_jit_info.restype = ctypes.c_int32
EXPORTS += ["sg_jit_info"]


def jit_info():
    """{mode, ready, compiling, failed, hits, misses, compile_ms} of the NVRTC-specialized kernels."""
    out = (ctypes.c_int64 * 7)()
    _check(_lib.sg_jit_info(out, 7))
    v = list(out)
    return {"mode": v[0], "ready": v[1], "compiling": v[2], "failed": v[3], "hits": v[4], "misses": v[5],
            "compile_ms": v[6] / 1000.0}

_lib.sg_jit_selftest.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P(ctypes.c_int32), ctypes.c_int32,
                                 ctypes.c_char_p, ctypes.c_int64]
_lib.sg_jit_selftest.restype = ctypes.c_int32
_lib.sg_jit_set_mode.argtypes = [ctypes.c_int32]
_lib.sg_jit_set_mode.restype = ctypes.c_int32
_lib.sg_jit_shutdown.argtypes = []
_lib.sg_jit_shutdown.restype = ctypes.c_int32
EXPORTS += ["sg_jit_selftest", "sg_jit_set_mode", "sg_jit_shutdown"]


def jit_shutdown():
    """Stop the JIT (drop queued compiles, wait for in-flight ones): NVRTC's
    exit-time teardown under a running compile crashes the process."""
    _check(_lib.sg_jit_shutdown())


# Python atexit hooks run before any C exit handler (include/sg.h)
atexit.register(jit_shutdown)


def jit_set_mode(mode):
    """0 off, 1 asynchronous, 2 synchronous, -1 back to SG_JIT."""
    _check(_lib.sg_jit_set_mode(int(mode)))


def jit_selftest(ops, nd=3, gl=1, i32=False):
    """NVRTC-compile (no GPU) a specialized kernel for the op names; returns (ok, log)."""
    arr = (ctypes.c_int32 * len(ops))(*[OPS[o] for o in ops])
    log = ctypes.create_string_buffer(1 << 16)
    rc = _lib.sg_jit_selftest(nd, gl, int(i32), arr, len(ops), log, len(log))
    return rc == 0, log.value.decode(errors="replace")
