"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain single-threaded executor of the UNOPTIMIZED lowered task stream
(PAPER.md:84-85 eager execution; "transparent to users").  The
arithmetic lives in ``sg_oracle.cpp`` (C++17, compiled with
-ffp-contract=off); this file only loads it, maps op names to the oracle's own
ids, and performs the paper's lowering of user calls into tasks
("kernels are decomposed into tasks"; "3 tasks per
such a small kernel").

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It shares no code with
paper_2012_08141_b200/ and never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "sg_oracle.cpp")

ROOT, DENSE, BITMASKED, POINTER, PLACE = 0, 1, 2, 3, 4

# The oracle's own op ids (must match the enum in sg_oracle.cpp).
OPS = {"FILL": 1, "ADD_CONST": 2, "INC": 3, "AXPY": 4, "STENCIL": 5, "JACOBI": 6,
       "REDUCE_SUM": 7, "DOWNSAMPLE": 8, "JITTER": 9, "CLEAR_SCALAR": 10,
       "P2G": 20, "GRID_OP": 21, "G2P": 22,
       "LOSS_MEAN": 27, "ADJ_INIT": 28, "G2P_ADJ": 29, "P2G_ADJ": 30,
       "SMOOTH_RB": 31, "RESTRICT": 32, "PROLONG": 33, "RESID_NORM2": 34,
       "DOT": 35, "AXPY_RATIO": 36, "XPAY_RATIO": 37, "COPY_SCALAR": 38, "PERMUTE": 42}

ERRORS = {-1: "ARG", -2: "LAYOUT", -3: "RANGE", -6: "DEMOTION_TRAP", -7: "OVERFLOW"}


def build(force=False):
    """Compile the oracle (g++, -O2, no FMA contraction)."""
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC):
        return _LIB_PATH
    cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
           "-o", _LIB_PATH, _SRC]
    subprocess.check_call(cmd)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        P = ctypes.POINTER
        L.orc_create.restype = vp
        L.orc_create.argtypes = [P(i32), i32, ctypes.c_char_p, i32]
        L.orc_destroy.argtypes = [vp]
        L.orc_error.restype = ctypes.c_char_p
        L.orc_error.argtypes = [vp]
        L.orc_activate.argtypes = [vp, i32, P(i32), i64]
        L.orc_listgen.argtypes = [vp, i32]
        L.orc_clear_list.argtypes = [vp, i32]
        L.orc_struct_for.argtypes = [vp, i32, i32, P(i32), i32, P(ctypes.c_float), i32, u32]
        L.orc_serial.argtypes = [vp, i32, P(i32), i32, P(ctypes.c_float), i32]
        L.orc_deactivate.argtypes = [vp, i32]
        L.orc_export_mask.restype = i64
        L.orc_export_mask.argtypes = [vp, i32, P(i32), i64]
        L.orc_export_list.restype = i64
        L.orc_export_list.argtypes = [vp, i32, P(i32), i64]
        L.orc_read_field.argtypes = [vp, i32, P(ctypes.c_double), P(ctypes.c_double), i64]
        L.orc_load_field.argtypes = [vp, i32, P(ctypes.c_double), i64]
        L.orc_counters.argtypes = [vp, P(i64)]
        L.orc_register_array.argtypes = [vp, P(ctypes.c_float), i64, i32]
        L.orc_read_array.argtypes = [vp, i32, P(ctypes.c_double), P(ctypes.c_double), i64]
        L.orc_load_array.argtypes = [vp, i32, P(ctypes.c_double), i64]
        L.orc_set_exact.argtypes = [vp, i32]
        L.orc_range_for.argtypes = [vp, i32, i64, P(i32), i32, P(i32), i32, P(ctypes.c_float), i32, u32]
        for name in ("orc_activate", "orc_listgen", "orc_clear_list", "orc_struct_for", "orc_serial",
                     "orc_deactivate", "orc_read_field", "orc_load_field", "orc_counters", "orc_register_array",
                     "orc_read_array", "orc_load_array", "orc_range_for"):
            getattr(L, name).restype = i32
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle {ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class Oracle:
    """One oracle grid.  Methods mirror the LOWERED task vocabulary."""

    def __init__(self, desc):
        self.desc = np.ascontiguousarray(desc, dtype=np.int32)
        err = ctypes.create_string_buffer(256)
        self.h = lib().orc_create(_ptr(self.desc, ctypes.c_int32), len(self.desc), err, 256)
        if not self.h:
            raise OracleError(-2, err.value.decode())
        self._derive()
        self.tasks_eager_folded = 0
        self.tasks_eager_faithful = 0

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().orc_destroy(h)
            self.h = None

    # --- layout facts needed for lowering (independent of the product) ---
    def _derive(self):
        d = self.desc
        self.parent = [int(r[1]) for r in d]
        self.kind = [int(r[0]) for r in d]
        self.ndim = [int(r[2]) for r in d]
        self.place_rows = [i for i, r in enumerate(d) if r[0] == PLACE]
        # chain (root->leaf) of levels above each snode
        self.chain_of = {}
        for i in range(1, len(d)):
            c, n = [], i if self.kind[i] != PLACE else self.parent[i]
            while n > 0:
                c.append(n)
                n = self.parent[n]
            self.chain_of[i] = list(reversed(c))

    def field_leaf(self, f):
        return self.parent[self.place_rows[f]]

    def field_shape(self, f):
        row = self.place_rows[f]
        s = [1, 1, 1]
        n = self.parent[row]
        while n > 0:
            for a in range(3):
                s[a] *= int(self.desc[n][3 + a])
            n = self.parent[n]
        return tuple(s[: self.ndim[row]])

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, lib().orc_error(self.h).decode())

    # --- lowered tasks ---
    def activate(self, field, coords):
        c = np.ascontiguousarray(coords, dtype=np.int32)
        self._check(lib().orc_activate(self.h, field, _ptr(c, ctypes.c_int32), len(c)))

    def listgen(self, snode):
        self._check(lib().orc_listgen(self.h, snode))

    def clear_list(self, snode):
        self._check(lib().orc_clear_list(self.h, snode))

    def struct_for_task(self, op, snode, fields, params=(), activating=0):
        f = np.ascontiguousarray(fields, dtype=np.int32)
        p = np.ascontiguousarray(params if len(params) else [0.0], dtype=np.float32)
        self._check(lib().orc_struct_for(self.h, OPS[op], snode, _ptr(f, ctypes.c_int32), len(f),
                                         _ptr(p, ctypes.c_float), len(params), activating))

    def serial_task(self, op, fields, params=()):
        f = np.ascontiguousarray(fields, dtype=np.int32)
        p = np.ascontiguousarray(params if len(params) else [0.0], dtype=np.float32)
        self._check(lib().orc_serial(self.h, OPS[op], _ptr(f, ctypes.c_int32), len(f),
                                     _ptr(p, ctypes.c_float), len(params)))

    def deactivate_task(self, snode):
        self._check(lib().orc_deactivate(self.h, snode))

    def range_for_task(self, op, n, fields, arrays, params=(), activating=0):
        f = np.ascontiguousarray(fields, dtype=np.int32)
        a = np.ascontiguousarray(arrays, dtype=np.int32)
        p = np.ascontiguousarray(params if len(params) else [0.0], dtype=np.float32)
        self._check(lib().orc_range_for(self.h, OPS[op], n, _ptr(f, ctypes.c_int32), len(f), _ptr(a, ctypes.c_int32),
                                        len(a), _ptr(p, ctypes.c_float), len(params), activating))

    def set_exact(self, on=True):
        """f64 storage (no f32 rounding of fields/arrays): finite-difference pins."""
        lib().orc_set_exact(self.h, 1 if on else 0)

    # --- particle arrays (SoA: shape (ncomp, n)) ---
    def register_array(self, arr):
        a = np.ascontiguousarray(arr, dtype=np.float32)
        if a.ndim == 1:
            a = a[None]
        rc = lib().orc_register_array(self.h, _ptr(a, ctypes.c_float), a.shape[1], a.shape[0])
        self._check(0 if rc >= 0 else rc)
        self.array_shapes = getattr(self, "array_shapes", []) + [a.shape]
        return rc

    def array(self, i, with_mag=False):
        shape = self.array_shapes[i]
        v = np.zeros(shape, dtype=np.float64)
        m = np.zeros(shape, dtype=np.float64)
        self._check(lib().orc_read_array(self.h, i, _ptr(v, ctypes.c_double), _ptr(m, ctypes.c_double), v.size))
        return (v, m) if with_mag else v

    def load_array(self, i, data):
        d = np.ascontiguousarray(data, dtype=np.float64)
        self._check(lib().orc_load_array(self.h, i, _ptr(d, ctypes.c_double), d.size))

    # --- lowering (readings R3, R5) ---
    def listgen_levels(self, leaf):
        """Sparse levels a struct-for over `leaf` needs lists for: every
        pointer/bitmasked level on the root->leaf path except a bitmasked leaf."""
        out = []
        for s in self.chain_of[leaf]:
            if self.kind[s] in (BITMASKED, POINTER):
                if s == leaf and self.kind[s] == BITMASKED:
                    continue
                out.append(s)
        return out

    def _lower_lists(self, levels):
        for s in levels:
            self.clear_list(s)
            self.listgen(s)
        self.tasks_eager_faithful += 2 * len(levels)
        self.tasks_eager_folded += len(levels)

    def _count1(self):
        self.tasks_eager_faithful += 1
        self.tasks_eager_folded += 1

    def call(self, c):
        kind = c["call"]
        if kind == "activate":
            self.activate(c["field"], c["coords"])
            self._count1()
        elif kind == "struct_for":
            self._lower_lists(self.listgen_levels(c["snode"]))
            act = sum(1 << i for i, a in enumerate(c.get("activating", [])) if a)
            self.struct_for_task(c["op"], c["snode"], c["fields"], c.get("params", []), act)
            self._count1()
        elif kind == "serial":
            self.serial_task(c["op"], c["fields"], c.get("params", []))
            self._count1()
        elif kind == "range_for":
            act = sum(1 << i for i, a in enumerate(c.get("activating", [])) if a)
            self.range_for_task(c["op"], c["n"], c["fields"], c["arrays"], c.get("params", []), act)
            self._count1()
        elif kind == "clear":
            if c["mode"] == "values":
                f = c["target"]
                if self.ndim[self.place_rows[f]] == 0:
                    self.serial_task("CLEAR_SCALAR", [f])
                    self._count1()
                else:
                    leaf = self.field_leaf(f)
                    self._lower_lists(self.listgen_levels(leaf))
                    self.struct_for_task("FILL", leaf, [f], [0.0], 0)
                    self._count1()
            else:
                s = c["target"]
                leaf = self.chain_of[s][-1]
                # the tree's leaf level: follow structural children down
                n = s
                while True:
                    kids = [i for i in range(len(self.desc)) if self.parent[i] == n and self.kind[i] != PLACE]
                    if not kids:
                        break
                    n = kids[0]
                leaf = n
                self._lower_lists(self.listgen_levels(leaf))
                self.deactivate_task(s)
                self._count1()
        elif kind == "listgen":
            s = c["snode"]
            lv = [x for x in self.chain_of[s] if self.kind[x] in (BITMASKED, POINTER)]
            self._lower_lists(lv)
        elif kind == "flush":
            pass  # the oracle is eager: every task already ran
        else:
            raise ValueError(f"unknown call {kind}")

    # --- snapshots ---
    def mask(self, snode):
        nd = self.ndim[snode]
        n = lib().orc_export_mask(self.h, snode, None, 0)
        if n < 0:
            self._check(int(n))
        out = np.zeros((max(n, 1), max(nd, 1)), dtype=np.int32)
        lib().orc_export_mask(self.h, snode, _ptr(out, ctypes.c_int32), n)
        return out[:n, :nd]

    def list(self, snode):
        nd = self.ndim[snode]
        n = lib().orc_export_list(self.h, snode, None, 0)
        out = np.zeros((max(n, 1), max(nd, 1)), dtype=np.int32)
        lib().orc_export_list(self.h, snode, _ptr(out, ctypes.c_int32), n)
        return out[:n, :nd]

    def field(self, f, with_mag=False):
        shape = self.field_shape(f)
        n = int(np.prod(shape)) if shape else 1
        v = np.zeros(n, dtype=np.float64)
        m = np.zeros(n, dtype=np.float64)
        self._check(lib().orc_read_field(self.h, f, _ptr(v, ctypes.c_double), _ptr(m, ctypes.c_double), n))
        v, m = v.reshape(shape), m.reshape(shape)
        return (v, m) if with_mag else v

    def load_field(self, f, dense):
        d = np.ascontiguousarray(dense, dtype=np.float64).ravel()
        self._check(lib().orc_load_field(self.h, f, _ptr(d, ctypes.c_double), len(d)))

    def counters(self):
        out = np.zeros(4, dtype=np.int64)
        lib().orc_counters(self.h, _ptr(out, ctypes.c_int64))
        return dict(tasks=int(out[0]), listgens=int(out[1]), allocated=int(out[2]), freed=int(out[3]))


def run_program(prog, upto=None):
    """Replay a workloads program on a fresh oracle grid (eager, unoptimized)."""
    o = Oracle(prog["desc"])
    for name, arr in prog.get("arrays", {}).items():
        o.register_array(arr)
    calls = prog["calls"] if upto is None else prog["calls"][:upto]
    for c in calls:
        o.call(c)
    return o
