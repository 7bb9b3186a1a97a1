"""Brute-force dense checker for the oracle (tiny grids only).

A second, independent formulation of the sparse-grid semantics used to pin the
oracle (s4 tier T0): every sparse level is a dense
boolean array over its whole resolution, a leaf cell is active iff the
upsampled masks of all its sparse ancestors are set (PAPER.md:162 dense
constraint), fields are dense int64 arrays that hold 0 where inactive
(PAPER.md:195), and struct-for visits exactly the active leaf cells
(PAPER.md:138-143).  Ops are evaluated with whole-array numpy expressions
(shifted zero-padded views for stencils) instead of per-cell map lookups.
It implements only the EAGER program (lists are always fresh there).
"""
import numpy as np

ROOT, DENSE, BITMASKED, POINTER, PLACE = 0, 1, 2, 3, 4


class Brute:
    def __init__(self, desc):
        d = np.asarray(desc)
        self.d = d
        n = len(d)
        self.parent = d[:, 1].tolist()
        self.kind = d[:, 0].tolist()
        self.nd = d[:, 2].tolist()
        self.places = [i for i in range(n) if self.kind[i] == PLACE]
        self.chain = {}
        for i in range(1, n):
            c, x = [], (i if self.kind[i] != PLACE else self.parent[i])
            while x > 0:
                c.append(x)
                x = self.parent[x]
            self.chain[i] = c[::-1]
        self.res = {}
        for i in range(1, n):
            if self.kind[i] == PLACE:
                continue
            r = np.ones(3, dtype=int)
            for x in self.chain[i]:
                r *= d[x, 3:6]
            self.res[i] = tuple(int(v) for v in r[: self.nd[i]])
        self.masks = {i: np.zeros(self.res[i], dtype=bool) for i in self.res
                      if self.kind[i] in (BITMASKED, POINTER)}
        self.vals = []
        for p in self.places:
            lv = self.chain[p]
            shape = self.res[lv[-1]] if lv else ()
            self.vals.append(np.zeros(shape, dtype=np.int64))

    # --- structure ---
    def levels_of_field(self, f):
        return self.chain[self.places[f]]

    def active(self, levels):
        if not levels:
            return np.ones((), dtype=bool)
        shape = self.res[levels[-1]]
        a = np.ones(shape, dtype=bool)
        for l in levels:
            if l in self.masks:
                m = self.masks[l]
                for ax in range(len(shape)):
                    m = np.repeat(m, shape[ax] // self.res[l][ax], axis=ax)
                a &= m
        return a

    def field_active(self, f):
        return self.active(self.levels_of_field(f))

    def activate_cells(self, levels, cells):
        leaf = levels[-1]
        for l in levels:
            if l in self.masks:
                ratio = np.array(self.res[leaf]) // np.array(self.res[l])
                q = cells // ratio
                self.masks[l][tuple(q.T)] = True

    def read(self, f):
        return self.vals[f] * self.field_active(f)

    # --- program replay ---
    def call(self, c):
        k = c["call"]
        if k == "activate":
            self.activate_cells(self.levels_of_field(c["field"]), np.asarray(c["coords"]))
        elif k == "struct_for":
            self.struct_for(c["op"], c["snode"], c["fields"], c.get("params", []))
        elif k == "serial":
            assert c["op"] == "CLEAR_SCALAR"
            self.vals[c["fields"][0]][...] = 0
        elif k == "clear":
            if c["mode"] == "values":
                f = c["target"]
                self.vals[f] = np.where(self.field_active(f), 0, self.vals[f])
            else:
                s = c["target"]
                tree_levels = [l for l in self.chain if self.kind[l] != PLACE and s in self.chain[l]]
                for l in tree_levels:
                    if l in self.masks:
                        self.masks[l][...] = False
                for f, p in enumerate(self.places):
                    if s in self.chain[p]:
                        self.vals[f][...] = 0

    def struct_for(self, op, snode, f, p):
        levels = self.chain[snode]
        A = self.active(levels)
        P = lambda i: int(p[i]) if i < len(p) else 0
        D = len(A.shape)

        def shifted(R, ax, d):
            out = np.zeros_like(R)
            src = [slice(None)] * D
            dst = [slice(None)] * D
            if d > 0:
                src[ax], dst[ax] = slice(d, None), slice(None, -d)
            else:
                src[ax], dst[ax] = slice(None, d), slice(-d, None)
            out[tuple(dst)] = R[tuple(src)]
            return out

        if op == "FILL":
            self.vals[f[0]][A] = P(0)
        elif op == "INC":
            self.vals[f[0]][A] += P(0)
        elif op == "ADD_CONST":
            self.vals[f[0]][A] = (self.read(f[1]) + P(0))[A]
        elif op == "AXPY":
            self.vals[f[0]][A] = (P(0) * self.read(f[1]) + self.read(f[2]))[A]
        elif op == "STENCIL":
            R = self.read(f[1])
            S = sum(shifted(R, ax, +1) + shifted(R, ax, -1) for ax in range(D)) - 2 * D * R
            self.vals[f[0]][A] = S[A]
        elif op == "JACOBI":
            R = self.read(f[1])
            S = sum(shifted(R, ax, +1) + shifted(R, ax, -1) for ax in range(D)) + self.read(f[2])
            self.vals[f[0]][A] = S[A] / (2 * D)
        elif op == "JITTER":
            R = self.read(f[0])
            nb = shifted(R, 0, +1)
            even = (np.arange(A.shape[0]) % 2 == 0).reshape((-1,) + (1,) * (D - 1))
            sel = A & even
            self.vals[f[0]][sel] += nb[sel]
        elif op == "REDUCE_SUM":
            self.vals[f[0]][...] += self.read(f[1])[A].sum()
        elif op == "DOWNSAMPLE":
            R = self.read(f[1]) if len(f) > 1 and f[1] >= 0 else np.zeros(A.shape, dtype=np.int64)
            cells = np.argwhere(A)
            if len(cells):
                hl = self.levels_of_field(f[0])
                self.activate_cells(hl, cells // 2)
                np.add.at(self.vals[f[0]], tuple((cells // 2).T), P(0) * R[A] + P(1))
        else:
            raise ValueError(op)

    def mask(self, s):
        return np.argwhere(self.masks[s]).astype(np.int32)


def run(prog):
    b = Brute(prog["desc"])
    for c in prog["calls"]:
        b.call(c)
    return b
