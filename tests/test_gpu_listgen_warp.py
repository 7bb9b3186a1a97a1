"""GPU parity (-m gpu) of the warp-tile listgen (k_listgen_warp):
big bitmasked levels (>= 8 mask words per parent entry, parent capacity large
enough that the launcher picks warp tiles).  Lists bit-exact against the CPU
oracle as sorted sets (BASELINE.json north_star), plus the count and no
duplicates.  Covers sparse (10%, the LG-XL shape), empty, fully dense
containers (tiles above the 1024-entry staging buffer take the direct-write
path), single bits at word and container edges, and a ragged parent list."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2012_08141_b200 import sg  # noqa: E402


def as_set(a):
    return sorted(map(tuple, np.asarray(a).tolist()))


def layout(ptr=8, bm=16):
    L = W.Layout()
    lv = L.chain([("pointer", (ptr,) * 3), ("bitmasked", (bm,) * 3)], [("m", "f32")])
    return L, lv


def run(cells, ptr=8, bm=16):
    L, lv = layout(ptr, bm)
    calls = [W.activate(0, np.asarray(cells, dtype=np.int32).reshape(-1, 3)), W.listgen(lv[-1]), W.flush()]
    prog = W.program(L, calls)
    g, _ = sg.run_program(prog)
    o = oracle.run_program(prog)
    got = np.asarray(g.list(lv[-1]))
    want = as_set(o.list(lv[-1]))
    assert len(got) == len(want)
    assert len(set(map(tuple, got.tolist()))) == len(got), "duplicate entries"
    assert as_set(got) == want
    assert as_set(g.mask(lv[-1])) == as_set(o.mask(lv[-1]))
    return len(want)


def sparse_cells(rng, ptr, bm, p_ptr, p_bit):
    n = ptr ** 3
    on = rng.permutation(n)[: max(1, int(n * p_ptr))]
    k = int(bm ** 3 * p_bit)
    out = []
    for c in on:
        px, py, pz = c // (ptr * ptr), (c // ptr) % ptr, c % ptr
        loc = rng.choice(bm ** 3, size=k, replace=False)
        lx, ly, lz = loc // (bm * bm), (loc // bm) % bm, loc % bm
        out.append(np.stack([px * bm + lx, py * bm + ly, pz * bm + lz], 1))
    return np.concatenate(out)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_sparse_ten_percent(seed):
    rng = np.random.default_rng(seed)
    assert run(sparse_cells(rng, 8, 16, 0.3, 0.10)) > 10000


def test_empty():
    assert run(np.zeros((0, 3), dtype=np.int32)) == 0


def test_dense_containers_take_the_direct_path():
    # two whole 16^3 containers (4096 bits each): every warp tile holds 8192
    # set bits, far above the staging buffer
    cells = np.stack(np.meshgrid(np.arange(32), np.arange(16), np.arange(16), indexing="ij"), -1).reshape(-1, 3)
    assert run(cells) == 32 * 16 * 16


def test_edge_bits_and_mixed_density():
    rng = np.random.default_rng(7)
    edges = []
    for c in [(0, 0, 0), (7, 7, 7), (3, 0, 5)]:
        base = np.array(c) * 16
        for loc in [(0, 0, 0), (15, 15, 15), (0, 0, 31 % 16), (0, 1, 15), (8, 8, 0)]:
            edges.append(base + np.array(loc))
    dense = np.stack(np.meshgrid(np.arange(16, 32), np.arange(32, 48), np.arange(0, 16), indexing="ij"), -1).reshape(-1, 3)
    cells = np.concatenate([np.array(edges), dense, sparse_cells(rng, 8, 16, 0.05, 0.3)])
    run(cells)


def test_repeat_listgen_is_stable_across_epochs():
    # the look-back descriptors carry an epoch: back-to-back listgens of the
    # same level must each produce the full list
    rng = np.random.default_rng(3)
    L, lv = layout()
    cells = sparse_cells(rng, 8, 16, 0.2, 0.1).astype(np.int32)
    g = sg.Grid(L.desc())
    g.activate(0, torch.as_tensor(cells).cuda())
    g.flush("all")
    first = None
    for _ in range(4):
        g.listgen(lv[-1])
        g.flush(0)
        got = as_set(g.list(lv[-1]))
        first = first or got
        assert got == first
    assert len(first) == len({tuple(c) for c in cells.tolist()})


def test_lg_xl_full_size_exact_set():
    """LG-XL at the size bench.py times (2048^3 bound, pointer(64^3) -> bitmasked(32^3),
    25% of the containers, 10% of their bits): the list must be exactly the set of
    activated cells -- listgen's definition with no
    deactivation in between -- compared as sorted 64-bit cell keys on the device."""
    L = W.Layout()
    lv = L.chain([("pointer", (64,) * 3), ("bitmasked", (32,) * 3)], [("m", "f32")])
    gen = torch.Generator(device="cuda").manual_seed(0)
    n_ptr = 64 ** 3
    ptr_on = torch.randperm(n_ptr, device="cuda", generator=gen)[: n_ptr // 4]
    n_act = ptr_on.numel()
    cells_per = int(32768 * 0.10)
    g = sg.Grid(L.desc(), pool_capacity=n_act, list_capacity=int(n_act * cells_per * 1.05) + 1024)
    keys = []
    for s in range(0, n_act, 4096):
        pc = ptr_on[s:s + 4096]
        px, py, pz = pc // 4096, (pc // 64) % 64, pc % 64
        loc = torch.randint(0, 32768, (pc.numel(), cells_per), device="cuda", generator=gen)
        co = torch.stack([px[:, None] * 32 + loc // 1024, py[:, None] * 32 + (loc // 32) % 32,
                          pz[:, None] * 32 + loc % 32], -1).reshape(-1, 3).to(torch.int32).contiguous()
        g.activate(0, co)
        g.flush("all")
        c64 = co.to(torch.int64)
        keys.append((c64[:, 0] << 22) | (c64[:, 1] << 11) | c64[:, 2])
    g.sync()
    want = torch.unique(torch.cat(keys))
    del keys
    g.listgen(lv[-1])
    g.flush("all")
    got = torch.as_tensor(g.list(lv[-1])).cuda().to(torch.int64)
    assert got.shape[0] == want.numel()
    gk = torch.sort((got[:, 0] << 22) | (got[:, 1] << 11) | got[:, 2]).values
    assert torch.equal(gk, want)
