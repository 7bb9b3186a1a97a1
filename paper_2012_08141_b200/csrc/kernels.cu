// kernels.cu -- sm_100a kernels of the sparse-grid hot path: range-for (MPM
// transfers, binned; exchange ops), deactivation and the export helpers.
// Activation and listgen live in kernels_lg.cu, the struct-for launches in
// kernels_sf.cu (separate translation units compile in parallel).
//
//   k_deactivate    DEACTIVATE(S): zero payload of active blocks, clear masks,
//                   push pointer children to the free list (zero-on-free).
//   k_serial / k_range_for, export helpers.
// No host synchronization anywhere on the hot path: list counts are read on
// the device and every kernel grid-strides over them.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include "sg_internal.h"
#include "jit.h"

namespace cg = cooperative_groups;

namespace sg {

#include "device_common.cuh"

#include "mpm_ops.cuh"
#include "exchange_ops.cuh"
#include "mpm_adj.cuh"
#include "mpm_bin.cuh"

// ---------------------------------------------------------------------------
// Serial and range-for
// ---------------------------------------------------------------------------
struct SerArgs {
  DevCtx C;
  int nops;
  DOp ops[SG_MAXOPS];
  uint64_t aux[SG_MAXOPS];
};

__global__ void k_serial(const __grid_constant__ SerArgs A) {
  for (int o = 0; o < A.nops; o++) {
    if (A.ops[o].op == SG_OP_CLEAR_SCALAR) *(uint32_t*)A.aux[o] = 0u;
    if (A.ops[o].op == SG_OP_COPY_SCALAR)
      *(uint32_t*)A.aux[o] = A.C.scalars[A.C.fields[A.ops[o].f[1]].scalar];
    if (A.ops[o].op == SG_OP_ARRAY_COUNT) *A.C.arrays[A.ops[o].a[0]].dcount = (int32_t)A.ops[o].p[0];
  }
}

struct RFArgs {
  DevCtx C;
  int64_t n;
  const int32_t* dcount;   // device extent (range_n < 0), else null
  int nops;
  int task;
  DOp ops[SG_MAXOPS];
};

__global__ void __launch_bounds__(128) k_range_for(const __grid_constant__ RFArgs A) {
  const int64_t n = A.dcount ? (int64_t)*A.dcount : A.n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int o = 0; o < A.nops; o++) {
      const DOp& op = A.ops[o];
      switch (op.op) {
        case SG_OP_P2G: mpm_p2g<0>(A.C, A.C.trees[A.C.fields[op.f[0]].tree], op, i, A.task); break;
        case SG_OP_G2P: mpm_g2p<0>(A.C, A.C.trees[A.C.fields[op.f[0]].tree], op, i); break;
        case SG_OP_HALO_UNPACK: halo_unpack(A.C, op, i, A.task); break;
        case SG_OP_ADJ_INIT: adj_init(A.C, op, i); break;
        default: break;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Deactivate (reading R7): payload zeroed, masks cleared, children freed.
// ---------------------------------------------------------------------------
struct DeArgs {
  DTree T;
  DevCtx C;
  int ls;
  const uint32_t* drive_entries;
  const uint32_t* drive_count;
  const uint32_t* lent[SG_MAXL];
  const uint32_t* lcnt[SG_MAXL];
};

__global__ void __launch_bounds__(256) k_deactivate(const __grid_constant__ DeArgs A) {
  const DTree& T = A.T;
  const uint32_t nblk = A.drive_entries ? *A.drive_count : 1u;
  const uint32_t blk = 1u << T.lblk;
  const uint64_t fstride = 1ull << T.ln_leaf;
  // phase 1: zero the payload (and leaf bits) of every active block
  for (uint32_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    uint32_t* cont;
    uint32_t first;
    int org[3];
    if (!resolve_entry(T, A.drive_entries ? A.drive_entries[b] : 0u, cont, first, org)) continue;
    uint32_t* p0 = cont + T.payload_off + first;
    for (int f = 0; f < T.nfields; f++)
      for (uint32_t i = threadIdx.x; i < blk; i += blockDim.x) p0[(uint64_t)f * fstride + i] = 0u;
    if (T.leaf_bitmasked) {
      const DLevel& LL = T.lev[T.nlev - 1];
      for (uint32_t w = (first >> 5) + threadIdx.x; w < ((first + blk + 31) >> 5); w += blockDim.x)
        cont[LL.mask_off + w] = 0u;
    }
  }
  // phase 2: every listed level at/below S
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gsz = (uint64_t)gridDim.x * blockDim.x;
  for (int l = A.ls; l < T.nlev; l++) {
    if (!A.lent[l]) continue;
    const DLevel& L = T.lev[l];
    uint32_t n = *A.lcnt[l];
    for (uint64_t i = gtid; i < n; i += gsz) {
      uint32_t e = A.lent[l][i];
      uint32_t cs = e >> L.ln, idx = e & ((1u << L.ln) - 1u);
      uint32_t* cont = cont_ptr(T, L.seg, cs);
      if (L.kind == SG_BITMASKED) {
        cont[L.mask_off + (idx >> 5)] = 0u;
      } else if (L.kind == SG_POINTER) {
        uint32_t v = cont[L.slot_off + idx];
        cont[L.slot_off + idx] = SG_SLOT_NULL;
        if (v != SG_SLOT_NULL && v != SG_SLOT_BUSY) {
          const DSeg& S = T.seg[L.seg + 1];
          uint32_t* child = cont_ptr(T, L.seg + 1, v - 1u);
          for (uint32_t w = 0; w < S.header_words; w++) child[w] = 0u;
          int32_t pos = atomicAdd(&S.alloc[1], 1);
          S.free_list[pos] = v - 1u;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Export / handoff helpers (tests and exports only)
// ---------------------------------------------------------------------------
struct FieldIO {
  DTree T;
  int slot;
  uint32_t* dense;
  const uint32_t* src;
  int64_t total;
  int sh[3];
};

__device__ __forceinline__ void dense_coords(const FieldIO& a, int64_t i, int c[3]) {
  c[2] = (int)(i & ((1ll << a.sh[2]) - 1));
  c[1] = (int)((i >> a.sh[2]) & ((1ll << a.sh[1]) - 1));
  c[0] = (int)(i >> (a.sh[1] + a.sh[2]));
}

__global__ void k_read_field(const __grid_constant__ FieldIO a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.total; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
    dense_coords(a, i, c);
    uint32_t idx;
    uint32_t* cont = locate(a.T, c, idx);
    a.dense[i] = cont ? cont[a.T.payload_off + ((uint64_t)a.slot << a.T.ln_leaf) + idx] : 0u;
  }
}

__global__ void k_load_field(const __grid_constant__ FieldIO a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.total; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
    dense_coords(a, i, c);
    uint32_t idx;
    uint32_t* cont = locate_active(a.T, c, idx);
    if (cont) cont[a.T.payload_off + ((uint64_t)a.slot << a.T.ln_leaf) + idx] = a.src[i];
  }
}

struct MaskScan {
  DTree T;
  int level;
  uint8_t* flags;
  int64_t total;
  int sh[3];
};

__global__ void k_mask_scan(const __grid_constant__ MaskScan a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.total; i += (int64_t)gridDim.x * blockDim.x) {
    int g[3];
    g[2] = (int)(i & ((1ll << a.sh[2]) - 1));
    g[1] = (int)((i >> a.sh[2]) & ((1ll << a.sh[1]) - 1));
    g[0] = (int)(i >> (a.sh[1] + a.sh[2]));
    const DLevel& S = a.T.lev[a.level];
    int c[3] = {g[0] << S.lbelow[0], g[1] << S.lbelow[1], g[2] << S.lbelow[2]};
    uint32_t* cont = a.T.seg[0].base;
    uint32_t idx = 0;
    uint8_t act = 1;
    for (int l = 0; l <= a.level; l++) {
      const DLevel& L = a.T.lev[l];
      idx = (idx << L.lE) | local_lin(L, c);
      if (L.kind == SG_BITMASKED) {
        if (!((cont[L.mask_off + (idx >> 5)] >> (idx & 31)) & 1u)) { act = 0; break; }
      } else if (L.kind == SG_POINTER) {
        uint32_t v = cont[L.slot_off + idx];
        if (v == SG_SLOT_NULL || v == SG_SLOT_BUSY) { act = 0; break; }
        if (l < a.level) { cont = cont_ptr(a.T, L.seg + 1, v - 1u); idx = 0; }
      }
    }
    a.flags[i] = act;
  }
}

struct ListDecode {
  DTree T;
  int level;
  const uint32_t* entries;
  const uint32_t* count;
  int32_t* coords;
};

__global__ void k_list_decode(const __grid_constant__ ListDecode a) {
  uint32_t n = *a.count;
  const DLevel& L = a.T.lev[a.level];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t e = a.entries[i];
    int g[3];
    cell_coords(a.T, a.level, e >> L.ln, e & ((1u << L.ln) - 1u), g);
    for (int d = 0; d < a.T.nd; d++) a.coords[(uint64_t)i * a.T.nd + d] = g[d];
  }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
static int check_launch() { return cudaGetLastError() == cudaSuccess ? 0 : SG_ERR_CUDA; }
static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static bool lb2_tree(const DTree& t) {
  const DLevel& d = t.lev[t.driving];
  return d.lbelow[0] == 2 && d.lbelow[1] == 2 && d.lbelow[2] == 2 && t.lblk == 6;
}

uint32_t bin_ntiles(uint32_t nkeys) { return (nkeys + BIN_TILE - 1) / BIN_TILE; }

int launch_bin(const DBins& b, const float* x, int64_t xs, int64_t n, const int32_t* dcount, float inv_dx,
               void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  BinArgs a;
  a.B = b; a.x = x; a.xs = xs; a.n = n; a.dcount = dcount; a.inv_dx = inv_dx;
  a.ntiles = bin_ntiles(b.nkeys);
  const int gp = (int)std::max<int64_t>(1, std::min<int64_t>((n + BIN_TPB - 1) / BIN_TPB, (int64_t)num_sms() * 8));
  const int gt = (int)std::min<uint32_t>(a.ntiles, (uint32_t)num_sms() * 4);
  // (a shared-memory histogram variant, k_bin_count_smem, measured slower on C4:
  // 14.4 vs 10.0 us -- profiles/r01_launches_c4_t31.csv)
  k_bin_count<<<gp, BIN_TPB, 0, s>>>(a);
  k_bin_tiles<<<gt, BIN_TPB, 0, s>>>(a);
  k_bin_top<<<1, 1024, 0, s>>>(a);
  k_bin_apply<<<gt, BIN_TPB, 0, s>>>(a);
  k_bin_scatter<<<gp, BIN_TPB, 0, s>>>(a);
  return check_launch();
}

int launch_range_for(const DevCtx& c, int64_t n, const int32_t* dcount, const DOp* ops, int nops, int task,
                     void* stream, const RangeScratch* rs, const DTree* grid_tree, const DTree* tree2,
                     const DBins* bins) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (nops == 1 && ops[0].op == SG_OP_PERMUTE) {
    PermArgs m;
    m.C = c; m.op = ops[0]; m.n = n; m.dcount = dcount; m.binned = bins != nullptr;
    if (bins) m.B = *bins;
    int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    k_permute<<<std::max(grid, 1), 256, 0, s>>>(m);
    return check_launch();
  }
  if (nops == 1 && bins) {   // binned MPM kernels (LB = 2 trees; bins built by the caller)
    MpmBinArgs m;
    m.T = *grid_tree; m.TG = tree2 ? *tree2 : *grid_tree; m.C = c; m.op = ops[0]; m.B = *bins; m.task = task;
    // (bin, chunk) grid: x strides over the non-empty bins, y over a bin's chunks
    const dim3 grid((unsigned)num_sms() * MB_BINS_X, MB_CHUNKS_Y);
    switch (ops[0].op) {
      case SG_OP_P2G: k_p2g_bin<<<grid, MB_TPB, 0, s>>>(m); break;
      case SG_OP_G2P: k_g2p_bin<<<grid, MB_TPB, 0, s>>>(m); break;
      case SG_OP_G2P_ADJ: k_g2p_adj_bin<<<grid, MB_TPB, 0, s>>>(m); break;
      case SG_OP_P2G_ADJ: k_p2g_adj_bin<<<grid, MB_TPB, 0, s>>>(m); break;
      default: return -1;
    }
    return check_launch();
  }
  if (nops == 1 && (ops[0].op == SG_OP_G2P_ADJ || ops[0].op == SG_OP_P2G_ADJ)) {
    Mpm2Args m;
    m.T = *grid_tree; m.TG = tree2 ? *tree2 : *grid_tree; m.C = c; m.op = ops[0]; m.n = n; m.task = task;
    const bool lb2 = lb2_tree(m.T) && lb2_tree(m.TG);
    int grid = (int)std::min<int64_t>((n + 127) / 128, (int64_t)num_sms() * 16);
    if (ops[0].op == SG_OP_G2P_ADJ) {
      if (lb2) k_g2p_adj<2><<<grid, 128, 0, s>>>(m);
      else k_g2p_adj<0><<<grid, 128, 0, s>>>(m);
    } else {
      if (lb2) k_p2g_adj<2><<<grid, 128, 0, s>>>(m);
      else k_p2g_adj<0><<<grid, 128, 0, s>>>(m);
    }
    return check_launch();
  }
  if (nops == 1 && ops[0].op == SG_OP_LOSS_MEAN) {
    LossArgs m;
    m.C = c; m.op = ops[0]; m.n = n;
    m.target = c.scalars + (ops[0].scalar >= 0 ? ops[0].scalar : 0);
    int grid = (int)std::min<int64_t>((n + LM_TPB - 1) / LM_TPB, (int64_t)std::min(c.max_grid, num_sms() * 4));
    k_loss_mean<<<std::max(grid, 1), LM_TPB, 0, s>>>(m);
    return check_launch();
  }
  if (nops == 1 && grid_tree && (ops[0].op == SG_OP_P2G || ops[0].op == SG_OP_G2P)) {
    MpmArgs m;
    m.T = *grid_tree; m.C = c; m.op = ops[0]; m.n = n; m.dcount = dcount; m.task = task;
    const bool lb2 = lb2_tree(*grid_tree);
    int grid = (int)std::min<int64_t>((n + 127) / 128, (int64_t)num_sms() * 16);
    if (ops[0].op == SG_OP_P2G) {
      if (lb2) k_p2g<2><<<grid, 128, 0, s>>>(m);
      else k_p2g<0><<<grid, 128, 0, s>>>(m);
    } else {
      if (lb2) k_g2p<2><<<grid, 128, 0, s>>>(m);
      else k_g2p<0><<<grid, 128, 0, s>>>(m);
    }
    return check_launch();
  }
  if (nops == 1 && ops[0].op == SG_OP_G2P_MIGRATE) {
    MigArgs m;
    m.C = c; m.op = ops[0]; m.status = rs->status; m.ctl = rs->ctl; m.task = task;
    m.T = *grid_tree;
    int grid = (int)std::min<int64_t>((n + MG_TPB - 1) / MG_TPB, (int64_t)num_sms() * 6);
    k_g2p_migrate<<<std::max(grid, 1), MG_TPB, 0, s>>>(m);
    return check_launch();
  }
  if (nops == 1 && ops[0].op == SG_OP_MIGRATE_COMPACT) {
    CompactArgs m;
    m.C = c; m.op = ops[0]; m.holes = rs->holes; m.tail = rs->tail; m.cap = rs->hole_cap; m.task = task;
    int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    k_migrate_mark<<<std::max(grid, 1), 256, 0, s>>>(m);
    k_migrate_fill<<<1, 1024, 0, s>>>(m);
    return check_launch();
  }
  if (nops == 1 && ops[0].op == SG_OP_MIGRATE_APPEND) {
    AppArgs m;
    m.C = c; m.op = ops[0]; m.ctl = rs->ctl + 4;
    int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 4);
    k_migrate_append<<<std::max(grid, 1), 256, 0, s>>>(m);
    return check_launch();
  }
  RFArgs* a = new RFArgs();
  a->C = c; a->n = n; a->dcount = dcount; a->nops = nops; a->task = task;
  for (int o = 0; o < nops; o++) a->ops[o] = ops[o];
  int grid = (int)std::min<int64_t>((n + 127) / 128, (int64_t)num_sms() * 16);
  k_range_for<<<grid, 128, 0, s>>>(*a);
  delete a;
  return check_launch();
}

int launch_serial(const DevCtx& c, const DOp* ops, int nops, int, void* stream) {
  SerArgs* a = new SerArgs();
  a->C = c; a->nops = nops;
  for (int o = 0; o < nops; o++) {
    a->ops[o] = ops[o];
    a->aux[o] = (uint64_t)(c.scalars + (ops[o].scalar >= 0 ? ops[o].scalar : 0));
  }
  k_serial<<<1, 1, 0, (cudaStream_t)stream>>>(*a);
  delete a;
  return check_launch();
}

// DEACTIVATE as a pool reset (reading R33): the deactivated level is the
// tree's first sparse level, so every container of every pool is freed -- zero
// the root container and each pool's allocated containers (free-listed ones are
// already zero), then the last CTA resets the bump counters and free lists.
struct ResetArgs {
  DTree T;
};

__global__ void __launch_bounds__(256) k_deactivate_reset(const __grid_constant__ ResetArgs A) {
  const DTree& T = A.T;
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gsz = (uint64_t)gridDim.x * blockDim.x;
  for (int s = 0; s < T.nseg; s++) {
    const DSeg& S = T.seg[s];
    uint64_t n = 1;
    if (s > 0) {
      const int32_t b = S.alloc[0];
      n = (uint64_t)min((uint32_t)max(b, 0), S.capacity);
    }
    const uint64_t words = n * S.stride;   // containers are 128-byte aligned: stride % 4 == 0
    uint4* p = reinterpret_cast<uint4*>(S.base);
    for (uint64_t i = gtid; i < words / 4; i += gsz) p[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (T.nseg < 2) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&T.seg[1].alloc[2], 1) == (int)gridDim.x - 1) {
      for (int s = 1; s < T.nseg; s++) { T.seg[s].alloc[0] = 0; T.seg[s].alloc[1] = 0; }
      T.seg[1].alloc[2] = 0;
      __threadfence();
    }
  }
}

int launch_deactivate_reset(const DTree& t, void* stream) {
  ResetArgs a;
  a.T = t;
  k_deactivate_reset<<<num_sms() * 4, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_deactivate(const DevCtx& c, const DTree& t, int, int level, const DList* lists, int, void* stream) {
  DeArgs a;
  a.T = t; a.C = c; a.ls = level;
  a.drive_entries = t.driving >= 0 ? lists[t.driving].entries : nullptr;
  a.drive_count = t.driving >= 0 ? lists[t.driving].count : nullptr;
  for (int l = 0; l < SG_MAXL; l++) {
    bool listed = l < t.nlev && (t.lev[l].kind == SG_POINTER ||
                                 (t.lev[l].kind == SG_BITMASKED && !(l == t.nlev - 1)));
    a.lent[l] = listed ? lists[l].entries : nullptr;
    a.lcnt[l] = listed ? lists[l].count : nullptr;
  }
  k_deactivate<<<num_sms() * 4, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

static void dense_shifts(const DTree& t, int sh[3]) {
  const DLevel& L = t.lev[t.nlev - 1];
  for (int a = 0; a < 3; a++) sh[a] = L.lres[a];
}

int launch_read_field(const DevCtx&, const DTree& t, int, int slot, uint32_t* dense, void* stream) {
  FieldIO a;
  a.T = t; a.slot = slot; a.dense = dense; a.src = nullptr;
  dense_shifts(t, a.sh);
  a.total = 1ll << (a.sh[0] + a.sh[1] + a.sh[2]);
  k_read_field<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_load_field(const DevCtx&, const DTree& t, int, int slot, const uint32_t* dense, void* stream) {
  FieldIO a;
  a.T = t; a.slot = slot; a.dense = nullptr; a.src = dense;
  dense_shifts(t, a.sh);
  a.total = 1ll << (a.sh[0] + a.sh[1] + a.sh[2]);
  k_load_field<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_mask_scan(const DevCtx&, const DTree& t, int, int level, uint8_t* flags, void* stream) {
  MaskScan a;
  a.T = t; a.level = level; a.flags = flags;
  for (int d = 0; d < 3; d++) a.sh[d] = t.lev[level].lres[d];
  a.total = 1ll << (a.sh[0] + a.sh[1] + a.sh[2]);
  k_mask_scan<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_list_decode(const DTree& t, int level, const DList& l, int32_t* coords, void* stream) {
  ListDecode a{t, level, l.entries, l.count, coords};
  k_list_decode<<<num_sms() * 4, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

}  // namespace sg
