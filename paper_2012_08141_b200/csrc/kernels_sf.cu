// kernels_sf.cu -- struct-for launches (split out of kernels.cu so the
// translation units compile in parallel): the fused struct-for megakernel
// -- op-table tile interpreter, dedicated
// JACOBI kernel, 8^3 streaming kernel, N2 chains -- and the JIT group content.
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include "sg_internal.h"
#include "jit.h"

namespace sg {

#include "device_common.cuh"

#include "mpm_ops.cuh"
#include "struct_for.cuh"

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

template <typename V, int ND, bool PAIR, int GL>
static void sf_dispatch(SFArgs* a, int grid, cudaStream_t s, const ChainTab* chain) {
  if (!chain) {
    k_struct_for<V, ND, PAIR, GL><<<grid, SF_TPB, 0, s>>>(*a);
    return;
  }
  k_struct_chain<V, ND, PAIR, GL><<<1, SF_TPB, 0, s>>>(*a, *chain);
}

// A group of f32 quad ops on 8^3 dense blocks (k_stream8 / stream8_body).
static bool stream8_group(const DTree& t, const DOp* ops, int nops, int gl, bool i32) {
  if (gl != 1 || i32 || t.leaf_bitmasked) return false;
  for (int o = 0; o < nops; o++) {
    const int op = ops[o].op;
    if (!(op == SG_OP_FILL || op == SG_OP_ADD_CONST || op == SG_OP_INC || op == SG_OP_AXPY || op == SG_OP_STENCIL ||
          op == SG_OP_JACOBI || op == SG_OP_REDUCE_SUM || op == SG_OP_DOT || op == SG_OP_AXPY_RATIO ||
          op == SG_OP_XPAY_RATIO))
      return false;
  }
  return true;
}

// The JIT content of a struct-for group (same geometry decisions as
// launch_struct_for); false when the group runs a dedicated kernel instead.
bool jit_group_of(const DTree& t, const DOp* ops, int nops, JitGroup& G) {
  int lb[3] = {0, 0, 0};
  bool quad = false;
  if (t.nlev - 1 - t.driving == 1) {
    const DLevel& B = t.lev[t.nlev - 1];
    for (int d = 0; d < 3; d++) lb[d] = B.le[d];
    quad = B.le[t.nd - 1] >= 2;
  }
  const int nd = quad ? t.nd : 0;
  int gl = 0;
  if (nd == 3 && lb[0] == 3 && lb[1] == 3 && lb[2] == 3) gl = 1;
  else if (nd == 3 && lb[0] == 2 && lb[1] == 2 && lb[2] == 2) gl = 2;
  else if (nd == 2 && lb[0] == 2 && lb[1] == 2) gl = 3;
  const bool i32 = ops[0].dt == SG_I32;
  const bool jac_red = nops == 2 && ops[0].op == SG_OP_JACOBI && ops[1].op == SG_OP_REDUCE_SUM &&
                       ops[1].f[1] == ops[0].f[0] && ops[1].scalar >= 0;
  if ((nops == 1 || jac_red) && ops[0].op == SG_OP_JACOBI && gl == 1 && !i32 && !t.leaf_bitmasked)
    return false;   // k_jacobi8
  G.nops = nops; G.nd = nd; G.gl = gl; G.i32 = i32 ? 1 : 0;
  G.stream = stream8_group(t, ops, nops, gl, i32) && getenv("SG_NO_STREAM8") == nullptr ? 1 : 0;
  for (int o = 0; o < nops; o++) G.ops[o] = ops[o];
  return true;
}

int launch_struct_for(const DevCtx& c, const DTree& t, int, const DList* drive, const DOp* ops, int nops,
                      int task, void* stream, int grid_hint, const DOp* chain_ops, const int* chain_phase_end,
                      int nphases, int chain_needs_nbr) {
  SFArgs* a = new SFArgs();
  a->T = t; a->C = c; a->task = task; a->nops = nops;
  a->entries = drive ? drive->entries : nullptr;
  a->count = drive ? drive->count : nullptr;
  a->table = drive ? drive->table : nullptr;
  a->table_ctl = drive ? drive->ctl : nullptr;
  a->has_reduce = 0;
  for (int o = 0; o < nops; o++)
    a->has_reduce |= ops[o].op == SG_OP_REDUCE_SUM || ops[o].op == SG_OP_RESID_NORM2 || ops[o].op == SG_OP_DOT;
  a->need_nbr = 0;
  bool i32 = false;
  for (int o = 0; o < nops; o++) {
    a->ops[o] = ops[o];
    int op = ops[o].op;
    if (op == SG_OP_STENCIL || op == SG_OP_JACOBI || op == SG_OP_JITTER || op == SG_OP_SMOOTH_RB ||
        op == SG_OP_RESTRICT || op == SG_OP_RESID_NORM2)
      a->need_nbr = 1;
    a->aux[o] = 0;
  }
  if (chain_needs_nbr) a->need_nbr = 1;
  // dtype of the group (validated uniform by the host)
  i32 = ops[0].dt == SG_I32;
  for (int o = 0; o < nops; o++)
    if (ops[o].scalar >= 0) a->aux[o] = (uint64_t)(c.scalars + ops[o].scalar);
  const int lblk = t.lblk;
  // tile: 2048 cells (at most SF_MAXE blocks); larger blocks span several tiles
  const int TILE_LOG = 11;
  a->ltile = TILE_LOG;
  a->lept = 8;   // entries per tile chosen on the device (<= 256), see sf_tiles
  // QUAD path: the block is a single level whose fastest axis has extent >= 4
  bool quad = false;
  a->lb[0] = a->lb[1] = a->lb[2] = 0;
  if (t.nlev - 1 - t.driving == 1) {
    const DLevel& B = t.lev[t.nlev - 1];
    for (int d = 0; d < 3; d++) a->lb[d] = B.le[d];
    quad = B.le[t.nd - 1] >= 2;
  }
  // one resident wave: 5 CTAs per SM (__launch_bounds__(SF_TPB, 5)); tiles are
  // sized on the device so every CTA gets an equal share
  int grid = num_sms() * 5;
  (void)grid_hint;
  ChainTab* ct = nullptr;
  if (nphases > 1) {   // one-CTA chain (the caller checked the list is small and the table fits)
    ct = new ChainTab();
    const int tot = chain_phase_end[nphases - 1];
    for (int i = 0; i < tot && i < SG_CHAIN_OPS; i++) ct->ops[i] = chain_ops[i];
    for (int i = 0; i < nphases && i < SG_CHAIN_OPS; i++) ct->phase_end[i] = chain_phase_end[i];
    ct->nphases = nphases;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int nd = quad ? t.nd : 0;
  static int pair = -1;
  // measured on B200 (profiles/r01_*): one quad per thread at 6 CTAs/SM beats
  // two quads per thread at 3 CTAs/SM (JAC-XL 2.84 vs 1.75 TB/s)
  if (pair < 0) { const char* e = getenv("SG_SF_PAIR"); pair = e ? atoi(e) != 0 : 0; }
  const bool stencil = a->need_nbr;
  // constant-geometry instantiations for the block shapes of the configs
  int gl = 0;
  if (nd == 3 && a->lb[0] == 3 && a->lb[1] == 3 && a->lb[2] == 3) gl = 1;
  else if (nd == 3 && a->lb[0] == 2 && a->lb[1] == 2 && a->lb[2] == 2) gl = 2;
  else if (nd == 2 && a->lb[0] == 2 && a->lb[1] == 2) gl = 3;
  // dedicated kernel: a lone f32 JACOBI over 8^3 dense blocks with a block table
  // dedicated kernel: a lone f32 JACOBI over 8^3 dense blocks with a block
  // table, or JACOBI fused with the reduction of its output
  const bool jac_red = nops == 2 && ops[0].op == SG_OP_JACOBI && ops[1].op == SG_OP_REDUCE_SUM &&
                       ops[1].f[1] == ops[0].f[0] && ops[1].scalar >= 0;
  if ((nops == 1 || jac_red) && ops[0].op == SG_OP_JACOBI && gl == 1 && !i32 && !t.leaf_bitmasked && nphases <= 1 &&
      drive && drive->table && getenv("SG_NO_JAC8") == nullptr) {
    JacArgs j;
    j.T = t; j.entries = drive->entries; j.count = drive->count; j.table = drive->table; j.table_ctl = drive->ctl;
    const uint64_t fs = 1ull << t.ln_leaf;
    j.s_dst = (uint64_t)ops[0].slot[0] * fs; j.s_src = (uint64_t)ops[0].slot[1] * fs;
    j.s_rhs = (uint64_t)ops[0].slot[2] * fs;
    j.inv = 1.0f / 6.0f;
    j.red_target = jac_red ? c.scalars + ops[1].scalar : nullptr;
    j.partials = c.partials;
    j.red_done = c.red_done;
    // (programmatic dependent launch was measured here: 4.36 vs 4.12 us per
    // launch inside the graph -- slower, so plain launches)
    if (jac_red) k_jacobi8<true><<<num_sms() * SG_JAC8_MINB, 256, 0, s>>>(j);
    else k_jacobi8<false><<<num_sms() * SG_JAC8_MINB, 256, 0, s>>>(j);
    delete a;
    return check_launch();
  }
  // groups of quad ops on 8^3 dense blocks: the streaming kernel (k_jacobi8's
  // structure, no shared-memory tiles) instead of the tile interpreter
  const bool stream8 = stream8_group(t, ops, nops, gl, i32) && drive && drive->table && !ct &&
                       getenv("SG_NO_STREAM8") == nullptr;
  // JIT-specialized kernel of this group's content (jit.cpp);
  // the interpreter runs while it compiles
  if (!ct && !(pair && stencil)) {
    JitGroup G;
    const void* k = jit_group_of(t, ops, nops, G) ? jit_lookup(G) : nullptr;
    if (k) {
      void* args[] = {(void*)a};
      cudaLaunchKernel(k, dim3(G.stream ? num_sms() * 4 : grid), dim3(SF_TPB), args, 0, s);
      delete a;
      return check_launch();
    }
  }
  if (stream8) {
    k_stream8<<<num_sms() * 4, 256, 0, s>>>(*a);
    delete a;
    return check_launch();
  }
#define SG_SF_LAUNCH(V)                                                                           \
  switch (nd * 10 + gl) {                                                                         \
    case 10: sf_dispatch<V, 1, false, 0>(a, grid, s, ct); break;   \
    case 20: sf_dispatch<V, 2, false, 0>(a, grid, s, ct); break;   \
    case 23: sf_dispatch<V, 2, false, 3>(a, grid, s, ct); break;   \
    case 30: if (pair && stencil) sf_dispatch<V, 3, true, 0>(a, grid, s, ct); \
             else sf_dispatch<V, 3, false, 0>(a, grid, s, ct); break;          \
    case 31: sf_dispatch<V, 3, false, 1>(a, grid, s, ct); break;   \
    case 32: sf_dispatch<V, 3, false, 2>(a, grid, s, ct); break;   \
    default: sf_dispatch<V, 0, false, 0>(a, grid, s, ct); break;   \
  }
  if (i32) { SG_SF_LAUNCH(int) } else { SG_SF_LAUNCH(float) }
#undef SG_SF_LAUNCH
  delete a;
  delete ct;
  return check_launch();
}

}  // namespace sg
