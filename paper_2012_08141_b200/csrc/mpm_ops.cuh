// mpm_ops.cuh -- MLS-MPM transfer ops (hu2018moving, the method PAPER.md:444
// evaluates; P2G "requires atomic add").  Included by kernels.cu
// after the tree helpers.  Quadratic B-spline weights over 3x3x3 nodes; the base
// node is decided in f32 with round-to-nearest intrinsics (no FMA contraction)
// exactly as the oracle does (reading R16).
//
// Arrays: a0 x (3 comps), a1 v (3), a2 C (9, row-major), a3 J (1); SoA with
// component c at ptr + c*n.  Grid fields f0..f2 velocity (momentum during P2G),
// f3 mass; they live in one tree whose leaf blocks are dense.
#pragma once

struct MpmKernel {
  int base[3];
  float fx[3];
  float w[3][3];
};

__device__ __forceinline__ MpmKernel mpm_bspline(const float xp[3], float inv_dx) {
  MpmKernel k;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    float X = __fmul_rn(xp[a], inv_dx);
    k.base[a] = (int)floorf(__fsub_rn(X, 0.5f));
    float fx = __fsub_rn(X, (float)k.base[a]);
    k.fx[a] = fx;
    float q0 = 1.5f - fx, q1 = fx - 1.0f, q2 = fx - 0.5f;
    k.w[0][a] = 0.5f * q0 * q0;
    k.w[1][a] = 0.75f - q1 * q1;
    k.w[2][a] = 0.5f * q2 * q2;
  }
  return k;
}

// Leaf blocks touched by the 3x3x3 stencil: at most 2 per axis.  blk[] holds the
// first cell (field slot 0) of each block, null if absent.
struct MpmBlocks {
  uint32_t* blk[2][2][2];
  int b0[3];      // block coords of base
  int lb[3];      // log2 block extents
};

template <bool ACTIVATE>
__device__ __forceinline__ void mpm_blocks(const DevCtx& C, const DTree& T, const int base[3], MpmBlocks& B, int task) {
  const int d = T.driving;
#pragma unroll
  for (int a = 0; a < 3; a++) { B.lb[a] = T.lev[d].lbelow[a]; B.b0[a] = base[a] >> B.lb[a]; }
  const uint32_t blkmask = ~((1u << T.lblk) - 1u);
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int k = 0; k < 2; k++) {
        int q[3] = {(B.b0[0] + i) << B.lb[0], (B.b0[1] + j) << B.lb[1], (B.b0[2] + k) << B.lb[2]};
        bool need = (((base[0] + 2) >> B.lb[0]) >= B.b0[0] + i) && (((base[1] + 2) >> B.lb[1]) >= B.b0[1] + j) &&
                    (((base[2] + 2) >> B.lb[2]) >= B.b0[2] + k);
        uint32_t* p = nullptr;
        if (need && in_domain(T, q)) {
          uint32_t idx;
          uint32_t* cont;
          if (ACTIVATE) {
            // activate the block by activating its cells' ancestors (dense leaf: any cell)
            cont = activate_walk(C, T, q, idx, task);
          } else {
            cont = locate(T, q, idx);
          }
          if (cont) p = cont + T.payload_off + (idx & blkmask);
        }
        B.blk[i][j][k] = p;
      }
}

__device__ __forceinline__ uint32_t* mpm_node(const DTree& T, const MpmBlocks& B, const int n[3]) {
  int i = (n[0] >> B.lb[0]) - B.b0[0], j = (n[1] >> B.lb[1]) - B.b0[1], k = (n[2] >> B.lb[2]) - B.b0[2];
  uint32_t* p = B.blk[i][j][k];
  if (!p) return nullptr;
  return p + inblock_idx(T, n);
}

__device__ void mpm_p2g(const DevCtx& C, const DOp& op, int64_t i, int task) {
  const DArray X = C.arrays[op.a[0]], Vv = C.arrays[op.a[1]], Cm = C.arrays[op.a[2]], Jj = C.arrays[op.a[3]];
  const float* x = (const float*)X.ptr;
  const float* v = (const float*)Vv.ptr;
  const float* cm = (const float*)Cm.ptr;
  const float* jj = (const float*)Jj.ptr;
  const float dt = op.p[0], inv_dx = op.p[1], pm = op.p[2], pv = op.p[3], E = op.p[4];
  const float dx = 1.0f / inv_dx;
  float xp[3] = {x[i], x[X.n + i], x[2 * X.n + i]};
  MpmKernel k = mpm_bspline(xp, inv_dx);
  float J = jj[i];
  float stress = -dt * 4.0f * E * pv * (J - 1.0f) * inv_dx * inv_dx;
  float aff[3][3], vel[3];
#pragma unroll
  for (int r = 0; r < 3; r++) {
    vel[r] = v[r * Vv.n + i];
#pragma unroll
    for (int c = 0; c < 3; c++) aff[r][c] = pm * cm[(3 * r + c) * Cm.n + i] + (r == c ? stress : 0.0f);
  }
  const DField& F0 = C.fields[op.f[0]];
  const DTree& T = C.trees[F0.tree];
  const uint64_t fs = 1ull << T.ln_leaf;
  int sl[4];
#pragma unroll
  for (int r = 0; r < 4; r++) sl[r] = C.fields[op.f[r]].slot;
  MpmBlocks B;
  if (op.act) mpm_blocks<true>(C, T, k.base, B, task);
  else mpm_blocks<false>(C, T, k.base, B, task);
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++)
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const float wgt = k.w[a][0] * k.w[b][1] * k.w[c][2];
        const float dpos[3] = {((float)a - k.fx[0]) * dx, ((float)b - k.fx[1]) * dx, ((float)c - k.fx[2]) * dx};
        int n[3] = {k.base[0] + a, k.base[1] + b, k.base[2] + c};
        uint32_t* p = mpm_node(T, B, n);
        if (!p) {
          if (C.debug) set_err(C, op.act ? SG_ERR_RANGE : SG_ERR_DEMOTION_TRAP, task);
          continue;
        }
#pragma unroll
        for (int r = 0; r < 3; r++) {
          float mom = pm * vel[r] + aff[r][0] * dpos[0] + aff[r][1] * dpos[1] + aff[r][2] * dpos[2];
          atomicAdd((float*)(p + sl[r] * fs), wgt * mom);
        }
        atomicAdd((float*)(p + sl[3] * fs), wgt * pm);
      }
}

__device__ void mpm_g2p(const DevCtx& C, const DOp& op, int64_t i) {
  const DArray X = C.arrays[op.a[0]], Vv = C.arrays[op.a[1]], Cm = C.arrays[op.a[2]], Jj = C.arrays[op.a[3]];
  float* x = (float*)X.ptr;
  float* v = (float*)Vv.ptr;
  float* cm = (float*)Cm.ptr;
  float* jj = (float*)Jj.ptr;
  const float dt = op.p[0], inv_dx = op.p[1];
  const float dx = 1.0f / inv_dx;
  float xp[3] = {x[i], x[X.n + i], x[2 * X.n + i]};
  MpmKernel k = mpm_bspline(xp, inv_dx);
  const DField& F0 = C.fields[op.f[0]];
  const DTree& T = C.trees[F0.tree];
  const uint64_t fs = 1ull << T.ln_leaf;
  int sl[3];
#pragma unroll
  for (int r = 0; r < 3; r++) sl[r] = C.fields[op.f[r]].slot;
  MpmBlocks B;
  mpm_blocks<false>(C, T, k.base, B, 0);
  float nv[3] = {0, 0, 0}, nC[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  const float s4 = 4.0f * inv_dx * inv_dx;
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++)
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const float wgt = k.w[a][0] * k.w[b][1] * k.w[c][2];
        const float dpos[3] = {((float)a - k.fx[0]) * dx, ((float)b - k.fx[1]) * dx, ((float)c - k.fx[2]) * dx};
        int n[3] = {k.base[0] + a, k.base[1] + b, k.base[2] + c};
        const uint32_t* p = mpm_node(T, B, n);
        if (!p) continue;
#pragma unroll
        for (int r = 0; r < 3; r++) {
          float g = __uint_as_float(p[sl[r] * fs]);
          nv[r] += wgt * g;
#pragma unroll
          for (int d = 0; d < 3; d++) nC[r][d] += s4 * wgt * g * dpos[d];
        }
      }
#pragma unroll
  for (int r = 0; r < 3; r++) {
    v[r * Vv.n + i] = nv[r];
    x[r * X.n + i] = xp[r] + dt * nv[r];
#pragma unroll
    for (int d = 0; d < 3; d++) cm[(3 * r + d) * Cm.n + i] = nC[r][d];
  }
  jj[i] = jj[i] * (1.0f + dt * (nC[0][0] + nC[1][1] + nC[2][2]));
}

// Grid update for one cell (struct-for).  base points at the cell in field slot 0.
__device__ __forceinline__ void mpm_grid_op(const DOp& op, const int c[3], uint32_t* cell0, uint64_t fs) {
  uint32_t* pv[3] = {cell0 + op.slot[0] * fs, cell0 + op.slot[1] * fs, cell0 + op.slot[2] * fs};
  const float m = __uint_as_float(cell0[op.slot[3] * fs]);
  float v[3] = {__uint_as_float(*pv[0]), __uint_as_float(*pv[1]), __uint_as_float(*pv[2])};
  if (m > 0.0f) {
#pragma unroll
    for (int a = 0; a < 3; a++) v[a] = v[a] / m;
  }
  v[1] -= op.p[0] * op.p[1];
  const float bound = op.p[2], n = op.p[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    bool cond = ((float)c[a] < bound && v[a] < 0.0f) || ((float)c[a] > n - bound && v[a] > 0.0f);
    if (cond) v[a] = 0.0f;
  }
#pragma unroll
  for (int a = 0; a < 3; a++) *pv[a] = __float_as_uint(v[a]);
}
