// mpm_adj.cuh -- C4 differentiable MPM: the hand-written adjoints of the MPM
// transfer ops (every kernel has a gradient kernel; the particle
// states of all substeps are the checkpoints), the loss and the adjoint seed.
// Included by kernels.cu after mpm_ops.cuh.  The math is derived in DESIGN.md
// "C4" (reading R31); both sides follow it, the oracle in f64.
//
//   G2P_ADJ  adjoint of GRID_OP (folded: the grid velocity u = mask * (p/m -
//            dt g e_y) is recomputed from the recomputed P2G momentum p and mass
//            m) and of G2P.  Gathers p, m from the grid tree; scatters the
//            adjoints of p and m into a second tree (activating atomics).
//   P2G_ADJ  adjoint of P2G: gathers the grid adjoints at the 27 nodes.
//   LOSS_MEAN  deterministic f64 reduction over the particles into a 0-D field.
//   ADJ_INIT   d loss / d x_T seed.
#pragma once

// d w / d fx of the quadratic B-spline (per axis), fx from mpm_bspline.
__device__ __forceinline__ void mpm_dw(const MpmKernel& k, float dw[3][3]) {
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const float q = k.fx[a];
    dw[0][a] = q - 1.5f;
    dw[1][a] = -2.0f * (q - 1.0f);
    dw[2][a] = q - 0.5f;
  }
}

__device__ __forceinline__ const float* arr_f(const DevCtx& C, int id) { return (const float*)C.arrays[id].ptr; }

struct Mpm2Args {
  DTree T;     // grid tree (p, m)            -- G2P_ADJ; the adjoint tree for P2G_ADJ
  DTree TG;    // adjoint tree (p_bar, m_bar) -- G2P_ADJ only
  DevCtx C;
  DOp op;
  int64_t n;
  int task;
};

template <int LB>
__device__ __forceinline__ void mpm_g2p_adj(const DevCtx& C, const DTree& T, const DTree& TG, const DOp& op,
                                            int64_t i, int task) {
  const DArray X = C.arrays[op.a[0]];
  const int64_t nx = X.n;
  const float* x = (const float*)X.ptr;
  const float* jj = arr_f(C, op.a[1]);
  const float *xb1 = arr_f(C, op.a[2]), *vb1 = arr_f(C, op.a[3]), *cb1 = arr_f(C, op.a[4]), *jb1 = arr_f(C, op.a[5]);
  const int64_t n1x = C.arrays[op.a[2]].n, n1v = C.arrays[op.a[3]].n, n1c = C.arrays[op.a[4]].n;
  float* xb0 = (float*)C.arrays[op.a[6]].ptr;
  float* jb0 = (float*)C.arrays[op.a[7]].ptr;
  const int64_t n0x = C.arrays[op.a[6]].n;
  const float dt = op.p[0], inv_dx = op.p[1], grav = op.p[2], bound = op.p[3], ng = op.p[4];
  const float dx = 1.0f / inv_dx, s4 = 4.0f * inv_dx * inv_dx;

  float xp[3] = {x[i], x[nx + i], x[2 * nx + i]};
  const MpmKernel k = mpm_bspline(xp, inv_dx);
  float dw[3][3];
  mpm_dw(k, dw);
  const float J = jj[i], Jb1 = jb1[i];
  float vt[3], Ct[3][3];
#pragma unroll
  for (int r = 0; r < 3; r++) {
    vt[r] = vb1[r * n1v + i] + dt * xb1[r * n1x + i];
#pragma unroll
    for (int d = 0; d < 3; d++) Ct[r][d] = cb1[(3 * r + d) * n1c + i] + (r == d ? Jb1 * J * dt : 0.0f);
  }

  const uint64_t fs = 1ull << T.ln_leaf, fsg = 1ull << TG.ln_leaf;
  const uint32_t* pool = T.seg[T.nseg - 1].base;
  uint32_t* poolg = TG.seg[TG.nseg - 1].base;
  const float* gp[4];
  float* gb[4];
#pragma unroll
  for (int r = 0; r < 4; r++) {
    gp[r] = (const float*)(pool + (uint64_t)op.slot[r] * fs);
    gb[r] = (float*)(poolg + (uint64_t)op.slot[4 + r] * fsg);
  }
  MpmBlocks B, BG;
  mpm_blocks<false, LB>(C, T, k.base, B, task);
  if (op.act) mpm_blocks<true, LB>(C, TG, k.base, BG, task);
  else mpm_blocks<false, LB>(C, TG, k.base, BG, task);

  auto node_u = [&](uint32_t off, int a, int b, int c, float pn[3], float& m, float u[3], float mask[3]) {
    m = 0.0f;
    pn[0] = pn[1] = pn[2] = 0.0f;
    if (off != SG_NO_BLOCK) {
      pn[0] = gp[0][off]; pn[1] = gp[1][off]; pn[2] = gp[2][off]; m = gp[3][off];
    }
    const int node[3] = {k.base[0] + a, k.base[1] + b, k.base[2] + c};
#pragma unroll
    for (int r = 0; r < 3; r++) u[r] = m > 0.0f ? pn[r] / m : pn[r];
    u[1] -= dt * grav;
#pragma unroll
    for (int r = 0; r < 3; r++) {
      const bool z = ((float)node[r] < bound && u[r] < 0.0f) || ((float)node[r] > ng - bound && u[r] > 0.0f);
      mask[r] = z ? 0.0f : 1.0f;
      if (z) u[r] = 0.0f;
    }
  };

  // pass 1: tr C_{s+1} (for the J adjoint)
  float trC = 0.0f;
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++)
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const uint32_t off = mpm_node_off<LB>(T, B, k.base, a, b, c);
        float pn[3], m, u[3], mask[3];
        node_u(off, a, b, c, pn, m, u, mask);
        const float W = k.w[a][0] * k.w[b][1] * k.w[c][2];
        trC += s4 * W * (u[0] * ((float)a - k.fx[0]) + u[1] * ((float)b - k.fx[1]) + u[2] * ((float)c - k.fx[2])) * dx;
      }
  const float Jb = Jb1 * (1.0f + dt * trC);

  // pass 2: adjoints of the node velocities -> grid adjoints; particle x adjoint
  float xb[3] = {xb1[i], xb1[n1x + i], xb1[2 * n1x + i]};
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++)
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const uint32_t off = mpm_node_off<LB>(T, B, k.base, a, b, c);
        float pn[3], m, u[3], mask[3];
        node_u(off, a, b, c, pn, m, u, mask);
        const float W = k.w[a][0] * k.w[b][1] * k.w[c][2];
        const float gW[3] = {inv_dx * dw[a][0] * k.w[b][1] * k.w[c][2], inv_dx * k.w[a][0] * dw[b][1] * k.w[c][2],
                             inv_dx * k.w[a][0] * k.w[b][1] * dw[c][2]};
        const float dpos[3] = {((float)a - k.fx[0]) * dx, ((float)b - k.fx[1]) * dx, ((float)c - k.fx[2]) * dx};
        float Wbar = 0.0f, dposbar[3] = {0.0f, 0.0f, 0.0f}, gbar[3];
#pragma unroll
        for (int r = 0; r < 3; r++) {
          const float ct = Ct[r][0] * dpos[0] + Ct[r][1] * dpos[1] + Ct[r][2] * dpos[2];
          gbar[r] = W * (vt[r] + s4 * ct);
          Wbar += u[r] * (vt[r] + s4 * ct);
#pragma unroll
          for (int d = 0; d < 3; d++) dposbar[d] += s4 * W * Ct[r][d] * u[r];
        }
#pragma unroll
        for (int d = 0; d < 3; d++) xb[d] += Wbar * gW[d] - dposbar[d];
        const uint32_t og = mpm_node_off<LB>(TG, BG, k.base, a, b, c);
        if (og == SG_NO_BLOCK) {
          if (C.debug) set_err(C, op.act ? SG_ERR_RANGE : SG_ERR_DEMOTION_TRAP, task);
          continue;
        }
        float mb = 0.0f;
#pragma unroll
        for (int r = 0; r < 3; r++) {
          const float ub = gbar[r] * mask[r];
          const float pb = m > 0.0f ? ub / m : ub;
          atomicAdd(gb[r] + og, pb);
          if (m > 0.0f) mb -= pb * (pn[r] / m);   // (ub/m)(p/m): m*m underflows in f32 at the cloud's rim
        }
        atomicAdd(gb[3] + og, mb);
      }
#pragma unroll
  for (int d = 0; d < 3; d++) xb0[d * n0x + i] = xb[d];
  jb0[i] = Jb;
}

template <int LB>
__device__ __forceinline__ void mpm_p2g_adj(const DevCtx& C, const DTree& T, const DOp& op, int64_t i, int task) {
  const DArray X = C.arrays[op.a[0]];
  const int64_t nx = X.n, nv = C.arrays[op.a[1]].n, nc = C.arrays[op.a[2]].n;
  const float* x = (const float*)X.ptr;
  const float *v = arr_f(C, op.a[1]), *cm = arr_f(C, op.a[2]), *jj = arr_f(C, op.a[3]);
  float* xb = (float*)C.arrays[op.a[4]].ptr;
  float* vb = (float*)C.arrays[op.a[5]].ptr;
  float* cb = (float*)C.arrays[op.a[6]].ptr;
  float* jb = (float*)C.arrays[op.a[7]].ptr;
  const int64_t nxb = C.arrays[op.a[4]].n, nvb = C.arrays[op.a[5]].n, ncb = C.arrays[op.a[6]].n;
  const float dt = op.p[0], inv_dx = op.p[1], pm = op.p[2], pv = op.p[3], E = op.p[4];
  const float dx = 1.0f / inv_dx;
  const float kJ = -dt * 4.0f * E * pv * inv_dx * inv_dx;

  float xp[3] = {x[i], x[nx + i], x[2 * nx + i]};
  const MpmKernel k = mpm_bspline(xp, inv_dx);
  float dw[3][3];
  mpm_dw(k, dw);
  const float J = jj[i];
  float vv[3], Am[3][3];
#pragma unroll
  for (int r = 0; r < 3; r++) {
    vv[r] = v[r * nv + i];
#pragma unroll
    for (int c = 0; c < 3; c++) Am[r][c] = pm * cm[(3 * r + c) * nc + i] + (r == c ? kJ * (J - 1.0f) : 0.0f);
  }
  const uint64_t fs = 1ull << T.ln_leaf;
  const uint32_t* pool = T.seg[T.nseg - 1].base;
  const float* gb[4];
#pragma unroll
  for (int r = 0; r < 4; r++) gb[r] = (const float*)(pool + (uint64_t)op.slot[r] * fs);
  MpmBlocks B;
  mpm_blocks<false, LB>(C, T, k.base, B, task);
  float xbar[3] = {0.0f, 0.0f, 0.0f}, vbar[3] = {0.0f, 0.0f, 0.0f}, Ab[3][3];
#pragma unroll
  for (int r = 0; r < 3; r++)
#pragma unroll
    for (int d = 0; d < 3; d++) Ab[r][d] = 0.0f;
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++)
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const uint32_t off = mpm_node_off<LB>(T, B, k.base, a, b, c);
        if (off == SG_NO_BLOCK) continue;   // inactive adjoint node reads 0
        const float pb[3] = {gb[0][off], gb[1][off], gb[2][off]};
        const float mb = gb[3][off];
        const float W = k.w[a][0] * k.w[b][1] * k.w[c][2];
        const float gW[3] = {inv_dx * dw[a][0] * k.w[b][1] * k.w[c][2], inv_dx * k.w[a][0] * dw[b][1] * k.w[c][2],
                             inv_dx * k.w[a][0] * k.w[b][1] * dw[c][2]};
        const float dpos[3] = {((float)a - k.fx[0]) * dx, ((float)b - k.fx[1]) * dx, ((float)c - k.fx[2]) * dx};
        float Wbar = mb * pm, dposbar[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int r = 0; r < 3; r++) {
          const float mom = pm * vv[r] + Am[r][0] * dpos[0] + Am[r][1] * dpos[1] + Am[r][2] * dpos[2];
          Wbar += pb[r] * mom;
          vbar[r] += W * pm * pb[r];
#pragma unroll
          for (int d = 0; d < 3; d++) {
            Ab[r][d] += W * pb[r] * dpos[d];
            dposbar[d] += W * pb[r] * Am[r][d];
          }
        }
#pragma unroll
        for (int d = 0; d < 3; d++) xbar[d] += Wbar * gW[d] - dposbar[d];
      }
#pragma unroll
  for (int d = 0; d < 3; d++) {
    xb[d * nxb + i] += xbar[d];
    vb[d * nvb + i] = vbar[d];
#pragma unroll
    for (int c = 0; c < 3; c++) cb[(3 * d + c) * ncb + i] = pm * Ab[d][c];
  }
  jb[i] += kJ * (Ab[0][0] + Ab[1][1] + Ab[2][2]);
}

template <int LB>
__global__ void __launch_bounds__(128, 3) k_g2p_adj(const __grid_constant__ Mpm2Args A) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * blockDim.x)
    mpm_g2p_adj<LB>(A.C, A.T, A.TG, A.op, i, A.task);
}

template <int LB>
__global__ void __launch_bounds__(128, 4) k_p2g_adj(const __grid_constant__ Mpm2Args A) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * blockDim.x)
    mpm_p2g_adj<LB>(A.C, A.T, A.op, i, A.task);
}

// ADJ_INIT: a0[p0][i] = p1, every other entry of a0..a3 = 0 (generic range-for body).
__device__ __forceinline__ void adj_init(const DevCtx& C, const DOp& op, int64_t i) {
  const int comp = (int)op.p[0];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const DArray a = C.arrays[op.a[k]];
    float* p = (float*)a.ptr;
    for (int c = 0; c < a.ncomp; c++) p[c * a.n + i] = (k == 0 && c == comp) ? op.p[1] : 0.0f;
  }
}

// LOSS_MEAN: f0[] += p1 * sum_i a0[p0][i].  Each thread sums a fixed strided
// subsequence in f64, the CTA tree-reduces in shared memory, CTA partials go
// to global memory and the last CTA adds them in CTA order: deterministic.
constexpr int LM_TPB = 256;
struct LossArgs {
  DevCtx C;
  DOp op;
  int64_t n;
  uint32_t* target;
};

__global__ void __launch_bounds__(LM_TPB) k_loss_mean(const __grid_constant__ LossArgs A) {
  __shared__ double s[LM_TPB];
  __shared__ bool s_last;
  const DArray X = A.C.arrays[A.op.a[0]];
  const float* x = (const float*)X.ptr + (int64_t)(int)A.op.p[0] * X.n;
  double t = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)LM_TPB + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * LM_TPB)
    t += (double)x[i];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int w = LM_TPB / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) A.C.partials[blockIdx.x] = s[0];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(A.C.red_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double u = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += LM_TPB) u += __ldcg(&A.C.partials[b]);
  s[threadIdx.x] = u;
  __syncthreads();
  for (int w = LM_TPB / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float old = __uint_as_float(*A.target);
    *A.target = __float_as_uint((float)((double)old + (double)A.op.p[1] * s[0]));
    *A.C.red_done = 0u;
  }
}
