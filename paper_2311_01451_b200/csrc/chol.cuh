// Blocked left-looking Cholesky of the near-field Gram, batched over the boxes
// of a colour, with the panel updates / panel TRSMs / back substitution run as
// DMMA GEMM tiles (nt_tile / nn_tile).  One CholDesc per matrix; the per-panel
// GEMM descriptors are derived inside the kernels (no descriptor explosion).
//
// Matrix (logical rows): C = Omega_near Omega_near^* in rows [0, r) (lower
// triangle valid) and B = Y_b Omega_near^* in physical rows [uoff, uoff + mextra).
// Result: L (C = L L^*) in the lower triangle, u = B L^-* in the B rows, then
// W = u L^-1 = Y_b Omega_near^dagger in the B rows.
// Panels of width CB = 64; L_JJ^-1 of every panel is kept in CholDesc::linv.
// Template C: complex128 (interleaved doubles; leading dimensions in complex units).
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace rsrs {

constexpr int CB = 64;
// panel width: 64 (real), 32 (complex: one 32-column complex GEMM tile per panel, so the
// in-place panel TRSM / back substitution tiles never read columns another tile writes)
template <bool C> constexpr int cbw() { return C ? 32 : 64; }

// P[j0:, J] -= L[j0:, 0:j0] L[J, 0:j0]^*   (z = 2*matrix + part; part 0: C rows, 1: B rows)
template <bool C>
__global__ void __launch_bounds__(128) chol_update_kernel(const CholDesc* __restrict__ cds, int j0) {
  constexpr int CBW = cbw<C>();
  extern __shared__ __align__(16) double smem[];
  constexpr int SC = C ? 2 : 1;
  const CholDesc& cd = cds[blockIdx.z >> 1];
  const int part = blockIdx.z & 1;
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r || j0 == 0) return;
  const int n = min(CBW, r - j0);
  const int jt = blockIdx.x * tile_n<C>();
  if (jt >= n) return;
  NTDesc d{};
  d.A = part ? cd.A + (i64)cd.uoff * cd.lda * SC : cd.A + (i64)j0 * cd.lda * SC;
  const int m = part ? cd.mextra : r - j0;
  const int i0 = blockIdx.y * GT;
  if (i0 >= m) return;
  d.lda = cd.lda;
  d.B = cd.A + (i64)j0 * cd.lda * SC;
  d.ldb = cd.lda;
  d.C = const_cast<double*>(d.A) + (i64)j0 * SC;
  d.ldc = cd.lda;
  d.alpha = -1.0;
  d.beta = 1.0;
  nt_tile_t<C>(d, m, n, j0, i0, jt, smem);
}

// Cholesky of the diagonal block P[J, J] (in place) and L_JJ^-1 (to linv[J])
constexpr int CHOL_DIAG_SMEM = 2 * CB * (CB + 1) * 8;   // >= the complex 32 x 32 case

template <bool C>
__global__ void __launch_bounds__(256) chol_diag_kernel(const CholDesc* __restrict__ cds, int j0) {
  constexpr int CBW = cbw<C>();
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double dsm[];
  S (*Ls)[CBW + 1] = reinterpret_cast<S (*)[CBW + 1]>(dsm);
  S (*Is)[CBW + 1] = reinterpret_cast<S (*)[CBW + 1]>(reinterpret_cast<S*>(dsm) + CBW * (CBW + 1));
  __shared__ int bad;
  const CholDesc& cd = cds[blockIdx.x];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int jb = min(CBW, r - j0);
  const int tid = threadIdx.x;
  const S zero = s_zero(S());
  S* A = reinterpret_cast<S*>(cd.A) + (i64)j0 * cd.lda + j0;
  for (int idx = tid; idx < CBW * CBW; idx += 256) {
    const int i = idx / CBW, j = idx % CBW;
    Ls[i][j] = (i < jb && j <= i) ? A[(i64)i * cd.lda + j] : zero;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < jb; ++c) {
    const double dcc = s_real(Ls[c][c]);
    if (!(dcc > 0.0)) {
      if (tid == 0) bad = 1;
      break;
    }
    const double lcc = sqrt(dcc);
    __syncthreads();
    for (int i = c + 1 + tid; i < jb; i += 256) Ls[i][c] = s_scale(Ls[i][c], 1.0 / lcc);
    if (tid == 0) Ls[c][c] = s_scale(s_one(S()), lcc);
    __syncthreads();
    const int nt = jb - c - 1;
    for (int idx = tid; idx < nt * nt; idx += 256) {
      const int i = c + 1 + idx / nt, j = c + 1 + idx % nt;
      if (j <= i) Ls[i][j] = s_sub(Ls[i][j], s_mulc(Ls[i][c], Ls[j][c]));
    }
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (tid == 0 && cd.status) *cd.status = ST_SINGULAR_GRAM;
    return;
  }
  // L^-1 column by column (lower triangular), zero padded to 64 x 64
  if (tid < CBW) {
    const int j = tid;
    for (int i = 0; i < CBW; ++i) Is[i][j] = zero;
    if (j < jb) {
      Is[j][j] = s_div(s_one(S()), Ls[j][j]);
      for (int i = j + 1; i < jb; ++i) {
        S s = zero;
        for (int q = j; q < i; ++q) s = s_add(s, s_mul(Ls[i][q], Is[q][j]));
        Is[i][j] = s_neg(s_div(s, Ls[i][i]));
      }
    }
  }
  __syncthreads();
  S* linv = reinterpret_cast<S*>(cd.linv) + (i64)(j0 / CBW) * CBW * CBW;
  for (int idx = tid; idx < CBW * CBW; idx += 256) {
    const int i = idx / CBW, j = idx % CBW;
    linv[idx] = Is[i][j];
    if (i < jb && j <= i) A[(i64)i * cd.lda + j] = Ls[i][j];
  }
}

// rows below the diagonal block: X <- X L_JJ^-*  (part 0: C rows [j0+64, r), 1: B rows)
template <bool C>
__global__ void __launch_bounds__(128) chol_trsm_kernel(const CholDesc* __restrict__ cds, int j0) {
  constexpr int CBW = cbw<C>();
  extern __shared__ __align__(16) double smem[];
  constexpr int SC = C ? 2 : 1;
  const CholDesc& cd = cds[blockIdx.z >> 1];
  const int part = blockIdx.z & 1;
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int jb = min(CBW, r - j0);
  const int jt = blockIdx.x * tile_n<C>();
  if (jt >= jb) return;
  const int m = part ? cd.mextra : r - j0 - CBW;
  const int i0 = blockIdx.y * GT;
  if (i0 >= m) return;
  NTDesc d{};
  d.A = part ? cd.A + ((i64)cd.uoff * cd.lda + j0) * SC : cd.A + ((i64)(j0 + CBW) * cd.lda + j0) * SC;
  d.lda = cd.lda;
  d.B = cd.linv + (i64)(j0 / CBW) * CBW * CBW * SC;
  d.ldb = CBW;
  d.C = const_cast<double*>(d.A);
  d.ldc = cd.lda;
  d.alpha = 1.0;
  d.beta = 0.0;
  nt_tile_t<C>(d, m, jb, jb, i0, jt, smem);   // in place: one column tile reads all of K before it writes
}

// back substitution, block J: W[:, J] = u[:, J] - W[:, J+] L[J+, J]
template <bool C>
__global__ void __launch_bounds__(128) chol_back_a_kernel(const CholDesc* __restrict__ cds, int j0) {
  constexpr int CBW = cbw<C>();
  extern __shared__ __align__(16) double smem[];
  constexpr int SC = C ? 2 : 1;
  const CholDesc& cd = cds[blockIdx.z];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int K = r - j0 - CBW;
  const int m = cd.mextra;
  const int i0 = blockIdx.y * GT;
  const int jt = blockIdx.x * tile_n<C>();
  const int n = min(CBW, r - j0);
  if (K <= 0 || i0 >= m || jt >= n) return;
  double* U = cd.A + (i64)cd.uoff * cd.lda * SC;
  NNDesc d{};
  d.A = U + (i64)(j0 + CBW) * SC;
  d.lda = cd.lda;
  d.B = cd.A + ((i64)(j0 + CBW) * cd.lda + j0) * SC;
  d.ldb = cd.lda;
  d.D = U + (i64)j0 * SC;
  d.ldd = cd.lda;
  d.alpha = -1.0;
  d.beta = 1.0;
  nn_tile_t<C>(d, m, n, K, i0, jt, smem);
}

// back substitution, block J: W[:, J] <- W[:, J] L_JJ^-1
template <bool C>
__global__ void __launch_bounds__(128) chol_back_b_kernel(const CholDesc* __restrict__ cds, int j0) {
  constexpr int CBW = cbw<C>();
  extern __shared__ __align__(16) double smem[];
  constexpr int SC = C ? 2 : 1;
  const CholDesc& cd = cds[blockIdx.z];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int jb = min(CBW, r - j0);
  const int m = cd.mextra;
  const int i0 = blockIdx.y * GT;
  const int jt = blockIdx.x * tile_n<C>();
  if (i0 >= m || jt >= jb) return;
  double* U = cd.A + (i64)cd.uoff * cd.lda * SC;
  NNDesc d{};
  d.A = U + (i64)j0 * SC;
  d.lda = cd.lda;
  d.B = cd.linv + (i64)(j0 / CBW) * CBW * CBW * SC;
  d.ldb = CBW;
  d.D = U + (i64)j0 * SC;
  d.ldd = cd.lda;
  d.alpha = 1.0;
  d.beta = 0.0;
  nn_tile_t<C>(d, m, jb, jb, i0, jt, smem);   // in place: one column tile reads all of K before it writes
}

}  // namespace rsrs
