// Blocked left-looking Cholesky of the near-field Gram, batched over the boxes
// of a colour, with the panel updates / panel TRSMs / back substitution run as
// DMMA GEMM tiles (nt_tile / nn_tile).  One CholDesc per matrix; the per-panel
// GEMM descriptors are derived inside the kernels (no descriptor explosion).
//
// Matrix (logical rows): C = Omega_near Omega_near^T in rows [0, r) (lower
// triangle valid) and B = Y_b Omega_near^T in physical rows [uoff, uoff + mextra).
// Result: L (C = L L^T) in the lower triangle, u = B L^-T in the B rows, then
// W = u L^-1 = Y_b Omega_near^dagger in the B rows.
// Panels of width CB = 64; L_JJ^-1 of every panel is kept in CholDesc::linv.
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace rsrs {

constexpr int CB = 64;

// P[j0:, J] -= L[j0:, 0:j0] L[J, 0:j0]^T   (z = 2*matrix + part; part 0: C rows, 1: B rows)
__global__ void __launch_bounds__(128) chol_update_kernel(const CholDesc* __restrict__ cds, int j0) {
  extern __shared__ __align__(16) double smem[];
  const CholDesc& cd = cds[blockIdx.z >> 1];
  const int part = blockIdx.z & 1;
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r || j0 == 0) return;
  const int n = min(CB, r - j0);
  NTDesc d{};
  d.A = part ? cd.A + (i64)cd.uoff * cd.lda : cd.A + (i64)j0 * cd.lda;
  const int m = part ? cd.mextra : r - j0;
  const int i0 = blockIdx.y * GT;
  if (i0 >= m) return;
  d.lda = cd.lda;
  d.B = cd.A + (i64)j0 * cd.lda;
  d.ldb = cd.lda;
  d.C = const_cast<double*>(d.A) + j0;
  d.ldc = cd.lda;
  d.alpha = -1.0;
  d.beta = 1.0;
  nt_tile(d, m, n, j0, i0, 0, smem);
}

// Cholesky of the diagonal block P[J, J] (in place) and L_JJ^-1 (to linv[J])
constexpr int CHOL_DIAG_SMEM = 2 * CB * (CB + 1) * 8;

__global__ void __launch_bounds__(256) chol_diag_kernel(const CholDesc* __restrict__ cds, int j0) {
  extern __shared__ __align__(16) double dsm[];
  double (*Ls)[CB + 1] = reinterpret_cast<double (*)[CB + 1]>(dsm);
  double (*Is)[CB + 1] = reinterpret_cast<double (*)[CB + 1]>(dsm + CB * (CB + 1));
  __shared__ int bad;
  const CholDesc& cd = cds[blockIdx.x];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int jb = min(CB, r - j0);
  const int tid = threadIdx.x;
  double* A = cd.A + (i64)j0 * cd.lda + j0;
  for (int idx = tid; idx < CB * CB; idx += 256) {
    const int i = idx / CB, j = idx % CB;
    Ls[i][j] = (i < jb && j <= i) ? A[(i64)i * cd.lda + j] : 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < jb; ++c) {
    const double dcc = Ls[c][c];
    if (!(dcc > 0.0)) {
      if (tid == 0) bad = 1;
      break;
    }
    const double lcc = sqrt(dcc);
    __syncthreads();
    for (int i = c + 1 + tid; i < jb; i += 256) Ls[i][c] /= lcc;
    if (tid == 0) Ls[c][c] = lcc;
    __syncthreads();
    const int nt = jb - c - 1;
    for (int idx = tid; idx < nt * nt; idx += 256) {
      const int i = c + 1 + idx / nt, j = c + 1 + idx % nt;
      if (j <= i) Ls[i][j] -= Ls[i][c] * Ls[j][c];
    }
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (tid == 0 && cd.status) *cd.status = ST_SINGULAR_GRAM;
    return;
  }
  // L^-1 column by column (lower triangular), zero padded to 64 x 64
  if (tid < CB) {
    const int j = tid;
    for (int i = 0; i < CB; ++i) Is[i][j] = 0.0;
    if (j < jb) {
      Is[j][j] = 1.0 / Ls[j][j];
      for (int i = j + 1; i < jb; ++i) {
        double s = 0.0;
        for (int q = j; q < i; ++q) s += Ls[i][q] * Is[q][j];
        Is[i][j] = -s / Ls[i][i];
      }
    }
  }
  __syncthreads();
  double* linv = cd.linv + (i64)(j0 / CB) * CB * CB;
  for (int idx = tid; idx < CB * CB; idx += 256) {
    const int i = idx / CB, j = idx % CB;
    linv[idx] = Is[i][j];
    if (i < jb && j <= i) A[(i64)i * cd.lda + j] = Ls[i][j];
  }
}

// rows below the diagonal block: X <- X L_JJ^-T  (part 0: C rows [j0+64, r), 1: B rows)
__global__ void __launch_bounds__(128) chol_trsm_kernel(const CholDesc* __restrict__ cds, int j0) {
  extern __shared__ __align__(16) double smem[];
  const CholDesc& cd = cds[blockIdx.z >> 1];
  const int part = blockIdx.z & 1;
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int jb = min(CB, r - j0);
  const int m = part ? cd.mextra : r - j0 - CB;
  const int i0 = blockIdx.y * GT;
  if (i0 >= m) return;
  NTDesc d{};
  d.A = part ? cd.A + (i64)cd.uoff * cd.lda + j0 : cd.A + (i64)(j0 + CB) * cd.lda + j0;
  d.lda = cd.lda;
  d.B = cd.linv + (i64)(j0 / CB) * CB * CB;
  d.ldb = CB;
  d.C = const_cast<double*>(d.A);
  d.ldc = cd.lda;
  d.alpha = 1.0;
  d.beta = 0.0;
  nt_tile(d, m, jb, jb, i0, 0, smem);   // in place: the tile reads all of K before it writes
}

// back substitution, block J: W[:, J] = u[:, J] - W[:, J+] L[J+, J]
__global__ void __launch_bounds__(128) chol_back_a_kernel(const CholDesc* __restrict__ cds, int j0) {
  extern __shared__ __align__(16) double smem[];
  const CholDesc& cd = cds[blockIdx.z];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int K = r - j0 - CB;
  const int m = cd.mextra;
  const int i0 = blockIdx.y * GT;
  if (K <= 0 || i0 >= m) return;
  double* U = cd.A + (i64)cd.uoff * cd.lda;
  NNDesc d{};
  d.A = U + j0 + CB;
  d.lda = cd.lda;
  d.B = cd.A + (i64)(j0 + CB) * cd.lda + j0;
  d.ldb = cd.lda;
  d.D = U + j0;
  d.ldd = cd.lda;
  d.alpha = -1.0;
  d.beta = 1.0;
  nn_tile(d, m, min(CB, r - j0), K, i0, 0, smem);
}

// back substitution, block J: W[:, J] <- W[:, J] L_JJ^-1
__global__ void __launch_bounds__(128) chol_back_b_kernel(const CholDesc* __restrict__ cds, int j0) {
  extern __shared__ __align__(16) double smem[];
  const CholDesc& cd = cds[blockIdx.z];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int jb = min(CB, r - j0);
  const int m = cd.mextra;
  const int i0 = blockIdx.y * GT;
  if (i0 >= m) return;
  double* U = cd.A + (i64)cd.uoff * cd.lda;
  NNDesc d{};
  d.A = U + j0;
  d.lda = cd.lda;
  d.B = cd.linv + (i64)(j0 / CB) * CB * CB;
  d.ldb = CB;
  d.D = U + j0;
  d.ldd = cd.lda;
  d.alpha = 1.0;
  d.beta = 0.0;
  nn_tile(d, m, jb, jb, i0, 0, smem);   // in place: the tile reads all of K before it writes
}

}  // namespace rsrs
