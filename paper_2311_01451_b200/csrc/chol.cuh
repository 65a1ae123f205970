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

// Cholesky of the diagonal block P[J, J] (in place) and L_JJ^-1 (to linv[J]).
// Gaussian elimination without pivoting on the augmented [C_JJ | I] held in
// REGISTERS (thread t owns rows t/16 + 16a, columns t%16 + 16b): after step c,
// C = Lt D Lt^* gives L[:, c] = a[:, c] / sqrt(d_c) and the I part becomes
// Lt^-1, so L^-1 = D^-1/2 Lt^-1 comes out of the same sweep (no serial
// triangular inverse).  One barrier per column (column c and row c are
// broadcast through double-buffered shared memory).

template <bool C>
__global__ void __launch_bounds__(256, 3) chol_diag_kernel(const CholDesc* __restrict__ cds, int j0) {
  constexpr int CBW = cbw<C>();
  typedef typename ScalarOf<C>::T S;
  constexpr int RA = CBW / 16, CA = 2 * CBW / 16;      // owned rows / columns per thread
  __shared__ S colbuf[2][CBW];
  __shared__ S rowbuf[2][2 * CBW];
  __shared__ double pivs[CBW];
  const CholDesc& cd = cds[blockIdx.x];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  const int jb = min(CBW, r - j0);
  const int tid = threadIdx.x;
  const int tr = tid >> 4, tc = tid & 15;
  const S zero = s_zero(S()), one = s_one(S());
  S* A = reinterpret_cast<S*>(cd.A) + (i64)j0 * cd.lda + j0;
  S a[RA][CA];
#pragma unroll
  for (int ra = 0; ra < RA; ++ra) {
    const int i = tr + 16 * ra;
#pragma unroll
    for (int cb = 0; cb < CA; ++cb) {
      const int j = tc + 16 * cb;
      S v;
      if (j < CBW) {   // C part: Hermitian from the lower triangle; identity on padding rows
        if (i < jb && j < jb) v = (j <= i) ? A[(i64)i * cd.lda + j] : s_conj(A[(i64)j * cd.lda + i]);
        else v = (i == j) ? one : zero;
      } else {
        v = (j - CBW == i) ? one : zero;
      }
      a[ra][cb] = v;
    }
  }
  bool bad = false;
  // c = 16 * cblk + cc: the owned slot of column / row c is the compile-time cblk
#pragma unroll
  for (int cblk = 0; cblk < CBW / 16; ++cblk) {
    for (int cc = 0; cc < 16 && !bad; ++cc) {
      const int c = 16 * cblk + cc;
      if (c >= jb) break;
      const int buf = c & 1;
      if (tc == cc)                       // owners of column c (C part)
#pragma unroll
        for (int ra = 0; ra < RA; ++ra) colbuf[buf][tr + 16 * ra] = a[ra][cblk];
      if (tr == cc) {                     // owners of row c publish the multiplier row a[c, :] / piv
        // (the pivot a[c, c] sits in the same thread row; its owner is (tr, tc) = (cc, cc))
        const double pv = s_real(a[cblk][cblk]);
        const double rp = 1.0 / __shfl_sync(0xffffu << (threadIdx.x & 16), pv, cc, 16);
#pragma unroll
        for (int cb = 0; cb < CA; ++cb) rowbuf[buf][tc + 16 * cb] = s_scale(a[cblk][cb], rp);
      }
      __syncthreads();
      const double piv = s_real(colbuf[buf][c]);
      if (!(piv > 0.0)) {
        bad = true;
        break;
      }
      if (tid < jb && tid >= c) A[(i64)tid * cd.lda + c] = colbuf[buf][tid];   // unscaled L[:, c] * sqrt(piv)
      if (tid == 0) pivs[c] = piv;
      // rows i > c: a[i, :] -= a[i, c] (a[c, :] / piv)
      S rb[CA];
#pragma unroll
      for (int cb = 0; cb < CA; ++cb) rb[cb] = rowbuf[buf][tc + 16 * cb];
      // compile-time skips (cblk is unrolled): owned rows below 16 cblk are finished, C columns
      // below 16 cblk are never read again, I columns from 16 (cblk + 1) on are zero in row c
#pragma unroll
      for (int ra = 0; ra < RA; ++ra) {
        if (ra < cblk) continue;
        const int i = tr + 16 * ra;
        const S m = (i > c) ? colbuf[buf][i] : zero;
#pragma unroll
        for (int cb = 0; cb < CA; ++cb) {
          if (cb < CA / 2 && cb < cblk) continue;
          if (cb >= CA / 2 && cb - CA / 2 > cblk) continue;
          a[ra][cb] = s_sub(a[ra][cb], s_mul(m, rb[cb]));
        }
      }
    }
  }
  if (bad) {
    if (tid == 0 && cd.status) *cd.status = ST_SINGULAR_GRAM;
    return;
  }
  __syncthreads();
  if (tid < jb) pivs[tid] = rsqrt(pivs[tid]);
  __syncthreads();
  // L[:, c] = column c at step c / sqrt(piv_c)
  for (int idx = tid; idx < jb * jb; idx += 256) {
    const int i = idx / jb, c = idx - i * jb;
    if (i >= c) A[(i64)i * cd.lda + c] = s_scale(A[(i64)i * cd.lda + c], pivs[c]);
  }
  // L^-1 = D^-1/2 Lt^-1 (zero padded beyond jb)
  S* linv = reinterpret_cast<S*>(cd.linv) + (i64)(j0 / CBW) * CBW * CBW;
#pragma unroll
  for (int ra = 0; ra < RA; ++ra) {
    const int i = tr + 16 * ra;
#pragma unroll
    for (int cb = 0; cb < CA; ++cb) {
      const int j = tc + 16 * cb;
      if (j < CBW) continue;
      const int jj = j - CBW;
      linv[i * CBW + jj] = (i < jb && jj < jb) ? s_scale(a[ra][cb], pivs[i]) : zero;
    }
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

// ---------------------------------------------------------------------------
// Fused per-matrix Cholesky (real): one 128-thread CTA runs the whole blocked
// left-looking factorization of one near-field Gram (update tiles, diagonal
// block, TRSM tiles, panel after panel) and, in a second launch, the whole back
// substitution.  Same arithmetic as the per-panel kernels above (one launch per
// colour batch instead of ~3 per panel): small near fields (the sphere's leaves,
// r <= ~256) are latency-bound on the per-panel launch chain, and independent
// matrices now overlap each other's serial diagonal steps on the SM.

// 64 x 64 diagonal block by in-register elimination on [C_JJ | I], 128 threads:
// thread (tr, tc) = (tid / 16, tid % 16) owns rows tr + 8 ra (ra < 8) and columns
// tc + 16 cb (cb < 8; cb >= 4: the I part).  Row c = 8 cb8 + cc is owned by tr = cc
// in slot ra = cb8; column c by tc = c % 16 in slot cb = cb8 / 2 (both compile time).
RSRS_DI bool chol_diag_block128(const CholDesc& cd, int j0, int r, double* smem) {
  constexpr int TR = 8, RA = CB / TR, CA = 2 * CB / 16;
  // broadcast buffers alias the (idle) GEMM staging memory
  double (*colbuf)[CB] = reinterpret_cast<double (*)[CB]>(smem);
  double (*rowbuf)[2 * CB] = reinterpret_cast<double (*)[2 * CB]>(smem + 2 * CB);
  double* pivs = smem + 6 * CB;
  int& sbad = *reinterpret_cast<int*>(smem + 7 * CB);
  const int jb = min(CB, r - j0);
  const int tid = threadIdx.x;
  const int tr = tid >> 4, tc = tid & 15;
  double* A = cd.A + (i64)j0 * cd.lda + j0;
  double a[RA][CA];
#pragma unroll
  for (int ra = 0; ra < RA; ++ra) {
    const int i = tr + TR * ra;
#pragma unroll
    for (int cb = 0; cb < CA; ++cb) {
      const int j = tc + 16 * cb;
      double v;
      if (j < CB) {
        if (i < jb && j < jb) v = (j <= i) ? A[(i64)i * cd.lda + j] : A[(i64)j * cd.lda + i];
        else v = (i == j) ? 1.0 : 0.0;
      } else {
        v = (j - CB == i) ? 1.0 : 0.0;
      }
      a[ra][cb] = v;
    }
  }
  if (tid == 0) sbad = 0;
  bool bad = false;
#pragma unroll
  for (int cb8 = 0; cb8 < CB / TR; ++cb8) {
    const int cbc = cb8 >> 1;                 // column slot of c
    for (int cc = 0; cc < TR && !bad; ++cc) {
      const int c = TR * cb8 + cc;
      if (c >= jb) break;
      const int buf = c & 1;
      const int ctc = (cb8 & 1) * 8 + cc;     // c % 16
      if (tc == ctc)
#pragma unroll
        for (int ra = 0; ra < RA; ++ra) colbuf[buf][tr + TR * ra] = a[ra][cbc];
      if (tr == cc) {
        const double pv = a[cb8][cbc];
        const double rp = 1.0 / __shfl_sync(0xffffu << (threadIdx.x & 16), pv, ctc, 16);
#pragma unroll
        for (int cb = 0; cb < CA; ++cb) rowbuf[buf][tc + 16 * cb] = a[cb8][cb] * rp;
      }
      __syncthreads();
      const double piv = colbuf[buf][c];
      if (!(piv > 0.0)) {
        bad = true;
        break;
      }
      if (tid < jb && tid >= c) A[(i64)tid * cd.lda + c] = colbuf[buf][tid];
      if (tid == 0) pivs[c] = piv;
      double rb[CA];
#pragma unroll
      for (int cb = 0; cb < CA; ++cb) rb[cb] = rowbuf[buf][tc + 16 * cb];
#pragma unroll
      for (int ra = 0; ra < RA; ++ra) {
        if (ra < cb8) continue;               // rows below 8 cb8 are finished
        const int i = tr + TR * ra;
        const double m = (i > c) ? colbuf[buf][i] : 0.0;
#pragma unroll
        for (int cb = 0; cb < CA; ++cb) {
          if (cb < CA / 2 && cb < cbc) continue;               // C columns below 16 cbc: never read again
          if (cb >= CA / 2 && cb - CA / 2 > cbc) continue;     // I columns beyond 16 (cbc + 1): zero in row c
          a[ra][cb] -= m * rb[cb];
        }
      }
    }
  }
  if (bad) sbad = 1;                           // every thread sees the same pivot: uniform
  __syncthreads();
  if (sbad) return false;
  if (tid < jb) pivs[tid] = rsqrt(pivs[tid]);
  __syncthreads();
  for (int idx = tid; idx < jb * jb; idx += 128) {
    const int i = idx / jb, c = idx - i * jb;
    if (i >= c) A[(i64)i * cd.lda + c] *= pivs[c];
  }
  double* linv = cd.linv + (i64)(j0 / CB) * CB * CB;
#pragma unroll
  for (int ra = 0; ra < RA; ++ra) {
    const int i = tr + TR * ra;
#pragma unroll
    for (int cb = CA / 2; cb < CA; ++cb) {
      const int jj = tc + 16 * (cb - CA / 2);
      linv[i * CB + jj] = (i < jb && jj < jb) ? a[ra][cb] * pivs[i] : 0.0;
    }
  }
  return true;
}

// ---------------------------------------------------------------------------
// Two-level diagonal block (real, 128 threads).  The 64 x 64 block A_JJ is factored
// in 16 x 16 sub-blocks (right-looking): each diagonal sub-block is eliminated by ONE
// warp, warp-synchronously (lane j owns column j of the augmented [A_kk | I]; 16
// shuffle steps, no CTA barrier), giving L_kk and X_k = L_kk^-1 in the same sweep as
// chol_diag_kernel (Gaussian elimination without pivoting: A = Lt D Lt^T, the I part
// becomes Lt^-1, L = Lt D^1/2, L^-1 = D^-1/2 Lt^-1).  The sub-panel L_ik = A_ik X_k^T,
// the trailing update A_ij -= L_ik L_jk^T and the block inverse
// (L^-1)_ik = -X_i sum_{k<=m<i} L_im (L^-1)_mk run on all 128 threads from shared
// memory: about 20 CTA barriers per 64 columns instead of 64 column steps.
// Shared memory: S [64][65] (lower: A -> L; strictly upper blocks (k, i), k < i:
// (L^-1)_ik^T), X [4][16][17], T [3][16][17].  Same outputs as chol_diag_kernel
// (L in the lower triangle of A_JJ, L_JJ^-1 zero padded beyond jb in linv[J]).
constexpr int D16_LD = CB + 1;
constexpr int D16_XS = 16 * 17;
constexpr int D16_SMEM = (CB * D16_LD + 7 * D16_XS) * 8 + 16;

// warp: 16 x 16 diagonal sub-block k of S -> L_kk (lower, in S), X_k (to X); false on a
// non-positive pivot (uniform over the warp)
RSRS_DI bool chol16_warp(double* S, int k, double* X) {
  const int lane = threadIdx.x & 31;
  const int o = 16 * k;
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (lane < 16) a[i] = (i >= lane) ? S[(o + i) * D16_LD + o + lane] : S[(o + lane) * D16_LD + o + i];
    else a[i] = (i == lane - 16) ? 1.0 : 0.0;
  }
  double rs[16];
  double myrs = 1.0;
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    // the multipliers a[i][c] (lane c) are final before step c: issue their shuffles first
    double m[16];
#pragma unroll
    for (int i = c + 1; i < 16; ++i) m[i] = __shfl_sync(0xffffffffu, a[i], c);
    const double p = __shfl_sync(0xffffffffu, a[c], c);
    ok = ok && (p > 0.0);
    const double rp = 1.0 / p;
    rs[c] = rsqrt(p);
    if (lane == c) myrs = rs[c];
    // lane c keeps its column (= L[:, c] sqrt(d_c) for rows >= c); lanes < c hold a zero in row c
    const double rowc = (lane == c) ? 0.0 : a[c] * rp;
#pragma unroll
    for (int i = c + 1; i < 16; ++i) a[i] -= m[i] * rowc;
  }
  if (!ok) return false;
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i >= lane) S[(o + i) * D16_LD + o + lane] = a[i] * myrs;
  } else {
    const int jj = lane - 16;
#pragma unroll
    for (int i = 0; i < 16; ++i) X[i * 17 + jj] = a[i] * rs[i];   // zero above the diagonal
  }
  return true;
}

// false on a non-positive pivot (every thread)
RSRS_DI bool chol_diag16(const CholDesc& cd, int j0, int r, double* smem) {
  double* S = smem;
  double* Xb = S + CB * D16_LD;
  double* Tb = Xb + 4 * D16_XS;
  int& sbad = *reinterpret_cast<int*>(Tb + 3 * D16_XS);
  const int jb = min(CB, r - j0);
  const int nkb = (jb + 15) >> 4;
  const int tid = threadIdx.x, warp = tid >> 5;
  double* A = cd.A + (i64)j0 * cd.lda + j0;
  for (int idx = tid; idx < CB * CB; idx += 128) {
    const int i = idx >> 6, j = idx & 63;
    if (j <= i && i < 16 * nkb) S[i * D16_LD + j] = (i < jb && j < jb) ? A[(i64)i * cd.lda + j] : (i == j ? 1.0 : 0.0);
  }
  if (tid == 0) sbad = 0;
  __syncthreads();
  for (int k = 0; k < nkb; ++k) {
    if (warp == 0 && !chol16_warp(S, k, Xb + k * D16_XS) && (tid & 31) == 0) sbad = 1;
    __syncthreads();
    if (sbad) return false;
    const int nb = nkb - 1 - k;
    if (nb <= 0) break;
    // L_ik = A_ik X_k^T (k < i < nkb), in place through registers
    {
      const double* Xk = Xb + k * D16_XS;
      double v[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int idx = tid + 128 * q;
        v[q] = 0.0;
        if (idx < nb * 256) {
          const int ib = k + 1 + (idx >> 8), rr = (idx >> 4) & 15, cc = idx & 15;
          const double* srow = S + (16 * ib + rr) * D16_LD + 16 * k;
          double s = 0.0;
#pragma unroll
          for (int mm = 0; mm < 16; ++mm) s += (mm <= cc) ? srow[mm] * Xk[cc * 17 + mm] : 0.0;
          v[q] = s;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int idx = tid + 128 * q;
        if (idx < nb * 256) {
          const int ib = k + 1 + (idx >> 8), rr = (idx >> 4) & 15, cc = idx & 15;
          S[(16 * ib + rr) * D16_LD + 16 * k + cc] = v[q];
        }
      }
      __syncthreads();
    }
    // trailing A_ij -= L_ik L_jk^T, k < j <= i < nkb (lower triangle of the diagonal blocks)
    {
      const int npair = nb * (nb + 1) / 2;
      for (int idx = tid; idx < npair * 256; idx += 128) {
        int pi = idx >> 8, ib = k + 1, jbk = k + 1;
        // pair pi -> (ib, jbk) in the order (k+1,k+1), (k+2,k+1), (k+2,k+2), ...
        for (int t = 1; t <= nb; ++t) {
          if (pi < t) { ib = k + t; jbk = k + 1 + pi; break; }
          pi -= t;
        }
        const int rr = (idx >> 4) & 15, cc = idx & 15;
        if (ib == jbk && cc > rr) continue;
        const double* li = S + (16 * ib + rr) * D16_LD + 16 * k;
        const double* lj = S + (16 * jbk + cc) * D16_LD + 16 * k;
        double s = 0.0;
#pragma unroll
        for (int mm = 0; mm < 16; ++mm) s += li[mm] * lj[mm];
        S[(16 * ib + rr) * D16_LD + 16 * jbk + cc] -= s;
      }
      __syncthreads();
    }
  }
  // block rows of L^-1: T_k = sum_{m=k}^{i-1} L_im (L^-1)_mk, then (L^-1)_ik = -X_i T_k
  for (int i = 1; i < nkb; ++i) {
    for (int idx = tid; idx < i * 256; idx += 128) {
      const int k = idx >> 8, rr = (idx >> 4) & 15, cc = idx & 15;
      double s = 0.0;
      for (int m = k; m < i; ++m) {
        const double* lim = S + (16 * i + rr) * D16_LD + 16 * m;
        if (m == k) {
          const double* xk = Xb + k * D16_XS;
#pragma unroll
          for (int q = 0; q < 16; ++q) s += lim[q] * xk[q * 17 + cc];
        } else {
          const double* lmk = S + (16 * k + cc) * D16_LD + 16 * m;   // (L^-1)_mk[q][cc] at S[16k+cc][16m+q]
#pragma unroll
          for (int q = 0; q < 16; ++q) s += lim[q] * lmk[q];
        }
      }
      Tb[k * D16_XS + rr * 17 + cc] = s;
    }
    __syncthreads();
    for (int idx = tid; idx < i * 256; idx += 128) {
      const int k = idx >> 8, rr = (idx >> 4) & 15, cc = idx & 15;
      const double* xi = Xb + i * D16_XS + rr * 17;
      const double* tk = Tb + k * D16_XS;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q) s += (q <= rr) ? xi[q] * tk[q * 17 + cc] : 0.0;
      S[(16 * k + cc) * D16_LD + 16 * i + rr] = -s;
    }
    __syncthreads();
  }
  // L (lower triangle of A_JJ) and L_JJ^-1 (zero padded) to global memory
  double* linv = cd.linv + (i64)(j0 / CB) * CB * CB;
  for (int idx = tid; idx < CB * CB; idx += 128) {
    const int i = idx >> 6, j = idx & 63;
    const int bi = i >> 4, bj = j >> 4;
    double li = 0.0;
    if (i < jb && j < jb && j <= i) {
      A[(i64)i * cd.lda + j] = S[i * D16_LD + j];
      li = (bi == bj) ? Xb[bi * D16_XS + (i & 15) * 17 + (j & 15)] : S[j * D16_LD + i];
    }
    linv[idx] = li;
  }
  return true;
}

// standalone diagonal step of the per-panel chain (real): one 128-thread CTA per matrix
__global__ void __launch_bounds__(128) chol_diag16_kernel(const CholDesc* __restrict__ cds, int j0) {
  extern __shared__ __align__(16) double smem[];
  const CholDesc& cd = cds[blockIdx.x];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  if (j0 >= r) return;
  if (!chol_diag16(cd, j0, r, smem) && threadIdx.x == 0 && cd.status) *cd.status = ST_SINGULAR_GRAM;
}

// tiles of an NT product over m rows (row tile 32 when m <= 32)
RSRS_DI void nt_rows(const NTDesc& d, int m, int n, int K, double* smem) {
  if (m <= 32) {
    if (m > 0) nt_tile<32>(d, m, n, K, 0, 0, smem);
  } else {
    for (int i0 = 0; i0 < m; i0 += GT) nt_tile<GT>(d, m, n, K, i0, 0, smem);
  }
}
RSRS_DI void nn_rows(const NNDesc& d, int m, int n, int K, double* smem) {
  if (m <= 32) {
    if (m > 0) nn_tile<32>(d, m, n, K, 0, 0, smem);
  } else {
    for (int i0 = 0; i0 < m; i0 += GT) nn_tile<GT>(d, m, n, K, i0, 0, smem);
  }
}

__global__ void __launch_bounds__(128, 3) chol_fused_kernel(const CholDesc* __restrict__ cds, int d16) {
  extern __shared__ __align__(16) double smem[];
  const CholDesc& cd = cds[blockIdx.x];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  for (int j0 = 0; j0 < r; j0 += CB) {
    const int jb = min(CB, r - j0);
    if (j0 > 0) {
      // P[j0:, J] -= L[j0:, 0:j0] L[J, 0:j0]^T  (C rows, then the B rows)
      for (int part = 0; part < 2; ++part) {
        NTDesc d{};
        d.A = part ? cd.A + (i64)cd.uoff * cd.lda : cd.A + (i64)j0 * cd.lda;
        d.lda = cd.lda;
        d.B = cd.A + (i64)j0 * cd.lda;
        d.ldb = cd.lda;
        d.C = const_cast<double*>(d.A) + j0;
        d.ldc = cd.lda;
        d.alpha = -1.0;
        d.beta = 1.0;
        nt_rows(d, part ? cd.mextra : r - j0, jb, j0, smem);
      }
      __syncthreads();
    }
    if (!(d16 ? chol_diag16(cd, j0, r, smem) : chol_diag_block128(cd, j0, r, smem))) {
      if (threadIdx.x == 0 && cd.status) *cd.status = ST_SINGULAR_GRAM;
      return;
    }
    __syncthreads();
    // rows below the diagonal block: X <- X L_JJ^-T (in place; one column tile covers J)
    for (int part = 0; part < 2; ++part) {
      NTDesc d{};
      d.A = part ? cd.A + (i64)cd.uoff * cd.lda + j0 : cd.A + (i64)(j0 + CB) * cd.lda + j0;
      d.lda = cd.lda;
      d.B = cd.linv + (i64)(j0 / CB) * CB * CB;
      d.ldb = CB;
      d.C = const_cast<double*>(d.A);
      d.ldc = cd.lda;
      d.alpha = 1.0;
      d.beta = 0.0;
      nt_rows(d, part ? cd.mextra : r - j0 - CB, jb, jb, smem);
    }
    __syncthreads();
  }
}

// back substitution W = u L^-1 of one matrix per CTA, column blocks descending
__global__ void __launch_bounds__(128, 3) chol_back_fused_kernel(const CholDesc* __restrict__ cds) {
  extern __shared__ __align__(16) double smem[];
  const CholDesc& cd = cds[blockIdx.x];
  if (cd.status && *cd.status != ST_OK) return;
  const int r = *cd.pr;
  const int m = cd.mextra;
  double* U = cd.A + (i64)cd.uoff * cd.lda;
  for (int j0 = ((r - 1) / CB) * CB; j0 >= 0; j0 -= CB) {
    const int jb = min(CB, r - j0);
    const int K = r - j0 - CB;
    if (K > 0) {   // W[:, J] = u[:, J] - W[:, J+] L[J+, J]
      NNDesc d{};
      d.A = U + j0 + CB;
      d.lda = cd.lda;
      d.B = cd.A + (i64)(j0 + CB) * cd.lda + j0;
      d.ldb = cd.lda;
      d.D = U + j0;
      d.ldd = cd.lda;
      d.alpha = -1.0;
      d.beta = 1.0;
      nn_rows(d, m, jb, K, smem);
      __syncthreads();
    }
    {              // W[:, J] <- W[:, J] L_JJ^-1 (in place)
      NNDesc d{};
      d.A = U + j0;
      d.lda = cd.lda;
      d.B = cd.linv + (i64)(j0 / CB) * CB * CB;
      d.ldb = CB;
      d.D = U + j0;
      d.ldd = cd.lda;
      d.alpha = 1.0;
      d.beta = 0.0;
      nn_rows(d, m, jb, jb, smem);
      __syncthreads();
    }
  }
}

}  // namespace rsrs
