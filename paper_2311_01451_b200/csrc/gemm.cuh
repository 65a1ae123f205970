// Batched FP64 GEMMs with row gathers on the FP64 tensor cores (DMMA m8n8k4).
//
// Two shapes cover every dense contraction of the sweep:
//   gemm_nt: C = alpha * A_rows B_rows^T   (K = p long; near-field Gram
//            Omega_near Omega_near^T, B = Y_b Omega_near^T, ID Gram H)
//   gemm_nn: D_rows = beta C_rows + alpha opA B_rows  (Y'' = Y_b - W Omega_near,
//            E/F updates PAPER.md:1205-1212, L/U updates PAPER.md:1219-1227,
//            G_U = X_rr^-1 X_rc, G_L = X_cr X_rr^-1)
// Rows are gathered through int32 index lists straight from the row-major
// sample store (each row = one point's p samples, 256-B aligned), staged in
// shared memory with cp.async (16-B chunks, zero fill at the edges), two-stage
// pipeline, 64x64 output tile per 128-thread CTA, 4 warps x (32x32) each.
#pragma once
#include "common.cuh"

namespace rsrs {

constexpr int GT = 64;       // output tile
constexpr int GBK = 32;      // K chunk
constexpr int GPA = 36;      // smem row stride (doubles) of [64][32] tiles: conflict-free fragments
constexpr int GPB = 68;      // smem row stride of [32][64] tiles
constexpr int NT_SMEM = 2 * 2 * GT * GPA * 8;              // 73,728 B
constexpr int NN_SMEM = 2 * (GT * GPA + GBK * GPB) * 8;    // 71,680 B
// shared memory of a TM-row tile (C: complex variants)
constexpr int nt_smem(int TM, bool C) { return 2 * (TM + (C ? 32 : GT)) * GPA * 8; }
constexpr int nn_smem(int TM, bool C) { return 2 * (TM * GPA + (C ? GBK / 2 : GBK) * GPB) * 8; }

// dynamic size: min(cap, *p - off) when p is set, else cap
RSRS_DI int dyn(const int* p, int off, int cap) { return p ? min(cap, *p - off) : cap; }

// descriptors nn_kstream_kernel takes (the rest of a mixed list stays with gemm_nn_kernel)
constexpr int KS_KMAX = 1024;
RSRS_DI bool kstream_takes(const NNDesc& d, int K) { return K > 0 && K <= KS_KMAX && !d.transA; }

// One TM x 64 output tile (TM = 64 or 32 rows) of C = alpha A_rows B_rows^T + beta C (K columns).
// STAGES = 2: two cp.async stages, two barriers per k chunk; STAGES = 3: one barrier per chunk
template <int TM = GT, int STAGES = 2>
RSRS_DI void nt_tile(const NTDesc& d, int m, int n, int K, int i0, int j0, double* smem) {
  constexpr int MT = TM / 16, QA = TM / 8;
  double* As = smem;
  double* Bs = smem + STAGES * TM * GPA;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  constexpr int cw = 32;
  const int cofs = wc * 32;

  const double* aptr[QA];
  const double* bptr[8];
  bool aval[QA], bval[8];
  const int lrow = tid >> 4, kc = (tid & 15) * 2;
#pragma unroll
  for (int q = 0; q < QA; ++q) {
    const int gi = i0 + lrow + 8 * q;
    aval[q] = gi < m;
    const i64 ar = aval[q] ? (d.rowA ? (i64)d.rowA[gi] : (i64)gi) : 0;
    aptr[q] = d.A + ar * d.lda;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int gj = j0 + lrow + 8 * q;
    bval[q] = gj < n;
    const i64 br = bval[q] ? (d.rowB ? (i64)d.rowB[gj] : (i64)gj) : 0;
    bptr[q] = d.B + br * d.ldb;
  }
  auto load_stage = [&](int s, int kt) {
    const int k = kt * GBK + kc;
    const int bytes = (k + 2 <= K) ? 16 : (k < K ? 8 : 0);
    const int koff = bytes ? k : 0;
#pragma unroll
    for (int q = 0; q < QA; ++q)
      cp_async16(&As[(s * TM + lrow + 8 * q) * GPA + kc], aptr[q] + koff, aval[q] ? bytes : 0);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      cp_async16(&Bs[(s * GT + lrow + 8 * q) * GPA + kc], bptr[q] + koff, bval[q] ? bytes : 0);
  };
  double acc[MT][4][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  // a warp whose sub-tile lies wholly outside C (ragged near fields) or strictly above
  // the diagonal of the symmetric Gram (never consumed) skips its MMAs
  bool wact;
  {
    const int sym = d.psym ? *d.psym : d.sym_rows;
    const int rb = i0 + wr * (TM / 2), cb = j0 + cofs;
    // (same condition as the tile-level skip: every row of the warp's band below sym_rows)
    wact = rb < m && cb < n && !(rb + TM / 2 <= sym && cb >= rb + TM / 2);
  }

  const int nk = (K + GBK - 1) / GBK;
  if constexpr (STAGES == 2) {
    if (nk > 0) {
      load_stage(0, 0);
      cp_async_commit();
    }
  } else {
    if (nk > 0) load_stage(0, 0);
    cp_async_commit();
    if (nk > 1) load_stage(1, 1);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    int sb;
    if constexpr (STAGES == 2) {
      if (kt + 1 < nk) {
        load_stage((kt + 1) & 1, kt + 1);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      sb = kt & 1;
    } else {
      // chunk kt landed (one newer group may be pending); after the barrier every warp is done
      // with chunk kt - 1, so its buffer takes chunk kt + 2
      cp_async_wait<1>();
      __syncthreads();
      if (kt + 2 < nk) load_stage((kt + 2) % 3, kt + 2);
      cp_async_commit();
      sb = kt % 3;
    }
    const double* as = As + (sb * TM + wr * (TM / 2)) * GPA;
    const double* bs = Bs + (sb * GT + cofs) * GPA;
    if (wact) {
#pragma unroll
      for (int kk = 0; kk < GBK / 4; ++kk) {
        double a[MT], b[4];
#pragma unroll
        for (int t = 0; t < MT; ++t) a[t] = as[(t * 8 + gid) * GPA + kk * 4 + tig];
#pragma unroll
        for (int u = 0; u < 4; ++u) b[u] = (u * 8 < cw) ? bs[(u * 8 + gid) * GPA + kk * 4 + tig] : 0.0;
#pragma unroll
        for (int t = 0; t < MT; ++t)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u * 8 < cw) dmma884(acc[t][u][0], acc[t][u][1], a[t], b[u]);
      }
    }
    if constexpr (STAGES == 2) __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < MT; ++t) {
    const int i = i0 + wr * (TM / 2) + t * 8 + gid;
    if (i >= m) continue;
    double* crow = d.C + (i64)i * d.ldc;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u * 8 >= cw) continue;
      const int j = j0 + cofs + u * 8 + 2 * tig;
      if (j + 1 < n) {
        double2 c = make_double2(0.0, 0.0);
        if (d.beta != 0.0) c = *reinterpret_cast<const double2*>(crow + j);
        *reinterpret_cast<double2*>(crow + j) =
            make_double2(d.beta * c.x + d.alpha * acc[t][u][0], d.beta * c.y + d.alpha * acc[t][u][1]);
      } else if (j < n) {
        const double c = d.beta != 0.0 ? crow[j] : 0.0;
        crow[j] = d.beta * c + d.alpha * acc[t][u][0];
      }
    }
  }
}

// mlo < m <= mhi: the descriptors this launch takes (a level of small boxes is split into a 16-row
// tile launch for m <= 16 and a 32-row one for the rest)
template <int TM, int STAGES = 2>
__global__ void __launch_bounds__(128) gemm_nt_kernel(const NTDesc* __restrict__ descs, int mlo = 0,
                                                      int mhi = 1 << 30) {
  extern __shared__ __align__(16) double smem[];
  const NTDesc& d = descs[blockIdx.z];
  const int m = dyn(d.pm, 0, d.m);
  const int n = dyn(d.pn, 0, d.n);
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * GT;
  if (i0 >= m || j0 >= n || m <= mlo || m > mhi) return;
  const int sym = d.psym ? *d.psym : d.sym_rows;
  if (i0 + TM <= sym && j0 >= i0 + TM) return;  // strictly upper tile of the Gram
  const NTDesc dl = d;
  nt_tile<TM, STAGES>(dl, m, n, d.K, i0, j0, smem);
}

// One TM x 64 output tile (TM = 64 or 32 rows) of D_rows = beta C_rows + alpha opA B_rows.
template <int TM = GT>
RSRS_DI void nn_tile(const NNDesc& d, int m, int n, int K, int i0, int j0, double* smem) {
  constexpr int MT = TM / 16, QA = TM / 8, RP = TM / 2;
  const bool inplace = (d.Cin == nullptr);
  if (K <= 0 && inplace && d.beta == 1.0) return;
  double* As = smem;                       // [2][TM][GPA]  (i, k)
  double* Bs = smem + 2 * TM * GPA;        // [2][32][GPB]  (k, j)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  constexpr int cw = 32;
  const int cofs = wc * 32;

  // row indices of the B rows of the next stage to be loaded, fetched one stage ahead
  // so that the dependent index loads overlap the MMAs instead of stalling the cp.async
  int brow[8];
  auto fetch_rows = [&](int kt) {
    const int kr = tid >> 5;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = kt * GBK + kr + 4 * q;
      brow[q] = k < K ? (d.rowB ? d.rowB[k] : k) : 0;
    }
  };
  auto load_stage = [&](int s, int kt) {
    const int k0 = kt * GBK;
    if (!d.transA) {
      const int lrow = tid >> 4, kc = (tid & 15) * 2;
      const int k = k0 + kc;
      const int bytes = (k + 2 <= K) ? 16 : (k < K ? 8 : 0);
#pragma unroll
      for (int q = 0; q < QA; ++q) {
        const int row = lrow + 8 * q;
        const int gi = i0 + row;
        const bool v = gi < m && bytes > 0;
        const double* src = v ? d.A + (i64)gi * d.lda + k : d.A;
        cp_async16(&As[(s * TM + row) * GPA + kc], src, v ? bytes : 0);
      }
    } else {
      // A stored (K x m): opA(i, k) = A[k*lda + i]; transpose through registers
      const int kr = tid / RP, ic = (tid % RP) * 2;
#pragma unroll
      for (int q = 0; q < RP / 4; ++q) {
        const int kl = kr + (128 / RP) * q;
        const int k = k0 + kl;
        const int gi = i0 + ic;
        double v0 = 0.0, v1 = 0.0;
        if (k < K) {
          const double* src = d.A + (i64)k * d.lda + gi;
          if (gi + 1 < m) {
            const double2 v = *reinterpret_cast<const double2*>(src);
            v0 = v.x;
            v1 = v.y;
          } else if (gi < m) {
            v0 = src[0];
          }
        }
        As[(s * TM + ic) * GPA + kl] = v0;
        As[(s * TM + ic + 1) * GPA + kl] = v1;
      }
    }
    {
      const int kr = tid >> 5, jc = (tid & 31) * 2;
      const int gj = j0 + jc;
      const int cb = (gj + 2 <= n) ? 16 : (gj < n ? 8 : 0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int kl = kr + 4 * q;
        const int k = k0 + kl;
        const bool v = k < K && cb > 0;
        const double* src = v ? d.B + (i64)brow[q] * d.ldb + gj : d.B;
        cp_async16(&Bs[(s * GBK + kl) * GPB + jc], src, v ? cb : 0);
      }
    }
  };
  double acc[MT][4][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  // a warp whose sub-tile lies wholly outside D (skinny or ragged rows) skips its MMAs
  const bool wact = i0 + wr * (TM / 2) < m && j0 + cofs < n;

  // 32-row tiles: the beta * C operand of the epilogue is loaded before the K loop, so its
  // latency overlaps the GEMM instead of following it (ncu: the epilogue's dependent loads
  // held ~35% of the stall samples of the row-gathered L/U update)
  constexpr bool PRE = (TM <= 32);
  double2 cpre[PRE ? MT : 1][4];
  if constexpr (PRE) {
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const int i = i0 + wr * (TM / 2) + t * 8 + gid;
#pragma unroll
      for (int u = 0; u < 4; ++u) cpre[t][u] = make_double2(0.0, 0.0);
      if (i >= m || d.beta == 0.0) continue;
      const double* crow;
      if (inplace) crow = d.D + (d.rowD ? (i64)d.rowD[i] : (i64)i) * d.ldd;
      else crow = d.Cin + (d.rowC ? (i64)d.rowC[i] : (i64)i) * d.ldc;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + cofs + u * 8 + 2 * tig;
        if (j + 1 < n) cpre[t][u] = *reinterpret_cast<const double2*>(crow + j);
        else if (j < n) cpre[t][u].x = crow[j];
      }
    }
  }

  const int nk = K > 0 ? (K + GBK - 1) / GBK : 0;
  if (nk > 0) {
    fetch_rows(0);
    load_stage(0, 0);
    cp_async_commit();
    if (nk > 1) fetch_rows(1);
  }
  for (int kt = 0; kt < nk; ++kt) {
    if (kt + 1 < nk) {
      load_stage((kt + 1) & 1, kt + 1);
      cp_async_commit();
      if (kt + 2 < nk) fetch_rows(kt + 2);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + ((kt & 1) * TM + wr * (TM / 2)) * GPA;
    const double* bs = Bs + (kt & 1) * GBK * GPB + cofs;
    if (wact)
#pragma unroll
      for (int kk = 0; kk < GBK / 4; ++kk) {
        double a[MT], b[4];
#pragma unroll
        for (int t = 0; t < MT; ++t) a[t] = as[(t * 8 + gid) * GPA + kk * 4 + tig];
#pragma unroll
        for (int u = 0; u < 4; ++u) b[u] = (u * 8 < cw) ? bs[(kk * 4 + tig) * GPB + u * 8 + gid] : 0.0;
#pragma unroll
        for (int t = 0; t < MT; ++t)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u * 8 < cw) dmma884(acc[t][u][0], acc[t][u][1], a[t], b[u]);
      }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int t = 0; t < MT; ++t) {
    const int i = i0 + wr * (TM / 2) + t * 8 + gid;
    if (i >= m) continue;
    const i64 dr = d.rowD ? (i64)d.rowD[i] : (i64)i;
    double* drow = d.D + dr * d.ldd;
    const double* crow;
    if (inplace) {
      crow = drow;
    } else {
      const i64 cr = d.rowC ? (i64)d.rowC[i] : (i64)i;
      crow = d.Cin + cr * d.ldc;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u * 8 >= cw) continue;
      const int j = j0 + cofs + u * 8 + 2 * tig;
      if (j + 1 < n) {
        double2 c = make_double2(0.0, 0.0);
        if constexpr (PRE) c = cpre[t][u];
        else if (d.beta != 0.0) c = *reinterpret_cast<const double2*>(crow + j);
        *reinterpret_cast<double2*>(drow + j) =
            make_double2(d.beta * c.x + d.alpha * acc[t][u][0], d.beta * c.y + d.alpha * acc[t][u][1]);
      } else if (j < n) {
        double c = 0.0;
        if constexpr (PRE) c = cpre[t][u].x;
        else if (d.beta != 0.0) c = crow[j];
        drow[j] = d.beta * c + d.alpha * acc[t][u][0];
      }
    }
  }
}

template <int TM>
__global__ void __launch_bounds__(128) gemm_nn_kernel(const NNDesc* __restrict__ descs, int mlo = 0,
                                                      int mhi = 1 << 30, int klo = -1, int skipks = 0) {
  extern __shared__ __align__(16) double smem[];
  const NNDesc& d = descs[blockIdx.z];
  const int m = dyn(d.pm, 0, d.m);
  const int n = dyn(d.pn, 0, d.n);
  const int K = dyn(d.pK, 0, d.K);
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * GT;
  if (i0 >= m || j0 >= n || m <= mlo || m > mhi || K <= klo) return;   // K <= klo: nn_stream_kernel's
  if (skipks && kstream_takes(d, K)) return;                            // nn_kstream_kernel's
  const NNDesc dl = d;
  nn_tile<TM>(dl, m, n, K, i0, j0, smem);
}


// Streaming form of the rank-K row update D_rows = beta C_rows + alpha opA B_rows for a short inner
// dimension (K <= GBK: the L/U push of a box with n_r <= 32 redundant points).
// The update is pure HBM traffic (read and write m x n, ~2K flop per 16 B), so one CTA keeps a
// 32-row band and walks its share of the 64-column chunks through a cp.async ring (depth 2 or 3)
// holding the chunk of B (K rows, zero-filled to a multiple of 4) and of C: the descriptor / size /
// row-index prologue and the A fragments (registers) are paid once per band instead of once per
// 32 x 64 tile, and the next chunk(s) stay in flight while the current one is multiplied and stored.
// Same DMMA order per element as nn_tile<32>, so the results are bit-identical to it.
// Descriptors with K > GBK are left to gemm_nn_kernel (launched on the same list with klo = GBK).
constexpr int NS_TM = 32;
constexpr int NS_STAGE_DBL = (GBK + NS_TM) * GPB;                  // B chunk, then C tile
constexpr int ns_smem(int stages) { return stages * NS_STAGE_DBL * 8 + (NS_TM + GBK) * 8; }   // + row offsets

// NS_STAGES = 3: 2 CTAs per SM, two chunks in flight per CTA; 2: 3 CTAs per SM, one chunk in flight
template <int NS_STAGES>
__global__ void __launch_bounds__(128) nn_stream_kernel(const NNDesc* __restrict__ descs, int ngroups) {
  extern __shared__ __align__(16) double smem[];
  const NNDesc& dg = descs[blockIdx.z];
  const int m = dyn(dg.pm, 0, dg.m);
  const int n = dyn(dg.pn, 0, dg.n);
  const int K = dyn(dg.pK, 0, dg.K);
  const int i0 = blockIdx.y * NS_TM;
  if (i0 >= m || K > GBK) return;
  const NNDesc d = dg;
  const bool inplace = (d.Cin == nullptr);
  if (K <= 0 && inplace && d.beta == 1.0) return;
  const int nch = (n + GT - 1) / GT;
  const int c0 = (int)(((i64)nch * blockIdx.x) / ngroups), c1 = (int)(((i64)nch * (blockIdx.x + 1)) / ngroups);
  if (c0 >= c1) return;
  i64* drow_off = reinterpret_cast<i64*>(smem + NS_STAGES * NS_STAGE_DBL);   // [NS_TM] D row offsets
  i64* brow_off = drow_off + NS_TM;                                           // [GBK]   B row offsets
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  const int cofs = wc * 32;
  if (tid < NS_TM) {
    const int i = i0 + tid;
    drow_off[tid] = i < m ? (d.rowD ? (i64)d.rowD[i] : (i64)i) * d.ldd : -1;
  } else if (tid < NS_TM + GBK) {
    const int k = tid - NS_TM;
    brow_off[k] = k < K ? (d.rowB ? (i64)d.rowB[k] : (i64)k) * d.ldb : 0;
  }
  // A fragments of the band (zero beyond K / m)
  const int nkk = (K + 3) >> 2;
  double a[2][GBK / 4];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int i = i0 + wr * 16 + t * 8 + gid;
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      const int k = kk * 4 + tig;
      a[t][kk] = (i < m && k < K) ? (d.transA ? d.A[(i64)k * d.lda + i] : d.A[(i64)i * d.lda + k]) : 0.0;
    }
  }
  const bool needc = d.beta != 0.0;
  // C rows: rowC / Cin when out of place (only the in-place form is staged through drow_off)
  __syncthreads();
  const int krows = nkk * 4;
  auto load_chunk = [&](int s, int c) {
    double* Bs = smem + s * NS_STAGE_DBL;
    double* Cs = Bs + GBK * GPB;
    const int kr = tid >> 5, jc = (tid & 31) * 2;
    const int gj = c * GT + jc;
    const int cb = (gj + 2 <= n) ? 16 : (gj < n ? 8 : 0);
#pragma unroll
    for (int q = 0; q < GBK / 4; ++q) {
      const int kl = kr + 4 * q;
      if (kl < krows) {
        const bool v = kl < K && cb > 0;
        const double* src = v ? d.B + brow_off[kl] + gj : d.B;
        cp_async16(&Bs[kl * GPB + jc], src, v ? cb : 0);
      }
    }
    if (needc) {
#pragma unroll
      for (int q = 0; q < NS_TM / 4; ++q) {
        const int r = kr + 4 * q;
        const i64 off = drow_off[r];
        const bool v = off >= 0 && cb > 0;
        const double* src = d.D;
        if (v) {
          if (inplace) src = d.D + off + gj;
          else src = d.Cin + (d.rowC ? (i64)d.rowC[i0 + r] : (i64)(i0 + r)) * d.ldc + gj;
        }
        cp_async16(&Cs[r * GPB + jc], src, v ? cb : 0);
      }
    }
  };
  const int nc = c1 - c0;
#pragma unroll
  for (int s = 0; s < NS_STAGES - 1; ++s) {
    if (s < nc) load_chunk(s, c0 + s);
    cp_async_commit();
  }
  const bool wrow = i0 + wr * 16 < m;
  for (int c = 0; c < nc; ++c) {
    cp_async_wait<NS_STAGES - 2>();
    __syncthreads();       // chunk c landed; every warp is done with chunk c - 1, whose buffer is refilled
    if (c + NS_STAGES - 1 < nc) load_chunk((c + NS_STAGES - 1) % NS_STAGES, c0 + c + NS_STAGES - 1);
    cp_async_commit();
    const int j0 = (c0 + c) * GT;
    if (!wrow || j0 + cofs >= n) continue;
    const double* bs = smem + (c % NS_STAGES) * NS_STAGE_DBL + cofs;
    const double* cs = smem + (c % NS_STAGES) * NS_STAGE_DBL + GBK * GPB;
    double acc[2][4][2];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      if (kk < nkk) {
        double b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) b[u] = bs[(kk * 4 + tig) * GPB + u * 8 + gid];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma884(acc[t][u][0], acc[t][u][1], a[t][kk], b[u]);
      }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int rl = wr * 16 + t * 8 + gid;
      const i64 off = drow_off[rl];
      if (off < 0) continue;
      double* drow = d.D + off;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int jl = cofs + u * 8 + 2 * tig;
        const int j = j0 + jl;
        if (j >= n) continue;
        double2 cv = make_double2(0.0, 0.0);
        if (needc) cv = *reinterpret_cast<const double2*>(cs + rl * GPB + jl);
        if (j + 1 < n)
          *reinterpret_cast<double2*>(drow + j) =
              make_double2(d.beta * cv.x + d.alpha * acc[t][u][0], d.beta * cv.y + d.alpha * acc[t][u][1]);
        else
          drow[j] = d.beta * cv.x + d.alpha * acc[t][u][0];
      }
    }
  }
}

// Column-walking form of nn_tile<32> for the B-bound products with few output rows and a long
// inner dimension (projection Y'' = Y_b - W Omega_near; pulled L/U update):
// one CTA keeps a 32-row band and walks its 64-column chunks, the (chunk, k-stage) pairs flattened
// into one 4-stage cp.async ring, so the ring never drains between chunks and the descriptor /
// row-index prologue is paid once per band.  Same DMMA order per element as nn_tile<32>.
// Takes the descriptors with 0 < K <= KS_KMAX and transA == 0; the others are left to
// gemm_nn_kernel (launched on the same list with the complementary filter).
constexpr int KS_STAGES = 4;
constexpr int KS_STAGE_DBL = NS_TM * GPA + GBK * GPB;
constexpr int KS_SMEM = KS_STAGES * KS_STAGE_DBL * 8 + KS_KMAX * 4;

__global__ void __launch_bounds__(128) nn_kstream_kernel(const NNDesc* __restrict__ descs, int ngroups) {
  extern __shared__ __align__(16) double smem[];
  const NNDesc& dg = descs[blockIdx.z];
  const int m = dyn(dg.pm, 0, dg.m);
  const int n = dyn(dg.pn, 0, dg.n);
  const int K = dyn(dg.pK, 0, dg.K);
  const int i0 = blockIdx.y * NS_TM;
  if (i0 >= m || !kstream_takes(dg, K)) return;
  const NNDesc d = dg;
  const bool inplace = (d.Cin == nullptr);
  const int nch = (n + GT - 1) / GT;
  const int c0 = (int)(((i64)nch * blockIdx.x) / ngroups), c1 = (int)(((i64)nch * (blockIdx.x + 1)) / ngroups);
  if (c0 >= c1) return;
  int* browi = reinterpret_cast<int*>(smem + KS_STAGES * KS_STAGE_DBL);   // [K] gathered B rows
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  const int cofs = wc * 32;
  for (int k = tid; k < K; k += 128) browi[k] = d.rowB ? d.rowB[k] : k;
  __syncthreads();
  const int nk = (K + GBK - 1) / GBK;
  const int total = (c1 - c0) * nk;
  auto load = [&](int s, int it) {
    const int c = it / nk, kt = it - c * nk;
    double* As = smem + s * KS_STAGE_DBL;
    double* Bs = As + NS_TM * GPA;
    const int k0 = kt * GBK;
    {
      const int lrow = tid >> 4, kc = (tid & 15) * 2;
      const int k = k0 + kc;
      const int bytes = (k + 2 <= K) ? 16 : (k < K ? 8 : 0);
#pragma unroll
      for (int q = 0; q < NS_TM / 8; ++q) {
        const int row = lrow + 8 * q;
        const int gi = i0 + row;
        const bool v = gi < m && bytes > 0;
        const double* src = v ? d.A + (i64)gi * d.lda + k : d.A;
        cp_async16(&As[row * GPA + kc], src, v ? bytes : 0);
      }
    }
    {
      const int kr = tid >> 5, jc = (tid & 31) * 2;
      const int gj = (c0 + c) * GT + jc;
      const int cb = (gj + 2 <= n) ? 16 : (gj < n ? 8 : 0);
#pragma unroll
      for (int q = 0; q < GBK / 4; ++q) {
        const int kl = kr + 4 * q;
        const int k = k0 + kl;
        const bool v = k < K && cb > 0;
        const double* src = v ? d.B + (i64)browi[k] * d.ldb + gj : d.B;
        cp_async16(&Bs[kl * GPB + jc], src, v ? cb : 0);
      }
    }
  };
#pragma unroll
  for (int s = 0; s < KS_STAGES - 1; ++s) {
    if (s < total) load(s, s);
    cp_async_commit();
  }
  const bool wrow = i0 + wr * 16 < m;
  double acc[2][4][2];
  double2 cpre[2][4];
  int c = 0, kt = 0;
  for (int it = 0; it < total; ++it) {
    cp_async_wait<KS_STAGES - 2>();
    __syncthreads();
    if (it + KS_STAGES - 1 < total) load((it + KS_STAGES - 1) % KS_STAGES, it + KS_STAGES - 1);
    cp_async_commit();
    const int j0 = (c0 + c) * GT;
    const bool wact = wrow && j0 + cofs < n;
    if (kt == 0) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[t][u][0] = acc[t][u][1] = 0.0;
          cpre[t][u] = make_double2(0.0, 0.0);
        }
        const int i = i0 + wr * 16 + t * 8 + gid;
        if (!wact || i >= m || d.beta == 0.0) continue;
        const double* crow;
        if (inplace) crow = d.D + (d.rowD ? (i64)d.rowD[i] : (i64)i) * d.ldd;
        else crow = d.Cin + (d.rowC ? (i64)d.rowC[i] : (i64)i) * d.ldc;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + cofs + u * 8 + 2 * tig;
          if (j + 1 < n) cpre[t][u] = *reinterpret_cast<const double2*>(crow + j);
          else if (j < n) cpre[t][u].x = crow[j];
        }
      }
    }
    if (wact) {
      const double* as = smem + (it % KS_STAGES) * KS_STAGE_DBL + wr * 16 * GPA;
      const double* bs = smem + (it % KS_STAGES) * KS_STAGE_DBL + NS_TM * GPA + cofs;
#pragma unroll
      for (int kk = 0; kk < GBK / 4; ++kk) {
        double a[2], b[4];
#pragma unroll
        for (int t = 0; t < 2; ++t) a[t] = as[(t * 8 + gid) * GPA + kk * 4 + tig];
#pragma unroll
        for (int u = 0; u < 4; ++u) b[u] = bs[(kk * 4 + tig) * GPB + u * 8 + gid];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma884(acc[t][u][0], acc[t][u][1], a[t], b[u]);
      }
      if (kt == nk - 1) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int i = i0 + wr * 16 + t * 8 + gid;
          if (i >= m) continue;
          double* drow = d.D + (d.rowD ? (i64)d.rowD[i] : (i64)i) * d.ldd;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + cofs + u * 8 + 2 * tig;
            if (j + 1 < n)
              *reinterpret_cast<double2*>(drow + j) = make_double2(d.beta * cpre[t][u].x + d.alpha * acc[t][u][0],
                                                                   d.beta * cpre[t][u].y + d.alpha * acc[t][u][1]);
            else if (j < n)
              drow[j] = d.beta * cpre[t][u].x + d.alpha * acc[t][u][0];
          }
        }
      }
    }
    if (++kt == nk) {
      kt = 0;
      ++c;
    }
  }
}

// ---------------------------------------------------------------------------
// complex128 variants (RSRS_C128; interleaved {re, im} doubles).  Leading
// dimensions and sizes in the descriptors are in COMPLEX units.  Both shapes
// run as real DMMA GEMMs over the interleaved data (K_real = 2K):
//   NT  C = A B^H:  Re = A_r B_r^T, Im = A_r (B')^T with B'_q = sign(q) B_{q^1}
//                   (sign = -1 for an even real index q): Im(a conj b) = sum ai br - ar bi
//   NN  D = opA B:  B''_{2k} = B_k, B''_{2k+1} = rot(B_k), rot(br, bi) = (-bi, br)
//                   opA = conj(A)^T when transA (A^* in the sample updates)
// ---------------------------------------------------------------------------
constexpr int GTC = 32;      // complex output columns of the NT tile (64 rows x 32 complex)

template <int TM = GT>
RSRS_DI void nt_tile_c(const NTDesc& d, int m, int n, int K, int i0, int j0, double* smem) {
  constexpr int MT = TM / 16, QA = TM / 8;
  double* As = smem;                      // [2][TM][GPA]
  double* Bs = smem + 2 * TM * GPA;       // [2][32][GPA]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  const int K2 = 2 * K;
  const i64 lda2 = 2 * d.lda, ldb2 = 2 * d.ldb;
  const double* aptr[QA];
  const double* bptr[4];
  bool aval[QA], bval[4];
  const int lrow = tid >> 4, kc = (tid & 15) * 2;
#pragma unroll
  for (int q = 0; q < QA; ++q) {
    const int gi = i0 + lrow + 8 * q;
    aval[q] = gi < m;
    const i64 ar = aval[q] ? (d.rowA ? (i64)d.rowA[gi] : (i64)gi) : 0;
    aptr[q] = d.A + ar * lda2;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int gj = j0 + lrow + 8 * q;
    bval[q] = gj < n;
    const i64 br = bval[q] ? (d.rowB ? (i64)d.rowB[gj] : (i64)gj) : 0;
    bptr[q] = d.B + br * ldb2;
  }
  auto load_stage = [&](int s, int kt) {
    const int k = kt * GBK + kc;
    const int bytes = k < K2 ? 16 : 0;
    const int koff = bytes ? k : 0;
#pragma unroll
    for (int q = 0; q < QA; ++q)
      cp_async16(&As[(s * TM + lrow + 8 * q) * GPA + kc], aptr[q] + koff, aval[q] ? bytes : 0);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      cp_async16(&Bs[(s * GTC + lrow + 8 * q) * GPA + kc], bptr[q] + koff, bval[q] ? bytes : 0);
  };
  double ar_[MT][2][2], ai_[MT][2][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int u = 0; u < 2; ++u) ar_[t][u][0] = ar_[t][u][1] = ai_[t][u][0] = ai_[t][u][1] = 0.0;
  const double sgn = (tig & 1) ? 1.0 : -1.0;
  const int nk = (K2 + GBK - 1) / GBK;
  if (nk > 0) {
    load_stage(0, 0);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    if (kt + 1 < nk) {
      load_stage((kt + 1) & 1, kt + 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + ((kt & 1) * TM + wr * (TM / 2)) * GPA;
    const double* bs = Bs + ((kt & 1) * GTC + wc * 16) * GPA;
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      double a[MT], b[2], b2[2];
#pragma unroll
      for (int t = 0; t < MT; ++t) a[t] = as[(t * 8 + gid) * GPA + kk * 4 + tig];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        b[u] = bs[(u * 8 + gid) * GPA + kk * 4 + tig];
        b2[u] = sgn * bs[(u * 8 + gid) * GPA + kk * 4 + (tig ^ 1)];
      }
#pragma unroll
      for (int t = 0; t < MT; ++t)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          dmma884(ar_[t][u][0], ar_[t][u][1], a[t], b[u]);
          dmma884(ai_[t][u][0], ai_[t][u][1], a[t], b2[u]);
        }
    }
    __syncthreads();
  }
  const i64 ldc2 = 2 * d.ldc;
#pragma unroll
  for (int t = 0; t < MT; ++t) {
    const int i = i0 + wr * (TM / 2) + t * 8 + gid;
    if (i >= m) continue;
    double* crow = d.C + (i64)i * ldc2;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + wc * 16 + u * 8 + 2 * tig + e;
        if (j < n) {
          double2 c = make_double2(0.0, 0.0);
          if (d.beta != 0.0) c = *reinterpret_cast<const double2*>(crow + 2 * j);
          *reinterpret_cast<double2*>(crow + 2 * j) =
              make_double2(d.beta * c.x + d.alpha * ar_[t][u][e], d.beta * c.y + d.alpha * ai_[t][u][e]);
        }
      }
    }
  }
}

template <int TM>
__global__ void __launch_bounds__(128) gemm_nt_kernel_c(const NTDesc* __restrict__ descs) {
  extern __shared__ __align__(16) double smem[];
  const NTDesc& d = descs[blockIdx.z];
  const int m = dyn(d.pm, 0, d.m);
  const int n = dyn(d.pn, 0, d.n);
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * GTC;
  if (i0 >= m || j0 >= n) return;
  const int sym = d.psym ? *d.psym : d.sym_rows;
  if (i0 + TM <= sym && j0 >= i0 + TM) return;  // strictly upper part of the Hermitian Gram
  const NTDesc dl = d;
  nt_tile_c<TM>(dl, m, n, d.K, i0, j0, smem);
}

// One tile (64 rows x 32 complex columns) of D_rows = beta C_rows + alpha opA B_rows.
template <int TM = GT>
RSRS_DI void nn_tile_c(const NNDesc& d, int m, int n, int K, int i0, int j0, double* smem) {
  constexpr int MT = TM / 16, QA = TM / 8, RP = TM / 2;
  const bool inplace = (d.Cin == nullptr);
  if (K <= 0 && inplace && d.beta == 1.0) return;
  double* As = smem;                       // [2][TM][GPA]   (i, real k)
  double* Bs = smem + 2 * TM * GPA;        // [2][16][GPB]   (complex k, real j)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  const int K2 = 2 * K, n2 = 2 * n, j02 = 2 * j0;
  const i64 lda2 = 2 * d.lda, ldb2 = 2 * d.ldb;
  int brow[4];   // B row indices of the next stage (complex k), fetched one stage ahead
  auto fetch_rows = [&](int kt) {
    const int kr = tid >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = kt * (GBK / 2) + kr + 4 * q;
      brow[q] = k < K ? (d.rowB ? d.rowB[k] : k) : 0;
    }
  };
  auto load_stage = [&](int s, int kt) {
    const int k0 = kt * GBK;               // real k
    if (!d.transA) {
      const int lrow = tid >> 4, kc = (tid & 15) * 2;
      const int k = k0 + kc;
      const int bytes = k < K2 ? 16 : 0;
#pragma unroll
      for (int q = 0; q < QA; ++q) {
        const int row = lrow + 8 * q;
        const int gi = i0 + row;
        const bool v = gi < m && bytes > 0;
        const double* src = v ? d.A + (i64)gi * lda2 + k : d.A;
        cp_async16(&As[(s * TM + row) * GPA + kc], src, v ? bytes : 0);
      }
    } else {
      // opA(i, k) = conj(A[k][i]), A stored K x m (complex)
      const int kr = tid / RP, ic = (tid % RP) * 2;
#pragma unroll
      for (int q = 0; q < RP / 8; ++q) {
        const int kl = kr + (128 / RP) * q;   // complex k (local, 0..15)
        const int k = (k0 >> 1) + kl;
        const int gi = i0 + ic;
        double2 v0 = make_double2(0.0, 0.0), v1 = v0;
        if (k < K) {
          const double* src = d.A + (i64)k * lda2 + 2 * (i64)gi;
          if (gi < m) v0 = *reinterpret_cast<const double2*>(src);
          if (gi + 1 < m) v1 = *reinterpret_cast<const double2*>(src + 2);
        }
        As[(s * TM + ic) * GPA + 2 * kl] = v0.x;
        As[(s * TM + ic) * GPA + 2 * kl + 1] = -v0.y;
        As[(s * TM + ic + 1) * GPA + 2 * kl] = v1.x;
        As[(s * TM + ic + 1) * GPA + 2 * kl + 1] = -v1.y;
      }
    }
    {
      const int kr = tid >> 5, jc = (tid & 31) * 2;
      const int gj = j02 + jc;
      const int cb = (gj < n2) ? 16 : 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int kl = kr + 4 * q;            // complex k (local)
        const int k = (k0 >> 1) + kl;
        const bool v = k < K && cb > 0;
        const double* src = v ? d.B + (i64)brow[q] * ldb2 + gj : d.B;
        cp_async16(&Bs[(s * (GBK / 2) + kl) * GPB + jc], src, v ? cb : 0);
      }
    }
  };
  double acc[MT][4][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  const bool odd_k = tig & 1;
  const double sgn = (gid & 1) ? 1.0 : -1.0;
  // a warp whose sub-tile lies wholly outside D (skinny or ragged rows) skips its MMAs
  const bool wact = i0 + wr * (TM / 2) < m && 2 * j0 + wc * 32 < 2 * n;
  const int nk = K2 > 0 ? (K2 + GBK - 1) / GBK : 0;
  if (nk > 0) {
    fetch_rows(0);
    load_stage(0, 0);
    cp_async_commit();
    if (nk > 1) fetch_rows(1);
  }
  for (int kt = 0; kt < nk; ++kt) {
    if (kt + 1 < nk) {
      load_stage((kt + 1) & 1, kt + 1);
      cp_async_commit();
      if (kt + 2 < nk) fetch_rows(kt + 2);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + ((kt & 1) * TM + wr * (TM / 2)) * GPA;
    const double* bs = Bs + (kt & 1) * (GBK / 2) * GPB + wc * 32;
    if (wact)
#pragma unroll
      for (int kk = 0; kk < GBK / 4; ++kk) {
        double a[MT], b[4];
#pragma unroll
        for (int t = 0; t < MT; ++t) a[t] = as[(t * 8 + gid) * GPA + kk * 4 + tig];
        const double* brow = bs + (kk * 2 + (tig >> 1)) * GPB;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = u * 8 + gid;
          b[u] = odd_k ? sgn * brow[col ^ 1] : brow[col];
        }
#pragma unroll
        for (int t = 0; t < MT; ++t)
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma884(acc[t][u][0], acc[t][u][1], a[t], b[u]);
      }
    __syncthreads();
  }
  const i64 ldd2 = 2 * d.ldd, ldc2 = 2 * d.ldc;
#pragma unroll
  for (int t = 0; t < MT; ++t) {
    const int i = i0 + wr * (TM / 2) + t * 8 + gid;
    if (i >= m) continue;
    const i64 dr = d.rowD ? (i64)d.rowD[i] : (i64)i;
    double* drow = d.D + dr * ldd2;
    const double* crow;
    if (inplace) {
      crow = drow;
    } else {
      const i64 cr = d.rowC ? (i64)d.rowC[i] : (i64)i;
      crow = d.Cin + cr * ldc2;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j02 + wc * 32 + u * 8 + 2 * tig;     // real column (even: one complex entry)
      if (j < n2) {
        double2 c = make_double2(0.0, 0.0);
        if (d.beta != 0.0) c = *reinterpret_cast<const double2*>(crow + j);
        *reinterpret_cast<double2*>(drow + j) =
            make_double2(d.beta * c.x + d.alpha * acc[t][u][0], d.beta * c.y + d.alpha * acc[t][u][1]);
      }
    }
  }
}

template <int TM>
__global__ void __launch_bounds__(128) gemm_nn_kernel_c(const NNDesc* __restrict__ descs) {
  extern __shared__ __align__(16) double smem[];
  const NNDesc& d = descs[blockIdx.z];
  const int m = dyn(d.pm, 0, d.m);
  const int n = dyn(d.pn, 0, d.n);
  const int K = dyn(d.pK, 0, d.K);
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * GTC;
  if (i0 >= m || j0 >= n) return;
  const NNDesc dl = d;
  nn_tile_c<TM>(dl, m, n, K, i0, j0, smem);
}

// scalar-type dispatch used by the templated per-box kernels
template <bool C>
RSRS_DI void nt_tile_t(const NTDesc& d, int m, int n, int K, int i0, int j0, double* smem) {
  if constexpr (C) nt_tile_c(d, m, n, K, i0, j0, smem);
  else nt_tile(d, m, n, K, i0, j0, smem);
}
template <bool C>
RSRS_DI void nn_tile_t(const NNDesc& d, int m, int n, int K, int i0, int j0, double* smem) {
  if constexpr (C) nn_tile_c(d, m, n, K, i0, j0, smem);
  else nn_tile(d, m, n, K, i0, j0, smem);
}
template <bool C> constexpr int tile_n() { return C ? GTC : GT; }

// Skinny in-place update D_rows += alpha opA B_rows with m, K <= SK_MAX (the E/F
// updates Y_r -= T Y_s, Omega_s += T^* Omega_r: a few rows times p columns, HBM-bound).
// One CTA per (descriptor, SK_COLS-column chunk): opA is staged in shared memory as
// [K][mp] (mp = m rounded up to 16, zero padded) and every thread streams one column,
// 16 output rows per pass, reading each B row once per pass (coalesced over columns).
// Grid (descriptors, column chunks); dynamic shared memory skinny_smem<C>().
constexpr int SK_MAX = 64;
constexpr int SK_COLS = 128;   // default columns per CTA (RSRS_SKINNY_COLS overrides; multiple of 128)
template <bool C> constexpr int skinny_smem() { return SK_MAX * SK_MAX * (C ? 16 : 8) + 2 * SK_MAX * 4; }
// opA capacity (scalars) for a launch whose m, K <= mk: K rows of mp = round_up(m, 16)
constexpr int skinny_acap(int mk) { return mk * ((mk + 15) & ~15); }
template <bool C>
__global__ void __launch_bounds__(128) skinny_nn_kernel(const NNDesc* __restrict__ descs, int cols,
                                                        int acap = SK_MAX * SK_MAX) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double ssm[];
  S* As = reinterpret_cast<S*>(ssm);
  const NNDesc& d = descs[blockIdx.x];
  const int m = dyn(d.pm, 0, d.m), n = dyn(d.pn, 0, d.n), K = dyn(d.pK, 0, d.K);
  if (m <= 0 || K <= 0 || (int)blockIdx.y * cols >= n) return;
  const int mp = (m + 15) & ~15;
  const S* A = reinterpret_cast<const S*>(d.A);
  const S zero = s_zero(S());
  int* rB = reinterpret_cast<int*>(As + acap);   // gathered row indices, staged once
  int* rD = rB + SK_MAX;
  for (int t = threadIdx.x; t < K; t += 128) rB[t] = d.rowB ? d.rowB[t] : t;
  for (int i = threadIdx.x; i < m; i += 128) rD[i] = d.rowD ? d.rowD[i] : i;
  for (int idx = threadIdx.x; idx < K * mp; idx += 128) {
    const int t = idx / mp, i = idx - t * mp;
    S v = zero;
    if (i < m) v = d.transA ? s_conj(A[(i64)t * d.lda + i]) : A[(i64)i * d.lda + t];
    As[idx] = v;
  }
  __syncthreads();
  const S* B = reinterpret_cast<const S*>(d.B);
  S* D = reinterpret_cast<S*>(d.D);
  // SK_COLS columns per CTA (the staged opA serves all of them), one column per thread per pass
  for (int j = blockIdx.y * cols + threadIdx.x; j < min(n, (int)(blockIdx.y + 1) * cols); j += 128) {
    for (int i0 = 0; i0 < m; i0 += 16) {
      S acc[16], dv[16];
      // the D rows of this pass are read together with the first B rows (one round trip)
#pragma unroll
      for (int u = 0; u < 16; ++u) dv[u] = (i0 + u < m) ? D[(i64)rD[i0 + u] * d.ldd + j] : zero;
#pragma unroll
      for (int u = 0; u < 16; ++u) acc[u] = zero;
      // 8 independent B loads in flight per thread (one memory round trip per 8 rows of B)
      for (int t0 = 0; t0 < K; t0 += 8) {
        S bv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) bv[q] = (t0 + q < K) ? B[(i64)rB[t0 + q] * d.ldb + j] : zero;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (t0 + q >= K) break;
          const S* at = As + (t0 + q) * mp + i0;
#pragma unroll
          for (int u = 0; u < 16; ++u) acc[u] = s_add(acc[u], s_mul(at[u], bv[q]));
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int i = i0 + u;
        if (i < m) D[(i64)rD[i] * d.ldd + j] = s_add(dv[u], s_scale(acc[u], d.alpha));
      }
    }
  }
}

}  // namespace rsrs
