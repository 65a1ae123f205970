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

// dynamic size: min(cap, *p - off) when p is set, else cap
RSRS_DI int dyn(const int* p, int off, int cap) { return p ? min(cap, *p - off) : cap; }

// One 64x64 output tile of C = alpha A_rows B_rows^T + beta C (K columns).
RSRS_DI void nt_tile(const NTDesc& d, int m, int n, int K, int i0, int j0, double* smem) {
  double* As = smem;
  double* Bs = smem + 2 * GT * GPA;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;

  const double* aptr[8];
  const double* bptr[8];
  bool aval[8], bval[8];
  const int lrow = tid >> 4, kc = (tid & 15) * 2;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int gi = i0 + lrow + 8 * q;
    aval[q] = gi < m;
    const i64 ar = aval[q] ? (d.rowA ? (i64)d.rowA[gi] : (i64)gi) : 0;
    aptr[q] = d.A + ar * d.lda;
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
    for (int q = 0; q < 8; ++q) {
      const int row = lrow + 8 * q;
      cp_async16(&As[(s * GT + row) * GPA + kc], aptr[q] + koff, aval[q] ? bytes : 0);
      cp_async16(&Bs[(s * GT + row) * GPA + kc], bptr[q] + koff, bval[q] ? bytes : 0);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;

  const int nk = (K + GBK - 1) / GBK;
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
    const double* as = As + ((kt & 1) * GT + wr * 32) * GPA;
    const double* bs = Bs + ((kt & 1) * GT + wc * 32) * GPA;
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = as[(t * 8 + gid) * GPA + kk * 4 + tig];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = bs[(u * 8 + gid) * GPA + kk * 4 + tig];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma884(acc[t][u][0], acc[t][u][1], a[t], b[u]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int i = i0 + wr * 32 + t * 8 + gid;
    if (i >= m) continue;
    double* crow = d.C + (i64)i * d.ldc;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + wc * 32 + u * 8 + 2 * tig;
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

__global__ void __launch_bounds__(128) gemm_nt_kernel(const NTDesc* __restrict__ descs) {
  extern __shared__ __align__(16) double smem[];
  const NTDesc& d = descs[blockIdx.z];
  const int m = dyn(d.pm, 0, d.m);
  const int n = dyn(d.pn, 0, d.n);
  const int i0 = blockIdx.y * GT, j0 = blockIdx.x * GT;
  if (i0 >= m || j0 >= n) return;
  const int sym = d.psym ? *d.psym : d.sym_rows;
  if (i0 + GT <= sym && j0 >= i0 + GT) return;  // strictly upper tile of the Gram
  const NTDesc dl = d;
  nt_tile(dl, m, n, d.K, i0, j0, smem);
}

// One 64x64 output tile of D_rows = beta C_rows + alpha opA B_rows.
RSRS_DI void nn_tile(const NNDesc& d, int m, int n, int K, int i0, int j0, double* smem) {
  const bool inplace = (d.Cin == nullptr);
  if (K <= 0 && inplace && d.beta == 1.0) return;
  double* As = smem;                       // [2][64][GPA]  (i, k)
  double* Bs = smem + 2 * GT * GPA;        // [2][32][GPB]  (k, j)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;

  auto load_stage = [&](int s, int kt) {
    const int k0 = kt * GBK;
    if (!d.transA) {
      const int lrow = tid >> 4, kc = (tid & 15) * 2;
      const int k = k0 + kc;
      const int bytes = (k + 2 <= K) ? 16 : (k < K ? 8 : 0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int row = lrow + 8 * q;
        const int gi = i0 + row;
        const bool v = gi < m && bytes > 0;
        const double* src = v ? d.A + (i64)gi * d.lda + k : d.A;
        cp_async16(&As[(s * GT + row) * GPA + kc], src, v ? bytes : 0);
      }
    } else {
      // A stored (K x m): opA(i, k) = A[k*lda + i]; transpose through registers
      const int kr = tid >> 5, ic = (tid & 31) * 2;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int kl = kr + 4 * q;
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
        As[(s * GT + ic) * GPA + kl] = v0;
        As[(s * GT + ic + 1) * GPA + kl] = v1;
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
        const double* src = d.B;
        if (v) {
          const i64 br = d.rowB ? (i64)d.rowB[k] : (i64)k;
          src = d.B + br * d.ldb + gj;
        }
        cp_async16(&Bs[(s * GBK + kl) * GPB + jc], src, v ? cb : 0);
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;

  const int nk = K > 0 ? (K + GBK - 1) / GBK : 0;
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
    const double* as = As + ((kt & 1) * GT + wr * 32) * GPA;
    const double* bs = Bs + (kt & 1) * GBK * GPB + wc * 32;
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = as[(t * 8 + gid) * GPA + kk * 4 + tig];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = bs[(kk * 4 + tig) * GPB + u * 8 + gid];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma884(acc[t][u][0], acc[t][u][1], a[t], b[u]);
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int i = i0 + wr * 32 + t * 8 + gid;
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
      const int j = j0 + wc * 32 + u * 8 + 2 * tig;
      if (j + 1 < n) {
        double2 c = make_double2(0.0, 0.0);
        if (d.beta != 0.0) c = *reinterpret_cast<const double2*>(crow + j);
        *reinterpret_cast<double2*>(drow + j) =
            make_double2(d.beta * c.x + d.alpha * acc[t][u][0], d.beta * c.y + d.alpha * acc[t][u][1]);
      } else if (j < n) {
        const double c = d.beta != 0.0 ? crow[j] : 0.0;
        drow[j] = d.beta * c + d.alpha * acc[t][u][0];
      }
    }
  }
}

__global__ void __launch_bounds__(128) gemm_nn_kernel(const NNDesc* __restrict__ descs) {
  extern __shared__ __align__(16) double smem[];
  const NNDesc& d = descs[blockIdx.z];
  const int m = dyn(d.pm, 0, d.m);
  const int n = dyn(d.pn, 0, d.n);
  const int K = dyn(d.pK, 0, d.K);
  const int i0 = blockIdx.y * GT, j0 = blockIdx.x * GT;
  if (i0 >= m || j0 >= n) return;
  const NNDesc dl = d;
  nn_tile(dl, m, n, K, i0, j0, smem);
}

}  // namespace rsrs
