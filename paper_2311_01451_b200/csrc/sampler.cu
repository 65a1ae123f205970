// Harness operator (NOT the factorization path): on-the-fly kernel matvec
// Y = A X for the BASELINE.json workloads, A_ij = delta_ij + w k(|x_i - x_j|)
// (PAPER.md:119-126 eq. kernel_eval; black-box access PAPER.md:53-61).
// Used to draw the samples Y = A Omega, Z = A^* Psi (timed separately from the
// sweep, BASELINE.json north_star) and residuals ||A x - b||.
// A 64 x 32 kernel tile is evaluated into shared memory (FP64), then
// contracted with a 32 x 64 tile of X on the FP64 tensor cores (DMMA).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/rsrs_sampler.h"
#include "common.cuh"

namespace {

using rsrs::i64;

constexpr int TM = 64, TN = 64, TK = 32;
constexpr int SA = TK + 4;   // A tile [64][36]
constexpr int SB = TN + 4;   // X tile [32][68]

__device__ __forceinline__ double kval(int kind, double r, double w) {
  if (kind == 0) return w * log(r);        // 2D log kernel
  return w / r;                            // 3D Laplace single layer
}

// rows [row0, row0 + nrows) of Y = A X (Y holds only those rows)
__global__ void __launch_bounds__(128) matvec_real_kernel(const double* __restrict__ pts, int64_t N, int64_t row0,
                                                          int64_t nrows, const double* __restrict__ X, int64_t ldx,
                                                          double* __restrict__ Y, int64_t ldy, int ncol,
                                                          int kind, double w) {
  __shared__ double As[TM * SA];
  __shared__ double Bs[TK * SB];
  __shared__ double Pi[TM * 3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;
  const int64_t i0 = row0 + (int64_t)blockIdx.y * TM;
  const int64_t iend = row0 + nrows;
  const int j0 = blockIdx.x * TN;
  for (int t = tid; t < TM * 3; t += 128) {
    const int64_t gi = i0 + t / 3;
    Pi[t] = gi < iend ? pts[gi * 3 + t % 3] : 0.0;
  }
  double acc[4][4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  __syncthreads();
  for (int64_t k0 = 0; k0 < N; k0 += TK) {
    // kernel tile A[i0:i0+64, k0:k0+32]
    for (int t = tid; t < TM * TK; t += 128) {
      const int ii = t / TK, kk = t % TK;
      const int64_t gi = i0 + ii, gk = k0 + kk;
      double v = 0.0;
      if (gi < iend && gk < N) {
        if (gi == gk) {
          v = 1.0;
        } else {
          const double dx = Pi[ii * 3] - pts[gk * 3];
          const double dy = Pi[ii * 3 + 1] - pts[gk * 3 + 1];
          const double dz = Pi[ii * 3 + 2] - pts[gk * 3 + 2];
          v = kval(kind, sqrt(dx * dx + dy * dy + dz * dz), w);
        }
      }
      As[ii * SA + kk] = v;
    }
    for (int t = tid; t < TK * TN; t += 128) {
      const int kk = t / TN, jj = t % TN;
      const int64_t gk = k0 + kk;
      Bs[kk * SB + jj] = (gk < N && j0 + jj < ncol) ? X[gk * ldx + j0 + jj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = As[(wr * 32 + t * 8 + gid) * SA + kk * 4 + tig];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = Bs[(kk * 4 + tig) * SB + wc * 32 + u * 8 + gid];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) rsrs::dmma884(acc[t][u][0], acc[t][u][1], a[t], b[u]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int64_t i = i0 + wr * 32 + t * 8 + gid;
    if (i >= iend) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + wc * 32 + u * 8 + 2 * tig;
      if (j < ncol) Y[(i - row0) * ldy + j] = acc[t][u][0];
      if (j + 1 < ncol) Y[(i - row0) * ldy + j + 1] = acc[t][u][1];
    }
  }
}

// Real kernels, wide tile: 64 rows x 128 columns per CTA (256 threads, 8 warps of
// 32 x 32), X tiles double-buffered with cp.async.  The kernel values of a 64 x 32
// A tile are evaluated once per 128 output columns (twice the reuse of the 64-wide
// tile above: the log / rsqrt evaluations and the scattered point loads were the
// bound), so Y = A Omega, Z = A Psi of c5 need ~half the evaluations.
constexpr int WTN = 128;
constexpr int WSB = WTN + 4;
constexpr int WIDE_SMEM = (TM * SA + 2 * TK * WSB + TM * 3) * 8;

__global__ void __launch_bounds__(256, 2) matvec_real_wide_kernel(const double* __restrict__ pts, int64_t N,
                                                                  int64_t row0, int64_t nrows,
                                                                  const double* __restrict__ X, int64_t ldx,
                                                                  double* __restrict__ Y, int64_t ldy, int ncol,
                                                                  int kind, double w) {
  extern __shared__ __align__(16) double wsm[];
  double* As = wsm;                       // [TM][SA]
  double* Bs = As + TM * SA;              // [2][TK][WSB]
  double* Pi = Bs + 2 * TK * WSB;         // [TM][3]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 2, wc = warp & 3;
  const int64_t i0 = row0 + (int64_t)blockIdx.y * TM;
  const int64_t iend = row0 + nrows;
  const int j0 = blockIdx.x * WTN;
  for (int t = tid; t < TM * 3; t += 256) {
    const int64_t gi = i0 + t / 3;
    Pi[t] = gi < iend ? pts[gi * 3 + t % 3] : 0.0;
  }
  // X tile loader: 32 rows x 128 columns = 2048 16-byte chunks, 8 per thread
  auto load_b = [&](int st, int64_t k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = tid + 256 * q;
      const int kk = c >> 6, jj = 2 * (c & 63);
      const int64_t gk = k0 + kk;
      const int j = j0 + jj;
      const int nb = (gk < N && j < ncol) ? ((j + 1 < ncol) ? 16 : 8) : 0;
      rsrs::cp_async16(&Bs[(st * TK + kk) * WSB + jj], nb ? (const void*)(X + gk * ldx + j) : (const void*)X, nb);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  const int nk = (int)((N + TK - 1) / TK);
  load_b(0, 0);
  rsrs::cp_async_commit();
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int64_t k0 = (int64_t)kt * TK;
    if (kt + 1 < nk) load_b((kt + 1) & 1, k0 + TK);
    rsrs::cp_async_commit();
    // kernel tile A[i0:i0+64, k0:k0+32]: a warp evaluates one row against 32 consecutive points
    {
      const int kk = lane;
      const int64_t gk = k0 + kk;
      double px = 0.0, py = 0.0, pz = 0.0;
      if (gk < N) {
        px = pts[gk * 3];
        py = pts[gk * 3 + 1];
        pz = pts[gk * 3 + 2];
      }
#pragma unroll 2
      for (int ii = warp; ii < TM; ii += 8) {
        const int64_t gi = i0 + ii;
        double v = 0.0;
        if (gi < iend && gk < N) {
          if (gi == gk) {
            v = 1.0;
          } else {
            const double dx = Pi[ii * 3] - px;
            const double dy = Pi[ii * 3 + 1] - py;
            const double dz = Pi[ii * 3 + 2] - pz;
            v = kval(kind, sqrt(dx * dx + dy * dy + dz * dz), w);
          }
        }
        As[ii * SA + kk] = v;
      }
    }
    rsrs::cp_async_wait<1>();
    __syncthreads();
    const double* bs = Bs + (kt & 1) * TK * WSB;
#pragma unroll
    for (int kk = 0; kk < TK / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = As[(wr * 32 + t * 8 + gid) * SA + kk * 4 + tig];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = bs[(kk * 4 + tig) * WSB + wc * 32 + u * 8 + gid];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) rsrs::dmma884(acc[t][u][0], acc[t][u][1], a[t], b[u]);
    }
    __syncthreads();
  }
  rsrs::cp_async_wait<0>();
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int64_t i = i0 + wr * 32 + t * 8 + gid;
    if (i >= iend) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + wc * 32 + u * 8 + 2 * tig;
      if (j < ncol) Y[(i - row0) * ldy + j] = acc[t][u][0];
      if (j + 1 < ncol) Y[(i - row0) * ldy + j + 1] = acc[t][u][1];
    }
  }
}

// Complex operator (kind 2, config c4): A_ij = delta_ij + w (i/4) H0^(1)(kappa r)
// = delta_ij + w (-Y0(kappa r) + i J0(kappa r)) / 4, complex symmetric, so
// A^* = conj(A).  X, Y are complex128 (interleaved doubles).  Y = A X runs as
// Y_real = A_r X_real + A_i rot(X_real) with rot(xr, xi) = (-xi, xr) per
// entry, i.e. two real DMMAs per step.  64 rows x 64 complex columns per CTA.
constexpr int CTN = 128;          // real columns of the X tile (64 complex)
constexpr int CSB = CTN + 4;
constexpr int CPLX_SMEM = (2 * TM * SA + TK * CSB + TM * 3) * 8;

__global__ void __launch_bounds__(256) matvec_cplx_kernel(const double* __restrict__ pts, int64_t N,
                                                          int64_t row0, int64_t nrows,
                                                          const double* __restrict__ X, int64_t ldx,
                                                          double* __restrict__ Y, int64_t ldy, int ncol,
                                                          double w, double kappa, int adjoint) {
  extern __shared__ __align__(16) double csm[];
  double* Ar = csm;
  double* Ai = Ar + TM * SA;
  double* Bs = Ai + TM * SA;
  double* Pi = Bs + TK * CSB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 2, wc = warp & 3;
  const int64_t i0 = row0 + (int64_t)blockIdx.y * TM;
  const int64_t iend = row0 + nrows;
  const int c0 = blockIdx.x * (CTN / 2);            // complex column
  const int ncol2 = 2 * ncol;
  const double sgn_im = adjoint ? -1.0 : 1.0;
  for (int t = tid; t < TM * 3; t += 256) {
    const int64_t gi = i0 + t / 3;
    Pi[t] = gi < iend ? pts[gi * 3 + t % 3] : 0.0;
  }
  double acc[4][4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
  __syncthreads();
  for (int64_t k0 = 0; k0 < N; k0 += TK) {
    for (int t = tid; t < TM * TK; t += 256) {
      const int ii = t / TK, kk = t % TK;
      const int64_t gi = i0 + ii, gk = k0 + kk;
      double vr = 0.0, vi = 0.0;
      if (gi < iend && gk < N) {
        if (gi == gk) {
          vr = 1.0;
        } else {
          const double dx = Pi[ii * 3] - pts[gk * 3];
          const double dy = Pi[ii * 3 + 1] - pts[gk * 3 + 1];
          const double dz = Pi[ii * 3 + 2] - pts[gk * 3 + 2];
          const double kr = kappa * sqrt(dx * dx + dy * dy + dz * dz);
          vr = -0.25 * w * ::y0(kr);
          vi = sgn_im * 0.25 * w * ::j0(kr);
        }
      }
      Ar[ii * SA + kk] = vr;
      Ai[ii * SA + kk] = vi;
    }
    for (int t = tid; t < TK * CTN; t += 256) {
      const int kk = t / CTN, jj = t % CTN;
      const int64_t gk = k0 + kk;
      Bs[kk * CSB + jj] = (gk < N && 2 * c0 + jj < ncol2) ? X[gk * 2 * ldx + 2 * c0 + jj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK / 4; ++kk) {
      double ar[4], ai[4], b[4], br[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        ar[t] = Ar[(wr * 32 + t * 8 + gid) * SA + kk * 4 + tig];
        ai[t] = Ai[(wr * 32 + t * 8 + gid) * SA + kk * 4 + tig];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int col = wc * 32 + u * 8 + gid;
        const double* brow = Bs + (kk * 4 + tig) * CSB;
        b[u] = brow[col];
        br[u] = (gid & 1) ? brow[col - 1] : -brow[col + 1];
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          rsrs::dmma884(acc[t][u][0], acc[t][u][1], ar[t], b[u]);
          rsrs::dmma884(acc[t][u][0], acc[t][u][1], ai[t], br[u]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int64_t i = i0 + wr * 32 + t * 8 + gid;
    if (i >= iend) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = 2 * c0 + wc * 32 + u * 8 + 2 * tig;   // real column (even)
      if (j < ncol2) {
        Y[(i - row0) * 2 * ldy + j] = acc[t][u][0];
        Y[(i - row0) * 2 * ldy + j + 1] = acc[t][u][1];
      }
    }
  }
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* rsrs_sampler_last_error(void) { return g_err.c_str(); }

int rsrs_sample_matvec_rows(int kind, const double* pts, int64_t N, int64_t row0, int64_t nrows, double weight,
                            double kappa, const void* X, int64_t ldx, void* Y, int64_t ldy, int64_t ncol,
                            int adjoint, void* stream) {
  if (kind < 0 || kind > 2 || !pts || !X || !Y || N < 1 || row0 < 0 || nrows < 0 || row0 + nrows > N ||
      ncol < 1 || ldx < ncol || ldy < ncol) {
    g_err = "rsrs_sample_matvec_rows: invalid argument";
    return 1;
  }
  if (nrows == 0) return 0;
  if (kind == 2) {
    dim3 grid((unsigned)((ncol + CTN / 2 - 1) / (CTN / 2)), (unsigned)((nrows + TM - 1) / TM));
    cudaFuncSetAttribute(matvec_cplx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CPLX_SMEM);
    matvec_cplx_kernel<<<grid, 256, CPLX_SMEM, (cudaStream_t)stream>>>(pts, N, row0, nrows, (const double*)X, ldx,
                                                                       (double*)Y, ldy, (int)ncol, weight, kappa,
                                                                       adjoint);
  } else {
    // the real kernels here are symmetric: A^* = A
    if ((ldx & 1) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {   // 16-byte aligned X rows
      dim3 grid((unsigned)((ncol + WTN - 1) / WTN), (unsigned)((nrows + TM - 1) / TM));
      cudaFuncSetAttribute(matvec_real_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WIDE_SMEM);
      matvec_real_wide_kernel<<<grid, 256, WIDE_SMEM, (cudaStream_t)stream>>>(pts, N, row0, nrows, (const double*)X,
                                                                             ldx, (double*)Y, ldy, (int)ncol, kind,
                                                                             weight);
    } else {
      dim3 grid((unsigned)((ncol + TN - 1) / TN), (unsigned)((nrows + TM - 1) / TM));
      matvec_real_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(pts, N, row0, nrows, (const double*)X, ldx,
                                                                 (double*)Y, ldy, (int)ncol, kind, weight);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string("rsrs_sample_matvec_rows: ") + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

int rsrs_sample_matvec(int kind, const double* pts, int64_t N, double weight, const void* X, int64_t ldx,
                       void* Y, int64_t ldy, int64_t ncol, int adjoint, void* stream) {
  if (kind < 0 || kind > 1) {
    g_err = "rsrs_sample_matvec: invalid kind (0 log2d, 1 lap3d; complex kinds: rsrs_sample_matvec_c128)";
    return 1;
  }
  return rsrs_sample_matvec_rows(kind, pts, N, 0, N, weight, 0.0, X, ldx, Y, ldy, ncol, adjoint, stream);
}

int rsrs_sample_matvec_c128(const double* pts, int64_t N, double weight, double kappa, const void* X,
                            int64_t ldx, void* Y, int64_t ldy, int64_t ncol, int adjoint, void* stream) {
  return rsrs_sample_matvec_rows(2, pts, N, 0, N, weight, kappa, X, ldx, Y, ldy, ncol, adjoint, stream);
}

}  // extern "C"
