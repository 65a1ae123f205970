// Solve / apply sweeps and permutation kernels (HBM-bound; one CTA per box).
// K = V_1..V_n A~_diag W_n..W_1, V = E L, W = U F;
// inverses of elim() toggle the sign of the off-diagonal block.
#pragma once
#include "common.cuh"

namespace rsrs {

RSRS_DI double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
RSRS_DI double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// right-hand sides per tile of the multi-RHS sweep (factor bytes are read once per tile)
template <bool C>
constexpr int sweep_nrb() { return C ? 4 : 16; }

// Matrix-times-tile from shared memory, the core of every sweep kernel:
//   acc(i, c) = sum_j M[i, j] X[j, c],  rows i in [0, m), X = xsm[j * NRB + c] (n x NRB)
// An 8-lane group per row (4 rows per warp in flight), each lane streaming its own
// 16-byte chunks of the row (coalesced 128-byte row segments per group), so that a CTA
// keeps many independent loads in flight (the 1-RHS sweep is latency / HBM bound);
// emit(i, acc) runs on the group leader.  NRB right-hand sides share each factor load.
template <int NRB, class F>
RSRS_DI void gemv_rows(const double* __restrict__ M, i64 ld, int m, int n, const double* __restrict__ xsm,
                       F&& emit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 3, gl = lane & 7;
  for (int i0 = warp * 4; i0 < m; i0 += nw * 4) {
    const int i = i0 + g;
    double acc[NRB];
#pragma unroll
    for (int c = 0; c < NRB; ++c) acc[c] = 0.0;
    if (i < m) {
      const double* row = M + (i64)i * ld;
      const int n2 = n >> 1;            // rows are 16-byte aligned (even leading dimensions)
      const double2* row2 = reinterpret_cast<const double2*>(row);
#pragma unroll 4
      for (int j2 = gl; j2 < n2; j2 += 8) {
        const double2 a = __ldg(row2 + j2);
        if constexpr (NRB == 1) {
          acc[0] = fma(a.x, xsm[2 * j2], fma(a.y, xsm[2 * j2 + 1], acc[0]));
        } else {
          // right-hand-side pairs as 16-byte shared loads (the x tile is the shared-memory traffic)
          const double2* x0 = reinterpret_cast<const double2*>(xsm + (2 * j2) * NRB);
          const double2* x1 = reinterpret_cast<const double2*>(xsm + (2 * j2 + 1) * NRB);
#pragma unroll
          for (int c = 0; c < NRB / 2; ++c) {
            const double2 u = x0[c], v = x1[c];
            acc[2 * c] = fma(a.x, u.x, fma(a.y, v.x, acc[2 * c]));
            acc[2 * c + 1] = fma(a.x, u.y, fma(a.y, v.y, acc[2 * c + 1]));
          }
        }
      }
      if ((n & 1) && gl == 0) {
        const double a = __ldg(row + n - 1);
#pragma unroll
        for (int c = 0; c < NRB; ++c) acc[c] = fma(a, xsm[(n - 1) * NRB + c], acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < NRB; ++c) {
      acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 4);
      acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 2);
      acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 1);
    }
    if (i < m && gl == 0) emit(i, acc);
  }
}
template <int NRB, class F>
RSRS_DI void gemv_rows(const double2* __restrict__ M, i64 ld, int m, int n, const double2* __restrict__ xsm,
                       F&& emit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 3, gl = lane & 7;
  for (int i0 = warp * 4; i0 < m; i0 += nw * 4) {
    const int i = i0 + g;
    double2 acc[NRB];
#pragma unroll
    for (int c = 0; c < NRB; ++c) acc[c] = make_double2(0.0, 0.0);
    if (i < m) {
      const double2* row = M + (i64)i * ld;
#pragma unroll 4
      for (int j = gl; j < n; j += 8) {
        const double2 a = __ldg(row + j);
#pragma unroll
        for (int c = 0; c < NRB; ++c) {
          const double2 xv = xsm[j * NRB + c];
          acc[c].x = fma(a.x, xv.x, fma(-a.y, xv.y, acc[c].x));
          acc[c].y = fma(a.x, xv.y, fma(a.y, xv.x, acc[c].y));
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NRB; ++c)
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, o);
        acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, o);
      }
    if (i < m && gl == 0) emit(i, acc);
  }
}

// x rows -> shared tile (rows idx[0..n), columns c0 .. c0 + NRB; zero beyond nrhs)
template <class S, int NRB>
RSRS_DI void load_rows(S* __restrict__ dst, const S* __restrict__ x, const int* __restrict__ idx, int n, i64 ldx,
                       int c0, int nrhs) {
  for (int t = threadIdx.x; t < n * NRB; t += blockDim.x) {
    const int i = t / NRB, c = t % NRB;
    dst[t] = (c0 + c < nrhs) ? x[(i64)idx[i] * ldx + c0 + c] : s_zero(S());
  }
}

// x_s (-|+)= T^* x_r  (T: n_r x k, ld ldn): a thread per (s, column); coalesced over s
template <class S, int NRB>
RSRS_DI void t_adjoint_update(S* __restrict__ x, const int* __restrict__ skel, const S* __restrict__ T, i64 ldn,
                              int k, int nr, const S* __restrict__ xr, i64 ldx, int c0, int nrhs, double sign) {
  for (int t = threadIdx.x; t < k * NRB; t += blockDim.x) {
    const int sidx = t % k, c = t / k;
    if (c0 + c >= nrhs) continue;
    S v = s_zero(S());
    for (int i = 0; i < nr; ++i) v = s_add(v, s_mul(s_conj(T[(i64)i * ldn + sidx]), xr[i * NRB + c]));
    S* xp = x + (i64)skel[sidx] * ldx + c0 + c;
    *xp = s_add(*xp, s_scale(v, sign));
  }
}

// forward solve of one box: x_r -= T x_s ; x_c -= G_L x_r ; x_r <- X_rr^-1 x_r
template <bool C, int NRB>
__global__ void __launch_bounds__(256) solve_fwd_kernel(const BoxDev* __restrict__ boxes,
                                                         const double* __restrict__ fpoold,
                                                         const int* __restrict__ ipool, double* __restrict__ xd,
                                                         i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  S* sm = reinterpret_cast<S*>(smd);
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* x = reinterpret_cast<S*>(xd);
  const BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn;
  S* xs = sm;
  S* xr = xs + k * NRB;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const S* T = fpool + b.f_T;
  const S* GL = fpool + b.f_GL;
  const S* Xi = fpool + b.f_Xinv;
  for (int c0 = 0; c0 < nrhs; c0 += NRB) {
    load_rows<S, NRB>(xs, x, skel, k, ldx, c0, nrhs);
    load_rows<S, NRB>(xr, x, red, nr, ldx, c0, nrhs);
    __syncthreads();
    gemv_rows<NRB>(T, ldn, nr, k, xs, [&](int i, const S* acc) {
#pragma unroll
      for (int c = 0; c < NRB; ++c) xr[i * NRB + c] = s_sub(xr[i * NRB + c], acc[c]);
    });
    __syncthreads();
    gemv_rows<NRB>(GL, ldn, nc, nr, xr, [&](int i, const S* acc) {
#pragma unroll
      for (int c = 0; c < NRB; ++c)
        if (c0 + c < nrhs) {
          S* xp = x + (i64)cc[i] * ldx + c0 + c;
          *xp = s_sub(*xp, acc[c]);
        }
    });
    gemv_rows<NRB>(Xi, ldn, nr, nr, xr, [&](int i, const S* acc) {
#pragma unroll
      for (int c = 0; c < NRB; ++c)
        if (c0 + c < nrhs) x[(i64)red[i] * ldx + c0 + c] = acc[c];
    });
    __syncthreads();
  }
}

// backward solve of one box: x_r -= G_U x_c ; x_s -= T^* x_r
template <bool C, int NRB>
__global__ void __launch_bounds__(256) solve_bwd_kernel(const BoxDev* __restrict__ boxes,
                                                         const double* __restrict__ fpoold,
                                                         const int* __restrict__ ipool, double* __restrict__ xd,
                                                         i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  S* sm = reinterpret_cast<S*>(smd);
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* x = reinterpret_cast<S*>(xd);
  const BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn, ldr = b.ldr;
  S* xc = sm;
  S* xr = xc + nc * NRB;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const S* T = fpool + b.f_T;
  const S* GU = fpool + b.f_GU;
  for (int c0 = 0; c0 < nrhs; c0 += NRB) {
    load_rows<S, NRB>(xc, x, cc, nc, ldx, c0, nrhs);
    load_rows<S, NRB>(xr, x, red, nr, ldx, c0, nrhs);
    __syncthreads();
    gemv_rows<NRB>(GU, ldr, nr, nc, xc, [&](int i, const S* acc) {
#pragma unroll
      for (int c = 0; c < NRB; ++c) {
        const S v = s_sub(xr[i * NRB + c], acc[c]);
        xr[i * NRB + c] = v;
        if (c0 + c < nrhs) x[(i64)red[i] * ldx + c0 + c] = v;
      }
    });
    __syncthreads();
    t_adjoint_update<S, NRB>(x, skel, T, ldn, k, nr, xr, ldx, c0, nrhs, -1.0);
    __syncthreads();
  }
}

// apply, forward half of one box: x_s += T^* x_r ; x_r += G_U x_c ; x_r <- X_rr x_r
template <bool C, int NRB>
__global__ void __launch_bounds__(256) apply_fwd_kernel(const BoxDev* __restrict__ boxes,
                                                         const double* __restrict__ fpoold,
                                                         const int* __restrict__ ipool, double* __restrict__ xd,
                                                         i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  S* sm = reinterpret_cast<S*>(smd);
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* x = reinterpret_cast<S*>(xd);
  const BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn, ldr = b.ldr;
  S* xc = sm;
  S* xr = xc + nc * NRB;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const S* T = fpool + b.f_T;
  const S* GU = fpool + b.f_GU;
  const S* Xrr = fpool + b.f_Xrr;
  for (int c0 = 0; c0 < nrhs; c0 += NRB) {
    load_rows<S, NRB>(xr, x, red, nr, ldx, c0, nrhs);
    __syncthreads();
    // x_s += T^* x_r first: c = near \ red holds b's skeletons, so x_c is read after it
    t_adjoint_update<S, NRB>(x, skel, T, ldn, k, nr, xr, ldx, c0, nrhs, 1.0);
    __syncthreads();
    load_rows<S, NRB>(xc, x, cc, nc, ldx, c0, nrhs);
    __syncthreads();
    gemv_rows<NRB>(GU, ldr, nr, nc, xc, [&](int i, const S* acc) {
#pragma unroll
      for (int c = 0; c < NRB; ++c) xr[i * NRB + c] = s_add(xr[i * NRB + c], acc[c]);
    });
    __syncthreads();
    gemv_rows<NRB>(Xrr, ldn, nr, nr, xr, [&](int i, const S* acc) {
#pragma unroll
      for (int c = 0; c < NRB; ++c)
        if (c0 + c < nrhs) x[(i64)red[i] * ldx + c0 + c] = acc[c];
    });
    __syncthreads();
  }
}

// apply, backward half of one box: x_c += G_L x_r ; x_r += T x_s
template <bool C, int NRB>
__global__ void __launch_bounds__(256) apply_bwd_kernel(const BoxDev* __restrict__ boxes,
                                                         const double* __restrict__ fpoold,
                                                         const int* __restrict__ ipool, double* __restrict__ xd,
                                                         i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  S* sm = reinterpret_cast<S*>(smd);
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* x = reinterpret_cast<S*>(xd);
  const BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn;
  S* xs = sm;
  S* xr = xs + k * NRB;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const S* T = fpool + b.f_T;
  const S* GL = fpool + b.f_GL;
  for (int c0 = 0; c0 < nrhs; c0 += NRB) {
    load_rows<S, NRB>(xr, x, red, nr, ldx, c0, nrhs);
    __syncthreads();
    gemv_rows<NRB>(GL, ldn, nc, nr, xr, [&](int i, const S* acc) {
#pragma unroll
      for (int c = 0; c < NRB; ++c)
        if (c0 + c < nrhs) {
          S* xp = x + (i64)cc[i] * ldx + c0 + c;
          *xp = s_add(*xp, acc[c]);
        }
    });
    __syncthreads();
    load_rows<S, NRB>(xs, x, skel, k, ldx, c0, nrhs);   // after the x_c update (skel is part of c)
    __syncthreads();
    gemv_rows<NRB>(T, ldn, nr, k, xs, [&](int i, const S* acc) {
#pragma unroll
      for (int c = 0; c < NRB; ++c)
        if (c0 + c < nrhs) x[(i64)red[i] * ldx + c0 + c] = s_add(xr[i * NRB + c], acc[c]);
    });
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Packed solve records (block-diagonal form).  At the end of a level the factor
// blocks the solve reads are copied into one compact, contiguous record per box
// (solve_pack_kernel) laid out so that every factor load of the sweep is
// coalesced and independent of the others (one memory round trip per phase):
//   forward  [Tt (k x nr) | GLt (nr x nc) | Xit (nr x nr)]   column-major T, G_L, X_rr^-1
//   backward [GU (nr x nc) | Tb (nr x k)]                   row-major, no padding
// Each sub-block starts on an even scalar offset (16-byte aligned).
RSRS_DI i64 ev2(i64 v) { return (v + 1) & ~(i64)1; }
RSRS_DI i64 pack_fwd_size(int nr, int k, int nc) { return ev2((i64)k * nr) + ev2((i64)nr * nc) + ev2((i64)nr * nr); }
RSRS_DI i64 pack_bwd_size(int nr, int k, int nc) { return ev2((i64)nr * nc) + ev2((i64)nr * k); }

template <bool C>
__global__ void __launch_bounds__(256) solve_pack_kernel(const BoxDev* __restrict__ boxes,
                                                          const double* __restrict__ fpoold,
                                                          const i64* __restrict__ pk, double* __restrict__ packd) {
  typedef typename ScalarOf<C>::T S;
  const BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  const S* T = fpool + b.f_T;
  const S* GL = fpool + b.f_GL;
  const S* GU = fpool + b.f_GU;
  const S* Xi = fpool + b.f_Xinv;
  const int ldn = b.ldn, ldr = b.ldr;
  S* P = reinterpret_cast<S*>(packd) + pk[blockIdx.x];
  S* Tt = P;
  S* GLt = Tt + ev2((i64)k * nr);
  S* Xit = GLt + ev2((i64)nr * nc);
  S* GUp = Xit + ev2((i64)nr * nr);
  S* Tb = GUp + ev2((i64)nr * nc);
  const int tid = threadIdx.x, nt = blockDim.x;
  // writes are contiguous in the packed index, reads strided (one-time copy)
  for (int t = tid; t < k * nr; t += nt) {
    const int j = t / nr, i = t % nr;
    Tt[t] = T[(i64)i * ldn + j];
  }
  for (i64 t = tid; t < (i64)nr * nc; t += nt) {
    const int j = (int)(t / nc), i = (int)(t % nc);
    GLt[t] = GL[(i64)i * ldn + j];
  }
  for (int t = tid; t < nr * nr; t += nt) {
    const int j = t / nr, i = t % nr;
    Xit[t] = Xi[(i64)i * ldn + j];
  }
  for (i64 t = tid; t < (i64)nr * nc; t += nt) {
    const int i = (int)(t / nc), j = (int)(t % nc);
    GUp[t] = GU[(i64)i * ldr + j];
  }
  for (int t = tid; t < nr * k; t += nt) {
    const int i = t / k, j = t % k;
    Tb[t] = T[(i64)i * ldn + j];
  }
}

// forward solve of one box from its packed record:
//   x_r -= T x_s ;  then (both from the updated x_r)  x_c -= G_L x_r ,  x_r <- X_rr^-1 x_r
// A thread per output row; its factor loads (a column-major column walk) are coalesced
// across the CTA and independent of each other.
template <bool C, int NRB>
__global__ void __launch_bounds__(256) solve_fwd_packed_kernel(const BoxDev* __restrict__ boxes,
                                                                const i64* __restrict__ pk,
                                                                const double* __restrict__ packd,
                                                                const int* __restrict__ ipool,
                                                                double* __restrict__ xd, i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  const BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  S* sm = reinterpret_cast<S*>(smd);
  S* x = reinterpret_cast<S*>(xd);
  const S* Tt = reinterpret_cast<const S*>(packd) + pk[blockIdx.x];
  const S* GLt = Tt + ev2((i64)k * nr);
  const S* Xit = GLt + ev2((i64)nr * nc);
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  S* xs = sm;
  S* xr = xs + k * NRB;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int c0 = 0; c0 < nrhs; c0 += NRB) {
    load_rows<S, NRB>(xs, x, skel, k, ldx, c0, nrhs);
    load_rows<S, NRB>(xr, x, red, nr, ldx, c0, nrhs);
    __syncthreads();
    for (int i = tid; i < nr; i += nt) {
      S acc[NRB];
#pragma unroll
      for (int c = 0; c < NRB; ++c) acc[c] = s_zero(S());
      // loads in predicated chunks of 8: all in flight at once whatever the trip count
      for (int j0 = 0; j0 < k; j0 += 8) {
        S tv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) tv[q] = (j0 + q < k) ? __ldg(Tt + (i64)(j0 + q) * nr + i) : s_zero(S());
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (j0 + q < k)
#pragma unroll
            for (int c = 0; c < NRB; ++c) acc[c] = s_add(acc[c], s_mul(tv[q], xs[(j0 + q) * NRB + c]));
      }
#pragma unroll
      for (int c = 0; c < NRB; ++c) xr[i * NRB + c] = s_sub(xr[i * NRB + c], acc[c]);
    }
    __syncthreads();
    for (int i = tid; i < nc + nr; i += nt) {
      const bool isc = i < nc;
      const int ii = isc ? i : i - nc;
      const S* col = isc ? GLt + ii : Xit + ii;
      const i64 ldc = isc ? nc : nr;
      S acc[NRB];
#pragma unroll
      for (int c = 0; c < NRB; ++c) acc[c] = s_zero(S());
      for (int j0 = 0; j0 < nr; j0 += 16) {
        S gv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) gv[q] = (j0 + q < nr) ? __ldg(col + (i64)(j0 + q) * ldc) : s_zero(S());
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (j0 + q < nr)
#pragma unroll
            for (int c = 0; c < NRB; ++c) acc[c] = s_add(acc[c], s_mul(gv[q], xr[(j0 + q) * NRB + c]));
      }
      if (isc) {
        S* xp = x + (i64)cc[ii] * ldx + c0;
#pragma unroll
        for (int c = 0; c < NRB; ++c)
          if (c0 + c < nrhs) xp[c] = s_sub(xp[c], acc[c]);
      } else {
        S* xp = x + (i64)red[ii] * ldx + c0;
#pragma unroll
        for (int c = 0; c < NRB; ++c)
          if (c0 + c < nrhs) xp[c] = acc[c];
      }
    }
    __syncthreads();
  }
}

// backward solve of one box from its packed record: x_r -= G_U x_c ; x_s -= T^* x_r
// G_U rows by whole warps (lanes over the coupled columns), T^* by a thread per skeleton.
template <bool C, int NRB>
__global__ void __launch_bounds__(256) solve_bwd_packed_kernel(const BoxDev* __restrict__ boxes,
                                                                const i64* __restrict__ pk,
                                                                const double* __restrict__ packd,
                                                                const int* __restrict__ ipool,
                                                                double* __restrict__ xd, i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  const BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  S* sm = reinterpret_cast<S*>(smd);
  S* x = reinterpret_cast<S*>(xd);
  const S* GU = reinterpret_cast<const S*>(packd) + pk[blockIdx.x] + pack_fwd_size(nr, k, nc);
  const S* Tb = GU + ev2((i64)nr * nc);
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  S* xc = sm;
  S* xr = xc + nc * NRB;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int c0 = 0; c0 < nrhs; c0 += NRB) {
    load_rows<S, NRB>(xc, x, cc, nc, ldx, c0, nrhs);
    load_rows<S, NRB>(xr, x, red, nr, ldx, c0, nrhs);
    __syncthreads();
    // RW rows per warp at a time, 8 column loads per row and lane: 8 RW loads in flight per lane
    constexpr int RW = NRB <= 4 ? 4 : 2;
    for (int i0 = warp * RW; i0 < nr; i0 += nw * RW) {
      S acc[RW][NRB];
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int c = 0; c < NRB; ++c) acc[r][c] = s_zero(S());
      for (int j0 = lane; j0 < nc; j0 += 32 * 8) {
        S gv[RW][8];
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            gv[r][q] = (i0 + r < nr && j0 + 32 * q < nc) ? __ldg(GU + (i64)(i0 + r) * nc + j0 + 32 * q) : s_zero(S());
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (j0 + 32 * q < nc)
#pragma unroll
            for (int c = 0; c < NRB; ++c) {
              const S xv = xc[(j0 + 32 * q) * NRB + c];
#pragma unroll
              for (int r = 0; r < RW; ++r) acc[r][c] = s_add(acc[r][c], s_mul(gv[r][q], xv));
            }
      }
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int c = 0; c < NRB; ++c) acc[r][c] = warp_sum(acc[r][c]);
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < RW; ++r) {
          const int i = i0 + r;
          if (i >= nr) break;
#pragma unroll
          for (int c = 0; c < NRB; ++c) {
            const S v = s_sub(xr[i * NRB + c], acc[r][c]);
            xr[i * NRB + c] = v;
            if (c0 + c < nrhs) x[(i64)red[i] * ldx + c0 + c] = v;
          }
        }
      }
    }
    __syncthreads();
    for (int sidx = tid; sidx < k; sidx += nt) {
      S acc[NRB];
#pragma unroll
      for (int c = 0; c < NRB; ++c) acc[c] = s_zero(S());
      for (int i0 = 0; i0 < nr; i0 += 8) {
        S tv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) tv[q] = (i0 + q < nr) ? s_conj(__ldg(Tb + (i64)(i0 + q) * k + sidx)) : s_zero(S());
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (i0 + q < nr)
#pragma unroll
            for (int c = 0; c < NRB; ++c) acc[c] = s_add(acc[c], s_mul(tv[q], xr[(i0 + q) * NRB + c]));
      }
      S* xp = x + (i64)skel[sidx] * ldx + c0;
#pragma unroll
      for (int c = 0; c < NRB; ++c)
        if (c0 + c < nrhs) xp[c] = s_sub(xp[c], acc[c]);
    }
    __syncthreads();
  }
}

// top block: x_S <- A~_SS^-1 x_S (LU with pivots) or x_S <- A~_SS x_S
// Blocked substitution: a 32 x 32 diagonal block is solved by one warp with shuffles (no
// CTA barrier per row), the rows below / above are updated by the whole CTA: 2 barriers
// per 32 rows instead of 2 per row.
template <bool C>
__global__ void __launch_bounds__(1024) top_solve_kernel(const double* __restrict__ LUd, i64 lda, int n,
                                                          const int* __restrict__ ipiv,
                                                          const int* __restrict__ Sidx, double* __restrict__ xd,
                                                          i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double xsd[];
  S* xs = reinterpret_cast<S*>(xsd);
  const S* LU = reinterpret_cast<const S*>(LUd);
  S* x = reinterpret_cast<S*>(xd);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = blockIdx.x; col < nrhs; col += gridDim.x) {   // columns over the grid (explicit inverse)
    for (int i = tid; i < n; i += blockDim.x) xs[i] = x[(i64)Sidx[i] * ldx + col];
    __syncthreads();
    if (tid == 0)
      for (int c = 0; c < n; ++c)
        if (ipiv[c] != c) {
          const S t = xs[c];
          xs[c] = xs[ipiv[c]];
          xs[ipiv[c]] = t;
        }
    __syncthreads();
    for (int p0 = 0; p0 < n; p0 += 32) {          // unit lower, panels top-down
      const int pn = min(32, n - p0);
      if (warp == 0) {
        S v = lane < pn ? xs[p0 + lane] : s_zero(S());
        for (int j = 0; j < pn; ++j) {
          S xj;
          if constexpr (C) {
            xj.x = __shfl_sync(0xffffffffu, v.x, j);
            xj.y = __shfl_sync(0xffffffffu, v.y, j);
          } else {
            xj = __shfl_sync(0xffffffffu, v, j);
          }
          if (lane > j && lane < pn) v = s_sub(v, s_mul(LU[(i64)(p0 + lane) * lda + p0 + j], xj));
        }
        if (lane < pn) xs[p0 + lane] = v;
      }
      __syncthreads();
      for (int i = p0 + pn + warp; i < n; i += blockDim.x / 32) {
        S v = s_zero(S());
        if (lane < pn) v = s_mul(LU[(i64)i * lda + p0 + lane], xs[p0 + lane]);
        v = warp_sum(v);
        if (lane == 0) xs[i] = s_sub(xs[i], v);
      }
      __syncthreads();
    }
    for (int p1 = n; p1 > 0; p1 -= 32) {          // upper, panels bottom-up
      const int p0 = max(0, p1 - 32), pn = p1 - p0;
      if (warp == 0) {
        S v = lane < pn ? xs[p0 + lane] : s_zero(S());
        for (int j = pn - 1; j >= 0; --j) {
          if (lane == j) v = s_div(v, LU[(i64)(p0 + j) * lda + p0 + j]);
          S xj;
          if constexpr (C) {
            xj.x = __shfl_sync(0xffffffffu, v.x, j);
            xj.y = __shfl_sync(0xffffffffu, v.y, j);
          } else {
            xj = __shfl_sync(0xffffffffu, v, j);
          }
          if (lane < j) v = s_sub(v, s_mul(LU[(i64)(p0 + lane) * lda + p0 + j], xj));
        }
        if (lane < pn) xs[p0 + lane] = v;
      }
      __syncthreads();
      for (int i = warp; i < p0; i += blockDim.x / 32) {
        S v = s_zero(S());
        if (lane < pn) v = s_mul(LU[(i64)i * lda + p0 + lane], xs[p0 + lane]);
        v = warp_sum(v);
        if (lane == 0) xs[i] = s_sub(xs[i], v);
      }
      __syncthreads();
    }
    for (int i = tid; i < n; i += blockDim.x) x[(i64)Sidx[i] * ldx + col] = xs[i];
    __syncthreads();
  }
}

template <bool C>
__global__ void __launch_bounds__(1024) top_apply_kernel(const double* __restrict__ Ad, i64 lda, int n,
                                                          const int* __restrict__ Sidx, double* __restrict__ xd,
                                                          i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double xsd[];
  S* xs = reinterpret_cast<S*>(xsd);
  const S* A = reinterpret_cast<const S*>(Ad);
  S* x = reinterpret_cast<S*>(xd);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int i = tid; i < n; i += blockDim.x) xs[i] = x[(i64)Sidx[i] * ldx + col];
    __syncthreads();
    for (int i = warp; i < n; i += blockDim.x / 32) {
      S v = s_zero(S());
      const S* row = A + (i64)i * lda;
      for (int j0 = lane; j0 < n; j0 += 32 * 8) {   // 8 row loads in flight per lane
        S a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = (j0 + 32 * q < n) ? row[j0 + 32 * q] : s_zero(S());
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (j0 + 32 * q < n) v = s_add(v, s_mul(a[q], xs[j0 + 32 * q]));
      }
      v = warp_sum(v);
      if (lane == 0) x[(i64)Sidx[i] * ldx + col] = v;
    }
    __syncthreads();
  }
}

// X = I (n x n, ld in scalars of sc doubles) and iota[i] = i
__global__ void identity_iota_kernel(double* __restrict__ X, i64 ld, int n, int sc, int* __restrict__ iota) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* row = X + (i64)i * ld * sc;
  for (int j = 0; j < n * sc; ++j) row[j] = (j == i * sc) ? 1.0 : 0.0;
  iota[i] = i;
}

// x_tree[t, :] = b[perm[t], :]  /  b[perm[t], :] = x_tree[t, :]
__global__ void permute_rows_kernel(const double* __restrict__ src, i64 lds, double* __restrict__ dst, i64 ldd,
                                    const int64_t* __restrict__ perm, int64_t N, int ncol, int inverse) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (t >= N) return;
  const int64_t o = perm[t];
  for (int j = threadIdx.x; j < ncol; j += blockDim.x) {
    if (!inverse)
      dst[t * ldd + j] = src[o * lds + j];
    else
      dst[o * ldd + j] = src[t * lds + j];
  }
}

// the same for narrow right-hand sides (ncol < 32): a thread per (row, column)
__global__ void permute_rows_flat_kernel(const double* __restrict__ src, i64 lds, double* __restrict__ dst, i64 ldd,
                                         const int64_t* __restrict__ perm, int64_t N, int ncol, int inverse) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * ncol) return;
  const int64_t t = e / ncol;
  const int j = (int)(e - t * ncol);
  const int64_t o = perm[t];
  if (!inverse)
    dst[t * ldd + j] = src[o * lds + j];
  else
    dst[o * ldd + j] = src[t * lds + j];
}

// ---------------------------------------------------------------------------
// Triangular form (Remark PAPER.md:577-611), real symmetric spd:
//   V = E [C 0; M_U^T I],  W = [C^T M_U; 0 I] F,  eliminated blocks of the middle factor = I.
// Stored per box: T (f_T), C (f_Xrr, lower), C^-1 (f_Xinv, lower), M_U = C^-1 X_rc (f_GU).
// ---------------------------------------------------------------------------
// forward solve: x_r -= T x_s ; x_r <- C^-1 x_r ; x_c -= M_U^T x_r
__global__ void __launch_bounds__(256) solve_fwd_tri_kernel(const BoxDev* __restrict__ boxes,
                                                             const double* __restrict__ fpool,
                                                             const int* __restrict__ ipool, double* __restrict__ x,
                                                             i64 ldx, int nrhs) {
  extern __shared__ __align__(16) double smd[];
  const BoxDev b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn, ldr = b.ldr;
  double* xs = smd;
  double* xr = xs + k;
  double* yr = xr + nr;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const double* T = fpool + b.f_T;
  const double* Ci = fpool + b.f_Xinv;
  const double* MU = fpool + b.f_GU;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int s = tid; s < k; s += blockDim.x) xs[s] = x[(i64)skel[s] * ldx + col];
    __syncthreads();
    for (int i = tid; i < nr; i += blockDim.x) {
      double v = x[(i64)red[i] * ldx + col];
      for (int s = 0; s < k; ++s) v -= T[(i64)i * ldn + s] * xs[s];
      xr[i] = v;
    }
    __syncthreads();
    for (int i = warp; i < nr; i += blockDim.x / 32) {       // y_r = C^-1 x_r (lower)
      double v = 0.0;
      for (int j = lane; j <= i; j += 32) v += Ci[(i64)i * ldn + j] * xr[j];
      v = warp_sum(v);
      if (lane == 0) {
        yr[i] = v;
        x[(i64)red[i] * ldx + col] = v;
      }
    }
    __syncthreads();
    for (int j = tid; j < nc; j += blockDim.x) {              // x_c -= M_U^T y_r
      double v = 0.0;
      for (int i = 0; i < nr; ++i) v += MU[(i64)i * ldr + j] * yr[i];
      x[(i64)cc[j] * ldx + col] -= v;
    }
    __syncthreads();
  }
}

// backward solve: x_r <- C^-T (x_r - M_U x_c) ; x_s -= T^T x_r
__global__ void __launch_bounds__(256) solve_bwd_tri_kernel(const BoxDev* __restrict__ boxes,
                                                             const double* __restrict__ fpool,
                                                             const int* __restrict__ ipool, double* __restrict__ x,
                                                             i64 ldx, int nrhs) {
  extern __shared__ __align__(16) double smd[];
  const BoxDev b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn, ldr = b.ldr;
  double* xc = smd;
  double* tr = xc + nc;
  double* xr = tr + nr;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const double* T = fpool + b.f_T;
  const double* Ci = fpool + b.f_Xinv;
  const double* MU = fpool + b.f_GU;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int j = tid; j < nc; j += blockDim.x) xc[j] = x[(i64)cc[j] * ldx + col];
    __syncthreads();
    for (int i = warp; i < nr; i += blockDim.x / 32) {        // t_r = x_r - M_U x_c
      double v = 0.0;
      for (int j = lane; j < nc; j += 32) v += MU[(i64)i * ldr + j] * xc[j];
      v = warp_sum(v);
      if (lane == 0) tr[i] = x[(i64)red[i] * ldx + col] - v;
    }
    __syncthreads();
    for (int i = tid; i < nr; i += blockDim.x) {              // x_r = C^-T t_r (upper)
      double v = 0.0;
      for (int m = i; m < nr; ++m) v += Ci[(i64)m * ldn + i] * tr[m];
      xr[i] = v;
      x[(i64)red[i] * ldx + col] = v;
    }
    __syncthreads();
    for (int s = tid; s < k; s += blockDim.x) {               // x_s -= T^T x_r
      double v = 0.0;
      for (int i = 0; i < nr; ++i) v += T[(i64)i * ldn + s] * xr[i];
      x[(i64)skel[s] * ldx + col] -= v;
    }
    __syncthreads();
  }
}

// apply, forward half (W = [C^T M_U; 0 I] F): x_s += T^T x_r ; x_r <- C^T x_r + M_U x_c
__global__ void __launch_bounds__(256) apply_fwd_tri_kernel(const BoxDev* __restrict__ boxes,
                                                             const double* __restrict__ fpool,
                                                             const int* __restrict__ ipool, double* __restrict__ x,
                                                             i64 ldx, int nrhs) {
  extern __shared__ __align__(16) double smd[];
  const BoxDev b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn, ldr = b.ldr;
  double* xc = smd;
  double* xr = xc + nc;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const double* T = fpool + b.f_T;
  const double* Cf = fpool + b.f_Xrr;
  const double* MU = fpool + b.f_GU;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int i = tid; i < nr; i += blockDim.x) xr[i] = x[(i64)red[i] * ldx + col];
    __syncthreads();
    for (int s = tid; s < k; s += blockDim.x) {
      double v = 0.0;
      for (int i = 0; i < nr; ++i) v += T[(i64)i * ldn + s] * xr[i];
      x[(i64)skel[s] * ldx + col] += v;
    }
    __syncthreads();
    // c = near \ red holds b's skeletons: read x_c after the F update
    for (int j = tid; j < nc; j += blockDim.x) xc[j] = x[(i64)cc[j] * ldx + col];
    __syncthreads();
    for (int i = warp; i < nr; i += blockDim.x / 32) {
      double v = 0.0;
      for (int m = i + lane; m < nr; m += 32) v += Cf[(i64)m * ldn + i] * xr[m];
      for (int j = lane; j < nc; j += 32) v += MU[(i64)i * ldr + j] * xc[j];
      v = warp_sum(v);
      if (lane == 0) x[(i64)red[i] * ldx + col] = v;
    }
    __syncthreads();
  }
}

// apply, backward half (V = E [C 0; M_U^T I]): x_c += M_U^T x_r ; x_r <- C x_r ; x_r += T x_s
__global__ void __launch_bounds__(256) apply_bwd_tri_kernel(const BoxDev* __restrict__ boxes,
                                                             const double* __restrict__ fpool,
                                                             const int* __restrict__ ipool, double* __restrict__ x,
                                                             i64 ldx, int nrhs) {
  extern __shared__ __align__(16) double smd[];
  const BoxDev b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn, ldr = b.ldr;
  double* xs = smd;
  double* xr = xs + k;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const double* T = fpool + b.f_T;
  const double* Cf = fpool + b.f_Xrr;
  const double* MU = fpool + b.f_GU;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int i = tid; i < nr; i += blockDim.x) xr[i] = x[(i64)red[i] * ldx + col];
    __syncthreads();
    for (int j = tid; j < nc; j += blockDim.x) {
      double v = 0.0;
      for (int i = 0; i < nr; ++i) v += MU[(i64)i * ldr + j] * xr[i];
      x[(i64)cc[j] * ldx + col] += v;
    }
    __syncthreads();
    // the skeletons are part of c: read x_s after the L update
    for (int s = tid; s < k; s += blockDim.x) xs[s] = x[(i64)skel[s] * ldx + col];
    __syncthreads();
    for (int i = warp; i < nr; i += blockDim.x / 32) {
      double v = 0.0;
      for (int j = lane; j <= i; j += 32) v += Cf[(i64)i * ldn + j] * xr[j];
      for (int s = lane; s < k; s += 32) v += T[(i64)i * ldn + s] * xs[s];
      v = warp_sum(v);
      if (lane == 0) x[(i64)red[i] * ldx + col] = v;
    }
    __syncthreads();
  }
}

}  // namespace rsrs
