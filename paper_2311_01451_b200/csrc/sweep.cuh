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

// forward solve of one box: x_r -= T x_s ; x_c -= G_L x_r ; x_r <- X_rr^-1 x_r
template <bool C>
__global__ void __launch_bounds__(256) solve_fwd_kernel(const BoxDev* __restrict__ boxes,
                                                         const double* __restrict__ fpoold,
                                                         const int* __restrict__ ipool, double* __restrict__ xd,
                                                         i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  S* sm = reinterpret_cast<S*>(smd);
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* x = reinterpret_cast<S*>(xd);
  const S zero = s_zero(S());
  const BoxDev b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn;
  S* xs = sm;
  S* xr = xs + k;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const S* T = fpool + b.f_T;
  const S* GL = fpool + b.f_GL;
  const S* Xi = fpool + b.f_Xinv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int s = tid; s < k; s += blockDim.x) xs[s] = x[(i64)skel[s] * ldx + col];
    __syncthreads();
    for (int i = tid; i < nr; i += blockDim.x) {
      S v = x[(i64)red[i] * ldx + col];
      for (int s = 0; s < k; ++s) v = s_sub(v, s_mul(T[(i64)i * ldn + s], xs[s]));
      xr[i] = v;
    }
    __syncthreads();
    for (int ci = warp; ci < nc; ci += blockDim.x / 32) {
      S v = zero;
      for (int j = lane; j < nr; j += 32) v = s_add(v, s_mul(GL[(i64)ci * ldn + j], xr[j]));
      v = warp_sum(v);
      if (lane == 0) x[(i64)cc[ci] * ldx + col] = s_sub(x[(i64)cc[ci] * ldx + col], v);
    }
    for (int i = warp; i < nr; i += blockDim.x / 32) {
      S v = zero;
      for (int j = lane; j < nr; j += 32) v = s_add(v, s_mul(Xi[(i64)i * ldn + j], xr[j]));
      v = warp_sum(v);
      if (lane == 0) x[(i64)red[i] * ldx + col] = v;
    }
    __syncthreads();
  }
}

// backward solve of one box: x_r -= G_U x_c ; x_s -= T^T x_r
template <bool C>
__global__ void __launch_bounds__(256) solve_bwd_kernel(const BoxDev* __restrict__ boxes,
                                                         const double* __restrict__ fpoold,
                                                         const int* __restrict__ ipool, double* __restrict__ xd,
                                                         i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  S* sm = reinterpret_cast<S*>(smd);
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* x = reinterpret_cast<S*>(xd);
  const S zero = s_zero(S());
  const BoxDev b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn;
  const int ldr = b.ldr;
  S* xc = sm;
  S* xr = xc + nc;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const S* T = fpool + b.f_T;
  const S* GU = fpool + b.f_GU;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int j = tid; j < nc; j += blockDim.x) xc[j] = x[(i64)cc[j] * ldx + col];
    __syncthreads();
    for (int i = warp; i < nr; i += blockDim.x / 32) {
      S v = zero;
      for (int j = lane; j < nc; j += 32) v = s_add(v, s_mul(GU[(i64)i * ldr + j], xc[j]));
      v = warp_sum(v);
      if (lane == 0) {
        const S nv = s_sub(x[(i64)red[i] * ldx + col], v);
        x[(i64)red[i] * ldx + col] = nv;
        xr[i] = nv;
      }
    }
    __syncthreads();
    for (int s = tid; s < k; s += blockDim.x) {   // x_s -= T^* x_r
      S v = zero;
      for (int i = 0; i < nr; ++i) v = s_add(v, s_mul(s_conj(T[(i64)i * ldn + s]), xr[i]));
      x[(i64)skel[s] * ldx + col] = s_sub(x[(i64)skel[s] * ldx + col], v);
    }
    __syncthreads();
  }
}

// apply, forward half of one box: x_s += T^T x_r ; x_r += G_U x_c ; x_r <- X_rr x_r
template <bool C>
__global__ void __launch_bounds__(256) apply_fwd_kernel(const BoxDev* __restrict__ boxes,
                                                         const double* __restrict__ fpoold,
                                                         const int* __restrict__ ipool, double* __restrict__ xd,
                                                         i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  S* sm = reinterpret_cast<S*>(smd);
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* x = reinterpret_cast<S*>(xd);
  const S zero = s_zero(S());
  const BoxDev b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn;
  const int ldr = b.ldr;
  S* xc = sm;
  S* xr = xc + nc;
  S* xr2 = xr + nr;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const S* T = fpool + b.f_T;
  const S* GU = fpool + b.f_GU;
  const S* Xrr = fpool + b.f_Xrr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int i = tid; i < nr; i += blockDim.x) xr[i] = x[(i64)red[i] * ldx + col];
    __syncthreads();
    for (int s = tid; s < k; s += blockDim.x) {   // x_s += T^* x_r
      S v = zero;
      for (int i = 0; i < nr; ++i) v = s_add(v, s_mul(s_conj(T[(i64)i * ldn + s]), xr[i]));
      x[(i64)skel[s] * ldx + col] = s_add(x[(i64)skel[s] * ldx + col], v);
    }
    __syncthreads();
    for (int j = tid; j < nc; j += blockDim.x) xc[j] = x[(i64)cc[j] * ldx + col];
    __syncthreads();
    for (int i = warp; i < nr; i += blockDim.x / 32) {
      S v = zero;
      for (int j = lane; j < nc; j += 32) v = s_add(v, s_mul(GU[(i64)i * ldr + j], xc[j]));
      v = warp_sum(v);
      if (lane == 0) xr[i] = s_add(xr[i], v);
    }
    __syncthreads();
    for (int i = warp; i < nr; i += blockDim.x / 32) {
      S v = zero;
      for (int j = lane; j < nr; j += 32) v = s_add(v, s_mul(Xrr[(i64)i * ldn + j], xr[j]));
      v = warp_sum(v);
      if (lane == 0) xr2[i] = v;
    }
    __syncthreads();
    for (int i = tid; i < nr; i += blockDim.x) x[(i64)red[i] * ldx + col] = xr2[i];
    __syncthreads();
  }
}

// apply, backward half of one box: x_c += G_L x_r ; x_r += T x_s
template <bool C>
__global__ void __launch_bounds__(256) apply_bwd_kernel(const BoxDev* __restrict__ boxes,
                                                         const double* __restrict__ fpoold,
                                                         const int* __restrict__ ipool, double* __restrict__ xd,
                                                         i64 ldx, int nrhs) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double smd[];
  S* sm = reinterpret_cast<S*>(smd);
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* x = reinterpret_cast<S*>(xd);
  const S zero = s_zero(S());
  const BoxDev b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, nc = b.nc;
  if (nr <= 0) return;
  const int ldn = b.ldn;
  S* xs = sm;
  S* xr = xs + k;
  const int* red = ipool + b.f_red;
  const int* skel = ipool + b.f_skel;
  const int* cc = ipool + b.f_c;
  const S* T = fpool + b.f_T;
  const S* GL = fpool + b.f_GL;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int col = 0; col < nrhs; ++col) {
    for (int i = tid; i < nr; i += blockDim.x) xr[i] = x[(i64)red[i] * ldx + col];
    __syncthreads();
    for (int ci = warp; ci < nc; ci += blockDim.x / 32) {
      S v = zero;
      for (int j = lane; j < nr; j += 32) v = s_add(v, s_mul(GL[(i64)ci * ldn + j], xr[j]));
      v = warp_sum(v);
      if (lane == 0) x[(i64)cc[ci] * ldx + col] = s_add(x[(i64)cc[ci] * ldx + col], v);
    }
    __syncthreads();
    for (int s = tid; s < k; s += blockDim.x) xs[s] = x[(i64)skel[s] * ldx + col];
    __syncthreads();
    for (int i = tid; i < nr; i += blockDim.x) {
      S v = xr[i];
      for (int s = 0; s < k; ++s) v = s_add(v, s_mul(T[(i64)i * ldn + s], xs[s]));
      x[(i64)red[i] * ldx + col] = v;
    }
    __syncthreads();
  }
}

// top block: x_S <- A~_SS^-1 x_S (LU with pivots) or x_S <- A~_SS x_S
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
  const int tid = threadIdx.x;
  for (int col = 0; col < nrhs; ++col) {
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
    for (int c = 0; c < n; ++c) {  // unit lower
      const S xc = xs[c];
      for (int i = c + 1 + tid; i < n; i += blockDim.x) xs[i] = s_sub(xs[i], s_mul(LU[(i64)i * lda + c], xc));
      __syncthreads();
    }
    for (int c = n - 1; c >= 0; --c) {  // upper
      if (tid == 0) xs[c] = s_div(xs[c], LU[(i64)c * lda + c]);
      __syncthreads();
      const S xc = xs[c];
      for (int i = tid; i < c; i += blockDim.x) xs[i] = s_sub(xs[i], s_mul(LU[(i64)i * lda + c], xc));
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
      for (int j = lane; j < n; j += 32) v = s_add(v, s_mul(A[(i64)i * lda + j], xs[j]));
      v = warp_sum(v);
      if (lane == 0) x[(i64)Sidx[i] * ldx + col] = v;
    }
    __syncthreads();
  }
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
    for (int j = tid; j < nc; j += blockDim.x) xc[j] = x[(i64)cc[j] * ldx + col];
    __syncthreads();
    for (int s = tid; s < k; s += blockDim.x) {
      double v = 0.0;
      for (int i = 0; i < nr; ++i) v += T[(i64)i * ldn + s] * xr[i];
      x[(i64)skel[s] * ldx + col] += v;
    }
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
    for (int s = tid; s < k; s += blockDim.x) xs[s] = x[(i64)skel[s] * ldx + col];
    __syncthreads();
    for (int j = tid; j < nc; j += blockDim.x) {
      double v = 0.0;
      for (int i = 0; i < nr; ++i) v += MU[(i64)i * ldr + j] * xr[i];
      x[(i64)cc[j] * ldx + col] += v;
    }
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
