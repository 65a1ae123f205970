// Per-box dense kernels of the RSRS sweep (one CTA per box / matrix).
#pragma once
#include "common.cuh"

namespace rsrs {

// ---------------------------------------------------------------------------
// Interpolative decomposition of S = [Y'', Z''] / sqrt(2w)
// through its Gram H = S S^* (Hermitian for complex128): greedy max-residual-norm pivoting (the pivots and
// R of column-pivoted QR of S^T), stop at R_jj <= atol(l), T = (R11^-1 R12)^T.
// Also writes the skeleton / redundant / coupled index lists of the box.
// ---------------------------------------------------------------------------
template <bool C>
__global__ void __launch_bounds__(256) id_kernel(BoxDev* __restrict__ boxes, const double* __restrict__ wsd,
                                                 int* __restrict__ iws, double* __restrict__ fpoold,
                                                 int* __restrict__ ipool, const int* __restrict__ gidx,
                                                 double atol2, int p, int oversample, int hsame,
                                                 int pullmode) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double Hsd[];
  S* Hs = reinterpret_cast<S*>(Hsd);
  const S* ws = reinterpret_cast<const S*>(wsd);
  S* fpool = reinterpret_cast<S*>(fpoold);
  BoxDev& b = boxes[blockIdx.x];
  const int nb = b.nb, r = b.r;
  if (b.status != ST_OK) {                 // e.g. too few samples for this near field
    // keep every row as a skeleton so that later near lists / compaction stay in range
    // (the factorization is abandoned at the end of the level)
    int* skelrow = iws + b.off_skelrow;
    const int* near = iws + b.off_rows;
    for (int t = threadIdx.x; t < nb; t += blockDim.x) skelrow[t] = b.row0 + t;
    for (int t = threadIdx.x; t < r; t += blockDim.x) {
      iws[b.off_crow + t] = near[t];
      iws[b.off_cpos + t] = t;
    }
    if (threadIdx.x == 0) {
      b.k = nb;
      b.nr = 0;
      b.nc = r;
      b.ncp = r;
    }
    return;
  }
  const int ldh = nb + 1;
  // H = [Y'' Z''][Y'' Z'']^T is unnormalised: S = [Y' Z'] / sqrt(2w) => compare
  // H_jj against 2 w atol^2 (T = (R11^-1 R12)^T is scale invariant)
  const double thr = atol2 * 2.0 * (double)(p - r);
  int* perm = reinterpret_cast<int*>(Hs + nb * ldh);
  int* rank_of = perm + nb;        // sorted position of pivot-order entries
  int* is_red = rank_of + nb;
  __shared__ double pval;
  __shared__ int pidx, kfinal;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const S* H = ws + b.off_h;
  const int ldhg = b.ldn;
  // H = H_Y + H_Z = Y'' Y''^* + Z'' Z''^* (the two halves of S S^*, written by gemm_nt)
  // symmetric shortcuts (hsame): 1 = Z'' = Y'' (A = A^*, Psi = Omega): H = 2 H_Y;
  // 2 = Z'' = conj(Y'') (complex symmetric A = A^T, Psi = conj(Omega)): H = H_Y + conj(H_Y) = 2 Re(H_Y)
  const S* H2 = hsame ? H : H + (i64)nb * ldhg;
  for (int idx = tid; idx < nb * nb; idx += 256) {
    const i64 g = (i64)(idx / nb) * ldhg + idx % nb;
    Hs[(idx / nb) * ldh + idx % nb] = s_add(H[g], hsame == 2 ? s_conj(H2[g]) : H2[g]);
  }
  for (int i = tid; i < nb; i += 256) perm[i] = i;
  if (tid == 0) kfinal = nb;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (warp == 0) {
      double bv = -1.0;
      int bi = nb;
      for (int i = j + lane; i < nb; i += 32) {
        const double v = s_real(Hs[i * ldh + i]);
        if (v > bv || (v == bv && i < bi)) {
          bv = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        pval = bv;
        pidx = bi;
      }
    }
    __syncthreads();
    if (!(pval > thr)) {
      if (tid == 0) kfinal = j;
      break;
    }
    const int q = pidx;
    if (q != j) {
      for (int c = tid; c < nb; c += 256) {
        const S t = Hs[j * ldh + c];
        Hs[j * ldh + c] = Hs[q * ldh + c];
        Hs[q * ldh + c] = t;
      }
      __syncthreads();
      for (int c = tid; c < nb; c += 256) {
        const S t = Hs[c * ldh + j];
        Hs[c * ldh + j] = Hs[c * ldh + q];
        Hs[c * ldh + q] = t;
      }
      if (tid == 0) {
        const int t = perm[j];
        perm[j] = perm[q];
        perm[q] = t;
      }
      __syncthreads();
    }
    const double rjj = sqrt(s_real(Hs[j * ldh + j]));
    __syncthreads();
    for (int c = j + 1 + tid; c < nb; c += 256) Hs[j * ldh + c] = s_scale(Hs[j * ldh + c], 1.0 / rjj);
    if (tid == 0) Hs[j * ldh + j] = s_scale(s_one(S()), rjj);
    __syncthreads();
    // Schur complement H_il -= conj(R_ji) R_jl  (H = R^* R)
    const int nt = nb - j - 1;
    for (int idx = tid; idx < nt * nt; idx += 256) {
      const int i = j + 1 + idx / nt, l = j + 1 + idx % nt;
      Hs[i * ldh + l] = s_sub(Hs[i * ldh + l], s_mul(s_conj(Hs[j * ldh + i]), Hs[j * ldh + l]));
    }
    __syncthreads();
  }
  __syncthreads();
  const int k = kfinal;
  const int nr = nb - k;
  const int w = p - r;
  // sorted ranks of skeleton (pivot positions 0..k-1) and redundant (k..nb-1) entries
  for (int s = tid; s < nb; s += 256) {
    const bool sk = s < k;
    const int lo = sk ? 0 : k, hi = sk ? k : nb;
    int rk = 0;
    for (int q2 = lo; q2 < hi; ++q2) rk += perm[q2] < perm[s];
    rank_of[s] = rk;
    is_red[perm[s]] = sk ? 0 : 1;
  }
  __syncthreads();
  int* skelrow = iws + b.off_skelrow;
  int* redrow = iws + b.off_redrow;
  int* red_tp = ipool + b.f_red;
  int* skel_tp = ipool + b.f_skel;
  for (int s = tid; s < nb; s += 256) {
    const int row = b.row0 + perm[s];
    if (s < k) {
      skelrow[rank_of[s]] = row;
      skel_tp[rank_of[s]] = gidx[row];
    } else {
      redrow[rank_of[s]] = row;
      red_tp[rank_of[s]] = gidx[row];
    }
  }
  // T = (R11^-1 R12)^*, rows = redundant (sorted), cols = skeleton (sorted)
  if (nr > 0 && k > 0) {
    S* T = fpool + b.f_T;
    const int ldn = b.ldn;
    for (int c = tid; c < nr; c += 256) {
      // back substitution R11 x = R12[:, c]  (x kept in the R12 column of Hs)
      const int col = k + c;
      for (int s = k - 1; s >= 0; --s) {
        S v = Hs[s * ldh + col];
        for (int q2 = s + 1; q2 < k; ++q2) v = s_sub(v, s_mul(Hs[s * ldh + q2], Hs[q2 * ldh + col]));
        Hs[s * ldh + col] = s_div(v, Hs[s * ldh + s]);
      }
      const int ri = rank_of[col];
      for (int s = 0; s < k; ++s) T[(i64)ri * ldn + rank_of[s]] = s_conj(Hs[s * ldh + col]);
    }
  }
  // coupled set c = near \ red, as two groups in near order (ballot compaction by warp 0):
  // rows that will not be eliminated later on this level (own skeletons, skeletons of
  // eliminated neighbours) first, then the rows of not-yet-eliminated neighbours -- those
  // take their L/U update by a pull when their own box comes up (single GPU)
  __shared__ int ncp_s;
  if (warp == 0) {
    const int* near = iws + b.off_rows;
    const int* nflag = iws + b.off_nflag;
    int* crow = iws + b.off_crow;
    int* cpos = iws + b.off_cpos;
    int* c_tp = ipool + b.f_c;
    int base = 0;
    for (int grp = 0; grp < 2; ++grp) {
      if (grp == 1 && lane == 0) ncp_s = base;
      for (int p0 = 0; p0 < r; p0 += 32) {
        const int pp = p0 + lane;
        bool keep = false;
        int row = 0;
        if (pp < r) {
          row = near[pp];
          const int loc = pp - b.self_pos;
          // push mode: one group in near order (the order does not depend on rank ownership)
          keep = !(loc >= 0 && loc < nb && is_red[loc]) && (pullmode ? nflag[pp] : 0) == grp;
        }
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (keep) {
          const int o = base + __popc(mask & ((1u << lane) - 1u));
          crow[o] = row;
          cpos[o] = pp;
          c_tp[o] = gidx[row];
        }
        base += __popc(mask);
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    b.k = k;
    b.nr = nr;
    b.nc = r - nr;
    b.ncp = ncp_s;
    if (k > w - oversample) b.status = ST_SAMPLES;   // rank not resolvable with p samples
  }
}

// ---------------------------------------------------------------------------
// X^-1 of an n x n matrix (n <= 64) by Gauss-Jordan elimination with partial
// pivoting on the augmented [X | I] held in REGISTERS (256 threads; thread t
// owns rows t/16 + 16a, columns t%16 + 16b of the 64 x 128 block).  Pivot rows
// are not swapped: step c eliminates column c from every other row with the
// largest remaining |x_ic| (argmax computed redundantly by every warp with
// shuffles), so the left half ends as a permutation and X^-1[c, :] is the
// right half of the step-c pivot row.  Two barriers per column.
// Returns false (on every thread) if a pivot is exactly zero.
// ---------------------------------------------------------------------------
template <class S>
__device__ bool gj_inverse_reg(const S* __restrict__ Xs, int ldx, int n, S* __restrict__ Xinv, int ldo,
                               S* colbuf /* smem [2][64] */, S* rowbuf /* smem [2][128] */, int* prow /* smem [64] */) {
  constexpr int RA = 4, CA = 8;
  const int tid = threadIdx.x, lane = tid & 31;
  const int tr = tid >> 4, tc = tid & 15;
  const S zero = s_zero(S()), one = s_one(S());
  S a[RA][CA];
#pragma unroll
  for (int ra = 0; ra < RA; ++ra) {
    const int i = tr + 16 * ra;
#pragma unroll
    for (int cb = 0; cb < CA; ++cb) {
      const int j = tc + 16 * cb;
      S v;
      if (j < 64) v = (i < n && j < n) ? Xs[i * ldx + j] : (i == j ? one : zero);
      else v = (j - 64 == i) ? one : zero;
      a[ra][cb] = v;
    }
  }
  unsigned long long used = 0;           // rows already used as pivots (same on every thread)
  bool ok = true;
#pragma unroll
  for (int cblk = 0; cblk < 4; ++cblk) {
    for (int cc = 0; cc < 16 && ok; ++cc) {
      const int c = 16 * cblk + cc;
      if (c >= n) break;
      const int buf = c & 1;
      if (tc == cc)
#pragma unroll
        for (int ra = 0; ra < RA; ++ra) colbuf[buf * 64 + tr + 16 * ra] = a[ra][cblk];
      __syncthreads();
      // argmax |x_ic| over unused rows i < n (lowest index on ties), in every warp
      double bv = -1.0;
      int bi = 64;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        if (i < n && !((used >> i) & 1ull)) {
          const double v = s_abs(colbuf[buf * 64 + i]);
          if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (!(bv > 0.0)) {
        ok = false;
        break;
      }
      const int pr = bi;
      used |= 1ull << pr;
      if (tid == 0) prow[c] = pr;
      if (tr == (pr & 15)) {              // owners of the pivot row publish it (select chain:
        const int sel = pr >> 4;          // no dynamic register indexing)
#pragma unroll
        for (int cb = 0; cb < CA; ++cb) {
          S v = a[0][cb];
#pragma unroll
          for (int ra = 1; ra < RA; ++ra) v = (ra == sel) ? a[ra][cb] : v;
          rowbuf[buf * 128 + tc + 16 * cb] = v;
        }
      }
      __syncthreads();
      const S piv = colbuf[buf * 64 + pr];
      const S rpiv = s_div(one, piv);
#pragma unroll
      for (int ra = 0; ra < RA; ++ra) {
        const int i = tr + 16 * ra;
        if (i == pr) {
#pragma unroll
          for (int cb = 0; cb < CA; ++cb) a[ra][cb] = s_mul(a[ra][cb], rpiv);
        } else {
          const S m = s_mul(colbuf[buf * 64 + i], rpiv);
#pragma unroll
          for (int cb = 0; cb < CA; ++cb) a[ra][cb] = s_sub(a[ra][cb], s_mul(m, rowbuf[buf * 128 + tc + 16 * cb]));
        }
      }
    }
  }
  if (!ok) return false;
  __syncthreads();
  // X^-1[c, :] = right half of pivot row prow[c]; invert the map through colbuf's int view
  int* pos = reinterpret_cast<int*>(rowbuf);   // row -> step
  if (tid < n) pos[prow[tid]] = tid;
  __syncthreads();
#pragma unroll
  for (int ra = 0; ra < RA; ++ra) {
    const int i = tr + 16 * ra;
    if (i >= n) continue;
    const int c = pos[i];
#pragma unroll
    for (int cb = 4; cb < CA; ++cb) {
      const int j = tc + 16 * cb - 64;
      if (j < n) Xinv[(i64)c * ldo + j] = a[ra][cb];
    }
  }
  return true;
}

// ---------------------------------------------------------------------------
// Block extraction + elimination factors of one box (PAPER.md:1213-1218,
// 934-955).  X_Y = Yhat_r Omegahat_near^dagger evaluated through the
// pre-update pseudo-inverse: Omegahat_near = F_loc Omega_near =>
// Omegahat^dagger = Omega^dagger F_loc^-1, so X_Y = (W_r - T W_s) F_loc^-1
// with W = Y_b Omega_near^dagger (reading R5).  Same for X_Z.
// Then LU(X_rr) with partial pivoting and X_rr^-1; X_rc and X_cr are written
// densely for the G_U / G_L GEMMs.
// ---------------------------------------------------------------------------
template <bool C>
__global__ void __launch_bounds__(256) extract_lu_kernel(BoxDev* __restrict__ boxes, double* __restrict__ wsd,
                                                         const int* __restrict__ iws,
                                                         double* __restrict__ fpoold, int sym, int tri) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double Xsd[];
  S* Xs = reinterpret_cast<S*>(Xsd);
  S* ws = reinterpret_cast<S*>(wsd);
  S* fpool = reinterpret_cast<S*>(fpoold);
  const S zero = s_zero(S());
  BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr, k = b.k, r = b.r, nb = b.nb, nc = b.nc;
  if (nr <= 0 || b.status != ST_OK) return;
  const int ldn = b.ldn;
  const int ldx = nr + 1;
  // X_rr (LU factors) in shared memory; inverses / triangular factors go straight to the
  // factor pool (ld ldn), so that boxes up to ~165 rows (real) fit.  Before X_rr is gathered
  // the same space holds T (n_r x k <= n_b^2 / 4); the index lists sit behind n_b (n_b + 1).
  int* ipiv = reinterpret_cast<int*>(Xs + (i64)nb * (nb + 1));
  int* redloc = ipiv + nr;
  int* skelloc = redloc + nb;
  __shared__ int singular;
  __shared__ double pv;
  __shared__ int pi;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int* redrow = iws + b.off_redrow;
  const int* skelrow = iws + b.off_skelrow;
  const int* cpos = iws + b.off_cpos;
  for (int i = tid; i < nr; i += 256) redloc[i] = redrow[i] - b.row0;
  for (int s = tid; s < k; s += 256) skelloc[s] = skelrow[s] - b.row0;
  if (tid == 0) singular = 0;
  __syncthreads();
  const S* T = fpool + b.f_T;
  const i64 ldr = b.ldr;
  const S* WY = ws + b.off_aug + (i64)b.rmax * ldr;
  // symmetric shortcut (Psi = Omega, Z = Y): the Z side equals the Y side
  const S* WZ = sym ? WY : ws + b.off_aug + (i64)(b.rmax + nb) * ldr + (i64)b.rmax * ldr;
  S* XY = ws + b.off_xy;
  S* XZ = ws + b.off_xz;
  // T staged in shared memory (the X_rr space, not yet in use)
  S* Ts = Xs;
  for (int idx = tid; idx < nr * k; idx += 256) Ts[idx] = T[(i64)(idx / k) * ldn + idx % k];
  __syncthreads();
  // 1. row combination X = W_r - T W_s: a thread per near column j; the column's skeleton entries
  //    (chunks of 16) are held in registers and the redundant rows go 8 at a time, every load of a
  //    group independent (a thread-per-element loop waited one memory round trip per element)
  constexpr int SKC = 8;
  for (int j = tid; j < r; j += 256) {
    for (int s0 = 0; s0 < k || s0 == 0; s0 += SKC) {
      S wy[SKC], wz[SKC];
#pragma unroll
      for (int q = 0; q < SKC; ++q) {
        const bool ok = s0 + q < k;
        wy[q] = ok ? WY[(i64)skelloc[s0 + q] * ldr + j] : zero;
        wz[q] = ok ? WZ[(i64)skelloc[s0 + q] * ldr + j] : zero;
      }
      for (int i0 = 0; i0 < nr; i0 += 8) {
        S vy[8], vz[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u;
          if (i < nr) {
            // first chunk starts from W_r, later ones from the partial sums
            vy[u] = s0 == 0 ? WY[(i64)redloc[i] * ldr + j] : XY[(i64)i * ldr + j];
            vz[u] = s0 == 0 ? WZ[(i64)redloc[i] * ldr + j] : XZ[(i64)i * ldr + j];
          } else {
            vy[u] = vz[u] = zero;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u;
          if (i >= nr) break;
#pragma unroll
          for (int q = 0; q < SKC; ++q)
            if (s0 + q < k) {
              const S t = Ts[i * k + s0 + q];
              vy[u] = s_sub(vy[u], s_mul(t, wy[q]));
              vz[u] = s_sub(vz[u], s_mul(t, wz[q]));
            }
          XY[(i64)i * ldr + j] = vy[u];
          XZ[(i64)i * ldr + j] = vz[u];
        }
      }
    }
  }
  __syncthreads();
  // 2. column fix X[:, red] -= X[:, skel] T^*  (F_loc^-1 on b's own columns): a thread per row i,
  //    X[i, skel] in registers (chunks of 16), the redundant columns 8 at a time
  if (k > 0) {
    for (int i = tid; i < nr; i += 256) {
      for (int s0 = 0; s0 < k; s0 += SKC) {
        S xy[SKC], xz[SKC];
#pragma unroll
        for (int q = 0; q < SKC; ++q) {
          const bool ok = s0 + q < k;
          xy[q] = ok ? XY[(i64)i * ldr + b.self_pos + skelloc[s0 + q]] : zero;
          xz[q] = ok ? XZ[(i64)i * ldr + b.self_pos + skelloc[s0 + q]] : zero;
        }
        for (int j0 = 0; j0 < nr; j0 += 8) {
          S vy[8], vz[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int jj = j0 + u;
            vy[u] = jj < nr ? XY[(i64)i * ldr + b.self_pos + redloc[jj]] : zero;
            vz[u] = jj < nr ? XZ[(i64)i * ldr + b.self_pos + redloc[jj]] : zero;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int jj = j0 + u;
            if (jj >= nr) break;
#pragma unroll
            for (int q = 0; q < SKC; ++q)
              if (s0 + q < k) {
                const S t = Ts[jj * k + s0 + q];
                vy[u] = s_sub(vy[u], s_mulc(xy[q], t));
                vz[u] = s_sub(vz[u], s_mulc(xz[q], t));
              }
            XY[(i64)i * ldr + b.self_pos + redloc[jj]] = vy[u];
            XZ[(i64)i * ldr + b.self_pos + redloc[jj]] = vz[u];
          }
        }
      }
    }
  }
  __syncthreads();   // Ts (the X_rr space) is dead from here on
  // 3. gather X_rr (shared + factor), X_rc (nr x nc), X_cr (nc x nr)
  S* Xrr = fpool + b.f_Xrr;
  for (int idx = tid; idx < nr * nr; idx += 256) {
    const int i = idx / nr, j = idx % nr;
    Xs[i * ldx + j] = XY[(i64)i * ldr + b.self_pos + redloc[j]];
  }
  if (sym) {
    // symmetric shortcuts: sym = 1 (A = A^*, Z = Y): X_rr := (X_rr + X_rr^*) / 2, so
    // G_L = G_U^* and the Z-side update equals the Y-side one (Z stays equal to Y);
    // sym = 2 (complex symmetric A = A^T, Z = conj(Y)): X_rr := (X_rr + X_rr^T) / 2, so
    // G_L = G_U^T and the Z-side update is the conjugate of the Y-side one
    __syncthreads();
    for (int idx = tid; idx < nr * nr; idx += 256) {
      const int i = idx / nr, j = idx % nr;
      if (i < j) {
        const S xji = sym == 2 ? Xs[j * ldx + i] : s_conj(Xs[j * ldx + i]);
        const S v = s_scale(s_add(Xs[i * ldx + j], xji), 0.5);
        Xs[i * ldx + j] = v;
        Xs[j * ldx + i] = sym == 2 ? v : s_conj(v);
      }
    }
    if (sym == 1 && C)
      for (int i = tid; i < nr; i += 256) Xs[i * ldx + i] = s_scale(s_add(Xs[i * ldx + i], s_conj(Xs[i * ldx + i])), 0.5);
  }
  __syncthreads();
  for (int idx = tid; idx < nr * nr; idx += 256) {
    const int i = idx / nr, j = idx % nr;
    Xrr[(i64)i * ldn + j] = Xs[i * ldx + j];
  }
  S* Xrc = ws + b.off_xrc;
  S* Xcr = ws + b.off_xcr;
  // gathers 4 elements per thread per round (loads first, then stores: one round trip per 4)
  for (int idx0 = tid; idx0 < nr * nc; idx0 += 4 * 256) {
    S v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = idx0 + u * 256;
      v[u] = idx < nr * nc ? XY[(i64)(idx / nc) * ldr + cpos[idx % nc]] : zero;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = idx0 + u * 256;
      if (idx < nr * nc) Xrc[(i64)(idx / nc) * ldr + idx % nc] = v[u];
    }
  }
  for (int idx0 = tid; idx0 < nr * nc; idx0 += 4 * 256) {
    S v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = idx0 + u * 256;
      // X_cr = (X_Z)^*; complex-symmetric shortcut: X_Z = conj(X_Y) (held as X_Y), X_cr = X_Y^T
      v[u] = idx < nr * nc ? XZ[(i64)(idx % nr) * ldr + cpos[idx / nr]] : zero;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = idx0 + u * 256;
      if (idx < nr * nc) Xcr[(i64)(idx / nr) * ldn + idx % nr] = sym == 2 ? v[u] : s_conj(v[u]);
    }
  }
  __syncthreads();
  if (tri) {
    // triangular form (Remark PAPER.md:577-611): X_rr (symmetrised above) = C C^T
    // by a right-looking Cholesky in shared memory; C -> f_Xrr (apply), C^-1 -> f_Xinv (solve,
    // and M_U = C^-1 X_rc by the G-stage GEMM).  Real symmetric shortcut only.
    for (int c = 0; c < nr; ++c) {
      const S d = Xs[c * ldx + c];
      if (!(s_real(d) > 0.0)) {            // not positive definite
        if (tid == 0) singular = 1;
        break;
      }
      const double dc = sqrt(s_real(d));
      __syncthreads();
      for (int i = c + 1 + tid; i < nr; i += 256) Xs[i * ldx + c] = s_scale(Xs[i * ldx + c], 1.0 / dc);
      if (tid == 0) Xs[c * ldx + c] = s_scale(s_one(S()), dc);
      __syncthreads();
      const int nt = nr - c - 1;
      for (int idx = tid; idx < nt * nt; idx += 256) {
        const int i = c + 1 + idx / nt, j = c + 1 + idx % nt;
        if (j <= i) Xs[i * ldx + j] = s_sub(Xs[i * ldx + j], s_mul(Xs[i * ldx + c], s_conj(Xs[j * ldx + c])));
      }
      __syncthreads();
    }
    __syncthreads();
    if (singular) {
      if (tid == 0) b.status = ST_SINGULAR_XRR;
      return;
    }
    // C^-1 (lower) column by column: C z = e_j (a thread per column, written to the pool)
    S* Cf = fpool + b.f_Xrr;
    S* Ci = fpool + b.f_Xinv;
    for (int j = tid; j < nr; j += 256) {
      for (int i = 0; i < nr; ++i) {
        S v = (i == j) ? s_one(S()) : zero;
        for (int q = j; q < i; ++q) v = s_sub(v, s_mul(Xs[i * ldx + q], Ci[(i64)q * ldn + j]));
        Ci[(i64)i * ldn + j] = (i < j) ? zero : s_div(v, Xs[i * ldx + i]);
      }
    }
    for (int idx = tid; idx < nr * nr; idx += 256) {
      const int i = idx / nr, j = idx % nr;
      Cf[(i64)i * ldn + j] = j <= i ? Xs[i * ldx + j] : zero;
    }
    return;
  }
  if (nr <= 64) {
    // 4-5. X_rr^-1 by register Gauss-Jordan (the LU factors themselves are not stored)
    __shared__ S gj_col[2 * 64];
    __shared__ S gj_row[2 * 128];
    __shared__ int gj_prow[64];
    if (!gj_inverse_reg<S>(Xs, ldx, nr, fpool + b.f_Xinv, ldn, gj_col, gj_row, gj_prow)) {
      if (threadIdx.x == 0) b.status = ST_SINGULAR_XRR;
    }
    return;
  }
  // 4. LU with partial pivoting
  for (int c = 0; c < nr; ++c) {
    if (warp == 0) {
      double bv = -1.0;
      int bi = nr;
      for (int i = c + lane; i < nr; i += 32) {
        const double v = s_abs(Xs[i * ldx + c]);
        if (v > bv || (v == bv && i < bi)) {
          bv = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        pv = bv;
        pi = bi;
        ipiv[c] = bi;
        if (!(bv > 0.0)) singular = 1;
      }
    }
    __syncthreads();
    if (singular) break;
    if (pi != c) {
      for (int j = tid; j < nr; j += 256) {
        const S t = Xs[c * ldx + j];
        Xs[c * ldx + j] = Xs[pi * ldx + j];
        Xs[pi * ldx + j] = t;
      }
      __syncthreads();
    }
    const S piv = Xs[c * ldx + c];
    for (int i = c + 1 + tid; i < nr; i += 256) Xs[i * ldx + c] = s_div(Xs[i * ldx + c], piv);
    __syncthreads();
    const int nt = nr - c - 1;
    for (int idx = tid; idx < nt * nt; idx += 256) {
      const int i = c + 1 + idx / nt, j = c + 1 + idx % nt;
      Xs[i * ldx + j] = s_sub(Xs[i * ldx + j], s_mul(Xs[i * ldx + c], Xs[c * ldx + j]));
    }
    __syncthreads();
  }
  if (singular) {
    if (tid == 0) b.status = ST_SINGULAR_XRR;
    return;
  }
  // 5. X_rr^-1 = U^-1 L^-1 P, column by column (a thread per column, in the factor pool)
  S* Is = fpool + b.f_Xinv;
  for (int j = tid; j < nr; j += 256) {
    for (int i = 0; i < nr; ++i) Is[(i64)i * ldn + j] = (i == j) ? s_one(S()) : zero;
    for (int c = 0; c < nr; ++c) {
      const int q = ipiv[c];
      if (q != c) {
        const S t = Is[(i64)c * ldn + j];
        Is[(i64)c * ldn + j] = Is[(i64)q * ldn + j];
        Is[(i64)q * ldn + j] = t;
      }
    }
    for (int i = 0; i < nr; ++i) {
      S s = Is[(i64)i * ldn + j];
      for (int q = 0; q < i; ++q) s = s_sub(s, s_mul(Xs[i * ldx + q], Is[(i64)q * ldn + j]));
      Is[(i64)i * ldn + j] = s;
    }
    for (int i = nr - 1; i >= 0; --i) {
      S s = Is[(i64)i * ldn + j];
      for (int q = i + 1; q < nr; ++q) s = s_sub(s, s_mul(Xs[i * ldx + q], Is[(i64)q * ldn + j]));
      Is[(i64)i * ldn + j] = s_div(s, Xs[i * ldx + i]);
    }
  }
}

// ---------------------------------------------------------------------------
// Pulled L/U update (single GPU).  When a box j comes up, the eliminated
// neighbours n have not pushed Y_c -= G_L Y_r into j's rows (they only updated
// rows that are never eliminated later on the level); j applies all of them at
// once:  Y_j -= [G_L^(n1)[j, :] G_L^(n2)[j, :] ..] [Y_r(n1); Y_r(n2); ..]  and
// Z_j -= [G_U^(n1)[:, j]^* ..] [Z_r(n1); ..]  -- one GEMM with K = sum n_r instead
// of up to 3^d - 1 read-modify-write passes over j's rows.  This kernel gathers
// the operands (A_Y, A_Z: n_b x K into ws at off_pull; the Y_r row list at off_prow).
// j's rows are one contiguous, ascending run in the second group of c(n).
// ---------------------------------------------------------------------------
template <bool C>
__global__ void __launch_bounds__(256) pull_assemble_kernel(BoxDev* __restrict__ boxes,
                                                            const BoxDev* __restrict__ level_boxes,
                                                            int* __restrict__ iws, const int* __restrict__ nbrrec,
                                                            const double* __restrict__ fpoold, double* __restrict__ wsd,
                                                            int zside) {
  typedef typename ScalarOf<C>::T S;
  BoxDev& b = boxes[blockIdx.x];
  const int nb = b.nb;
  const int* nd = nbrrec + b.off_nbr;
  const S* fpool = reinterpret_cast<const S*>(fpoold);
  S* AY = reinterpret_cast<S*>(wsd) + b.off_pull;
  S* AZ = AY + (i64)nb * b.ldr;
  int* prow = iws + b.off_prow;
  // K offsets of the eliminated neighbours (prefix sum in neighbour order), then one warp per
  // neighbour: warp-parallel lower bound of b's first row in c(n) (two probes of 32 lanes instead of
  // a serial binary search) and the copy of the G_L rows / G_U columns that touch b
  __shared__ int kofs[65], nrs[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int nn = b.nnbr;
  if (tid < nn) {
    const int idx = nd[4 * tid];
    int nr = 0;
    if (idx >= 0) {
      const BoxDev& n = level_boxes[idx];
      if (n.nr > 0 && n.status == ST_OK) nr = n.nr;
    }
    nrs[tid] = nr;
  }
  __syncthreads();
  if (tid == 0) {
    int o = 0;
    for (int q = 0; q < nn; ++q) {
      kofs[q] = o;
      o += nrs[q];
    }
    kofs[nn] = o;
    b.kpull = o;
  }
  __syncthreads();
  for (int q = warp; q < nn; q += nw) {
    const int nr = nrs[q];
    if (nr == 0) continue;
    const BoxDev& n = level_boxes[nd[4 * q]];
    const int* crow = iws + n.off_crow;
    // lower bound of row0 in crow[ncp, nc) (sorted): coarse probe on a 32-point grid, then exact
    int lo = n.ncp, hi = n.nc;
    while (hi - lo > 32) {
      const int step = (hi - lo + 31) / 32;
      const int pos = lo + lane * step;
      const bool below = pos < hi && crow[pos] < b.row0;
      const int cnt = __popc(__ballot_sync(0xffffffffu, below));   // probes below row0 (a prefix)
      const int nlo = cnt > 0 ? lo + (cnt - 1) * step + 1 : lo;
      hi = min(hi, lo + cnt * step);
      lo = nlo;
    }
    {
      const int pos = lo + lane;
      const bool below = pos < hi && crow[pos] < b.row0;
      lo += __popc(__ballot_sync(0xffffffffu, below));
    }
    const int o = lo, K0 = kofs[q];
    const S* GL = fpool + n.f_GL;      // nc x nr, ld ldn(n)
    const S* GU = fpool + n.f_GU;      // nr x nc, ld ldr(n)
    for (int idx2 = lane; idx2 < nb * nr; idx2 += 32) {
      const int a = idx2 / nr, i = idx2 % nr;
      AY[(i64)a * b.ldr + K0 + i] = GL[(i64)(o + a) * n.ldn + i];
      if (zside) AZ[(i64)a * b.ldr + K0 + i] = s_conj(GU[(i64)i * n.ldr + o + a]);
    }
    for (int i = lane; i < nr; i += 32) prow[K0 + i] = iws[n.off_redrow + i];
  }
}


// ---------------------------------------------------------------------------
// Near-field row list of every box of a colour batch, built on the device:
// near = active(I_b u I_n) in Morton order of the neighbour boxes
// (R2).  Neighbours processed by an earlier
// colour contribute only their skeleton rows (their redundant rows are
// decoupled); the others contribute all their rows.
// Records {boxdev index or -1, first row, count, box}: a foreign neighbour on the
// multi-GPU path is a contiguous halo block holding exactly its active rows.
// ---------------------------------------------------------------------------
__global__ void build_near_kernel(BoxDev* __restrict__ boxes, const BoxDev* __restrict__ level_boxes,
                                  int* __restrict__ iws, const int* __restrict__ nbrrec, int p, int oversample) {
  BoxDev& b = boxes[blockIdx.x];
  const int lane = threadIdx.x;
  const int* nd = nbrrec + b.off_nbr;
  int* near = iws + b.off_rows;
  for (int t = lane; t < b.nb; t += 32) near[b.rmax + t] = b.row0 + t;   // the box's own rows (cross product)
  int* nflag = iws + b.off_nflag;
  int o = 0, selfp = 0;
  for (int q = 0; q < b.nnbr; ++q) {
    const int idx = nd[4 * q], r0 = nd[4 * q + 1];
    int cnt = nd[4 * q + 2];
    if (idx >= 0) {
      const BoxDev& nbx = level_boxes[idx];
      cnt = nbx.k;
      const int* src = iws + nbx.off_skelrow;
      for (int t = lane; t < cnt; t += 32) {
        near[o + t] = src[t];
        nflag[o + t] = 0;
      }
    } else {
      const bool self = (r0 == b.row0);
      if (self) selfp = o;
      // 1: rows of a not-yet-eliminated neighbour on this rank (pulled later); own rows and
      // halo blocks (-2, -3: foreign, pushed and returned) are 0
      const int fl = (self || idx <= -2) ? 0 : 1;
      for (int t = lane; t < cnt; t += 32) {
        near[o + t] = r0 + t;
        nflag[o + t] = fl;
      }
    }
    o += cnt;
  }
  if (lane == 0) {
    b.r = o;
    b.self_pos = selfp;
    b.status = (p - o < oversample + 1) ? ST_SAMPLES : ST_OK;
    b.k = 0;
    b.nr = 0;
    b.nc = 0;
  }
}

// ---------------------------------------------------------------------------
// Level-to-level merge: gather the skeleton rows of every
// box into the next level's store, parent-major (children in Morton order).
// ---------------------------------------------------------------------------
__global__ void compact_kernel(const BoxDev* __restrict__ boxes, const int* __restrict__ iws,
                               const int* __restrict__ dst_row0, const double* __restrict__ Y,
                               const double* __restrict__ Z, const double* __restrict__ Om,
                               const double* __restrict__ Ps, i64 ld, const int* __restrict__ gidx,
                               double* __restrict__ nY, double* __restrict__ nZ, double* __restrict__ nOm,
                               double* __restrict__ nPs, i64 nld, int* __restrict__ ngidx, int p) {
  const BoxDev& b = boxes[blockIdx.x];
  const int k = b.k;
  const int* skelrow = iws + b.off_skelrow;
  const int base = dst_row0[blockIdx.x];
  if (base < 0) return;                    // skeletons move to another rank (dist.h plan_moves)
  for (int s = blockIdx.y; s < k; s += gridDim.y) {
    const int src = skelrow[s];
    const int dst = base + s;
    if (threadIdx.x == 0) ngidx[dst] = gidx[src];
    const double* y = Y + (i64)src * ld;
    const double* z = Z + (i64)src * ld;
    const double* o = Om + (i64)src * ld;
    const double* q = Ps + (i64)src * ld;
    const bool zs = nZ != nullptr;      // symmetric shortcut: no Z / Psi stores
    for (int j = threadIdx.x; j < p; j += blockDim.x) {
      nY[(i64)dst * nld + j] = y[j];
      nOm[(i64)dst * nld + j] = o[j];
      if (zs) {
        nZ[(i64)dst * nld + j] = z[j];
        nPs[(i64)dst * nld + j] = q[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Top block: LU with partial pivoting of A~_SS (single CTA, in global memory).
// ---------------------------------------------------------------------------
template <bool C>
__global__ void __launch_bounds__(1024) top_lu_kernel(double* __restrict__ Ad, i64 lda, int n,
                                                       int* __restrict__ ipiv, int* __restrict__ status) {
  typedef typename ScalarOf<C>::T S;
  S* A = reinterpret_cast<S*>(Ad);
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int pidx;
  __shared__ double pval;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c = 0; c < n; ++c) {
    double bv = -1.0;
    int bi = n;
    for (int i = c + tid; i < n; i += 1024) {
      const double v = s_abs(A[(i64)i * lda + c]);
      if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      rv[warp] = bv;
      ri[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
      bv = rv[lane];
      bi = ri[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        pval = bv;
        pidx = bi;
        ipiv[c] = bi;
      }
    }
    __syncthreads();
    if (!(pval > 0.0)) {
      if (tid == 0) *status = ST_SINGULAR_XRR;
      return;
    }
    const int q = pidx;
    if (q != c) {
      for (int j = tid; j < n; j += 1024) {
        const S t = A[(i64)c * lda + j];
        A[(i64)c * lda + j] = A[(i64)q * lda + j];
        A[(i64)q * lda + j] = t;
      }
      __syncthreads();
    }
    const S piv = A[(i64)c * lda + c];
    for (int i = c + 1 + tid; i < n; i += 1024) A[(i64)i * lda + c] = s_div(A[(i64)i * lda + c], piv);
    __syncthreads();
    const int nt = n - c - 1;
    for (int idx = tid; idx < nt * nt; idx += 1024) {
      const int i = c + 1 + idx / nt, j = c + 1 + idx % nt;
      A[(i64)i * lda + j] = s_sub(A[(i64)i * lda + j], s_mul(A[(i64)i * lda + c], A[(i64)c * lda + j]));
    }
    __syncthreads();
  }
}

}  // namespace rsrs

// ---------------------------------------------------------------------------
// Multi-GPU data movement (dist.h plans): flat row lists, row gathers into
// message buffers and scatters back.  A message holds `narr` sections of n rows
// x w doubles (Y, Z[, Omega, Psi]) followed, optionally, by the n tree
// positions (as doubles, exact below 2^53).
// ---------------------------------------------------------------------------
namespace rsrs {

// recs[i] = {boxdev index (>= 0: the box's skeleton rows) or -1 (rows row0 ..), row0, count, out offset}
__global__ void rowlist_kernel(const BoxDev* __restrict__ boxes, const int* __restrict__ iws,
                               const int4* __restrict__ recs, int* __restrict__ out) {
  const int4 r = recs[blockIdx.x];
  if (r.x >= 0) {
    const int* src = iws + boxes[r.x].off_skelrow;
    for (int t = threadIdx.x; t < r.z; t += blockDim.x) out[r.w + t] = src[t];
  } else {
    for (int t = threadIdx.x; t < r.z; t += blockDim.x) out[r.w + t] = r.y + t;
  }
}

// out[a][i][:] = A_a[rows[i]][:w] ; out_g[i] = gidx[rows[i]]   (rows == nullptr: row0 + i)
__global__ void gather_rows_kernel(const double* __restrict__ A0, const double* __restrict__ A1,
                                   const double* __restrict__ A2, const double* __restrict__ A3, i64 ldd,
                                   const int* __restrict__ gidx, const int* __restrict__ rows, int row0, int n,
                                   int w, int narr, int with_gidx, double* __restrict__ out) {
  const int i = blockIdx.x, a = blockIdx.y;
  if (i >= n) return;
  const int row = rows ? rows[i] : row0 + i;
  if (a < narr) {
    const double* A = a == 0 ? A0 : a == 1 ? A1 : a == 2 ? A2 : A3;
    const double* src = A + (i64)row * ldd;
    double* dst = out + ((i64)a * n + i) * w;
    for (int j = threadIdx.x; j < w; j += blockDim.x) dst[j] = src[j];
  } else if (with_gidx && threadIdx.x == 0) {
    out[(i64)narr * n * w + i] = (double)gidx[row];
  }
}

// A_a[rows[i]][:w] = in[a][i][:] ; gidx[rows[i]] = in_g[i]
__global__ void scatter_rows_kernel(const double* __restrict__ in, double* __restrict__ A0, double* __restrict__ A1,
                                    double* __restrict__ A2, double* __restrict__ A3, i64 ldd,
                                    int* __restrict__ gidx, const int* __restrict__ rows, int row0, int n, int w,
                                    int narr, int with_gidx) {
  const int i = blockIdx.x, a = blockIdx.y;
  if (i >= n) return;
  const int row = rows ? rows[i] : row0 + i;
  if (a < narr) {
    double* A = a == 0 ? A0 : a == 1 ? A1 : a == 2 ? A2 : A3;
    double* dst = A + (i64)row * ldd;
    const double* src = in + ((i64)a * n + i) * w;
    for (int j = threadIdx.x; j < w; j += blockDim.x) dst[j] = src[j];
  } else if (with_gidx && threadIdx.x == 0) {
    gidx[row] = (int)in[(i64)narr * n * w + i];
  }
}

// solve merge: rows a box touched (lists of tree positions in the factor's index
// pool) -> contrib[pos] = x[pos], mask[pos] = 1.  which: 0 = red and c
// (forward / apply-backward), 1 = red and skel (backward / apply-forward).
__global__ void mark_rows_kernel(const BoxDev* __restrict__ boxes, const int* __restrict__ ipool,
                                 const double* __restrict__ x, i64 ldx, int w, double* __restrict__ contrib,
                                 double* __restrict__ mask, int which) {
  const BoxDev& b = boxes[blockIdx.x];
  if (b.nr <= 0) return;
  const int* l1 = ipool + b.f_red;
  const int n1 = b.nr;
  const int* l2 = ipool + (which == 0 ? b.f_c : b.f_skel);
  const int n2 = which == 0 ? b.nc : b.k;
  for (int t = threadIdx.x; t < (n1 + n2) * w; t += blockDim.x) {
    const int i = t / w, j = t % w;
    const int pos = i < n1 ? l1[i] : l2[i - n1];
    contrib[(i64)pos * w + j] = x[(i64)pos * ldx + j];
    if (j == 0) mask[pos] = 1.0;
  }
}

__global__ void mark_list_kernel(const int* __restrict__ list, int n, const double* __restrict__ x, i64 ldx, int w,
                                 double* __restrict__ contrib, double* __restrict__ mask) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n * w; t += gridDim.x * blockDim.x) {
    const int i = t / w, j = t % w;
    const int pos = list[i];
    contrib[(i64)pos * w + j] = x[(i64)pos * ldx + j];
    if (j == 0) mask[pos] = 1.0;
  }
}

// after the sum over ranks: x[pos] = contrib[pos] where some rank touched pos (exactly one did)
__global__ void merge_finalize_kernel(int64_t N, double* __restrict__ x, i64 ldx, int w, double* __restrict__ contrib,
                                      double* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (mask[i] != 0.0) {
      for (int j = 0; j < w; ++j) {
        x[i * ldx + j] = contrib[i * w + j];
        contrib[i * w + j] = 0.0;
      }
      mask[i] = 0.0;
    }
  }
}

// Compact multi-GPU solve merge (factor.cu Merger): the rows a colour batch touches on this rank, in
// box order (the box's redundant rows, then its c rows (which 0) or skeleton rows (which 1)), the
// same rows mark_rows_kernel marks.  Same-colour near sets are disjoint, so the lists of the ranks
// are disjoint and their concatenation (rank order) is the batch's merge list.
__global__ void merge_count_kernel(const BoxDev* __restrict__ boxes, int nbox, int* __restrict__ cnt) {
  int c0 = 0, c1 = 0;
  for (int i = threadIdx.x; i < nbox; i += blockDim.x) {
    const BoxDev& b = boxes[i];
    if (b.nr <= 0) continue;
    c0 += b.nr + b.nc;
    c1 += b.nr + b.k;
  }
  if (c0) atomicAdd(cnt, c0);
  if (c1) atomicAdd(cnt + 1, c1);
}

// one 1024-thread CTA: out[t] = the t-th touched row (as a double: the lists are summed over ranks)
__global__ void __launch_bounds__(1024) merge_list_kernel(const BoxDev* __restrict__ boxes, int nbox,
                                                          const int* __restrict__ ipool, int which,
                                                          double* __restrict__ out) {
  __shared__ int sc[1024];
  __shared__ int sbase;
  const int tid = threadIdx.x;
  if (tid == 0) sbase = 0;
  __syncthreads();
  for (int c0 = 0; c0 < nbox; c0 += 1024) {
    const int i = c0 + tid;
    int len = 0, n1 = 0;
    const int *l1 = nullptr, *l2 = nullptr;
    if (i < nbox && boxes[i].nr > 0) {
      const BoxDev& b = boxes[i];
      n1 = b.nr;
      l1 = ipool + b.f_red;
      l2 = ipool + (which == 0 ? b.f_c : b.f_skel);
      len = n1 + (which == 0 ? b.nc : b.k);
    }
    sc[tid] = len;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {      // inclusive scan
      const int v = tid >= off ? sc[tid - off] : 0;
      __syncthreads();
      sc[tid] += v;
      __syncthreads();
    }
    const int base = sbase + sc[tid] - len;
    for (int t = 0; t < len; ++t) out[base + t] = (double)(t < n1 ? l1[t] : l2[t - n1]);
    __syncthreads();
    if (tid == 1023) sbase += sc[1023];
    __syncthreads();
  }
}

__global__ void merge_rows_to_int_kernel(const double* __restrict__ in, int* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int)in[i];
}

// buf[t, :] = x[rows[t], :]  (this rank's part of the batch's merge buffer)
__global__ void merge_pack_kernel(const int* __restrict__ rows, int n, const double* __restrict__ x, int w,
                                  double* __restrict__ buf) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * w; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / w, j = t - i * w;
    buf[t] = x[(int64_t)rows[i] * w + j];
  }
}

// x[rows[t], :] = buf[t, :]  (after the sum over ranks: every touched row has exactly one writer)
__global__ void merge_scatter_kernel(const int* __restrict__ rows, int n, const double* __restrict__ buf,
                                     double* __restrict__ x, int w) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)n * w; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / w, j = t - i * w;
    x[(int64_t)rows[i] * w + j] = buf[t];
  }
}

__global__ void add_into_kernel(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

}  // namespace rsrs
