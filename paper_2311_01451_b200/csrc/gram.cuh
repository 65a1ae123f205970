// Level-wide near-field Gram blocks (single GPU).
//
// Every near field of a level is a concatenation of whole neighbour boxes, and
// the Omega / Psi rows of a box change exactly once during the level: when the
// box is eliminated, its skeleton rows take the E/F update Omega_s += T^* Omega_r
// (the Omega_r rows are dead afterwards, R15).
// So the near-field Gram of box b, C_b = Omega_near Omega_near^*, is a matrix of
// blocks G(i, j) = Omega_i Omega_j^* over pairs of boxes i, j that meet in some
// near field (both neighbours of one nonempty box).  The blocks are computed once
// per level (one batched DMMA GEMM over the box pairs instead of one r x r x p
// GEMM per box), kept current by applying F (rows) / F^* (columns) when a box
// is eliminated, and each C_b is assembled from them by a gather.
#pragma once
#include "common.cuh"

namespace rsrs {

// One partner entry of a box (entries of a box sorted by partner).
struct GBlk {
  int j;       // partner box
  int mode;    // 0: stored block is (this, j) -- rows are this box; 1: stored (j, this) -- columns; 2: (this, this)
  int nrow, ncol;   // shape of the stored block
  i64 off;     // scalar offset of the stored block in the pool (row-major, leading dimension ld)
  int ld, pad;
};

// Descriptors of the level's Gram-block precompute: box i, side (Omega / Psi) computes its row
// block [G(i, j) for partners j >= i] = M_i M_partners^* (one NT GEMM; empty boxes get m = 0).
__global__ void pre_desc_kernel(int nbox, int sides, const int* __restrict__ nb, const int* __restrict__ row0,
                                const i64* __restrict__ roff, const int* __restrict__ rld,
                                const i64* __restrict__ rowl_at, const double* Om, const double* Ps, i64 ld,
                                const int* rowl, double* pool, i64 poff, int p, int SC, NTDesc* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sides * nbox) return;
  const int side = t / nbox, i = t - side * nbox;
  const double* M = side ? Ps : Om;
  NTDesc d{};
  d.A = M + SC * (i64)max(row0[i], 0) * ld; d.rowA = nullptr; d.lda = ld;
  d.B = M; d.rowB = rowl + rowl_at[i]; d.ldb = ld;
  d.C = pool + SC * (side * poff + roff[i]); d.ldc = rld[i];
  d.m = nb[i] > 0 ? nb[i] : 0; d.n = (int)(rowl_at[i + 1] - rowl_at[i]); d.K = p; d.sym_rows = 0; d.alpha = 1.0;
  out[t] = d;
}

// Partner table and B-row lists of the level (one warp per box i; partner lists sorted).
// Entry t of box i points at G(i, j) inside i's row block (j >= i: mode 0, or 2 on the
// diagonal) or at G(j, i) inside j's row block (j < i: mode 1, columns offset by the
// partners of j below i).  rowl[rowl_at[i] + ...] = store rows of i's partners j >= i.
__global__ void __launch_bounds__(256) gblk_tables_kernel(int nbox, const int* __restrict__ gpstart,
                                                          const int* __restrict__ plist, const int* __restrict__ nb,
                                                          const int* __restrict__ row0, const i64* __restrict__ roff,
                                                          const int* __restrict__ rld,
                                                          const i64* __restrict__ rowl_at, GBlk* __restrict__ tab,
                                                          int* __restrict__ rowl) {
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nbox) return;
  int col = 0;
  for (int t = gpstart[i]; t < gpstart[i + 1]; ++t) {
    const int j = plist[t];
    GBlk e;
    e.j = j;
    e.pad = 0;
    if (j >= i) {
      e.mode = j == i ? 2 : 0;
      e.off = roff[i] + col;
      e.ld = rld[i];
      e.nrow = nb[i];
      e.ncol = nb[j];
      int* rl = rowl + rowl_at[i] + col;
      for (int r = lane; r < nb[j]; r += 32) rl[r] = row0[j] + r;
      col += nb[j];
    } else {
      int c = 0;
      for (int u = gpstart[j]; u < gpstart[j + 1]; ++u) {
        const int v = plist[u];
        if (v >= i) break;
        if (v >= j) c += nb[v];
      }
      e.mode = 1;
      e.off = roff[j] + c;
      e.ld = rld[j];
      e.nrow = nb[j];
      e.ncol = nb[i];
    }
    if (lane == 0) tab[t] = e;
  }
}

// Partner table of a level whose row blocks are shared by packs of consecutive boxes (small-box
// levels, factor.cu): box i's rows sit at roff[i] (ld rld[i]) inside its pack's block, and the
// column of partner j is j's offset in the pack's sorted union list (binary search).
RSRS_DI int pack_col(const int* __restrict__ upstart, const int* __restrict__ ulist, const int* __restrict__ ucol,
                     int P, int j) {
  int lo = upstart[P], hi = upstart[P + 1] - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ulist[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  return ucol[lo];   // j is in the list by construction
}
__global__ void __launch_bounds__(256) gblk_tables_packed_kernel(int nbox, const int* __restrict__ gpstart,
                                                                 const int* __restrict__ plist, const int* __restrict__ nb,
                                                                 const i64* __restrict__ roff, const int* __restrict__ rld,
                                                                 const int* __restrict__ pack_of,
                                                                 const int* __restrict__ upstart,
                                                                 const int* __restrict__ ulist,
                                                                 const int* __restrict__ ucol, GBlk* __restrict__ tab) {
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nbox) return;
  for (int t = gpstart[i] + lane; t < gpstart[i + 1]; t += 32) {
    const int j = plist[t];
    GBlk e;
    e.j = j;
    e.pad = 0;
    if (j >= i) {
      e.mode = j == i ? 2 : 0;
      e.off = roff[i] + pack_col(upstart, ulist, ucol, pack_of[i], j);
      e.ld = rld[i];
      e.nrow = nb[i];
      e.ncol = nb[j];
    } else {
      e.mode = 1;
      e.off = roff[j] + pack_col(upstart, ulist, ucol, pack_of[j], i);
      e.ld = rld[j];
      e.nrow = nb[j];
      e.ncol = nb[i];
    }
    tab[t] = e;
  }
}
// B-row lists of the packed precompute GEMMs: pack P's union columns in order
__global__ void __launch_bounds__(256) pack_rowl_kernel(int npack, const int* __restrict__ upstart,
                                                        const int* __restrict__ ulist, const int* __restrict__ ucol,
                                                        const int* __restrict__ nb, const int* __restrict__ row0,
                                                        const i64* __restrict__ prowl_at, int* __restrict__ rowl) {
  const int P = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (P >= npack) return;
  for (int u = upstart[P]; u < upstart[P + 1]; ++u) {
    const int j = ulist[u];
    int* rl = rowl + prowl_at[P] + ucol[u];
    for (int r = lane; r < nb[j]; r += 32) rl[r] = row0[j] + r;
  }
}

// (box, block) work items of the block update: my box q (level order) -> its partner entries.
__global__ void __launch_bounds__(256) gblk_work_kernel(int nq, const BoxDev* __restrict__ level_boxes,
                                                        const int* __restrict__ gpstart,
                                                        const i64* __restrict__ wpre, int2* __restrict__ work) {
  const int q = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  const int i = level_boxes[q].box;
  const int t0 = gpstart[i], cnt = gpstart[i + 1] - t0;
  for (int u = lane; u < cnt; u += 32) work[wpre[q] + u] = make_int2(q, t0 + u);
}

// After the colour batch's E/F updates: for every (eliminated box, block) work item
// (grid x; grid y = side), stage the block (<= 64 x 64) and T in shared memory,
// apply F = [rows s += T^* rows r] to the box's rows and / or F^* to its columns,
// and write the block back.  Boxes of one colour never share a block.
constexpr int GB_MAX = 64;
constexpr int GB_LD = GB_MAX + 1;
template <bool C> constexpr int gblk_smem() { return 2 * GB_MAX * GB_LD * (C ? 16 : 8) + 2 * GB_MAX * 4; }
// shared memory of one launch whose blocks are at most mb x mb (the level's largest box): the sphere's
// leaf blocks are <= 30 x 30, so sizing for 64 x 64 held occupancy at 3 CTAs per SM
template <bool C> inline int gblk_smem_for(int mb) { return 2 * mb * (mb + 1) * (C ? 16 : 8) + 2 * mb * 4; }
template <bool C>
__global__ void __launch_bounds__(256) gblk_update_kernel(const BoxDev* __restrict__ level_boxes,
                                                          const int2* __restrict__ work,
                                                          const GBlk* __restrict__ tab, double* __restrict__ poolO,
                                                          double* __restrict__ poolP, const double* __restrict__ fpoold,
                                                          const int* __restrict__ iws, int mb) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ __align__(16) double gsm[];
  const int GB_LD = mb + 1;                 // blocks and T are at most mb x mb (mb = launch's largest box)
  S* Bs = reinterpret_cast<S*>(gsm);        // block (nrow x ncol), ld GB_LD
  S* Ts = Bs + mb * GB_LD;                  // T (n_r x k), ld GB_LD
  int* skl = reinterpret_cast<int*>(Ts + mb * GB_LD);
  int* red = skl + mb;
  const int2 w = work[blockIdx.x];
  const BoxDev& b = level_boxes[w.x];
  const int k = b.k, nr = b.nr;
  if (b.status != ST_OK || nr <= 0 || k <= 0) return;
  const GBlk e = tab[w.y];
  const int tid = threadIdx.x;
  const S* T = reinterpret_cast<const S*>(fpoold) + b.f_T;
  S* B = reinterpret_cast<S*>(blockIdx.y ? poolP : poolO) + e.off;
  const int nt = blockDim.x, nT = nr * k, nB = e.nrow * e.ncol;
  // staging in rounds of 4 block + 4 T elements per thread, all loads of a round in flight together
  for (int r0 = tid; r0 < max(nT, nB); r0 += 4 * nt) {
    S vb[4], vt[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = r0 + u * nt;
      vb[u] = idx < nB ? B[(i64)(idx / e.ncol) * e.ld + idx % e.ncol] : s_zero(S());
      vt[u] = idx < nT ? T[(i64)(idx / k) * b.ldn + idx % k] : s_zero(S());
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = r0 + u * nt;
      if (idx < nB) Bs[(idx / e.ncol) * GB_LD + idx % e.ncol] = vb[u];
      if (idx < nT) Ts[(idx / k) * GB_LD + idx % k] = vt[u];
    }
  }
  for (int q = tid; q < k; q += nt) skl[q] = iws[b.off_skelrow + q] - b.row0;
  for (int i = tid; i < nr; i += nt) red[i] = iws[b.off_redrow + i] - b.row0;
  __syncthreads();
  if (e.mode != 1) {   // rows: B[s, :] += T^* B[r, :]   (red and skel rows are disjoint)
    for (int idx = tid; idx < k * e.ncol; idx += blockDim.x) {
      const int q = idx / e.ncol, c = idx % e.ncol;
      S acc = Bs[skl[q] * GB_LD + c];
      for (int i = 0; i < nr; ++i) acc = s_add(acc, s_mul(s_conj(Ts[i * GB_LD + q]), Bs[red[i] * GB_LD + c]));
      Bs[skl[q] * GB_LD + c] = acc;
    }
    __syncthreads();
  }
  if (e.mode != 0) {   // columns: B[:, s] += B[:, r] T
    for (int idx = tid; idx < e.nrow * k; idx += blockDim.x) {
      const int r = idx / k, q = idx % k;
      S acc = Bs[r * GB_LD + skl[q]];
      for (int i = 0; i < nr; ++i) acc = s_add(acc, s_mul(Bs[r * GB_LD + red[i]], Ts[i * GB_LD + q]));
      Bs[r * GB_LD + skl[q]] = acc;
    }
    __syncthreads();
  }
  // write back only what changed: the box's rows (mode 0, 2) and columns (mode 1, 2)
  if (e.mode != 1)
    for (int idx = tid; idx < k * e.ncol; idx += blockDim.x) {
      const int q = idx / e.ncol, c = idx % e.ncol;
      B[(i64)skl[q] * e.ld + c] = Bs[skl[q] * GB_LD + c];
    }
  if (e.mode != 0)
    for (int idx = tid; idx < e.nrow * k; idx += blockDim.x) {
      const int r = idx / k, q = idx % k;
      B[(i64)r * e.ld + skl[q]] = Bs[r * GB_LD + skl[q]];
    }
}

// C_b[pos(q1) + a, pos(q2) + c] = G(n_q1, n_q2)[act_q1[a], act_q2[c]] for slots q2 <= q1
// of b's neighbour list (the lower block triangle of the near-field Gram).
// Grid (boxes of the batch, neighbour slots q1).  The slot table, the partner entries
// and the active-row map of the whole row band are staged in shared memory by all
// threads at once; the band is then copied in one flat pass (blocks stored as (this, j)
// and small transposed blocks), with large transposed blocks (mode 1) going through a
// 32 x 32 shared-memory tile so that both sides stay coalesced.
// Dynamic shared memory: gram_assemble_smem(max r of the batch).
inline size_t gram_assemble_smem(int rmax) { return sizeof(int) * 2 * (size_t)(rmax > 0 ? rmax : 1); }
template <bool C>
__global__ void __launch_bounds__(256) gram_assemble_kernel(const BoxDev* __restrict__ boxes,
                                                            const BoxDev* __restrict__ level_boxes,
                                                            const int* __restrict__ iws, const int* __restrict__ nbrrec,
                                                            const GBlk* __restrict__ tab, const int* __restrict__ pstart,
                                                            const double* __restrict__ poolO,
                                                            const double* __restrict__ poolP,
                                                            double* __restrict__ wsd, int sides) {
  typedef typename ScalarOf<C>::T S;
  extern __shared__ int gasm[];
  __shared__ int pos[65], cnt[64], bx[64], idxs[64], ent[64];
  __shared__ GBlk sE[64];
  __shared__ S tile[32][33];
  const BoxDev& b = boxes[blockIdx.x];
  const int q1 = blockIdx.y;
  if (q1 >= b.nnbr || b.status != ST_OK) return;
  const int nn = b.nnbr;
  const int* nd = nbrrec + b.off_nbr;
  const int tid = threadIdx.x;
  if (tid < nn) {
    const int idx = nd[4 * tid];
    cnt[tid] = idx >= 0 ? level_boxes[idx].k : nd[4 * tid + 2];
    bx[tid] = nd[4 * tid + 3];
    idxs[tid] = idx;
    ent[tid] = 0;
  }
  __syncthreads();
  if (cnt[q1] == 0) return;   // uniform
  if (tid == 0) {
    int o = 0;
    for (int q = 0; q < nn; ++q) {
      pos[q] = o;
      o += cnt[q];
    }
    pos[nn] = o;
  }
  // partner entries of slot q1's box for every slot q2 <= q1 (each partner matches at most one slot)
  const int box1 = bx[q1];
  const GBlk* t1 = tab + pstart[box1];
  const int np1 = pstart[box1 + 1] - pstart[box1];
  for (int u = tid; u < np1; u += 256) {
    const int j = t1[u].j;
    for (int q = 0; q <= q1; ++q)
      if (bx[q] == j) ent[q] = u;
  }
  __syncthreads();
  if (tid <= q1) sE[tid] = t1[ent[tid]];
  // active local row of every column of the band, and its slot
  int* act = gasm;
  int* colq = gasm + b.rmax;
  const int p1 = pos[q1], n1 = cnt[q1], ncols = p1 + n1;
  for (int col = tid; col < ncols; col += 256) {
    int lo = 0, hi = q1;   // last slot with pos <= col
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pos[mid] <= col) lo = mid;
      else hi = mid - 1;
    }
    const int a = col - pos[lo], idx = idxs[lo];
    colq[col] = lo;
    act[col] = idx >= 0 ? iws[level_boxes[idx].off_skelrow + a] - level_boxes[idx].row0 : a;
  }
  __syncthreads();
  const int* act1 = act + p1;
  const i64 ldr = b.ldr;
  const bool big1 = n1 >= 16;
  for (int side = 0; side < sides; ++side) {
    const S* P = reinterpret_cast<const S*>(side ? poolP : poolO);
    S* Cb = reinterpret_cast<S*>(wsd) + b.off_aug + (side ? (i64)(b.rmax + b.nb) * ldr : 0);
    // 4 elements per thread per round: the pool loads go out together, then the stores
    for (int idx0 = tid; idx0 < n1 * ncols; idx0 += 4 * 256) {
      S v[4];
      bool w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = idx0 + u * 256;
        w[u] = false;
        v[u] = s_zero(S());
        if (idx >= n1 * ncols) continue;
        const int a = idx / ncols, col = idx - a * ncols;
        const int q2 = colq[col];
        const GBlk& e = sE[q2];
        if (e.mode != 1) {
          v[u] = P[e.off + (i64)act1[a] * e.ld + act[col]];
          w[u] = true;
        } else if (!(big1 && cnt[q2] >= 16)) {   // large transposed blocks: tiled below
          v[u] = s_conj(P[e.off + (i64)act[col] * e.ld + act1[a]]);
          w[u] = true;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = idx0 + u * 256;
        if (!w[u]) continue;
        const int a = idx / ncols, col = idx - a * ncols;
        Cb[(i64)(p1 + a) * ldr + col] = v[u];
      }
    }
    if (!big1) continue;
    // large blocks stored transposed: 32 x 32 tiles through shared memory
    const int tx = tid & 31, ty = tid >> 5;
    for (int q2 = 0; q2 < q1; ++q2) {
      const GBlk e = sE[q2];
      const int n2 = cnt[q2];
      if (e.mode != 1 || n2 < 16) continue;
      const S* B = P + e.off;
      const int* act2 = act + pos[q2];
      for (int a0 = 0; a0 < n1; a0 += 32)
        for (int c0 = 0; c0 < n2; c0 += 32) {
          for (int cc = ty; cc < 32; cc += 8)
            if (c0 + cc < n2 && a0 + tx < n1) tile[cc][tx] = B[(i64)act2[c0 + cc] * e.ld + act1[a0 + tx]];
          __syncthreads();
          for (int aa = ty; aa < 32; aa += 8)
            if (a0 + aa < n1 && c0 + tx < n2) Cb[(i64)(p1 + a0 + aa) * ldr + pos[q2] + c0 + tx] = s_conj(tile[tx][aa]);
          __syncthreads();
        }
    }
  }
}

}  // namespace rsrs
