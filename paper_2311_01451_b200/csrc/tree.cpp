// Uniform 2^d-tree planner (host C++): Morton order, box CSR, neighbour and
// colour lists.  PAPER.md:799-820 (section 4.1, "split the root node into 2^d
// children ... until the size of each node is below some given threshold m");
// PAPER.md:182-184 (Fig. 1: neighbours share an edge or corner).
// Readings: DESIGN.md section 3 (R11 depth, R12 neighbours, R10 colours).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>

#include "internal.h"

namespace rsrs {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
void clear_error() { g_err.clear(); }
const char* last_error() { return g_err.c_str(); }

static inline uint64_t interleave(const int32_t* c, int d) {
  uint64_t key = 0;
  for (int b = 0; b < 21; ++b)
    for (int i = 0; i < d; ++i) key |= (uint64_t)((c[i] >> b) & 1) << (b * d + i);
  return key;
}
static inline void deinterleave(uint64_t key, int d, int32_t* c) {
  for (int i = 0; i < d; ++i) c[i] = 0;
  for (int b = 0; b < 21; ++b)
    for (int i = 0; i < d; ++i) c[i] |= (int32_t)((key >> (b * d + i)) & 1) << b;
}

static rsrs_status build(const double* pts, int64_t N, int d, int leaf_max, const double* lo_in,
                         double side_in, int nranks, Tree& T) {
  if (!pts || N < 1 || d < 1 || d > 3 || leaf_max < 1 || nranks < 1) {
    set_error("rsrs_build_tree: invalid argument");
    return RSRS_ERR_INVALID;
  }
  double lo[3] = {0, 0, 0};
  double side = side_in;
  if (lo_in) {
    for (int i = 0; i < d; ++i) lo[i] = lo_in[i];
    if (!(side > 0)) {
      set_error("rsrs_build_tree: root_side must be > 0");
      return RSRS_ERR_INVALID;
    }
  } else {
    double hi[3];
    for (int i = 0; i < d; ++i) lo[i] = hi[i] = pts[i];
    for (int64_t n = 0; n < N; ++n)
      for (int i = 0; i < d; ++i) {
        lo[i] = std::min(lo[i], pts[n * d + i]);
        hi[i] = std::max(hi[i], pts[n * d + i]);
      }
    side = 0;
    for (int i = 0; i < d; ++i) side = std::max(side, hi[i] - lo[i]);
    side = side > 0 ? side * (1 + 1e-12) : 1.0;
  }
  T.d = d;
  T.N = N;
  T.nranks = nranks;
  // depth: smallest L with max leaf occupancy <= leaf_max
  std::vector<int32_t> coords(N * d);
  std::vector<uint64_t> key(N);
  int L = 0;
  for (;; ++L) {
    if (L > 20) {
      set_error("rsrs_build_tree: depth exceeds 20 (coincident points?)");
      return RSRS_ERR_INVALID;
    }
    const double n = (double)(1 << L);
    for (int64_t p = 0; p < N; ++p) {
      for (int i = 0; i < d; ++i) {
        double c = std::floor((pts[p * d + i] - lo[i]) / side * n);
        int32_t ci = (int32_t)std::min(std::max(c, 0.0), n - 1);
        coords[p * d + i] = ci;
      }
      key[p] = interleave(&coords[p * d], d);
    }
    std::vector<uint64_t> sk(key);
    std::sort(sk.begin(), sk.end());
    int64_t occ = 0, run = 0;
    for (int64_t p = 0; p < N; ++p) {
      run = (p > 0 && sk[p] == sk[p - 1]) ? run + 1 : 1;
      occ = std::max(occ, run);
    }
    if (occ <= leaf_max) break;
  }
  T.L = L;
  T.perm.resize(N);
  std::iota(T.perm.begin(), T.perm.end(), 0);
  std::stable_sort(T.perm.begin(), T.perm.end(),
                   [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  std::vector<uint64_t> skey(N);
  for (int64_t p = 0; p < N; ++p) skey[p] = key[T.perm[p]];

  T.levels.assign(L + 1, TreeLevel());
  for (int lev = 0; lev <= L; ++lev) {
    TreeLevel& lv = T.levels[lev];
    const int shift = d * (L - lev);
    lv.start.clear();
    lv.keys.clear();
    for (int64_t p = 0; p < N; ++p) {
      uint64_t k = skey[p] >> shift;
      if (p == 0 || k != (skey[p - 1] >> shift)) {
        lv.start.push_back(p);
        lv.keys.push_back(k);
      }
    }
    lv.start.push_back(N);
    lv.nboxes = (int64_t)lv.keys.size();
    lv.coords.resize(lv.nboxes * d);
    lv.colour.resize(lv.nboxes);
    for (int64_t b = 0; b < lv.nboxes; ++b) {
      deinterleave(lv.keys[b], d, &lv.coords[b * d]);
      int col = 0, pw = 1;
      for (int i = 0; i < d; ++i) {
        col += (lv.coords[b * d + i] % 3) * pw;
        pw *= 3;
      }
      lv.colour[b] = col;
    }
    // neighbours: Chebyshev distance <= 1, nonempty, ascending Morton key
    lv.nbr_off.assign(lv.nboxes + 1, 0);
    lv.nbr.clear();
    const int32_t nside = 1 << lev;
    int noff = 1;
    for (int i = 0; i < d; ++i) noff *= 3;
    for (int64_t b = 0; b < lv.nboxes; ++b) {
      std::vector<int32_t> nb;
      for (int o = 0; o < noff; ++o) {
        int32_t c[3];
        int oo = o;
        bool ok = true;
        for (int i = 0; i < d; ++i) {
          c[i] = lv.coords[b * d + i] + (oo % 3) - 1;
          oo /= 3;
          if (c[i] < 0 || c[i] >= nside) ok = false;
        }
        if (!ok) continue;
        uint64_t k = interleave(c, d);
        auto it = std::lower_bound(lv.keys.begin(), lv.keys.end(), k);
        if (it != lv.keys.end() && *it == k) nb.push_back((int32_t)(it - lv.keys.begin()));
      }
      std::sort(nb.begin(), nb.end());
      lv.nbr.insert(lv.nbr.end(), nb.begin(), nb.end());
      lv.nbr_off[b + 1] = (int32_t)lv.nbr.size();
    }
    lv.parent.assign(lv.nboxes, -1);
    if (lev > 0) {
      const TreeLevel& pl = T.levels[lev - 1];
      for (int64_t b = 0; b < lv.nboxes; ++b) {
        uint64_t pk = lv.keys[b] >> d;
        auto it = std::lower_bound(pl.keys.begin(), pl.keys.end(), pk);
        lv.parent[b] = (int32_t)(it - pl.keys.begin());
      }
    }
  }
  // partners: boxes that meet in some near field (neighbours of a common box)
  for (int lev = 0; lev <= L; ++lev) {
    TreeLevel& lv = T.levels[lev];
    lv.part_off.assign(lv.nboxes + 1, 0);
    lv.part.clear();
    std::vector<int32_t> stamp(lv.nboxes, -1);
    for (int64_t i = 0; i < lv.nboxes; ++i) {
      const size_t at = lv.part.size();
      for (int32_t q = lv.nbr_off[i]; q < lv.nbr_off[i + 1]; ++q) {
        const int32_t m = lv.nbr[q];
        for (int32_t q2 = lv.nbr_off[m]; q2 < lv.nbr_off[m + 1]; ++q2) {
          const int32_t j = lv.nbr[q2];
          if (stamp[j] != (int32_t)i) {
            stamp[j] = (int32_t)i;
            lv.part.push_back(j);
          }
        }
      }
      std::sort(lv.part.begin() + at, lv.part.end());
      lv.part_off[i + 1] = (int32_t)lv.part.size();
    }
  }
  for (int lev = 0; lev <= L; ++lev) {
    TreeLevel& lv = T.levels[lev];
    lv.child_off.assign(lv.nboxes + 1, 0);
    lv.child.clear();
    if (lev < L) {
      const TreeLevel& cl = T.levels[lev + 1];
      for (int64_t c = 0; c < cl.nboxes; ++c) lv.child_off[cl.parent[c] + 1]++;
      for (int64_t b = 0; b < lv.nboxes; ++b) lv.child_off[b + 1] += lv.child_off[b];
      lv.child.resize(cl.nboxes);
      std::vector<int32_t> fill(lv.child_off.begin(), lv.child_off.end() - 1);
      for (int64_t c = 0; c < cl.nboxes; ++c) lv.child[fill[cl.parent[c]]++] = (int32_t)c;
    }
  }
  return RSRS_OK;
}

}  // namespace rsrs

extern "C" {

const char* rsrs_last_error(void) { return rsrs::last_error(); }

const char* rsrs_version(void) { return "rsrs-b200 0.1 (sm_100a)"; }

rsrs_status rsrs_build_tree(const double* pts, int64_t N, int d, int leaf_max,
                            const double* root_lo, double root_side, int nranks,
                            rsrs_tree* out) {
  rsrs::clear_error();
  if (!out) {
    rsrs::set_error("rsrs_build_tree: out is NULL");
    return RSRS_ERR_INVALID;
  }
  *out = nullptr;
  rsrs_tree t = nullptr;
  try {
    t = new rsrs_tree_s();
  } catch (...) {
    rsrs::set_error("rsrs_build_tree: out of host memory");
    return RSRS_ERR_NOMEM;
  }
  rsrs_status st;
  try {
    st = rsrs::build(pts, N, d, leaf_max, root_lo, root_side, nranks, t->t);
  } catch (...) {
    rsrs::set_error("rsrs_build_tree: out of host memory");
    st = RSRS_ERR_NOMEM;
  }
  if (st != RSRS_OK) {
    delete t;
    return st;
  }
  *out = t;
  return RSRS_OK;
}

rsrs_status rsrs_tree_info(rsrs_tree t, int* L, int* d, int64_t* N) {
  if (!t) {
    rsrs::set_error("rsrs_tree_info: null tree");
    return RSRS_ERR_INVALID;
  }
  if (L) *L = t->t.L;
  if (d) *d = t->t.d;
  if (N) *N = t->t.N;
  return RSRS_OK;
}

rsrs_status rsrs_tree_perm(rsrs_tree t, int64_t* perm) {
  if (!t || !perm) {
    rsrs::set_error("rsrs_tree_perm: null argument");
    return RSRS_ERR_INVALID;
  }
  std::memcpy(perm, t->t.perm.data(), sizeof(int64_t) * t->t.N);
  return RSRS_OK;
}

rsrs_status rsrs_tree_level_size(rsrs_tree t, int level, int64_t* nboxes, int64_t* nnbr) {
  if (!t || level < 0 || level > t->t.L) {
    rsrs::set_error("rsrs_tree_level_size: invalid tree or level");
    return RSRS_ERR_INVALID;
  }
  const auto& lv = t->t.levels[level];
  if (nboxes) *nboxes = lv.nboxes;
  if (nnbr) *nnbr = (int64_t)lv.nbr.size();
  return RSRS_OK;
}

rsrs_status rsrs_tree_level(rsrs_tree t, int level, uint64_t* keys, int64_t* start,
                            int32_t* parent, int32_t* colour, int32_t* nbr_off, int32_t* nbr) {
  if (!t || level < 0 || level > t->t.L) {
    rsrs::set_error("rsrs_tree_level: invalid tree or level");
    return RSRS_ERR_INVALID;
  }
  const auto& lv = t->t.levels[level];
  if (keys) std::memcpy(keys, lv.keys.data(), sizeof(uint64_t) * lv.nboxes);
  if (start) std::memcpy(start, lv.start.data(), sizeof(int64_t) * (lv.nboxes + 1));
  if (parent) std::memcpy(parent, lv.parent.data(), sizeof(int32_t) * lv.nboxes);
  if (colour) std::memcpy(colour, lv.colour.data(), sizeof(int32_t) * lv.nboxes);
  if (nbr_off) std::memcpy(nbr_off, lv.nbr_off.data(), sizeof(int32_t) * (lv.nboxes + 1));
  if (nbr) std::memcpy(nbr, lv.nbr.data(), sizeof(int32_t) * lv.nbr.size());
  return RSRS_OK;
}

rsrs_status rsrs_plan_samples(rsrs_tree t, int kmax_guess, int oversample, int64_t* p_min) {
  if (!t || !p_min || kmax_guess < 0 || oversample < 0) {
    rsrs::set_error("rsrs_plan_samples: invalid argument");
    return RSRS_ERR_INVALID;
  }
  const auto& lv = t->t.levels[t->t.L];
  int64_t rmax = 0;
  for (int64_t b = 0; b < lv.nboxes; ++b) {
    int64_t r = 0;
    for (int32_t q = lv.nbr_off[b]; q < lv.nbr_off[b + 1]; ++q)
      r += lv.start[lv.nbr[q] + 1] - lv.start[lv.nbr[q]];
    rmax = std::max(rmax, r);
  }
  int64_t p = rmax + kmax_guess + oversample;
  *p_min = (p + 31) / 32 * 32;
  return RSRS_OK;
}

void rsrs_tree_destroy(rsrs_tree t) { delete t; }

}  // extern "C"
