// Multi-GPU planning of the RSRS sweep (see dist.h).
#include "dist.h"

#include <algorithm>

namespace rsrs {

Partition make_partition(const Tree& T, int nranks, int gather_level, int top_level) {
  Partition P;
  P.nranks = std::max(1, nranks);
  const TreeLevel& lv = T.levels[T.L];
  // modelled work of a leaf box: (points of the box and its neighbours)^2
  std::vector<double> w(lv.nboxes, 0.0);
  double tot = 0;
  for (int64_t b = 0; b < lv.nboxes; ++b) {
    double r = 0;
    for (int32_t q = lv.nbr_off[b]; q < lv.nbr_off[b + 1]; ++q)
      r += (double)(lv.start[lv.nbr[q] + 1] - lv.start[lv.nbr[q]]);
    w[b] = r * r;
    tot += w[b];
  }
  P.first.assign(P.nranks + 1, T.N);
  P.first[0] = 0;
  double acc = 0;
  int q = 1;
  for (int64_t b = 0; b < lv.nboxes && q < P.nranks; ++b) {
    // cut before box b once the work so far reaches q / nranks of the total
    while (q < P.nranks && acc >= tot * q / P.nranks) P.first[q++] = lv.start[b];
    acc += w[b];
  }
  for (; q < P.nranks; ++q) P.first[q] = T.N;
  if (gather_level < 0) {
    gather_level = 0;
    for (int l = 0; l <= T.L; ++l)
      if (T.levels[l].nboxes <= 16 * (int64_t)P.nranks) gather_level = l;
  }
  P.gather_level = std::max(gather_level, top_level - 1);
  if (P.nranks == 1) P.gather_level = T.L;
  if (P.gather_level >= T.L)              // nothing is distributed: rank 0 holds every row
    for (int r = 1; r <= P.nranks; ++r) P.first[r] = T.N;
  return P;
}

HaloPlan plan_halo(const Tree& T, const Partition& P, int level, int colour, const std::vector<int>& nb,
                   const std::vector<int>& cnt, int rank) {
  HaloPlan H;
  H.recv.assign(P.nranks, {});
  H.send.assign(P.nranks, {});
  if (P.nranks == 1 || level <= P.gather_level) return H;
  const TreeLevel& lv = T.levels[level];
  const int64_t nbox = lv.nboxes;
  // mark[j] = bitmask-free: for each box j, the set of ranks whose colour-c boxes touch j
  // (a box has at most 3^d neighbours, so collect pairs and deduplicate)
  std::vector<std::pair<int, int>> rx, tx;   // (peer, box)
  for (int64_t b = 0; b < nbox; ++b) {
    if (lv.colour[b] != colour || nb[b] <= 0) continue;
    const int ob = P.owner(T, level, b);
    for (int32_t q = lv.nbr_off[b]; q < lv.nbr_off[b + 1]; ++q) {
      const int j = lv.nbr[q];
      if (cnt[j] <= 0) continue;
      const int oj = P.owner(T, level, j);
      if (oj == ob) continue;
      if (ob == rank) rx.push_back({oj, j});
      if (oj == rank) tx.push_back({ob, j});
    }
  }
  auto fill = [&](std::vector<std::pair<int, int>>& v, std::vector<std::vector<BoxCount>>& out, int64_t& rows) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    for (const auto& pj : v) {
      out[pj.first].push_back({pj.second, cnt[pj.second]});
      rows += cnt[pj.second];
    }
  };
  fill(rx, H.recv, H.recv_rows);
  fill(tx, H.send, H.send_rows);
  return H;
}

MovePlan plan_moves(const Tree& T, const Partition& P, int level, const std::vector<int>& k, int rank) {
  MovePlan M;
  M.send.assign(P.nranks, {});
  M.recv.assign(P.nranks, {});
  if (P.nranks == 1 || level < 1) return M;
  const TreeLevel& lv = T.levels[level];
  for (int64_t b = 0; b < lv.nboxes; ++b) {
    if (k[b] <= 0) continue;
    const int src = P.owner(T, level, b);
    const int dst = P.owner(T, level - 1, lv.parent[b]);
    if (src == dst) continue;
    if (src == rank) M.send[dst].push_back({(int)b, k[b]});
    if (dst == rank) M.recv[src].push_back({(int)b, k[b]});
  }
  return M;
}

}  // namespace rsrs

// ---------------------------------------------------------------------------
// C ABI: host-only views of the multi-GPU plan (include/rsrs.h)
// ---------------------------------------------------------------------------
extern "C" {

rsrs_status rsrs_tree_partition(rsrs_tree t, int nranks, int gather_level, int top_level, int64_t* first,
                                int* gather_out) {
  rsrs::clear_error();
  if (!t || nranks < 1 || top_level < 1) {
    rsrs::set_error("rsrs_tree_partition: invalid argument");
    return RSRS_ERR_INVALID;
  }
  const rsrs::Partition P = rsrs::make_partition(t->t, nranks, gather_level, top_level);
  if (first)
    for (int q = 0; q <= nranks; ++q) first[q] = P.first[q];
  if (gather_out) *gather_out = P.gather_level;
  return RSRS_OK;
}

static rsrs_status put_records(const std::vector<std::vector<rsrs::BoxCount>>& send,
                               const std::vector<std::vector<rsrs::BoxCount>>& recv, int32_t* out, int64_t cap,
                               int64_t* len) {
  int64_t n = 0;
  for (int kind = 0; kind < 2; ++kind) {
    const auto& v = kind == 0 ? send : recv;
    for (size_t q = 0; q < v.size(); ++q)
      for (const auto& bc : v[q]) {
        if (out && n + 4 <= 4 * cap) {
          out[n] = kind;
          out[n + 1] = (int32_t)q;
          out[n + 2] = bc.box;
          out[n + 3] = bc.count;
        }
        n += 4;
      }
  }
  if (len) *len = n / 4;
  if (out && n / 4 > cap) {
    rsrs::set_error("plan: capacity too small");
    return RSRS_ERR_INVALID;
  }
  return RSRS_OK;
}

rsrs_status rsrs_dist_halo_plan(rsrs_tree t, int nranks, int gather_level, int top_level, int level, int colour,
                                const int32_t* nb, const int32_t* cnt, int rank, int32_t* out, int64_t cap,
                                int64_t* len) {
  rsrs::clear_error();
  if (!t || !nb || !cnt || level < 0 || level > t->t.L || rank < 0 || rank >= nranks) {
    rsrs::set_error("rsrs_dist_halo_plan: invalid argument");
    return RSRS_ERR_INVALID;
  }
  const rsrs::Partition P = rsrs::make_partition(t->t, nranks, gather_level, top_level);
  const int64_t n = t->t.levels[level].nboxes;
  std::vector<int> vnb(nb, nb + n), vcnt(cnt, cnt + n);
  const rsrs::HaloPlan H = rsrs::plan_halo(t->t, P, level, colour, vnb, vcnt, rank);
  return put_records(H.send, H.recv, out, cap, len);
}

rsrs_status rsrs_dist_move_plan(rsrs_tree t, int nranks, int gather_level, int top_level, int level,
                                const int32_t* k, int rank, int32_t* out, int64_t cap, int64_t* len) {
  rsrs::clear_error();
  if (!t || !k || level < 1 || level > t->t.L || rank < 0 || rank >= nranks) {
    rsrs::set_error("rsrs_dist_move_plan: invalid argument");
    return RSRS_ERR_INVALID;
  }
  const rsrs::Partition P = rsrs::make_partition(t->t, nranks, gather_level, top_level);
  const int64_t n = t->t.levels[level].nboxes;
  std::vector<int> vk(k, k + n);
  const rsrs::MovePlan M = rsrs::plan_moves(t->t, P, level, vk, rank);
  return put_records(M.send, M.recv, out, cap, len);
}

rsrs_status rsrs_dist_owner(rsrs_tree t, int nranks, int gather_level, int top_level, int level, int32_t* owner) {
  rsrs::clear_error();
  if (!t || !owner || level < 0 || level > t->t.L) {
    rsrs::set_error("rsrs_dist_owner: invalid argument");
    return RSRS_ERR_INVALID;
  }
  const rsrs::Partition P = rsrs::make_partition(t->t, nranks, gather_level, top_level);
  for (int64_t b = 0; b < t->t.levels[level].nboxes; ++b) owner[b] = P.owner(t->t, level, b);
  return RSRS_OK;
}

}  // extern "C"
