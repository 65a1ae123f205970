// Multi-GPU planning of the RSRS sweep (host C++, no CUDA): box ownership by
// Morton range, per-(level, colour) halo exchange lists and the level-to-level
// row moves.  Pure functions of the tree, the partition and the box sizes, so
// every rank derives the same plan independently (checked across processes by
// tests/test_dist_plan.py with torch.distributed/gloo).
//
// Method facts this relies on (section 5, R10/R15):
//  - box b reads the samples of near(b) = active rows of b and its neighbours
//    and writes Y/Z rows of c = near \ red plus its own rows;
//  - boxes of one colour are >= 3 apart, so their near sets are disjoint: a
//    foreign row is read and written by at most one box per colour, and the
//    owner does not touch it meanwhile -> fetch, update, return is exact;
//  - active(j) = all rows of j before j is processed, its skeletons after.
#pragma once
#include <cstdint>
#include <utility>
#include <vector>

#include "internal.h"

namespace rsrs {

struct Partition {
  int nranks = 1;
  int gather_level = 0;              // boxes on levels <= gather_level belong to rank 0
  std::vector<int64_t> first;        // nranks + 1 tree positions: rank q owns leaves in [first[q], first[q+1])
  int owner_pos(int64_t pos) const {
    int lo = 0, hi = nranks;         // largest q with first[q] <= pos
    while (hi - lo > 1) {
      const int m = (lo + hi) / 2;
      if (first[m] <= pos) lo = m;
      else hi = m;
    }
    return lo;
  }
  int owner(const Tree& T, int level, int64_t box) const {
    if (nranks == 1 || level <= gather_level) return 0;
    return owner_pos(T.levels[level].start[box]);
  }
};

// Leaves split into nranks Morton-contiguous ranges of about equal modelled work
// (near-field Gram ~ r_b^2 p, r_b = points of b and its neighbours).
// gather_level < 0: the largest level with at most 16 * nranks boxes (at least
// top_level - 1, so the top block is always on one rank).
Partition make_partition(const Tree& T, int nranks, int gather_level, int top_level);

struct BoxCount {
  int box;
  int count;
  bool operator==(const BoxCount& o) const { return box == o.box && count == o.count; }
};

// Halo lists of one (level, colour) on `rank`:
//   recv[q] = foreign boxes of owner q adjacent to my colour-c boxes (Morton order)
//   send[q] = my boxes adjacent to q's colour-c boxes (Morton order)
// with count = active rows of the box (cnt[j]); boxes with cnt 0 are skipped.
struct HaloPlan {
  std::vector<std::vector<BoxCount>> recv, send;
  int64_t recv_rows = 0, send_rows = 0;
};
HaloPlan plan_halo(const Tree& T, const Partition& P, int level, int colour, const std::vector<int>& nb,
                   const std::vector<int>& cnt, int rank);

// Moves of the skeleton rows of level `level` into the stores of level-1
// (parent order, children in Morton order inside a parent):
//   send[q] = my level-`level` boxes whose skeletons go to rank q != rank (Morton order)
//   recv[q] = boxes of rank q whose skeletons come to me (Morton order)
// k = skeleton count per box of `level` (global).
struct MovePlan {
  std::vector<std::vector<BoxCount>> send, recv;
};
MovePlan plan_moves(const Tree& T, const Partition& P, int level, const std::vector<int>& k, int rank);

}  // namespace rsrs
