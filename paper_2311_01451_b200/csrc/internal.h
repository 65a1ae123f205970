// Internal host-side structures of librsrs (not part of the C ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rsrs.h"

namespace rsrs {

// thread-local last-error message (rsrs_last_error)
void set_error(const std::string& msg);
void clear_error();

struct TreeLevel {
  int64_t nboxes = 0;
  std::vector<uint64_t> keys;      // Morton keys, ascending
  std::vector<int32_t> coords;     // nboxes * d
  std::vector<int64_t> start;      // nboxes + 1 (tree positions)
  std::vector<int32_t> parent;     // box index on level - 1
  std::vector<int32_t> colour;     // sum_i (c_i mod 3) 3^i
  std::vector<int32_t> nbr_off;    // nboxes + 1
  std::vector<int32_t> nbr;        // neighbour lists (self included, ascending)
  std::vector<int32_t> child_off;  // nboxes + 1 (children on level + 1)
  std::vector<int32_t> child;
  std::vector<int32_t> part_off;   // nboxes + 1: boxes sharing a near field (neighbours of neighbours)
  std::vector<int32_t> part;       // ascending per box (Gram blocks, gram.cuh)
};

struct Tree {
  int d = 0;
  int64_t N = 0;
  int L = 0;
  int nranks = 1;
  std::vector<int64_t> perm;       // tree position -> original index
  std::vector<TreeLevel> levels;   // 0..L
};

}  // namespace rsrs

struct rsrs_tree_s {
  rsrs::Tree t;
};
