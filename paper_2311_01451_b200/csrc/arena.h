// Device memory arena of librsrs (host C++).
//
// rsrs_factor needs a few GB of workspace per call (near-field Grams, the
// compacted sample stores of the next level, factor pools sized by upper
// bounds).  Growing the CUDA stream-ordered pool for that on every call costs
// 0.1-3 s of driver time (measured with RSRS_TRACE=1 on B200), so the library
// keeps its own arena: chunks obtained with cudaMalloc once, never returned to
// the driver while the process lives (rsrs_release_memory() returns the idle
// ones), sub-allocated best-fit with coalescing.  Host bookkeeping only: a free
// is immediately reusable, so callers free only memory no queued kernel still
// uses (rsrs_factor synchronises its stream before releasing workspace, and
// rsrs_factor_destroy synchronises the device).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

namespace rsrs {

class Arena {
 public:
  static Arena& get() {
    static Arena a;
    return a;
  }
  // nullptr on failure (cudaMalloc of a new chunk failed)
  void* alloc(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    bytes = round(bytes);
    auto best = free_by_addr_.end();
    for (auto it = free_by_addr_.begin(); it != free_by_addr_.end(); ++it)
      if (it->second >= bytes && (best == free_by_addr_.end() || it->second < best->second)) best = it;
    if (best == free_by_addr_.end()) {
      // new chunk: at least 1 GiB, at least a quarter of what is reserved
      size_t sz = bytes;
      sz = sz < (size_t(1) << 30) ? (size_t(1) << 30) : sz;
      sz = sz < reserved_ / 4 ? round(reserved_ / 4) : sz;
      void* p = nullptr;
      if (cudaMalloc(&p, sz) != cudaSuccess) {
        cudaGetLastError();
        if (sz > bytes && cudaMalloc(&p, bytes) == cudaSuccess) {
          sz = bytes;
        } else {
          cudaGetLastError();
          // fragmented: hand the wholly idle chunks back to the driver and try once more
          release_idle_locked();
          sz = bytes;
          if (cudaMalloc(&p, sz) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
          }
        }
      }
      chunks_.push_back({(char*)p, sz});
      reserved_ += sz;
      best = free_by_addr_.emplace((char*)p, sz).first;
    }
    char* base = best->first;
    const size_t have = best->second;
    free_by_addr_.erase(best);
    if (have > bytes) free_by_addr_.emplace(base + bytes, have - bytes);
    used_.emplace(base, bytes);
    in_use_ += bytes;
    return base;
  }
  void free(void* pv) {
    if (!pv) return;
    std::lock_guard<std::mutex> lk(mu_);
    char* p = (char*)pv;
    auto u = used_.find(p);
    if (u == used_.end()) return;
    size_t sz = u->second;
    used_.erase(u);
    in_use_ -= sz;
    // coalesce with the following and preceding free blocks of the same chunk
    auto nx = free_by_addr_.lower_bound(p);
    if (nx != free_by_addr_.end() && nx->first == p + sz && same_chunk(p, nx->first)) {
      sz += nx->second;
      nx = free_by_addr_.erase(nx);
    }
    if (nx != free_by_addr_.begin()) {
      auto pr = std::prev(nx);
      if (pr->first + pr->second == p && same_chunk(pr->first, p)) {
        pr->second += sz;
        return;
      }
    }
    free_by_addr_.emplace(p, sz);
  }
  // return wholly idle chunks to the driver
  void release_idle() {
    std::lock_guard<std::mutex> lk(mu_);
    release_idle_locked();
  }
  size_t reserved() const { return reserved_; }
  size_t in_use() const { return in_use_; }

 private:
  void release_idle_locked() {
    std::vector<Chunk> keep;
    for (const Chunk& c : chunks_) {
      auto it = free_by_addr_.find(c.base);
      if (it != free_by_addr_.end() && it->second == c.size) {
        free_by_addr_.erase(it);
        cudaFree(c.base);
        reserved_ -= c.size;
      } else {
        keep.push_back(c);
      }
    }
    chunks_ = keep;
  }
  struct Chunk {
    char* base;
    size_t size;
  };
  static size_t round(size_t b) { return (b + 255) & ~size_t(255); }
  bool same_chunk(const char* a, const char* b) const {
    for (const Chunk& c : chunks_)
      if (a >= c.base && a < c.base + c.size) return b >= c.base && b < c.base + c.size;
    return false;
  }
  std::mutex mu_;
  std::vector<Chunk> chunks_;
  std::map<char*, size_t> free_by_addr_;
  std::map<char*, size_t> used_;
  size_t reserved_ = 0, in_use_ = 0;
};

}  // namespace rsrs
