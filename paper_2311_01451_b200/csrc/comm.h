// Transports of the multi-GPU sweep (host C++).
//
//   NcclComm    one process per GPU; grouped ncclSend/ncclRecv for the halo and
//               row-move exchanges, ncclAllReduce for the per-colour rank
//               vector and the solve merges.  NCCL is loaded with dlopen (the
//               library has no link-time NCCL dependency; in a PyTorch process
//               this resolves to the libnccl.so.2 torch already loaded).
//   InProcComm  G ranks as G host threads of one process on one GPU (the
//               single-GPU emulation of the partitioned sweep): exchanges are
//               device-to-device copies between the ranks' buffers, fenced by
//               host barriers.  No kernel ever waits on another kernel.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace rsrs {

struct CommError {
  std::string msg;
};

struct Msg {
  int peer;
  void* buf;        // device
  size_t bytes;
};

class Comm {
 public:
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  // grouped point-to-point exchange on stream s; returns after completion
  virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) = 0;
  // elementwise max over ranks of a HOST int array (in place)
  virtual void allreduce_max_i32(int* host, size_t n, cudaStream_t s) = 0;
  // elementwise sum over ranks of a DEVICE double array (in place); every rank
  // receives identical values
  virtual void allreduce_sum_f64(double* dev, size_t n, cudaStream_t s) = 0;
};

// ---------------------------------------------------------------------------
// NCCL (dlopen)
// ---------------------------------------------------------------------------
// NCCL enum values (nccl.h): ncclUint8 = 1, ncclInt32 = 2, ncclFloat64 = 8; ncclSum = 0, ncclMax = 2
constexpr int NCCL_UINT8 = 1, NCCL_INT32 = 2, NCCL_FLOAT64 = 8, NCCL_SUM = 0, NCCL_MAX = 2;
struct NcclUid {   // ncclUniqueId
  char internal[128];
};

struct NcclApi {
  typedef int (*GroupFn)();
  typedef int (*SendFn)(const void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*RecvFn)(void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*AllReduceFn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*UidFn)(void*);
  typedef int (*InitFn)(void**, int, NcclUid, int);   // ncclCommInitRank(comm*, nranks, id, rank)
  typedef const char* (*ErrFn)(int);
  typedef int (*DestroyFn)(void*);
  void* h = nullptr;
  GroupFn groupStart = nullptr, groupEnd = nullptr;
  SendFn send = nullptr;
  RecvFn recv = nullptr;
  AllReduceFn allReduce = nullptr;
  UidFn getUniqueId = nullptr;
  InitFn commInitRank = nullptr;
  ErrFn errStr = nullptr;
  DestroyFn commDestroy = nullptr;
  static NcclApi& get() {
    static NcclApi a;
    static bool tried = false;
    if (!tried) {
      tried = true;
      a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (a.h) {
        a.groupStart = (GroupFn)dlsym(a.h, "ncclGroupStart");
        a.groupEnd = (GroupFn)dlsym(a.h, "ncclGroupEnd");
        a.send = (SendFn)dlsym(a.h, "ncclSend");
        a.recv = (RecvFn)dlsym(a.h, "ncclRecv");
        a.allReduce = (AllReduceFn)dlsym(a.h, "ncclAllReduce");
        a.getUniqueId = (UidFn)dlsym(a.h, "ncclGetUniqueId");
        a.commInitRank = (InitFn)dlsym(a.h, "ncclCommInitRank");
        a.errStr = (ErrFn)dlsym(a.h, "ncclGetErrorString");
        a.commDestroy = (DestroyFn)dlsym(a.h, "ncclCommDestroy");
      }
    }
    return a;
  }
  bool ok() const { return h && groupStart && groupEnd && send && recv && allReduce && getUniqueId && commInitRank; }
};

class NcclComm : public Comm {
 public:
  NcclComm(void* comm, int rank_, int nranks_) : comm_(comm) {
    rank = rank_;
    nranks = nranks_;
  }
  ~NcclComm() override {
    if (stage_) cudaFree(stage_);
  }
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
    NcclApi& A = NcclApi::get();
    chk(A.groupStart(), "ncclGroupStart");
    for (const Msg& m : sends)
      if (m.bytes) chk(A.send(m.buf, m.bytes, NCCL_UINT8, m.peer, comm_, s), "ncclSend");
    for (const Msg& m : recvs)
      if (m.bytes) chk(A.recv(m.buf, m.bytes, NCCL_UINT8, m.peer, comm_, s), "ncclRecv");
    chk(A.groupEnd(), "ncclGroupEnd");
    // stream-ordered: the scatter kernels that consume the received rows follow on `s`
    // (no host round trip; errors surface at the next synchronising call)
  }
  void allreduce_max_i32(int* host, size_t n, cudaStream_t s) override {
    if (!n) return;
    ensure(n * sizeof(int));
    cudaMemcpyAsync(stage_, host, n * sizeof(int), cudaMemcpyHostToDevice, s);
    chk(NcclApi::get().allReduce(stage_, stage_, n, NCCL_INT32, NCCL_MAX, comm_, s), "ncclAllReduce");
    cudaMemcpyAsync(host, stage_, n * sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) throw CommError{"allreduce: stream synchronize failed"};
  }
  void allreduce_sum_f64(double* dev, size_t n, cudaStream_t s) override {
    if (!n) return;
    chk(NcclApi::get().allReduce(dev, dev, n, NCCL_FLOAT64, NCCL_SUM, comm_, s), "ncclAllReduce");
  }

 private:
  void chk(int r, const char* what) {
    if (r != 0) {
      NcclApi& A = NcclApi::get();
      throw CommError{std::string(what) + ": " + (A.errStr ? A.errStr(r) : std::to_string(r))};
    }
  }
  void ensure(size_t b) {
    if (b > stage_bytes_) {
      if (stage_) cudaFree(stage_);
      cudaMalloc(&stage_, b);
      stage_bytes_ = b;
    }
  }
  void* comm_;
  void* stage_ = nullptr;
  size_t stage_bytes_ = 0;
};

// ---------------------------------------------------------------------------
// In-process emulation: G host threads on one GPU
// ---------------------------------------------------------------------------
class InProcHub {
 public:
  explicit InProcHub(int G) : G_(G), sends_(G * G), ibuf_(G), dbuf_(G) {}
  int size() const { return G_; }
  // cyclic barrier; throws if some rank aborted
  void barrier() {
    std::unique_lock<std::mutex> lk(mu_);
    if (aborted_) throw CommError{"another emulated rank failed"};
    const long gen = gen_;
    if (++arrived_ == G_) {
      arrived_ = 0;
      ++gen_;
      cv_.notify_all();
      return;
    }
    cv_.wait(lk, [&] { return gen_ != gen || aborted_; });
    if (aborted_) throw CommError{"another emulated rank failed"};
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu_);
    aborted_ = true;
    cv_.notify_all();
  }
  std::vector<Msg>& send_slot(int src, int dst) { return sends_[src * G_ + dst]; }
  std::vector<int>& ibuf(int r) { return ibuf_[r]; }
  double*& dbuf(int r) { return dbuf_[r]; }

 private:
  int G_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  long gen_ = 0;
  bool aborted_ = false;
  std::vector<std::vector<Msg>> sends_;
  std::vector<std::vector<int>> ibuf_;
  std::vector<double*> dbuf_;
};

class InProcComm : public Comm {
 public:
  InProcComm(InProcHub* hub, int rank_) : hub_(hub) {
    rank = rank_;
    nranks = hub->size();
  }
  ~InProcComm() override {
    if (tmp_) cudaFree(tmp_);
  }
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
    for (int q = 0; q < nranks; ++q) hub_->send_slot(rank, q).clear();
    for (const Msg& m : sends) hub_->send_slot(rank, m.peer).push_back(m);
    cudaStreamSynchronize(s);   // send buffers complete before peers read them
    hub_->barrier();
    std::vector<size_t> used(nranks, 0);
    for (const Msg& m : recvs) {
      // the k-th message from a peer matches the k-th message it posted to me
      std::vector<Msg>& v = hub_->send_slot(m.peer, rank);
      size_t& u = used[m.peer];
      if (u >= v.size() || v[u].bytes != m.bytes)
        throw CommError{"emulated exchange: size mismatch from rank " + std::to_string(m.peer)};
      if (m.bytes) cudaMemcpyAsync(m.buf, v[u].buf, m.bytes, cudaMemcpyDeviceToDevice, s);
      ++u;
    }
    cudaStreamSynchronize(s);
    hub_->barrier();            // peers finished reading my send buffers
  }
  void allreduce_max_i32(int* host, size_t n, cudaStream_t) override {
    hub_->ibuf(rank).assign(host, host + n);
    hub_->barrier();
    for (int q = 0; q < nranks; ++q) {
      const std::vector<int>& v = hub_->ibuf(q);
      if (v.size() != n) throw CommError{"emulated allreduce: size mismatch"};
      for (size_t i = 0; i < n; ++i) host[i] = (q == 0) ? v[i] : std::max(host[i], v[i]);
    }
    hub_->barrier();
  }
  void allreduce_sum_f64(double* dev, size_t n, cudaStream_t s) override;   // factor.cu (needs a kernel)
  InProcHub* hub() { return hub_; }
  double* tmp(size_t n) {
    if (n > tmp_n_) {
      if (tmp_) cudaFree(tmp_);
      cudaMalloc(&tmp_, n * sizeof(double));
      tmp_n_ = n;
    }
    return tmp_;
  }

 private:
  InProcHub* hub_;
  double* tmp_ = nullptr;
  size_t tmp_n_ = 0;
};

}  // namespace rsrs
