// comm.cuh — the multi-GPU exchange of the sharded MWU iteration.
//
// One process per GPU; the edges (variables of bmatch / densest) are split into contiguous
// ranges of the L2-blocked internal order, the vertex rows (packing side) are replicated.  Per
// MWU iteration the only vector exchange is ONE sum-allreduce of the scattered forward product
// d^(y) (the box-level analog of the paper's reductions for M x); every partial
// phase reduction (column, search pass, init) exchanges its few reduced slots with an allgather
// and every rank combines them in rank order, so all ranks take identical control decisions.
//
//  * NcclComm: NCCL over NVLink / NVSwitch, loaded with dlopen (libnccl.so.2 of the PyTorch
//    wheel, or $MWU_NCCL_LIB) so that a single-GPU run has no NCCL dependency.
//    NCCL collectives are stream-ordered device work, so the sharded probe loop is captured
//    into the same CUDA graph as the one-GPU loop (conditional WHILE nodes).
//  * SimComm: an in-process group of `world` contexts on ONE device (one host thread per rank,
//    host-side barriers, device copies / sums issued by rank 0 in rank order).  No kernel ever
//    waits on another; it exists so that the sharded engine is testable on a one-GPU box.  Its
//    barriers are host work, so SimComm runs are host-driven (not captured).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdlib.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace mwu {

struct Comm {
  int world = 1, rank = 0;
  virtual ~Comm() {}
  // in-place sum over ranks of buf[0..n) (fp64); result identical on every rank
  virtual void allreduce_sum(double* buf, int64_t n, cudaStream_t st) = 0;
  // out[r * n + i] = in_r[i] for every rank r
  virtual void allgather(const double* in, double* out, int64_t n, cudaStream_t st) = 0;
  // collectives may be captured into a CUDA graph (enqueued on the stream, no host work)
  virtual bool capturable() const { return false; }
};

// ---------------------------------------------------------------------------------- NCCL
// Minimal NCCL ABI (stable since NCCL 2.x): opaque communicator, 128-byte unique id.
typedef struct ncclComm* ncclComm_t_;
struct NcclUid { char internal[128]; };
typedef int (*fn_getUniqueId)(NcclUid*);
typedef int (*fn_commInitRank)(ncclComm_t_*, int, NcclUid, int);
typedef int (*fn_allReduce)(const void*, void*, size_t, int, int, ncclComm_t_, cudaStream_t);
typedef int (*fn_allGather)(const void*, void*, size_t, int, ncclComm_t_, cudaStream_t);
typedef int (*fn_commDestroy)(ncclComm_t_);
typedef int (*fn_commAbort)(ncclComm_t_);
typedef const char* (*fn_getErrorString)(int);
enum { NCCL_FLOAT64_ = 8, NCCL_SUM_ = 0 };

struct NcclLib {
  void* h = nullptr;
  fn_getUniqueId getUniqueId = nullptr;
  fn_commInitRank commInitRank = nullptr;
  fn_allReduce allReduce = nullptr;
  fn_allGather allGather = nullptr;
  fn_commDestroy commDestroy = nullptr;
  fn_commAbort commAbort = nullptr;
  fn_getErrorString errStr = nullptr;
  static NcclLib& get() {
    static NcclLib L;
    if (!L.h) {
      const char* env = getenv("MWU_NCCL_LIB");
      const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
      for (const char* n : names)
        if (n && (L.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
      if (!L.h) throw std::runtime_error("NCCL library not found (set MWU_NCCL_LIB)");
      L.getUniqueId = (fn_getUniqueId)dlsym(L.h, "ncclGetUniqueId");
      L.commInitRank = (fn_commInitRank)dlsym(L.h, "ncclCommInitRank");
      L.allReduce = (fn_allReduce)dlsym(L.h, "ncclAllReduce");
      L.allGather = (fn_allGather)dlsym(L.h, "ncclAllGather");
      L.commDestroy = (fn_commDestroy)dlsym(L.h, "ncclCommDestroy");
      L.commAbort = (fn_commAbort)dlsym(L.h, "ncclCommAbort");
      L.errStr = (fn_getErrorString)dlsym(L.h, "ncclGetErrorString");
      if (!L.getUniqueId || !L.commInitRank || !L.allReduce || !L.allGather || !L.commDestroy)
        throw std::runtime_error("NCCL library lacks required symbols");
    }
    return L;
  }
  void check(int r, const char* what) {
    if (r != 0) throw std::runtime_error(std::string(what) + ": " + (errStr ? errStr(r) : "NCCL error"));
  }
};

struct NcclComm : Comm {
  ncclComm_t_ c = nullptr;
  NcclComm(int w, int r, const void* uid) {
    world = w; rank = r;
    NcclLib& L = NcclLib::get();
    NcclUid id;
    memcpy(id.internal, uid, 128);
    L.check(L.commInitRank(&c, w, id, r), "ncclCommInitRank");
  }
  ~NcclComm() override { if (c) NcclLib::get().commDestroy(c); }
  bool capturable() const override { return true; }
  // a failed collective aborts the communicator (pending operations on every rank return
  // instead of hanging) before the error reaches the caller as MWU_ERR_NCCL
  void checked(int r, const char* what) {
    NcclLib& L = NcclLib::get();
    if (r != 0) {
      if (L.commAbort && c) { L.commAbort(c); c = nullptr; }
      L.check(r, what);
    }
  }
  void allreduce_sum(double* buf, int64_t n, cudaStream_t st) override {
    if (!c) throw std::runtime_error("NCCL communicator aborted by an earlier error");
    NcclLib& L = NcclLib::get();
    checked(L.allReduce(buf, buf, (size_t)n, NCCL_FLOAT64_, NCCL_SUM_, c, st), "ncclAllReduce");
  }
  void allgather(const double* in, double* out, int64_t n, cudaStream_t st) override {
    if (!c) throw std::runtime_error("NCCL communicator aborted by an earlier error");
    NcclLib& L = NcclLib::get();
    checked(L.allGather(in, out, (size_t)n, NCCL_FLOAT64_, c, st), "ncclAllGather");
  }
};

// ---------------------------------------------------------------------------------- SimComm
__global__ void k_add_into(double* a, const double* b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = a[i] + b[i];
}

struct SimGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<const double*> in;
  std::vector<double*> out;
  std::vector<cudaStream_t> st;
  explicit SimGroup(int w) : world(w), in(w), out(w), st(w) {}
  // a rank that failed (and will never arrive) turns the others' wait into an error after
  // 120 s instead of a hang
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const int64_t g = gen;
    if (++arrived == world) { arrived = 0; ++gen; cv.notify_all(); }
    else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; }))
      throw std::runtime_error("SimGroup barrier timeout (another rank failed)");
  }
};

struct SimComm : Comm {
  SimGroup* g;
  SimComm(SimGroup* grp, int r) : g(grp) { world = grp->world; rank = r; }
  void allreduce_sum(double* buf, int64_t n, cudaStream_t st) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("sim allreduce: stream");
    g->out[rank] = buf;
    g->st[rank] = st;
    g->barrier();
    if (rank == 0 && n > 0) {   // fixed order: ((b0 + b1) + b2) + ...
      for (int r = 1; r < world; ++r) k_add_into<<<592, 256, 0, st>>>(g->out[0], g->out[r], n);
      for (int r = 1; r < world; ++r)
        cudaMemcpyAsync(g->out[r], g->out[0], n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("sim allreduce: sum");
    }
    g->barrier();
  }
  void allgather(const double* in, double* out, int64_t n, cudaStream_t st) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("sim allgather: stream");
    g->in[rank] = in;
    g->out[rank] = out;
    g->barrier();
    if (rank == 0 && n > 0) {
      for (int d = 0; d < world; ++d)
        for (int r = 0; r < world; ++r)
          cudaMemcpyAsync(g->out[d] + (int64_t)r * n, g->in[r], n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("sim allgather: copy");
    }
    g->barrier();
  }
};

}  // namespace mwu
