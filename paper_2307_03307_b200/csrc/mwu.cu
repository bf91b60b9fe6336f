// mwu.cu — context, structure build, probe engine (host-driven or one CUDA-graph launch per
// probe via conditional WHILE nodes), outer bisection and the C ABI of include/mwu.h.
#include "../../include/mwu.h"
#include "kernels.cuh"
#include "storage.cuh"
#include "comm.cuh"

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: host ranges for nsys / ncu timelines

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

using namespace mwu;

namespace {

thread_local std::string g_create_err;

enum Kind { K_CSR = 0, K_MATCH = 1, K_VCOVER = 2, K_DOMSET = 3, K_DENSEST = 4 };

struct MwuError {
  mwu_status st;
  std::string msg;
};

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      throw MwuError{e_ == cudaErrorMemoryAllocation ? MWU_ERR_OOM : MWU_ERR_CUDA,                 \
                     std::string(#call) + ": " + cudaGetErrorString(e_)};                          \
  } while (0)
#define CKL() CK(cudaGetLastError())

struct Seg {
  int64_t nrows = 0, nnz = 0;
  int64_t* rowptr = nullptr;
  uint32_t* idx = nullptr;
  double* val = nullptr;
  int64_t ntiles = 0;
  int64_t* tile_row = nullptr;
  int64_t nlong = 0, nchunks = 0;
  int64_t* long_rows = nullptr;
  int64_t* long_cptr = nullptr;
  double* chunk_sum = nullptr;
  SegView view() const {
    SegView s;
    s.rowptr = rowptr; s.nrows = nrows; s.idx = idx; s.val = val; s.tile_row = tile_row; s.ntiles = ntiles;
    s.long_rows = long_rows; s.long_cptr = long_cptr; s.nlong = nlong; s.nchunks = nchunks; s.chunk_sum = chunk_sum;
    return s;
  }
};

}  // namespace

struct mwu_ctx {
  mwu_options opt{};
  int dev = 0;
  cudaStream_t st = nullptr;
  std::string err;
  bool poisoned = false;
  int kind = K_CSR, mode = MWU_MIXED;
  int64_t n = 0, nv = 0, E = 0, nleft = 0;
  int64_t mP = 0, mC = 0;
  int pSing = 0, cSing = 0;
  int64_t nnzP = 0, nnzC = 0, empty_dropped = 0;
  bool empty_cover = false;
  // graph storage
  int32_t *src = nullptr, *dst = nullptr, *srow = nullptr, *drow = nullptr, *deg = nullptr, *prow = nullptr;
  Seg inc_all, inc_p;
  int inc_fast = 0;          // fast edge-variable path: incidence rowptrs only (no slot list / plan)
  int64_t maxdeg = 0, nprime = 0;
  // CSR storage
  Seg csrP, cscP, csrC, cscC;
  double *colmaxP = nullptr, *colsumC = nullptr, *crecipC = nullptr, *crecipP = nullptr;
  // fast densest path (lazyC): compacted covering-row records per MWU_CT-edge tile
  int lazyC = 0;
  int scatterP = 0;          // graph kinds with edge variables: d^(y) scattered by the column kernel
  uint32_t* perm = nullptr;  // scatterP: internal (L2-blocked) edge position -> original edge id
  uint32_t* rowperm = nullptr;  // scatterP: fast (degree-ordered) packing row -> vertex-order row
  int compC = 0;             // vcover (fast, one rank): forward product writes compacted covering records
  int fastC = 0;             // vcover / domset: transposed (and domset forward) products scattered
  double* exptab = nullptr;  // 2^(j/256), j < 256 (fastmath.cuh mwu_exp_tab)
  double* emtab = nullptr;   // 2^(j/256), j in [-128, 128), and 2^(j/256) - 1 as hi + lo
  double* hsum = nullptr;    // fastC: C^T v per variable
  int32_t* rowidC = nullptr; // fastC domset: row id of every nonzero of C = I + A
  // multi-GPU (edge-sharded): this rank owns internal edges [e0, e0 + E)
  int world = 1, rank = 0;
  int sharded = 0;                            // a communicator drives the exchange (world >= 1)
  Comm* comm = nullptr;
  int64_t Eg = 0, ng = 0, mCg = 0, e0 = 0;   // global edges / variables / covering rows
  std::vector<int64_t> rb;                    // [world+1] ranges of the sharded dimension
  // owner-partitioned bipartite matching (sharded): right rows [own_rows[r], own_rows[r+1]) and
  // the internal edges [own_rb[r], own_rb[r+1]) belong to rank r; rows [0, nLx) are replicated
  int own = 0;
  int64_t nLx = 0, R0 = 0, R1 = 0;
  std::vector<int64_t> own_rows, own_rb;
  int64_t r0 = 0, k0 = 0, nnzL = 0;           // domset: first local row, first local nonzero, count
  uint32_t* perm_full = nullptr;
  double* gslots = nullptr;                   // [world][MWU_SLOTS] gathered reduction slots
  double* gfull = nullptr;                    // full internal-order vector (hooks)
  double* gsend = nullptr;                    // padded local slice (hooks)
  int64_t ntilesC = 0;
  double *rz = nullptr, *rdz = nullptr, *rv = nullptr;
  int32_t* tcnt = nullptr;   // records per stream (one stream per warp of the compacting kernel)
  int64_t rec_grid = 0, rec_cap = 0;   // compacting kernel's grid; records per warp stream
  uint32_t* act = nullptr;   // activity bits of d (bit e: edge e's pair of directions is nonzero)
  // vectors
  double *x = nullptr, *d = nullptr, *y = nullptr, *dy = nullptr, *u = nullptr, *z = nullptr, *dz = nullptr,
         *v = nullptr, *gtmp = nullptr, *gdbg = nullptr, *hdbg = nullptr, *xbest = nullptr, *tmp = nullptr,
         *tmp2 = nullptr;
  Ctl* ctl = nullptr;
  Ctl* hctl = nullptr;  // pinned host mirror
  double* part = nullptr;
  unsigned int* counter = nullptr;
  int sms = 148, grid_rows = 592, grid_max = 1184;
  std::vector<void*> allocs;
  bool probe_active = false;
  double aguess[32] = {0};   // accepted step sizes of the last probe by iteration (first-window guess)
  double bound = 0, eps = 0;
  int record = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  unsigned long long h_iter = 0, h_search = 0;
  bool graph_ok = false;
  mwu_stats stats{};
  int64_t launches = 0;
  double bytes_alg = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evin = nullptr;   // caller-stream ordering (mwu_options.stream)
  cudaStream_t ust = nullptr;   // the caller's stream (nullptr: legacy default stream)
};

namespace {

// ------------------------------------------------------------------------------ memory
template <class T>
T* dalloc(mwu_ctx* c, int64_t n) {
  if (n <= 0) n = 1;
  n += 4;  // padding: 16-byte bulk copies of a ragged tail stay inside the allocation
  void* p = nullptr;
  CK(cudaMalloc(&p, (size_t)n * sizeof(T)));
  c->allocs.push_back(p);
  return (T*)p;
}
template <class T>
T* talloc(int64_t n) {  // temporary (caller frees with tfree)
  if (n <= 0) n = 1;
  void* p = nullptr;
  CK(cudaMalloc(&p, (size_t)n * sizeof(T)));
  return (T*)p;
}
void tfree(void* p) {
  if (p) cudaFree(p);
}

int grid_for(mwu_ctx* c, int64_t n) {
  int64_t g = (n + MWU_NT - 1) / MWU_NT;
  if (g < 1) g = 1;
  if (g > c->grid_max) g = c->grid_max;
  return (int)g;
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 63 && (int64_t(1) << b) < n) ++b;
  return b;
}

void sync(mwu_ctx* c) { CK(cudaStreamSynchronize(c->st)); }

// Order the library stream after the work the caller queued on its stream (mwu_options.stream):
// called before every read of caller memory; outputs are complete when a call returns.
void wait_caller(mwu_ctx* c) {
  CK(cudaEventRecord(c->evin, c->ust ? c->ust : cudaStreamLegacy));
  CK(cudaStreamWaitEvent(c->st, c->evin, 0));
}

template <class T>
T read_scalar(mwu_ctx* c, const T* dptr) {
  T h;
  CK(cudaMemcpyAsync(&h, dptr, sizeof(T), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  return h;
}

void pull_ctl(mwu_ctx* c) {
  CK(cudaMemcpyAsync(c->hctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->st));
  sync(c);
}

template <class T>
void push_field(mwu_ctx* c, T* dfield, T val) {
  CK(cudaMemcpyAsync(dfield, &val, sizeof(T), cudaMemcpyHostToDevice, c->st));
  sync(c);  // val is a stack value
}

// exclusive scan of n int64 values into out[n+1] (out[n] = total)
void exclusive_scan_total(mwu_ctx* c, const int64_t* in_n, int64_t* out, int64_t n) {
  int64_t* tmp = talloc<int64_t>(n + 1);
  CK(cudaMemsetAsync(tmp + n, 0, sizeof(int64_t), c->st));
  if (n > 0) CK(cudaMemcpyAsync(tmp, in_n, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->st));
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, tmp, out, n + 1, c->st));
  void* t = talloc<char>(tb);
  CK(cub::DeviceScan::ExclusiveSum(t, tb, tmp, out, n + 1, c->st));
  sync(c);
  tfree(t);
  tfree(tmp);
}

// tile plan + long rows of a segmented structure
void build_plan(mwu_ctx* c, Seg& s) {
  s.ntiles = s.nnz / MWU_TILE + 1;
  s.tile_row = dalloc<int64_t>(c, s.ntiles + 1);
  k_tile_rows<<<grid_for(c, s.ntiles + 1), MWU_NT, 0, c->st>>>(s.rowptr, s.nrows, s.ntiles, s.tile_row);
  CKL();
  if (s.nrows == 0) return;
  uint8_t* flags = talloc<uint8_t>(s.nrows);
  k_long_flags<<<grid_for(c, s.nrows), MWU_NT, 0, c->st>>>(s.rowptr, s.nrows, flags);
  CKL();
  int64_t* sel = talloc<int64_t>(s.nrows);
  int64_t* nsel = talloc<int64_t>(1);
  cub::CountingInputIterator<int64_t> it(0);
  size_t tb = 0;
  CK(cub::DeviceSelect::Flagged(nullptr, tb, it, flags, sel, nsel, s.nrows, c->st));
  void* t = talloc<char>(tb);
  CK(cub::DeviceSelect::Flagged(t, tb, it, flags, sel, nsel, s.nrows, c->st));
  s.nlong = read_scalar(c, nsel);
  tfree(t);
  if (s.nlong > 0) {
    s.long_rows = dalloc<int64_t>(c, s.nlong);
    CK(cudaMemcpyAsync(s.long_rows, sel, s.nlong * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->st));
    int64_t* nch = talloc<int64_t>(s.nlong);
    k_long_nchunks<<<grid_for(c, s.nlong), MWU_NT, 0, c->st>>>(s.rowptr, s.long_rows, s.nlong, nch);
    CKL();
    s.long_cptr = dalloc<int64_t>(c, s.nlong + 1);
    exclusive_scan_total(c, nch, s.long_cptr, s.nlong);
    s.nchunks = read_scalar(c, s.long_cptr + s.nlong);
    s.chunk_sum = dalloc<double>(c, s.nchunks);
    tfree(nch);
  }
  sync(c);
  tfree(sel);
  tfree(nsel);
  tfree(flags);
}

// CSC copy of a CSR (rows x cols): stable sort of entries by column keeps rows ascending.
void build_csc(mwu_ctx* c, const Seg& A, int64_t cols, Seg& T) {
  T.nrows = cols;
  T.nnz = A.nnz;
  T.rowptr = dalloc<int64_t>(c, cols + 1);
  T.idx = dalloc<uint32_t>(c, A.nnz);
  T.val = A.val ? dalloc<double>(c, A.nnz) : nullptr;
  if (A.nnz > 0) {
    uint32_t* rid = talloc<uint32_t>(A.nnz);
    k_row_ids<<<grid_for(c, A.nrows), MWU_NT, 0, c->st>>>(A.nrows, A.rowptr, rid);
    CKL();
    uint32_t* kout = talloc<uint32_t>(A.nnz);
    uint64_t* vin = talloc<uint64_t>(A.nnz);
    uint64_t* vout = talloc<uint64_t>(A.nnz);
    k_iota64<<<grid_for(c, A.nnz), MWU_NT, 0, c->st>>>(A.nnz, vin);
    CKL();
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, A.idx, kout, vin, vout, A.nnz, 0, bits_for(cols + 1), c->st));
    void* t = talloc<char>(tb);
    CK(cub::DeviceRadixSort::SortPairs(t, tb, A.idx, kout, vin, vout, A.nnz, 0, bits_for(cols + 1), c->st));
    k_gather_csc<<<grid_for(c, A.nnz), MWU_NT, 0, c->st>>>(A.nnz, vout, rid, A.val, T.idx, T.val);
    CKL();
    int64_t* cnt = talloc<int64_t>(cols);
    CK(cudaMemsetAsync(cnt, 0, cols * sizeof(int64_t), c->st));
    k_col_count<<<grid_for(c, A.nnz), MWU_NT, 0, c->st>>>(A.nnz, A.idx, cnt);
    CKL();
    exclusive_scan_total(c, cnt, T.rowptr, cols);
    sync(c);
    tfree(t); tfree(rid); tfree(kout); tfree(vin); tfree(vout); tfree(cnt);
  } else {
    CK(cudaMemsetAsync(T.rowptr, 0, (cols + 1) * sizeof(int64_t), c->st));
  }
  build_plan(c, T);
}

double rp_bytes(int64_t nnz) { return nnz < (int64_t(1) << 31) ? 4.0 : 8.0; }

void alloc_vectors(mwu_ctx* c) {
  c->x = dalloc<double>(c, c->n);
  c->d = dalloc<double>(c, c->n);
  c->xbest = dalloc<double>(c, c->n);
  c->y = dalloc<double>(c, c->mP);
  c->dy = dalloc<double>(c, c->mP);
  c->u = dalloc<double>(c, c->mP);
  c->z = dalloc<double>(c, c->mC);
  if (c->lazyC || c->compC) {
    c->ntilesC = (c->mC + MWU_CT - 1) / MWU_CT;
    // one dense record stream per warp of the compacting kernel (column kernel / edge_sum_compact)
    c->rec_grid = std::max<int64_t>(1, std::min<int64_t>(c->ntilesC, (c->lazyC ? MWU_COL_MINB : 4) * (int64_t)c->sms));
    c->rec_cap = (c->ntilesC + c->rec_grid - 1) / c->rec_grid * kWarpSeg;
    const int64_t nrec = c->rec_grid * (MWU_NT / 32) * c->rec_cap;
    c->rz = dalloc<double>(c, nrec);
    c->rdz = dalloc<double>(c, nrec);
    c->rv = dalloc<double>(c, nrec);
    c->tcnt = dalloc<int32_t>(c, c->rec_grid * (MWU_NT / 32));
  }
  if (c->kind == K_MATCH && c->scatterP) {   // matching fast path: activity bits of d
    c->act = dalloc<uint32_t>(c, (c->E + 31) / 32 + 1);
    CK(cudaMemsetAsync(c->act, 0, ((c->E + 31) / 32 + 1) * sizeof(uint32_t), c->st));
  }
  if (c->lazyC) {
    c->act = dalloc<uint32_t>(c, c->ntilesC * (MWU_CT / 32));
    CK(cudaMemsetAsync(c->act, 0, c->ntilesC * (MWU_CT / 32) * sizeof(uint32_t), c->st));
  } else {
    c->dz = dalloc<double>(c, c->mC);
    c->v = dalloc<double>(c, c->mC);
  }
  int64_t mx = c->n;
  if (c->mP > mx) mx = c->mP;
  if (c->mC > mx) mx = c->mC;
  c->tmp = dalloc<double>(c, mx);
  if (c->scatterP) c->tmp2 = dalloc<double>(c, std::max(c->ng > 0 ? c->ng : c->n, c->mP));
  if (c->fastC) c->hsum = dalloc<double>(c, c->n);
  if (c->kind == K_CSR && !c->pSing && !c->cSing) c->gtmp = dalloc<double>(c, c->n);
  CK(cudaMemsetAsync(c->d, 0, c->n * sizeof(double), c->st));
  CK(cudaMemsetAsync(c->x, 0, c->n * sizeof(double), c->st));
  CK(cudaMemsetAsync(c->xbest, 0, c->n * sizeof(double), c->st));
  CK(cudaMemsetAsync(c->dy, 0, (c->mP > 0 ? c->mP : 1) * sizeof(double), c->st));
  if (c->dz) CK(cudaMemsetAsync(c->dz, 0, (c->mC > 0 ? c->mC : 1) * sizeof(double), c->st));
}

void init_ctx_common(mwu_ctx* c, const mwu_options* opt) {
  if (opt) c->opt = *opt; else mwu_default_options(&c->opt);
  c->world = c->opt.world > 1 ? c->opt.world : 1;
  c->rank = c->world > 1 ? c->opt.rank : 0;
  // a communicator is built for world > 1, and also for world = 1 when an NCCL id or a rank
  // group is passed (the sharded engine with one rank: exercises the exchange plumbing)
  if (c->world > 1 || c->opt.nccl_id || c->opt.comm_group) {
    if (c->rank < 0 || c->rank >= c->world) throw MwuError{MWU_ERR_ARG, "rank out of range"};
    try {
      if (c->opt.comm_group) c->comm = new SimComm((SimGroup*)c->opt.comm_group, c->rank);
      else if (c->opt.nccl_id) c->comm = new NcclComm(c->world, c->rank, c->opt.nccl_id);
      else throw std::runtime_error("world > 1 needs nccl_id or comm_group");
      c->sharded = 1;
    } catch (const std::exception& e) { throw MwuError{MWU_ERR_NCCL, e.what()}; }
    // NCCL collectives are captured into the probe graph with the kernels; the in-process test
    // group synchronises on the host, so its runs are host-driven
    if (!c->comm->capturable()) c->opt.use_graph = 0;
  }
  if (c->opt.device >= 0) CK(cudaSetDevice(c->opt.device));
  CK(cudaGetDevice(&c->dev));
  CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->dev));
  c->grid_rows = c->sms * 4;
  c->grid_max = c->sms * 8;
  CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  c->ctl = dalloc<Ctl>(c, 1);
  CK(cudaMallocHost(&c->hctl, sizeof(Ctl)));
  memset(c->hctl, 0, sizeof(Ctl));
  CK(cudaMemsetAsync(c->ctl, 0, sizeof(Ctl), c->st));
  c->part = dalloc<double>(c, (int64_t)c->grid_max * MWU_SLOTS);
  c->counter = dalloc<unsigned int>(c, 1);
  {
    double T[256];
    mwu_exp_table(T);
    c->exptab = dalloc<double>(c, 256);
    CK(cudaMemcpy(c->exptab, T, sizeof(T), cudaMemcpyHostToDevice));
    double E3[768];
    mwu_expm1_tables(E3, E3 + 256, E3 + 512);
    c->emtab = dalloc<double>(c, 768);
    CK(cudaMemcpy(c->emtab, E3, sizeof(E3), cudaMemcpyHostToDevice));
  }
  CK(cudaFuncSetAttribute(search_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSearchSmem));
  CK(cudaFuncSetAttribute(col_densest_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kColSmem));
  CK(cudaFuncSetAttribute(col_match_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMSmem));
  CK(cudaMemsetAsync(c->counter, 0, sizeof(unsigned int), c->st));
  CK(cudaEventCreate(&c->ev0));
  CK(cudaEventCreate(&c->ev1));
  CK(cudaEventCreateWithFlags(&c->evin, cudaEventDisableTiming));
  c->ust = (cudaStream_t)c->opt.stream;
  wait_caller(c);
}

// ------------------------------------------------------------------------------ graph build
void build_graph_storage(mwu_ctx* c, const mwu_graph* g) {
  const int64_t E = g->n_edges, nv = g->n_vertices;
  c->E = E; c->nv = nv; c->nleft = g->n_left;
  c->src = dalloc<int32_t>(c, E);
  c->dst = dalloc<int32_t>(c, E);
  if (E > 0) {
    CK(cudaMemcpyAsync(c->src, g->src, E * sizeof(int32_t), cudaMemcpyDefault, c->st));
    CK(cudaMemcpyAsync(c->dst, g->dst, E * sizeof(int32_t), cudaMemcpyDefault, c->st));
  }
  // validation: range, self-loops, bipartite sides, duplicate edges
  unsigned int* err = talloc<unsigned int>(1);
  CK(cudaMemsetAsync(err, 0, sizeof(unsigned int), c->st));
  if (E > 0) {
    unsigned long long* keys = talloc<unsigned long long>(E);
    unsigned long long* keys2 = talloc<unsigned long long>(E);
    k_validate_edges<<<grid_for(c, E), MWU_NT, 0, c->st>>>(E, c->src, c->dst, nv, g->n_left,
                                                            g->kind == MWU_G_BMATCH && g->n_left > 0, err, keys);
    CKL();
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, E, 0, 64, c->st));
    void* t = talloc<char>(tb);
    CK(cub::DeviceRadixSort::SortKeys(t, tb, keys, keys2, E, 0, 64, c->st));
    k_adjacent_dups<<<grid_for(c, E), MWU_NT, 0, c->st>>>(E, keys2, err);
    CKL();
    sync(c);
    tfree(t); tfree(keys); tfree(keys2);
  }
  const unsigned int ebits = read_scalar(c, err);
  tfree(err);
  if (ebits) {
    std::string m = "invalid graph:";
    if (ebits & 1) m += " vertex id out of range;";
    if (ebits & 2) m += " self-loop;";
    if (ebits & 4) m += " BMATCH edge not between the two sides split at n_left;";
    if (ebits & 8) m += " duplicate edge;";
    throw MwuError{MWU_ERR_ARG, m};
  }
  // degrees
  c->deg = dalloc<int32_t>(c, nv);
  CK(cudaMemsetAsync(c->deg, 0, nv * sizeof(int32_t), c->st));
  if (E > 0) { k_degree<<<grid_for(c, E), MWU_NT, 0, c->st>>>(E, c->src, c->dst, c->deg); CKL(); }
  {
    int64_t* deg64 = talloc<int64_t>(nv);
    k_to_int64<int32_t><<<grid_for(c, nv), MWU_NT, 0, c->st>>>(nv, c->deg, deg64, 0);
    CKL();
    int64_t* outm = talloc<int64_t>(1);
    size_t tb = 0;
    CK(cub::DeviceReduce::Max(nullptr, tb, deg64, outm, nv, c->st));
    void* t = talloc<char>(tb);
    CK(cub::DeviceReduce::Max(t, tb, deg64, outm, nv, c->st));
    c->maxdeg = read_scalar(c, outm);
    tfree(t);
    // incidence CSR over all vertices (rowptr = exclusive scan of deg)
    if (g->kind != MWU_G_DOMSET) {
      c->inc_all.nrows = nv;
      c->inc_all.nnz = 2 * E;
      c->inc_all.rowptr = dalloc<int64_t>(c, nv + 1);
      exclusive_scan_total(c, deg64, c->inc_all.rowptr, nv);
    }
    // non-isolated vertex count n'
    int64_t* fl = talloc<int64_t>(nv);
    k_nonzero_flags<<<grid_for(c, nv), MWU_NT, 0, c->st>>>(nv, c->deg, fl);
    CKL();
    int64_t* scan = talloc<int64_t>(nv + 1);
    exclusive_scan_total(c, fl, scan, nv);
    c->nprime = read_scalar(c, scan + nv);
    if (g->kind == MWU_G_MATCH || g->kind == MWU_G_BMATCH || g->kind == MWU_G_DENSEST) {
      c->prow = dalloc<int32_t>(c, nv);
      c->inc_p.nrows = c->nprime;
      c->inc_p.nnz = 2 * E;
      c->inc_p.rowptr = dalloc<int64_t>(c, c->nprime + 1);
    }
    // the fast path of the edge-variable kinds (d^(y) scattered by the column kernel over the
    // blocked edge order) never walks the vertex -> slot incidence: skip its 2E-slot sort
    const bool fastE = !c->opt.deterministic &&
                       (g->kind == MWU_G_MATCH || g->kind == MWU_G_BMATCH ||
                        (g->kind == MWU_G_DENSEST && E < (int64_t(1) << 31) - MWU_CT));
    // slots sorted by vertex (stable radix sort keeps slot order within a vertex)
    if (g->kind != MWU_G_DOMSET && !fastE) {
      c->inc_all.idx = dalloc<uint32_t>(c, 2 * E);
      if (E > 0) {
        uint32_t *keys = talloc<uint32_t>(2 * E), *kout = talloc<uint32_t>(2 * E), *vals = talloc<uint32_t>(2 * E);
        k_slot_keys<<<grid_for(c, 2 * E), MWU_NT, 0, c->st>>>(E, c->src, c->dst, keys, vals);
        CKL();
        size_t tb2 = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, keys, kout, vals, c->inc_all.idx, 2 * E, 0, bits_for(nv + 1), c->st));
        void* t2 = talloc<char>(tb2);
        CK(cub::DeviceRadixSort::SortPairs(t2, tb2, keys, kout, vals, c->inc_all.idx, 2 * E, 0, bits_for(nv + 1), c->st));
        sync(c);
        tfree(t2); tfree(keys); tfree(kout); tfree(vals);
      }
    }
    if (c->prow) {
      k_compact_rows<<<grid_for(c, nv), MWU_NT, 0, c->st>>>(nv, c->deg, scan, c->inc_all.rowptr, c->prow, c->inc_p.rowptr);
      CKL();
      const int64_t tot = 2 * E;
      CK(cudaMemcpyAsync(c->inc_p.rowptr + c->nprime, &tot, sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
      c->inc_p.idx = c->inc_all.idx;
      c->srow = dalloc<int32_t>(c, E);
      c->drow = dalloc<int32_t>(c, E);
      if (E > 0 && !fastE) {                  // fast path: written in the blocked order later
        k_map_endpoints<<<grid_for(c, E), MWU_NT, 0, c->st>>>(E, c->src, c->dst, c->prow, c->srow, c->drow);
        CKL();
      }
      sync(c);
      c->inc_fast = fastE ? 1 : 0;
    }
    sync(c);
    tfree(deg64); tfree(outm); tfree(fl); tfree(scan);
  }
  if (g->kind == MWU_G_DOMSET) {
    // C = I + A as CSR: sort (row << 32 | col) keys of diagonal and both edge directions
    const int64_t tot = nv + 2 * E;
    unsigned long long *keys = talloc<unsigned long long>(tot), *kout = talloc<unsigned long long>(tot);
    k_domset_keys<<<grid_for(c, tot), MWU_NT, 0, c->st>>>(nv, E, c->src, c->dst, keys);
    CKL();
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, kout, tot, 0, 64, c->st));
    void* t = talloc<char>(tb);
    CK(cub::DeviceRadixSort::SortKeys(t, tb, keys, kout, tot, 0, 64, c->st));
    c->csrC.nrows = nv;
    c->csrC.nnz = tot;
    c->csrC.idx = dalloc<uint32_t>(c, tot);
    k_low32<<<grid_for(c, tot), MWU_NT, 0, c->st>>>(tot, kout, c->csrC.idx);
    CKL();
    int64_t* deg1 = talloc<int64_t>(nv);
    k_to_int64<int32_t><<<grid_for(c, nv), MWU_NT, 0, c->st>>>(nv, c->deg, deg1, 1);
    CKL();
    c->csrC.rowptr = dalloc<int64_t>(c, nv + 1);
    exclusive_scan_total(c, deg1, c->csrC.rowptr, nv);
    sync(c);
    tfree(t); tfree(keys); tfree(kout); tfree(deg1);
    build_plan(c, c->csrC);
    c->cscC = c->csrC;  // symmetric: the CSR doubles as the CSC (column side)
    c->nnzC = tot;
  }
  if (c->inc_p.rowptr && !c->inc_fast) build_plan(c, c->inc_p);
  if (g->kind == MWU_G_VCOVER) build_plan(c, c->inc_all);
}

// ------------------------------------------------------------------------------ multi-GPU
// contiguous ranges on MWU_CT-edge tile boundaries (keeps the sliced per-edge arrays 16-byte
// aligned for the bulk copies and the activity words whole)
void shard_range(int64_t n, int world, int rank, int64_t& a, int64_t& b) {
  const int64_t tiles = (n + MWU_CT - 1) / MWU_CT;
  a = std::min(n, (int64_t)((__int128)tiles * rank / world) * MWU_CT);
  b = (rank + 1 == world) ? n : std::min(n, (int64_t)((__int128)tiles * (rank + 1) / world) * MWU_CT);
}

// complete a deferred partial reduction: gather every rank's slots, combine in rank order
void exchange(mwu_ctx* c) {
  if (!c->sharded) return;
  try {
    c->comm->allgather(c->ctl->dslots, c->gslots, MWU_SLOTS, c->st);
  } catch (const std::exception& e) { throw MwuError{MWU_ERR_NCCL, e.what()}; }
  finalize_multi<<<1, 32, 0, c->st>>>(c->ctl, c->gslots, c->world);
  CKL();
}

void allreduce_rows(mwu_ctx* c, double* v, int64_t n) {
  if (!c->sharded) return;
  try {
    c->comm->allreduce_sum(v, n, c->st);
  } catch (const std::exception& e) { throw MwuError{MWU_ERR_NCCL, e.what()}; }
}

// Restrict the context to this rank's internal edge range (after the global structure build).
void localize(mwu_ctx* c) {
  const int w = (c->kind == K_DENSEST) ? 2 : 1;
  c->Eg = c->E; c->ng = c->n; c->mCg = c->mC;
  c->perm_full = c->perm;
  if (!c->sharded) return;
  c->gslots = dalloc<double>(c, (int64_t)c->world * MWU_SLOTS);
  c->rb.assign(c->world + 1, 0);
  if (c->kind == K_DOMSET) {
    // covering rows (vertices) by nnz-balanced ranges on even rows (16-byte aligned row slices)
    std::vector<int64_t> rp(c->nv + 1);
    CK(cudaMemcpyAsync(rp.data(), c->csrC.rowptr, (c->nv + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    for (int r = 1; r < c->world; ++r) {
      const int64_t target = (int64_t)((__int128)c->nnzC * r / c->world);
      int64_t row = std::lower_bound(rp.begin(), rp.end(), target) - rp.begin();
      row &= ~int64_t(1);
      c->rb[r] = std::max(c->rb[r - 1], std::min(row, c->nv));
    }
    c->rb[c->world] = c->nv;
    c->r0 = c->rb[c->rank];
    c->mC = c->rb[c->rank + 1] - c->r0;
    c->k0 = rp[c->r0];
    c->nnzL = rp[c->r0 + c->mC] - c->k0;
    return;                                    // variables (vertices) replicated
  }
  if (c->own) c->rb = c->own_rb;              // edges of the rank's own right rows
  else
    for (int r = 0; r <= c->world; ++r) {
      int64_t a, b;
      shard_range(c->Eg, c->world, std::min(r, c->world - 1), a, b);
      c->rb[r] = (r == c->world) ? c->Eg : a;
    }
  const int64_t a = c->rb[c->rank], b = c->rb[c->rank + 1];
  c->e0 = a;
  c->E = b - a;
  if (c->kind == K_VCOVER) {                   // covering rows = edges local, vertices replicated
    c->mC = c->E;
    c->src += a;
    c->dst += a;
    return;
  }
  c->n = w * c->E;
  if (c->kind == K_DENSEST) c->mC = c->E;
  c->perm += a;
  if (c->own) {
    // owner edge ranges are not tile-aligned: the local rows move to aligned buffers (the
    // column kernel bulk-copies them), and the rank's rows are [0, nLx) + [R0, R1)
    int32_t *sr = dalloc<int32_t>(c, c->E), *dr = dalloc<int32_t>(c, c->E);
    if (c->E > 0) {
      CK(cudaMemcpyAsync(sr, c->srow + a, c->E * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(dr, c->drow + a, c->E * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->st));
    }
    c->srow = sr; c->drow = dr;
    c->R0 = std::max(c->own_rows[c->rank], c->nLx);
    c->R1 = std::max(c->own_rows[c->rank + 1], c->R0);
    return;
  }
  c->srow += a;
  c->drow += a;
}

// full vector of a sharded quantity (w per item of the sharded dimension: edges, or domset
// rows) from every rank's slice
const double* gather_full(mwu_ctx* c, const double* local, int w) {
  if (!c->sharded) return local;
  const int64_t total = c->rb[c->world];
  int64_t maxE = 0;
  for (int r = 0; r < c->world; ++r) maxE = std::max(maxE, c->rb[r + 1] - c->rb[r]);
  if (!c->gfull) { c->gfull = dalloc<double>(c, w * total); c->gsend = dalloc<double>(c, w * maxE * c->world + w * maxE); }
  double* recv = c->gsend + w * maxE;
  const int64_t mine = c->rb[c->rank + 1] - c->rb[c->rank];
  if (mine > 0) CK(cudaMemcpyAsync(c->gsend, local, w * mine * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  try {
    c->comm->allgather(c->gsend, recv, w * maxE, c->st);
  } catch (const std::exception& e) { throw MwuError{MWU_ERR_NCCL, e.what()}; }
  for (int r = 0; r < c->world; ++r) {
    const int64_t a = c->rb[r], b = c->rb[r + 1];
    if (b > a) CK(cudaMemcpyAsync(c->gfull + w * a, recv + (int64_t)r * w * maxE, w * (b - a) * sizeof(double),
                                  cudaMemcpyDeviceToDevice, c->st));
  }
  return c->gfull;
}

// Fast edge-variable kinds: L2-blocked internal edge order (storage.cuh k_block_keys) and the
// endpoint rows of the internal order.  perm maps internal -> original edge ids (Q29 order is
// restored by every vector hook and mwu_get_x).
constexpr int kBlockLDefault = 22, kBlockRDefault = 20;   // src blocks of 4M rows, dst blocks of 1M rows
void build_blocked_order(mwu_ctx* c) {
  const int64_t E = c->E;
  if (E <= 0) return;
  // matching (random bipartite, degree ~16: no src-block reuse): one source block
  // (edges sorted by src row) and 4M-row destination blocks whose u / d^(y) slices stay in L2
  int defL = kBlockLDefault, defR = kBlockRDefault;
  if (c->kind == K_MATCH) {
    defL = 1;
    while (defL < 31 && (int64_t(1) << defL) < c->nprime) ++defL;
    defR = 22;
  }
  const int kBlockL = c->opt.block_l > 0 ? c->opt.block_l : defL;
  const int kBlockR = c->opt.block_r > 0 ? c->opt.block_r : defR;
  if (kBlockL > 31 || kBlockR > 31) throw MwuError{MWU_ERR_ARG, "block_l / block_r must be <= 31"};
  // packing rows in degree-descending order (fast path only; hooks restore vertex order)
  int32_t* prowf = talloc<int32_t>(c->nv);
  uint32_t* dvo = talloc<uint32_t>(c->nv);   // vertices in row order
  {
    unsigned long long *dk = talloc<unsigned long long>(c->nv), *dko = talloc<unsigned long long>(c->nv);
    uint32_t *dv = talloc<uint32_t>(c->nv);
    k_deg_keys<<<grid_for(c, c->nv), MWU_NT, 0, c->st>>>(c->nv, c->deg, c->kind == K_MATCH ? c->nleft : 0, dk, dv);
    CKL();
    size_t tb2 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, dk, dko, dv, dvo, c->nv, 0, 64, c->st));
    void* t2 = talloc<char>(tb2);
    CK(cub::DeviceRadixSort::SortPairs(t2, tb2, dk, dko, dv, dvo, c->nv, 0, 64, c->st));
    c->rowperm = dalloc<uint32_t>(c, c->nprime);
    k_deg_rows<<<grid_for(c, c->nprime), MWU_NT, 0, c->st>>>(c->nprime, dvo, c->prow, prowf, c->rowperm);
    CKL();
    sync(c);
    tfree(t2); tfree(dk); tfree(dko); tfree(dv);
  }
  // L2 blocks over ROW ranges of the (degree-ordered) packing-row vectors: key = (srow >> BL,
  // drow >> BR, srow, drow)
  const int64_t nr = std::max<int64_t>(c->nprime, 1);
  const int nbL = (int)((nr + (int64_t(1) << kBlockL) - 1) >> kBlockL);
  const int nbR = (int)((nr + (int64_t(1) << kBlockR) - 1) >> kBlockR);
  unsigned long long *keys = talloc<unsigned long long>(E), *kout = talloc<unsigned long long>(E);
  uint32_t* vals = talloc<uint32_t>(E);
  c->perm = dalloc<uint32_t>(c, E);
  int bits = kBlockL + kBlockR;
  int64_t* d_ob = nullptr;
  if (c->own) {
    // right rows split into W ranges of about E / W edges each (degree prefix sums), boundaries
    // even (16-byte aligned row slices for the search's bulk copies)
    const int W = c->world;
    unsigned long long* cnt = talloc<unsigned long long>(1);
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c->st));
    k_count_left<<<grid_for(c, c->nleft), MWU_NT, 0, c->st>>>(c->nleft, c->deg, cnt);
    CKL();
    const int64_t nLp = (int64_t)read_scalar(c, cnt);
    tfree(cnt);
    const int64_t nR = c->nprime - nLp;
    int64_t *rd = talloc<int64_t>(std::max<int64_t>(nR, 1)), *cum = talloc<int64_t>(std::max<int64_t>(nR, 1));
    k_right_deg<<<grid_for(c, std::max<int64_t>(nR, 1)), MWU_NT, 0, c->st>>>(nR, nLp, dvo, c->deg, rd);
    CKL();
    size_t tb3 = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb3, rd, cum, nR, c->st));
    void* t3 = talloc<char>(tb3);
    CK(cub::DeviceScan::InclusiveSum(t3, tb3, rd, cum, nR, c->st));
    int64_t* d_b = talloc<int64_t>(W + 1);
    if (W > 1) k_owner_bounds<<<1, 64, 0, c->st>>>(cum, nR, E, W, d_b);
    CKL();
    std::vector<int64_t> hb(W + 1, 0);
    CK(cudaMemcpyAsync(hb.data(), d_b, (W + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    tfree(t3); tfree(rd); tfree(cum); tfree(d_b);
    c->nLx = std::min(c->nprime, nLp + (nLp & 1));
    c->own_rows.assign(W + 1, 0);
    c->own_rows[0] = nLp;
    for (int r = 1; r < W; ++r) {
      int64_t row = nLp + hb[r] + 1;                       // the row reaching the target stays below
      row = (row + 1) & ~int64_t(1);
      c->own_rows[r] = std::min(c->nprime, std::max(row, std::max(c->own_rows[r - 1], c->nLx)));
    }
    c->own_rows[W] = c->nprime;
    int64_t maxrows = 1;
    for (int r = 0; r < W; ++r) maxrows = std::max(maxrows, c->own_rows[r + 1] - c->own_rows[r]);
    const int nbRo = (int)((maxrows + (int64_t(1) << kBlockR) - 1) >> kBlockR);
    d_ob = talloc<int64_t>(W + 1);
    CK(cudaMemcpyAsync(d_ob, c->own_rows.data(), (W + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
    k_block_keys_own<<<grid_for(c, E), MWU_NT, 0, c->st>>>(E, c->src, c->dst, prowf, d_ob, W, nbRo, kBlockL, kBlockR,
                                                          keys, vals);
    while (bits < 64 && (1ull << (bits - kBlockL - kBlockR)) < (unsigned long long)W * (unsigned long long)nbRo) ++bits;
  } else {
    k_block_keys<<<grid_for(c, E), MWU_NT, 0, c->st>>>(E, c->src, c->dst, prowf, nbR, kBlockL, kBlockR, keys, vals);
    while (bits < 64 && (1ull << (bits - kBlockL - kBlockR)) < (unsigned long long)nbL * (unsigned long long)nbR) ++bits;
  }
  CKL();
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, kout, vals, c->perm, E, 0, bits, c->st));
  void* t = talloc<char>(tb);
  CK(cub::DeviceRadixSort::SortPairs(t, tb, keys, kout, vals, c->perm, E, 0, bits, c->st));
  k_map_endpoints_perm<<<grid_for(c, E), MWU_NT, 0, c->st>>>(E, c->perm, c->src, c->dst, prowf, c->srow, c->drow);
  CKL();
  if (c->own) {                              // edge range of every owner along the internal order
    k_orient<<<grid_for(c, E), MWU_NT, 0, c->st>>>(E, c->srow, c->drow);
    CKL();
    const int W = c->world;
    int64_t* d_e = talloc<int64_t>(W + 1);
    k_owner_edges<<<1, 128, 0, c->st>>>(c->drow, E, d_ob, W, d_e);
    CKL();
    c->own_rb.assign(W + 1, 0);
    CK(cudaMemcpyAsync(c->own_rb.data(), d_e, (W + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    tfree(d_e); tfree(d_ob);
  }
  sync(c);
  tfree(prowf); tfree(dvo);
  tfree(t); tfree(keys); tfree(kout); tfree(vals);
}

// internal -> original order of an edge-variable (w = 1 match, 2 densest) or edge-row (w = 1) vector
const double* unperm(mwu_ctx* c, const double* in, int w) {
  if (!c->perm) return in;
  in = gather_full(c, in, w);
  k_unperm<<<grid_for(c, c->Eg), MWU_NT, 0, c->st>>>(c->Eg, c->perm_full, in, c->tmp2, w);
  CKL();
  return c->tmp2;
}

// ------------------------------------------------------------------------------ CSR build
void copy_csr_checked(mwu_ctx* c, const mwu_csr* A, Seg& S, int64_t cols, const char* name) {
  if (A->rows < 0 || A->cols != cols || A->nnz < 0 || !A->rowptr || (A->nnz > 0 && !A->colidx))
    throw MwuError{MWU_ERR_ARG, std::string(name) + ": bad dimensions or null pointers"};
  S.nrows = A->rows;
  S.nnz = A->nnz;
  S.rowptr = dalloc<int64_t>(c, A->rows + 1);
  S.idx = dalloc<uint32_t>(c, A->nnz);
  CK(cudaMemcpyAsync(S.rowptr, A->rowptr, (A->rows + 1) * sizeof(int64_t), cudaMemcpyDefault, c->st));
  if (A->nnz > 0) CK(cudaMemcpyAsync(S.idx, A->colidx, A->nnz * sizeof(int32_t), cudaMemcpyDefault, c->st));
  if (A->vals) {
    S.val = dalloc<double>(c, A->nnz);
    if (A->nnz > 0) CK(cudaMemcpyAsync(S.val, A->vals, A->nnz * sizeof(double), cudaMemcpyDefault, c->st));
  }
  int64_t ends[2];
  CK(cudaMemcpyAsync(&ends[0], S.rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(&ends[1], S.rowptr + A->rows, sizeof(int64_t), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  if (ends[0] != 0 || ends[1] != A->nnz) throw MwuError{MWU_ERR_ARG, std::string(name) + ": rowptr[0] != 0 or rowptr[rows] != nnz"};
  unsigned int* err = talloc<unsigned int>(1);
  int32_t* rl = talloc<int32_t>(A->rows);
  CK(cudaMemsetAsync(err, 0, sizeof(unsigned int), c->st));
  if (A->rows > 0) { k_validate_csr<<<grid_for(c, A->rows), MWU_NT, 0, c->st>>>(A->rows, cols, S.rowptr, S.idx, S.val, err, rl); CKL(); }
  const unsigned int eb = read_scalar(c, err);
  tfree(err);
  tfree(rl);
  if (eb & 16) throw MwuError{MWU_ERR_ARG, std::string(name) + ": column index out of range or not strictly increasing in a row"};
  if (eb & 32) throw MwuError{MWU_ERR_ARG, std::string(name) + ": negative or non-finite value (positive LP required)"};
}

// drop empty rows of P (Q17): compacted rowptr over the same item arrays
void compact_rows(mwu_ctx* c, Seg& S) {
  int64_t* fl = talloc<int64_t>(S.nrows);
  if (S.nrows > 0) { k_row_nonempty<<<grid_for(c, S.nrows), MWU_NT, 0, c->st>>>(S.nrows, S.rowptr, fl); CKL(); }
  int64_t* scan = talloc<int64_t>(S.nrows + 1);
  exclusive_scan_total(c, fl, scan, S.nrows);
  const int64_t kept = read_scalar(c, scan + S.nrows);
  if (kept != S.nrows) {
    int64_t* rp = dalloc<int64_t>(c, kept + 1);
    k_compact_csr_rows<<<grid_for(c, S.nrows), MWU_NT, 0, c->st>>>(S.nrows, S.rowptr, scan, rp);
    CKL();
    CK(cudaMemcpyAsync(rp + kept, &S.nnz, sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
    sync(c);
    c->empty_dropped = S.nrows - kept;
    S.rowptr = rp;
    S.nrows = kept;
  }
  tfree(fl);
  tfree(scan);
}

// packing side of an explicit instance, after csrP holds the CSR: drop empty rows (Q17), tile
// plan, CSC copy, column maxima ||P_{:,i}||_inf for x0
void finish_csr_packing(mwu_ctx* c, int64_t n) {
  compact_rows(c, c->csrP);                       // Q17
  c->mP = c->csrP.nrows; c->nnzP = c->csrP.nnz;
  build_plan(c, c->csrP);
  build_csc(c, c->csrP, n, c->cscP);
  c->colmaxP = dalloc<double>(c, n);
  c->crecipP = dalloc<double>(c, n);
  k_col_stats<<<grid_for(c, n), MWU_NT, 0, c->st>>>(n, c->cscP.rowptr, c->cscP.val, c->colmaxP, nullptr, c->crecipP);
  CKL();
  // an all-zero packing column leaves x_i = eps/(n*0) undefined
  double* mn = talloc<double>(1);
  size_t tb = 0;
  CK(cub::DeviceReduce::Min(nullptr, tb, c->colmaxP, mn, n, c->st));
  void* t = talloc<char>(tb);
  CK(cub::DeviceReduce::Min(t, tb, c->colmaxP, mn, n, c->st));
  const double mincol = read_scalar(c, mn);
  tfree(t); tfree(mn);
  if (!(mincol > 0.0)) throw MwuError{MWU_ERR_ARG, "P has an all-zero column: initialisation x_i = eps/(n ||P_:,i||) undefined"};
}

// covering side: record empty covering rows (infeasible, Q17), tile plan, CSC copy, column sums
void finish_csr_covering(mwu_ctx* c, int64_t n) {
  c->mC = c->csrC.nrows; c->nnzC = c->csrC.nnz;
  // empty covering rows make the LP infeasible (0 >= 1), Q17
  {
    Seg tmpS = c->csrC;
    const int64_t before = tmpS.nrows;
    int64_t saved = c->empty_dropped;
    compact_rows(c, tmpS);
    c->empty_cover = (tmpS.nrows != before);
    c->empty_dropped = saved;
  }
  build_plan(c, c->csrC);
  build_csc(c, c->csrC, n, c->cscC);
  c->colsumC = dalloc<double>(c, n);
  c->crecipC = dalloc<double>(c, n);
  k_col_stats<<<grid_for(c, n), MWU_NT, 0, c->st>>>(n, c->cscC.rowptr, c->cscC.val, nullptr, c->colsumC, c->crecipC);
  CKL();
}

// Generalized matching (NEXT#3): rows of diag(1/b) M for the vertices selected by
// sel (the vertex -> incident-slot CSR gives each row's edges in ascending edge id: canonical CSR)
__global__ void k_gm_count(int64_t nrows, const int32_t* __restrict__ sel, const int64_t* __restrict__ inc_rowptr,
                           int64_t* __restrict__ cnt) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = sel[r];
    cnt[r] = inc_rowptr[v + 1] - inc_rowptr[v];
  }
}
__global__ void k_gm_fill(int64_t nrows, const int32_t* __restrict__ sel, const int64_t* __restrict__ inc_rowptr,
                          const uint32_t* __restrict__ slots, const double* __restrict__ bound,
                          const int64_t* __restrict__ rowptr, uint32_t* __restrict__ col, double* __restrict__ val) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = sel[r];
    const double w = 1.0 / bound[v];                    // row v of M scaled by 1/u(v) or 1/l(v)
    const int64_t a = inc_rowptr[v], b = inc_rowptr[v + 1], o = rowptr[r];
    for (int64_t k = a; k < b; ++k) { col[o + (k - a)] = slots[k] >> 1; val[o + (k - a)] = w; }
  }
}
__global__ void k_gm_flags(int64_t nv, const double* __restrict__ lb, const double* __restrict__ ub,
                           uint8_t* __restrict__ fp, uint8_t* __restrict__ fc, unsigned int* __restrict__ err) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const double l = lb[v], u = ub[v];
    if (!(l >= 0.0) || !(u > 0.0) || !(l <= u) || isinf(l)) atomicOr(err, 64u);
    fp[v] = isfinite(u) ? 1 : 0;                         // packing row  (1/u(v)) M_v x <= 1
    fc[v] = (l > 0.0) ? 1 : 0;                           // covering row (1/l(v)) M_v x >= 1
  }
}

// select the flagged vertex ids, build the scaled CSR of their incidence rows
void build_gm_side(mwu_ctx* c, const uint8_t* flags, const double* bound, Seg& S) {
  const int64_t nv = c->nv;
  int32_t* sel = talloc<int32_t>(nv);
  int64_t* nsel = talloc<int64_t>(1);
  cub::CountingInputIterator<int32_t> it(0);
  size_t tb = 0;
  CK(cub::DeviceSelect::Flagged(nullptr, tb, it, flags, sel, nsel, nv, c->st));
  void* t = talloc<char>(tb);
  CK(cub::DeviceSelect::Flagged(t, tb, it, flags, sel, nsel, nv, c->st));
  const int64_t rows = read_scalar(c, nsel);
  tfree(t);
  S.nrows = rows;
  S.rowptr = dalloc<int64_t>(c, rows + 1);
  int64_t* cnt = talloc<int64_t>(rows);
  if (rows > 0) { k_gm_count<<<grid_for(c, rows), MWU_NT, 0, c->st>>>(rows, sel, c->inc_all.rowptr, cnt); CKL(); }
  exclusive_scan_total(c, cnt, S.rowptr, rows);
  S.nnz = read_scalar(c, S.rowptr + rows);
  S.idx = dalloc<uint32_t>(c, S.nnz);
  S.val = dalloc<double>(c, S.nnz);
  if (rows > 0) {
    k_gm_fill<<<grid_for(c, rows), MWU_NT, 0, c->st>>>(rows, sel, c->inc_all.rowptr, c->inc_all.idx, bound, S.rowptr,
                                                      S.idx, S.val);
    CKL();
  }
  sync(c);
  tfree(cnt); tfree(sel); tfree(nsel);
}

// ------------------------------------------------------------------------------ kernel launchers
template <class Ep>
void launch_seg(mwu_ctx* c, cudaStream_t st, const Seg& S, ItemGather it, Ep ep, int action) {
  const SegView sv = S.view();
  if (S.nlong > 0) {
    seg_long_chunks<ItemGather><<<grid_for(c, S.nchunks * MWU_NT), MWU_NT, 0, st>>>(sv, it, c->ctl);
    c->launches++;
  }
  int g = (int)((S.ntiles < c->grid_rows) ? (S.ntiles < 1 ? 1 : S.ntiles) : c->grid_rows);
  if (S.nlong > 0 && g < 8) g = 8;
  seg_main<ItemGather, Ep><<<g, MWU_NT, 0, st>>>(sv, it, ep, c->ctl, c->part, c->counter, action);
  c->launches++;
}

ItemGather item_of(const Seg& S, const double* vec, int shift, const double* scale_ptr) {
  ItemGather it;
  it.idx = S.idx; it.val = S.val; it.vec = vec; it.shift = shift; it.scale_ptr = scale_ptr;
  return it;
}

int rows_grid(mwu_ctx* c, int64_t rows) {
  const int g = grid_for(c, rows > 0 ? rows : 1);
  return g < c->grid_rows ? g : c->grid_rows;
}

EpColumn make_col(mwu_ctx* c, int s_is_h, const double* gtmp) {
  EpColumn ep;
  ep.x = c->x; ep.d = c->d; ep.gtmp = gtmp; ep.gdbg = c->record ? c->gdbg : nullptr; ep.hdbg = c->record ? c->hdbg : nullptr;
  ep.c = c->ctl; ep.s_is_h = s_is_h; ep.kind_step = 0;
  return ep;
}

void enqueue_column(mwu_ctx* c, cudaStream_t st) {
  switch (c->kind) {
    case K_MATCH:
      if (c->scatterP) {
        CK(cudaMemsetAsync(c->dy, 0, (c->mP > 0 ? c->mP : 1) * sizeof(double), st));
        const int64_t tiles = (c->E + MWU_CT - 1) / MWU_CT;
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, MWU_MT_MINB * c->sms));
        col_match_fast<<<g, MWU_NT, kMSmem, st>>>(c->E, c->srow, c->drow, c->u, c->x, c->d, c->dy,
                                                c->record ? c->gdbg : nullptr, c->record ? c->hdbg : nullptr,
                                                c->ctl, c->part, c->counter, c->act);
        c->launches++;
        break;
      }
      col_match<<<rows_grid(c, c->E), MWU_NT, 0, st>>>(c->E, c->srow, c->drow, c->u, c->x, c->d,
                                                      c->record ? c->gdbg : nullptr, c->record ? c->hdbg : nullptr,
                                                      c->ctl, c->part, c->counter);
      c->launches++;
      break;
    case K_DENSEST:
      if (c->lazyC) {
        CK(cudaMemsetAsync(c->dy, 0, (c->mP > 0 ? c->mP : 1) * sizeof(double), st));
        const int g = (int)c->rec_grid;
        col_densest_fast<<<g, MWU_NT, kColSmem, st>>>(c->E, c->srow, c->drow, c->u, c->x, c->d, c->z, c->dy, c->act, c->rz,
                                              c->rdz, c->rv, c->tcnt, c->rec_cap, c->record ? c->gdbg : nullptr,
                                              c->record ? c->hdbg : nullptr, c->ctl, c->part, c->counter, c->exptab);
        inactive_exact<<<rows_grid(c, c->E), MWU_NT, 0, st>>>(c->E, c->act, c->z, c->ctl, c->part, c->counter);
        c->launches += 2;
        break;
      }
      col_densest<<<rows_grid(c, c->E), MWU_NT, 0, st>>>(c->E, c->srow, c->drow, c->u, c->v, c->x, c->d, c->dz,
                                                        c->record ? c->gdbg : nullptr, c->record ? c->hdbg : nullptr,
                                                        c->ctl, c->part, c->counter);
      c->launches++;
      break;
    case K_VCOVER:
    case K_DOMSET:
      if (c->fastC) {
        CK(cudaMemsetAsync(c->hsum, 0, c->n * sizeof(double), st));
        if (c->kind == K_VCOVER)
          vc_scatter<<<(int)std::min<int64_t>(MWU_VC_GRID * c->sms, (c->E + 4 * MWU_NT - 1) / (4 * MWU_NT) + 1), MWU_NT, 0, st>>>(
              c->E, c->src, c->dst, c->v, c->hsum, c->ctl);
        else if (!c->sharded)
          csr_scatter<<<(int)std::min<int64_t>(MWU_CSR_GRID * c->sms, (c->nnzC + 4 * MWU_NT - 1) / (4 * MWU_NT) + 1), MWU_NT, 0, st>>>(
              c->nnzC, c->rowidC, c->csrC.idx, c->v, c->hsum, c->ctl, 0);
        else   // local rows: C^T v by scattering each local row's weight to its columns (C symmetric)
          csr_scatter_T<<<(int)std::min<int64_t>(4 * c->sms, (c->nnzL + 4 * MWU_NT - 1) / (4 * MWU_NT) + 1), MWU_NT, 0, st>>>(
              c->nnzL, c->rowidC + c->k0, c->csrC.idx + c->k0, c->v, c->r0, c->hsum, c->ctl);
        allreduce_rows(c, c->hsum, c->n);     // sharded: partial column gradient of the local rows
        col_vertex<<<rows_grid(c, c->n), MWU_NT, 0, st>>>(c->n, c->hsum, c->x, c->d, c->record ? c->gdbg : nullptr,
                                                        c->record ? c->hdbg : nullptr, c->ctl, c->part, c->counter);
        c->launches += 2;
        break;
      }
      if (c->kind == K_VCOVER)
        launch_seg(c, st, c->inc_all, item_of(c->inc_all, c->v, 1, nullptr), make_col(c, 1, nullptr), A_COL);
      else
        launch_seg(c, st, c->cscC, item_of(c->cscC, c->v, 0, nullptr), make_col(c, 1, nullptr), A_COL);
      break;
    case K_CSR:
      if (!c->pSing && !c->cSing) {
        EpStoreG eg; eg.g = c->gtmp; eg.c = c->ctl; eg.kind_step = 0;
        launch_seg(c, st, c->cscP, item_of(c->cscP, c->u, 0, nullptr), eg, A_NONE);
        launch_seg(c, st, c->cscC, item_of(c->cscC, c->v, 0, nullptr), make_col(c, 1, c->gtmp), A_COL);
      } else if (c->cSing) {
        launch_seg(c, st, c->cscP, item_of(c->cscP, c->u, 0, nullptr), make_col(c, 0, nullptr), A_COL);
      } else {
        launch_seg(c, st, c->cscC, item_of(c->cscC, c->v, 0, nullptr), make_col(c, 1, nullptr), A_COL);
      }
      break;
  }
}

// forward products: out_y = P in, out_z = C in.  init: actions A_NONE; iteration: step actions
void enqueue_forward(mwu_ctx* c, cudaStream_t st, const double* in, double* oy, double* oz, bool init) {
  EpOut ey; ey.out = oy; ey.kind_step = init ? 0 : 1;
  EpOut ez; ez.out = oz; ez.kind_step = init ? 0 : 1;
  double* invB = &c->ctl->invB;
  const int a_done_p = init ? A_NONE : A_STEP_DONE + 100;
  const int a_done = init ? A_NONE : A_STEP_DONE;
  switch (c->kind) {
    case K_MATCH:
      if (!init && c->scatterP) {            // d^(y) was scattered by the column kernel
        dy_finalize<<<rows_grid(c, c->mP), MWU_NT, 0, st>>>(c->mP, c->dy, c->ctl, c->part, c->counter);
        c->launches++;
        break;
      }
      if (init && c->scatterP) {
        CK(cudaMemsetAsync(oy, 0, (c->mP > 0 ? c->mP : 1) * sizeof(double), st));
        scatter_init<<<rows_grid(c, c->E), MWU_NT, 0, st>>>(c->E, c->srow, c->drow, in, oy, c->ctl, 0);
        c->launches++;
        break;
      }
      launch_seg(c, st, c->inc_p, item_of(c->inc_p, in, 1, nullptr), ey, a_done_p);
      break;
    case K_DENSEST:
      if (!init && c->lazyC) {               // d^(y) was scattered by the column kernel
        dy_finalize<<<rows_grid(c, c->mP), MWU_NT, 0, st>>>(c->mP, c->dy, c->ctl, c->part, c->counter);
        c->launches++;
        break;
      }
      if (init) {
        pair_sum<<<rows_grid(c, c->E), MWU_NT, 0, st>>>(c->E, in, oz, c->ctl);
        c->launches++;
      }
      if (init && c->scatterP) {
        CK(cudaMemsetAsync(oy, 0, (c->mP > 0 ? c->mP : 1) * sizeof(double), st));
        scatter_init<<<rows_grid(c, c->E), MWU_NT, 0, st>>>(c->E, c->srow, c->drow, in, oy, c->ctl, 1);
        c->launches++;
        break;
      }
      launch_seg(c, st, c->inc_p, item_of(c->inc_p, in, 0, invB), ey, a_done_p);
      break;
    case K_VCOVER:
      if (!init && c->compC) {
        edge_sum_compact<<<(int)c->rec_grid, MWU_NT, 0, st>>>(c->E, c->src, c->dst, in, oz, c->z, c->v, c->rz, c->rdz,
                                                              c->rv, c->tcnt, c->rec_cap, c->ctl, c->part, c->counter);
        inactive_exact_dz<<<rows_grid(c, c->E), MWU_NT, 0, st>>>(c->E, oz, c->z, c->ctl, c->part, c->counter);
        c->launches += 2;
        break;
      }
      edge_sum<<<rows_grid(c, c->E), MWU_NT, 0, st>>>(c->E, c->src, c->dst, in, oz, c->ctl, c->part, c->counter, a_done);
      c->launches++;
      break;
    case K_DOMSET:
      if (c->fastC) {
        CK(cudaMemsetAsync(oz, 0, (c->mC > 0 ? c->mC : 1) * sizeof(double), st));
        const int64_t nz = c->sharded ? c->nnzL : c->nnzC;
        csr_scatter<<<(int)std::min<int64_t>(MWU_CSR_GRID * c->sms, (nz + 4 * MWU_NT - 1) / (4 * MWU_NT) + 1), MWU_NT, 0, st>>>(
            nz, c->rowidC + c->k0, c->csrC.idx + c->k0, in, oz, c->ctl, c->r0);
        c->launches++;
        if (!init && c->compC) {
          edge_sum_compact<<<(int)c->rec_grid, MWU_NT, 0, st>>>(c->mC, nullptr, nullptr, oz, oz, c->z, c->v, c->rz,
                                                                c->rdz, c->rv, c->tcnt, c->rec_cap, c->ctl, c->part,
                                                                c->counter);
          inactive_exact_dz<<<rows_grid(c, c->mC), MWU_NT, 0, st>>>(c->mC, oz, c->z, c->ctl, c->part, c->counter);
          c->launches += 2;
        } else if (!init) {
          step_done<<<1, 32, 0, st>>>(c->ctl);
          c->launches++;
        }
        break;
      }
      launch_seg(c, st, c->csrC, item_of(c->csrC, in, 0, nullptr), ez, a_done);
      break;
    case K_CSR:
      if (!c->pSing && !c->cSing) {
        launch_seg(c, st, c->csrP, item_of(c->csrP, in, 0, nullptr), ey, init ? A_NONE : A_STEP_MAXDY);
        launch_seg(c, st, c->csrC, item_of(c->csrC, in, 0, nullptr), ez, a_done);
      } else if (c->cSing) {
        launch_seg(c, st, c->csrP, item_of(c->csrP, in, 0, nullptr), ey, a_done_p);
      } else {
        launch_seg(c, st, c->csrC, item_of(c->csrC, in, 0, nullptr), ez, a_done);
      }
      break;
  }
}

void enqueue_search(mwu_ctx* c, cudaStream_t st) {
  const int64_t chunks = (std::max(c->mP, c->mC) + MWU_SCH - 1) / MWU_SCH;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(MWU_SEARCH_MINB * c->sms, chunks));
  SearchArgs A;
  int64_t p0 = 0, p1 = c->mP;                // sharded: each rank sums a slice of the replicated rows
  const int64_t rep = c->own ? c->nLx : c->mP;
  if (c->sharded) {
    shard_range(rep, c->world, c->rank, p0, p1);
    p0 &= ~int64_t(1);                       // 16-byte aligned bulk copies
    if (c->rank + 1 < c->world) p1 &= ~int64_t(1);
  }
  A.mP = p1 - p0; A.y = c->y + p0; A.dy = c->dy + p0; A.u = c->u + p0;
  A.mP2 = c->own ? c->R1 - c->R0 : 0;       // + the rank's own rows (owner-partitioned matching)
  A.y2 = c->y + c->R0; A.dy2 = c->dy + c->R0; A.u2 = c->u + c->R0;
  A.mC = c->mC; A.z = c->z; A.dz = c->dz; A.v = c->v;
  A.rz = c->rz; A.rdz = c->rdz; A.rv = c->rv; A.tcnt = c->tcnt;
  A.nstreams = c->rec_grid * (MWU_NT / 32); A.rcap = c->rec_cap;
  A.emtab = c->emtab;
  search_pass<<<g, MWU_NT, kSearchSmem, st>>>(A, c->ctl, c->part, c->counter);
  c->launches++;
}

void enqueue_update(mwu_ctx* c, cudaStream_t st, int has_delta) {
  // lazyC: the covering side is updated lazily by the next column kernel (only at init are its
  // weight sums formed here, without storing v)
  const int64_t mC = (c->lazyC && has_delta) ? 0 : c->mC;
  const int64_t mP = c->own ? c->nLx : c->mP;   // owner-partitioned: replicated rows + own rows
  update_rows<<<rows_grid(c, c->mP + mC), MWU_NT, 0, st>>>(mP, c->y, c->dy, c->u, mC, c->z, c->dz, c->v,
                                                          c->ctl, c->part, c->counter, has_delta,
                                                          c->own ? c->R0 : 0, c->own ? c->R1 : 0);
  c->launches++;
}

// ------------------------------------------------------------------------------ graph (probe loop)
void enqueue_col_step(mwu_ctx* c);
void enqueue_search_pass(mwu_ctx* c);
void enqueue_update_phase(mwu_ctx* c);

void build_probe_graph(mwu_ctx* c) {
  if (c->graph_ok) return;
  cudaGraph_t top;
  CK(cudaGraphCreate(&top, 0));
  cudaGraphConditionalHandle hi;
  CK(cudaGraphConditionalHandleCreate(&hi, top, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = hi;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t wn;
  CK(cudaGraphAddNode(&wn, top, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  cudaGraphConditionalHandle hs;
  CK(cudaGraphConditionalHandleCreate(&hs, body, 0, 0));
  // part A: column + step
  const int64_t l0 = c->launches;
  CK(cudaStreamBeginCaptureToGraph(c->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  enqueue_col_step(c);
  cudaStreamCaptureStatus cst;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CK(cudaStreamGetCaptureInfo(c->st, &cst, nullptr, nullptr, &deps, &ndeps));
  std::vector<cudaGraphNode_t> leaf(deps, deps + ndeps);
  cudaGraph_t g2;
  CK(cudaStreamEndCapture(c->st, &g2));
  // inner WHILE: search passes
  cudaGraphNodeParams p2 = {};
  p2.type = cudaGraphNodeTypeConditional;
  p2.conditional.handle = hs;
  p2.conditional.type = cudaGraphCondTypeWhile;
  p2.conditional.size = 1;
  cudaGraphNode_t sn;
  CK(cudaGraphAddNode(&sn, body, leaf.data(), leaf.size(), &p2));
  cudaGraph_t sbody = p2.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(c->st, sbody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  enqueue_search_pass(c);
  CK(cudaStreamEndCapture(c->st, &g2));
  // part C: update, after the search loop
  CK(cudaStreamBeginCaptureToGraph(c->st, body, &sn, nullptr, 1, cudaStreamCaptureModeRelaxed));
  enqueue_update_phase(c);
  CK(cudaStreamEndCapture(c->st, &g2));
  CK(cudaGraphInstantiate(&c->gexec, top, 0));
  c->graph = top;
  c->h_iter = (unsigned long long)hi;
  c->h_search = (unsigned long long)hs;
  c->launches = l0;  // captured launches are not executed launches
  c->graph_ok = true;
}

// ------------------------------------------------------------------------------ probe engine
int64_t m_total(mwu_ctx* c) { return (c->pSing ? 1 : c->mP) + (c->cSing ? 1 : (c->mCg > 0 ? c->mCg : c->mC)); }

void probe_begin(mwu_ctx* c, double bound, double eps) {
  if (!(eps > 0.0 && eps < 1.0)) throw MwuError{MWU_ERR_ARG, "eps must be in (0, 1)"};
  if (!(bound > 0.0) || !std::isfinite(bound)) throw MwuError{MWU_ERR_ARG, "bound must be positive and finite"};
  if ((c->ng > 0 ? c->ng : c->n) <= 0) throw MwuError{MWU_ERR_ARG, "instance has no variables"};   // a shard may be empty
  if (c->opt.use_graph) build_probe_graph(c);
  Ctl& h = *c->hctl;
  memset(&h, 0, sizeof(Ctl));
  const int64_t m = m_total(c);
  h.eps = eps;
  h.B = bound;
  h.invB = 1.0 / bound;                                    // (1/M) 1^T or 1/D
  h.eta = c->opt.eta_factor * std::log((double)m) / eps;   // P:271, Q1, Q2
  h.sigma = (c->mode == MWU_MIXED) ? 1.0 / (2.0 * h.eta) : 1.0 / h.eta;   // P:279, P:322 (Q13)
  h.max_iter = c->opt.max_iter;
  h.pSing = c->pSing;
  h.cSing = c->cSing;
  h.mode = c->mode;
  h.tol_prose = c->opt.tol_prose;
  h.max_evals = c->opt.max_evals;
  h.bisect_depth = c->opt.bisect_depth;
  if (c->opt.step_rule < MWU_STEP_BINARY || c->opt.step_rule > MWU_STEP_STANDARD)
    throw MwuError{MWU_ERR_ARG, "unknown step_rule"};
  h.step_rule = c->opt.step_rule;
  h.use_graph = c->opt.use_graph;
  h.lazyC = c->lazyC;
  h.compC = c->compC;
  h.world = c->sharded ? std::max(2, c->world) : 1;   // device: defer partial reductions when sharded
  h.repvars = c->fastC ? 1 : 0;                          // covering kinds: variables replicated
  h.partupd = ((c->sharded && c->fastC) || c->own) ? 1 : 0;   // their covering rows / owned rows are local
  h.ownrows = c->own;
  for (int i = 0; i < 32; ++i) h.aguess[i] = c->aguess[i];
  h.status = c->empty_cover ? ST_INFEASIBLE : ST_RUNNING;
  h.reason = c->empty_cover ? R_EMPTY_COVER : R_NONE;
  h.record = c->record;
  h.iter_stop = INT64_MAX;
  h.h_iter = 0;     // conditional handles are live only while the probe graph runs
  h.h_search = 0;
  CK(cudaMemcpyAsync(c->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, c->st));
  if (c->lazyC) CK(cudaMemsetAsync(c->act, 0, c->ntilesC * (MWU_CT / 32) * sizeof(uint32_t), c->st));
  else if (c->act) CK(cudaMemsetAsync(c->act, 0, ((c->E + 31) / 32 + 1) * sizeof(uint32_t), c->st));
  // x_i = eps / (n ||P_{:,i}||_inf)
  double cm = 1.0;
  const double* colmax = nullptr;
  if (c->kind == K_DENSEST) cm = h.invB;                          // P = O/D
  else if (c->kind == K_VCOVER || c->kind == K_DOMSET) cm = h.invB; // P = (1/M)1^T
  else if (c->kind == K_CSR) { if (c->pSing) cm = h.invB; else colmax = c->colmaxP; }
  init_x<<<rows_grid(c, c->n), MWU_NT, 0, c->st>>>(c->n, c->x, colmax, cm, c->ctl, c->part, c->counter,
                                                  c->ng > 0 ? c->ng : c->n);
  c->launches++;
  CKL();
  exchange(c);
  // y = P x, z = C x
  enqueue_forward(c, c->st, c->x, c->y, c->z, true);
  if (c->scatterP) allreduce_rows(c, c->y, c->own ? c->nLx : c->mP);   // sharded: partial rows of the local edges
  init_ext<<<rows_grid(c, c->mP + c->mC), MWU_NT, 0, c->st>>>(c->mP, c->y, c->mC, c->z, c->ctl, c->part, c->counter);
  c->launches++;
  exchange(c);
  enqueue_update(c, c->st, 0);
  exchange(c);
  CKL();
  sync(c);
  c->probe_active = true;
  c->bound = bound;
  c->eps = eps;
}

// The phases of one MWU iteration as stream work (host-driven loop and probe-graph capture
// alike).  Sharded runs add the exchange steps: on the graph path (NCCL) they are captured too.
void enqueue_col_step(mwu_ctx* c) {          // column + forward products
  enqueue_column(c, c->st);
  if (c->sharded && c->scatterP) {
    allreduce_rows(c, c->dy, c->own ? c->nLx : c->mP);   // the one vector exchange per iteration
    exchange(c);                             // column reductions (max d, sums, inactive rows)
    if (c->lazyC) {
      inactive_exact<<<rows_grid(c, c->E), MWU_NT, 0, c->st>>>(c->E, c->act, c->z, c->ctl, c->part, c->counter);
      exchange(c);
    }
  }
  enqueue_forward(c, c->st, c->d, c->dy, c->dz, false);
  if (c->own) exchange(c);                   // max d^(y) over the owned rows
}
void enqueue_search_pass(mwu_ctx* c) {       // one HBM pass of the step search
  enqueue_search(c, c->st);
  exchange(c);
}
void enqueue_update_phase(mwu_ctx* c) {      // y, z, weights of the accepted step
  enqueue_update(c, c->st, 1);
  exchange(c);                               // sharded covering kinds: S_C over local rows
}

// host-driven iteration (debug / lockstep parity path); alpha > 0 fixes the step
void host_iteration(mwu_ctx* c, double alpha) {
  push_field(c, &c->ctl->fixed_alpha, alpha > 0.0 ? alpha : 0.0);
  pull_ctl(c);
  if (c->hctl->status != ST_RUNNING) return;
  enqueue_col_step(c);
  CKL();
  for (int guard = 0; guard < 100000; ++guard) {
    pull_ctl(c);
    if (c->hctl->status != ST_RUNNING || !c->hctl->sactive) break;
    enqueue_search_pass(c);
    CKL();
  }
  enqueue_update_phase(c);
  CKL();
  sync(c);
  if (alpha > 0.0) push_field(c, &c->ctl->fixed_alpha, 0.0);
}

float run_loop(mwu_ctx* c, int64_t k) {
  pull_ctl(c);
  if (c->hctl->status != ST_RUNNING) return 0.f;
  const int64_t stop = (k < 0) ? INT64_MAX : c->hctl->t + k;
  if (k == 0) return 0.f;
  float ms = 0.f;
  if (c->opt.use_graph) {
    build_probe_graph(c);
    push_field(c, &c->ctl->iter_stop, stop);
    push_field(c, &c->ctl->h_iter, c->h_iter);
    push_field(c, &c->ctl->h_search, c->h_search);
    CK(cudaEventRecord(c->ev0, c->st));
    CK(cudaGraphLaunch(c->gexec, c->st));
    CK(cudaEventRecord(c->ev1, c->st));
    sync(c);
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    push_field(c, &c->ctl->h_iter, 0ull);
    push_field(c, &c->ctl->h_search, 0ull);
    push_field(c, &c->ctl->iter_stop, (int64_t)INT64_MAX);
  } else {
    CK(cudaEventRecord(c->ev0, c->st));
    for (;;) {
      pull_ctl(c);
      if (c->hctl->status != ST_RUNNING || c->hctl->t >= stop) break;
      host_iteration(c, 0.0);
    }
    CK(cudaEventRecord(c->ev1, c->st));
    sync(c);
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  }
  pull_ctl(c);
  if (c->hctl->nan_flag) throw MwuError{MWU_ERR_NUMERIC, "non-finite weight sums"};
  for (int i = 0; i < 32 && i < c->hctl->t; ++i) c->aguess[i] = c->hctl->ahist[i];
  return ms;
}

// Host-driven iterations with CUDA events around every phase (per-kernel roofline in bench.py).
// out[2p] = total ms, out[2p+1] = kernel launches, for p = column, step, search, update;
// out[8] = iterations run, out[9] = search passes.
void profile_iters(mwu_ctx* c, int64_t k, double* out) {
  for (int i = 0; i < 10; ++i) out[i] = 0.0;
  cudaEvent_t e[2];
  CK(cudaEventCreate(&e[0]));
  CK(cudaEventCreate(&e[1]));
  auto timed = [&](int p, auto&& fn) {
    const int64_t l0 = c->launches;
    CK(cudaEventRecord(e[0], c->st));
    fn();
    CK(cudaEventRecord(e[1], c->st));
    CK(cudaEventSynchronize(e[1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e[0], e[1]));
    out[2 * p] += ms;
    out[2 * p + 1] += (double)(c->launches - l0);
  };
  for (int64_t it = 0; it < k; ++it) {
    pull_ctl(c);
    if (c->hctl->status != ST_RUNNING) break;
    timed(0, [&] {
      enqueue_column(c, c->st);
      if (c->sharded && c->scatterP) {
        allreduce_rows(c, c->dy, c->own ? c->nLx : c->mP);
        exchange(c);
        if (c->lazyC) {
          inactive_exact<<<rows_grid(c, c->E), MWU_NT, 0, c->st>>>(c->E, c->act, c->z, c->ctl, c->part, c->counter);
          exchange(c);
        }
      }
    });
    timed(1, [&] {
      enqueue_forward(c, c->st, c->d, c->dy, c->dz, false);
      if (c->own) exchange(c);
    });
    for (int guard = 0; guard < 100000; ++guard) {
      pull_ctl(c);
      if (c->hctl->status != ST_RUNNING || !c->hctl->sactive) break;
      timed(2, [&] { enqueue_search(c, c->st); exchange(c); });
      out[9] += 1;
    }
    timed(3, [&] { enqueue_update(c, c->st, 1); exchange(c); });
    out[8] += 1;
  }
  cudaEventDestroy(e[0]);
  cudaEventDestroy(e[1]);
}

void flush(mwu_ctx* c) {
  if (c->lazyC) flush_pairs<<<rows_grid(c, c->E), MWU_NT, 0, c->st>>>(c->E, c->x, c->d, c->z, c->act, c->ctl);
  else if (c->act) flush_act1<<<rows_grid(c, c->E), MWU_NT, 0, c->st>>>(c->E, c->x, c->d, c->act, c->ctl);
  else flush_x<<<rows_grid(c, c->n), MWU_NT, 0, c->st>>>(c->n, c->x, c->d, c->ctl);
  CKL();
  int zero = 0;
  CK(cudaMemcpyAsync(&c->ctl->apply_prev, &zero, sizeof(int), cudaMemcpyHostToDevice, c->st));
  sync(c);
}

// sum / max of a device vector (ctl->scratch[0], [1])
void reduce_dev(mwu_ctx* c, const double* a, int64_t n, double& sum, double& mx) {
  reduce_vec<<<rows_grid(c, n), MWU_NT, 0, c->st>>>(n, a, c->ctl, c->part, c->counter);
  CKL();
  exchange(c);
  double s[2];
  CK(cudaMemcpyAsync(s, c->ctl->scratch, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  sum = s[0];
  mx = s[1];
}

// Q14 brackets (L, H) and witness x into xbest
void brackets(mwu_ctx* c, double eps, double& L, double& H) {
  double s, mx;
  if (c->kind == K_DENSEST) {
    L = (double)(c->Eg > 0 ? c->Eg : c->E) / (double)c->nprime;
    H = (double)c->maxdeg / 2.0;
    k_fill<<<rows_grid(c, c->n), MWU_NT, 0, c->st>>>(c->n, c->xbest, 0.5);
    CKL();
    return;
  }
  if (c->kind == K_VCOVER || c->kind == K_DOMSET) {
    L = (c->kind == K_VCOVER) ? (double)(c->Eg > 0 ? c->Eg : c->E) / (double)c->maxdeg
                              : (double)c->nv / (double)(c->maxdeg + 1);
    if (c->kind == K_VCOVER) k_fill_nonzero<<<rows_grid(c, c->n), MWU_NT, 0, c->st>>>(c->n, c->deg, c->xbest, 1.0);
    else k_fill<<<rows_grid(c, c->n), MWU_NT, 0, c->st>>>(c->n, c->xbest, 1.0);
    CKL();
    reduce_dev(c, c->xbest, c->n, s, mx);
    H = s;
    return;
  }
  if (c->kind == K_CSR && c->mode == MWU_PURE_COVERING) {
    reduce_dev(c, c->colsumC, c->n, s, mx);
    L = (double)c->mC / mx;
    CK(cudaMemcpyAsync(c->xbest, c->crecipC, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    reduce_dev(c, c->xbest, c->n, s, mx);
    H = s;
    return;
  }
  // packing: witness x0 / max(P x0) (x0 of P:272), H = sum_i max_j 1/p_ji
  Ctl& h = *c->hctl;
  memset(&h, 0, sizeof(Ctl));
  h.eps = eps; h.invB = 1.0; h.status = ST_RUNNING; h.iter_stop = INT64_MAX; h.world = c->sharded ? std::max(2, c->world) : 1;
  h.repvars = c->fastC ? 1 : 0;
  CK(cudaMemcpyAsync(c->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, c->st));
  init_x<<<rows_grid(c, c->n), MWU_NT, 0, c->st>>>(c->n, c->x, c->kind == K_CSR ? c->colmaxP : nullptr, 1.0, c->ctl,
                                                  c->part, c->counter, c->ng > 0 ? c->ng : c->n);
  CKL();
  exchange(c);
  enqueue_forward(c, c->st, c->x, c->y, c->z, true);
  if (c->scatterP) allreduce_rows(c, c->y, c->mP);
  reduce_dev(c, c->y, c->mP, s, mx);
  CK(cudaMemcpyAsync(c->tmp, &mx, sizeof(double), cudaMemcpyHostToDevice, c->st));
  scale_div<<<rows_grid(c, c->n), MWU_NT, 0, c->st>>>(c->n, c->x, c->xbest, c->tmp);
  CKL();
  sync(c);
  reduce_dev(c, c->xbest, c->n, s, mx);
  L = s;
  if (c->kind == K_MATCH) H = (double)(c->Eg > 0 ? c->Eg : c->E);
  else { reduce_dev(c, c->crecipP, c->n, s, mx); H = s; }
}

void finish_feasible(mwu_ctx* c) {
  // x_out = x / min(Cx) (Q15) with min(Cx) = s_C (cached)
  flush(c);
  scale_div<<<rows_grid(c, c->n), MWU_NT, 0, c->st>>>(c->n, c->x, c->xbest, &c->ctl->sC);
  CKL();
  sync(c);
}

void solve(mwu_ctx* c, double eps, int64_t max_iter, int32_t* outcome) {
  if (max_iter > 0) c->opt.max_iter = max_iter;
  mwu_stats& S = c->stats;
  const int64_t l0 = c->launches;
  S.probes = 0; S.iters_total = 0; S.search_evals = 0; S.search_passes = 0;
  S.near_tie_count = 0;
  for (int p = 0; p < 4; ++p) S.t_phase_ms[p] = 0.0;
  const double qnan = std::numeric_limits<double>::quiet_NaN();
  S.max_Px_raw = S.min_Cx_raw = S.max_Px = S.min_Cx = qnan;
  S.certificate = std::numeric_limits<double>::quiet_NaN();
  S.objective = std::numeric_limits<double>::quiet_NaN();
  cudaEvent_t s0, s1;                        // solve timing (run_loop uses ev0 / ev1 itself)
  CK(cudaEventCreate(&s0)); CK(cudaEventCreate(&s1));
  CK(cudaEventRecord(s0, c->st));
  float loop_ms_total = 0.f;
  struct Nvtx {                               // one NVTX range per probe (SURVEY §5 tracing)
    explicit Nvtx(const char* m) { nvtxRangePushA(m); }
    ~Nvtx() { nvtxRangePop(); }
  };
  Nvtx solve_range("mwu_solve");
  auto run_one = [&](double B) -> int {
    Nvtx probe_range("mwu_probe");
    probe_begin(c, B, eps);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, c->st));
    (void)run_loop(c, -1);
    CK(cudaEventRecord(b, c->st));
    CK(cudaEventSynchronize(b));
    float ms = 0; CK(cudaEventElapsedTime(&ms, a, b)); loop_ms_total += ms;
    cudaEventDestroy(a); cudaEventDestroy(b);
    pull_ctl(c);
    const Ctl& h = *c->hctl;
    S.probes++;
    S.iters_total += h.t;
    S.iters_last = h.t;
    S.search_evals += h.evals_total;
    S.search_passes += h.passes_total;
    S.near_tie_count += h.near_ties;
    for (int p = 0; p < 4; ++p) S.t_phase_ms[p] += h.tph[p] * 1e-6;
    S.outcome = h.status; S.reason = h.reason; S.eta = h.eta; S.alpha_last = h.alpha_last;
    if (h.status == ST_FEASIBLE) {
      S.certificate = h.sP / h.sC;      // rho = max y / min z (Q6)
      if (std::fabs(S.certificate - (1.0 + eps)) <= 1e-12 * (1.0 + eps)) S.near_tie_count++;
      S.max_Px_raw = h.sP; S.min_Cx_raw = h.sC;     // of the probe's final iterate
      S.max_Px = S.certificate; S.min_Cx = 1.0;    // of x_out = x / min(Cx) (Q15)
      finish_feasible(c);
    }
    return h.status;
  };
  if (c->kind == K_CSR && c->mode == MWU_MIXED) {
    const int st = run_one(1.0);
    if (st != ST_FEASIBLE) { flush(c); CK(cudaMemcpyAsync(c->xbest, c->x, c->n * sizeof(double), cudaMemcpyDeviceToDevice, c->st)); }
    S.bound = std::numeric_limits<double>::quiet_NaN();
    *outcome = st;
  } else {
    double L, H;
    brackets(c, eps, L, H);
    const double rt = c->opt.outer_rel_tol > 0 ? c->opt.outer_rel_tol : eps / 4.0;
    const int sense = (c->mode == MWU_PURE_PACKING) ? +1 : -1;
    bool any = false;
    double cert = std::numeric_limits<double>::quiet_NaN(), raw[2] = {qnan, qnan};
    while (H > (1.0 + rt) * L) {
      const double B = std::sqrt(L * H);
      const int st = run_one(B);
      const bool ok = (st == ST_FEASIBLE);
      if (ok) { any = true; cert = S.certificate; raw[0] = S.max_Px_raw; raw[1] = S.min_Cx_raw; }
      if ((ok && sense > 0) || (!ok && sense < 0)) L = B; else H = B;
    }
    S.certificate = any ? cert : std::numeric_limits<double>::quiet_NaN();
    S.max_Px_raw = raw[0]; S.min_Cx_raw = raw[1];
    S.max_Px = S.certificate; S.min_Cx = any ? 1.0 : qnan;
    S.bound = sense > 0 ? L : H;
    if (c->kind == K_DENSEST) S.objective = S.bound;
    else { double s, mx; reduce_dev(c, c->xbest, c->n, s, mx); S.objective = s; }
    S.outcome = ST_FEASIBLE;
    *outcome = ST_FEASIBLE;
  }
  CK(cudaEventRecord(s1, c->st));
  CK(cudaEventSynchronize(s1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, s0, s1));
  cudaEventDestroy(s0); cudaEventDestroy(s1);
  S.t_solve_ms = ms;
  S.t_loop_ms = loop_ms_total;
  S.kernel_launches = c->launches - l0;
  S.probe_graph = c->opt.use_graph ? 1 : 0;
}

void fill_static_stats(mwu_ctx* c) {
  mwu_stats& S = c->stats;
  S.n = c->n; S.m_P = c->pSing ? 1 : c->mP; S.m_C = c->cSing ? 1 : c->mC;
  S.nnz_P = c->nnzP; S.nnz_C = c->nnzC; S.empty_rows_dropped = c->empty_dropped;
  // algorithmic bytes per MWU iteration: structure of the two forward and two
  // transposed products + 32 B per variable (x r/w, d r/w) + 40 B per stored row
  double sfwd_tr = 0;
  const double rowsB = 40.0 * (double)(c->mP + c->mC);
  auto implicit = [&](int64_t rp_rows) { return 4.0 * (double)c->E + 8.0 * (double)(rp_rows + 1); };
  switch (c->kind) {
    case K_MATCH: sfwd_tr = 2 * implicit(c->nleft > 0 ? c->nleft : c->nv); break;
    case K_VCOVER: case K_DENSEST: sfwd_tr = 2 * implicit(c->nv); break;
    case K_DOMSET: sfwd_tr = 2 * (4.0 * c->nnzC + rp_bytes(c->nnzC) * (c->nv + 1)); break;
    case K_CSR: {
      auto side = [&](const Seg& A) {
        return A.rowptr ? 4.0 * A.nnz + rp_bytes(A.nnz) * (A.nrows + 1) + (A.val ? 8.0 * A.nnz : 0.0) : 0.0;
      };
      sfwd_tr = side(c->csrP) + side(c->cscP) + side(c->csrC) + side(c->cscC);
      break;
    }
  }
  c->bytes_alg = sfwd_tr + 32.0 * (double)c->n + rowsB;
  S.bytes_alg_per_iter = c->bytes_alg;
}

mwu_status fail(mwu_ctx* c, const MwuError& e) {
  if (c) {
    c->err = e.msg;
    if (e.st == MWU_ERR_CUDA) c->poisoned = true;
  }
  return e.st;
}

void destroy_ctx(mwu_ctx* c) {
  if (!c) return;
  if (c->comm) { delete c->comm; c->comm = nullptr; }
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->st) cudaStreamSynchronize(c->st);
  for (void* p : c->allocs) cudaFree(p);
  if (c->hctl) cudaFreeHost(c->hctl);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->evin) cudaEventDestroy(c->evin);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
}

}  // namespace

// ================================================================================== C ABI
extern "C" {

void mwu_default_options(mwu_options* o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->eta_factor = 10.0;
  o->max_iter = 5000;
  o->tol_prose = 1;
  o->max_evals = 200;
  o->outer_rel_tol = 0.0;
  o->use_graph = 1;
  o->bisect_depth = 3;
  o->device = -1;
  o->world = 1;
  o->rank = 0;
  o->nccl_id = nullptr;
  o->comm_group = nullptr;
  o->deterministic = 0;
  o->stream = nullptr;
  o->block_l = 0;
  o->block_r = 0;
  o->compact_cover = 1;
  o->step_rule = MWU_STEP_BINARY;
}

const char* mwu_last_error(const mwu_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

mwu_status mwu_create_graph(const mwu_graph* g, const mwu_options* opt, mwu_ctx** out) {
  if (!out) return MWU_ERR_ARG;
  *out = nullptr;
  if (!g || g->n_vertices <= 0 || g->n_edges < 0 || (g->n_edges > 0 && (!g->src || !g->dst)) ||
      g->kind < MWU_G_BMATCH || g->kind > MWU_G_DENSEST || g->n_vertices > INT32_MAX || g->n_edges > (int64_t(1) << 31)) {
    g_create_err = "mwu_create_graph: bad descriptor";
    return MWU_ERR_ARG;
  }
  mwu_ctx* c = new mwu_ctx();
  try {
    init_ctx_common(c, opt);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, c->st));
    build_graph_storage(c, g);
    switch (g->kind) {
      case MWU_G_BMATCH: case MWU_G_MATCH:
        if (g->n_edges == 0) throw MwuError{MWU_ERR_ARG, "matching needs at least one edge"};
        c->kind = K_MATCH; c->mode = MWU_PURE_PACKING; c->n = c->E; c->mP = c->nprime; c->cSing = 1;
        c->scatterP = c->opt.deterministic ? 0 : 1;
        c->nnzP = 2 * c->E; c->nnzC = c->E; c->empty_dropped = c->nv - c->nprime;
        break;
      case MWU_G_VCOVER:
        if (g->n_edges == 0) throw MwuError{MWU_ERR_ARG, "vertex cover needs at least one edge"};
        c->kind = K_VCOVER; c->mode = MWU_PURE_COVERING; c->n = c->nv; c->mC = c->E; c->pSing = 1;
        c->nnzC = 2 * c->E; c->nnzP = c->nv;
        c->fastC = c->opt.deterministic ? 0 : 1;
        break;
      case MWU_G_DOMSET:
        c->kind = K_DOMSET; c->mode = MWU_PURE_COVERING; c->n = c->nv; c->mC = c->nv; c->pSing = 1; c->nnzP = c->nv;
        c->fastC = c->opt.deterministic ? 0 : 1;
        if (c->fastC && c->nnzC > 0) {
          c->rowidC = dalloc<int32_t>(c, c->nnzC);
          k_row_ids<<<grid_for(c, c->nv), MWU_NT, 0, c->st>>>(c->nv, c->csrC.rowptr, (uint32_t*)c->rowidC);
          CKL();
        }
        break;
      case MWU_G_DENSEST:
        if (g->n_edges == 0) throw MwuError{MWU_ERR_ARG, "densest subgraph needs at least one edge"};
        c->kind = K_DENSEST; c->mode = MWU_MIXED; c->n = 2 * c->E; c->mP = c->nprime; c->mC = c->E;
        c->lazyC = (c->opt.deterministic || c->E >= (int64_t(1) << 31) - MWU_CT) ? 0 : 1;
        c->scatterP = c->lazyC;
        c->nnzP = 2 * c->E; c->nnzC = 2 * c->E; c->empty_dropped = c->nv - c->nprime;
        break;
    }
    // sharded bipartite matching: right rows owned by one rank each, only the left rows exchanged
    c->own = (c->sharded && c->kind == K_MATCH && c->scatterP && c->nleft > 0) ? 1 : 0;
    if (c->scatterP) build_blocked_order(c);
    fill_static_stats(c);                    // global sizes
    if (c->sharded && !c->scatterP && !c->fastC)
      throw MwuError{MWU_ERR_ARG, "multi-GPU sharding needs a graph kind with deterministic = 0"};
    localize(c);
    // vcover / domset, one rank: the forward product compacts the covering rows with d^(z) > 0
    // for the search passes (sharded runs keep the dense rows: their step reductions are not exchanged)
    c->compC = ((c->kind == K_VCOVER || c->kind == K_DOMSET) && c->fastC && !c->sharded && c->mC > 0 &&
                c->mC < (int64_t(1) << 31) - MWU_CT && c->opt.compact_cover) ? 1 : 0;
    alloc_vectors(c);
    {                                        // exchange flags for reductions before a probe
      Ctl& h = *c->hctl;
      memset(&h, 0, sizeof(Ctl));
      h.world = c->sharded ? std::max(2, c->world) : 1;
      h.repvars = c->fastC ? 1 : 0;
      h.partupd = ((c->sharded && c->fastC) || c->own) ? 1 : 0;
      h.ownrows = c->own;
      CK(cudaMemcpyAsync(c->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, c->st));
      sync(c);
    }
    CK(cudaEventRecord(b, c->st));
    CK(cudaEventSynchronize(b));
    float ms = 0; CK(cudaEventElapsedTime(&ms, a, b));
    c->stats.t_create_ms = ms;
    cudaEventDestroy(a); cudaEventDestroy(b);
    sync(c);
  } catch (const MwuError& e) {
    g_create_err = e.msg;
    destroy_ctx(c);
    return e.st;
  }
  *out = c;
  return MWU_OK;
}

mwu_status mwu_create_gmatch(const mwu_graph* g, const double* lb, const double* ub, const mwu_options* opt,
                             mwu_ctx** out) {
  if (!out) return MWU_ERR_ARG;
  *out = nullptr;
  if (!g || !lb || !ub || g->n_vertices <= 0 || g->n_edges <= 0 || !g->src || !g->dst || g->n_vertices > INT32_MAX ||
      g->n_edges > INT32_MAX) {
    g_create_err = "mwu_create_gmatch: bad descriptor or bounds";
    return MWU_ERR_ARG;
  }
  mwu_ctx* c = new mwu_ctx();
  try {
    init_ctx_common(c, opt);
    if (c->world > 1 || c->sharded) throw MwuError{MWU_ERR_ARG, "generalized matching runs on one rank"};
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, c->st));
    mwu_graph gv = *g;
    gv.kind = MWU_G_VCOVER;                    // validation + vertex -> incident-slot CSR (sorted slots)
    build_graph_storage(c, &gv);
    const int64_t nv = c->nv, E = c->E;
    double* dlb = dalloc<double>(c, nv);
    double* dub = dalloc<double>(c, nv);
    CK(cudaMemcpyAsync(dlb, lb, nv * sizeof(double), cudaMemcpyDefault, c->st));
    CK(cudaMemcpyAsync(dub, ub, nv * sizeof(double), cudaMemcpyDefault, c->st));
    uint8_t* fp = talloc<uint8_t>(nv);
    uint8_t* fc = talloc<uint8_t>(nv);
    unsigned int* err = talloc<unsigned int>(1);
    CK(cudaMemsetAsync(err, 0, sizeof(unsigned int), c->st));
    k_gm_flags<<<grid_for(c, nv), MWU_NT, 0, c->st>>>(nv, dlb, dub, fp, fc, err);
    CKL();
    const unsigned int eb = read_scalar(c, err);
    tfree(err);
    if (eb) throw MwuError{MWU_ERR_ARG, "mwu_create_gmatch: need 0 <= lb <= ub, ub > 0, lb finite"};
    c->kind = K_CSR; c->mode = MWU_MIXED; c->n = E;
    build_gm_side(c, fp, dub, c->csrP);        // P = diag(1/u) M over the vertices with finite u
    build_gm_side(c, fc, dlb, c->csrC);        // C = diag(1/l) M over the vertices with l > 0
    tfree(fp); tfree(fc);
    if (c->csrP.nrows == 0 || c->csrC.nrows == 0)
      throw MwuError{MWU_ERR_ARG, "mwu_create_gmatch: needs a finite upper bound and a positive lower bound somewhere"};
    finish_csr_packing(c, E);
    finish_csr_covering(c, E);
    alloc_vectors(c);
    fill_static_stats(c);
    CK(cudaEventRecord(b, c->st));
    CK(cudaEventSynchronize(b));
    float ms = 0; CK(cudaEventElapsedTime(&ms, a, b));
    c->stats.t_create_ms = ms;
    cudaEventDestroy(a); cudaEventDestroy(b);
  } catch (const MwuError& e) {
    g_create_err = e.msg;
    destroy_ctx(c);
    return e.st;
  }
  *out = c;
  return MWU_OK;
}

mwu_status mwu_create_csr(const mwu_csr* P, const mwu_csr* C, mwu_mode mode, const mwu_options* opt, mwu_ctx** out) {
  if (!out) return MWU_ERR_ARG;
  *out = nullptr;
  const bool needP = (mode == MWU_MIXED || mode == MWU_PURE_PACKING);
  const bool needC = (mode == MWU_MIXED || mode == MWU_PURE_COVERING);
  if ((needP && !P) || (needC && !C) || (mode < MWU_MIXED || mode > MWU_PURE_COVERING)) {
    g_create_err = "mwu_create_csr: missing matrix for this mode";
    return MWU_ERR_ARG;
  }
  const int64_t n = needP ? P->cols : C->cols;
  if (needP && needC && P->cols != C->cols) { g_create_err = "mwu_create_csr: P.cols != C.cols"; return MWU_ERR_ARG; }
  if (n <= 0 || n > INT32_MAX) { g_create_err = "mwu_create_csr: bad number of columns"; return MWU_ERR_ARG; }
  mwu_ctx* c = new mwu_ctx();
  try {
    init_ctx_common(c, opt);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, c->st));
    c->kind = K_CSR; c->mode = mode; c->n = n;
    if (needP) {
      copy_csr_checked(c, P, c->csrP, n, "P");
      finish_csr_packing(c, n);
    } else {
      c->pSing = 1; c->nnzP = n;
    }
    if (needC) {
      copy_csr_checked(c, C, c->csrC, n, "C");
      finish_csr_covering(c, n);
    } else {
      c->cSing = 1; c->nnzC = n;
    }
    alloc_vectors(c);
    fill_static_stats(c);
    CK(cudaEventRecord(b, c->st));
    CK(cudaEventSynchronize(b));
    float ms = 0; CK(cudaEventElapsedTime(&ms, a, b));
    c->stats.t_create_ms = ms;
    cudaEventDestroy(a); cudaEventDestroy(b);
  } catch (const MwuError& e) {
    g_create_err = e.msg;
    destroy_ctx(c);
    return e.st;
  }
  *out = c;
  return MWU_OK;
}

#define GUARD(c)                                          \
  if (!(c)) return MWU_ERR_ARG;                           \
  if ((c)->poisoned) return MWU_ERR_CUDA;

mwu_status mwu_solve(mwu_ctx* c, double eps, int64_t max_iter, int32_t* outcome) {
  GUARD(c);
  int32_t dummy;
  if (!outcome) outcome = &dummy;
  try {
    solve(c, eps, max_iter, outcome);
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_get_x(mwu_ctx* c, double* x, int64_t len) {
  GUARD(c);
  const int64_t n = c->ng > 0 ? c->ng : c->n;
  if (!x || len != n) { c->err = "mwu_get_x: len must equal n"; return MWU_ERR_ARG; }
  try {
    wait_caller(c);
    const double* src = unperm(c, c->xbest, c->kind == K_DENSEST ? 2 : 1);
    CK(cudaMemcpyAsync(x, src, n * sizeof(double), cudaMemcpyDefault, c->st));
    sync(c);
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_get_stats(mwu_ctx* c, mwu_stats* out) {
  GUARD(c);
  if (!out) return MWU_ERR_ARG;
  *out = c->stats;
  return MWU_OK;
}

void mwu_destroy(mwu_ctx* c) { destroy_ctx(c); }

mwu_status mwu_probe_begin(mwu_ctx* c, double bound, double eps) {
  GUARD(c);
  try {
    if (c->kind == K_CSR && c->mode == MWU_MIXED) bound = 1.0;
    probe_begin(c, bound, eps);
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_step(mwu_ctx* c, double alpha, int32_t* state) {
  GUARD(c);
  if (!c->probe_active) { c->err = "mwu_step: no active probe"; return MWU_ERR_STATE; }
  try {
    host_iteration(c, alpha);
    pull_ctl(c);
    if (c->hctl->nan_flag) throw MwuError{MWU_ERR_NUMERIC, "non-finite weight sums"};
    if (state) *state = c->hctl->status;
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_run_iters(mwu_ctx* c, int64_t k, int32_t* state) {
  GUARD(c);
  if (!c->probe_active) { c->err = "mwu_run_iters: no active probe"; return MWU_ERR_STATE; }
  try {
    const int64_t l0 = c->launches;
    c->stats.t_loop_ms = run_loop(c, k);
    pull_ctl(c);
    if (state) *state = c->hctl->status;
    // probe-cumulative diagnostics of the current probe
    c->stats.near_tie_count = c->hctl->near_ties;
    for (int p = 0; p < 4; ++p) c->stats.t_phase_ms[p] = c->hctl->tph[p] * 1e-6;
    c->stats.kernel_launches = c->launches - l0;
    c->stats.probe_graph = c->opt.use_graph ? 1 : 0;
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_run_probe(mwu_ctx* c, int32_t* state) { return mwu_run_iters(c, -1, state); }

int64_t mwu_vec_len(mwu_ctx* c, int which) {
  if (!c) return 0;
  const int64_t n = c->ng > 0 ? c->ng : c->n, mC = c->mCg > 0 ? c->mCg : c->mC;   // whole vectors
  switch (which) {
    case MWU_VEC_X: case MWU_VEC_D: case MWU_VEC_XBEST: return n;
    case MWU_VEC_G: case MWU_VEC_H: return c->record ? n : 0;
    case MWU_VEC_Y: case MWU_VEC_DY: case MWU_VEC_WP: return c->pSing ? 1 : c->mP;
    case MWU_VEC_Z: case MWU_VEC_DZ: case MWU_VEC_WC: return c->cSing ? 1 : mC;
  }
  return 0;
}

mwu_status mwu_get_vec(mwu_ctx* c, int which, double* out, int64_t len) {
  GUARD(c);
  const int64_t L = mwu_vec_len(c, which);
  if (!out || L <= 0 || len != L) { c->err = "mwu_get_vec: unknown vector or wrong length"; return MWU_ERR_ARG; }
  try {
    wait_caller(c);
    pull_ctl(c);
    const Ctl h = *c->hctl;
    const double* src = nullptr;
    double scal = 0;
    bool use_scal = false;
    switch (which) {
      case MWU_VEC_X: flush(c); src = c->x; break;
      case MWU_VEC_D:
        if (c->lazyC) {
          d_from_act<<<rows_grid(c, c->E), MWU_NT, 0, c->st>>>(c->E, c->d, c->act, c->tmp, nullptr);
          CKL();
          src = c->tmp;
        } else if (c->act) {
          d_from_act1<<<rows_grid(c, c->E), MWU_NT, 0, c->st>>>(c->E, c->d, c->act, c->tmp);
          CKL();
          src = c->tmp;
        } else src = c->d;
        break;
      case MWU_VEC_XBEST: src = c->xbest; break;
      case MWU_VEC_G: src = c->gdbg; break;
      case MWU_VEC_H: src = c->hdbg; break;
      case MWU_VEC_Y: if (c->pSing) { scal = h.yS; use_scal = true; } else src = c->y; break;
      case MWU_VEC_DY: if (c->pSing) { scal = h.dyS; use_scal = true; } else src = c->dy; break;
      case MWU_VEC_Z:
        if (c->cSing) { scal = h.zS; use_scal = true; }
        else { if (c->lazyC) flush(c); src = c->z; }
        break;
      case MWU_VEC_DZ:
        if (c->cSing) { scal = h.dzS; use_scal = true; }
        else if (c->lazyC) {
          d_from_act<<<rows_grid(c, c->E), MWU_NT, 0, c->st>>>(c->E, c->d, c->act, nullptr, c->tmp);
          CKL();
          src = c->tmp;
        }
        else src = c->dz;
        break;
      case MWU_VEC_WP:
        if (c->pSing) { scal = 1.0; use_scal = true; }
        else { scale_div<<<rows_grid(c, c->mP), MWU_NT, 0, c->st>>>(c->mP, c->u, c->tmp, &c->ctl->SP); CKL(); src = c->tmp; }
        break;
      case MWU_VEC_WC:
        if (c->cSing) { scal = 1.0; use_scal = true; }
        else if (c->lazyC) {
          flush(c);
          wc_from_z<<<rows_grid(c, c->mC), MWU_NT, 0, c->st>>>(c->mC, c->z, c->tmp, c->ctl);
          CKL();
          src = c->tmp;
        }
        else { scale_div<<<rows_grid(c, c->mC), MWU_NT, 0, c->st>>>(c->mC, c->v, c->tmp, &c->ctl->SC); CKL(); src = c->tmp; }
        break;
    }
    if (c->own && !use_scal && (which == MWU_VEC_Y || which == MWU_VEC_DY || which == MWU_VEC_WP)) {
      // every rank's own rows (replicated prefix from rank 0): zeros elsewhere, summed over ranks
      own_mask<<<rows_grid(c, c->mP), MWU_NT, 0, c->st>>>(c->mP, src, c->tmp, c->nLx, c->R0, c->R1, c->rank == 0);
      CKL();
      allreduce_rows(c, c->tmp, c->mP);
      src = c->tmp;
    }
    if (c->rowperm && !use_scal && (which == MWU_VEC_Y || which == MWU_VEC_DY || which == MWU_VEC_WP)) {
      k_unperm<<<grid_for(c, c->mP), MWU_NT, 0, c->st>>>(c->mP, c->rowperm, src, c->tmp2, 1);   // vertex order
      CKL();
      src = c->tmp2;
    }
    if (!c->perm && c->sharded && !use_scal && (which == MWU_VEC_Z || which == MWU_VEC_DZ || which == MWU_VEC_WC))
      src = gather_full(c, src, 1);          // covering rows of every rank (vcover / domset)
    if (c->perm && !use_scal) {              // internal (L2-blocked) edge order -> original (Q29)
      const int w = (c->kind == K_DENSEST) ? 2 : 1;
      if (which == MWU_VEC_X || which == MWU_VEC_D || which == MWU_VEC_XBEST || which == MWU_VEC_G ||
          which == MWU_VEC_H)
        src = unperm(c, src, w);
      else if (c->kind == K_DENSEST && (which == MWU_VEC_Z || which == MWU_VEC_DZ || which == MWU_VEC_WC))
        src = unperm(c, src, 1);
    }
    if (use_scal) CK(cudaMemcpyAsync(out, &scal, sizeof(double), cudaMemcpyDefault, c->st));
    else CK(cudaMemcpyAsync(out, src, L * sizeof(double), cudaMemcpyDefault, c->st));
    sync(c);
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_set_stream(mwu_ctx* c, void* stream) {
  GUARD(c);
  c->ust = (cudaStream_t)stream;
  c->opt.stream = stream;
  return MWU_OK;
}

mwu_status mwu_set_record(mwu_ctx* c, int on) {
  GUARD(c);
  try {
    if (on && !c->gdbg) { c->gdbg = dalloc<double>(c, c->n); c->hdbg = dalloc<double>(c, c->n); }
    if (on != c->record && c->graph_ok) {  // epilogue pointers are baked into the graph
      cudaGraphExecDestroy(c->gexec); cudaGraphDestroy(c->graph);
      c->gexec = nullptr; c->graph = nullptr; c->graph_ok = false;
    }
    c->record = on ? 1 : 0;
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_get_structure(mwu_ctx* c, int which, void* out, int64_t* bytes) {
  GUARD(c);
  if (!bytes) return MWU_ERR_ARG;
  const void* src = nullptr;
  int64_t nb = 0;
  switch (which) {
    case MWU_ST_INC_ROWPTR: src = c->inc_all.rowptr; nb = c->inc_all.rowptr ? (c->nv + 1) * 8 : 0; break;
    case MWU_ST_INC_SLOTS: src = c->inc_all.idx; nb = c->inc_all.idx ? 2 * c->E * 4 : 0; break;
    case MWU_ST_DEGREE: src = c->deg; nb = c->deg ? c->nv * 4 : 0; break;
    case MWU_ST_PROW_OF_VERTEX: src = c->prow; nb = c->prow ? c->nv * 4 : 0; break;
    case MWU_ST_C_ROWPTR: src = c->csrC.rowptr; nb = c->csrC.rowptr ? (c->csrC.nrows + 1) * 8 : 0; break;
    case MWU_ST_C_COLIDX: src = c->csrC.idx; nb = c->csrC.rowptr ? c->csrC.nnz * 4 : 0; break;
    case MWU_ST_CT_ROWPTR: src = c->cscC.rowptr; nb = c->cscC.rowptr ? (c->cscC.nrows + 1) * 8 : 0; break;
    case MWU_ST_CT_ROWIDX: src = c->cscC.idx; nb = c->cscC.rowptr ? c->cscC.nnz * 4 : 0; break;
    case MWU_ST_PT_ROWPTR: src = c->cscP.rowptr; nb = c->cscP.rowptr ? (c->cscP.nrows + 1) * 8 : 0; break;
    case MWU_ST_PT_ROWIDX: src = c->cscP.idx; nb = c->cscP.rowptr ? c->cscP.nnz * 4 : 0; break;
    case MWU_ST_P_ROWPTR: src = c->csrP.rowptr; nb = c->csrP.rowptr ? (c->csrP.nrows + 1) * 8 : 0; break;
    case MWU_ST_P_COLIDX: src = c->csrP.idx; nb = c->csrP.rowptr ? c->csrP.nnz * 4 : 0; break;
    default: break;
  }
  if (!src || nb <= 0) {
    if (nb == 0 && src) { *bytes = 0; return MWU_OK; }
    c->err = "mwu_get_structure: structure not present for this kind";
    return MWU_ERR_ARG;
  }
  if (*bytes < nb || !out) { *bytes = nb; c->err = "mwu_get_structure: buffer too small"; return MWU_ERR_ARG; }
  try {
    wait_caller(c);
    CK(cudaMemcpyAsync(out, src, nb, cudaMemcpyDefault, c->st));
    sync(c);
  } catch (const MwuError& e) { return fail(c, e); }
  *bytes = nb;
  return MWU_OK;
}

mwu_status mwu_get_scalars(mwu_ctx* c, double* o) {
  GUARD(c);
  if (!o) return MWU_ERR_ARG;
  try {
    pull_ctl(c);
    const Ctl& h = *c->hctl;
    o[0] = h.eta; o[1] = h.sigma; o[2] = h.sP; o[3] = h.SP; o[4] = h.sC; o[5] = h.SC;
    o[6] = (double)h.t; o[7] = h.alpha_last; o[8] = (double)h.evals_total; o[9] = (double)h.passes_total;
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_profile_iters(mwu_ctx* c, int64_t k, double* out10) {
  GUARD(c);
  if (!out10) return MWU_ERR_ARG;
  if (!c->probe_active) { c->err = "mwu_profile_iters: no active probe"; return MWU_ERR_STATE; }
  try {
    profile_iters(c, k, out10);
  } catch (const MwuError& e) { return fail(c, e); }
  return MWU_OK;
}

mwu_status mwu_get_unique_id(void* out128) {
  if (!out128) return MWU_ERR_ARG;
  try {
    NcclLib& L = NcclLib::get();
    NcclUid id;
    if (L.getUniqueId(&id) != 0) { g_create_err = "ncclGetUniqueId failed"; return MWU_ERR_NCCL; }
    memcpy(out128, id.internal, 128);
  } catch (const std::exception& e) {
    g_create_err = e.what();
    return MWU_ERR_NCCL;
  }
  return MWU_OK;
}

mwu_status mwu_shard_range(int64_t n, int world, int rank, int64_t* e0, int64_t* e1) {
  if (!e0 || !e1 || n < 0 || world < 1 || rank < 0 || rank >= world) return MWU_ERR_ARG;
  shard_range(n, world, rank, *e0, *e1);
  return MWU_OK;
}

mwu_status mwu_simgroup_create(int world, void** group) {
  if (!group || world < 1) return MWU_ERR_ARG;
  *group = new SimGroup(world);
  return MWU_OK;
}

void mwu_simgroup_destroy(void* group) { delete (SimGroup*)group; }

}  // extern "C"
