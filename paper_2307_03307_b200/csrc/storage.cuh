// storage.cuh — device-side structure build (one-off per context, bit-exact integer work).
//
//  * graph kinds: edge list -> degrees, vertex -> incident-slot CSR (slot 2e+b, sorted within
//    a vertex by a stable radix sort), compacted packing rows without isolated vertices (Q17),
//    endpoint row ids; DOMSET: I + A as CSR via a 64-bit key sort.
//  * CSR kinds: validation, empty-row compaction of P, CSC copies of P and C (stable sort by
//    column keeps rows ascending inside a column), column maxima of P.
//  * tile plans for the segmented kernels (load balance on power-law degrees).
#pragma once
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include "common.cuh"

namespace mwu {

__global__ void k_tile_rows(const int64_t* rowptr, int64_t nrows, int64_t ntiles, int64_t* tile_row) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= ntiles; k += (int64_t)gridDim.x * blockDim.x) {
    if (k == ntiles) { tile_row[k] = nrows; continue; }
    const int64_t target = k * (int64_t)MWU_TILE;
    int64_t lo = 0, hi = nrows;                 // first r in [0,nrows) with rowptr[r] >= target
    while (lo < hi) { int64_t m = (lo + hi) >> 1; if (rowptr[m] >= target) hi = m; else lo = m + 1; }
    tile_row[k] = lo;
  }
}

__global__ void k_long_flags(const int64_t* rowptr, int64_t nrows, uint8_t* flag) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x)
    flag[r] = (rowptr[r + 1] - rowptr[r]) > MWU_TILE;
}

__global__ void k_long_nchunks(const int64_t* rowptr, const int64_t* rows, int64_t nlong, int64_t* nch) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < nlong; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[l];
    nch[l] = (rowptr[r + 1] - rowptr[r] + MWU_LCH - 1) / MWU_LCH;
  }
}

// ---------------------------------------------------------------- graph build kernels
// error bits: 1 id out of range, 2 self-loop, 4 bipartite side violation, 8 duplicate edge
__global__ void k_validate_edges(int64_t E, const int32_t* src, const int32_t* dst, int64_t nv, int64_t nleft,
                                 int bip, unsigned int* err, unsigned long long* keys) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], b = dst[e];
    unsigned int f = 0;
    if (a < 0 || b < 0 || a >= nv || b >= nv) f |= 1u;
    if (a == b) f |= 2u;
    if (bip && ((a < nleft) == (b < nleft))) f |= 4u;
    if (f) atomicOr(err, f);
    const unsigned long long lo = (unsigned long long)(a < b ? a : b), hi = (unsigned long long)(a < b ? b : a);
    keys[e] = (lo << 32) | (hi & 0xffffffffull);
  }
}

__global__ void k_adjacent_dups(int64_t n, const unsigned long long* keys, unsigned int* err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (keys[i] == keys[i - 1]) atomicOr(err, 8u);
}

__global__ void k_degree(int64_t E, const int32_t* src, const int32_t* dst, int32_t* deg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(deg + src[e], 1);
    atomicAdd(deg + dst[e], 1);
  }
}

__global__ void k_slot_keys(int64_t E, const int32_t* src, const int32_t* dst, uint32_t* keys, uint32_t* vals) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < 2 * E; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = s >> 1;
    keys[s] = (uint32_t)((s & 1) ? dst[e] : src[e]);
    vals[s] = (uint32_t)s;
  }
}

template <class T>
__global__ void k_to_int64(int64_t n, const T* in, int64_t* out, int64_t add) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)in[i] + add;
}

__global__ void k_nonzero_flags(int64_t n, const int32_t* deg, int64_t* flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = deg[i] > 0 ? 1 : 0;
}

// prow[v] = compacted row id (exclusive scan of the nonzero flags) or -1; rowptrP[prow] = rowptr[v]
__global__ void k_compact_rows(int64_t nv, const int32_t* deg, const int64_t* scan, const int64_t* rowptr_all,
                               int32_t* prow, int64_t* rowptrP) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    if (deg[v] > 0) { prow[v] = (int32_t)scan[v]; rowptrP[scan[v]] = rowptr_all[v]; }
    else prow[v] = -1;
  }
}

__global__ void k_map_endpoints(int64_t E, const int32_t* src, const int32_t* dst, const int32_t* prow,
                                int32_t* srow, int32_t* drow) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    srow[e] = prow[src[e]];
    drow[e] = prow[dst[e]];
  }
}

// L2-blocked edge order (the paper's CSB blocking, at L2 scale): key = (block pair
// (src >> BL, dst >> BR), src & maskL, dst & maskR).  A wide src block (2^BL vertices) stays
// L2-resident (its gathered u and scattered d^(y) slices) while the narrow dst blocks (2^BR)
// stream past it, so each random-access slice is fetched ~once per src block instead of once
// per access.
// vrow: vertex -> packing row (the blocks are row ranges of the gathered / scattered vectors)
__global__ void k_block_keys(int64_t E, const int32_t* src, const int32_t* dst, const int32_t* vrow, int nbR,
                             int BL, int BR, unsigned long long* keys, uint32_t* vals) {
  const unsigned long long mL = (1ull << BL) - 1ull, mR = (1ull << BR) - 1ull;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long a = (unsigned long long)vrow[src[e]], b = (unsigned long long)vrow[dst[e]];
    const unsigned long long pair = (a >> BL) * (unsigned long long)nbR + (b >> BR);
    keys[e] = (pair << (BL + BR)) | ((a & mL) << BR) | (b & mR);
    vals[e] = (uint32_t)e;
  }
}

// Owner-partitioned destination rows of a sharded bipartite matching: right
// rows [ob[r], ob[r+1]) belong to rank r (ob[0] = first right row); key = (owner, dst block
// within the owner's rows, src row, dst row), so each rank's edges are one contiguous range and
// no other rank touches its right rows.
__global__ void k_block_keys_own(int64_t E, const int32_t* src, const int32_t* dst, const int32_t* vrow,
                                 const int64_t* ob, int W, int nbR, int BL, int BR, unsigned long long* keys,
                                 uint32_t* vals) {
  const unsigned long long mR = (1ull << BR) - 1ull;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = vrow[src[e]], q = vrow[dst[e]];          // left rows come first: a left, b right
    const unsigned long long a = (unsigned long long)(p < q ? p : q);
    const int64_t b = p < q ? q : p;
    int r = 0;
    while (r + 1 < W && b >= ob[r + 1]) ++r;
    const unsigned long long rel = (unsigned long long)(b - ob[0] < 0 ? 0 : b - ob[r]);
    const unsigned long long blk = (unsigned long long)r * (unsigned long long)nbR + (rel >> BR);
    keys[e] = (blk << (BL + BR)) | (a << BR) | (rel & mR);
    vals[e] = (uint32_t)e;
  }
}
// srow = the left endpoint's row, drow = the right endpoint's (rows of the left side come first)
__global__ void k_orient(int64_t E, int32_t* srow, int32_t* drow) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = srow[i], b = drow[i];
    if (a > b) { srow[i] = b; drow[i] = a; }
  }
}
// number of non-isolated left vertices (their rows come first in the degree order)
__global__ void k_count_left(int64_t nleft, const int32_t* deg, unsigned long long* out) {
  unsigned long long k = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nleft; v += (int64_t)gridDim.x * blockDim.x)
    k += deg[v] > 0 ? 1ull : 0ull;
  for (int o = 16; o > 0; o >>= 1) k += __shfl_down_sync(0xffffffffu, k, o);
  if ((threadIdx.x & 31) == 0 && k) atomicAdd(out, k);
}
// degrees of the right rows in row order: rd[i] = deg[vertex of row nL + i]
__global__ void k_right_deg(int64_t nR, int64_t nL, const uint32_t* vsorted, const int32_t* deg, int64_t* rd) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nR; i += (int64_t)gridDim.x * blockDim.x)
    rd[i] = deg[vsorted[nL + i]];
}
// out[r] = first i with cum[i] >= target_r = r * total / W (r = 1 .. W-1), by binary search
__global__ void k_owner_bounds(const int64_t* cum, int64_t n, int64_t total, int W, int64_t* out) {
  const int r = threadIdx.x + 1;
  if (r >= W) return;
  const int64_t t = (int64_t)((__int128)total * r / W);
  int64_t lo = 0, hi = n;
  while (lo < hi) { const int64_t m = (lo + hi) / 2; if (cum[m] >= t) hi = m; else lo = m + 1; }
  out[r] = lo;
}
// out[r] = first internal edge whose dst row is >= ob[r] (owners ascend along the internal order)
__global__ void k_owner_edges(const int32_t* drow, int64_t E, const int64_t* ob, int W, int64_t* out) {
  const int r = threadIdx.x;
  if (r > W) return;
  if (r == 0) { out[0] = 0; return; }
  if (r == W) { out[W] = E; return; }
  int64_t lo = 0, hi = E;
  while (lo < hi) { const int64_t m = (lo + hi) / 2; if (drow[m] >= ob[r]) hi = m; else lo = m + 1; }
  out[r] = lo;
}

// degree-descending row order (hot rows of power-law graphs cluster in a small, L2-resident
// prefix of the packing-row vectors): key = (~deg, v)
// (bipartite: the left side's rows first, so a source sweep never touches right-side rows)
__global__ void k_deg_keys(int64_t nv, const int32_t* deg, int64_t nleft, unsigned long long* keys, uint32_t* vals) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    // isolated vertices last (rows [0, n') are the non-isolated ones), then side, then degree
    const unsigned long long iso = deg[v] == 0 ? (1ull << 63) : 0ull;
    const unsigned long long side = (nleft > 0 && v >= nleft) ? (1ull << 62) : 0ull;
    keys[v] = iso | side | ((unsigned long long)(0x3fffffffu - ((uint32_t)deg[v] & 0x3fffffffu)) << 32) |
              (unsigned long long)v;
    vals[v] = (uint32_t)v;
  }
}
// sorted vertices -> fast row ids: prowf[v_i] = i (i < n'), rowperm[i] = prow[v_i]
__global__ void k_deg_rows(int64_t nprime, const uint32_t* vsorted, const int32_t* prow, int32_t* prowf,
                           uint32_t* rowperm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nprime; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = vsorted[i];
    prowf[v] = (int32_t)i;
    rowperm[i] = (uint32_t)prow[v];
  }
}

__global__ void k_map_endpoints_perm(int64_t E, const uint32_t* perm, const int32_t* src, const int32_t* dst,
                                     const int32_t* prow, int32_t* srow, int32_t* drow) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = perm[i];
    srow[i] = prow[src[e]];
    drow[i] = prow[dst[e]];
  }
}

// internal (blocked) order -> original order: out[perm[i] * w + b] = in[i * w + b]
__global__ void k_unperm(int64_t E, const uint32_t* perm, const double* in, double* out, int w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (int64_t)perm[i] * w;
    for (int b = 0; b < w; ++b) out[o + b] = in[i * w + b];
  }
}

__global__ void k_domset_keys(int64_t nv, int64_t E, const int32_t* src, const int32_t* dst, unsigned long long* keys) {
  const int64_t tot = nv + 2 * E;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long r, c;
    if (i < nv) { r = i; c = i; }
    else {
      const int64_t s = i - nv, e = s >> 1;
      if (s & 1) { r = (unsigned long long)dst[e]; c = (unsigned long long)src[e]; }
      else { r = (unsigned long long)src[e]; c = (unsigned long long)dst[e]; }
    }
    keys[i] = (r << 32) | c;
  }
}

__global__ void k_low32(int64_t n, const unsigned long long* keys, uint32_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)(keys[i] & 0xffffffffull);
}

// ---------------------------------------------------------------- CSR build kernels
// error bits: 16 column out of range / not strictly increasing, 32 negative or non-finite value
__global__ void k_validate_csr(int64_t rows, int64_t cols, const int64_t* rowptr, const uint32_t* col,
                               const double* val, unsigned int* err, int32_t* rowlen_nz) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = rowptr[r], b = rowptr[r + 1];
    unsigned int f = 0;
    int64_t prev = -1;
    for (int64_t k = a; k < b; ++k) {
      const int64_t cc = (int64_t)(int32_t)col[k];
      if (cc < 0 || cc >= cols || cc <= prev) f |= 16u;
      prev = cc;
      if (val && !(val[k] >= 0.0 && isfinite(val[k]))) f |= 32u;
    }
    if (f) atomicOr(err, f);
    rowlen_nz[r] = (int32_t)(b - a);
  }
}

__global__ void k_row_ids(int64_t rows, const int64_t* rowptr, uint32_t* rid) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) rid[k] = (uint32_t)r;
}

__global__ void k_iota64(int64_t n, uint64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = i;
}

__global__ void k_col_count(int64_t nnz, const uint32_t* col, int64_t* cnt) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)(cnt + col[k]), 1ull);
}

__global__ void k_gather_csc(int64_t nnz, const uint64_t* perm, const uint32_t* rid, const double* val,
                             uint32_t* rowT, double* valT) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t p = perm[k];
    rowT[k] = rid[p];
    if (val) valT[k] = val[p];
  }
}

// per column: max value (||P_{:,i}||_inf), sum (||C_{:,i}||_1), max 1/value (Q14 witness)
__global__ void k_col_stats(int64_t n, const int64_t* colptr, const double* valT, double* cmax, double* csum,
                            double* crecip) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double mx = 0.0, sm = 0.0, rc = 0.0;
    for (int64_t k = colptr[i]; k < colptr[i + 1]; ++k) {
      const double a = valT ? valT[k] : 1.0;
      mx = fmax(mx, a);
      sm += a;
      if (a > 0.0) rc = fmax(rc, 1.0 / a);
    }
    if (cmax) cmax[i] = mx;
    if (csum) csum[i] = sm;
    if (crecip) crecip[i] = rc;
  }
}

__global__ void k_compact_csr_rows(int64_t rows, const int64_t* rowptr, const int64_t* scan, int64_t* rowptrP) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    if (rowptr[r + 1] > rowptr[r]) rowptrP[scan[r]] = rowptr[r];
}

__global__ void k_row_nonempty(int64_t rows, const int64_t* rowptr, int64_t* flag) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    flag[r] = rowptr[r + 1] > rowptr[r] ? 1 : 0;
}

__global__ void k_fill(int64_t n, double* a, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) a[i] = v;
}

__global__ void k_fill_nonzero(int64_t n, const int32_t* deg, double* a, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = deg[i] > 0 ? v : 0.0;
}

}  // namespace mwu
