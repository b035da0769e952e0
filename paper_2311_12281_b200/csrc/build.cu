// build.cu -- degree-rank relabel + CSR build on the device (replaces
// build_graph, graph.py:162-259), the reference-layout build, and the
// synthetic R-MAT workload generator.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "engine.cuh"

namespace gs {

// ---------------------------------------------------------------------------
// small helpers

template <class F>
static int cub_call(gs_engine* e, F&& f) {
  size_t bytes = 0;
  GS_CUDA(f(nullptr, bytes));
  void* tmp = nullptr;
  GS_TRY(e->alloc(&tmp, bytes > 0 ? bytes : 1));
  cudaError_t err = f(tmp, bytes);
  e->release(tmp);
  GS_CUDA(err);
  return GS_OK;
}

static int bits_for(int64_t x) {  // bits needed to represent values in [0, x]
  int b = 0;
  while (b < 62 && (int64_t(1) << b) <= x) ++b;
  return b < 1 ? 1 : b;
}

__device__ __forceinline__ int64_t upper_bound_i64(const int64_t* a, int64_t lo, int64_t hi,
                                                   int64_t x) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// kernels

// Degrees of a normalised edge list.  Sets bad[0] for invalid pairs and
// bad[1] when the list is not strictly increasing with u < v (informational:
// the sort-based build checks duplicates itself).  Consecutive edges of a
// sorted list share u, so the u-side increments are warp-aggregated.
__global__ void k_count_deg_edges(const int32_t* __restrict__ uv, int64_t m, int64_t n,
                                  uint32_t* __restrict__ deg, int* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t mm = (m + 31) / 32 * 32;  // whole warps iterate together
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < mm; k += stride) {
    const bool in = k < m;
    int2 p = in ? reinterpret_cast<const int2*>(uv)[k] : make_int2(-1, -1);
    bool ok = in && !(p.x < 0 || p.y < 0 || p.x >= n || p.y >= n || p.x == p.y);
    if (in && !ok) atomicExch(&bad[0], 1);
    if (in && !(p.x < p.y)) bad[1] = 1;
    if (in && k > 0) {
      const int2 q = reinterpret_cast<const int2*>(uv)[k - 1];
      if (q.x > p.x || (q.x == p.x && q.y >= p.y)) bad[1] = 1;
    }
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    const int key = ok ? p.x : -1 - (int)(threadIdx.x & 31);
    const unsigned grp = __match_any_sync(0xffffffffu, key) & act;
    if (ok) {
      if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&deg[p.x], (unsigned)__popc(grp));
      atomicAdd(&deg[p.y], 1u);
    }
  }
}

__global__ void k_deg_from_off(const int64_t* __restrict__ off, int64_t n,
                               uint32_t* __restrict__ deg, int* __restrict__ bad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = off[v + 1] - off[v];
    if (d < 0 || d > 0x7fffffff) { atomicExch(bad, 2); d = 0; }
    deg[v] = (uint32_t)d;
  }
}

__global__ void k_arc_keys_edges(const int32_t* __restrict__ uv, int64_t m,
                                 const int32_t* __restrict__ rank, int B,
                                 uint64_t* __restrict__ keys) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    int2 p = reinterpret_cast<const int2*>(uv)[k];
    uint64_t ru = rank ? (uint64_t)rank[p.x] : (uint64_t)p.x;
    uint64_t rv = rank ? (uint64_t)rank[p.y] : (uint64_t)p.y;
    keys[2 * k] = (ru << B) | rv;
    keys[2 * k + 1] = (rv << B) | ru;
  }
}

// CSR input: owner of each slot by a binary search narrowed per block.
__global__ void k_arc_keys_csr(const int64_t* __restrict__ off, int64_t n,
                               const int32_t* __restrict__ adj, int64_t slots,
                               const int32_t* __restrict__ rank, int B,
                               uint64_t* __restrict__ keys, int* __restrict__ bad) {
  int64_t base = blockIdx.x * (int64_t)blockDim.x;
  int64_t i = base + threadIdx.x;
  __shared__ int64_t vlo, vhi;
  if (threadIdx.x == 0) {
    int64_t last = base + blockDim.x - 1;
    if (last >= slots) last = slots - 1;
    vlo = upper_bound_i64(off, 0, n + 1, base) - 1;
    vhi = upper_bound_i64(off, 0, n + 1, last);
  }
  __syncthreads();
  if (i >= slots) return;
  int64_t u = upper_bound_i64(off, vlo, vhi, i) - 1;
  int32_t v = adj[i];
  if (v < 0 || v >= n || v == u) { atomicExch(bad, 3); v = 0; }
  if (i > off[u] && adj[i - 1] >= v) atomicExch(bad, 4);  // runs strictly increasing
  uint64_t ru = rank ? (uint64_t)rank[u] : (uint64_t)u;
  uint64_t rv = rank ? (uint64_t)rank[v] : (uint64_t)v;
  keys[i] = (ru << B) | rv;
}

__global__ void k_extract_adj(const uint64_t* __restrict__ keys, int64_t slots, int B,
                              int32_t* __restrict__ adj, int* __restrict__ bad) {
  const uint64_t mask = (uint64_t(1) << B) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < slots;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    adj[i] = (int32_t)(k & mask);
    if (i > 0 && keys[i - 1] == k) atomicExch(bad, 5);  // duplicate undirected edge
  }
}

// number of neighbours with smaller rank (the prefix owned by b)
__global__ void k_lowcnt(const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                         int64_t n, int64_t* __restrict__ cnt) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = off[b], hi = off[b + 1];
    int64_t l = lo, h = hi;
    while (l < h) {
      int64_t mid = (l + h) >> 1;
      if (adj[mid] < (int32_t)b) l = mid + 1; else h = mid;
    }
    cnt[b] = l - lo;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[n] = 0;
}

// expand oriented edges: light vertices, one thread each
__global__ void k_expand_light(const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                               const int64_t* __restrict__ eoff, int64_t rlo, int64_t rhi,
                               int32_t* __restrict__ elo, int32_t* __restrict__ ehi) {
  for (int64_t b = rlo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < rhi;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t e0 = eoff[b], e1 = eoff[b + 1], s = off[b];
    for (int64_t e = e0; e < e1; ++e) {
      elo[e] = adj[s + (e - e0)];
      ehi[e] = (int32_t)b;
    }
  }
}

// heavy vertices: one block per vertex
__global__ void k_expand_heavy(const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                               const int64_t* __restrict__ eoff, int64_t rlo, int64_t rhi,
                               int32_t* __restrict__ elo, int32_t* __restrict__ ehi) {
  for (int64_t b = rlo + blockIdx.x; b < rhi; b += gridDim.x) {
    int64_t e0 = eoff[b], e1 = eoff[b + 1], s = off[b];
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      elo[e] = adj[s + (e - e0)];
      ehi[e] = (int32_t)b;
    }
  }
}

// first rank whose degree >= each class threshold (degrees sorted ascending)
__global__ void k_class_bounds(const int64_t* __restrict__ ndeg, int64_t n,
                               int64_t* __restrict__ out) {
  int c = threadIdx.x;
  if (c < DevGraph::kClasses) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (ndeg[mid] < deg_class(c)) lo = mid + 1; else hi = mid;
    }
    out[c] = lo;
  }
  if (c == DevGraph::kClasses) out[c] = n > 0 ? ndeg[n - 1] : 0;
}

// ---------------------------------------------------------------------------
// shared tail of both builds: given rank[] (or null) and arc keys, finish CSR

// offsets (rank space) from rank-ordered degrees, class bounds, dmax
static int finish_offsets(gs_engine* e, int64_t n, int64_t* ndeg, int64_t* h_cls) {
  DevGraph& g = e->g;
  cudaStream_t st = e->stream;
  GS_TRY(e->alloc_n(&g.off, n + 1));
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, ndeg, g.off, n + 1, st);
  }));
  int64_t* d_cls = nullptr;
  GS_TRY(e->alloc_n(&d_cls, DevGraph::kClasses + 1));
  k_class_bounds<<<1, 32, 0, st>>>(ndeg, n, d_cls);
  e->launches++;
  GS_CUDA(cudaMemcpyAsync(h_cls, d_cls, sizeof(int64_t) * (DevGraph::kClasses + 1),
                          cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  e->release(d_cls);
  return GS_OK;
}

// oriented-edge offsets, validation, endpoint arrays
static int finish_rest(gs_engine* e, int64_t n, int64_t m, const int64_t* h_cls, int* d_bad) {
  DevGraph& g = e->g;
  cudaStream_t st = e->stream;
  int64_t* cnt = nullptr;
  GS_TRY(e->alloc_n(&cnt, n + 1));
  if (n > 0) {
    k_lowcnt<<<grid_for(n, 256), 256, 0, st>>>(g.off, g.adj, n, cnt);
    e->launches++;
  }
  GS_TRY(e->alloc_n(&g.eoff, n + 1));
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cnt, g.eoff, n + 1, st);
  }));
  e->release(cnt);
  int h_bad = 0;
  GS_CUDA(cudaMemcpyAsync(&h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  e->release(d_bad);
  if (h_bad) {
    const char* why = h_bad == 1   ? "edge has an id outside [0, n) or is a self-loop"
                      : h_bad == 2 ? "vertex_offsets not monotone"
                      : h_bad == 3 ? "adjacency entry outside [0, n) or a self-loop"
                      : h_bad == 4 ? "adjacency runs not strictly increasing"
                                   : "duplicate undirected edge";
    set_error(std::string("invalid graph: ") + why);
    return GS_EINVAL;
  }
  for (int c = 0; c < DevGraph::kClasses; ++c) g.rclass[c] = h_cls[c];
  g.dmax = h_cls[DevGraph::kClasses];
  int64_t mm = 0;
  GS_CUDA(cudaMemcpy(&mm, g.eoff + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (mm != m) {
    set_error("invalid graph: adjacency is not symmetric");
    return GS_EINVAL;
  }
  GS_CUDA(cudaGetLastError());
  g.n = n;
  g.m = m;
  return GS_OK;  // the endpoint arrays are built on first use (ensure_endpoints)
}

// elo/ehi (endpoints of every oriented edge) for the edge-parallel cluster
// kernels and the state export; a scan without cores never needs them
int ensure_endpoints(gs_engine* e) {
  DevGraph& g = e->g;
  if (g.elo || g.m == 0) return GS_OK;
  cudaStream_t st = e->stream;
  const int64_t n = g.n, m = g.m;
  GS_TRY(e->alloc_n(&g.elo, m));
  GS_TRY(e->alloc_n(&g.ehi, m));
  const int64_t rsplit = g.rclass[1];  // degree >= 64 -> block per vertex
  if (rsplit > 0) {
    k_expand_light<<<grid_for(rsplit, 256), 256, 0, st>>>(g.off, g.adj, g.eoff, 0, rsplit,
                                                          g.elo, g.ehi);
    e->launches++;
  }
  if (n > rsplit) {
    int64_t nb = n - rsplit;
    k_expand_heavy<<<(unsigned)(nb < 65535 * 4 ? nb : 65535 * 4), 256, 0, st>>>(
        g.off, g.adj, g.eoff, rsplit, n, g.elo, g.ehi);
    e->launches++;
  }
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// ---------------------------------------------------------------------------
// CSR assembly without a global sort: every arc is scattered straight into its
// rank-space run (offsets are known from the degrees), then each run is sorted
// on its own (segmented sort over 4-byte ranks).  This moves 4 B per arc per
// pass instead of the 8-byte (rank_u, rank_v) keys of a 6-pass global radix
// sort, and needs 2 x 4 B x 2m of scratch instead of 2 x 8 B x 2m.

// Edge input: rank-space arcs (ru -> rv) and (rv -> ru) of every valid pair.
// Sorted input puts consecutive pairs on the same u, so the u-side cursor
// increments are warp-aggregated (match_any + one atomic per group).
__global__ void k_scatter_edges(const int32_t* __restrict__ uv, int64_t m, int64_t n,
                                const int32_t* __restrict__ rank,
                                unsigned long long* __restrict__ cur,
                                int32_t* __restrict__ out) {
  // cur[r] starts at off[r]: the atomic returns the absolute slot
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t mm = (m + 31) / 32 * 32;
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < mm; k += stride) {
    const bool in = k < m;
    const int2 p = in ? reinterpret_cast<const int2*>(uv)[k] : make_int2(-1, -1);
    const bool ok = in && !(p.x < 0 || p.y < 0 || p.x >= n || p.y >= n || p.x == p.y);
    const int32_t ru = ok ? rank[p.x] : -1 - lane;
    const int32_t rv = ok ? rank[p.y] : -1 - lane;
    const unsigned gu = __match_any_sync(0xffffffffu, ru);
    const unsigned gv = __match_any_sync(0xffffffffu, rv);
    unsigned long long bu = 0, bv = 0;
    if (ok && lane == __ffs(gu) - 1) bu = atomicAdd(&cur[ru], (unsigned long long)__popc(gu));
    if (ok && lane == __ffs(gv) - 1) bv = atomicAdd(&cur[rv], (unsigned long long)__popc(gv));
    bu = __shfl_sync(0xffffffffu, bu, __ffs(gu) - 1);
    bv = __shfl_sync(0xffffffffu, bv, __ffs(gv) - 1);
    if (ok) {
      out[bu + __popc(gu & below)] = rv;
      out[bv + __popc(gv & below)] = ru;
    }
  }
}

// Edge input, bucketed: the direct scatter above issues one random 8-byte
// cursor atomic and one random 4-byte write per arc over the whole 2m-slot
// array (ncu at s24: 14.7 ms, 17 GB read + 8 GB written for 4.2 GB of arcs, 95%
// of cycles with no eligible warp).  Instead (1) each tile of edges sorts its
// 2 x 2048 arcs into B rank-range buckets of ~equal arc counts (bucket b = the
// slots of runs [bstart[b], bstart[b+1]), so the (run, neighbour) pairs land
// in the bucket's own slot range, one global reservation per bucket per tile),
// then (2) one grid-stride pass over that bucket-ordered array places each
// arc in its run: at any moment the whole grid works inside one or two
// buckets, whose cursors and output slots stay in L2.
static constexpr int kEdgeTile = 8;    // edges per thread per tile
static constexpr int kMaxBuckets = 1024;

__global__ void __launch_bounds__(256) k_bucket_arcs(const int32_t* __restrict__ uv, int64_t m,
                                                     int64_t n, const int32_t* __restrict__ rank,
                                                     const int32_t* __restrict__ bstart, int nbk,
                                                     unsigned long long* __restrict__ bcur,
                                                     int2* __restrict__ arcs2,
                                                     int* __restrict__ bad) {
  __shared__ int s_cnt[kMaxBuckets], s_pos[kMaxBuckets];
  __shared__ unsigned long long s_base[kMaxBuckets];
  __shared__ int32_t s_bst[kMaxBuckets + 1];
  for (int i = threadIdx.x; i <= nbk; i += blockDim.x) s_bst[i] = bstart[i];
  const int64_t tile = (int64_t)blockDim.x * kEdgeTile;
  bool b3 = false;
  auto bucket_of = [&](int32_t r) {
    int lo = 0, hi = nbk;  // last b with bstart[b] <= r
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_bst[mid] <= r) lo = mid; else hi = mid;
    }
    return lo;
  };
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < m; t0 += (int64_t)gridDim.x * tile) {
    for (int i = threadIdx.x; i < nbk; i += blockDim.x) { s_cnt[i] = 0; s_pos[i] = 0; }
    __syncthreads();
    int32_t ru[kEdgeTile], rv[kEdgeTile];
    int bu[kEdgeTile], bv[kEdgeTile];
#pragma unroll
    for (int k = 0; k < kEdgeTile; ++k) {
      const int64_t e = t0 + (int64_t)k * blockDim.x + threadIdx.x;
      ru[k] = rv[k] = -1;
      if (e < m) {
        const int2 p = reinterpret_cast<const int2*>(uv)[e];
        if (p.x < 0 || p.y < 0 || p.x >= n || p.y >= n || p.x == p.y) { b3 = true; continue; }
        ru[k] = rank[p.x];
        rv[k] = rank[p.y];
      }
    }
#pragma unroll
    for (int k = 0; k < kEdgeTile; ++k) {
      if (ru[k] < 0) continue;
      bu[k] = bucket_of(ru[k]);
      bv[k] = bucket_of(rv[k]);
      atomicAdd(&s_cnt[bu[k]], 1);
      atomicAdd(&s_cnt[bv[k]], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nbk; i += blockDim.x)
      if (s_cnt[i]) s_base[i] = atomicAdd(&bcur[i], (unsigned long long)s_cnt[i]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kEdgeTile; ++k) {
      if (ru[k] < 0) continue;
      arcs2[s_base[bu[k]] + atomicAdd(&s_pos[bu[k]], 1)] = make_int2(ru[k], rv[k]);
      arcs2[s_base[bv[k]] + atomicAdd(&s_pos[bv[k]], 1)] = make_int2(rv[k], ru[k]);
    }
    __syncthreads();
  }
  if (b3) atomicExch(bad, 1);
}

__global__ void k_bucket_starts(const int64_t* __restrict__ rows, int nbk,
                                const int64_t* __restrict__ off, int32_t* __restrict__ bst,
                                unsigned long long* __restrict__ bcur) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nbk) return;
  bst[k] = (int32_t)rows[k];
  if (k < nbk) bcur[k] = (unsigned long long)off[rows[k]];
}

// (arcs of one hub run arrive together in its bucket: lanes holding the same
// run share one cursor atomic, or a hub's cursor serialises the bucket)
__global__ void k_place_arcs(const int2* __restrict__ arcs2, int64_t slots,
                             unsigned long long* __restrict__ cur, int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  const int64_t ss = (slots + 31) / 32 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ss;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool in = i < slots;
    const int2 a = in ? arcs2[i] : make_int2(-1 - lane, 0);
    const unsigned grp = __match_any_sync(0xffffffffu, a.x);
    const int lead = __ffs(grp) - 1;
    unsigned long long base = 0;
    if (in && lane == lead) base = atomicAdd(&cur[a.x], (unsigned long long)__popc(grp));
    base = __shfl_sync(0xffffffffu, base, lead);
    if (in) out[base + __popc(grp & below)] = a.y;
  }
}

// CSR input: slot i of caller vertex u lands at the same position of u's
// rank-space run (no atomics); validates ids and the strictly increasing runs.
static constexpr int64_t kHeavyScatter = 512;  // == deg_class(2): rclass[2] starts them

__global__ void k_scatter_csr(const int64_t* __restrict__ off, int64_t n, int64_t u0, int64_t u1,
                              const int32_t* __restrict__ chunk, int64_t i0, int64_t i1,
                              int32_t prev, const int32_t* __restrict__ rank,
                              const int64_t* __restrict__ noff, int32_t* __restrict__ out,
                              int* __restrict__ bad, int64_t row_lo, int64_t row_hi) {
  // One warp per caller vertex u in [u0, u1): the slots of u's run inside
  // [i0, i1) (values in chunk[i - i0]) go, relabelled, to the same positions
  // of u's rank-space run -- coalesced reads and writes per run, three
  // broadcast loads per vertex.  prev = the caller's adjacency[i0 - 1] (the
  // run-order check across chunks).
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = u0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); u < u1;
       u += nw) {
    const int64_t ou = off[u], eu = off[u + 1];
    if (eu - ou >= kHeavyScatter) continue;  // k_scatter_csr_heavy
    const int64_t lo = max(ou, i0), hi = min(eu, i1);
    if (lo >= hi) continue;
    const int64_t ru = rank[u];
    if (ru < row_lo || ru >= row_hi) continue;  // another part's row
    const int64_t base = noff[ru] - ou;
    bool b3 = false, b4 = false;
    for (int64_t i = lo + lane; i < hi; i += 32) {
      int32_t v = chunk[i - i0];
      if (v < 0 || v >= n || v == u) { b3 = true; v = (int32_t)u; }
      if (i > ou && (i > i0 ? chunk[i - 1 - i0] : prev) >= v) b4 = true;  // runs increasing
      out[base + i] = rank[v];
    }
    if (b3) atomicExch(bad, 3);
    if (b4) atomicExch(bad, 4);
  }
}

// Runs of kHeavyScatter+ neighbours (a contiguous rank range [rh, n)): one CTA
// per run, so a hub's run does not serialise on one warp.
__global__ void k_scatter_csr_heavy(const int64_t* __restrict__ off, int64_t n, int64_t rh,
                                    int64_t rhi, const int32_t* __restrict__ orig,
                                    const int32_t* __restrict__ chunk, int64_t i0, int64_t i1,
                                    int32_t prev, const int32_t* __restrict__ rank,
                                    const int64_t* __restrict__ noff, int32_t* __restrict__ out,
                                    int* __restrict__ bad) {
  for (int64_t r = rh + blockIdx.x; r < rhi; r += gridDim.x) {
    const int64_t u = orig[r];
    const int64_t ou = off[u];
    const int64_t lo = max(ou, i0), hi = min(off[u + 1], i1);
    if (lo >= hi) continue;
    const int64_t base = noff[r] - ou;
    bool b3 = false, b4 = false;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      int32_t v = chunk[i - i0];
      if (v < 0 || v >= n || v == u) { b3 = true; v = (int32_t)u; }
      if (i > ou && (i > i0 ? chunk[i - 1 - i0] : prev) >= v) b4 = true;
      out[base + i] = rank[v];
    }
    if (b3) atomicExch(bad, 3);
    if (b4) atomicExch(bad, 4);
  }
}

// ---------------------------------------------------------------------------
// Per-run sorts, in place.  Degrees ascend with the rank, so each size class
// is a contiguous rank range: [2, 32] one warp per run (register bitonic
// network over shuffles), (32, 512] one warp per run (2-16 keys per lane in
// registers, k_sort_runs_wreg), (512, 4096) one CTA per run (block radix
// sort), >= 4096 (a few thousand hub runs holding a large share of the arcs)
// a segmented radix sort over the neighbour bits.  A repeated neighbour after
// sorting is a duplicate undirected edge (bad = 5).

static constexpr int32_t kPad = 0x7fffffff;

// first rank whose degree is >= x (degrees are non-decreasing in rank)
__device__ __forceinline__ int64_t rank_of_degree(const int64_t* off, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid + 1] - off[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// The runs a sort kernel handles: a contiguous rank range [rlo, rhi), or the
// ranks listed in list[0, *count) (the host-streamed build sorts each chunk's
// completed runs while later chunks are still in flight)
struct RunSet {
  int64_t rlo, rhi;
  const int32_t* list;
  const int* count;
};
__device__ __forceinline__ int64_t rs_size(const RunSet& R) {
  return R.list ? (int64_t)*R.count : R.rhi - R.rlo;
}
__device__ __forceinline__ int64_t rs_at(const RunSet& R, int64_t i) {
  return R.list ? (int64_t)R.list[i] : R.rlo + i;
}

__global__ void k_sort_classes(const int64_t* __restrict__ off, int64_t n,
                               int64_t* __restrict__ out) {
  const int64_t th[7] = {2, 33, 257, 513, 1025, 2049, 4096};
  const int c = threadIdx.x;
  if (c < 7) out[c] = rank_of_degree(off, n, th[c]);
}

// Warp-wide bitonic sort of 32 K keys held K per lane, "blocked" (lane l holds
// positions lK .. lK + K - 1), ascending.  Partner distances j < K are register
// compare-swaps, j >= K shuffles; the direction bit (i & k) is a compile-time
// constant for k < K and a function of the lane alone for k >= K.  (The
// shared-memory network it replaces issued ~2x the instructions: two loads,
// two stores and the index arithmetic per compare, plus a __syncwarp per stage.)
template <int K>
__device__ __forceinline__ void warp_bitonic_sort(int32_t (&x)[K], int lane) {
  constexpr int P = 32 * K;
#pragma unroll
  for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < K) {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const int p = r ^ j;
          if (p > r) {
            const bool up = k < K ? (r & k) == 0 : (lane & (k / K)) == 0;
            const int32_t lo = min(x[r], x[p]), hi = max(x[r], x[p]);
            x[r] = up ? lo : hi;
            x[p] = up ? hi : lo;
          }
        }
      } else {
        const int lj = j / K;
        const bool keep_lo = ((lane & lj) == 0) == ((lane & (k / K)) == 0);
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const int32_t y = __shfl_xor_sync(0xffffffffu, x[r], lj);
          x[r] = keep_lo ? min(x[r], y) : max(x[r], y);
        }
      }
    }
  }
}

// one run of d in (32 (K / 2), 32 K] slots of `o`, sorted in place by the warp
// (registers; a padded shared-memory transpose for the coalesced write-back)
template <int K>
__device__ __forceinline__ void sort_run_inplace(int32_t* o, int d, int32_t* sbuf, int lane,
                                                 bool& dup) {
  int32_t x[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = lane + 32 * r;
    x[r] = i < d ? o[i] : kPad;
  }
  warp_bitonic_sort<K>(x, lane);
#pragma unroll
  for (int r = 0; r < K; ++r) sbuf[lane * (K + 1) + r] = x[r];
  __syncwarp();
  for (int i = lane; i < d; i += 32) {
    const int32_t v = sbuf[(i / K) * (K + 1) + i % K];
    o[i] = v;
    if (i + 1 < d) dup |= sbuf[((i + 1) / K) * (K + 1) + (i + 1) % K] == v;
  }
  __syncwarp();
}

// runs of 33..512 slots: one warp per run, K = 2..16 keys per lane (replaces a
// shared-memory bitonic network for 33..256 and a 128-thread block radix sort
// for 257..512)
__global__ void __launch_bounds__(256) k_sort_runs_wreg(const int64_t* __restrict__ off,
                                                        RunSet R, int32_t* __restrict__ arcs,
                                                        int* __restrict__ bad) {
  __shared__ int32_t buf[8 * 32 * 17];
  const int lane = threadIdx.x & 31;
  int32_t* sbuf = buf + (threadIdx.x >> 5) * (32 * 17);
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nr = rs_size(R);
  bool dup = false;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < nr; it += nw) {
    const int64_t v = rs_at(R, it);
    const int64_t o = off[v];
    const int d = (int)(off[v + 1] - o);
    if (d <= 64) sort_run_inplace<2>(arcs + o, d, sbuf, lane, dup);
    else if (d <= 128) sort_run_inplace<4>(arcs + o, d, sbuf, lane, dup);
    else if (d <= 256) sort_run_inplace<8>(arcs + o, d, sbuf, lane, dup);
    else sort_run_inplace<16>(arcs + o, d, sbuf, lane, dup);
  }
  if (dup) atomicExch(bad, 5);
}

__global__ void __launch_bounds__(256) k_sort_runs_reg(const int64_t* __restrict__ off,
                                                       RunSet R, int32_t* __restrict__ arcs,
                                                       int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nr = rs_size(R);
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < nr; it += nw) {
    const int64_t v = rs_at(R, it);
    const int64_t o = off[v];
    const int d = (int)(off[v + 1] - o);
    int32_t x = lane < d ? arcs[o + lane] : kPad;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const int32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        const bool up = (lane & k) == 0, low = (lane & j) == 0;
        x = (low == up) ? min(x, y) : max(x, y);
      }
    }
    const int32_t nx = __shfl_down_sync(0xffffffffu, x, 1);
    if (lane < d) {
      arcs[o + lane] = x;
      if (lane + 1 < d && nx == x) atomicExch(bad, 5);
    }
  }
}

// bitonic sort of s[0, P) (P a power of two) by the `nt` threads of a group
// one CTA per run of up to 256*ITEMS neighbours: block radix sort over the
// rank bits (+ one bit that sends the padding to the end)
template <int NT, int ITEMS>
__global__ void __launch_bounds__(NT) k_sort_runs_block(const int64_t* __restrict__ off,
                                                         RunSet R, int endbit,
                                                         int32_t* __restrict__ arcs,
                                                         int* __restrict__ bad) {
  using Sort = cub::BlockRadixSort<uint32_t, NT, ITEMS>;
  __shared__ typename Sort::TempStorage tmp;
  __shared__ int s_dup;
  const int t = threadIdx.x;
  if (t == 0) s_dup = 0;
  const int64_t nr = rs_size(R);
  for (int64_t it = blockIdx.x; it < nr; it += gridDim.x) {
    const int64_t v = rs_at(R, it);
    const int64_t o = off[v];
    const int d = (int)(off[v + 1] - o);
    uint32_t k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {  // striped load; the sort ignores input order
      const int idx = i * NT + t;
      k[i] = idx < d ? (uint32_t)arcs[o + idx] : 0xFFFFFFFFu;
    }
    Sort(tmp).SortBlockedToStriped(k, 0, endbit);
    bool dup = false;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      if (idx < d) arcs[o + idx] = (int32_t)k[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      if (idx + 1 < d) dup |= arcs[o + idx] == arcs[o + idx + 1];
    }
    if (dup) s_dup = 1;
    __syncthreads();
  }
  if (t == 0 && s_dup) atomicExch(bad, 5);
}

// ... and runs of up to NT*ITEMS (16384) neighbours in place, one 1024-thread
// CTA per run, the radix sort's scratch in dynamic shared memory (the hub runs
// of the host-CSR chunk pipeline, sorted while later chunks are in flight)
template <int NT, int ITEMS, int RB>
__global__ void __launch_bounds__(NT, 1) k_sort_runs_block_dyn(const int64_t* __restrict__ off,
                                                                RunSet R, int endbit,
                                                                int32_t* __restrict__ arcs,
                                                                int* __restrict__ bad) {
  using Sort = cub::BlockRadixSort<uint32_t, NT, ITEMS, cub::NullType, RB>;
  extern __shared__ __align__(16) unsigned char dsm[];
  typename Sort::TempStorage& tmp = *reinterpret_cast<typename Sort::TempStorage*>(dsm);
  __shared__ int s_dup;
  const int t = threadIdx.x;
  if (t == 0) s_dup = 0;
  const int64_t nr = rs_size(R);
  for (int64_t it = blockIdx.x; it < nr; it += gridDim.x) {
    const int64_t v = rs_at(R, it);
    const int64_t o = off[v];
    const int d = (int)(off[v + 1] - o);
    uint32_t k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      k[i] = idx < d ? (uint32_t)arcs[o + idx] : 0xFFFFFFFFu;
    }
    Sort(tmp).SortBlockedToStriped(k, 0, endbit);
    bool dup = false;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      if (idx < d) arcs[o + idx] = (int32_t)k[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      if (idx + 1 < d) dup |= arcs[o + idx] == arcs[o + idx + 1];
    }
    if (dup) s_dup = 1;
    __syncthreads();
  }
  if (t == 0 && s_dup) atomicExch(bad, 5);
}

// segment bounds of the listed runs for a segmented sort; slots past the
// list's count are empty segments (the launch is sized for every hub run)
__global__ void k_list_segments(const int64_t* __restrict__ off, const int32_t* __restrict__ list,
                                const int* __restrict__ count, int64_t nseg,
                                int64_t* __restrict__ beg, int64_t* __restrict__ end) {
  const int64_t c = *count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nseg;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i < c ? (int64_t)list[i] : -1;
    beg[i] = v >= 0 ? off[v] : 0;
    end[i] = v >= 0 ? off[v + 1] : 0;
  }
}

// the listed runs back from the sort's alternate buffer (src, when the sort
// ended there) and their duplicate check, one CTA per run
__global__ void k_list_finish(const int64_t* __restrict__ off, const int32_t* __restrict__ list,
                              const int* __restrict__ count, const int32_t* __restrict__ src,
                              int32_t* __restrict__ arcs, int* __restrict__ bad) {
  __shared__ int s_dup;
  if (threadIdx.x == 0) s_dup = 0;
  const int64_t c = *count;
  for (int64_t it = blockIdx.x; it < c; it += gridDim.x) {
    const int64_t v = list[it], lo = off[v], hi = off[v + 1];
    if (src)
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) arcs[i] = src[i];
    __syncthreads();
    bool dup = false;
    for (int64_t i = lo + threadIdx.x; i + 1 < hi; i += blockDim.x) dup |= arcs[i] == arcs[i + 1];
    if (dup) s_dup = 1;
    __syncthreads();
  }
  if (threadIdx.x == 0 && s_dup) atomicExch(bad, 5);
}

// composite keys (run index within the tail, neighbour) of the long runs
__global__ void k_tail_keys(const int64_t* __restrict__ off, int64_t rlo, int64_t rhi,
                            const int32_t* __restrict__ arcs, int B,
                            uint64_t* __restrict__ keys) {
  const int64_t base = off[rlo];
  for (int64_t v = rlo + blockIdx.x; v < rhi; v += gridDim.x) {
    const uint64_t hi = (uint64_t)(v - rlo) << B;
    for (int64_t i = off[v] + threadIdx.x; i < off[v + 1]; i += blockDim.x)
      keys[i - base] = hi | (uint64_t)(uint32_t)arcs[i];
  }
}

__global__ void k_tail_extract(const uint64_t* __restrict__ keys, int64_t cnt, int B,
                               int32_t* __restrict__ out, int* __restrict__ bad) {
  const uint64_t mask = (uint64_t(1) << B) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    out[i] = (int32_t)(k & mask);
    if (i > 0 && keys[i - 1] == k) atomicExch(bad, 5);
  }
}

__global__ void k_rebase(const int64_t* __restrict__ in, int64_t k, int64_t base,
                         int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] - base;
}

// a repeated neighbour in a sorted run is a duplicate edge (bad = 5): flat
// over the slots [s0, s1) of runs [rlo, rhi); an equal pair is checked against
// the run boundaries only when it occurs (rare), by binary search
__global__ void k_run_dups(const int64_t* __restrict__ off, int64_t rlo, int64_t rhi,
                           int64_t s0, int64_t s1, const int32_t* __restrict__ arcs,
                           int* __restrict__ bad) {
  bool dup = false;
  for (int64_t i = s0 + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s1;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (arcs[i] != arcs[i - 1]) continue;
    int64_t lo = rlo, hi = rhi;  // run holding slot i: last v with off[v] <= i
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid] <= i) lo = mid; else hi = mid;
    }
    dup |= off[lo] < i;  // i - 1 in the same run
  }
  if (dup) atomicExch(bad, 5);
}

// The long runs (ranks [rbig, row_hi), >= 4096 neighbours, already
// scattered into `arcs`) sorted on stream `st`: as segments over the neighbour
// bits (cub segmented radix sort), then the duplicate check.  With `defer`
// the scratch blocks are handed back to the caller, who releases them once
// `st` has joined the engine stream (the engine's block cache is ordered by
// the engine stream only).
static int sort_hub_tail(gs_engine* e, cudaStream_t st, int64_t n, int32_t* arcs, int* d_bad,
                         int64_t rbig, int64_t row_hi, std::vector<void*>* defer) {
  DevGraph& g = e->g;
  if (row_hi <= rbig) return GS_OK;
  int64_t hbig = 0, hend = 0;
  GS_CUDA(cudaMemcpyAsync(&hbig, g.off + rbig, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaMemcpyAsync(&hend, g.off + row_hi, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  const int64_t cnt = hend - hbig;
  const bool seg_tail = !(getenv("GS_SEG_TAIL") && atoi(getenv("GS_SEG_TAIL")) == 0);
  auto drop = [&](void* p) {
    if (defer) defer->push_back(p); else e->release(p);
  };
  if (cnt > 0 && seg_tail) {
    // the long runs sorted as segments over the neighbour bits only (int32
    // keys, B bits) instead of one radix sort of 64-bit (run, neighbour) keys
    // (batches of runs holding < 2^30 slots: the segmented sort counts items in int)
    const int B = bits_for(n - 1);
    const int64_t nseg = row_hi - rbig;
    std::vector<int64_t> hoff(nseg + 1);
    GS_CUDA(cudaMemcpyAsync(hoff.data(), g.off + rbig, sizeof(int64_t) * (size_t)(nseg + 1),
                            cudaMemcpyDeviceToHost, st));
    GS_CUDA(cudaStreamSynchronize(st));
    int64_t kBatch = (int64_t)1 << 30;
    if (const char* v = getenv("GS_SEG_BATCH")) kBatch = std::max<int64_t>(1, atoll(v));  // tests
    std::vector<int64_t> cut{0};  // batch boundaries (run indices); a batch holds >= 1 run
    int64_t most = 0;
    for (int64_t a = 0; a < nseg;) {
      int64_t z = a + 1;
      while (z < nseg && hoff[z + 1] - hoff[a] <= kBatch) ++z;
      most = std::max(most, hoff[z] - hoff[a]);
      cut.push_back(z);
      a = z;
    }
    int64_t* segoff = nullptr;
    int32_t* tmp = nullptr;
    GS_TRY(e->alloc_n(&segoff, nseg + 1));
    GS_TRY(e->alloc_n(&tmp, most));
    for (size_t bi = 0; bi + 1 < cut.size(); ++bi) {
      const int64_t a = cut[bi], z = cut[bi + 1];  // runs [a, z)
      const int64_t base = hoff[a], items = hoff[z] - base;
      k_rebase<<<grid_for(z - a + 1, 256), 256, 0, st>>>(g.off + rbig + a, z - a + 1, base,
                                                          segoff);
      cub::DoubleBuffer<int32_t> db(arcs + base, tmp);
      size_t tb = 0;
      GS_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tb, db, (int)items, (int)(z - a),
                                                      segoff, segoff + 1, 0, B, st));
      void* t = nullptr;
      GS_TRY(e->alloc(&t, tb > 0 ? tb : 1));
      GS_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(t, tb, db, (int)items, (int)(z - a), segoff,
                                                      segoff + 1, 0, B, st));
      if (db.Current() != arcs + base)
        GS_CUDA(cudaMemcpyAsync(arcs + base, db.Current(), sizeof(int32_t) * (size_t)items,
                                cudaMemcpyDeviceToDevice, st));
      GS_CUDA(cudaStreamSynchronize(st));  // segoff / tmp reuse across batches
      drop(t);
      e->launches += 2;
    }
    k_run_dups<<<(unsigned)std::min<int64_t>(grid_for(cnt, 256), (int64_t)e->sms * 16), 256, 0,
                 st>>>(g.off, rbig, row_hi, hbig, hend, arcs, d_bad);
    e->launches++;
    drop(segoff);
    drop(tmp);
  } else if (cnt > 0) {
    const int B = bits_for(n - 1);
    const int R = bits_for(row_hi - 1 - rbig);
    uint64_t *k1 = nullptr, *k2 = nullptr;
    GS_TRY(e->alloc_n(&k1, cnt));
    GS_TRY(e->alloc_n(&k2, cnt));
    const int64_t nv = row_hi - rbig;
    k_tail_keys<<<(unsigned)(nv < 65535 * 4 ? nv : 65535 * 4), 256, 0, st>>>(g.off, rbig, row_hi,
                                                                            arcs, B, k1);
    cub::DoubleBuffer<uint64_t> db(k1, k2);
    size_t tb = 0;
    GS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, cnt, 0, B + R, st));
    void* t = nullptr;
    GS_TRY(e->alloc(&t, tb > 0 ? tb : 1));
    GS_CUDA(cub::DeviceRadixSort::SortKeys(t, tb, db, cnt, 0, B + R, st));
    k_tail_extract<<<e->sms * 16, 256, 0, st>>>(db.Current(), cnt, B, arcs + hbig, d_bad);
    e->launches += 3;
    drop(t);
    drop(k1);
    drop(k2);
  }
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// Sort every run of `arcs` (offsets g.off) in place.
static int sort_runs(gs_engine* e, int64_t n, int64_t slots, int32_t* arcs, int* d_bad,
                     int64_t row_lo, int64_t row_hi, bool classes_done = false) {
  DevGraph& g = e->g;
  cudaStream_t st = e->stream;
  if (slots == 0 || n == 0) return GS_OK;
  int64_t* d_cls = nullptr;
  GS_TRY(e->alloc_n(&d_cls, 7));
  k_sort_classes<<<1, 32, 0, st>>>(g.off, n, d_cls);
  int64_t r[7];
  GS_CUDA(cudaMemcpyAsync(r, d_cls, sizeof(r), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  e->release(d_cls);
  e->launches++;
  for (int k = 0; k < 7; ++k) r[k] = std::min(std::max(r[k], row_lo), row_hi);  // this part
  const int64_t r2 = std::max(r[0], row_lo), r33 = r[1], r257 = r[2], rbig = r[6];
  auto warps_grid = [&](int64_t runs) {
    const int64_t gr = (runs + 7) / 8;
    return (unsigned)(gr < (int64_t)e->sms * 64 ? gr : (int64_t)e->sms * 64);
  };
  auto blocks_grid = [&](int64_t runs) {
    return (unsigned)(runs < (int64_t)e->sms * 16 ? runs : (int64_t)e->sms * 16);
  };
  const int endbit = std::min(32, bits_for(n - 1) + 1);
  if (classes_done) r[6] = std::max(r[6], r2);  // runs < 4096 sorted chunk by chunk
  if (!classes_done && r33 > r2) {
    k_sort_runs_reg<<<warps_grid(r33 - r2), 256, 0, st>>>(g.off, RunSet{r2, r33, nullptr, nullptr},
                                                          arcs, d_bad);
    e->launches++;
  }
  if (!classes_done && r257 > r33) {
    k_sort_runs_wreg<<<warps_grid(r257 - r33), 256, 0, st>>>(g.off, RunSet{r33, r257, nullptr, nullptr}, arcs,
                                                                        d_bad);
    e->launches++;
  }
  // CTA classes sized to the run: (256,512] 128x4, (512,1024] 128x8, (1024,2048] 256x8,
  // (2048,4096) 256x16 slots
  if (!classes_done && r[3] > r[2]) {
    k_sort_runs_wreg<<<warps_grid(r[3] - r[2]), 256, 0, st>>>(g.off, RunSet{r[2], r[3], nullptr, nullptr},
                                                               arcs, d_bad);
    e->launches++;
  }
  if (!classes_done && r[4] > r[3]) {
    k_sort_runs_block<128, 8><<<blocks_grid(r[4] - r[3]), 128, 0, st>>>(g.off, RunSet{r[3], r[4], nullptr, nullptr}, endbit,
                                                                        arcs, d_bad);
    e->launches++;
  }
  if (!classes_done && r[5] > r[4]) {
    k_sort_runs_block<256, 8><<<blocks_grid(r[5] - r[4]), 256, 0, st>>>(g.off, RunSet{r[4], r[5], nullptr, nullptr}, endbit,
                                                                        arcs, d_bad);
    e->launches++;
  }
  if (!classes_done && r[6] > r[5]) {
    k_sort_runs_block<256, 16><<<blocks_grid(r[6] - r[5]), 256, 0, st>>>(g.off, RunSet{r[5], r[6], nullptr, nullptr},
                                                                         endbit, arcs, d_bad);
    e->launches++;
  }
  GS_CUDA(cudaGetLastError());
  return sort_hub_tail(e, st, n, arcs, d_bad, rbig, row_hi, nullptr);
}

// shared tail: arcs scattered into their runs (`arcs`, 2m) -> sorted CSR
static int finish_scatter_build(gs_engine* e, int64_t n, int64_t m, int32_t* arcs,
                                const int64_t* h_cls, int* d_bad) {
  e->g.adj_external = false;
  GS_TRY(sort_runs(e, n, 2 * m, arcs, d_bad, 0, n));
  e->g.adj = arcs;
  return finish_rest(e, n, m, h_cls, d_bad);
}

// degrees -> (degree, id) order: orig[rank], rank[orig], rank-space offsets
__global__ void k_iota(int64_t n, uint32_t* __restrict__ x) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    x[v] = (uint32_t)v;
}

// sorted (degree key, id value) -> orig[rank], rank[orig], ndeg[rank]
__global__ void k_rank_scatter_pairs(const uint32_t* __restrict__ dk,
                                     const uint32_t* __restrict__ ids, int64_t n,
                                     int32_t* __restrict__ orig, int32_t* __restrict__ rank,
                                     int64_t* __restrict__ ndeg) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = (int32_t)ids[r];
    orig[r] = v;
    rank[v] = (int32_t)r;
    ndeg[r] = (int64_t)dk[r];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ndeg[n] = 0;
}

// degrees -> (degree, id) order: orig[rank], rank[orig], rank-space offsets.
// A stable radix sort of the degrees with the ids as values (ids enter in
// ascending order, so equal degrees keep id order) over only the bits the
// largest degree needs: 3 passes at s24 instead of 8 over (degree, id) keys.
static int rank_and_offsets(gs_engine* e, int64_t n, uint32_t* deg, int64_t* h_cls) {
  DevGraph& g = e->g;
  cudaStream_t st = e->stream;
  uint32_t *dk2 = nullptr, *ids = nullptr, *ids2 = nullptr, *dmx = nullptr;
  GS_TRY(e->alloc_n(&dk2, n));
  GS_TRY(e->alloc_n(&ids, n));
  GS_TRY(e->alloc_n(&ids2, n));
  GS_TRY(e->alloc_n(&dmx, 1));
  uint32_t hmax = 0;
  if (n > 0) {
    k_iota<<<grid_for(n, 256), 256, 0, st>>>(n, ids);
    e->launches++;
    GS_TRY(cub_call(e, [&](void* t, size_t& b) {
      return cub::DeviceReduce::Max(t, b, deg, dmx, n, st);
    }));
    GS_CUDA(cudaMemcpyAsync(&hmax, dmx, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    GS_CUDA(cudaStreamSynchronize(st));
  }
  e->release(dmx);
  cub::DoubleBuffer<uint32_t> dbk(deg, dk2), dbv(ids, ids2);
  const int endbit = bits_for((int64_t)hmax);
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, dbk, dbv, n, 0, endbit, st);
  }));
  int64_t* ndeg = nullptr;
  GS_TRY(e->alloc_n(&g.orig, n));
  GS_TRY(e->alloc_n(&g.rank, n));
  GS_TRY(e->alloc_n(&ndeg, n + 1));
  if (n > 0) {
    k_rank_scatter_pairs<<<grid_for(n, 256), 256, 0, st>>>(dbk.Current(), dbv.Current(), n,
                                                           g.orig, g.rank, ndeg);
    e->launches++;
  } else {
    GS_CUDA(cudaMemsetAsync(ndeg, 0, sizeof(int64_t), st));
  }
  e->release(dk2);
  e->release(ids);
  e->release(ids2);
  GS_TRY(finish_offsets(e, n, ndeg, h_cls));
  e->release(ndeg);
  return GS_OK;
}

__global__ void k_row_split(const int64_t* __restrict__ off, int64_t n, int64_t slots, int world,
                            int64_t* __restrict__ rows);

int build_from_edges(gs_engine* e, int64_t n, int64_t m, const int32_t* uv) {
  cudaStream_t st = e->stream;
  DevGraph& g = e->g;
  e->free_graph();
  int* d_bad = nullptr;
  GS_TRY(e->alloc_n(&d_bad, 2));
  GS_CUDA(cudaMemsetAsync(d_bad, 0, 2 * sizeof(int), st));
  uint32_t* deg = nullptr;
  GS_TRY(e->alloc_n(&deg, n));
  GS_CUDA(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * (size_t)(n > 0 ? n : 1), st));
  if (m > 0) {
    k_count_deg_edges<<<e->sms * 8, 256, 0, st>>>(uv, m, n, deg, d_bad);
    e->launches++;
  }
  int64_t h_cls[DevGraph::kClasses + 1];
  GS_TRY(rank_and_offsets(e, n, deg, h_cls));
  e->release(deg);
  unsigned long long* cur = nullptr;
  GS_TRY(e->alloc_n(&cur, n));
  if (n > 0)
    GS_CUDA(cudaMemcpyAsync(cur, g.off, sizeof(int64_t) * (size_t)n, cudaMemcpyDeviceToDevice, st));
  int32_t* arcs = nullptr;
  GS_TRY(e->alloc_n(&arcs, 2 * m));
  // bucketed placement (GS_EDGE_BUCKETS=1, when its 8-byte arc buffer fits):
  // measured 25.2 -> 20.9 ms at R-MAT s24 but 181 -> 209 ms on the skewed
  // Chung-Lu graph (its hub runs' cursors serialise inside their buckets), so
  // the direct scatter stays the default
  static const bool buckets_on = getenv("GS_EDGE_BUCKETS") && atoi(getenv("GS_EDGE_BUCKETS")) == 1;
  int2* arcs2 = nullptr;
  if (m > 0 && buckets_on) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t need = 16 * (size_t)m;
    if (need < fr / 2 && (!e->cap || e->reserved + need + (64ull << 20) < e->cap)) {
      if (e->alloc_n(&arcs2, 2 * m) != GS_OK) { cudaGetLastError(); arcs2 = nullptr; }
    }
  }
  if (m > 0 && arcs2) {
    // ~32 M arcs per bucket (measured best of 2^19..2^25 at s24: 20.9 vs 25.2 ms direct)
    static const int bshift = getenv("GS_EDGE_BSHIFT") ? atoi(getenv("GS_EDGE_BSHIFT")) : 25;
    const int nbk = (int)std::min<int64_t>(kMaxBuckets, std::max<int64_t>(1, (2 * m) >> bshift));
    int64_t* rows = nullptr;
    int32_t* bst = nullptr;
    unsigned long long* bcur = nullptr;
    GS_TRY(e->alloc_n(&rows, nbk + 1));
    GS_TRY(e->alloc_n(&bst, nbk + 1));
    GS_TRY(e->alloc_n(&bcur, nbk));
    k_row_split<<<grid_for(nbk + 1, 256), 256, 0, st>>>(g.off, n, 2 * m, nbk, rows);
    k_bucket_starts<<<grid_for(nbk + 1, 256), 256, 0, st>>>(rows, nbk, g.off, bst, bcur);
    const int64_t tiles = (m + 256 * kEdgeTile - 1) / (256 * kEdgeTile);
    k_bucket_arcs<<<(unsigned)std::min<int64_t>(tiles, (int64_t)e->sms * 8), 256, 0, st>>>(
        uv, m, n, g.rank, bst, nbk, bcur, arcs2, d_bad);
    // one launch per bucket (GS_EDGE_PERBUCKET=0: one sweep of the resident
    // grid): the whole GPU places one bucket's arcs at a time, so its cursors
    // and output slots are all that is live in L2
    int occ = 0;
    GS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_place_arcs, 256, 0));
    const unsigned gp = (unsigned)(std::max(occ, 1) * e->sms);
    static const bool per_bucket = !(getenv("GS_EDGE_PERBUCKET") && atoi(getenv("GS_EDGE_PERBUCKET")) == 0);
    if (per_bucket) {
      std::vector<int64_t> hrows(nbk + 1), hoff(nbk + 1);
      GS_CUDA(cudaMemcpyAsync(hrows.data(), rows, sizeof(int64_t) * (nbk + 1), cudaMemcpyDeviceToHost, st));
      GS_CUDA(cudaStreamSynchronize(st));
      for (int k = 0; k <= nbk; ++k) {
        GS_CUDA(cudaMemcpyAsync(&hoff[k], g.off + hrows[k], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      }
      GS_CUDA(cudaStreamSynchronize(st));
      for (int k = 0; k < nbk; ++k) {
        const int64_t a0 = hoff[k], a1 = hoff[k + 1];
        if (a1 <= a0) continue;
        k_place_arcs<<<(unsigned)std::min<int64_t>(gp, grid_for(a1 - a0, 256)), 256, 0, st>>>(
            arcs2 + a0, a1 - a0, cur, arcs);
      }
      e->launches += nbk;
    } else {
      k_place_arcs<<<gp, 256, 0, st>>>(arcs2, 2 * m, cur, arcs);
    }
    e->launches += 4;
    GS_CUDA(cudaGetLastError());
    GS_CUDA(cudaStreamSynchronize(st));  // arcs2 / bcur are released below
    e->release(rows);
    e->release(bst);
    e->release(bcur);
    e->release(arcs2);
  } else if (m > 0) {
    k_scatter_edges<<<e->sms * 8, 256, 0, st>>>(uv, m, n, g.rank, cur, arcs);
    e->launches++;
  }
  e->release(cur);
  return finish_scatter_build(e, n, m, arcs, h_cls, d_bad);
}

// rank-space row bounds of every part: first row whose offset reaches
// k * slots / world (k = 0..world); parts get ~equal numbers of arcs
__global__ void k_row_split(const int64_t* __restrict__ off, int64_t n, int64_t slots, int world,
                            int64_t* __restrict__ rows) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > world) return;
  if (k == world) { rows[k] = n; return; }
  const int64_t target = (int64_t)((__int128)slots * k / world);
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] < target) lo = mid + 1; else hi = mid;
  }
  rows[k] = lo;
}

// rows (and slot bounds) of every part; [row_lo, row_hi) of part_rank
int part_rows(gs_engine* e, int64_t n, int64_t slots, int part_rank, int part_world,
                     int64_t* row_lo, int64_t* row_hi, int64_t* slot_bounds) {
  if (part_world <= 1) {
    *row_lo = 0;
    *row_hi = n;
    if (slot_bounds) { slot_bounds[0] = 0; slot_bounds[1] = slots; }
    return GS_OK;
  }
  DevGraph& g = e->g;
  int64_t* d_rows = nullptr;
  GS_TRY(e->alloc_n(&d_rows, part_world + 1));
  k_row_split<<<grid_for(part_world + 1, 64), 64, 0, e->stream>>>(g.off, n, slots, part_world,
                                                                 d_rows);
  e->launches++;
  std::vector<int64_t> rows(part_world + 1), sb(part_world + 1);
  GS_CUDA(cudaMemcpyAsync(rows.data(), d_rows, sizeof(int64_t) * (part_world + 1),
                          cudaMemcpyDeviceToHost, e->stream));
  GS_CUDA(cudaStreamSynchronize(e->stream));
  e->release(d_rows);
  for (int k = 0; k <= part_world; ++k)
    GS_CUDA(cudaMemcpyAsync(&sb[k], g.off + rows[k], sizeof(int64_t), cudaMemcpyDeviceToHost,
                            e->stream));
  GS_CUDA(cudaStreamSynchronize(e->stream));
  *row_lo = rows[part_rank];
  *row_hi = rows[part_rank + 1];
  if (slot_bounds)
    for (int k = 0; k <= part_world; ++k) slot_bounds[k] = sb[k];
  return GS_OK;
}

// the arcs buffer: the caller's (partitioned builds) or a fresh one
static int arcs_buffer(gs_engine* e, int64_t slots, int32_t* adj_out, int32_t** arcs) {
  if (adj_out) {
    *arcs = adj_out;
    e->g.adj_external = true;
    return GS_OK;
  }
  e->g.adj_external = false;
  return e->alloc_n(arcs, slots);
}

// after the scatter: sort this part's runs, then finish now or on finish_build
static int finish_part(gs_engine* e, int64_t n, int64_t m, int32_t* arcs, const int64_t* h_cls,
                       int* d_bad, int64_t row_lo, int64_t row_hi, bool defer,
                       bool classes_done = false, bool all_sorted = false) {
  if (!all_sorted) GS_TRY(sort_runs(e, n, 2 * m, arcs, d_bad, row_lo, row_hi, classes_done));
  e->g.adj = arcs;
  if (!defer) return finish_rest(e, n, m, h_cls, d_bad);
  GS_CUDA(cudaStreamSynchronize(e->stream));  // the part is complete for the exchange
  e->pend_finish = true;
  e->pend_n = n;
  e->pend_m = m;
  for (int c = 0; c <= DevGraph::kClasses; ++c) e->pend_cls[c] = h_cls[c];
  e->pend_bad = d_bad;
  return GS_OK;
}

int finish_build(gs_engine* e) {
  if (!e->pend_finish) { set_error("no partitioned build waiting to be finished"); return GS_EINVAL; }
  e->pend_finish = false;
  int* d_bad = e->pend_bad;
  e->pend_bad = nullptr;
  return finish_rest(e, e->pend_n, e->pend_m, e->pend_cls, d_bad);
}

static int fused_scatter_sort(gs_engine* e, int64_t n, int64_t m, const int64_t* off,
                              const int32_t* adj, int32_t* arcs, int* d_bad, int64_t row_lo,
                              int64_t row_hi, int64_t r512);

int build_from_csr(gs_engine* e, int64_t n, int64_t m, const int64_t* off, const int32_t* adj,
                   int part_rank, int part_world, int32_t* adj_out, int64_t* slot_bounds) {
  cudaStream_t st = e->stream;
  DevGraph& g = e->g;
  e->free_graph();
  int* d_bad = nullptr;
  GS_TRY(e->alloc_n(&d_bad, 1));
  GS_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
  uint32_t* deg = nullptr;
  GS_TRY(e->alloc_n(&deg, n));
  if (n > 0) {
    k_deg_from_off<<<grid_for(n, 256), 256, 0, st>>>(off, n, deg, d_bad);
    e->launches++;
  }
  int64_t h_cls[DevGraph::kClasses + 1];
  GS_TRY(rank_and_offsets(e, n, deg, h_cls));
  e->release(deg);
  int64_t row_lo = 0, row_hi = n;
  GS_TRY(part_rows(e, n, 2 * m, part_rank, part_world, &row_lo, &row_hi, slot_bounds));
  int32_t* arcs = nullptr;
  GS_TRY(arcs_buffer(e, 2 * m, adj_out, &arcs));
  const bool fused = m > 0 && !(getenv("GS_FUSED_BUILD") && atoi(getenv("GS_FUSED_BUILD")) == 0);
  if (fused) {
    GS_TRY(fused_scatter_sort(e, n, m, off, adj, arcs, d_bad, row_lo, row_hi, h_cls[2]));
    return finish_part(e, n, m, arcs, h_cls, d_bad, row_lo, row_hi, part_world > 1, true, true);
  }
  if (m > 0) {
    k_scatter_csr<<<(unsigned)std::min<int64_t>(grid_for(n * 32, 256), (int64_t)e->sms * 64), 256,
                    0, st>>>(off, n, 0, n, adj, 0, 2 * m, 0, g.rank, g.off, arcs, d_bad, row_lo,
                             row_hi);
    const int64_t rh = std::max<int64_t>(h_cls[2], row_lo);
    if (row_hi > rh)
      k_scatter_csr_heavy<<<(unsigned)std::min<int64_t>(row_hi - rh, (int64_t)e->sms * 16), 256,
                            0, st>>>(off, n, rh, row_hi, g.orig, adj, 0, 2 * m, 0, g.rank, g.off,
                                     arcs, d_bad);
    e->launches += 2;
  }
  return finish_part(e, n, m, arcs, h_cls, d_bad, row_lo, row_hi, part_world > 1);
}

// Per-run sort classes of the runs a host chunk completed (caller vertices
// [ua, ub), their rank-space runs in [row_lo, row_hi)): ranks appended to
// eight class lists (the six classes of sort_runs below 4096, then [4096,
// 16384] and longer hub runs; runs < 2 need no sort), one shared-memory count
// + one global reservation per class per block.  With `hubs` false the hub
// runs are left to the final pass.
static constexpr int kChunkClasses = 8;
__global__ void __launch_bounds__(256) k_chunk_classes(const int64_t* __restrict__ off, int64_t ua,
                                                       int64_t ub, const int32_t* __restrict__ rank,
                                                       int64_t row_lo, int64_t row_hi,
                                                       int32_t* __restrict__ lists, int64_t stride,
                                                       int* __restrict__ counts, bool hubs) {
  __shared__ int s_cnt[kChunkClasses], s_base[kChunkClasses];
  for (int64_t base = ua + (int64_t)blockIdx.x * blockDim.x; base < ub;
       base += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < kChunkClasses) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t u = base + threadIdx.x;
    int cls = -1, pos = 0;
    int32_t r = 0;
    if (u < ub) {
      const int64_t d = off[u + 1] - off[u];
      r = rank[u];
      if (r >= row_lo && r < row_hi && d >= 2 && (hubs || d < 4096))
        cls = d <= 32 ? 0 : d <= 256 ? 1 : d <= 512 ? 2 : d <= 1024 ? 3 : d <= 2048 ? 4
            : d < 4096 ? 5 : d <= 16384 ? 6 : 7;
      if (cls >= 0) pos = atomicAdd(&s_cnt[cls], 1);
    }
    __syncthreads();
    if (threadIdx.x < kChunkClasses)
      s_base[threadIdx.x] = s_cnt[threadIdx.x] ? atomicAdd(&counts[threadIdx.x], s_cnt[threadIdx.x]) : 0;
    __syncthreads();
    if (cls >= 0) lists[cls * stride + s_base[cls] + pos] = r;
    __syncthreads();
  }
}

// Hub runs of the chunk pipeline: [4096, 16384] by k_sort_runs_block_dyn, longer
// ones by one segmented radix sort per chunk over the listed runs (segments
// where they lie in `arcs`, the alternate buffer as long as `arcs`; the launch
// covers nseg = every hub run of the part, the unlisted ones empty).
struct HubChunkSort {
  int64_t nseg = 0;
  int64_t *beg = nullptr, *end = nullptr;
  int32_t* alt = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  int smem = 0;
  int nitems = 0;
  int bits = 0;  // key bits (rank ids of the n vertices)
};
using HubSortT = cub::BlockRadixSort<uint32_t, 1024, 16, cub::NullType, 5>;

static int sort_chunk_runs(gs_engine* e, const int64_t* d_off, int64_t ua, int64_t ub,
                           int64_t row_lo, int64_t row_hi, int32_t* lists, int64_t stride,
                           int* counts, int endbit, int32_t* arcs, int* d_bad,
                           const HubChunkSort* hub) {
  cudaStream_t st = e->stream;
  const DevGraph& g = e->g;
  if (ub <= ua) return GS_OK;
  GS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int) * kChunkClasses, st));
  k_chunk_classes<<<(unsigned)std::min<int64_t>(grid_for(ub - ua, 256), (int64_t)e->sms * 8), 256,
                    0, st>>>(d_off, ua, ub, g.rank, row_lo, row_hi, lists, stride, counts,
                             hub != nullptr);
  auto L = [&](int c) { return RunSet{0, 0, lists + c * stride, counts + c}; };
  const unsigned wg = (unsigned)std::min<int64_t>((ub - ua + 7) / 8, (int64_t)e->sms * 16);
  const unsigned bg = (unsigned)std::min<int64_t>(ub - ua, (int64_t)e->sms * 8);
  k_sort_runs_reg<<<wg, 256, 0, st>>>(g.off, L(0), arcs, d_bad);
  k_sort_runs_wreg<<<wg, 256, 0, st>>>(g.off, L(1), arcs, d_bad);
  k_sort_runs_wreg<<<wg, 256, 0, st>>>(g.off, L(2), arcs, d_bad);
  k_sort_runs_block<128, 8><<<bg, 128, 0, st>>>(g.off, L(3), endbit, arcs, d_bad);
  k_sort_runs_block<256, 8><<<bg, 256, 0, st>>>(g.off, L(4), endbit, arcs, d_bad);
  k_sort_runs_block<256, 16><<<bg, 256, 0, st>>>(g.off, L(5), endbit, arcs, d_bad);
  e->launches += 7;
  if (hub) {
    k_sort_runs_block_dyn<1024, 16, 5><<<(unsigned)e->sms, 1024, hub->smem, st>>>(
        g.off, L(6), endbit, arcs, d_bad);
    e->launches++;
  }
  if (hub && hub->nseg > 0) {
    k_list_segments<<<grid_for(hub->nseg, 256), 256, 0, st>>>(g.off, lists + 7 * stride,
                                                              counts + 7, hub->nseg, hub->beg,
                                                              hub->end);
    cub::DoubleBuffer<int32_t> db(arcs, hub->alt);
    size_t tb = hub->tb;
    GS_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(hub->tmp, tb, db, hub->nitems,
                                                    (int)hub->nseg, hub->beg, hub->end, 0,
                                                    hub->bits, st));
    k_list_finish<<<(unsigned)e->sms * 2, 256, 0, st>>>(
        g.off, lists + 7 * stride, counts + 7, db.Current() == arcs ? nullptr : hub->alt, arcs,
        d_bad);
    e->launches += 4;
  }
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// ---------------------------------------------------------------------------
// Fused relabel + sort for a device-resident reference CSR: each caller run is
// read, relabelled, sorted where it is held (registers / shared memory) and
// written once, sorted, to its rank-space run -- instead of scatter, then a
// second read-sort-write pass.  Runs of 4096+ neighbours still go through the
// scatter + the radix sort of (run, neighbour) keys (sort_runs' tail).

// validate caller slot i of u (value v): ids, self-loops, strictly increasing runs
__device__ __forceinline__ int32_t fused_check(const int32_t* __restrict__ adj, int64_t i,
                                               int64_t ou, int64_t n, int64_t u, bool& b3,
                                               bool& b4) {
  int32_t v = adj[i];
  if (v < 0 || v >= n || v == u) { b3 = true; v = (int32_t)u; }
  if (i > ou && adj[i - 1] >= v) b4 = true;
  return v;
}

// W-lane segments of a warp each sort one run of <= W neighbours (register
// bitonic network within the segment): 32 / W runs per round; `runs` is the
// warp-uniform mask of the group's lanes whose vertex qualifies
template <int W>
__device__ __forceinline__ void segmented_runs(uint32_t runs, int lane, int64_t g0, int64_t myo,
                                               int myd, int64_t myr,
                                               const int32_t* __restrict__ adj,
                                               const int32_t* __restrict__ rank,
                                               const int64_t* __restrict__ noff,
                                               int32_t* __restrict__ out, int64_t n, bool& b3,
                                               bool& b4, bool& b5) {
  const int seg = lane / W, sl = lane % W;
  while (runs) {
    uint32_t t = runs;
    int src = -1;
    for (int k = 0; k <= seg && t; ++k) {
      const int b = __ffs(t) - 1;
      t &= t - 1;
      if (k == seg) src = b;
    }
    for (int k = 0; k < 32 / W && runs; ++k) runs &= runs - 1;  // consumed this round
    const int sb = src < 0 ? 0 : src;
    const int64_t ou = __shfl_sync(0xffffffffu, myo, sb);  // every lane shuffles
    const int dsb = __shfl_sync(0xffffffffu, myd, sb);
    const int64_t ru = __shfl_sync(0xffffffffu, myr, sb);
    const int d = src < 0 ? 0 : dsb;
    const int64_t u = g0 + sb;
    int32_t x = kPad;
    if (sl < d) x = rank[fused_check(adj, ou + sl, ou, n, u, b3, b4)];
#pragma unroll
    for (int k = 2; k <= W; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const int32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        const bool up = (sl & k) == 0, low = (sl & j) == 0;
        x = (low == up) ? min(x, y) : max(x, y);
      }
    }
    const int32_t nx = __shfl_down_sync(0xffffffffu, x, 1);
    if (sl < d) {
      out[noff[ru] + sl] = x;
      b5 |= sl + 1 < d && nx == x;
    }
  }
}

// one caller run of d in (32 (K / 2), 32 K] neighbours: coalesced gather into
// registers (any order: the network sorts it), warp sort, then a padded
// shared-memory transpose (lane stride K + 1: no bank conflicts) so the
// rank-space run is written coalesced
template <int K>
__device__ __forceinline__ void fused_run_regs(const int32_t* __restrict__ adj,
                                               const int32_t* __restrict__ rank, int64_t ou,
                                               int d, int64_t n, int64_t u, int32_t* o,
                                               int32_t* sbuf, int lane, bool& b3, bool& b4,
                                               bool& b5) {
  int32_t x[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = lane + 32 * r;
    x[r] = i < d ? rank[fused_check(adj, ou + i, ou, n, u, b3, b4)] : kPad;
  }
  warp_bitonic_sort<K>(x, lane);
#pragma unroll
  for (int r = 0; r < K; ++r) sbuf[lane * (K + 1) + r] = x[r];
  __syncwarp();
  for (int i = lane; i < d; i += 32) {
    const int32_t v = sbuf[(i / K) * (K + 1) + i % K];
    o[i] = v;
    if (i + 1 < d) b5 |= sbuf[((i + 1) / K) * (K + 1) + (i + 1) % K] == v;
  }
  __syncwarp();
}

// warp per caller vertex with d <= 32 (lane i holds element i): register
// bitonic network; d in (32, 511]: warp per vertex, K = 2..16 keys per lane
// (warp_bitonic_sort).  Longer runs are skipped (CTA kernels below).
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_fused_warp(const int64_t* __restrict__ off, int64_t n,
                                                    const int32_t* __restrict__ adj,
                                                    const int32_t* __restrict__ rank,
                                                    const int64_t* __restrict__ noff,
                                                    int32_t* __restrict__ out,
                                                    int* __restrict__ bad, int64_t row_lo,
                                                    int64_t row_hi) {
  constexpr int CAP = 32 * 17;  // the K = 16 transpose
  __shared__ int32_t buf[8 * CAP];
  const int lane = threadIdx.x & 31;
  int32_t* sbuf = buf + (threadIdx.x >> 5) * CAP;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool b3 = false, b4 = false, b5 = false;
  // groups of 32 consecutive caller vertices per warp: runs of <= 8 are
  // handled four at a time (8 lanes each: 4x the gathers in flight), the rest
  // one by one
  for (int64_t g0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32; g0 < n;
       g0 += nw * 32) {
    const int64_t myu = g0 + lane;
    int myd = 0;
    int64_t myo = 0, myr = -1;
    if (myu < n) {
      myo = off[myu];
      myd = (int)(off[myu + 1] - myo);
      myr = rank[myu];
      if (myr < row_lo || myr >= row_hi) myd = 0;
    }
    // the group's runs are then read one after another: pull their first
    // 512 bytes into L2 now, so each run's reads wait for L2, not DRAM
    if (myd > 0 && myd <= 256)
      for (int t = 0; t < myd && t < 128; t += 32)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(adj + myo + t));
    // 257..511: k_fused_warp16 (its 16 keys per lane would set this kernel's
    // register budget; at 32 registers it runs 64 warps per SM)
    uint32_t rest = __ballot_sync(0xffffffffu, myd > 16 && myd <= 256);
    // runs of <= 8: four per round (8 lanes each), of 9..16: two per round
    segmented_runs<8>(__ballot_sync(0xffffffffu, myd > 0 && myd <= 8), lane, g0, myo, myd, myr,
                      adj, rank, noff, out, n, b3, b4, b5);
    segmented_runs<16>(__ballot_sync(0xffffffffu, myd > 8 && myd <= 16), lane, g0, myo, myd,
                       myr, adj, rank, noff, out, n, b3, b4, b5);
    while (rest) {
    const int src = __ffs(rest) - 1;
    rest &= rest - 1;
    const int64_t u = g0 + src;
    const int64_t ou = __shfl_sync(0xffffffffu, myo, src);
    const int d = __shfl_sync(0xffffffffu, myd, src);
    const int64_t ru = __shfl_sync(0xffffffffu, myr, src);
    int32_t* o = out + noff[ru];
    if (d <= 32) {
      int32_t x = kPad;
      if (lane < d) x = rank[fused_check(adj, ou + lane, ou, n, u, b3, b4)];
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const int32_t y = __shfl_xor_sync(0xffffffffu, x, j);
          const bool up = (lane & k) == 0, low = (lane & j) == 0;
          x = (low == up) ? min(x, y) : max(x, y);
        }
      }
      const int32_t nx = __shfl_down_sync(0xffffffffu, x, 1);
      if (lane < d) {
        o[lane] = x;
        b5 |= lane + 1 < d && nx == x;
      }
    } else if (d <= 64) {
      fused_run_regs<2>(adj, rank, ou, d, n, u, o, sbuf, lane, b3, b4, b5);
    } else if (d <= 128) {
      fused_run_regs<4>(adj, rank, ou, d, n, u, o, sbuf, lane, b3, b4, b5);
    } else {
      fused_run_regs<8>(adj, rank, ou, d, n, u, o, sbuf, lane, b3, b4, b5);
    }
    }
  }
  if (b3) atomicExch(bad, 3);
  if (b4) atomicExch(bad, 4);
  if (b5) atomicExch(bad, 5);
}

// runs of 257..511 neighbours (the rank range [rlo, rhi)): warp per run, 16 keys
// per lane in registers (fused_run_regs<16>)
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_fused_warp16(const int64_t* __restrict__ off,
                                                            int64_t n, int64_t rlo, int64_t rhi,
                                                            const int32_t* __restrict__ orig,
                                                            const int32_t* __restrict__ adj,
                                                            const int32_t* __restrict__ rank,
                                                            const int64_t* __restrict__ noff,
                                                            int32_t* __restrict__ out,
                                                            int* __restrict__ bad) {
  __shared__ int32_t buf[8 * 32 * 17];
  const int lane = threadIdx.x & 31;
  int32_t* sbuf = buf + (threadIdx.x >> 5) * (32 * 17);
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool b3 = false, b4 = false, b5 = false;
  for (int64_t r = rlo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); r < rhi;
       r += nw) {
    const int64_t u = orig[r];
    const int64_t ou = off[u];
    const int d = (int)(off[u + 1] - ou);
    fused_run_regs<16>(adj, rank, ou, d, n, u, out + noff[r], sbuf, lane, b3, b4, b5);
  }
  if (b3) atomicExch(bad, 3);
  if (b4) atomicExch(bad, 4);
  if (b5) atomicExch(bad, 5);
}

// CTA per run of a rank range whose degrees lie in [kHeavyScatter, NT * ITEMS]:
// block radix sort over the rank bits
template <int NT, int ITEMS, int RB = 4>
__global__ void __launch_bounds__(NT) k_fused_block(const int64_t* __restrict__ off, int64_t n,
                                                    int64_t rlo, int64_t rhi,
                                                    const int32_t* __restrict__ orig,
                                                    const int32_t* __restrict__ adj,
                                                    const int32_t* __restrict__ rank,
                                                    const int64_t* __restrict__ noff, int endbit,
                                                    int32_t* __restrict__ out,
                                                    int* __restrict__ bad) {
  using Sort = cub::BlockRadixSort<uint32_t, NT, ITEMS, cub::NullType, RB>;
  __shared__ typename Sort::TempStorage tmp;
  const int t = threadIdx.x;
  bool b3 = false, b4 = false, b5 = false;
  for (int64_t r = rlo + blockIdx.x; r < rhi; r += gridDim.x) {
    const int64_t u = orig[r];
    const int64_t ou = off[u];
    const int d = (int)(off[u + 1] - ou);
    uint32_t k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      k[i] = idx < d ? (uint32_t)rank[fused_check(adj, ou + idx, ou, n, u, b3, b4)] : 0xFFFFFFFFu;
    }
    Sort(tmp).SortBlockedToStriped(k, 0, endbit);
    int32_t* o = out + noff[r];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      if (idx < d) o[idx] = (int32_t)k[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      if (idx + 1 < d) b5 |= o[idx] == o[idx + 1];
    }
    __syncthreads();
  }
  if (b3) atomicExch(bad, 3);
  if (b4) atomicExch(bad, 4);
  if (b5) atomicExch(bad, 5);
}

// ... for runs of up to 16384 neighbours: one 1024-thread CTA per run, the
// block radix sort's scratch in dynamic shared memory (beyond the 48 KB static
// limit); replaces scatter + segmented radix sort for these hub runs
template <int NT, int ITEMS, int RB = 4>
__global__ void __launch_bounds__(NT, 1) k_fused_block_dyn(const int64_t* __restrict__ off,
                                                           int64_t n, int64_t rlo, int64_t rhi,
                                                           const int32_t* __restrict__ orig,
                                                           const int32_t* __restrict__ adj,
                                                           const int32_t* __restrict__ rank,
                                                           const int64_t* __restrict__ noff,
                                                           int endbit, int32_t* __restrict__ out,
                                                           int* __restrict__ bad) {
  using Sort = cub::BlockRadixSort<uint32_t, NT, ITEMS, cub::NullType, RB>;
  extern __shared__ __align__(16) unsigned char dsm[];
  typename Sort::TempStorage& tmp = *reinterpret_cast<typename Sort::TempStorage*>(dsm);
  const int t = threadIdx.x;
  bool b3 = false, b4 = false, b5 = false;
  for (int64_t r = rlo + blockIdx.x; r < rhi; r += gridDim.x) {
    const int64_t u = orig[r];
    const int64_t ou = off[u];
    const int d = (int)(off[u + 1] - ou);
    uint32_t k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      k[i] = idx < d ? (uint32_t)rank[fused_check(adj, ou + idx, ou, n, u, b3, b4)] : 0xFFFFFFFFu;
    }
    Sort(tmp).SortBlockedToStriped(k, 0, endbit);
    int32_t* o = out + noff[r];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      if (idx < d) o[idx] = (int32_t)k[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * NT + t;
      if (idx + 1 < d) b5 |= o[idx] == o[idx + 1];
    }
    __syncthreads();
  }
  if (b3) atomicExch(bad, 3);
  if (b4) atomicExch(bad, 4);
  if (b5) atomicExch(bad, 5);
}

__global__ void k_fused_classes(const int64_t* __restrict__ off, int64_t n,
                                int64_t* __restrict__ out) {
  const int64_t th[5] = {1025, 2049, 4096, 16385, 257};
  const int c = threadIdx.x;
  if (c < 5) out[c] = rank_of_degree(off, n, th[c]);
}

// the device-CSR build's relabel + per-run sorts, fused.  Runs of > 16384
// neighbours are scattered and sorted as segments on the copy stream (idle in
// this build) while the engine stream sorts everything shorter; the engine
// stream joins it before the CSR is finished.
static int fused_scatter_sort(gs_engine* e, int64_t n, int64_t m, const int64_t* off,
                              const int32_t* adj, int32_t* arcs, int* d_bad, int64_t row_lo,
                              int64_t row_hi, int64_t r512) {
  DevGraph& g = e->g;
  cudaStream_t st = e->stream, cs = e->cstream;
  int64_t* d_cls = nullptr;
  GS_TRY(e->alloc_n(&d_cls, 5));
  k_fused_classes<<<1, 32, 0, st>>>(g.off, n, d_cls);
  int64_t r[5];
  GS_CUDA(cudaMemcpyAsync(r, d_cls, 5 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  e->release(d_cls);
  e->launches++;
  const int endbit = std::min(32, bits_for(n - 1) + 1);
  auto clip = [&](int64_t x) { return std::min(std::max(x, row_lo), row_hi); };
  // rank ranges by degree (ranks ascend with the degree): [512, 1024], [1025, 2048],
  // [2049, 4095], [4096, 16384], > 16384 (r512 = first rank of degree >= 512, h_cls[2])
  const int64_t h512 = clip(r512), h1025 = clip(r[0]), h2049 = clip(r[1]), h4096 = clip(r[2]),
                h16k = clip(r[3]), h257 = clip(r[4]);
  static const bool two_streams = !(getenv("GS_BUILD_STREAMS") && atoi(getenv("GS_BUILD_STREAMS")) == 1);
  // the longest runs first, on the copy stream: scatter, then the segmented sort
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<void*> deferred;
  cudaStream_t hs = two_streams ? cs : st;
  if (row_hi > h16k && two_streams) {
    GS_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
    GS_CUDA(cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming));
    GS_CUDA(cudaEventRecord(ev0, st));
    GS_CUDA(cudaStreamWaitEvent(cs, ev0, 0));
  }
  if (row_hi > h16k) {
    k_scatter_csr_heavy<<<(unsigned)std::min<int64_t>(row_hi - h16k, (int64_t)e->sms * 16), 256,
                          0, hs>>>(off, n, h16k, row_hi, g.orig, adj, 0, 2 * m, 0, g.rank,
                                   g.off, arcs, d_bad);
    e->launches++;
  }
  static const int fminb = getenv("GS_FUSED_MINB") ? atoi(getenv("GS_FUSED_MINB")) : 8;
  auto fk = fminb >= 8 ? k_fused_warp<8> : fminb == 7 ? k_fused_warp<7> : fminb == 6 ? k_fused_warp<6> : fminb == 5 ? k_fused_warp<5> : k_fused_warp<4>;
  fk<<<(unsigned)std::min<int64_t>(grid_for(n * 32, 256), (int64_t)e->sms * 64), 256,
                 0, st>>>(off, n, adj, g.rank, g.off, arcs, d_bad, row_lo, row_hi);
  e->launches++;
  if (h512 > h257) {
    static const int f16 = getenv("GS_FUSED16_MINB") ? atoi(getenv("GS_FUSED16_MINB")) : 4;
    auto fk16 = f16 >= 6 ? k_fused_warp16<6> : f16 == 5 ? k_fused_warp16<5> : k_fused_warp16<4>;
    fk16<<<(unsigned)std::min<int64_t>(grid_for((h512 - h257) * 32, 256), (int64_t)e->sms * 32),
           256, 0, st>>>(off, n, h257, h512, g.orig, adj, g.rank, g.off, arcs, d_bad);
    e->launches++;
  }
  auto blocks = [&](int64_t runs) {
    return (unsigned)std::min<int64_t>(std::max<int64_t>(runs, 1), (int64_t)e->sms * 16);
  };
  if (h1025 > h512)
    k_fused_block<128, 8><<<blocks(h1025 - h512), 128, 0, st>>>(
        off, n, h512, h1025, g.orig, adj, g.rank, g.off, endbit, arcs, d_bad);
  // radix bits per pass of the CTA sorts (25-bit keys at s24: 5 passes of 5 bits
  // beat 7 of 4 -- 12.07 -> 11.57 ms -- and 5 of 6)
  static const int rb = getenv("GS_SORT_RB") ? atoi(getenv("GS_SORT_RB")) : 5;
  static const int rbd = getenv("GS_SORT_RBD") ? atoi(getenv("GS_SORT_RBD")) : 5;
  // CTA shape of the two mid classes: fewer threads holding more keys each
  // (measured at s24, build ms: 256 x 8 / 256 x 16 keys 8.95, 512 x 4 / 512 x 8
  // 10.5, 128 x 16 / 128 x 32 8.60, 64 x 32 / 128 x 32 8.49, 64 x 32 / 64 x 64
  // 8.42; GS_FB_SHAPE 0 / 1 / 2 / 5 / 6, default 5)
  static const int fbs = getenv("GS_FB_SHAPE") ? atoi(getenv("GS_FB_SHAPE")) : 5;
  auto kb8 = rb == 4 ? k_fused_block<256, 8, 4> : k_fused_block<256, 8, 5>;
  auto kb16 = rb == 4 ? k_fused_block<256, 16, 4> : k_fused_block<256, 16, 5>;
  int nt8 = 256, nt16 = 256;
  if (fbs == 1) { kb8 = k_fused_block<512, 4, 5>; kb16 = k_fused_block<512, 8, 5>; nt8 = nt16 = 512; }
  if (fbs == 2) { kb8 = k_fused_block<128, 16, 5>; kb16 = k_fused_block<128, 32, 5>; nt8 = nt16 = 128; }
  if (fbs == 3) { kb8 = k_fused_block<128, 16, 5>; nt8 = 128; }
  if (fbs == 4) { kb16 = k_fused_block<128, 32, 5>; nt16 = 128; }
  if (fbs == 5) { kb8 = k_fused_block<64, 32, 5>; kb16 = k_fused_block<128, 32, 5>; nt8 = 64; nt16 = 128; }
  if (fbs == 6) { kb8 = k_fused_block<64, 32, 5>; kb16 = k_fused_block<64, 64, 5>; nt8 = nt16 = 64; }
  if (h2049 > h1025)
    kb8<<<blocks(h2049 - h1025), nt8, 0, st>>>(
        off, n, h1025, h2049, g.orig, adj, g.rank, g.off, endbit, arcs, d_bad);
  if (h4096 > h2049)
    kb16<<<blocks(h4096 - h2049), nt16, 0, st>>>(
        off, n, h2049, h4096, g.orig, adj, g.rank, g.off, endbit, arcs, d_bad);
  if (h16k > h4096) {
    // 4096-16384: 512 threads x 32 keys (GS_FBD_SHAPE=1, default; with the mid
    // classes at 64 x 32 / 128 x 32 the build is 8.31 ms against 8.49 with
    // 1024 x 16 (0) and 8.36 with 256 x 64 (2))
    static const int fbd = getenv("GS_FBD_SHAPE") ? atoi(getenv("GS_FBD_SHAPE")) : 1;
    auto kb = rbd == 5 ? k_fused_block_dyn<1024, 16, 5> : k_fused_block_dyn<1024, 16, 4>;
    int ntd = 1024;
    int sm = (int)std::max({sizeof(typename cub::BlockRadixSort<uint32_t, 1024, 16, cub::NullType, 4>::TempStorage),
                            sizeof(typename cub::BlockRadixSort<uint32_t, 1024, 16, cub::NullType, 5>::TempStorage)});
    if (fbd == 1) {
      kb = k_fused_block_dyn<512, 32, 5>;
      ntd = 512;
      sm = (int)sizeof(typename cub::BlockRadixSort<uint32_t, 512, 32, cub::NullType, 5>::TempStorage);
    } else if (fbd == 2) {
      kb = k_fused_block_dyn<256, 64, 5>;
      ntd = 256;
      sm = (int)sizeof(typename cub::BlockRadixSort<uint32_t, 256, 64, cub::NullType, 5>::TempStorage);
    }
    GS_CUDA(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    kb<<<(unsigned)std::min<int64_t>(h16k - h4096, (int64_t)e->sms * (1024 / ntd)), ntd, sm,
         st>>>(off, n, h4096, h16k, g.orig, adj, g.rank, g.off, endbit, arcs, d_bad);
  }
  e->launches += 4;
  GS_CUDA(cudaGetLastError());
  if (row_hi > h16k) {  // host syncs on the copy stream only: the engine stream keeps running
    GS_TRY(sort_hub_tail(e, hs, n, arcs, d_bad, h16k, row_hi, two_streams ? &deferred : nullptr));
    if (two_streams) {
      GS_CUDA(cudaEventRecord(ev1, cs));
      GS_CUDA(cudaStreamWaitEvent(st, ev1, 0));
    }
  }
  for (void* p : deferred) e->release(p);  // stream-ordered after the join
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  return GS_OK;
}

// Host CSR (the reference Graph in pinned or pageable memory): the offsets
// are copied first (degrees -> ranks -> rank-space offsets); the adjacency
// follows in kSlots x kChunk-element chunks on the copy stream, and each chunk
// is scattered into the rank-space runs as soon as it lands, so the PCIe
// transfer overlaps the relabel and the scatter.  HBM holds the chunk ring,
// not a second copy of the adjacency.
int build_from_csr_host(gs_engine* e, int64_t n, int64_t m, const int64_t* off_host,
                        const int32_t* adj_host, int part_rank, int part_world,
                        int32_t* adj_out, int64_t* slot_bounds) {
  constexpr int kSlots = 4;
  int64_t kChunk = (int64_t)1 << 24;  // 64 MB of adjacency per chunk
  if (const char* c = getenv("GS_H2D_CHUNK")) {  // test hook: many small chunks
    const long long v = atoll(c);
    if (v >= 64) kChunk = v;
  }
  cudaStream_t st = e->stream, cs = e->cstream;
  DevGraph& g = e->g;
  e->free_graph();
  const int64_t slots = 2 * m;
  const int64_t nchunks = (slots + kChunk - 1) / kChunk;
  int* d_bad = nullptr;
  int64_t* d_off = nullptr;
  GS_TRY(e->alloc_n(&d_bad, 1));
  GS_TRY(e->alloc_n(&d_off, n + 1));
  int32_t* ring[kSlots] = {nullptr};
  const int nring = (int)std::min<int64_t>(kSlots, nchunks);
  for (int k = 0; k < nring; ++k) GS_TRY(e->alloc_n(&ring[k], kChunk));
  cudaEvent_t copied[kSlots], freed[kSlots], ready;
  for (int k = 0; k < kSlots; ++k) {
    cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&freed[k], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  GS_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
  // Pageable caller arrays (numpy, array.array) go through a pinned staging
  // ring filled by a multi-threaded host copy, so the DMA stays asynchronous
  // and the link saturated; pinned arrays are streamed directly.
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, adj_host) == cudaSuccess &&
                      pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  int32_t* hring[kSlots] = {nullptr};
  // small inputs copy directly (a pinned allocation would cost more than it saves)
  const bool stage = !pinned && slots * (int64_t)sizeof(int32_t) >= ((int64_t)32 << 20);
  if (stage) {
    const size_t need = (size_t)std::min<int64_t>(kSlots, nchunks) * (size_t)kChunk * sizeof(int32_t);
    if (e->hstage_bytes < need) {
      if (e->hstage) cudaFreeHost(e->hstage);
      e->hstage = nullptr;
      e->hstage_bytes = 0;
      GS_CUDA(cudaHostAlloc(&e->hstage, need, cudaHostAllocDefault));
      e->hstage_bytes = need;
    }
    for (int k = 0; k < (int)std::min<int64_t>(kSlots, nchunks); ++k)
      hring[k] = static_cast<int32_t*>(e->hstage) + (size_t)k * (size_t)kChunk;
  }
  if (stage) {  // the offsets through the staging slots too, slot by slot
    const size_t ob = sizeof(int64_t) * (size_t)(n + 1);
    const size_t sb = (size_t)kChunk * sizeof(int32_t);
    const int nslots = (int)std::min<int64_t>(kSlots, nchunks);
    for (size_t at = 0, i = 0; at < ob; at += sb, ++i) {
      const int k = (int)(i % nslots);
      const size_t len = std::min(sb, ob - at);
      if (i >= (size_t)nslots) GS_CUDA(cudaEventSynchronize(copied[k]));
      gs_parallel_copy(hring[k], reinterpret_cast<const char*>(off_host) + at, len);
      GS_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(d_off) + at, hring[k], len,
                              cudaMemcpyHostToDevice, st));
      GS_CUDA(cudaEventRecord(copied[k], st));
    }
  } else {
    GS_CUDA(cudaMemcpyAsync(d_off, off_host, sizeof(int64_t) * (size_t)(n + 1),
                            cudaMemcpyHostToDevice, st));
  }
  cudaEventRecord(ready, st);  // the ring is allocated and free from here on
  GS_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  auto issue = [&](int64_t c) -> int {
    const int k = (int)(c % kSlots);
    const int64_t i0 = c * kChunk, len = std::min<int64_t>(kChunk, slots - i0);
    if (c >= kSlots) GS_CUDA(cudaStreamWaitEvent(cs, freed[k], 0));
    const int32_t* src = adj_host + i0;
    if (stage) {  // the staging slot's previous DMA must be done before refilling it
      GS_CUDA(cudaEventSynchronize(copied[k]));  // (the offsets' or chunk c - kSlots's)
      gs_parallel_copy(hring[k], adj_host + i0, sizeof(int32_t) * (size_t)len);
      src = hring[k];
    }
    GS_CUDA(cudaMemcpyAsync(ring[k], src, sizeof(int32_t) * (size_t)len,
                            cudaMemcpyHostToDevice, cs));
    GS_CUDA(cudaEventRecord(copied[k], cs));
    return GS_OK;
  };
  int64_t next = 0;
  for (; next < nring; ++next) GS_TRY(issue(next));  // overlaps the relabel below
  uint32_t* deg = nullptr;
  GS_TRY(e->alloc_n(&deg, n));
  if (n > 0) {
    k_deg_from_off<<<grid_for(n, 256), 256, 0, st>>>(d_off, n, deg, d_bad);
    e->launches++;
  }
  int64_t h_cls[DevGraph::kClasses + 1];
  GS_TRY(rank_and_offsets(e, n, deg, h_cls));
  e->release(deg);
  int64_t row_lo = 0, row_hi = n;
  GS_TRY(part_rows(e, n, slots, part_rank, part_world, &row_lo, &row_hi, slot_bounds));
  int32_t* arcs = nullptr;
  GS_TRY(arcs_buffer(e, slots, adj_out, &arcs));
  const int64_t rh = std::max<int64_t>(h_cls[2], row_lo);
  // Runs completed by chunk c (caller vertices whose whole run has arrived)
  // are sorted right after its scatter, while later chunks are in flight;
  // only the hub runs (>= 4096) wait for the final pass.
  std::vector<int64_t> done(nchunks + 1, 0);
  int64_t maxv = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t end = std::min<int64_t>((c + 1) * kChunk, slots);
    done[c + 1] = c + 1 == nchunks ? n
                                   : std::upper_bound(off_host + 1, off_host + n + 1, end) -
                                         (off_host + 1);
    maxv = std::max(maxv, done[c + 1] - done[c]);
  }
  int32_t* clists = nullptr;
  int* ccounts = nullptr;
  bool chunk_sort = nchunks > 1 && !(getenv("GS_CHUNK_SORT") && atoi(getenv("GS_CHUNK_SORT")) == 0);
  if (chunk_sort && (e->alloc_n(&clists, kChunkClasses * std::max<int64_t>(maxv, 1)) != GS_OK ||
                     e->alloc_n(&ccounts, kChunkClasses) != GS_OK)) {
    chunk_sort = false;  // no room (HBM cap): sort everything at the end
    cudaGetLastError();
  }
  const int endbit = std::min(32, bits_for(n - 1) + 1);
  // the hub runs (>= 4096) sorted chunk by chunk as well, so that none of the
  // sorting waits for the last chunk (GS_HUB_CHUNK=0: at the end, as before;
  // off when the alternate buffer does not fit or the slots exceed an int)
  HubChunkSort hub;
  bool hub_chunk = chunk_sort && slots <= INT32_MAX &&
                   !(getenv("GS_HUB_CHUNK") && atoi(getenv("GS_HUB_CHUNK")) == 0);
  if (hub_chunk) {
    hub.nseg = std::max<int64_t>(row_hi - std::max<int64_t>(h_cls[3], row_lo), 0);
    hub.nitems = (int)slots;
    hub.bits = bits_for(n - 1);
    hub.smem = (int)sizeof(HubSortT::TempStorage);
    GS_CUDA(cudaFuncSetAttribute(k_sort_runs_block_dyn<1024, 16, 5>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, hub.smem));
    if (hub.nseg > 0) {
      bool ok = e->alloc_n(&hub.beg, hub.nseg) == GS_OK && e->alloc_n(&hub.end, hub.nseg) == GS_OK &&
                e->alloc_n(&hub.alt, slots) == GS_OK;
      if (ok) {
        cub::DoubleBuffer<int32_t> db(arcs, hub.alt);
        GS_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, hub.tb, db, hub.nitems,
                                                        (int)hub.nseg, hub.beg, hub.end, 0,
                                                        hub.bits, st));
        ok = e->alloc(&hub.tmp, hub.tb > 0 ? hub.tb : 1) == GS_OK;
      }
      if (!ok) {
        hub_chunk = false;
        cudaGetLastError();
      }
    }
  }
  auto release_hub = [&]() {
    for (void* p : {(void*)hub.beg, (void*)hub.end, (void*)hub.alt, hub.tmp})
      if (p) e->release(p);
    hub = HubChunkSort();
  };
  if (!hub_chunk) release_hub();
  // GS_SK_STREAM=1: the sketch rows (sketch.cu) of every run a chunk
  // completes, built while later chunks are in flight, at the resolution of
  // eps >= 0.33 (k = 4, rows from degree 32; a scan at another resolution
  // rebuilds them).  Needs every run listed (hub_chunk).  Measured and off by
  // default: the chunk pipeline is not idle enough to hide them (s24 e2e from
  // the pinned host CSR 58.2 -> 60.9 ms, the scan's prep 2.2 ms shorter).
  constexpr int kSkLk = 2;
  constexpr int64_t kSkDmin = 32;
  int32_t* sk_rdeg = nullptr;
  const int64_t dmax_b = h_cls[DevGraph::kClasses];
  if (hub_chunk && part_world == 1 &&
      getenv("GS_SK_STREAM") && atoi(getenv("GS_SK_STREAM")) == 1)
    GS_TRY(sketch_stream_begin(e, n, dmax_b, kSkLk, kSkDmin, &sk_rdeg));
  for (int64_t c = 0; c < nchunks; ++c) {
    const int k = (int)(c % kSlots);
    const int64_t i0 = c * kChunk, len = std::min<int64_t>(kChunk, slots - i0);
    GS_CUDA(cudaStreamWaitEvent(st, copied[k], 0));
    // caller vertices whose runs meet [i0, i0 + len): host binary search
    const int64_t ua = std::upper_bound(off_host, off_host + n + 1, i0) - off_host - 1;
    const int64_t ub = std::upper_bound(off_host, off_host + n + 1, i0 + len - 1) - off_host;
    k_scatter_csr<<<(unsigned)std::min<int64_t>(grid_for((ub - ua) * 32, 256), (int64_t)e->sms * 64),
                    256, 0, st>>>(d_off, n, ua, ub, ring[k], i0, i0 + len,
                                  i0 > 0 ? adj_host[i0 - 1] : 0, g.rank, g.off, arcs, d_bad,
                                  row_lo, row_hi);
    if (row_hi > rh)
      k_scatter_csr_heavy<<<(unsigned)std::min<int64_t>(row_hi - rh, (int64_t)e->sms * 16), 256,
                            0, st>>>(d_off, n, rh, row_hi, g.orig, ring[k], i0, i0 + len,
                                     i0 > 0 ? adj_host[i0 - 1] : 0, g.rank, g.off, arcs, d_bad);
    e->launches += 2;
    GS_CUDA(cudaEventRecord(freed[k], st));
    if (next < nchunks) GS_TRY(issue(next++));
    if (chunk_sort)
      GS_TRY(sort_chunk_runs(e, d_off, done[c], done[c + 1], row_lo, row_hi, clists,
                             std::max<int64_t>(maxv, 1), ccounts, endbit, arcs, d_bad,
                             hub_chunk ? &hub : nullptr));
    if (sk_rdeg)
      GS_TRY(sketch_stream_rows(e, dmax_b, kSkLk, kSkDmin, sk_rdeg, arcs, clists,
                                std::max<int64_t>(maxv, 1), ccounts, done[c + 1] - done[c]));
  }
  if (sk_rdeg) {
    e->release(sk_rdeg);
    g.sk_lk = kSkLk;
    g.sk_dmin = kSkDmin;
  }
  e->release(clists);
  e->release(ccounts);
  release_hub();
  GS_CUDA(cudaGetLastError());
  GS_CUDA(cudaStreamSynchronize(cs));
  for (int k = 0; k < nring; ++k) e->release(ring[k]);
  e->release(d_off);
  for (int k = 0; k < kSlots; ++k) {
    cudaEventDestroy(copied[k]);
    cudaEventDestroy(freed[k]);
  }
  return finish_part(e, n, m, arcs, h_cls, d_bad, row_lo, row_hi, part_world > 1, chunk_sort,
                     hub_chunk);
}

__global__ void k_widen(const uint32_t* __restrict__ d, int64_t n, int64_t* __restrict__ o) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    o[v] = d[v];
}

// ---------------------------------------------------------------------------
// reference-layout build (gs_build_graph): original ids, edge_list, edge_ids

__global__ void k_orient_flags(const int64_t* __restrict__ off, int64_t n,
                               const int32_t* __restrict__ adj, int64_t slots,
                               int64_t* __restrict__ flag) {
  int64_t base = blockIdx.x * (int64_t)blockDim.x;
  int64_t i = base + threadIdx.x;
  __shared__ int64_t vlo, vhi;
  if (threadIdx.x == 0) {
    int64_t last = base + blockDim.x - 1;
    if (last >= slots) last = slots - 1;
    vlo = upper_bound_i64(off, 0, n + 1, base) - 1;
    vhi = upper_bound_i64(off, 0, n + 1, last);
  }
  __syncthreads();
  if (i >= slots) return;
  int64_t a = upper_bound_i64(off, vlo, vhi, i) - 1;
  int32_t b = adj[i];
  int64_t da = off[a + 1] - off[a], db = off[b + 1] - off[b];
  flag[i] = (da < db || (da == db && a < b)) ? 1 : 0;  // graph.py:226
}

__global__ void k_orient_emit(const int64_t* __restrict__ off, int64_t n,
                              const int32_t* __restrict__ adj, int64_t slots,
                              const int64_t* __restrict__ pos, int32_t* __restrict__ edge_ids,
                              int32_t* __restrict__ edge_list) {
  int64_t base = blockIdx.x * (int64_t)blockDim.x;
  int64_t i = base + threadIdx.x;
  __shared__ int64_t vlo, vhi;
  if (threadIdx.x == 0) {
    int64_t last = base + blockDim.x - 1;
    if (last >= slots) last = slots - 1;
    vlo = upper_bound_i64(off, 0, n + 1, base) - 1;
    vhi = upper_bound_i64(off, 0, n + 1, last);
  }
  __syncthreads();
  if (i >= slots) return;
  if (pos[i + 1] == pos[i]) return;  // not an owned slot
  int64_t k = pos[i];
  int32_t a = (int32_t)(upper_bound_i64(off, vlo, vhi, i) - 1);
  int32_t b = adj[i];
  edge_list[2 * k] = a;
  edge_list[2 * k + 1] = b;
  edge_ids[i] = (int32_t)k;
  int64_t l = off[b], h = off[b + 1];  // bisect_left(adjacency, a, ...) graph.py:236
  while (l < h) {
    int64_t mid = (l + h) >> 1;
    if (adj[mid] < a) l = mid + 1; else h = mid;
  }
  edge_ids[l] = (int32_t)k;
}

int build_reference_layout(gs_engine* e, int64_t n, int64_t m, const int32_t* uv_dev,
                           int64_t* off_dev, int32_t* adj_dev, int32_t* eids_dev,
                           int32_t* elist_dev, bool csr_only) {
  cudaStream_t st = e->stream;
  int* d_bad = nullptr;
  GS_TRY(e->alloc_n(&d_bad, 2));
  GS_CUDA(cudaMemsetAsync(d_bad, 0, 2 * sizeof(int), st));
  uint32_t* deg = nullptr;
  GS_TRY(e->alloc_n(&deg, n));
  GS_CUDA(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * (size_t)(n > 0 ? n : 1), st));
  if (m > 0) {
    k_count_deg_edges<<<e->sms * 8, 256, 0, st>>>(uv_dev, m, n, deg, d_bad);
    e->launches++;
  }
  int64_t* deg64 = nullptr;
  GS_TRY(e->alloc_n(&deg64, n + 1));
  GS_CUDA(cudaMemsetAsync(deg64, 0, sizeof(int64_t) * (size_t)(n + 1), st));
  if (n > 0) {
    k_widen<<<grid_for(n, 256), 256, 0, st>>>(deg, n, deg64);
    e->launches++;
  }
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, deg64, off_dev, n + 1, st);
  }));
  e->release(deg64);
  e->release(deg);
  const int B = bits_for(n > 0 ? n - 1 : 0);
  const int64_t slots = 2 * m;
  uint64_t *keys = nullptr, *keys2 = nullptr;
  GS_TRY(e->alloc_n(&keys, slots));
  GS_TRY(e->alloc_n(&keys2, slots));
  if (m > 0) {
    k_arc_keys_edges<<<e->sms * 8, 256, 0, st>>>(uv_dev, m, nullptr, B, keys);
    e->launches++;
  }
  cub::DoubleBuffer<uint64_t> db(keys, keys2);
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, db, slots, 0, 2 * B, st);
  }));
  if (slots > 0) {
    k_extract_adj<<<e->sms * 16, 256, 0, st>>>(db.Current(), slots, B, adj_dev, d_bad);
    e->launches++;
  }
  e->release(keys);
  e->release(keys2);
  if (csr_only) {
    GS_CUDA(cudaStreamSynchronize(st));
    int h_bad = 0;
    GS_CUDA(cudaMemcpy(&h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost));
    e->release(d_bad);
    if (h_bad) {
      set_error(h_bad == 1 ? "invalid edge list: id outside [0, n) or self-loop"
                           : "invalid edge list: duplicate undirected edge");
      return GS_EINVAL;
    }
    return GS_OK;
  }
  int64_t* flag = nullptr;
  int64_t* pos = nullptr;
  GS_TRY(e->alloc_n(&flag, slots + 1));
  GS_TRY(e->alloc_n(&pos, slots + 1));
  GS_CUDA(cudaMemsetAsync(flag + slots, 0, sizeof(int64_t), st));
  if (slots > 0) {
    k_orient_flags<<<grid_for(slots, 256), 256, 0, st>>>(off_dev, n, adj_dev, slots, flag);
    e->launches++;
  }
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, flag, pos, slots + 1, st);
  }));
  if (slots > 0) {
    k_orient_emit<<<grid_for(slots, 256), 256, 0, st>>>(off_dev, n, adj_dev, slots, pos,
                                                        eids_dev, elist_dev);
    e->launches++;
  }
  GS_CUDA(cudaStreamSynchronize(st));
  e->release(flag);
  e->release(pos);
  int h_bad = 0;
  GS_CUDA(cudaMemcpy(&h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost));
  e->release(d_bad);
  if (h_bad) {
    set_error(h_bad == 1 ? "invalid edge list: id outside [0, n) or self-loop"
                         : "invalid edge list: duplicate undirected edge");
    return GS_EINVAL;
  }
  return GS_OK;
}

// ---------------------------------------------------------------------------
// R-MAT generator (same stream as oracle/gscan_oracle.c orc_rmat_edges)

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t rmat_scramble(uint32_t x, int scale, uint64_t sm) {
  const uint64_t mask = (scale >= 32) ? 0xFFFFFFFFull : ((1ull << scale) - 1);
  const int h = (scale + 1) / 2;
  uint64_t y = x;
  y = (y * 0x9E3779B97F4A7C15ULL + (sm & mask)) & mask;
  y ^= y >> h;
  y = (y * 0xD6E8FEB86659FD93ULL) & mask;
  y ^= y >> h;
  return (uint32_t)y;
}

__global__ void k_rmat(int scale, uint64_t sm, int64_t count, int32_t* __restrict__ src,
                       int32_t* __restrict__ dst) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)t;
    uint32_t u = 0, v = 0;
    uint64_t r = 0;
    for (int l = 0; l < scale; ++l) {
      uint32_t x;
      if ((l & 1) == 0) {
        r = mix64(sm ^ (i * 32u + (uint64_t)(l >> 1)));
        x = (uint32_t)(r >> 32);
      } else {
        x = (uint32_t)r;
      }
      const uint32_t qd = x < 2448131358u ? 0u : x < 3264175144u ? 1u : x < 4080218931u ? 2u : 3u;
      u = (u << 1) | (qd >> 1);
      v = (v << 1) | (qd & 1u);
    }
    src[t] = (int32_t)rmat_scramble(u, scale, sm);
    dst[t] = (int32_t)rmat_scramble(v, scale, sm ^ 0x5bd1e995u);
  }
}

__global__ void k_pair_keys(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                            int64_t count, uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t u = (uint32_t)src[i], v = (uint32_t)dst[i];
    if (u > v) { uint32_t t = u; u = v; v = t; }
    keys[i] = (u == v) ? ~0ull : (((uint64_t)u << 32) | v);
  }
}

__global__ void k_unpack_pairs(const uint64_t* __restrict__ keys, int64_t count,
                               int32_t* __restrict__ uv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    reinterpret_cast<int2*>(uv)[i] = make_int2((int32_t)(k >> 32), (int32_t)(uint32_t)k);
  }
}

// Chung-Lu (expected-degree) workload: vertex i has weight
// w_i ~ (i + i0)^-alpha, alpha = 1/(gamma-1); both endpoints of every sample
// are drawn with probability ~ w by the closed-form inverse CDF of the
// continuous power law, then ids are scrambled like the R-MAT ones.
// i0 is chosen so that the largest expected degree is ~wmax.
__global__ void k_chunglu(int logn, double alpha, double i0, double span_lo, double span,
                          uint64_t sm, int64_t count, int32_t* __restrict__ src,
                          int32_t* __restrict__ dst) {
  const double n = (double)(1ull << logn);
  const double inv = 1.0 / (1.0 - alpha);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix64(sm ^ ((uint64_t)t * 0x9E3779B97F4A7C15ULL));
    const double ru = ((r >> 11) & ((1ull << 26) - 1)) * (1.0 / 67108864.0) +
                      (r >> 37) * (1.0 / 67108864.0 / 134217728.0);
    const uint64_t r2 = mix64(r ^ 0xD1B54A32D192ED03ULL);
    const double rv = ((r2 >> 11) & ((1ull << 26) - 1)) * (1.0 / 67108864.0) +
                      (r2 >> 37) * (1.0 / 67108864.0 / 134217728.0);
    double xu = pow(span_lo + ru * span, inv) - i0;
    double xv = pow(span_lo + rv * span, inv) - i0;
    uint32_t u = (uint32_t)fmin(fmax(xu, 0.0), n - 1.0);
    uint32_t v = (uint32_t)fmin(fmax(xv, 0.0), n - 1.0);
    src[t] = (int32_t)rmat_scramble(u, logn, sm);
    dst[t] = (int32_t)rmat_scramble(v, logn, sm);
  }
}

int chunglu_generate(int logn, double gamma, double wmax, int64_t count, uint64_t seed,
                     int32_t* src, int32_t* dst, cudaStream_t st) {
  const double alpha = 1.0 / (gamma - 1.0);
  const double n = (double)(1ull << logn);
  // expected degree of i: 2*count * w_i / sum(w); pick i0 so that i = 0 gets ~wmax
  // (bisection on i0; sum(w) by the integral of the continuous law)
  auto mass = [&](double i0) {
    return (pow(n + i0, 1.0 - alpha) - pow(i0, 1.0 - alpha)) / (1.0 - alpha);
  };
  double lo = 1e-3, hi = n;
  for (int it = 0; it < 200; ++it) {
    const double mid = sqrt(lo * hi);
    const double d0 = 2.0 * (double)count * pow(mid, -alpha) / mass(mid);
    if (d0 > wmax) lo = mid; else hi = mid;
  }
  const double i0 = sqrt(lo * hi);
  const double a = pow(i0, 1.0 - alpha), b = pow(n + i0, 1.0 - alpha);
  if (count > 0)
    k_chunglu<<<148 * 16, 256, 0, st>>>(logn, alpha, i0, a, b - a, mix64(seed), count, src, dst);
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

int rmat_generate(int scale, uint64_t seed, int64_t count, int32_t* src, int32_t* dst,
                  cudaStream_t st) {
  if (count > 0) k_rmat<<<148 * 16, 256, 0, st>>>(scale, mix64(seed), count, src, dst);
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

int normalize_edges(gs_engine* e, int64_t count, const int32_t* src, const int32_t* dst,
                    int32_t* uv, int64_t* m_out) {
  cudaStream_t st = e->stream;
  uint64_t *k1 = nullptr, *k2 = nullptr;
  GS_TRY(e->alloc_n(&k1, count));
  GS_TRY(e->alloc_n(&k2, count));
  if (count > 0) {
    k_pair_keys<<<e->sms * 8, 256, 0, st>>>(src, dst, count, k1);
    e->launches++;
  }
  cub::DoubleBuffer<uint64_t> db(k1, k2);
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, db, count, 0, 64, st);
  }));
  uint64_t* sorted = db.Current();
  uint64_t* other = db.Alternate();
  int64_t* d_num = nullptr;
  GS_TRY(e->alloc_n(&d_num, 1));
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Unique(t, b, sorted, other, d_num, count, st);
  }));
  int64_t nu = 0;
  GS_CUDA(cudaMemcpyAsync(&nu, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  uint64_t last = 0;
  if (nu > 0) {
    GS_CUDA(cudaMemcpy(&last, other + nu - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (last == ~0ull) --nu;  // the self-loop sentinel sorts last
  }
  if (nu > 0) {
    k_unpack_pairs<<<e->sms * 8, 256, 0, st>>>(other, nu, uv);
    e->launches++;
  }
  GS_CUDA(cudaStreamSynchronize(st));
  e->release(k1);
  e->release(k2);
  e->release(d_num);
  *m_out = nu;
  return GS_OK;
}


// ---------------------------------------------------------------------------
// sparse input ids -> dense ranks (parse_edge_list's remap, graph.py:114-117)

__global__ void k_concat_ids(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                             int64_t count, uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = a[i];
    out[count + i] = b[i];
  }
}

__global__ void k_remap_ids(const uint32_t* __restrict__ ids, int64_t n, uint32_t* __restrict__ x,
                            int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = x[i];
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ids[mid] < key) lo = mid + 1; else hi = mid;
    }
    x[i] = (uint32_t)lo;
  }
}

int normalize_sparse(gs_engine* e, int64_t count, uint32_t* src, uint32_t* dst, uint32_t* ids,
                     int64_t* n_out, int32_t* uv, int64_t* m_out) {
  cudaStream_t st = e->stream;
  *n_out = 0;
  *m_out = 0;
  if (count == 0) return GS_OK;
  uint32_t *k1 = nullptr, *k2 = nullptr;
  GS_TRY(e->alloc_n(&k1, 2 * count));
  GS_TRY(e->alloc_n(&k2, 2 * count));
  k_concat_ids<<<e->sms * 8, 256, 0, st>>>(src, dst, count, k1);
  cub::DoubleBuffer<uint32_t> db(k1, k2);
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, db, 2 * count, 0, 32, st);
  }));
  int64_t* d_num = nullptr;
  GS_TRY(e->alloc_n(&d_num, 1));
  GS_TRY(cub_call(e, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Unique(t, b, db.Current(), ids, d_num, 2 * count, st);
  }));
  int64_t n = 0;
  GS_CUDA(cudaMemcpyAsync(&n, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  e->release(k1);
  e->release(k2);
  e->release(d_num);
  if (n > 0x7fffffffLL) { set_error("vertex count exceeds the 4-byte id range"); return GS_EINVAL; }
  k_remap_ids<<<e->sms * 8, 256, 0, st>>>(ids, n, src, count);
  k_remap_ids<<<e->sms * 8, 256, 0, st>>>(ids, n, dst, count);
  e->launches += 5;
  GS_CUDA(cudaGetLastError());
  *n_out = n;
  return normalize_edges(e, count, reinterpret_cast<const int32_t*>(src),
                         reinterpret_cast<const int32_t*>(dst), uv, m_out);
}

}  // namespace gs
