// cluster.cu -- the scan driver: state init, identify (Alg. 2) via sim.cu,
// role resolution (scan.py:390-449), detectClusters (Alg. 3, scan.py:701-773)
// as lock-free union-find + canonical labels + member attachment, and
// classifyHubOutlier (Alg. 4, scan.py:779-852), then the result scatter back
// to caller vertex ids.
//
// Canonical output: a core's cluster id is the minimum caller id
// of the cores in its class; a member's id is the minimum over the clusters
// it is eligible for; shared members (eligible for >= 2 clusters, the
// reference's ROLE_MEMBER_SHARED) are recognised by min != max, which is the
// exact information classify_vertex_from_neighbors needs (scan.py:794-808).
#include <algorithm>

#include <cub/cub.cuh>

#include "simcore.cuh"

namespace gs {

__device__ __forceinline__ int32_t uf_root(const int32_t* parent, int32_t x) {
  const volatile int32_t* p = parent;
  int32_t px = p[x];
  while (px != x) { x = px; px = p[x]; }
  return x;
}

__global__ void k_init_state(const int64_t* __restrict__ off, int64_t n, int32_t mu,
                             uint64_t* __restrict__ bounds, uint8_t* __restrict__ role) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t upper = (uint64_t)(off[v + 1] - off[v] + 1);
    bounds[v] = 1ull | (upper << 32);  // lower = 1, upper = deg+1 (Alg. 1 lines 1-2)
    // a vertex with deg+1 < mu can never be a core: decide it up front
    role[v] = (int64_t)upper < mu ? ROLE_NONCORE : ROLE_UNKNOWN;
  }
}

// resolve_roles_from_bounds (scan.py:390-412)
__global__ void k_resolve(int64_t n, int32_t mu, const uint64_t* __restrict__ bounds,
                          uint8_t* __restrict__ role, unsigned long long* __restrict__ ctr) {
  unsigned long long unresolved = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] != ROLE_UNKNOWN) continue;
    const uint64_t b = bounds[v];
    const int32_t lower = (int32_t)(uint32_t)b, upper = (int32_t)(uint32_t)(b >> 32);
    if (lower >= mu) role[v] = ROLE_CORE;
    else if (upper < mu) role[v] = ROLE_NONCORE;
    else ++unresolved;
  }
  if (unresolved) atomicAdd(&ctr[CTR_UNRESOLVED], unresolved);
}

// singletons: every core is its own tree (scan.py:725-727)
__global__ void k_singletons(int64_t n, const uint8_t* __restrict__ role,
                             int32_t* __restrict__ parent, unsigned long long* __restrict__ ctr) {
  unsigned long long cores = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const bool core = role[v] == ROLE_CORE;
    parent[v] = core ? (int32_t)v : -1;
    cores += core;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cores += __shfl_xor_sync(0xffffffffu, cores, o);
  if (ctr && (threadIdx.x & 31) == 0 && cores) atomicAdd(&ctr[CTR_CORES_PRE], cores);
}

__device__ __forceinline__ int32_t uf_find_h(int32_t* parent, int32_t x) {
  volatile int32_t* p = parent;
  for (;;) {
    int32_t px = p[x];
    if (px == x) return x;
    int32_t gp = p[px];
    if (gp == px) return px;
    p[x] = gp;
    x = gp;
  }
}

// unions over already-similar core-core edges (scan.py:601-618)
__global__ void k_union_known(int64_t m, const int32_t* __restrict__ elo,
                              const int32_t* __restrict__ ehi, const uint8_t* __restrict__ sim,
                              const uint8_t* __restrict__ role, int32_t* parent,
                              unsigned long long* __restrict__ ctr, int rank, int world) {
  unsigned long long retries = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (sim[e] != SIM_SIMILAR) continue;
    int32_t a = elo[e], b = ehi[e];
    if (!owns(b, rank, world)) continue;
    if (role[a] != ROLE_CORE || role[b] != ROLE_CORE) continue;
    for (;;) {
      a = uf_find_h(parent, a);
      b = uf_find_h(parent, b);
      if (a == b) break;
      if (a > b) { int32_t t = a; a = b; b = t; }
      if (atomicCAS(&parent[b], b, a) == b) break;
      ++retries;
    }
  }
  if (retries) atomicAdd(&ctr[CTR_UNION_RETRIES], retries);
}

// flatten (scan.py:730-732) and canonical label = min caller id per class
__global__ void k_flatten(int64_t n, const uint8_t* __restrict__ role, int32_t* parent,
                          const int32_t* __restrict__ orig, int32_t* __restrict__ label,
                          unsigned long long* __restrict__ ctr) {
  unsigned long long roots = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] != ROLE_CORE) continue;
    const int32_t r = uf_root(parent, (int32_t)v);
    if (r == (int32_t)v) ++roots;
    atomicMin(&label[r], orig[v]);
  }
  if (roots) atomicAdd(&ctr[CTR_N_CLUSTERS], roots);
}

__global__ void k_core_labels(int64_t n, const uint8_t* __restrict__ role,
                              const int32_t* __restrict__ parent,
                              const int32_t* __restrict__ label, int32_t* __restrict__ lmin,
                              int32_t* __restrict__ lmax) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] == ROLE_CORE) {
      const int32_t L = label[uf_root(parent, (int32_t)v)];
      lmin[v] = L;
      lmax[v] = L;
    } else {
      lmin[v] = 0x7fffffff;
      lmax[v] = -1;
    }
  }
}

// member attachment over similar core/non-core edges (scan.py:662-698):
// min/max of eligible cluster labels per non-core vertex
__global__ void k_attach(int64_t m, const int32_t* __restrict__ elo,
                         const int32_t* __restrict__ ehi, const uint8_t* __restrict__ sim,
                         const uint8_t* __restrict__ role, int32_t* __restrict__ lmin,
                         int32_t* __restrict__ lmax, int rank, int world) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (sim[e] != SIM_SIMILAR) continue;
    const int32_t a = elo[e], b = ehi[e];
    if (!owns(b, rank, world)) continue;
    const bool ca = role[a] == ROLE_CORE, cb = role[b] == ROLE_CORE;
    if (ca == cb) continue;
    const int32_t core = ca ? a : b, w = ca ? b : a;
    const int32_t L = lmin[core];
    atomicMin(&lmin[w], L);
    atomicMax(&lmax[w], L);
  }
}

// hub / outlier (scan.py:779-829): an unclustered vertex is a hub iff it has
// >= 2 clustered neighbours whose label sets have >= 2 labels in union.
__device__ __forceinline__ void hub_scan(const int32_t* __restrict__ adj, int64_t lo, int64_t hi,
                                         const int32_t* __restrict__ lmin,
                                         const int32_t* __restrict__ lmax, int& cnt, int32_t& umin,
                                         int32_t& umax) {
  for (int64_t i = lo; i < hi; ++i) {
    const int32_t x = adj[i];
    const int32_t hx = lmax[x];
    if (hx < 0) continue;
    ++cnt;
    const int32_t lx = lmin[x];
    umin = lx < umin ? lx : umin;
    umax = hx > umax ? hx : umax;
  }
}

__global__ void k_classify_thread(int64_t rlo, int64_t rhi, const int64_t* __restrict__ off,
                                  const int32_t* __restrict__ adj, const uint8_t* __restrict__ role,
                                  const int32_t* __restrict__ lmin, const int32_t* __restrict__ lmax,
                                  const uint8_t* __restrict__ near, uint8_t* __restrict__ fin) {
  for (int64_t v = rlo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < rhi;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] == ROLE_CORE) { fin[v] = ROLE_CORE; continue; }
    if (lmax[v] >= 0) { fin[v] = ROLE_MEMBER; continue; }
    if (near && !near[v]) { fin[v] = ROLE_OUTLIER; continue; }  // no clustered neighbour
    int cnt = 0;
    int32_t umin = 0x7fffffff, umax = -1;
    hub_scan(adj, off[v], off[v + 1], lmin, lmax, cnt, umin, umax);
    fin[v] = (cnt >= 2 && umin != umax) ? ROLE_HUB : ROLE_OUTLIER;
  }
}

__global__ void k_classify_warp(int64_t rlo, int64_t rhi, const int64_t* __restrict__ off,
                                const int32_t* __restrict__ adj, const uint8_t* __restrict__ role,
                                const int32_t* __restrict__ lmin, const int32_t* __restrict__ lmax,
                                const uint8_t* __restrict__ near, uint8_t* __restrict__ fin) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = rlo + wid; v < rhi; v += nw) {
    if (role[v] == ROLE_CORE) { if (lane == 0) fin[v] = ROLE_CORE; continue; }
    if (lmax[v] >= 0) { if (lane == 0) fin[v] = ROLE_MEMBER; continue; }
    if (near && !near[v]) { if (lane == 0) fin[v] = ROLE_OUTLIER; continue; }
    int cnt = 0;
    int32_t umin = 0x7fffffff, umax = -1;
    const int64_t lo = off[v], hi = off[v + 1];
    for (int64_t i = lo + lane; i < hi; i += 32) {
      const int32_t x = adj[i];
      const int32_t hx = lmax[x];
      if (hx < 0) continue;
      ++cnt;
      const int32_t lx = lmin[x];
      umin = lx < umin ? lx : umin;
      umax = hx > umax ? hx : umax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      umin = min(umin, __shfl_xor_sync(0xffffffffu, umin, o));
      umax = max(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    }
    if (lane == 0) fin[v] = (cnt >= 2 && umin != umax) ? ROLE_HUB : ROLE_OUTLIER;
  }
}

// scatter to caller ids + role counts
__global__ void k_output(int64_t n, const int32_t* __restrict__ orig,
                         const uint8_t* __restrict__ fin, const int32_t* __restrict__ lmin,
                         uint8_t* __restrict__ role_out, int32_t* __restrict__ cluster_out,
                         unsigned long long* __restrict__ ctr) {
  unsigned long long c[4] = {0, 0, 0, 0};
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t f = fin[v];
    const int32_t o = orig[v];
    if (role_out) role_out[o] = f;
    if (cluster_out) cluster_out[o] = (f == ROLE_CORE || f == ROLE_MEMBER) ? lmin[v] : -1;
    c[f == ROLE_CORE ? 0 : f == ROLE_MEMBER ? 1 : f == ROLE_HUB ? 2 : 3]++;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c[i] += __shfl_xor_sync(0xffffffffu, c[i], o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (c[0]) atomicAdd(&ctr[CTR_N_CORE], c[0]);
    if (c[1]) atomicAdd(&ctr[CTR_N_MEMBER], c[1]);
    if (c[2]) atomicAdd(&ctr[CTR_N_HUB], c[2]);
    if (c[3]) atomicAdd(&ctr[CTR_N_OUTLIER], c[3]);
  }
}

// ---------------------------------------------------------------------------
// exchange kernels of the sharded scan (dist.py runs the collectives)

// local Lemma-1 evidence -> per-vertex counts: [0,n) similar, [n,2n) dissimilar
__global__ void k_export_counts(int64_t n, const uint64_t* __restrict__ bounds,
                                const int64_t* __restrict__ off, int32_t* __restrict__ cnt) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t b = bounds[v];
    cnt[v] = (int32_t)(uint32_t)b - 1;
    cnt[n + v] = (int32_t)(off[v + 1] - off[v] + 1) - (int32_t)(uint32_t)(b >> 32);
  }
}

// summed counts of all shards -> exact global bounds (then k_resolve)
__global__ void k_import_counts(int64_t n, const int32_t* __restrict__ cnt,
                                const int64_t* __restrict__ off, uint64_t* __restrict__ bounds) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t lower = (uint64_t)(1 + cnt[v]);
    const uint64_t upper = (uint64_t)(off[v + 1] - off[v] + 1 - cnt[n + v]);
    bounds[v] = lower | (upper << 32);
  }
}

// the local forest as (core, root) pairs, roots excluded
__global__ void k_export_pairs(int64_t n, const uint8_t* __restrict__ role,
                               const int32_t* __restrict__ parent, int32_t* __restrict__ pairs,
                               unsigned long long* __restrict__ count) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] != ROLE_CORE) continue;
    const int32_t r = uf_root(parent, (int32_t)v);
    if (r == (int32_t)v) continue;
    const unsigned long long i = atomicAdd(count, 1ull);
    pairs[2 * i] = (int32_t)v;
    pairs[2 * i + 1] = r;
  }
}

// every shard's pairs unioned into a fresh forest: the merged components
__global__ void k_union_pairs(int64_t np, const int32_t* __restrict__ pairs, int32_t* parent,
                              unsigned long long* __restrict__ ctr) {
  unsigned long long retries = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = pairs[2 * i], b = pairs[2 * i + 1];
    for (;;) {
      a = uf_find_h(parent, a);
      b = uf_find_h(parent, b);
      if (a == b) break;
      if (a > b) { int32_t t = a; a = b; b = t; }
      if (atomicCAS(&parent[b], b, a) == b) break;
      ++retries;
    }
  }
  if (retries) atomicAdd(&ctr[CTR_UNION_RETRIES], retries);
}

// ---------------------------------------------------------------------------

struct PhaseTimer {
  gs_engine* e;
  cudaEvent_t ev[12];
  int k = 0;
  explicit PhaseTimer(gs_engine* eng) : e(eng) {
    for (auto& x : ev) cudaEventCreate(&x);
  }
  ~PhaseTimer() {
    for (auto& x : ev) cudaEventDestroy(x);
  }
  void mark() { cudaEventRecord(ev[k++], e->stream); }
  float ms(int i, int j) {
    float t = 0;
    cudaEventElapsedTime(&t, ev[i], ev[j]);
    return t;
  }
};

static inline unsigned gridv(gs_engine* e, int64_t n) {
  return (unsigned)std::min<int64_t>(grid_for(n, 256), (int64_t)e->sms * 32);
}

// state, thresholds, Alg. 1 lines 1-4
int phase_begin(gs_engine* e, int32_t mu, const Eps2& eps) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  cudaStream_t str = e->stream;
  const int64_t n = g.n, m = g.m;
  e->mu = mu;
  e->eps = eps;
  e->ncores = 0;
  e->free_state();
  e->kev_mark(0);
  GS_TRY(e->alloc_n(&s.sim, m));
  GS_TRY(e->alloc_n(&s.bounds, n));
  GS_TRY(e->alloc_n(&s.role, n));
  GS_TRY(e->alloc_n(&s.parent, n));
  GS_TRY(e->alloc_n(&s.label, n));
  GS_TRY(e->alloc_n(&s.lmin, n));
  GS_TRY(e->alloc_n(&s.lmax, n));
  GS_TRY(e->alloc_n(&s.ctr, CTR_COUNT));
  GS_TRY(e->alloc_n(&s.wq, 8));
  GS_CUDA(cudaMemsetAsync(s.sim, 0, (size_t)(m > 0 ? m : 1), str));
  GS_CUDA(cudaMemsetAsync(s.ctr, 0, sizeof(unsigned long long) * CTR_COUNT, str));
  GS_CUDA(cudaMemsetAsync(s.label, 0x7f, sizeof(int32_t) * (size_t)(n > 0 ? n : 1), str));
  GS_TRY(prepare_similarity(e, eps));
  GS_TRY(run_prepass(e, mu));  // initial Lemma-1 bounds incl. every O(1)-decided edge
  e->kev_mark(1);
  return GS_OK;
}

// phase 1 on this shard's edges (Alg. 2)
int phase_identify(gs_engine* e) { return run_similarity(e, MODE_IDENTIFY, e->eps, e->mu); }

int phase_export_counts(gs_engine* e, int32_t* counts) {
  if (e->g.n == 0) return GS_OK;
  k_export_counts<<<gridv(e, e->g.n), 256, 0, e->stream>>>(e->g.n, e->s.bounds, e->g.off, counts);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

int phase_import_counts(gs_engine* e, const int32_t* counts) {
  if (e->g.n == 0) return GS_OK;
  k_import_counts<<<gridv(e, e->g.n), 256, 0, e->stream>>>(e->g.n, counts, e->g.off, e->s.bounds);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// resolve_roles_from_bounds / _cleanup_unknown_roles (scan.py:390-449)
int phase_resolve(gs_engine* e, bool allow_cleanup) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  cudaStream_t str = e->stream;
  const int64_t n = g.n;
  if (n > 0) {
    k_resolve<<<gridv(e, n), 256, 0, str>>>(n, e->mu, s.bounds, s.role, s.ctr);
    e->launches++;
  }
  unsigned long long unresolved = 0;
  GS_CUDA(cudaMemcpyAsync(&unresolved, s.ctr + CTR_UNRESOLVED, sizeof(unresolved),
                          cudaMemcpyDeviceToHost, str));
  GS_CUDA(cudaStreamSynchronize(str));
  if (unresolved && allow_cleanup) {
    GS_CUDA(cudaMemsetAsync(s.ctr + CTR_UNRESOLVED, 0, sizeof(unsigned long long), str));
    GS_TRY(run_similarity(e, MODE_CLEANUP, e->eps, e->mu));
    k_resolve<<<gridv(e, n), 256, 0, str>>>(n, e->mu, s.bounds, s.role, s.ctr);
    e->launches++;
    GS_CUDA(cudaMemcpyAsync(&unresolved, s.ctr + CTR_UNRESOLVED, sizeof(unresolved),
                            cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaStreamSynchronize(str));
  }
  if (unresolved) {
    set_error("role resolution incomplete after full edge sweep");
    return GS_EINTERNAL;
  }
  // singletons (scan.py:725-727) and the core count
  if (n > 0) {
    k_singletons<<<gridv(e, n), 256, 0, str>>>(n, s.role, s.parent, s.ctr);
    e->launches++;
    GS_CUDA(cudaMemcpyAsync(&e->ncores, s.ctr + CTR_CORES_PRE, sizeof(e->ncores),
                            cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaStreamSynchronize(str));
  }
  return GS_OK;
}


// ---------------------------------------------------------------------------
// Core-centric cluster phases.  When the cores' adjacency is a small part of
// the graph (R-MAT s24: <= 500 cores for every eps >= 0.2), union and attach
// only concern edges incident to a core, so they walk the cores' own lists
// instead of sweeping every oriented edge and every high endpoint b of the
// graph (elo / ehi endpoint arrays, neighbour flags, five class launches of
// the similarity kernels), and classification starts from the clustered
// vertices.  Decisions are exact and recorded as in the dense passes
// (sim[e], counters), so the canonical output is identical.

// position of w in the sorted slots [lo, hi) (w present: its index)
__device__ __forceinline__ int64_t run_find(const int32_t* __restrict__ adj, int64_t lo,
                                            int64_t hi, int32_t w) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (adj[mid] < w) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// sigma(a, b) >= eps?  a < b in rank (deg a <= deg b), one warp.  The O(1)
// degree bounds first (such an edge is not counted again: the identify
// pre-pass counted it), then N(a) from its high end, each lane locating its
// element in N(b) by binary search in a window that only shrinks (its next
// element is smaller), with the scan's exact early exits.
__device__ bool warp_decide(const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                            const int2* __restrict__ thr, const Eps2& eps, int32_t a, int32_t b,
                            int lane, bool& counted, unsigned long long& probes) {
  const int64_t oa = off[a], da = off[a + 1] - oa, ob = off[b], db = off[b + 1] - ob;
  const int2 t = thr[db];
  counted = false;
  if (da + 1 < t.x) return false;
  if (da <= t.y) return true;
  counted = true;
  const int64_t cmin = c_min_exact(da, db, da - 1, eps);
  int64_t hi = db;  // this lane's window in N(b): positions [0, hi]
  int64_t c = 0;
  for (int64_t s = 0; s < da; s += 32) {
    const int64_t j = s + lane;
    bool hit = false;
    if (j < da) {
      const int32_t x = adj[oa + da - 1 - j];
      const int64_t pos = run_find(adj, ob, ob + hi, x) - ob;
      hit = pos < db && adj[ob + pos] == x;
      hi = pos;
    }
    c += __popc(__ballot_sync(0xffffffffu, hit));
    const int64_t scanned = min(da, s + 32);
    probes += (unsigned long long)(scanned - s);
    if (c >= cmin) return true;
    if (c + (da - scanned) < cmin) return false;
  }
  return c >= cmin;
}

// Work items of the list kernels: 32-arc chunks of each listed vertex's run
// (its owned prefix, or its whole run), so a hub's thousands of arcs spread
// over many warps.  ipre = inclusive prefix of the per-entry chunk counts.
__global__ void k_list_chunks(const int* __restrict__ cnt, const int32_t* __restrict__ list,
                              const int64_t* __restrict__ off, const int64_t* __restrict__ eoff,
                              bool owned, int32_t* __restrict__ ch) {
  const int64_t c = *cnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = list[i];
    const int64_t len = owned ? eoff[v + 1] - eoff[v] : off[v + 1] - off[v];
    ch[i] = (int32_t)max((int64_t)1, (len + 31) >> 5);  // >= 1: every entry is visited
  }
}

// item -> (list index k, first arc of the chunk)
__device__ __forceinline__ int64_t item_entry(const int32_t* __restrict__ ipre, int64_t cnt,
                                              int64_t item, int64_t& base) {
  int64_t lo = 0, hi = cnt;  // first k with ipre[k] > item
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)ipre[mid] <= item) lo = mid + 1; else hi = mid;
  }
  base = (item - (lo > 0 ? (int64_t)ipre[lo - 1] : 0)) * 32;
  return lo;
}

// the cores as a list, and the sum of their degrees (the sparse paths' work)
// (deg_sum[0] += degrees, deg_sum[1] = max degree)
__global__ void k_core_list(int64_t n, const uint8_t* __restrict__ role,
                            const int64_t* __restrict__ off, int32_t* __restrict__ list,
                            int* __restrict__ cnt, unsigned long long* __restrict__ deg_sum) {
  unsigned long long ds = 0, dm = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] != ROLE_CORE) continue;
    list[atomicAdd(cnt, 1)] = (int32_t)v;
    const unsigned long long d = (unsigned long long)(off[v + 1] - off[v]);
    ds += d;
    dm = d > dm ? d : dm;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ds += __shfl_xor_sync(0xffffffffu, ds, o);
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, dm, o);
    dm = x > dm ? x : dm;
  }
  if ((threadIdx.x & 31) == 0 && ds) {
    atomicAdd(deg_sum, ds);
    atomicMax(deg_sum + 1, dm);
  }
}

// union over the core-core edges: warp per core c, the cores w < c of its run
// (c is their high endpoint: e = eoff[c] + i); known-similar edges union, an
// unknown one is decided unless both ends already share a root (scan.py:601-660)
// (DECIDE false: the known-similar unions only -- the dense path, whose class
// kernels decide the unknown edges after it)
template <bool DECIDE>
__global__ void k_union_sparse(const int* __restrict__ ncores, const int32_t* __restrict__ clist,
                               const int32_t* __restrict__ ipre,
                               const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                               const int64_t* __restrict__ eoff, const int2* __restrict__ thr,
                               Eps2 eps, uint8_t* __restrict__ sim,
                               const uint8_t* __restrict__ role, int32_t* parent,
                               unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nc = *ncores;
  const int64_t items = nc > 0 ? ipre[nc - 1] : 0;
  unsigned long long evals = 0, probes = 0, retries = 0;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    int64_t base = 0;
    const int32_t c = clist[item_entry(ipre, nc, it, base)];
    const int64_t oc = off[c], e0 = eoff[c], nlow = eoff[c + 1] - e0;
    {
      const int64_t i = base + lane;
      int32_t w = -1;
      uint8_t st = SIM_DISSIMILAR;
      if (i < nlow) {
        w = adj[oc + i];
        if (role[w] == ROLE_CORE) st = sim[e0 + i];
      }
      if (st == SIM_SIMILAR) uf_union(parent, w, c, retries);
      uint32_t mask = DECIDE ? __ballot_sync(0xffffffffu, st == SIM_UNKNOWN) : 0u;
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int32_t ww = __shfl_sync(0xffffffffu, w, src);
        int same = 0;
        if (lane == 0) same = uf_find(parent, ww) == uf_find(parent, c);
        if (__shfl_sync(0xffffffffu, same, 0)) continue;
        bool counted = false;
        unsigned long long pr = 0;
        const bool similar = warp_decide(off, adj, thr, eps, ww, c, lane, counted, pr);
        if (lane == 0) {
          sim[e0 + base + src] = similar ? SIM_SIMILAR : SIM_DISSIMILAR;
          evals += counted;
          probes += pr;
          if (similar) uf_union(parent, ww, c, retries);
        }
      }
    }
  }
  if (lane == 0 && evals) {
    atomicAdd(&ctr[CTR_SIM_EVALS], evals);
    atomicAdd(&ctr[CTR_INTERSECTIONS], evals);
  }
  if (lane == 0 && probes) atomicAdd(&ctr[CTR_PROBES], probes);
  if (retries) atomicAdd(&ctr[CTR_UNION_RETRIES], retries);
}

// attach over the core / non-core edges: warp per core c, every non-core
// neighbour w (e = eoff[high] + position of low in high's run); similar ->
// w's member labels take c's canonical label (scan.py:662-698)
// (DECIDE false: the known-similar edges only, after the dense path's class
// kernels decided the rest)
template <bool DECIDE>
__global__ void k_attach_sparse(const int* __restrict__ ncores, const int32_t* __restrict__ clist,
                                const int32_t* __restrict__ ipre,
                                const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                                const int64_t* __restrict__ eoff, const int2* __restrict__ thr,
                                Eps2 eps, uint8_t* __restrict__ sim,
                                const uint8_t* __restrict__ role, int32_t* __restrict__ lmin,
                                int32_t* __restrict__ lmax, unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nc = *ncores;
  const int64_t items = nc > 0 ? ipre[nc - 1] : 0;
  unsigned long long evals = 0, probes = 0;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    int64_t base = 0;
    const int32_t c = clist[item_entry(ipre, nc, it, base)];
    const int32_t L = lmin[c];
    const int64_t oc = off[c], dc = off[c + 1] - oc, nlow = eoff[c + 1] - eoff[c];
    {
      const int64_t i = base + lane;
      int32_t w = -1;
      int64_t e = -1;
      uint8_t st = SIM_DISSIMILAR;
      if (i < dc) {
        w = adj[oc + i];
        if (role[w] != ROLE_CORE) {
          e = i < nlow ? eoff[c] + i
                       : eoff[w] + (run_find(adj, off[w], off[w] + (eoff[w + 1] - eoff[w]), c) -
                                    off[w]);
          st = sim[e];
        }
      }
      if (st == SIM_SIMILAR) {
        atomicMin(&lmin[w], L);
        atomicMax(&lmax[w], L);
      }
      uint32_t mask = DECIDE ? __ballot_sync(0xffffffffu, st == SIM_UNKNOWN) : 0u;
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int32_t ww = __shfl_sync(0xffffffffu, w, src);
        const int64_t ee = __shfl_sync(0xffffffffu, e, src);
        bool counted = false;
        unsigned long long pr = 0;
        const bool similar = ww < c ? warp_decide(off, adj, thr, eps, ww, c, lane, counted, pr)
                                    : warp_decide(off, adj, thr, eps, c, ww, lane, counted, pr);
        if (lane == 0) {
          sim[ee] = similar ? SIM_SIMILAR : SIM_DISSIMILAR;
          evals += counted;
          probes += pr;
          if (similar) {
            atomicMin(&lmin[ww], L);
            atomicMax(&lmax[ww], L);
          }
        }
      }
    }
  }
  if (lane == 0 && evals) {
    atomicAdd(&ctr[CTR_SIM_EVALS], evals);
    atomicAdd(&ctr[CTR_INTERSECTIONS], evals);
  }
  if (lane == 0 && probes) atomicAdd(&ctr[CTR_PROBES], probes);
}

// flag[w] = 1 for every neighbour w of a listed core (32-arc items of the
// whole runs): the dense attach pass's core-adjacency marks from the core list
__global__ void k_flag_list(const int* __restrict__ ncores, const int32_t* __restrict__ clist,
                            const int32_t* __restrict__ ipre, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ adj, uint8_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nc = *ncores;
  const int64_t items = nc > 0 ? ipre[nc - 1] : 0;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    int64_t base = 0;
    const int32_t c = clist[item_entry(ipre, nc, it, base)];
    const int64_t i = base + lane, oc = off[c];
    if (i < off[c + 1] - oc) flag[adj[oc + i]] = 1;
  }
}

// classification from the clustered side: the clustered vertices (lmax >= 0)
// as a list, ...
__global__ void k_clustered_list(int64_t n, const int32_t* __restrict__ lmax,
                                 int32_t* __restrict__ list, int* __restrict__ cnt,
                                 unsigned long long* __restrict__ deg_sum,
                                 const int64_t* __restrict__ off) {
  unsigned long long ds = 0, dm = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (lmax[v] < 0) continue;
    list[atomicAdd(cnt, 1)] = (int32_t)v;
    const unsigned long long d = (unsigned long long)(off[v + 1] - off[v]);
    ds += d;
    dm = d > dm ? d : dm;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ds += __shfl_xor_sync(0xffffffffu, ds, o);
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, dm, o);
    dm = x > dm ? x : dm;
  }
  if ((threadIdx.x & 31) == 0 && ds) {
    atomicAdd(deg_sum, ds);
    atomicMax(deg_sum + 1, dm);
  }
}

// ... whose final roles are set here, and whose unclustered neighbours (the
// only hub candidates) are listed once each (first setter of their mark byte)
__global__ void k_near_list(const int* __restrict__ nclu, const int32_t* __restrict__ clu,
                            const int32_t* __restrict__ ipre,
                            const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                            const int32_t* __restrict__ lmax, const uint8_t* __restrict__ role,
                            uint8_t* __restrict__ mark, int32_t* __restrict__ near,
                            int* __restrict__ nnear, uint8_t* __restrict__ fin,
                            const int32_t* __restrict__ lmin, int32_t* __restrict__ hacc,
                            int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nc = *nclu;
  const int64_t items = nc > 0 ? ipre[nc - 1] : 0;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    int64_t base = 0;
    const int32_t u = clu[item_entry(ipre, nc, it, base)];
    if (lane == 0 && base == 0) fin[u] = role[u] == ROLE_CORE ? ROLE_CORE : ROLE_MEMBER;
    const int64_t i = off[u] + base + lane;
    if (i < off[u + 1]) {
      const int32_t w = adj[i];
      if (lmax[w] >= 0) continue;
      const unsigned bit = 1u << (8 * (w & 3));
      const unsigned old = atomicOr(reinterpret_cast<unsigned*>(mark) + (w >> 2), bit);
      if (!(old & bit)) near[atomicAdd(nnear, 1)] = w;
      // u's contribution to w's hub test, pushed from the clustered side
      // (zero-initialised: count, INT_MAX - min label, max label + 1)
      atomicAdd(&hacc[w], 1);
      atomicMax(&hacc[n + w], 0x7fffffff - lmin[u]);
      atomicMax(&hacc[2 * n + w], lmax[u] + 1);
    }
  }
}

// hub or outlier for each listed candidate (scan.py:779-829) from what its
// clustered neighbours pushed (k_near_list): >= 2 of them, >= 2 labels
__global__ void k_classify_near(const int* __restrict__ nnear, const int32_t* __restrict__ near,
                                const int32_t* __restrict__ hacc, int64_t n,
                                uint8_t* __restrict__ fin) {
  const int64_t nn = *nnear;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nn;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = near[k];
    const int32_t umin = 0x7fffffff - hacc[n + v], umax = hacc[2 * n + v] - 1;
    fin[v] = (hacc[v] >= 2 && umin != umax) ? ROLE_HUB : ROLE_OUTLIER;
  }
}

// unions over this shard's similar core-core edges (Alg. 3 lines 1-18)
// Sparse (core-centric) union / attach iff the cores' arcs are at most this
// fraction of all arcs (GS_SPARSE_CLUSTER=0 / 1 forces the dense / sparse path)
static constexpr int64_t kSparseDiv = 16;
// ... and no core above this degree: a hub core's edges are decided by binary
// searches in its run one by one (eps 0.2 at s24, a core of degree 92 K:
// cluster 9.2 ms dense, 13.5 sparse; eps 0.15 mu 3, cores <= 31: 13.2 -> 5.1)
static constexpr int64_t kSparseMaxDeg = 4096;
// classification from the clustered side iff their arcs are <= 2m / kListDiv:
// with the hub test pushed from the clustered side (k_near_list) the listed
// path only walks the clustered vertices' arcs, so it always wins (s24 eps
// 0.15 mu 3, 1.5 M hub candidates: 5.4 ms dense, 3.2 at 2m/4, 3.0 at 2m;
// eps 0.2: 2.7 -> 0.39 ms)
static constexpr int64_t kListDiv = 1;

// inclusive prefix of the 32-arc chunk counts of list[0, cnt) (owned prefix or
// whole run); the caller releases *ipre once the launch using it is ordered
static int list_chunks(gs_engine* e, int64_t cnt, const int* d_cnt, const int32_t* list,
                       bool owned, int32_t** ipre) {
  DevGraph& g = e->g;
  int32_t* ch = nullptr;
  GS_TRY(e->alloc_n(&ch, cnt));
  GS_TRY(e->alloc_n(ipre, cnt));
  k_list_chunks<<<gridv(e, cnt), 256, 0, e->stream>>>(d_cnt, list, g.off, g.eoff, owned, ch);
  size_t tb = 0;
  GS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, ch, *ipre, (int)cnt, e->stream));
  void* t = nullptr;
  GS_TRY(e->alloc(&t, tb > 0 ? tb : 1));
  GS_CUDA(cub::DeviceScan::InclusiveSum(t, tb, ch, *ipre, (int)cnt, e->stream));
  e->release(t);
  e->release(ch);
  e->launches += 2;
  return GS_OK;
}

static int sparse_mode() {
  static const int v = getenv("GS_SPARSE_CLUSTER") ? atoi(getenv("GS_SPARSE_CLUSTER")) : -1;
  return v;
}

int phase_union(gs_engine* e) {
  if (e->ncores == 0) return GS_OK;  // no core, no cluster
  DevGraph& g = e->g;
  DevState& s = e->s;
  s.sparse = false;
  if (e->shard_world == 1 && g.m > 0 && sparse_mode() != 0) {
    // the cores as a list and their degree sum: the sparse passes' work
    GS_TRY(e->alloc_n(&s.clist, (int64_t)e->ncores));
    GS_TRY(e->alloc_n(&s.lcnt, 4));
    unsigned long long* dsum = nullptr;
    GS_TRY(e->alloc_n(&dsum, 2));
    GS_CUDA(cudaMemsetAsync(s.lcnt, 0, 4 * sizeof(int), e->stream));
    GS_CUDA(cudaMemsetAsync(dsum, 0, 2 * sizeof(unsigned long long), e->stream));
    k_core_list<<<gridv(e, g.n), 256, 0, e->stream>>>(g.n, s.role, g.off, s.clist, s.lcnt, dsum);
    unsigned long long h[2] = {0, 0};
    GS_CUDA(cudaMemcpyAsync(h, dsum, sizeof(h), cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    e->release(dsum);
    e->launches++;
    s.sparse = sparse_mode() == 1 ||
               ((int64_t)h[0] <= 2 * g.m / kSparseDiv && (int64_t)h[1] <= kSparseMaxDeg);
  }
  if (s.sparse) {
    int32_t* ipre = nullptr;
    GS_TRY(list_chunks(e, (int64_t)e->ncores, s.lcnt, s.clist, true, &ipre));
    k_union_sparse<true><<<(unsigned)e->sms * 16, 256, 0, e->stream>>>(s.lcnt, s.clist, ipre, g.off, g.adj,
                                                                g.eoff, s.thr, e->eps, s.sim,
                                                                s.role, s.parent, s.ctr);
    e->launches++;
    e->release(ipre);  // stream-ordered reuse
    GS_CUDA(cudaGetLastError());
    return GS_OK;
  }
  if (g.m > 0 && s.clist) {  // known-similar core-core unions from the core list
    int32_t* ipre = nullptr;
    GS_TRY(list_chunks(e, (int64_t)e->ncores, s.lcnt, s.clist, true, &ipre));
    k_union_sparse<false><<<(unsigned)e->sms * 16, 256, 0, e->stream>>>(
        s.lcnt, s.clist, ipre, g.off, g.adj, g.eoff, s.thr, e->eps, s.sim, s.role, s.parent,
        s.ctr);
    e->launches++;
    e->release(ipre);
  } else if (g.m > 0) {  // ... or by a sweep over every edge (sharded, or GS_SPARSE_CLUSTER=0)
    GS_TRY(ensure_endpoints(e));
    k_union_known<<<gridv(e, g.m), 256, 0, e->stream>>>(g.m, g.elo, g.ehi, s.sim, s.role, s.parent,
                                                       s.ctr, e->shard_rank, e->shard_world);
    e->launches++;
  }
  return run_similarity(e, MODE_UNION, e->eps, e->mu);
}

int phase_export_pairs(gs_engine* e, int32_t* pairs, int64_t* npairs) {
  *npairs = 0;
  if (e->ncores == 0 || e->g.n == 0) return GS_OK;
  DevState& s = e->s;
  unsigned long long* cnt = nullptr;
  GS_TRY(e->alloc_n(&cnt, 1));
  GS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), e->stream));
  k_export_pairs<<<gridv(e, e->g.n), 256, 0, e->stream>>>(e->g.n, s.role, s.parent, pairs, cnt);
  e->launches++;
  unsigned long long h = 0;
  GS_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, e->stream));
  GS_CUDA(cudaStreamSynchronize(e->stream));
  e->release(cnt);
  *npairs = (int64_t)h;
  return GS_OK;
}

int phase_merge_pairs(gs_engine* e, const int32_t* pairs, int64_t npairs) {
  if (e->ncores == 0 || e->g.n == 0) return GS_OK;
  DevState& s = e->s;
  k_singletons<<<gridv(e, e->g.n), 256, 0, e->stream>>>(e->g.n, s.role, s.parent, nullptr);
  e->launches++;
  if (npairs > 0) {
    k_union_pairs<<<gridv(e, npairs), 256, 0, e->stream>>>(npairs, pairs, s.parent, s.ctr);
    e->launches++;
  }
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// flatten + canonical labels (min caller id per class); member labels init
int phase_labels(gs_engine* e) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  const int64_t n = g.n;
  if (n == 0) return GS_OK;
  if (e->ncores > 0) {
    k_flatten<<<gridv(e, n), 256, 0, e->stream>>>(n, s.role, s.parent, g.orig, s.label, s.ctr);
    e->launches++;
  }
  k_core_labels<<<gridv(e, n), 256, 0, e->stream>>>(n, s.role, s.parent, s.label, s.lmin, s.lmax);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// member attachment over this shard's similar core-noncore edges
// flag[w] = 1 for every neighbour w of a vertex v with key[v] >= 0 (cores:
// role; clustered vertices: lmax).  Ranks [0, rh) one warp per vertex, the
// heavy ranks [rh, n) (degree >= 512) one CTA per vertex, so a hub's list does
// not serialise on one warp.  The attach pass skips the b's whose owned edges
// cannot join a core and a non-core; classify skips the hub scan of vertices
// with no clustered neighbour.
template <bool CORES>
__global__ void k_flag_neighbours(int64_t rlo, int64_t rhi, bool per_cta,
                                  const int64_t* __restrict__ off,
                                  const int32_t* __restrict__ adj,
                                  const uint8_t* __restrict__ role,
                                  const int32_t* __restrict__ lmax, uint8_t* __restrict__ flag) {
  const int lane = per_cta ? threadIdx.x : (threadIdx.x & 31);
  const int step = per_cta ? blockDim.x : 32;
  const int64_t g0 = per_cta ? blockIdx.x : (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ng = per_cta ? gridDim.x : ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = rlo + g0; v < rhi; v += ng) {
    if (CORES ? role[v] != ROLE_CORE : lmax[v] < 0) continue;
    for (int64_t i = off[v] + lane; i < off[v + 1]; i += step) flag[adj[i]] = 1;
  }
}

__global__ void k_clustered_degree(int64_t n, const int64_t* __restrict__ off,
                                   const int32_t* __restrict__ lmax,
                                   unsigned long long* __restrict__ sum) {
  unsigned long long acc = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    if (lmax[v] >= 0) acc += (unsigned long long)(off[v + 1] - off[v]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(sum, acc);
}

template <bool CORES>
static void flag_neighbours(gs_engine* e, uint8_t* flag) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  const int64_t n = g.n, rh = g.rclass[2];
  if (rh > 0)
    k_flag_neighbours<CORES><<<(unsigned)std::min<int64_t>(grid_for(rh * 32, 256),
                                                            (int64_t)e->sms * 64),
                               256, 0, e->stream>>>(0, rh, false, g.off, g.adj, s.role, s.lmax,
                                                    flag);
  if (n > rh)
    k_flag_neighbours<CORES><<<(unsigned)std::min<int64_t>(n - rh, (int64_t)e->sms * 16), 256, 0,
                               e->stream>>>(rh, n, true, g.off, g.adj, s.role, s.lmax, flag);
  e->launches += 2;
}

int phase_attach(gs_engine* e) {
  if (e->ncores == 0) return GS_OK;
  DevGraph& g = e->g;
  DevState& s = e->s;
  if (s.sparse) {
    int32_t* ipre = nullptr;
    GS_TRY(list_chunks(e, (int64_t)e->ncores, s.lcnt, s.clist, false, &ipre));
    k_attach_sparse<true><<<(unsigned)e->sms * 16, 256, 0, e->stream>>>(s.lcnt, s.clist, ipre, g.off,
                                                                 g.adj, g.eoff, s.thr, e->eps,
                                                                 s.sim, s.role, s.lmin, s.lmax,
                                                                 s.ctr);
    e->launches++;
    e->release(ipre);
    GS_CUDA(cudaGetLastError());
    return GS_OK;
  }
  if (!s.coreadj) GS_TRY(e->alloc_n(&s.coreadj, (g.n + 3) & ~int64_t(3)));
  GS_CUDA(cudaMemsetAsync(s.coreadj, 0, (size_t)(g.n > 0 ? g.n : 1), e->stream));
  // with the core list (single GPU): the cores' neighbours flagged and the
  // known-similar edges attached from the cores' runs instead of sweeping
  // every vertex / every edge
  int32_t* ipre = nullptr;
  if (g.m > 0 && s.clist) {
    GS_TRY(list_chunks(e, (int64_t)e->ncores, s.lcnt, s.clist, false, &ipre));
    k_flag_list<<<(unsigned)e->sms * 16, 256, 0, e->stream>>>(s.lcnt, s.clist, ipre, g.off, g.adj,
                                                             s.coreadj);
    e->launches++;
  } else if (g.n > 0) {
    flag_neighbours<true>(e, s.coreadj);
  }
  GS_TRY(run_similarity(e, MODE_ATTACH, e->eps, e->mu));
  if (ipre) {
    k_attach_sparse<false><<<(unsigned)e->sms * 16, 256, 0, e->stream>>>(
        s.lcnt, s.clist, ipre, g.off, g.adj, g.eoff, s.thr, e->eps, s.sim, s.role, s.lmin, s.lmax,
        s.ctr);
    e->launches++;
    e->release(ipre);
  } else if (g.m > 0) {
    GS_TRY(ensure_endpoints(e));
    k_attach<<<gridv(e, g.m), 256, 0, e->stream>>>(g.m, g.elo, g.ehi, s.sim, s.role, s.lmin, s.lmax,
                                                  e->shard_rank, e->shard_world);
    e->launches++;
  }
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

int phase_export_labels(gs_engine* e, int32_t* labels) {
  const size_t b = sizeof(int32_t) * (size_t)e->g.n;
  if (b == 0) return GS_OK;
  GS_CUDA(cudaMemcpyAsync(labels, e->s.lmin, b, cudaMemcpyDeviceToDevice, e->stream));
  GS_CUDA(cudaMemcpyAsync(labels + e->g.n, e->s.lmax, b, cudaMemcpyDeviceToDevice, e->stream));
  return GS_OK;
}

int phase_import_labels(gs_engine* e, const int32_t* labels) {
  const size_t b = sizeof(int32_t) * (size_t)e->g.n;
  if (b == 0) return GS_OK;
  GS_CUDA(cudaMemcpyAsync(e->s.lmin, labels, b, cudaMemcpyDeviceToDevice, e->stream));
  GS_CUDA(cudaMemcpyAsync(e->s.lmax, labels + e->g.n, b, cudaMemcpyDeviceToDevice, e->stream));
  return GS_OK;
}

// phase 3 (Alg. 4) and the result scatter to caller ids
int phase_finish(gs_engine* e, uint8_t* role_out, int32_t* cluster_out, int out_on_device,
                 gs_stats* st) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  cudaStream_t str = e->stream;
  const int64_t n = g.n, m = g.m;
  uint8_t* fin = nullptr;
  GS_TRY(e->alloc_n(&fin, n));
  uint8_t* d_role_out = role_out;
  int32_t* d_cluster_out = cluster_out;
  if (!out_on_device) {
    d_role_out = nullptr;
    d_cluster_out = nullptr;
    if (role_out) GS_TRY(e->alloc_n(&d_role_out, n));
    if (cluster_out) GS_TRY(e->alloc_n(&d_cluster_out, n));
  }
  const int64_t rsplit = e->ncores > 0 ? g.rclass[1] : 0;
  // From the clustered side when its arcs are few: the clustered vertices are
  // listed (their roles set), their unclustered neighbours listed once each
  // and only those scanned for a hub; everyone else is an outlier.
  bool listed = false;
  if (e->ncores > 0 && n > 0 && sparse_mode() != 0) {
    int32_t* clu = nullptr;
    unsigned long long* dsum = nullptr;
    int* cnt = nullptr;
    GS_TRY(e->alloc_n(&clu, n));
    GS_TRY(e->alloc_n(&dsum, 2));
    GS_TRY(e->alloc_n(&cnt, 2));
    GS_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), str));
    GS_CUDA(cudaMemsetAsync(dsum, 0, 2 * sizeof(unsigned long long), str));
    k_clustered_list<<<gridv(e, n), 256, 0, str>>>(n, s.lmax, clu, cnt, dsum, g.off);
    unsigned long long h[2] = {0, 0};
    int hc = 0;
    GS_CUDA(cudaMemcpyAsync(h, dsum, sizeof(h), cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaMemcpyAsync(&hc, cnt, sizeof(int), cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaStreamSynchronize(str));
    e->launches++;
    static const int64_t list_div = getenv("GS_LIST_DIV") ? atoll(getenv("GS_LIST_DIV")) : kListDiv;
    listed = sparse_mode() == 1 || (int64_t)h[0] <= 2 * m / std::max<int64_t>(list_div, 1);
    if (listed) {
      int32_t* nearl = nullptr;
      GS_TRY(e->alloc_n(&nearl, n));
      if (!s.coreadj) GS_TRY(e->alloc_n(&s.coreadj, (n + 3) & ~int64_t(3)));
      GS_CUDA(cudaMemsetAsync(s.coreadj, 0, (size_t)((n + 3) & ~int64_t(3)), str));
      GS_CUDA(cudaMemsetAsync(fin, ROLE_OUTLIER, (size_t)n, str));
      const unsigned gw = (unsigned)std::min<int64_t>(grid_for((int64_t)n * 32, 256), (int64_t)e->sms * 16);
      int32_t* ipre = nullptr;
      int32_t* hacc = nullptr;  // per vertex: clustered-neighbour count, min / max label
      GS_TRY(e->alloc_n(&hacc, 3 * n));
      GS_CUDA(cudaMemsetAsync(hacc, 0, sizeof(int32_t) * 3 * (size_t)n, str));
      GS_TRY(list_chunks(e, std::max(hc, 1), cnt, clu, false, &ipre));
      k_near_list<<<gw, 256, 0, str>>>(cnt, clu, ipre, g.off, g.adj, s.lmax, s.role, s.coreadj,
                                       nearl, cnt + 1, fin, s.lmin, hacc, n);
      e->release(ipre);
      k_classify_near<<<gridv(e, n), 256, 0, str>>>(cnt + 1, nearl, hacc, n, fin);
      e->launches += 2;
      e->release(hacc);
      GS_CUDA(cudaGetLastError());
      GS_CUDA(cudaStreamSynchronize(str));  // the lists are released below
      e->release(nearl);
    }
    e->release(clu);
    e->release(dsum);
    e->release(cnt);
  }
  // near[v]: v has a clustered neighbour (only those can be hubs).  Flagging
  // costs the clustered vertices' degrees, the hub scan it saves the rest's:
  // flag only when the clustered side is the smaller one.
  bool use_near = false;
  if (!listed && e->ncores > 0 && n > 0) {
    unsigned long long* d_sum = nullptr;
    GS_TRY(e->alloc_n(&d_sum, 1));
    GS_CUDA(cudaMemsetAsync(d_sum, 0, sizeof(unsigned long long), str));
    k_clustered_degree<<<gridv(e, n), 256, 0, str>>>(n, g.off, s.lmax, d_sum);
    unsigned long long h_sum = 0;
    GS_CUDA(cudaMemcpyAsync(&h_sum, d_sum, sizeof(h_sum), cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaStreamSynchronize(str));
    e->release(d_sum);
    e->launches++;
    use_near = (int64_t)h_sum < g.m;  // < half of the 2m arcs
    if (use_near) {
      if (!s.coreadj) GS_TRY(e->alloc_n(&s.coreadj, (n + 3) & ~int64_t(3)));
      GS_CUDA(cudaMemsetAsync(s.coreadj, 0, (size_t)n, str));
      flag_neighbours<false>(e, s.coreadj);
    }
  }
  const uint8_t* near = use_near ? s.coreadj : nullptr;
  if (e->ncores == 0 && n > 0)  // nothing is clustered: every vertex is an outlier
    GS_CUDA(cudaMemsetAsync(fin, ROLE_OUTLIER, (size_t)n, str));
  if (rsplit > 0 && !listed) {
    k_classify_thread<<<gridv(e, rsplit), 256, 0, str>>>(0, rsplit, g.off, g.adj, s.role, s.lmin,
                                                        s.lmax, near, fin);
    e->launches++;
  }
  if (e->ncores > 0 && n > rsplit && !listed) {
    k_classify_warp<<<gridv(e, (n - rsplit) * 32), 256, 0, str>>>(rsplit, n, g.off, g.adj, s.role,
                                                                 s.lmin, s.lmax, near, fin);
    e->launches++;
  }
  cudaEvent_t c0, c1;
  cudaEventCreate(&c0);
  cudaEventCreate(&c1);
  cudaEventRecord(c0, str);
  if (n > 0) {
    k_output<<<gridv(e, n), 256, 0, str>>>(n, g.orig, fin, s.lmin, d_role_out, d_cluster_out, s.ctr);
    e->launches++;
  }
  if (!out_on_device) {
    if (role_out && n > 0)
      GS_CUDA(cudaMemcpyAsync(role_out, d_role_out, (size_t)n, cudaMemcpyDeviceToHost, str));
    if (cluster_out && n > 0)
      GS_CUDA(cudaMemcpyAsync(cluster_out, d_cluster_out, (size_t)n * 4, cudaMemcpyDeviceToHost,
                              str));
  }
  cudaEventRecord(c1, str);
  unsigned long long h[CTR_COUNT];
  GS_CUDA(cudaMemcpyAsync(h, s.ctr, sizeof(h), cudaMemcpyDeviceToHost, str));
  GS_CUDA(cudaStreamSynchronize(str));
  GS_CUDA(cudaGetLastError());
  if (!out_on_device) {
    if (d_role_out) e->release(d_role_out);
    if (d_cluster_out) e->release(d_cluster_out);
  }
  if (n > 0)  // final roles stay on the device (state export, scan.py ClusterState.role)
    GS_CUDA(cudaMemcpyAsync(s.role, fin, (size_t)n, cudaMemcpyDeviceToDevice, str));
  GS_CUDA(cudaStreamSynchronize(str));
  e->release(fin);
  if (st) {
    float d2h = 0;
    cudaEventElapsedTime(&d2h, c0, c1);
    fill_counters(st, n, m, h);
    st->phase_ms[GS_PH_D2H] = d2h;
  }
  cudaEventDestroy(c0);
  cudaEventDestroy(c1);
  return GS_OK;
}

void fill_counters(gs_stats* st, int64_t n, int64_t m, const unsigned long long* h) {
    st->n = n;
    st->m = m;
    st->sim_evals = (int64_t)h[CTR_SIM_EVALS];
    st->adj_probes = (int64_t)h[CTR_PROBES];
    st->union_retries = (int64_t)h[CTR_UNION_RETRIES];
    st->probe_bound_violations = 0;
    st->sim_decided_by_bound = (int64_t)h[CTR_BOUND_DECIDED];
    st->sim_intersections = (int64_t)h[CTR_INTERSECTIONS];
    st->alg_bytes_sim = (int64_t)h[CTR_ALG_BYTES];
    st->n_core = (int64_t)h[CTR_N_CORE];
    st->n_member = (int64_t)h[CTR_N_MEMBER];
    st->n_hub = (int64_t)h[CTR_N_HUB];
    st->n_outlier = (int64_t)h[CTR_N_OUTLIER];
    st->n_clusters = (int64_t)h[CTR_N_CLUSTERS];
    st->sim_decided_by_sketch = (int64_t)h[CTR_SKETCH_DECIDED];
    int64_t tot = 0;
    for (int c = 0; c < kKernelClasses; ++c) {
      st->kernel_bytes[c] = (int64_t)h[CTR_B_PREP + c];
      tot += st->kernel_bytes[c];
    }
    // the state initialisation of phase_begin (memset of sim[m] and label[n])
    if (h[CTR_B_PREP]) {
      st->kernel_bytes[0] += m + 4 * n;
      tot += m + 4 * n;
    }
    st->alg_bytes_sim = tot;
    st->wsim_bytes = h[CTR_WSIM] ? (int64_t)h[CTR_WSIM] + 9 * st->sim_evals + 8 * (n + 1) : 0;
    st->pcie_bytes = (int64_t)h[CTR_PCIE];
}

int read_counters(gs_engine* e, gs_stats* st) {
  unsigned long long h[CTR_COUNT] = {0};
  if (e->s.ctr) {
    GS_CUDA(cudaMemcpyAsync(h, e->s.ctr, sizeof(h), cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
  }
  fill_counters(st, e->g.n, e->g.m, h);
  return GS_OK;
}

// the single-GPU scan: every phase in a row, no exchange
int run_scan(gs_engine* e, int32_t mu, const Eps2& eps, uint8_t* role_out,
             int32_t* cluster_out, int out_on_device, gs_stats* st) {
  PhaseTimer tm(e);
  e->kev_on = st != nullptr;
  tm.mark();  // 0
  GS_TRY(phase_begin(e, mu, eps));
  GS_TRY(phase_identify(e));
  tm.mark();  // 1
  GS_TRY(phase_resolve(e, e->shard_world == 1));
  tm.mark();  // 2
  GS_TRY(phase_union(e));
  GS_TRY(phase_labels(e));
  GS_TRY(phase_attach(e));
  tm.mark();  // 3
  tm.mark();  // 4 (classify is timed inside finish with the output scatter)
  GS_TRY(phase_finish(e, role_out, cluster_out, out_on_device, st));
  tm.mark();  // 5
  GS_CUDA(cudaStreamSynchronize(e->stream));
  if (st) {
    st->phase_ms[GS_PH_IDENTIFY] = tm.ms(0, 1);
    st->phase_ms[GS_PH_CLEANUP] = tm.ms(1, 2);
    st->phase_ms[GS_PH_CLUSTER] = tm.ms(2, 3);
    st->phase_ms[GS_PH_CLASSIFY] = tm.ms(4, 5) - st->phase_ms[GS_PH_D2H];
    e->kev_class_ms(st->phase_ms + GS_PH_K_PREP);
  }
  e->kev_on = false;
  return GS_OK;
}


// ---------------------------------------------------------------------------
// ClusterState export (scan.py:87-134): the device state re-expressed in the
// reference's per-vertex layout, indexed by caller ids.
//   stage 0 (after identify_core): lower/upper, role core|noncore, parent -2
//   stage 1 (after detect_clusters): + members (3, shared 4), parent = the
//            canonical cluster label (a core id; its own parent)
//   stage 2 (after classify_hub_outlier): + hubs (5, parent -1), outliers (6)
__global__ void k_export_vertices(int64_t n, int stage, const int32_t* __restrict__ orig,
                                  const uint64_t* __restrict__ bounds,
                                  const uint8_t* __restrict__ role,
                                  const int32_t* __restrict__ lmin,
                                  const int32_t* __restrict__ lmax, int32_t* __restrict__ lower,
                                  int32_t* __restrict__ upper, uint8_t* __restrict__ role_out,
                                  int32_t* __restrict__ parent_out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = orig[v];
    const uint64_t b = bounds[v];
    lower[o] = (int32_t)(uint32_t)b;
    upper[o] = (int32_t)(uint32_t)(b >> 32);
    uint8_t r = role[v];
    int32_t par = -2;
    if (stage >= 1) {
      const bool clustered = lmin[v] != 0x7fffffff;
      if (stage == 1 && r == ROLE_NONCORE && clustered) r = ROLE_MEMBER;
      if (r == ROLE_MEMBER && lmin[v] != lmax[v]) r = 4;  // ROLE_MEMBER_SHARED
      if (r == ROLE_CORE || r == ROLE_MEMBER || r == 4) par = lmin[v];
      else if (r == ROLE_HUB) par = -1;
    }
    role_out[o] = r;
    parent_out[o] = par;
  }
}

// per oriented edge: status (O(1)-decided edges, folded into the initial
// bounds by the pre-pass, get their status here) and the caller-id pair
__global__ void k_export_edges(int64_t m, const int32_t* __restrict__ elo,
                               const int32_t* __restrict__ ehi, const int32_t* __restrict__ orig,
                               const int64_t* __restrict__ off, const int2* __restrict__ thr,
                               const uint8_t* __restrict__ sim, uint8_t* __restrict__ sim_out,
                               int32_t* __restrict__ pairs) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = elo[e], b = ehi[e];
    uint8_t st = sim[e];
    if (st == SIM_UNKNOWN && thr) {
      const int64_t da = off[a + 1] - off[a], db = off[b + 1] - off[b];
      const int2 t = thr[db];
      if (da + 1 < t.x) st = SIM_DISSIMILAR;
      else if (da <= t.y) st = SIM_SIMILAR;
    }
    if (sim_out) sim_out[e] = st;
    if (pairs) {
      pairs[2 * e] = orig[a];
      pairs[2 * e + 1] = orig[b];
    }
  }
}

int export_state(gs_engine* e, int stage, int32_t* lower, int32_t* upper, uint8_t* role,
                 int32_t* parent, uint8_t* sim, int32_t* pairs) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  cudaStream_t str = e->stream;
  const int64_t n = g.n, m = g.m;
  if (!s.bounds) { set_error("no scan state: run the identify phase first"); return GS_EINVAL; }
  if (n > 0 && (lower || upper || role || parent)) {
    int32_t *dl = nullptr, *du = nullptr, *dp = nullptr;
    uint8_t* dr = nullptr;
    GS_TRY(e->alloc_n(&dl, n));
    GS_TRY(e->alloc_n(&du, n));
    GS_TRY(e->alloc_n(&dp, n));
    GS_TRY(e->alloc_n(&dr, n));
    k_export_vertices<<<gridv(e, n), 256, 0, str>>>(n, stage, g.orig, s.bounds, s.role, s.lmin,
                                                    s.lmax, dl, du, dr, dp);
    e->launches++;
    if (lower) GS_CUDA(cudaMemcpyAsync(lower, dl, 4 * (size_t)n, cudaMemcpyDeviceToHost, str));
    if (upper) GS_CUDA(cudaMemcpyAsync(upper, du, 4 * (size_t)n, cudaMemcpyDeviceToHost, str));
    if (parent) GS_CUDA(cudaMemcpyAsync(parent, dp, 4 * (size_t)n, cudaMemcpyDeviceToHost, str));
    if (role) GS_CUDA(cudaMemcpyAsync(role, dr, (size_t)n, cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaStreamSynchronize(str));
    e->release(dl);
    e->release(du);
    e->release(dp);
    e->release(dr);
  }
  if (m > 0 && (sim || pairs)) {
    uint8_t* ds = nullptr;
    int32_t* dpairs = nullptr;
    if (sim) GS_TRY(e->alloc_n(&ds, m));
    if (pairs) GS_TRY(e->alloc_n(&dpairs, 2 * m));
    GS_TRY(ensure_endpoints(e));
    k_export_edges<<<gridv(e, m), 256, 0, str>>>(m, g.elo, g.ehi, g.orig, g.off, s.thr, s.sim, ds,
                                                 dpairs);
    e->launches++;
    if (sim) GS_CUDA(cudaMemcpyAsync(sim, ds, (size_t)m, cudaMemcpyDeviceToHost, str));
    if (pairs) GS_CUDA(cudaMemcpyAsync(pairs, dpairs, 8 * (size_t)m, cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaStreamSynchronize(str));
    if (ds) e->release(ds);
    if (dpairs) e->release(dpairs);
  }
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

}  // namespace gs
