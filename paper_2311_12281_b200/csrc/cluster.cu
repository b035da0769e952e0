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
#include "engine.cuh"

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
  if ((threadIdx.x & 31) == 0 && cores) atomicAdd(&ctr[CTR_CORES_PRE], cores);
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
                              unsigned long long* __restrict__ ctr) {
  unsigned long long retries = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (sim[e] != SIM_SIMILAR) continue;
    int32_t a = elo[e], b = ehi[e];
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
                         int32_t* __restrict__ lmax) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (sim[e] != SIM_SIMILAR) continue;
    const int32_t a = elo[e], b = ehi[e];
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
                                  uint8_t* __restrict__ fin) {
  for (int64_t v = rlo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < rhi;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] == ROLE_CORE) { fin[v] = ROLE_CORE; continue; }
    if (lmax[v] >= 0) { fin[v] = ROLE_MEMBER; continue; }
    int cnt = 0;
    int32_t umin = 0x7fffffff, umax = -1;
    hub_scan(adj, off[v], off[v + 1], lmin, lmax, cnt, umin, umax);
    fin[v] = (cnt >= 2 && umin != umax) ? ROLE_HUB : ROLE_OUTLIER;
  }
}

__global__ void k_classify_warp(int64_t rlo, int64_t rhi, const int64_t* __restrict__ off,
                                const int32_t* __restrict__ adj, const uint8_t* __restrict__ role,
                                const int32_t* __restrict__ lmin, const int32_t* __restrict__ lmax,
                                uint8_t* __restrict__ fin) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = rlo + wid; v < rhi; v += nw) {
    if (role[v] == ROLE_CORE) { if (lane == 0) fin[v] = ROLE_CORE; continue; }
    if (lmax[v] >= 0) { if (lane == 0) fin[v] = ROLE_MEMBER; continue; }
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

int run_scan(gs_engine* e, int32_t mu, const Eps2& eps, uint8_t* role_out,
             int32_t* cluster_out, int out_on_device, gs_stats* st) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  cudaStream_t str = e->stream;
  const int64_t n = g.n, m = g.m;
  const int T = 256;
  const unsigned gv = (unsigned)std::min<int64_t>(grid_for(n, T), (int64_t)e->sms * 32);
  const unsigned ge = (unsigned)std::min<int64_t>(grid_for(m, T), (int64_t)e->sms * 32);
  e->free_state();
  GS_TRY(e->alloc_n(&s.sim, m));
  GS_TRY(e->alloc_n(&s.bounds, n));
  GS_TRY(e->alloc_n(&s.role, n));
  GS_TRY(e->alloc_n(&s.parent, n));
  GS_TRY(e->alloc_n(&s.label, n));
  GS_TRY(e->alloc_n(&s.lmin, n));
  GS_TRY(e->alloc_n(&s.lmax, n));
  GS_TRY(e->alloc_n(&s.ctr, CTR_COUNT));
  GS_TRY(e->alloc_n(&s.wq, 8));
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
  PhaseTimer tm(e);
  tm.mark();  // 0
  GS_CUDA(cudaMemsetAsync(s.sim, 0, (size_t)(m > 0 ? m : 1), str));
  GS_CUDA(cudaMemsetAsync(s.ctr, 0, sizeof(unsigned long long) * CTR_COUNT, str));
  GS_CUDA(cudaMemsetAsync(s.label, 0x7f, sizeof(int32_t) * (size_t)(n > 0 ? n : 1), str));
  if (n > 0) {
    k_init_state<<<gv, T, 0, str>>>(g.off, n, mu, s.bounds, s.role);
    e->launches++;
  }
  // ---- phase 1: identify cores (Alg. 2)
  GS_TRY(prepare_similarity(e, eps));
  GS_TRY(run_similarity(e, MODE_IDENTIFY, eps, mu));
  tm.mark();  // 1
  // ---- cleanup (scan.py:415-449): resolve from bounds; re-evaluate if open
  if (n > 0) {
    k_resolve<<<gv, T, 0, str>>>(n, mu, s.bounds, s.role, s.ctr);
    e->launches++;
  }
  unsigned long long unresolved = 0;
  GS_CUDA(cudaMemcpyAsync(&unresolved, s.ctr + CTR_UNRESOLVED, sizeof(unresolved),
                          cudaMemcpyDeviceToHost, str));
  GS_CUDA(cudaStreamSynchronize(str));
  if (unresolved) {
    GS_CUDA(cudaMemsetAsync(s.ctr + CTR_UNRESOLVED, 0, sizeof(unsigned long long), str));
    GS_TRY(run_similarity(e, MODE_CLEANUP, eps, mu));
    k_resolve<<<gv, T, 0, str>>>(n, mu, s.bounds, s.role, s.ctr);
    e->launches++;
    GS_CUDA(cudaMemcpyAsync(&unresolved, s.ctr + CTR_UNRESOLVED, sizeof(unresolved),
                            cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaStreamSynchronize(str));
    if (unresolved) {
      set_error("role resolution incomplete after full edge sweep");
      return GS_EINTERNAL;
    }
  }
  tm.mark();  // 2
  // ---- phase 2: detect clusters (Alg. 3)
  unsigned long long ncores = 0;
  if (n > 0) {
    k_singletons<<<gv, T, 0, str>>>(n, s.role, s.parent, s.ctr);
    e->launches++;
    GS_CUDA(cudaMemcpyAsync(&ncores, s.ctr + CTR_CORES_PRE, sizeof(ncores),
                            cudaMemcpyDeviceToHost, str));
    GS_CUDA(cudaStreamSynchronize(str));
  }
  if (ncores > 0) {  // no core, no cluster: the union / attach passes have no edge
    if (m > 0) {
      k_union_known<<<ge, T, 0, str>>>(m, g.elo, g.ehi, s.sim, s.role, s.parent, s.ctr);
      e->launches++;
    }
    GS_TRY(run_similarity(e, MODE_UNION, eps, mu));
    k_flatten<<<gv, T, 0, str>>>(n, s.role, s.parent, g.orig, s.label, s.ctr);
    e->launches++;
  }
  if (n > 0) {
    k_core_labels<<<gv, T, 0, str>>>(n, s.role, s.parent, s.label, s.lmin, s.lmax);
    e->launches++;
  }
  if (ncores > 0) {
    GS_TRY(run_similarity(e, MODE_ATTACH, eps, mu));
    if (m > 0) {
      k_attach<<<ge, T, 0, str>>>(m, g.elo, g.ehi, s.sim, s.role, s.lmin, s.lmax);
      e->launches++;
    }
  }
  tm.mark();  // 3
  // ---- phase 3: hubs and outliers (Alg. 4)
  const int64_t rsplit = ncores > 0 ? g.rclass[1] : 0;
  if (ncores == 0 && n > 0)  // nothing is clustered: every vertex is an outlier
    GS_CUDA(cudaMemsetAsync(fin, ROLE_OUTLIER, (size_t)n, str));
  if (rsplit > 0) {
    k_classify_thread<<<(unsigned)std::min<int64_t>(grid_for(rsplit, T), (int64_t)e->sms * 32),
                        T, 0, str>>>(0, rsplit, g.off, g.adj, s.role, s.lmin, s.lmax, fin);
    e->launches++;
  }
  if (ncores > 0 && n > rsplit) {
    const int64_t nwarps = n - rsplit;
    k_classify_warp<<<(unsigned)std::min<int64_t>(grid_for(nwarps * 32, T), (int64_t)e->sms * 32),
                      T, 0, str>>>(rsplit, n, g.off, g.adj, s.role, s.lmin, s.lmax, fin);
    e->launches++;
  }
  tm.mark();  // 4
  if (n > 0) {
    k_output<<<gv, T, 0, str>>>(n, g.orig, fin, s.lmin, d_role_out, d_cluster_out, s.ctr);
    e->launches++;
  }
  if (!out_on_device) {
    if (role_out && n > 0)
      GS_CUDA(cudaMemcpyAsync(role_out, d_role_out, (size_t)n, cudaMemcpyDeviceToHost, str));
    if (cluster_out && n > 0)
      GS_CUDA(cudaMemcpyAsync(cluster_out, d_cluster_out, (size_t)n * 4, cudaMemcpyDeviceToHost,
                              str));
  }
  tm.mark();  // 5
  unsigned long long h[CTR_COUNT];
  GS_CUDA(cudaMemcpyAsync(h, s.ctr, sizeof(h), cudaMemcpyDeviceToHost, str));
  GS_CUDA(cudaStreamSynchronize(str));
  GS_CUDA(cudaGetLastError());
  if (!out_on_device) {
    if (d_role_out) e->release(d_role_out);
    if (d_cluster_out) e->release(d_cluster_out);
  }
  e->release(fin);
  if (st) {
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
    st->phase_ms[GS_PH_IDENTIFY] = tm.ms(0, 1);
    st->phase_ms[GS_PH_CLEANUP] = tm.ms(1, 2);
    st->phase_ms[GS_PH_CLUSTER] = tm.ms(2, 3);
    st->phase_ms[GS_PH_CLASSIFY] = tm.ms(3, 4);
    st->phase_ms[GS_PH_D2H] = tm.ms(4, 5);
  }
  return GS_OK;
}

}  // namespace gs
