// sim.cu -- the structural-similarity sweep (identifyCore, Alg. 2; the
// checkSim procedure, scan.py:203-233) and its reuse by the union and attach
// passes of detectClusters (Alg. 3, scan.py:621-698).
//
// Work is grouped by the HIGH-degree endpoint b of each oriented edge (a, b):
//   * tiny b   (deg < 64)          one thread per edge, merge of two short runs
//   * small/medium/large b         one CTA per b (persistent, largest first):
//        N(b) is staged once into a shared-memory open-addressing table,
//        then every a in b's owned prefix streams N(a) with coalesced loads,
//        one warp per a, probing the table; ballot/popc counts hits
//   * huge b   (deg >= 28672)      same, table in an L2-resident global slab
// Before any intersection the exact O(1) degree bounds decide the edge when
// c in [0, deg(a)-1] cannot change the answer, and during the scan the warp
// stops as soon as c >= c_min or c + remaining < c_min (exact, c_min is
// computed with the integer predicate).  Progressive pruning (Lemma 1): in
// MODE_IDENTIFY an edge whose endpoints both have a decided role is skipped.
#include "engine.cuh"

namespace gs {

static constexpr uint32_t kEmpty = 0xFFFFFFFFu;

__device__ __forceinline__ uint8_t ld_role(const uint8_t* role, int64_t v) {
  return *reinterpret_cast<const volatile uint8_t*>(role + v);
}

__device__ __forceinline__ int32_t uf_find(int32_t* parent, int32_t x) {
  volatile int32_t* p = parent;
  for (;;) {
    int32_t px = p[x];
    if (px == x) return x;
    int32_t gp = p[px];
    if (gp == px) return px;
    p[x] = gp;  // path halving: gp is an ancestor of x, safe under races
    x = gp;
  }
}

// Lock-free union: hook the larger root under the smaller (roots are then the
// minimum rank of their class; parent[v] <= v keeps the forest acyclic).
__device__ __forceinline__ void uf_union(int32_t* parent, int32_t a, int32_t b,
                                         unsigned long long& retries) {
  for (;;) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a > b) { int32_t t = a; a = b; b = t; }
    int32_t old = atomicCAS(&parent[b], b, a);
    if (old == b) return;
    ++retries;
  }
}

// Apply nsim similar / ndis dissimilar outcomes to x's packed bounds and
// decide its role the moment a bound crosses mu (scan.py:302-345).
__device__ __forceinline__ void apply_bounds(uint64_t* bounds, uint8_t* role, int64_t x,
                                             uint32_t nsim, uint32_t ndis, int32_t mu) {
  const uint64_t delta = (uint64_t)nsim - ((uint64_t)ndis << 32);
  const uint64_t old = atomicAdd(reinterpret_cast<unsigned long long*>(&bounds[x]),
                                 (unsigned long long)delta);
  const uint64_t nw = old + delta;
  const int32_t lower = (int32_t)(uint32_t)nw;
  const int32_t upper = (int32_t)(uint32_t)(nw >> 32);
  if (lower >= mu) role[x] = ROLE_CORE;
  else if (upper < mu) role[x] = ROLE_NONCORE;
}

// Does edge (a, b) need a decision in this mode?
__device__ __forceinline__ bool edge_needed(const SimParams& P, int64_t e, int32_t a,
                                            int32_t b) {
  if (P.sim[e] != SIM_UNKNOWN) return false;
  const uint8_t ra = ld_role(P.role, a), rb = ld_role(P.role, b);
  switch (P.mode) {
    case MODE_IDENTIFY:  // Alg. 2 line 2: defer if both roles are known
      return ra == ROLE_UNKNOWN || rb == ROLE_UNKNOWN;
    case MODE_CLEANUP:
      return ra == ROLE_UNKNOWN || rb == ROLE_UNKNOWN;
    case MODE_UNION:  // scan.py:642-648
      if (ra != ROLE_CORE || rb != ROLE_CORE) return false;
      return uf_find(P.parent, a) != uf_find(P.parent, b);
    default:  // MODE_ATTACH, scan.py:681-686
      return (ra == ROLE_CORE) != (rb == ROLE_CORE);
  }
}

struct LocalCtr {
  unsigned long long evals = 0, probes = 0, bound = 0, inters = 0, bytes = 0, retries = 0;
};

// Record one decided edge.  b's bound update is returned to the caller
// (aggregated per CTA for the shared-b kernels) unless apply_b is set.
__device__ __forceinline__ void record_edge(const SimParams& P, int64_t e, int32_t a,
                                            int32_t b, bool similar, bool apply_b,
                                            LocalCtr& lc) {
  P.sim[e] = similar ? SIM_SIMILAR : SIM_DISSIMILAR;
  lc.evals++;
  if (P.mode == MODE_IDENTIFY || P.mode == MODE_CLEANUP) {
    apply_bounds(P.bounds, P.role, a, similar ? 1u : 0u, similar ? 0u : 1u, P.mu);
    if (apply_b) apply_bounds(P.bounds, P.role, b, similar ? 1u : 0u, similar ? 0u : 1u, P.mu);
  } else if (P.mode == MODE_UNION && similar) {
    uf_union(P.parent, a, b, lc.retries);
  }
}

__device__ void flush_ctr(const SimParams& P, LocalCtr& lc) {
  // warp reduce then one atomic per warp
  unsigned long long v[6] = {lc.evals, lc.probes, lc.bound, lc.inters, lc.bytes, lc.retries};
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (v[0]) atomicAdd(&P.ctr[CTR_SIM_EVALS], v[0]);
    if (v[1]) atomicAdd(&P.ctr[CTR_PROBES], v[1]);
    if (v[2]) atomicAdd(&P.ctr[CTR_BOUND_DECIDED], v[2]);
    if (v[3]) atomicAdd(&P.ctr[CTR_INTERSECTIONS], v[3]);
    if (v[4]) atomicAdd(&P.ctr[CTR_ALG_BYTES], v[4]);
    if (v[5]) atomicAdd(&P.ctr[CTR_UNION_RETRIES], v[5]);
  }
}

// ---------------------------------------------------------------------------
// tiny b: one thread per high endpoint b (deg < 64), its owned edges in
// order, merging two short runs.  Walking b's edges sequentially lets each
// decision (b's bounds are applied immediately) prune b's later edges, the
// progressive deferral of Alg. 2 line 2.

__global__ void __launch_bounds__(256) k_sim_tiny(SimParams P, int64_t rlo, int64_t rhi) {
  LocalCtr lc;
  for (int64_t b = rlo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < rhi;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = P.eoff[b], e1 = P.eoff[b + 1];
    if (e0 == e1) continue;
    const int64_t ob = P.off[b], eb = P.off[b + 1], db = eb - ob;
    for (int64_t e = e0; e < e1; ++e) {
      const int32_t a = P.adj[ob + (e - e0)];
      if (!edge_needed(P, e, a, (int32_t)b)) continue;
      const int64_t ia0 = P.off[a], ea = P.off[a + 1];
      const int64_t da = ea - ia0;
      const int64_t cmax = da - 1;
      bool res;
      if (!is_similar(cmax, da, db, P.eps)) { res = false; lc.bound++; }
      else if (is_similar(0, da, db, P.eps)) { res = true; lc.bound++; }
      else {
        const int64_t cmin = c_min_exact(da, db, cmax, P.eps);
        int64_t c = 0, ia = ia0, ib = ob;
        res = false;
        while (ia < ea && ib < eb) {
          const int32_t x = P.adj[ia], y = P.adj[ib];
          if (x == y) { ++c; ++ia; ++ib; }
          else if (x < y) ++ia;
          else ++ib;
          if (c >= cmin) { res = true; break; }
          if (c + (ea - ia) < cmin) break;
        }
        lc.probes += (unsigned long long)(ia - ia0);
        lc.inters++;
        lc.bytes += 4ull * (unsigned long long)(da + db);
      }
      record_edge(P, e, a, (int32_t)b, res, true, lc);
    }
  }
  flush_ctr(P, lc);
}

// ---------------------------------------------------------------------------
// CTA per high endpoint b with a hash table of N(b)

// Bucketed open addressing: T buckets of 4 keys (16 B).  A key hashes to a
// bucket; inserters claim the bucket's slots in order 0..3 with atomicCAS and
// spill to the next bucket only when all four are taken, so slots fill as a
// prefix and a bucket whose last slot is empty ends a miss.  One 16-byte
// load answers almost every probe (load <= 0.55 keys/slot), which keeps the
// 32 lanes of a warp in lock-step instead of waiting for the longest
// linear-probing chain.
__device__ __forceinline__ void bucket_insert(uint32_t* tab, uint32_t T, uint32_t w) {
  uint32_t h = hslot(w, T);
  for (;;) {
    uint32_t* bk = tab + 4 * h;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint32_t old = atomicCAS(&bk[s], kEmpty, w);
      if (old == kEmpty || old == w) return;
    }
    h = (h + 1 == T) ? 0 : h + 1;
  }
}

template <bool GTAB>
__device__ __forceinline__ bool probe(const uint32_t* __restrict__ tab, uint32_t T, uint32_t w) {
  uint32_t h = hslot(w, T);
  for (;;) {
    // L2-resident tables are written with atomics at L2: bypass L1 (.cg)
    const uint4 q = GTAB ? __ldcg(reinterpret_cast<const uint4*>(tab) + h)
                         : reinterpret_cast<const uint4*>(tab)[h];
    if (q.x == w || q.y == w || q.z == w || q.w == w) return true;
    if (q.w == kEmpty) return false;
    h = (h + 1 == T) ? 0 : h + 1;
  }
}

template <int NT, bool GTAB, int U>
__global__ void __launch_bounds__(NT) k_sim_hash(SimParams P, int64_t rlo, int64_t rhi,
                                                 uint32_t tcap, int qi, int chunk) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* table = GTAB ? (P.gtab + (int64_t)blockIdx.x * P.gtab_stride) : smem;
  // survivors of the O(1) filter: where N(a) starts, (a, deg a), (j, c_min)
  int64_t* surv_oa = reinterpret_cast<int64_t*>(smem + (GTAB ? 0 : 4 * (size_t)tcap));
  int2* surv_ad = reinterpret_cast<int2*>(surv_oa + chunk);
  int2* surv_jc = surv_ad + chunk;
  __shared__ int s_item, s_nsurv, s_next;
  __shared__ unsigned int s_bsim, s_bdis;
  const int tid = threadIdx.x, lane = tid & 31;
  LocalCtr lc;

  for (;;) {
    if (tid == 0) s_item = atomicAdd(&P.wq[qi], 1);
    __syncthreads();
    const int64_t b = rhi - 1 - (int64_t)s_item;
    if (b < rlo) break;
    const int64_t ob = P.off[b], db = P.off[b + 1] - ob;
    const int64_t e0 = P.eoff[b], nlow = P.eoff[b + 1] - e0;
    uint32_t T = (uint32_t)(db / 2 + 1);  // buckets: <= 0.5 keys per slot
    if (T > tcap) T = tcap;
    bool built = false;
    for (int64_t base = 0; base < nlow; base += chunk) {
      if (tid == 0) { s_nsurv = 0; s_next = 0; s_bsim = 0; s_bdis = 0; }
      __syncthreads();
      const int64_t lim = base + chunk < nlow ? base + chunk : nlow;
      // filter + O(1) bounds, one candidate a per thread
      for (int64_t j = base + tid; j < lim; j += NT) {
        const int64_t e = e0 + j;
        const int32_t a = P.adj[ob + j];
        if (!edge_needed(P, e, a, (int32_t)b)) continue;
        const int64_t oa = P.off[a];
        const int64_t da = P.off[a + 1] - oa;
        const int64_t cmax = da - 1;
        if (!is_similar(cmax, da, db, P.eps)) {
          lc.bound++;
          record_edge(P, e, a, (int32_t)b, false, false, lc);
          atomicAdd(&s_bdis, 1u);
        } else if (is_similar(0, da, db, P.eps)) {
          lc.bound++;
          record_edge(P, e, a, (int32_t)b, true, false, lc);
          atomicAdd(&s_bsim, 1u);
        } else {
          const int slot = atomicAdd(&s_nsurv, 1);
          surv_oa[slot] = oa;
          surv_ad[slot] = make_int2(a, (int32_t)da);
          surv_jc[slot] = make_int2((int32_t)j, (int32_t)c_min_exact(da, db, cmax, P.eps));
        }
      }
      __syncthreads();
      const int ns = s_nsurv;
      if (ns > 0) {
        if (!built) {  // stage N(b) once per b
          for (uint32_t i = tid; i < T; i += NT)
            reinterpret_cast<uint4*>(table)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
          __syncthreads();
          for (int64_t i = tid; i < db; i += NT) bucket_insert(table, T, (uint32_t)P.adj[ob + i]);
          __syncthreads();
          built = true;
          if (tid == 0) lc.bytes += 4ull * (unsigned long long)db;  // N(b) read once
        }
        // one warp per surviving a, dynamic
        for (;;) {
          int s = 0;
          if (lane == 0) s = atomicAdd(&s_next, 1);
          s = __shfl_sync(0xffffffffu, s, 0);
          if (s >= ns) break;
          const int2 jc = surv_jc[s];
          const int2 ad = surv_ad[s];
          const int64_t j = jc.x;
          const int32_t cmin = jc.y;
          const int32_t a = ad.x;
          const int64_t da = ad.y;
          const int32_t* __restrict__ na = P.adj + surv_oa[s];
          int32_t c = 0;
          int64_t scanned = 0;
          bool res = false;
          for (int64_t k0 = 0;; k0 += 32 * U) {
            int32_t w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int64_t idx = k0 + u * 32 + lane;
              w[u] = idx < da ? __ldg(na + idx) : -1;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const bool hit = w[u] >= 0 && probe<GTAB>(table, T, (uint32_t)w[u]);
              c += __popc(__ballot_sync(0xffffffffu, hit));
            }
            scanned = k0 + 32 * U < da ? k0 + 32 * U : da;
            if (c >= cmin) { res = true; break; }
            if ((int64_t)c + (da - scanned) < cmin) { res = false; break; }
          }
          if (lane == 0) {
            lc.probes += (unsigned long long)scanned;
            lc.inters++;
            lc.bytes += 4ull * (unsigned long long)da;
            record_edge(P, e0 + j, a, (int32_t)b, res, false, lc);
            atomicAdd(res ? &s_bsim : &s_bdis, 1u);
          }
        }
      }
      __syncthreads();
      if (tid == 0 && (s_bsim | s_bdis) &&
          (P.mode == MODE_IDENTIFY || P.mode == MODE_CLEANUP))
        apply_bounds(P.bounds, P.role, b, s_bsim, s_bdis, P.mu);
      __syncthreads();
    }
    __syncthreads();  // everyone has read s_item before it is rewritten
  }
  flush_ctr(P, lc);
}

// ---------------------------------------------------------------------------
// host driver

template <int NT, bool GTAB, int U>
static int launch_hash(gs_engine* e, const SimParams& P, int64_t rlo, int64_t rhi,
                       uint32_t tcap, int qi, int chunk) {
  if (rhi <= rlo) return GS_OK;
  const size_t smem = (GTAB ? 0 : (size_t)tcap * 16) + (size_t)chunk * 24;
  auto kern = k_sim_hash<NT, GTAB, U>;
  GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  GS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)occ * e->sms;
  if (grid > rhi - rlo) grid = rhi - rlo;
  if (GTAB && grid > e->sms * 2) grid = e->sms * 2;
  kern<<<(unsigned)grid, NT, smem, e->stream>>>(P, rlo, rhi, tcap, qi, chunk);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

int run_similarity(gs_engine* e, int mode, const Eps2& eps, int32_t mu) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  if (g.m == 0) return GS_OK;
  SimParams P;
  P.off = g.off;
  P.adj = g.adj;
  P.eoff = g.eoff;
  P.elo = g.elo;
  P.ehi = g.ehi;
  P.sim = s.sim;
  P.bounds = s.bounds;
  P.role = s.role;
  P.parent = s.parent;
  P.ctr = s.ctr;
  P.wq = s.wq;
  P.eps = eps;
  P.mu = mu;
  P.mode = mode;
  P.gtab = nullptr;
  P.gtab_stride = 0;
  GS_CUDA(cudaMemsetAsync(s.wq, 0, 8 * sizeof(int32_t), e->stream));
  const int64_t* rc = g.rclass;
  // huge b first (longest work items), with an L2-resident table per CTA
  const int64_t rhuge = rc[4];
  if (g.n > rhuge) {
    const int64_t tcap_g = g.dmax / 2 + 1;  // buckets
    const int64_t nblk = (int64_t)e->sms * 2;
    GS_TRY(e->alloc_n(&P.gtab, 4 * tcap_g * nblk));
    P.gtab_stride = 4 * tcap_g;
    GS_TRY((launch_hash<1024, true, 4>(e, P, rhuge, g.n, (uint32_t)tcap_g, 4, 1024)));
  }
  // table capacities in 16-byte buckets: large 12544 (196 KB, <= 0.572
  // keys/slot for deg < 28672), medium 2048 (32 KB), small 256 (4 KB);
  // survivor lists take 24 B per candidate of a chunk
  GS_TRY((launch_hash<1024, false, 4>(e, P, rc[3], rc[4], 12544, 3, 1024)));
  GS_TRY((launch_hash<256, false, 4>(e, P, rc[2], rc[3], 2048, 2, 512)));
  GS_TRY((launch_hash<128, false, 2>(e, P, rc[1], rc[2], 256, 1, 512)));
  if (rc[1] > rc[0]) {
    int64_t grid = (rc[1] - rc[0] + 255) / 256;
    if (grid > e->sms * 16) grid = e->sms * 16;
    k_sim_tiny<<<(unsigned)grid, 256, 0, e->stream>>>(P, rc[0], rc[1]);
    e->launches++;
    GS_CUDA(cudaGetLastError());
  }
  if (P.gtab) {
    GS_CUDA(cudaStreamSynchronize(e->stream));
    e->release(P.gtab);
  }
  return GS_OK;
}

}  // namespace gs
