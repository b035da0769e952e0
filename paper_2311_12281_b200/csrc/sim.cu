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
#include <algorithm>

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

// Two-choice bucketed cuckoo table: T buckets of 4 keys (16 B).  Every key
// lives in one of its two buckets h1(w), h2(w), so a lookup is exactly two
// independent 16-byte loads and eight compares -- no probe loop, so the 32
// lanes of a warp never wait for the longest chain.  The CTA builds it in
// parallel: claim an empty slot with atomicCAS in either bucket, otherwise
// atomicExch a resident key out and re-home it in its other bucket.  A key
// still homeless after kMaxKicks goes to a small shared stash; if the stash
// overflows the b is marked and lookups fall back to binary search of N(b)
// (exact, never taken at the load factors used here, <= 0.6 keys/slot).
static constexpr int kMaxKicks = 64;
static constexpr int kStash = 32;

struct Cuckoo {
  uint32_t* tab;      // 4*T words (shared or global)
  uint32_t T;
  int* nstash;        // shared
  uint32_t* stash;    // shared [kStash]
};

__device__ __forceinline__ uint32_t h1_of(uint32_t x, uint32_t T) { return __umulhi(x, T); }
__device__ __forceinline__ uint32_t h2_of(uint32_t x, uint32_t T) {
  return __umulhi(x * 0x85EBCA6Bu ^ (x >> 15), T);
}

__device__ __forceinline__ void cuckoo_insert(const Cuckoo& C, uint32_t w) {
  uint32_t key = w;
  uint32_t x = key * 0x9E3779B1u;
  uint32_t h = h1_of(x, C.T);
  for (int kick = 0; kick < kMaxKicks; ++kick) {
    const uint32_t ha = h1_of(x, C.T), hb = h2_of(x, C.T);
    const uint32_t alt = (h == ha) ? hb : ha;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      uint32_t* bk = C.tab + 4 * (pass == 0 ? h : alt);
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (atomicCAS(&bk[s], kEmpty, key) == kEmpty) return;
    }
    // both buckets full: displace a resident of `alt` and re-home it
    const uint32_t victim = atomicExch(&C.tab[4 * alt + (kick & 3)], key);
    if (victim == kEmpty) return;
    key = victim;
    x = key * 0x9E3779B1u;
    const uint32_t va = h1_of(x, C.T), vb = h2_of(x, C.T);
    h = (alt == va) ? vb : va;  // the victim's other bucket
  }
  const int i = atomicAdd(C.nstash, 1);
  if (i < kStash) C.stash[i] = key;
}

template <bool GTAB>
__device__ __forceinline__ bool cuckoo_find(const Cuckoo& C, uint32_t w, int nstash,
                                            const int32_t* __restrict__ nb, int64_t db) {
  const uint32_t x = w * 0x9E3779B1u;
  const uint4* t4 = reinterpret_cast<const uint4*>(C.tab);
  const uint32_t ha = h1_of(x, C.T), hb = h2_of(x, C.T);
  // L2-resident tables are written with atomics at L2: bypass L1 (.cg)
  const uint4 p = GTAB ? __ldcg(t4 + ha) : t4[ha];
  const uint4 q = GTAB ? __ldcg(t4 + hb) : t4[hb];
  bool hit = (p.x == w) | (p.y == w) | (p.z == w) | (p.w == w) | (q.x == w) | (q.y == w) |
             (q.z == w) | (q.w == w);
  if (nstash > 0) {  // CTA-uniform
    if (nstash <= kStash) {
      for (int i = 0; i < nstash; ++i) hit |= (C.stash[i] == w);
    } else {  // stash overflow: exact binary search of sorted N(b)
      int64_t lo = 0, hi = db;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((uint32_t)nb[mid] < w) lo = mid + 1; else hi = mid;
      }
      hit = lo < db && (uint32_t)nb[lo] == w;
    }
  }
  return hit;
}

// Per-b O(1) thresholds (exact): with cmax = deg(a) - 1,
//   dissimilar without intersecting  iff (da+1) q <  p (db+1)  iff da + 1 < xmin_b
//   similar without intersecting     iff 4 q >= p (da+1)(db+1)  iff da <= simmax_b
__device__ __forceinline__ void b_thresholds(int64_t db, const Eps2& e, int64_t& xmin,
                                             int64_t& simmax) {
  double est = e.ratio * (double)(db + 1);
  int64_t x = (int64_t)est;
  if (x < 1) x = 1;
  while (x > 1 && pred_ge((uint64_t)(x - 1), (uint64_t)(db + 1), e)) --x;
  while (!pred_ge((uint64_t)x, (uint64_t)(db + 1), e)) ++x;
  xmin = x;
  double es = 4.0 / (e.ratio * (double)(db + 1)) - 1.0;
  int64_t d = es < 0 ? -1 : (int64_t)(es > 4e18 ? 4e18 : es);
  if (d > (int64_t)1 << 40) d = (int64_t)1 << 40;
  while (d >= 0 && !pred_ge(4, (uint64_t)(d + 1) * (uint64_t)(db + 1), e)) --d;
  while (pred_ge(4, (uint64_t)(d + 2) * (uint64_t)(db + 1), e) && d < ((int64_t)1 << 40)) ++d;
  simmax = d;
}

// per-degree table of the O(1) thresholds, computed once per scan
__global__ void k_thresholds(int64_t dmax, Eps2 e, int2* __restrict__ thr) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d <= dmax;
       d += (int64_t)gridDim.x * blockDim.x) {
    int64_t xmin, simmax;
    b_thresholds(d, e, xmin, simmax);
    thr[d] = make_int2((int32_t)(xmin > 0x7fffffff ? 0x7fffffff : xmin),
                       (int32_t)(simmax > 0x7fffffff ? 0x7fffffff : simmax));
  }
}

// per-vertex split of the adjacency run at hub_lo (runs are sorted)
__global__ void k_hubsplit(const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                           int64_t n, uint32_t hub_lo, int32_t* __restrict__ nlo) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = off[v], h = off[v + 1];
    const int64_t lo0 = l;
    while (l < h) {
      const int64_t mid = (l + h) >> 1;
      if ((uint32_t)adj[mid] < hub_lo) l = mid + 1; else h = mid;
    }
    nlo[v] = (int32_t)(l - lo0);
  }
}

// Membership structure for N(b), per CTA:
//   * a direct-mapped bitmap over the top R ranks [hub_lo, n) in shared
//     memory: the high-degree vertices hold almost every element a warp
//     scans (N(a) is walked from its high-rank end), one LDS + bit test each
//   * a two-choice cuckoo table for the rest of N(b)
template <bool GTAB>
__device__ __forceinline__ bool member(const uint32_t* bm, uint32_t hub_lo, const Cuckoo& C,
                                       uint32_t w, int nstash, const int32_t* __restrict__ nb,
                                       int64_t nlo) {
  if (w >= hub_lo) {
    const uint32_t r = w - hub_lo;
    return (bm[r >> 5] >> (r & 31)) & 1u;
  }
  return cuckoo_find<GTAB>(C, w, nstash, nb, nlo);
}

// Decide one surviving edge (a, b): a warp walks N(a) from its high-rank
// end (hubs first).  The first step covers 32 elements -- a survivor near the
// degree bound is rejected after one or two misses -- later steps 128 (4
// coalesced loads per lane); the next step is prefetched only when this one
// cannot decide the edge.  Steps whose elements all lie in the hub range
// (warp vote) take a branch-free bitmap path; past-the-end slots hold a
// sentinel >= n that lands on an always-zero bitmap guard word.
template <bool GTAB>
__device__ __forceinline__ bool scan_survivor(const int32_t* __restrict__ a_run, int32_t da,
                                              int32_t cmin, const uint32_t* bm, uint32_t hub_lo,
                                              uint32_t rmax, const Cuckoo& C, int nstash,
                                              const int32_t* __restrict__ nb, int64_t nlo,
                                              int lane, int32_t& scanned) {
  const int32_t* __restrict__ na = a_run + (da - 1);  // walk downwards
  const int32_t need_miss = da - cmin + 1;            // misses that decide "dissimilar"
  constexpr uint32_t kPast = 0x7fffffffu;             // sentinel, >= n
  uint32_t cur[4], nxt[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) cur[u] = nxt[u] = kPast;
  if (lane < da) cur[0] = (uint32_t)__ldg(na - lane);
  int32_t cu = 1;  // loads per lane in the current step
  int32_t c = 0;
  scanned = 0;
  for (;;) {
    const int32_t wstep = min(32 * cu, da - scanned);
    const int32_t nbase = scanned + wstep;
    const bool pre =
        (cmin - c > wstep) && (need_miss - (scanned - c) > wstep) && (nbase < da);
    if (pre) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t idx = nbase + u * 32 + lane;
        nxt[u] = idx < da ? (uint32_t)__ldg(na - idx) : kPast;
      }
    }
    const uint32_t lo4 = min(min(cur[0], cur[1]), min(cur[2], cur[3]));
    uint32_t hits = 0;
    if (__all_sync(0xffffffffu, lo4 >= hub_lo)) {  // bitmap only, branch-free
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t r = min(cur[u] - hub_lo, rmax);
        hits += (bm[r >> 5] >> (r & 31)) & 1u;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (cur[u] != kPast) hits += member<GTAB>(bm, hub_lo, C, cur[u], nstash, nb, nlo);
    }
    c += (int32_t)__reduce_add_sync(0xffffffffu, hits);
    scanned = nbase;
    if (c >= cmin) return true;
    if (c + (da - scanned) < cmin) return false;
    if (pre) {
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t idx = scanned + u * 32 + lane;
        cur[u] = idx < da ? (uint32_t)__ldg(na - idx) : kPast;
      }
    }
    cu = 4;
  }
}

template <int NT, bool GTAB>
__global__ void __launch_bounds__(NT, 2048 / NT > 2 ? 2048 / NT / 2 : 1) k_sim_hash(SimParams P, int64_t rlo, int64_t rhi,
                                                 uint32_t tcap, int qi, int chunk,
                                                 uint32_t hub_lo, uint32_t bm_words) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* bm = smem;  // [bm_words] + zero guard words (kept 16-byte aligned)
  uint32_t* tab_s = smem + bm_words + 4;
  // survivors of the O(1) filter: where N(a) starts, (a, deg a), (j, c_min)
  int64_t* surv_oa = reinterpret_cast<int64_t*>(tab_s + (GTAB ? 0 : 4 * (size_t)tcap));
  int2* surv_ad = reinterpret_cast<int2*>(surv_oa + chunk);
  int2* surv_jc = surv_ad + chunk;
  __shared__ int s_item, s_nsurv, s_next, s_nstash;
  __shared__ unsigned int s_bsim, s_bdis;
  __shared__ int64_t s_nlo;
  __shared__ uint32_t s_stash[kStash];
  const int tid = threadIdx.x, lane = tid & 31;
  LocalCtr lc;
  Cuckoo C;
  C.tab = GTAB ? (P.gtab + (int64_t)blockIdx.x * P.gtab_stride) : tab_s;
  C.nstash = &s_nstash;
  C.stash = s_stash;
  for (uint32_t i = tid; i < bm_words + 4; i += NT) bm[i] = 0u;

  for (;;) {
    if (tid == 0) s_item = atomicAdd(&P.wq[qi], 1);
    __syncthreads();
    const int64_t b = rhi - 1 - (int64_t)s_item;
    if (b < rlo) break;
    const int64_t ob = P.off[b], db = P.off[b + 1] - ob;
    const int64_t e0 = P.eoff[b], nlow = P.eoff[b + 1] - e0;
    const int32_t* __restrict__ nb = P.adj + ob;
    const int2 th = P.thr[db];
    const int64_t xmin = th.x, simmax = th.y;
    bool built = false;
    for (int64_t base = 0; base < nlow; base += chunk) {
      if (tid == 0) { s_nsurv = 0; s_next = 0; s_bsim = 0; s_bdis = 0; }
      __syncthreads();
      const int64_t lim = base + chunk < nlow ? base + chunk : nlow;
      // filter + O(1) bounds, one candidate a per thread
      for (int64_t j = base + tid; j < lim; j += NT) {
        const int64_t e = e0 + j;
        const int32_t a = nb[j];
        if (!edge_needed(P, e, a, (int32_t)b)) continue;
        const int64_t oa = P.off[a];
        const int64_t da = P.off[a + 1] - oa;
        if (da + 1 < xmin) {
          lc.bound++;
          record_edge(P, e, a, (int32_t)b, false, false, lc);
          atomicAdd(&s_bdis, 1u);
        } else if (da <= simmax) {
          lc.bound++;
          record_edge(P, e, a, (int32_t)b, true, false, lc);
          atomicAdd(&s_bsim, 1u);
        } else {
          const int slot = atomicAdd(&s_nsurv, 1);
          surv_oa[slot] = oa;
          surv_ad[slot] = make_int2(a, (int32_t)da);
          surv_jc[slot] = make_int2((int32_t)j, (int32_t)c_min_exact(da, db, da - 1, P.eps));
        }
      }
      __syncthreads();
      const int ns = s_nsurv;
      if (ns > 0) {
        if (!built) {  // stage N(b) once per b: hub suffix -> bitmap, rest -> cuckoo
          if (tid == 0) {
            s_nlo = P.nlo[b];
            s_nstash = 0;
          }
          __syncthreads();
          const int64_t nlo = s_nlo;
          uint32_t T = (uint32_t)((nlo * 5) / 12 + 1);  // <= 0.6 keys per slot
          if (T > tcap) T = tcap;
          C.T = T;
          for (uint32_t i = tid; i < T; i += NT)
              reinterpret_cast<uint4*>(C.tab)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
          __syncthreads();
          for (int64_t i = tid; i < db; i += NT) {
            const uint32_t w = (uint32_t)nb[i];
            if (i >= nlo) {
              const uint32_t r = w - hub_lo;
              atomicOr(&bm[r >> 5], 1u << (r & 31));
            } else {
              cuckoo_insert(C, w);
            }
          }
          __syncthreads();
          built = true;
          if (tid == 0) lc.bytes += 4ull * (unsigned long long)db;  // N(b) read once
        }
        const int nstash = s_nstash;
        const int64_t nlo = s_nlo;
        const uint32_t rmax = bm_words * 32u;  // first bit of the zero guard word
        // one warp per surviving a, dynamic (scan_survivor)
        for (;;) {
          int s = 0;
          if (lane == 0) s = atomicAdd(&s_next, 1);
          s = __shfl_sync(0xffffffffu, s, 0);
          if (s >= ns) break;
          const int2 jc = surv_jc[s];
          const int2 ad = surv_ad[s];
          int32_t scanned;
          const bool res = scan_survivor<GTAB>(P.adj + surv_oa[s], ad.y, jc.y, bm, hub_lo, rmax,
                                               C, nstash, nb, nlo, lane, scanned);
          if (lane == 0) {
            lc.probes += (unsigned long long)scanned;
            lc.inters++;
            lc.bytes += 4ull * (unsigned long long)ad.y;
            record_edge(P, e0 + jc.x, ad.x, (int32_t)b, res, false, lc);
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
    if (built) {  // clear the bitmap words this b set (O(deg b), not O(R))
      for (int64_t i = s_nlo + tid; i < db; i += NT) bm[((uint32_t)nb[i] - hub_lo) >> 5] = 0u;
    }
    __syncthreads();  // bitmap clean and s_item read by all before the next b
  }
  flush_ctr(P, lc);
}

// ---------------------------------------------------------------------------
// small b (64 <= deg < 512): one warp per b, no CTA barriers.  Each warp owns
// a private cuckoo table of N(b) in shared memory; the 32 lanes filter 32
// candidates at a time (O(1) bounds), and the surviving edges are decided one
// by one by the whole warp with scan_survivor (data broadcast by shuffles).
static constexpr int kWarpBuckets = 256;  // 4 KB: deg < 512 -> <= 0.5 keys per slot
static constexpr int kWarpWords = 4 * kWarpBuckets + kStash + 4;

template <int NT>
__global__ void __launch_bounds__(NT, 2048 / NT / 2) k_sim_warp(SimParams P, int64_t rlo,
                                                               int64_t rhi, int qi) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* tab = smem + (size_t)wid * kWarpWords;
  Cuckoo C;
  C.tab = tab;
  C.stash = tab + 4 * kWarpBuckets;
  C.nstash = reinterpret_cast<int*>(C.stash + kStash);
  LocalCtr lc;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(&P.wq[qi], 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    const int64_t b = rhi - 1 - (int64_t)item;
    if (b < rlo) break;
    const int64_t ob = P.off[b], db = P.off[b + 1] - ob;
    const int64_t e0 = P.eoff[b], nlow = P.eoff[b + 1] - e0;
    const int32_t* __restrict__ nb = P.adj + ob;
    const int2 th = P.thr[db];
    bool built = false;
    uint32_t bsim = 0, bdis = 0;
    for (int64_t base = 0; base < nlow; base += 32) {
      const int64_t j = base + lane;
      int st = 0;  // 0 none, 1 dissimilar by bound, 2 similar by bound, 3 survivor
      int32_t a = 0, da = 0, cmin = 0;
      int64_t oa = 0;
      if (j < nlow) {
        a = nb[j];
        if (edge_needed(P, e0 + j, a, (int32_t)b)) {
          oa = P.off[a];
          da = (int32_t)(P.off[a + 1] - oa);
          if (da + 1 < th.x) st = 1;
          else if (da <= th.y) st = 2;
          else {
            st = 3;
            cmin = (int32_t)c_min_exact(da, db, da - 1, P.eps);
          }
          if (st == 1 || st == 2) {
            lc.bound++;
            record_edge(P, e0 + j, a, (int32_t)b, st == 2, false, lc);
          }
        }
      }
      bdis += __popc(__ballot_sync(0xffffffffu, st == 1));
      bsim += __popc(__ballot_sync(0xffffffffu, st == 2));
      uint32_t smask = __ballot_sync(0xffffffffu, st == 3);
      if (smask && !built) {  // stage N(b) once per b, warp-private
        uint32_t T = (uint32_t)((db * 5) / 12 + 1);
        if (T > kWarpBuckets) T = kWarpBuckets;
        C.T = T;
        for (uint32_t i = lane; i < T; i += 32)
          reinterpret_cast<uint4*>(tab)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        if (lane == 0) *C.nstash = 0;
        __syncwarp();
        for (int64_t i = lane; i < db; i += 32) cuckoo_insert(C, (uint32_t)nb[i]);
        __syncwarp();
        built = true;
        if (lane == 0) lc.bytes += 4ull * (unsigned long long)db;
      }
      const int nstash = built ? *C.nstash : 0;
      while (smask) {
        const int src = __ffs(smask) - 1;
        smask &= smask - 1;
        const int32_t sa = __shfl_sync(0xffffffffu, a, src);
        const int32_t sda = __shfl_sync(0xffffffffu, da, src);
        const int32_t scm = __shfl_sync(0xffffffffu, cmin, src);
        const int64_t soa = __shfl_sync(0xffffffffu, oa, src);
        int32_t scanned;
        const bool res = scan_survivor<false>(P.adj + soa, sda, scm, nullptr, 0xffffffffu, 0, C,
                                              nstash, nb, db, lane, scanned);
        if (res) ++bsim; else ++bdis;
        if (lane == 0) {
          lc.probes += (unsigned long long)scanned;
          lc.inters++;
          lc.bytes += 4ull * (unsigned long long)sda;
          record_edge(P, e0 + base + src, sa, (int32_t)b, res, false, lc);
        }
      }
    }
    if (lane == 0 && (bsim | bdis) && (P.mode == MODE_IDENTIFY || P.mode == MODE_CLEANUP))
      apply_bounds(P.bounds, P.role, b, bsim, bdis, P.mu);
    __syncwarp();
  }
  flush_ctr(P, lc);
}

// ---------------------------------------------------------------------------
// host driver

template <int NT, bool GTAB>
static int launch_hash(gs_engine* e, const SimParams& P, int64_t rlo, int64_t rhi,
                       uint32_t tcap, int qi, int chunk) {
  if (rhi <= rlo) return GS_OK;
  const size_t smem =
      (size_t)(P.bm_words + 4) * 4 + (GTAB ? 0 : (size_t)tcap * 16) + (size_t)chunk * 24;
  auto kern = k_sim_hash<NT, GTAB>;
  GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  GS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)occ * e->sms;
  if (grid > rhi - rlo) grid = rhi - rlo;
  if (GTAB && grid > e->sms * 2) grid = e->sms * 2;
  kern<<<(unsigned)grid, NT, smem, e->stream>>>(P, rlo, rhi, tcap, qi, chunk, P.hub_lo,
                                                P.bm_words);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

static int launch_warp(gs_engine* e, const SimParams& P, int64_t rlo, int64_t rhi, int qi) {
  if (rhi <= rlo) return GS_OK;
  constexpr int NT = 256;
  const size_t smem = (size_t)(NT / 32) * kWarpWords * 4;
  auto kern = k_sim_warp<NT>;
  GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  GS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)occ * e->sms;
  const int64_t nw = (rhi - rlo + NT / 32 - 1) / (NT / 32);
  if (grid > nw) grid = nw;
  kern<<<(unsigned)grid, NT, smem, e->stream>>>(P, rlo, rhi, qi);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// hub bitmap range: the top 2^18 ranks (32 KB of shared memory per CTA)
static constexpr int64_t kHubBits = 1 << 18;

int prepare_similarity(gs_engine* e, const Eps2& eps) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  GS_TRY(e->alloc_n(&s.thr, g.dmax + 1));
  GS_TRY(e->alloc_n(&s.nlo, g.n));
  k_thresholds<<<grid_for(g.dmax + 1, 256), 256, 0, e->stream>>>(g.dmax, eps, s.thr);
  const int64_t bits = std::min<int64_t>(kHubBits, ((g.n + 31) / 32) * 32);
  const uint32_t hub_lo = (uint32_t)std::max<int64_t>(0, g.n - bits);
  if (g.n > 0) {
    k_hubsplit<<<grid_for(g.n, 256), 256, 0, e->stream>>>(g.off, g.adj, g.n, hub_lo, s.nlo);
    e->launches += 2;
  }
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
  P.thr = s.thr;
  P.nlo = s.nlo;
  {
    const int64_t bits = std::min<int64_t>(kHubBits, ((g.n + 31) / 32) * 32);
    P.hub_lo = (uint32_t)std::max<int64_t>(0, g.n - bits);
    P.bm_words = (uint32_t)((g.n - P.hub_lo + 31) / 32);
  }
  GS_CUDA(cudaMemsetAsync(s.wq, 0, 8 * sizeof(int32_t), e->stream));
  const int64_t* rc = g.rclass;
  // huge b first (longest work items), with an L2-resident table per CTA
  const int64_t rhuge = rc[4];
  if (g.n > rhuge) {
    const int64_t tcap_g = (g.dmax * 5) / 12 + 1;  // buckets
    const int64_t nblk = (int64_t)e->sms * 2;
    GS_TRY(e->alloc_n(&P.gtab, 4 * tcap_g * nblk));
    P.gtab_stride = 4 * tcap_g;
    GS_TRY((launch_hash<1024, true>(e, P, rhuge, g.n, (uint32_t)tcap_g, 4, 1024)));
  }
  // shared memory per CTA: hub bitmap (top 2^18 ranks: 32 KB) + cuckoo table
  // for the non-hub part of N(b) (16-byte buckets) + survivor lists (24 B
  // per candidate of a chunk); the small class runs warp-per-b
  GS_TRY((launch_hash<1024, false>(e, P, rc[3], rc[4], 8192, 3, 1024)));
  GS_TRY((launch_hash<512, false>(e, P, rc[2], rc[3], 2048, 2, 1024)));
  GS_TRY(launch_warp(e, P, rc[1], rc[2], 1));
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
