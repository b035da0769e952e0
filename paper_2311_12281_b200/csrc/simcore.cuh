// simcore.cuh -- device building blocks of the similarity sweep shared by
// the in-HBM kernels (sim.cu) and the out-of-core kernels (ooc.cu): roles and
// Lemma-1 bounds, lock-free union-find, the two-choice cuckoo table, the
// per-degree O(1) thresholds and the early-exit survivor scan.
#pragma once
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

// Can any edge owned by b need a decision in this mode?  Union needs b core;
// attach needs b core or b adjacent to a core (coreadj, set before attach).
__device__ __forceinline__ bool b_needed(const SimParams& P, int64_t b) {
  if (P.mode == MODE_UNION) return ld_role(P.role, b) == ROLE_CORE;
  if (P.mode == MODE_ATTACH) return ld_role(P.role, b) == ROLE_CORE || P.coreadj[b];
  return true;
}

// Does edge (a, b) need a decision in this mode?
__device__ __forceinline__ bool edge_needed(const SimParams& P, int64_t e, int32_t a,
                                            int32_t b) {
  // identify visits every oriented edge once (by its high endpoint), so its
  // status is still unknown there: no load
  if (P.mode != MODE_IDENTIFY && P.sim[e] != SIM_UNKNOWN) return false;
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

// Work counters of the similarity kernels.  LocalCtr lives in registers
// (thread-level kernels); SharedCtr is one CTA-wide array in shared memory,
// updated with shared atomics -- the persistent CTA / warp kernels sit at their
// register limit, and eight 64-bit register counters per thread cost spills.
enum LCtrIdx { LC_EVALS, LC_PROBES, LC_BOUND, LC_INTERS, LC_BYTES, LC_RETRIES, LC_SKETCH, LC_WSIM,
               LC_N };

struct LocalCtr {
  unsigned long long evals = 0, probes = 0, bound = 0, inters = 0, bytes = 0, retries = 0,
                     sketch = 0, wsim = 0;
};

// Counters of the persistent CTA / warp kernels: a few registers per thread
// (bytes 64-bit, the rest 32-bit), folded into a CTA-wide shared array once per
// high endpoint b (warp reduction + one shared atomic per warp and counter):
// per-event shared atomics on one address serialise the whole CTA, and eight
// 64-bit register counters per thread cost spills at the 64-register limit.
// evals = sketch-decided + intersected here (the O(1)-decided edges these
// kernels re-meet in union / attach are not counted, see record_edge).
struct HotCtr {
  unsigned long long bytes = 0;
  uint32_t sketch = 0, inters = 0, probes = 0, wsim_d = 0;  // wsim in units of 4 bytes
};

__device__ __forceinline__ void ctr_add(LocalCtr& c, int i, unsigned long long x) {
  switch (i) {
    case LC_EVALS: c.evals += x; break;
    case LC_PROBES: c.probes += x; break;
    case LC_BOUND: c.bound += x; break;
    case LC_INTERS: c.inters += x; break;
    case LC_BYTES: c.bytes += x; break;
    case LC_RETRIES: c.retries += x; break;
    case LC_SKETCH: c.sketch += x; break;
    default: c.wsim += x; break;
  }
}

__device__ __forceinline__ void ctr_add(HotCtr& c, int i, unsigned long long x) {
  switch (i) {
    case LC_BYTES: c.bytes += x; break;
    case LC_SKETCH: c.sketch += (uint32_t)x; break;
    case LC_INTERS: c.inters += (uint32_t)x; break;
    case LC_PROBES: c.probes += (uint32_t)x; break;
    case LC_WSIM: c.wsim_d += (uint32_t)(x >> 2); break;
    default: break;  // LC_EVALS (derived), LC_BOUND (out of core only), LC_RETRIES (record_edge)
  }
}

// fold a warp's HotCtr into the CTA's shared array (all 32 lanes call it)
__device__ __forceinline__ void hot_flush_warp(HotCtr& c, unsigned long long* v) {
  const unsigned sk = __reduce_add_sync(0xffffffffu, c.sketch);
  const unsigned in = __reduce_add_sync(0xffffffffu, c.inters);
  const unsigned pr = __reduce_add_sync(0xffffffffu, c.probes);
  unsigned long long ws = c.wsim_d, by = c.bytes;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ws += __shfl_xor_sync(0xffffffffu, ws, o);
    by += __shfl_xor_sync(0xffffffffu, by, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (sk | in) atomicAdd(v + LC_EVALS, (unsigned long long)sk + in);
    if (sk) atomicAdd(v + LC_SKETCH, (unsigned long long)sk);
    if (in) atomicAdd(v + LC_INTERS, (unsigned long long)in);
    if (pr) atomicAdd(v + LC_PROBES, (unsigned long long)pr);
    if (ws) atomicAdd(v + LC_WSIM, 4ull * ws);
    if (by) atomicAdd(v + LC_BYTES, by);
  }
  c.bytes = 0;
  c.sketch = c.inters = c.probes = c.wsim_d = 0;
}

// global counter of each LC_* index (bytes go to the launch's class slot)
__device__ __forceinline__ int ctr_slot(const SimParams& P, int i) {
  switch (i) {
    case LC_EVALS: return CTR_SIM_EVALS;
    case LC_PROBES: return CTR_PROBES;
    case LC_BOUND: return CTR_BOUND_DECIDED;
    case LC_INTERS: return CTR_INTERSECTIONS;
    case LC_BYTES: return P.bslot;
    case LC_RETRIES: return CTR_UNION_RETRIES;
    case LC_SKETCH: return CTR_SKETCH_DECIDED;
    default: return CTR_WSIM;
  }
}

// zero / flush a SharedCtr: every thread of the CTA calls both (barriers inside)
__device__ __forceinline__ void shared_ctr_init(unsigned long long* v) {
  if (threadIdx.x < LC_N) v[threadIdx.x] = 0ull;
  __syncthreads();
}
__device__ __forceinline__ void shared_ctr_flush(const SimParams& P, const unsigned long long* v) {
  __syncthreads();
  if (threadIdx.x < LC_N && v[threadIdx.x]) atomicAdd(&P.ctr[ctr_slot(P, threadIdx.x)], v[threadIdx.x]);
}

// Algorithmic bytes (CTR_B_*, DESIGN 5) charged per unit of work:
static constexpr unsigned kBytesB = 40;     // per b: off[b..b+1], eoff[b..b+1], thr[deg b]
static constexpr unsigned kBytesCand = 22;  // per filtered candidate a: nb[j], off[a..a+1], 2 roles
static constexpr unsigned kBytesRec = 17;   // per decided edge: sim[e] + a's bounds (atomic RMW)

// Record one decided edge.  b's bound update is returned to the caller
// (aggregated per CTA for the shared-b kernels) unless apply_b is set.
// `count` is false for O(1)-decided edges re-met by the union / attach passes:
// the identify pre-pass already counted their decision (sim_evals).
template <class Ctr>
__device__ __forceinline__ void record_edge(const SimParams& P, int64_t e, int32_t a,
                                            int32_t b, bool similar, bool apply_b,
                                            Ctr& lc, bool count = true) {
  P.sim[e] = similar ? SIM_SIMILAR : SIM_DISSIMILAR;
  ctr_add(lc, LC_EVALS, count ? 1ull : 0ull);
  if (P.mode == MODE_IDENTIFY || P.mode == MODE_CLEANUP) {
    apply_bounds(P.bounds, P.role, a, similar ? 1u : 0u, similar ? 0u : 1u, P.mu);
    if (apply_b) apply_bounds(P.bounds, P.role, b, similar ? 1u : 0u, similar ? 0u : 1u, P.mu);
  } else if (P.mode == MODE_UNION && similar) {
    unsigned long long r = 0;
    uf_union(P.parent, a, b, r);
    if (r) atomicAdd(&P.ctr[CTR_UNION_RETRIES], r);  // failed CAS hooks: rare
  }
}

__device__ __forceinline__ void flush_ctr(const SimParams& P, LocalCtr& lc) {
  // warp reduce then one atomic per warp
  unsigned long long v[8] = {lc.evals, lc.probes, lc.bound, lc.inters, lc.bytes, lc.retries,
                             lc.sketch, lc.wsim};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (v[0]) atomicAdd(&P.ctr[CTR_SIM_EVALS], v[0]);
    if (v[1]) atomicAdd(&P.ctr[CTR_PROBES], v[1]);
    if (v[2]) atomicAdd(&P.ctr[CTR_BOUND_DECIDED], v[2]);
    if (v[3]) atomicAdd(&P.ctr[CTR_INTERSECTIONS], v[3]);
    if (v[4]) atomicAdd(&P.ctr[P.bslot], v[4]);
    if (v[5]) atomicAdd(&P.ctr[CTR_UNION_RETRIES], v[5]);
    if (v[6]) atomicAdd(&P.ctr[CTR_SKETCH_DECIDED], v[6]);
    if (v[7]) atomicAdd(&P.ctr[CTR_WSIM], v[7]);
  }
}

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
static constexpr uint32_t kPast = 0x7fffffffu;  // scan sentinel, >= n

// an element of N(a) for the scan: read once per edge, so not allocated in L1
#ifndef GS_SCAN_NA
#define GS_SCAN_NA 1
#endif
__device__ __forceinline__ uint32_t ld_scan(const int32_t* p) {
#if GS_SCAN_NA
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
#else
  return (uint32_t)__ldg(p);
#endif
}

// The first step's element of this lane (the top 32 of N(a)); issued early so
// the load of survivor s+1 overlaps the scan of survivor s.
__device__ __forceinline__ uint32_t first_element(const int32_t* __restrict__ a_run, int32_t da,
                                                  int lane) {
  return lane < da ? ld_scan(a_run + (da - 1 - lane)) : kPast;
}

template <bool GTAB>
__device__ __forceinline__ bool scan_survivor(const int32_t* __restrict__ a_run, int32_t da,
                                              int32_t cmin, const uint32_t* bm, uint32_t hub_lo,
                                              uint32_t rmax, const Cuckoo& C, int nstash,
                                              const int32_t* __restrict__ nb, int64_t nlo,
                                              int lane, int32_t& scanned, uint32_t first) {
  // Element j (0 = the top of N(a)) is a_run[da - 1 - j]; in a step based at
  // element s, lane l reads j = s + 32u + l for u < cu: one base pointer per
  // step, the four loads use immediate offsets.
  const int32_t* __restrict__ top = a_run + (da - 1 - lane);
  const int32_t need_miss = da - cmin + 1;  // misses that decide "dissimilar"
  // Any decision reads at least min(need_miss - misses, cmin - hits) more
  // elements, so a step of that many (rounded up to 32, at most 128) never
  // over-reads except in its last 31 slots; the next step is prefetched only
  // when this one cannot decide the edge.
  uint32_t cur[4], nxt[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) cur[u] = nxt[u] = kPast;
  cur[0] = first;
  int32_t cu = min(4, max(1, (min(need_miss, cmin) + 31) >> 5));
  {
    const int32_t rem = da - lane;
#pragma unroll
    for (int u = 1; u < 4; ++u)
      if (u < cu && 32 * u < rem) cur[u] = ld_scan(top - 32 * u);
  }
  int32_t c = 0;
  scanned = 0;
  for (;;) {
    const int32_t wstep = min(32 * cu, da - scanned);
    const int32_t nbase = scanned + wstep;
    const int32_t rest = min(need_miss - (scanned - c), cmin - c) - wstep;  // still certain
    const bool pre = rest > 0 && nbase < da;
    int32_t nu = 0;
    if (pre) {
      nu = min(4, (rest + 31) >> 5);
      const int32_t* __restrict__ q = top - nbase;
      const int32_t rem = da - nbase - lane;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        nxt[u] = (u < nu && 32 * u < rem) ? ld_scan(q - 32 * u) : kPast;
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
      cu = nu;
    } else {
      cu = min(4, max(1, (min(need_miss - (scanned - c), cmin - c) + 31) >> 5));
      const int32_t* __restrict__ q = top - scanned;
      const int32_t rem = da - scanned - lane;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        cur[u] = (u < cu && 32 * u < rem) ? ld_scan(q - 32 * u) : kPast;
    }
  }
}

// 32-bit mixer of the neighbourhood sketches (sketch.cu)
__device__ __forceinline__ uint32_t sk_hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  return x;
}

// Sketch bound (sketch.cu): U = |S_a & fold(S_b)| + d_a - |S_a| < c_min
// proves (a, b) dissimilar.  sk_try decides (warp-uniformly) whether to
// attempt it: the scan must have work to save (more than sk_minscan misses
// needed to reject) and the expected false hits, d_a (1 - e^(-d_b/M_a)) +
// d_a^2 / (2 M_a), must leave room below c_min -- otherwise U cannot decide
// and the read is wasted.
__device__ __forceinline__ bool sk_try(const SimParams& P, int64_t da, int64_t db, int32_t cmin) {
  if (P.sk == nullptr || da < P.sk_dmin || da - cmin + 1 < P.sk_minscan) return false;
  const float ma = 32.f * (float)sk_words(da, P.sk_lk), fa = (float)da;
  const float ef = fa * (1.f - __expf(-(float)db / ma)) + fa * fa / (2.f * ma);
  return ef < P.sk_gate * (float)cmin;
}

// v's sketch slot (2w words: S_v, then its levels; sketch.cu)
__device__ __forceinline__ const uint32_t* sk_row(const SimParams& P, int64_t v, int64_t d,
                                                  int64_t w) {
  return P.sk + P.skbase[d] + (v - P.rdeg[d]) * 2 * w;
}

// the levels of a row of w words held in `t` (2w words of room): level L
// (w >> L words) at 2 (w - (w >> L)); threads [i0, i0 + nt) of a warp
__device__ __forceinline__ void sk_fold_levels(uint32_t* t, int64_t w, int i0, int nt) {
  for (int64_t lo = 0, x = w; x > 4; lo += x, x >>= 1) {
    const int64_t h = x >> 1;
    for (int64_t i = i0; i < h; i += nt) t[lo + x + i] = t[lo + i] | t[lo + h + i];
    __syncwarp();
  }
}

// ... by a CTA (sync = __syncthreads)
template <class Sync>
__device__ __forceinline__ void sk_fold_levels(uint32_t* t, int64_t w, int i0, int nt, Sync sync) {
  for (int64_t lo = 0, x = w; x > 4; lo += x, x >>= 1) {
    const int64_t h = x >> 1;
    for (int64_t i = i0; i < h; i += nt) t[lo + x + i] = t[lo + i] | t[lo + h + i];
    sync();
  }
}

// B is S_b already folded to a's wa words (a shared-memory level, sim.cu)
__device__ __forceinline__ bool sk_rejects_lev(const uint32_t* __restrict__ A,
                                               const uint32_t* B, int64_t wa, int64_t da,
                                               int32_t cmin, int lane) {
  int acc = 0;
  for (int64_t j = lane; j < wa; j += 32) {
    const uint32_t x = __ldg(A + j);
    acc += __popc(x & B[j]) - __popc(x);
  }
  acc = __reduce_add_sync(0xffffffffu, acc);
  return da + acc < cmin;
}

// B is S_b in global memory (wb >= wa words), folded on the fly
__device__ __forceinline__ bool sk_rejects_fold(const uint32_t* __restrict__ A,
                                                const uint32_t* __restrict__ B, int64_t wa,
                                                int64_t wb, int64_t da, int32_t cmin, int lane) {
  int acc = 0;
  for (int64_t j = lane; j < wa; j += 32) {
    const uint32_t x = __ldg(A + j);
    uint32_t y = 0;
    for (int64_t t = j; t < wb; t += wa) y |= __ldg(B + t);
    acc += __popc(x & y) - __popc(x);
  }
  acc = __reduce_add_sync(0xffffffffu, acc);
  return da + acc < cmin;
}

// Wide variant of sk_rejects_fold for long rows (huge b): 16-byte loads
// (rows are 16-byte aligned, wa and wb multiples of 4 words).
__device__ __forceinline__ bool sk_rejects_fold4(const uint32_t* __restrict__ A,
                                                 const uint32_t* __restrict__ B, int64_t wa,
                                                 int64_t wb, int64_t da, int32_t cmin, int lane) {
  int acc = 0;
  for (int64_t j = 4 * lane; j < wa; j += 128) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(A + j));
    uint4 y = __ldg(reinterpret_cast<const uint4*>(B + j));
    for (int64_t t = j + wa; t < wb; t += wa) {
      const uint4 z = __ldg(reinterpret_cast<const uint4*>(B + t));
      y.x |= z.x; y.y |= z.y; y.z |= z.z; y.w |= z.w;
    }
    acc += __popc(x.x & y.x) + __popc(x.y & y.y) + __popc(x.z & y.z) + __popc(x.w & y.w) -
           __popc(x.x) - __popc(x.y) - __popc(x.z) - __popc(x.w);
  }
  acc = __reduce_add_sync(0xffffffffu, acc);
  return da + acc < cmin;
}

// Warp form over a shared-memory level with 16-byte loads (lane l: words
// 4l..4l+3 of each 128-word block) -- for rows read over PCIe (out-of-core),
// where the request size matters more than the latency.
__device__ __forceinline__ bool sk_rejects_lev4(const uint32_t* __restrict__ A,
                                                const uint32_t* B, int64_t wa, int64_t da,
                                                int32_t cmin, int lane,
                                                unsigned long long& abytes) {
  // U = d_a - sum popc(x & ~y) only decreases: stop after the first 512-byte
  // block that takes it below c_min (bytes over PCIe are the cost here);
  // abytes += the bytes of A requested
  int64_t u = da;
  for (int64_t j0 = 0; j0 < wa; j0 += 128) {
    abytes += 4ull * (unsigned long long)min((int64_t)128, wa - j0);
    const int64_t j = j0 + 4 * lane;
    int acc = 0;
    if (j < wa) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(A + j));
      const uint4 y = *reinterpret_cast<const uint4*>(B + j);
      acc = __popc(x.x & ~y.x) + __popc(x.y & ~y.y) + __popc(x.z & ~y.z) + __popc(x.w & ~y.w);
    }
    u -= __reduce_add_sync(0xffffffffu, acc);
    if (u < cmin) return true;
  }
  return false;
}

// Thread-per-survivor form of the sketch bound: one thread walks S_a in
// 16-byte steps against b's level (B: wa words, shared or global) or S_b
// folded on the fly (wb > wa), stopping as soon as U = d_a - sum popc(x & ~y)
// drops below c_min (U only decreases).  Used where many survivors are
// checked at once, so hundreds of rows are in flight per SM instead of one
// per warp.
// U = 16-byte steps in flight per early-exit check
// `gwords` += the global words read (S_a, plus S_b's slices when bglobal).
template <int SK_UNROLL = 2>
__device__ __forceinline__ bool sk_thread_rejects(const uint32_t* __restrict__ A,
                                                  const uint32_t* B, int64_t wa, int64_t wb,
                                                  int64_t da, int32_t cmin, bool bglobal,
                                                  unsigned long long& gwords) {
  const uint4* __restrict__ a4 = reinterpret_cast<const uint4*>(A);
  const uint4* b4 = reinterpret_cast<const uint4*>(B);
  const int64_t q = wa >> 2, qb = wb >> 2;
  int64_t u = da;
  for (int64_t j = 0; j < q; j += SK_UNROLL) {
    gwords += 4ull * (unsigned long long)min((int64_t)SK_UNROLL, q - j) *
              (unsigned long long)(1 + (bglobal ? qb / q : 0));
    uint4 x[SK_UNROLL], y[SK_UNROLL];
#pragma unroll
    for (int t = 0; t < SK_UNROLL; ++t) {
      x[t] = j + t < q ? __ldg(a4 + j + t) : make_uint4(0u, 0u, 0u, 0u);
      y[t] = j + t < q ? b4[j + t] : make_uint4(0u, 0u, 0u, 0u);
      for (int64_t f = j + t + q; f < qb; f += q) {  // fold (global S_b only)
        const uint4 z = __ldg(b4 + f);
        y[t].x |= z.x; y[t].y |= z.y; y[t].z |= z.z; y[t].w |= z.w;
      }
    }
#pragma unroll
    for (int t = 0; t < SK_UNROLL; ++t)
      u -= __popc(x[t].x & ~y[t].x) + __popc(x[t].y & ~y[t].y) + __popc(x[t].z & ~y[t].z) +
           __popc(x[t].w & ~y[t].w);
    if (u < cmin) return true;
  }
  return false;
}

// 256-bit global load (sm_100: LDG.E.256): one whole 32-byte sector per thread
__device__ __forceinline__ void ldg256(const uint32_t* p, uint32_t (&r)[8]) {
  asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "l"(p));
}

// ... without allocating in L1 (a row of S_a is read once per edge; 7% L1 hits)
__device__ __forceinline__ void ldg256_na(const uint32_t* p, uint32_t (&r)[8]) {
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "l"(p));
}

// Thread-per-edge sketch bound with 32-byte loads: the row walk of
// sk_thread_rejects, but every load fetches one whole sector, so an L1
// wavefront carries 32 useful bytes instead of 16 (a warp's lanes walk 32
// different rows: with 16-byte loads the L1 was the limiter, 86% busy).  A (S_a)
// and B (b's level at a's resolution) are global, 32-byte aligned (sketch
// slots are multiples of 8 words; wa >= 4).  `words` += the words of A read.
template <int UNROLL, bool NA = false, bool NAB = false>
__device__ __forceinline__ bool sk_rejects256(const uint32_t* __restrict__ A,
                                              const uint32_t* __restrict__ B, int64_t wa,
                                              int64_t da, int32_t cmin,
                                              unsigned long long& words) {
  int64_t u = da;
  if (wa < 8) {  // a 4-word row: one 16-byte step
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(A));
    const uint4 y = __ldg(reinterpret_cast<const uint4*>(B));
    words += 4;
    u -= __popc(x.x & ~y.x) + __popc(x.y & ~y.y) + __popc(x.z & ~y.z) + __popc(x.w & ~y.w);
    return u < cmin;
  }
  const int64_t q = wa >> 3;
  for (int64_t j = 0; j < q; j += UNROLL) {
    uint32_t x[UNROLL][8], y[UNROLL][8];
#pragma unroll
    for (int t = 0; t < UNROLL; ++t) {
      if (j + t < q) {
        if (NA) ldg256_na(A + 8 * (j + t), x[t]); else ldg256(A + 8 * (j + t), x[t]);
        if (NAB) ldg256_na(B + 8 * (j + t), y[t]); else ldg256(B + 8 * (j + t), y[t]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[t][k] = y[t][k] = 0u;
      }
    }
    words += 8ull * (unsigned long long)min((int64_t)UNROLL, q - j);
#pragma unroll
    for (int t = 0; t < UNROLL; ++t)
#pragma unroll
      for (int k = 0; k < 8; ++k) u -= __popc(x[t][k] & ~y[t][k]);
    if (u < cmin) return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk) 1-D copies into shared memory, completion on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// generic-proxy accesses of shared memory ordered before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// one elected thread: arm `bar` for `bytes` and copy them global -> shared
// (dst, src 16-byte aligned, bytes a multiple of 16)
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// Stage S_b (wb words) and its folds into `lev`: level L (wb >> L words)
// starts at word 2 (wb - (wb >> L)), so a's level (wa words) is at
// lev + 2 (wb - wa).  Threads [t0, t0 + nt) cooperate; sync() orders the
// levels (__syncthreads for a CTA, __syncwarp for a warp).
template <class Sync>
__device__ __forceinline__ void sk_stage_levels(const uint32_t* __restrict__ Bg, int64_t wb,
                                                uint32_t* lev, int t, int nt, Sync sync) {
  for (int64_t i = t; i < wb; i += nt) lev[i] = __ldg(Bg + i);
  sync();
  for (int64_t lo = 0, w = wb; w > 4; lo += w, w >>= 1) {
    const int64_t h = w >> 1;
    for (int64_t i = t; i < h; i += nt) lev[lo + w + i] = lev[lo + i] | lev[lo + h + i];
    sync();
  }
}

// host launcher of the per-degree threshold table (sim.cu)
int launch_thresholds(int64_t dmax, const Eps2& eps, int2* thr, cudaStream_t st);

}  // namespace gs
