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
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "simcore.cuh"

namespace gs {

__device__ __forceinline__ int64_t lower_bound_run(const int32_t* __restrict__ a, int64_t lo,
                                                   int64_t hi, int64_t key) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t rdeg_at(const int32_t* rdeg, int64_t dmax, int64_t d) {
  return rdeg[d < 0 ? 0 : (d > dmax + 2 ? dmax + 2 : d)];
}

// first index of b's owned prefix that can survive the O(1) bounds: the
// survivors are the suffix with deg(a) >= max(xmin - 1, simmax + 1)
__device__ __forceinline__ int64_t survivor_start(const SimParams& P, const int32_t* nb,
                                                  int64_t nlow, int2 th, int64_t dmax,
                                                  unsigned long long& bytes) {
  if (P.mode > MODE_CLEANUP) return 0;  // union / attach re-decide O(1) edges too
  const int64_t dstart = max((int64_t)th.x - 1, (int64_t)th.y + 1);
  bytes += 4ull * (unsigned long long)(64 - __clzll((unsigned long long)nlow));  // probes
  return lower_bound_run(nb, 0, nlow, rdeg_at(P.rdeg, dmax, dstart));
}

// The same search done by a whole CTA (NT threads, nlow <= NT^2 per round
// pair): NT sampled positions per round, __syncthreads_count brackets the
// answer, so two rounds of parallel loads replace ~log2(nlow) dependent ones.
template <int NT>
__device__ __forceinline__ int64_t survivor_start_cta(const SimParams& P, const int32_t* nb,
                                                      int64_t nlow, int2 th, int64_t dmax,
                                                      unsigned long long& bytes) {
  if (P.mode > MODE_CLEANUP || nlow == 0) return 0;
  const int64_t dstart = max((int64_t)th.x - 1, (int64_t)th.y + 1);
  const int64_t key = rdeg_at(P.rdeg, dmax, dstart);
  int64_t lo = 0, hi = nlow;  // answer in [lo, hi]: first index with nb[idx] >= key
  while (hi > lo) {
    const int64_t step = (hi - lo + NT - 1) / NT;
    const int64_t idx = lo + (int64_t)threadIdx.x * step;  // probes lo, lo+step, ...
    if (threadIdx.x == 0) bytes += 4ull * (unsigned long long)min((int64_t)NT, (hi - lo + step - 1) / step);
    const int cnt = __syncthreads_count(idx < hi && (int64_t)nb[idx] < key);
    // nb[lo + (cnt-1) step] < key <= nb[lo + cnt step] (if in range)
    const int64_t nlo = cnt == 0 ? lo : lo + (int64_t)(cnt - 1) * step + 1;
    const int64_t nhi = min(hi, lo + (int64_t)cnt * step);
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// The item-th high endpoint of a launch (largest first): from the stage-1 list
// of b's with a pending edge when the launch has one, else this shard's range.
__device__ __forceinline__ int64_t stage_b(const SimParams& P, int64_t rlo, int64_t rhi,
                                           int64_t item) {
  if (P.p1_list) {
    const int lo = P.p1_rng[0], hi = P.p1_rng[1];
    return item < hi - lo ? (int64_t)P.p1_list[hi - 1 - item] : rlo - 1;
  }
  return shard_top(rlo, rhi, item, P.shard_rank, P.shard_world);
}

// first index of the sorted run a[0, n) holding a value >= key, by a whole CTA
// (the same two-round sampled search)
template <int NT>
__device__ __forceinline__ int64_t cta_lower_bound(const int32_t* a, int64_t n, uint32_t key) {
  int64_t lo = 0, hi = n;
  while (hi > lo) {
    const int64_t step = (hi - lo + NT - 1) / NT;
    const int64_t idx = lo + (int64_t)threadIdx.x * step;
    const int cnt = __syncthreads_count(idx < hi && (uint32_t)a[idx] < key);
    const int64_t nlo = cnt == 0 ? lo : lo + (int64_t)(cnt - 1) * step + 1;
    const int64_t nhi = min(hi, lo + (int64_t)cnt * step);
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// ... and by one warp
__device__ __forceinline__ int64_t survivor_start_warp(const SimParams& P, const int32_t* nb,
                                                       int64_t nlow, int2 th, int64_t dmax,
                                                       int lane, unsigned long long& bytes) {
  if (P.mode > MODE_CLEANUP || nlow == 0) return 0;
  const int64_t dstart = max((int64_t)th.x - 1, (int64_t)th.y + 1);
  const int64_t key = rdeg_at(P.rdeg, dmax, dstart);
  int64_t lo = 0, hi = nlow;
  while (hi > lo) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t idx = lo + (int64_t)lane * step;
    if (lane == 0) bytes += 4ull * (unsigned long long)min((int64_t)32, (hi - lo + step - 1) / step);
    const int cnt = __popc(__ballot_sync(0xffffffffu, idx < hi && (int64_t)nb[idx] < key));
    const int64_t nlo = cnt == 0 ? lo : lo + (int64_t)(cnt - 1) * step + 1;
    const int64_t nhi = min(hi, lo + (int64_t)cnt * step);
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// tiny b: one thread per high endpoint b (deg < 64), its owned edges in
// order, merging two short runs.  Walking b's edges sequentially lets each
// decision (b's bounds are applied immediately) prune b's later edges, the
// progressive deferral of Alg. 2 line 2.

__global__ void __launch_bounds__(256) k_sim_tiny(SimParams P, int64_t rlo, int64_t rhi) {
  LocalCtr lc;
  const int w = P.shard_world;
  const int64_t first = rlo + ((P.shard_rank - rlo) % w + w) % w;  // first owned b >= rlo
  for (int64_t b = first + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * w; b < rhi;
       b += (int64_t)gridDim.x * blockDim.x * w) {
    const int64_t e0 = P.eoff[b], e1 = P.eoff[b + 1];
    if (e0 == e1) continue;
    if (P.mode >= MODE_UNION && !b_needed(P, b)) continue;
    const int64_t ob = P.off[b], eb = P.off[b + 1], db = eb - ob;
    lc.bytes += kBytesB;
    const int64_t j0 = survivor_start(P, P.adj + ob, e1 - e0, P.thr[db], P.dmax, lc.bytes);
    bool staged = false;
    for (int64_t e = e0 + j0; e < e1; ++e) {
      lc.bytes += kBytesCand;
      const int32_t a = P.adj[ob + (e - e0)];
      const int64_t ia0 = P.off[a], ea = P.off[a + 1];
      const int64_t da = ea - ia0;
      const int64_t cmax = da - 1;
      const int2 th = P.thr[db];
      const bool bdis = da + 1 < th.x, bsim = !bdis && da <= th.y;
      if ((bdis || bsim) && P.mode <= MODE_CLEANUP) continue;  // folded in by the pre-pass
      if (!edge_needed(P, e, a, (int32_t)b)) continue;
      bool res;
      if (bdis) res = false;  // union / attach: decided again, already counted
      else if (bsim) res = true;
      else {
        const int64_t cmin = c_min_exact(da, db, cmax, P.eps);
        int64_t c = 0, ia = ia0, ib = ob;
        res = false;
        // branch-free merge: both heads stay in registers, only the one that
        // advanced is reloaded (the loop issued two loads per step before)
        if (ia < ea && ib < eb) {
          int32_t x = P.adj[ia], y = P.adj[ib];
          for (;;) {
            const bool le = x <= y, ge = x >= y;
            c += (le && ge);
            ia += le;
            ib += ge;
            if (c >= cmin) { res = true; break; }
            if (ia >= ea || ib >= eb || c + (ea - ia) < cmin) break;
            if (le) x = P.adj[ia];
            if (ge) y = P.adj[ib];
          }
        }
        lc.probes += (unsigned long long)(ia - ia0);
        lc.inters++;
        lc.bytes += 4ull * (unsigned long long)((ia - ia0) + (ib - ob));  // the merge's reads
        lc.wsim += 4ull * (unsigned long long)da + (staged ? 0ull : 4ull * (unsigned long long)db);
        staged = true;
      }
      lc.bytes += kBytesRec + 16;  // + b's bounds (applied per edge here)
      record_edge(P, e, a, (int32_t)b, res, true, lc, !(bdis || bsim));
    }
  }
  flush_ctr(P, lc);
}

// ---------------------------------------------------------------------------
// CTA per high endpoint b with a hash table of N(b)

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

int launch_thresholds(int64_t dmax, const Eps2& eps, int2* thr, cudaStream_t st) {
  k_thresholds<<<grid_for(dmax + 1, 256), 256, 0, st>>>(dmax, eps, thr);
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// Lemma-1 pre-pass.  Whether an edge is decided by the O(1) degree bounds
// depends only on the two degrees, so every such edge is folded into the
// initial bounds here -- vertex-centric, no atomics -- and the identify sweep
// never touches it again (62.7% of the edges at s24 / eps 0.5).  Vertices the
// bounds already decide get their role before the sweep, so pruning starts
// immediately.  Sharded runs count only the edges they own.
__device__ __forceinline__ void prepass_edge(uint32_t dv, int64_t v, uint32_t dw, int64_t w,
                                             const int2* __restrict__ thr, int rank, int world,
                                             uint32_t& sim, uint32_t& dis, uint32_t& mine) {
  const bool vhi = w < v;  // rank order == (degree, id) order
  const uint32_t dlo = vhi ? dw : dv, dhi = vhi ? dv : dw;
  const int64_t hi = vhi ? v : w;
  if (!owns(hi, rank, world)) return;
  const int2 th = thr[dhi];
  const bool d = (int64_t)dlo + 1 < th.x;
  const bool s = !d && (int64_t)dlo <= th.y;
  dis += d;
  sim += s;
  mine += vhi && (d || s);
}

__device__ __forceinline__ void prepass_finish(int64_t v, uint32_t dv, uint32_t sim,
                                               uint32_t dis, int32_t mu,
                                               uint64_t* __restrict__ bounds,
                                               uint8_t* __restrict__ role) {
  const uint64_t lower = 1 + (uint64_t)sim, upper = (uint64_t)dv + 1 - dis;
  bounds[v] = lower | (upper << 32);
  role[v] = (int64_t)lower >= mu ? ROLE_CORE : (int64_t)upper < mu ? ROLE_NONCORE : ROLE_UNKNOWN;
}

// Degree tables for rank-space O(1) decisions.  Degrees ascend with the rank,
// so "deg(w) < d" is "w < rdeg[d]", and every O(1)-decided set of a vertex's
// neighbours is a prefix or suffix of its sorted run:
//   rdeg[d]  first rank with degree >= d (d in [0, dmax+2])
//   dx[d]    smallest high degree dh with d + 1 < xmin[dh] (low degree d is
//            dissimilar-by-bound against every dh >= dx[d]); dmax+1: none
//   ds[d]    largest high degree dh with d <= simmax[dh]; -1: none
__global__ void k_degree_tables(const int64_t* __restrict__ off, int64_t n, int64_t dmax,
                                const int2* __restrict__ thr, int32_t* __restrict__ rdeg,
                                int2* __restrict__ dxs) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d <= dmax + 2;
       d += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid + 1] - off[mid] < d) lo = mid + 1; else hi = mid;
    }
    rdeg[d] = (int32_t)lo;
    if (d > dmax) continue;
    int64_t a = 0, b = dmax + 1;  // xmin non-decreasing in dh: first dh with d + 1 < xmin
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (d + 1 < thr[mid].x) b = mid; else a = mid + 1;
    }
    int64_t c = 0, z = dmax + 1;  // simmax non-increasing in dh: first dh with simmax < d
    while (c < z) {
      const int64_t mid = (c + z) >> 1;
      if (thr[mid].y < d) z = mid; else c = mid + 1;
    }
    dxs[d] = make_int2((int32_t)a, (int32_t)(c - 1));
  }
}

// Lemma-1 pre-pass by binary search: four searches over v's sorted run give
// its O(1)-decided similar / dissimilar counts without touching each arc.
__global__ void k_prepass_bs(int64_t n, int64_t own_lo, int64_t own_hi, int64_t dmax,
                             const int64_t* __restrict__ off, const int64_t* __restrict__ eoff,
                             const int32_t* __restrict__ adj, const int2* __restrict__ thr,
                             const int32_t* __restrict__ rdeg, const int2* __restrict__ dxs,
                             int32_t mu, uint64_t* __restrict__ bounds,
                             uint8_t* __restrict__ role, unsigned long long* __restrict__ ctr) {
  unsigned long long decided = 0, bytes = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = off[v], dv = off[v + 1] - o;
    uint32_t sim = 0, dis = 0;
    bytes += 16 + 9;  // off[v..v+1]; bounds + role written
    if (v >= own_lo && v < own_hi && dv > 0) {
      const int64_t p0 = eoff[v + 1] - eoff[v];  // neighbours below v (v is their high end)
      const int2 th = thr[dv];
      const int64_t dl = lower_bound_run(adj, o, o + p0, rdeg_at(rdeg, dmax, (int64_t)th.x - 1)) - o;
      const int64_t sl = lower_bound_run(adj, o, o + p0, rdeg_at(rdeg, dmax, (int64_t)th.y + 1)) - o;
      const int2 xs = dxs[dv];
      const int64_t dh = dv - (lower_bound_run(adj, o + p0, o + dv, rdeg_at(rdeg, dmax, xs.x)) - o);
      const int64_t sh = lower_bound_run(adj, o + p0, o + dv,
                                         rdeg_at(rdeg, dmax, min(xs.y + 1, xs.x))) - o - p0;
      const int64_t slo = sl > dl ? sl - dl : 0;
      dis = (uint32_t)(dl + dh);
      sim = (uint32_t)(slo + (sh > 0 ? sh : 0));
      decided += (unsigned long long)(dl + slo);
      // eoff pair, thr, dxs, 4 rdeg entries + the four binary searches' probes
      const unsigned lp = 64 - __clzll((unsigned long long)p0),
                     lh = 64 - __clzll((unsigned long long)(dv - p0));
      bytes += 16 + 8 + 8 + 16 + 8ull * (lp + lh);
    }
    prepass_finish(v, (uint32_t)dv, sim, dis, mu, bounds, role);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    decided += __shfl_xor_sync(0xffffffffu, decided, o);
    bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
  }
  if ((threadIdx.x & 31) == 0 && decided) {
    atomicAdd(&ctr[CTR_SIM_EVALS], decided);
    atomicAdd(&ctr[CTR_BOUND_DECIDED], decided);
  }
  if ((threadIdx.x & 31) == 0 && bytes) atomicAdd(&ctr[CTR_B_PREP], bytes);
}

__global__ void k_prepass_thread(int64_t rlo, int64_t rhi, int64_t own_lo, int64_t own_hi,
                                 const int64_t* __restrict__ off,
                                 const int32_t* __restrict__ adj, const uint32_t* __restrict__ deg,
                                 const int2* __restrict__ thr, int32_t mu, int rank, int world,
                                 uint64_t* __restrict__ bounds, uint8_t* __restrict__ role,
                                 unsigned long long* __restrict__ ctr) {
  unsigned long long decided = 0;
  for (int64_t v = rlo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < rhi;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t dv = deg[v];
    uint32_t sim = 0, dis = 0, mine = 0;
    if (v < own_lo || v >= own_hi) {  // another rank's row: initial bounds only
      prepass_finish(v, dv, 0, 0, mu, bounds, role);
      continue;
    }
    for (int64_t i = off[v]; i < off[v + 1]; ++i) {
      const int32_t w = adj[i];
      prepass_edge(dv, v, deg[w], w, thr, rank, world, sim, dis, mine);
    }
    prepass_finish(v, dv, sim, dis, mu, bounds, role);
    decided += mine;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) decided += __shfl_xor_sync(0xffffffffu, decided, o);
  if ((threadIdx.x & 31) == 0 && decided) {
    atomicAdd(&ctr[CTR_SIM_EVALS], decided);
    atomicAdd(&ctr[CTR_BOUND_DECIDED], decided);
  }
}

__global__ void k_prepass_warp(int64_t rlo, int64_t rhi, int64_t own_lo, int64_t own_hi,
                                 const int64_t* __restrict__ off,
                               const int32_t* __restrict__ adj, const uint32_t* __restrict__ deg,
                               const int2* __restrict__ thr, int32_t mu, int rank, int world,
                               uint64_t* __restrict__ bounds, uint8_t* __restrict__ role,
                               unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long decided = 0;
  for (int64_t v = rlo + wid; v < rhi; v += nw) {
    const uint32_t dv = deg[v];
    uint32_t sim = 0, dis = 0, mine = 0;
    if (v < own_lo || v >= own_hi) {  // another rank's row: initial bounds only
      if (lane == 0) prepass_finish(v, dv, 0, 0, mu, bounds, role);
      continue;
    }
    for (int64_t i = off[v] + lane; i < off[v + 1]; i += 32) {
      const int32_t w = adj[i];
      prepass_edge(dv, v, deg[w], w, thr, rank, world, sim, dis, mine);
    }
    sim = __reduce_add_sync(0xffffffffu, sim);
    dis = __reduce_add_sync(0xffffffffu, dis);
    decided += mine;
    if (lane == 0) prepass_finish(v, dv, sim, dis, mu, bounds, role);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) decided += __shfl_xor_sync(0xffffffffu, decided, o);
  if (lane == 0 && decided) {
    atomicAdd(&ctr[CTR_SIM_EVALS], decided);
    atomicAdd(&ctr[CTR_BOUND_DECIDED], decided);
  }
}

__global__ void k_degrees(const int64_t* __restrict__ off, int64_t n, uint32_t* __restrict__ deg) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    deg[v] = (uint32_t)(off[v + 1] - off[v]);
}


// Claim the next b with a pending edge and start the bulk copy of N(b) into
// `buf` (16-byte aligned source: the list starts *pre words in).  Not inlined:
// its registers stay out of the kernel's scan loop (inlined: 142 B of spills).
__device__ __noinline__ int pf_claim_copy(int32_t* wq, const int32_t* pend, int64_t p1_lo,
                                          const int64_t* off, const int32_t* adj, int64_t rlo,
                                          int64_t rhi, int rank, int world, uint32_t* buf,
                                          int* pre_out, uint64_t* bar) {
  for (;;) {
    const int it = atomicAdd(wq, 1);
    const int64_t bb = shard_top(rlo, rhi, it, rank, world);
    if (bb < rlo) return it;
    if (pend[bb - p1_lo] == 0) continue;
    const int64_t o = off[bb], d = off[bb + 1] - o;
    const uintptr_t src = reinterpret_cast<uintptr_t>(adj + o);
    const uintptr_t s0 = src & ~uintptr_t(15);
    const uint32_t pre = (uint32_t)((src - s0) >> 2);
    const uint32_t bytes = (uint32_t)(((pre + d) * 4 + 15) & ~int64_t(15));
    *pre_out = (int)pre;
    fence_proxy_async_smem();  // the buffer's last reads (generic proxy) come first
    bulk_copy_g2s(buf, reinterpret_cast<const void*>(s0), bytes, bar);
    return it;
  }
}

// PF (identify stage 2, medium class): N(b) of the NEXT claimed b is copied
// into one of two shared-memory buffers by the bulk-copy engine (TMA,
// cp.async.bulk, completion on an mbarrier) while the CTA works on the current
// b, whose list is then read from shared memory by the survivor filter, the
// table build and the bitmap clean-up (`nbuf_words` words per buffer).
// S2: the identify stage-2 instance (SIM_PENDING edges only): the sketch
// machinery of the other modes is compiled out (fewer registers, no spills)
template <int NT, bool GTAB, bool PF = false, bool S2 = false>
__global__ void __launch_bounds__(NT, 2048 / NT > 2 ? 2048 / NT / 2 : 1) k_sim_hash(SimParams P, int64_t rlo, int64_t rhi,
                                                 uint32_t tcap, int qi, int chunk,
                                                 uint32_t hub_lo, uint32_t bm_words,
                                                 int64_t skw, uint32_t nbuf_words) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* bm = smem;  // [bm_words] + zero guard words (kept 16-byte aligned)
  // bitmap + >= 4 zero guard words, padded so the 16-byte buckets stay aligned
  uint32_t* tab_s = smem + ((bm_words + 4 + 3) & ~3u);
  // survivors of the O(1) filter: where N(a) starts, (a, deg a), (j, c_min)
  int64_t* surv_oa = reinterpret_cast<int64_t*>(tab_s + (GTAB ? 0 : 4 * (size_t)tcap));
  int2* surv_ad = reinterpret_cast<int2*>(surv_oa + chunk);
  int2* surv_jc = surv_ad + chunk;
  // sketch levels of b: S_b, then folded to 1/2, 1/4, ... (2 wb words, 16-byte aligned)
  uint32_t* sk_lev = reinterpret_cast<uint32_t*>(surv_jc + chunk);
  __shared__ int s_item, s_nsurv, s_next, s_nstash, s_nkeep;
  __shared__ unsigned int s_bsim, s_bdis;
  __shared__ int64_t s_nlo;
  __shared__ uint32_t s_stash[kStash];
  __shared__ unsigned long long s_ctr[LC_N];
  const int tid = threadIdx.x, lane = tid & 31;
  HotCtr lc;
  shared_ctr_init(s_ctr);
  Cuckoo C;
  C.tab = GTAB ? (P.gtab + (int64_t)blockIdx.x * P.gtab_stride) : tab_s;
  C.nstash = &s_nstash;
  C.stash = s_stash;
  for (uint32_t i = tid; i < ((bm_words + 4 + 3) & ~3u); i += NT) bm[i] = 0u;

  constexpr bool p1 = S2;  // identify stage 2: SIM_PENDING edges only
  // PF: the prefetched claim, its buffer's mbarrier phase and its list offset
  __shared__ int s_pitem;
  __shared__ int s_pref[2];
  __shared__ __align__(8) uint64_t s_mbar[2];
  uint32_t* nbuf = sk_lev + ((skw + 3) & ~int64_t(3));
  const bool pf = PF && p1;
  int cur = 0;
  uint32_t phase = 0;  // bit k: parity of buffer k's next completion
  auto pf_claim = [&](int k) -> int {
    return pf_claim_copy(P.wq + qi, P.p1_pend, P.p1_lo, P.off, P.adj, rlo, rhi, P.shard_rank,
                         P.shard_world, nbuf + (size_t)k * nbuf_words, &s_pref[k], &s_mbar[k]);
  };
  if (pf && tid == 0) {
    mbar_init(&s_mbar[0], 1);
    mbar_init(&s_mbar[1], 1);
    mbar_init_fence();
    s_pitem = pf_claim(0);
  }
  for (;;) {
    if (pf) {
      if (tid == 0) {
        s_item = s_pitem;
        if (shard_top(rlo, rhi, s_item, P.shard_rank, P.shard_world) >= rlo) s_pitem = pf_claim(cur ^ 1);
      }
    } else if (tid == 0) {
      s_item = atomicAdd(&P.wq[qi], 1);
    }
    __syncthreads();
    const int64_t b = stage_b(P, rlo, rhi, s_item);
    if (b < rlo) break;
    if ((P.mode >= MODE_UNION && !b_needed(P, b)) || (p1 && P.p1_pend[b - P.p1_lo] == 0)) {
      __syncthreads();  // s_item read by all before the next claim
      continue;
    }
    const int64_t ob = P.off[b], db = P.off[b + 1] - ob;
    const int64_t e0 = P.eoff[b], nlow = P.eoff[b + 1] - e0;
    const int32_t* __restrict__ nb = P.adj + ob;
    // N(b) as the CTA reads it: the landed shared-memory copy (PF) or global
    const int32_t* nbl = nb;
    if (pf) {
      mbar_wait(&s_mbar[cur], (phase >> cur) & 1u);
      phase ^= 1u << cur;
      nbl = reinterpret_cast<const int32_t*>(nbuf + (size_t)cur * nbuf_words) + s_pref[cur];
    }
    const int2 th = P.thr[db];
    const int64_t xmin = th.x, simmax = th.y;
    bool built = false, sk_staged = false, wsim_b = false;
    unsigned long long sb = kBytesB + (p1 ? 8 : 0);
    const int64_t j0 = p1 ? P.p1_j0[b - P.p1_lo] : survivor_start_cta<NT>(P, nb, nlow, th, P.dmax, sb);
    if (tid == 0) ctr_add(lc, LC_BYTES, sb);
    for (int64_t base = j0; base < nlow; base += chunk) {
      if (tid == 0) { s_nsurv = 0; s_next = 0; s_bsim = 0; s_bdis = 0; }
      __syncthreads();
      const int64_t lim = base + chunk < nlow ? base + chunk : nlow;
      if (tid == 0) ctr_add(lc, LC_BYTES, (unsigned long long)(lim - base) * (p1 ? 1u : kBytesCand));
      // filter + O(1) bounds, one candidate a per thread
      for (int64_t j = base + tid; j < lim; j += NT) {
        const int64_t e = e0 + j;
        if (p1 && P.sim[e] != SIM_PENDING) continue;  // decided (or skipped) by stage 1
        const int32_t a = nbl[j];
        const int64_t oa = P.off[a];
        const int64_t da = P.off[a + 1] - oa;
        if (p1) ctr_add(lc, LC_BYTES, kBytesCand);
        const bool bdec = da + 1 < xmin || da <= simmax;
        if (bdec && P.mode <= MODE_CLEANUP) continue;  // folded in by the pre-pass
        if (!edge_needed(P, e, a, (int32_t)b)) {
          if (p1) P.sim[e] = SIM_UNKNOWN;  // pruned since stage 1: undecided, as in Alg. 2
          continue;
        }
        if (da + 1 < xmin) {  // only union / attach get here (identify: pre-pass)
          record_edge(P, e, a, (int32_t)b, false, false, lc, false);
        } else if (da <= simmax) {
          record_edge(P, e, a, (int32_t)b, true, false, lc, false);
        } else {
          const int slot = atomicAdd(&s_nsurv, 1);
          ctr_add(lc, LC_WSIM, 4ull * (unsigned long long)da);  // SURVEY W_sim: 4 min(d)
          surv_oa[slot] = oa;
          surv_ad[slot] = make_int2(a, (int32_t)da);
          surv_jc[slot] = make_int2((int32_t)j, (int32_t)c_min_exact(da, db, da - 1, P.eps));
        }
      }
      __syncthreads();
      const int ns = s_nsurv;
      if (ns > 0) {
        if (tid == 0 && !wsim_b) ctr_add(lc, LC_WSIM, 4ull * (unsigned long long)db);  // once
        wsim_b = true;
        int ns_scan = ns;
        const bool tpass = !p1 && P.sk_thread && P.sk != nullptr && db >= P.sk_dmin &&
                           2 * sk_words(db, P.sk_lk) <= skw;
        if (!p1 && !sk_staged && P.sk != nullptr && db >= P.sk_dmin &&
            2 * sk_words(db, P.sk_lk) <= skw) {  // b's sketch and its folds, once per b
          const int64_t wb = sk_words(db, P.sk_lk);
          // the levels are precomputed (sketch.cu): one coalesced copy, one barrier
          const uint4* src = reinterpret_cast<const uint4*>(sk_row(P, b, db, wb));
          uint4* dst = reinterpret_cast<uint4*>(sk_lev);
          for (int64_t i = tid; i < (2 * wb - 4) / 4; i += NT) dst[i] = __ldg(src + i);
          __syncthreads();
          if (tid == 0) ctr_add(lc, LC_BYTES, 4ull * (unsigned long long)(2 * wb - 4));
          sk_staged = true;
        }
        if (tpass) {
          // thread-per-survivor sketch pass; the survivors it cannot decide
          // are compacted to the front for the warp scans
          const int64_t wbx = sk_words(db, P.sk_lk);
          int2 kad[2], kjc[2];
          int64_t koa[2];
          bool keep[2] = {false, false};
          if (tid == 0) s_nkeep = 0;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int i = tid + r * NT;
            if (i >= ns) continue;
            kad[r] = surv_ad[i];
            kjc[r] = surv_jc[i];
            koa[r] = surv_oa[i];
            keep[r] = true;
            if (sk_words(kad[r].y, P.sk_lk) <= P.sk_tmax && sk_try(P, kad[r].y, db, kjc[r].y)) {
              const int64_t wa = sk_words(kad[r].y, P.sk_lk);
              unsigned long long words = 0;
              const bool rej = sk_thread_rejects(sk_row(P, kad[r].x, kad[r].y, wa),
                                                 sk_lev + 2 * (wbx - wa), wa, wa, kad[r].y,
                                                 kjc[r].y, false, words);
              ctr_add(lc, LC_BYTES, 4ull * words + (rej ? kBytesRec : 0u));
              if (rej) {
                keep[r] = false;
                record_edge(P, e0 + kjc[r].x, kad[r].x, (int32_t)b, false, false, lc);
                ctr_add(lc, LC_SKETCH, 1);
                atomicAdd(&s_bdis, 1u);
              }
            }
          }
          __syncthreads();
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            if (!keep[r]) continue;
            const int k = atomicAdd(&s_nkeep, 1);
            surv_ad[k] = kad[r];
            surv_jc[k] = kjc[r];
            surv_oa[k] = koa[r];
          }
          __syncthreads();
          ns_scan = s_nkeep;
        }
        if (ns_scan > 0 && !built) {  // stage N(b) once per b: hub suffix -> bitmap, rest -> cuckoo
          // hub split of N(b), found by the CTA (no per-vertex table to build)
          const int64_t nlo = cta_lower_bound<NT>(nbl, db, hub_lo);
          if (tid == 0) {
            s_nlo = nlo;
            s_nstash = 0;
          }
          __syncthreads();
          uint32_t T = (uint32_t)((nlo * 5) / 12 + 1);  // <= 0.6 keys per slot
          if (T > tcap) T = tcap;
          C.T = T;
          for (uint32_t i = tid; i < T; i += NT)
              reinterpret_cast<uint4*>(C.tab)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
          __syncthreads();
          for (int64_t i = tid; i < db; i += NT) {
            const uint32_t w = (uint32_t)nbl[i];
            if (i >= nlo) {
              const uint32_t r = w - hub_lo;
              atomicOr(&bm[r >> 5], 1u << (r & 31));
            } else {
              cuckoo_insert(C, w);
            }
          }
          __syncthreads();
          built = true;
          if (tid == 0) ctr_add(lc, LC_BYTES, 4ull * (unsigned long long)db);  // N(b)
        }
        const int nstash = s_nstash;
        const int64_t nlo = s_nlo;
        const uint32_t rmax = bm_words * 32u;  // first bit of the zero guard word
        // one warp per surviving a, dynamic (scan_survivor), software-pipelined:
        // survivor s+1 is claimed and its first load issued before s is scanned
        const int64_t wb = P.sk != nullptr ? sk_words(db, P.sk_lk) : 0;
        const bool lev = 2 * wb <= skw && wb > 0 && sk_staged;
        int s = 0;
        if (lane == 0) s = atomicAdd(&s_next, 1);
        s = __shfl_sync(0xffffffffu, s, 0);
        uint32_t first = s < ns_scan ? first_element(P.adj + surv_oa[s], surv_ad[s].y, lane) : kPast;
        while (s < ns_scan) {
          int s2 = 0;
          if (lane == 0) s2 = atomicAdd(&s_next, 1);
          s2 = __shfl_sync(0xffffffffu, s2, 0);
          const uint32_t first2 =
              s2 < ns_scan ? first_element(P.adj + surv_oa[s2], surv_ad[s2].y, lane) : kPast;
          const int2 jc = surv_jc[s];
          const int2 ad = surv_ad[s];
          int32_t scanned = 0;
          bool skd = false;
          unsigned long long skbytes = 0;
          // long rows are left to the warp (thread-pass imbalance)
          if (!p1 && (!tpass || sk_words(ad.y, P.sk_lk) > P.sk_tmax) && sk_try(P, ad.y, db, jc.y)) {
            const int64_t wa = sk_words(ad.y, P.sk_lk);
            skbytes = 4ull * (unsigned long long)(lev ? wa : 2 * wa);
            const uint32_t* A = sk_row(P, ad.x, ad.y, wa);
            // b's level at a's resolution: staged in shared memory, or read from
            // its precomputed slot in global memory (huge b beyond the staged room)
            skd = sk_rejects_lev(A, lev ? sk_lev + 2 * (wb - wa) : sk_row(P, b, db, wb) + 2 * (wb - wa),
                                 wa, ad.y, jc.y, lane);
          }
          const bool res = !skd && scan_survivor<GTAB>(P.adj + surv_oa[s], ad.y, jc.y, bm, hub_lo,
                                                       rmax, C, nstash, nb, nlo, lane, scanned,
                                                       first);
          if (lane == 0) {
            ctr_add(lc, LC_PROBES, (unsigned long long)scanned);
            ctr_add(lc, skd ? LC_SKETCH : LC_INTERS, 1);
            ctr_add(lc, LC_BYTES, 4ull * (unsigned long long)scanned + kBytesRec + skbytes);
            surv_jc[s].y = res ? 1 : 0;  // recorded below, all survivors at once
            atomicAdd(res ? &s_bsim : &s_bdis, 1u);
          }
          s = s2;
          first = first2;
        }
        // record the chunk's decisions thread-per-edge: the bound atomics of
        // a (a returned value each) are all in flight together instead of one
        // per survivor on the deciding warp's critical path
        __syncthreads();
        for (int i = tid; i < ns_scan; i += NT)
          record_edge(P, e0 + surv_jc[i].x, surv_ad[i].x, (int32_t)b, surv_jc[i].y != 0, false, lc);
      }
      __syncthreads();
      if (tid == 0 && (s_bsim | s_bdis) &&
          (P.mode == MODE_IDENTIFY || P.mode == MODE_CLEANUP)) {
        apply_bounds(P.bounds, P.role, b, s_bsim, s_bdis, P.mu);
        ctr_add(lc, LC_BYTES, 16);
      }
      __syncthreads();
    }
    if (built) {  // clear the bitmap words this b set (O(deg b), not O(R))
      for (int64_t i = s_nlo + tid; i < db; i += NT) bm[((uint32_t)nbl[i] - hub_lo) >> 5] = 0u;
    }
    hot_flush_warp(lc, s_ctr);
    __syncthreads();  // bitmap clean and s_item read by all before the next b
    cur ^= 1;
  }
  hot_flush_warp(lc, s_ctr);
  shared_ctr_flush(P, s_ctr);
}

// ---------------------------------------------------------------------------
// small b (64 <= deg < 512): one warp per b, no CTA barriers.  Each warp owns
// a private cuckoo table of N(b) in shared memory; the 32 lanes filter 32
// candidates at a time (O(1) bounds), and the surviving edges are decided one
// by one by the whole warp with scan_survivor (data broadcast by shuffles).
static constexpr int kWarpBuckets = 256;  // 4 KB: deg < 512 -> <= 0.5 keys per slot
static constexpr int kWarpWords = 4 * kWarpBuckets + kStash + 4;

template <int NT, int MINB, bool S2 = false>
__global__ void __launch_bounds__(NT, MINB) k_sim_warp(SimParams P, int64_t rlo,
                                                               int64_t rhi, int qi) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* tab = smem + (size_t)wid * kWarpWords;
  Cuckoo C;
  C.tab = tab;
  C.stash = tab + 4 * kWarpBuckets;
  C.nstash = reinterpret_cast<int*>(C.stash + kStash);
  __shared__ unsigned long long s_ctr[LC_N];
  HotCtr lc;
  shared_ctr_init(s_ctr);
  constexpr bool p1 = S2;  // identify stage 2: SIM_PENDING edges only
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(&P.wq[qi], 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    const int64_t b = stage_b(P, rlo, rhi, item);
    if (b < rlo) break;
    if (P.mode >= MODE_UNION && !b_needed(P, b)) continue;
    if (p1 && P.p1_pend[b - P.p1_lo] == 0) continue;
    const int64_t ob = P.off[b], db = P.off[b + 1] - ob;
    const int64_t e0 = P.eoff[b], nlow = P.eoff[b + 1] - e0;
    const int32_t* __restrict__ nb = P.adj + ob;
    const int2 th = P.thr[db];
    bool built = false;
    uint32_t bsim = 0, bdis = 0;
    int64_t wb = 0;
    unsigned long long sb = kBytesB + (p1 ? 8 : 0);
    const int64_t j0 = p1 ? P.p1_j0[b - P.p1_lo] : survivor_start_warp(P, nb, nlow, th, P.dmax, lane, sb);
    if (lane == 0) ctr_add(lc, LC_BYTES, sb);
    for (int64_t base = j0; base < nlow; base += 32) {
      const int64_t j = base + lane;
      if (lane == 0)
        ctr_add(lc, LC_BYTES, (unsigned long long)min((int64_t)32, nlow - base) * (p1 ? 1u : kBytesCand));
      int st = 0;  // 0 none, 1 dissimilar by bound, 2 similar by bound, 3 survivor
      int32_t a = 0, da = 0, cmin = 0;
      int64_t oa = 0;
      if (j < nlow && (!p1 || P.sim[e0 + j] == SIM_PENDING)) {
        a = nb[j];
        oa = P.off[a];
        da = (int32_t)(P.off[a + 1] - oa);
        if (p1) ctr_add(lc, LC_BYTES, kBytesCand);
        const bool bdec = da + 1 < th.x || da <= th.y;
        const bool need = !(bdec && P.mode <= MODE_CLEANUP) && edge_needed(P, e0 + j, a, (int32_t)b);
        if (p1 && !need) P.sim[e0 + j] = SIM_UNKNOWN;  // pruned since stage 1
        if (need) {
          if (da + 1 < th.x) st = 1;
          else if (da <= th.y) st = 2;
          else {
            st = 3;
            cmin = (int32_t)c_min_exact(da, db, da - 1, P.eps);
            ctr_add(lc, LC_WSIM, 4ull * (unsigned long long)da);  // SURVEY W_sim: 4 min(d)
            // thread-per-candidate sketch bound (S_b folded from global, L1-resident)
            if (!p1 && P.sk_thread && P.sk != nullptr && db >= P.sk_dmin && sk_try(P, da, db, cmin)) {
              const int64_t wa = sk_words(da, P.sk_lk), wbb = sk_words(db, P.sk_lk);
              unsigned long long words = 0;
              const bool rej = sk_thread_rejects(sk_row(P, a, da, wa),
                                                 sk_row(P, b, db, wbb) + 2 * (wbb - wa), wa, wa,
                                                 da, cmin, true, words);
              ctr_add(lc, LC_BYTES, 4ull * words + (rej ? kBytesRec : 0u));
              if (rej) {
                st = 4;
                record_edge(P, e0 + j, a, (int32_t)b, false, false, lc);
                ctr_add(lc, LC_SKETCH, 1);
              }
            }
          }
          if (st == 1 || st == 2)  // only union / attach get here (identify: pre-pass)
            record_edge(P, e0 + j, a, (int32_t)b, st == 2, false, lc, false);
        }
      }
      bdis += __popc(__ballot_sync(0xffffffffu, st == 1 || st == 4));
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
        if (P.sk != nullptr && db >= P.sk_dmin) wb = sk_words(db, P.sk_lk);
        __syncwarp();
        built = true;
        if (lane == 0) {
          ctr_add(lc, LC_BYTES, 4ull * (unsigned long long)db);
          ctr_add(lc, LC_WSIM, 4ull * (unsigned long long)db);  // larger list once
        }
      }
      const int nstash = built ? *C.nstash : 0;
      // survivors of this batch, software-pipelined like the CTA kernel
      int src = smask ? __ffs(smask) - 1 : 0;
      uint32_t first = kPast;
      bool myres = false;
      if (smask) {
        const int32_t da0 = __shfl_sync(0xffffffffu, da, src);
        const int64_t oa0 = __shfl_sync(0xffffffffu, oa, src);
        first = first_element(P.adj + oa0, da0, lane);
      }
      while (smask) {
        smask &= smask - 1;
        const int src2 = smask ? __ffs(smask) - 1 : 0;
        const int32_t sa = __shfl_sync(0xffffffffu, a, src);
        const int32_t sda = __shfl_sync(0xffffffffu, da, src);
        const int32_t scm = __shfl_sync(0xffffffffu, cmin, src);
        const int64_t soa = __shfl_sync(0xffffffffu, oa, src);
        const int32_t da2 = __shfl_sync(0xffffffffu, da, src2);
        const int64_t oa2 = __shfl_sync(0xffffffffu, oa, src2);
        const uint32_t first2 = smask ? first_element(P.adj + oa2, da2, lane) : kPast;
        int32_t scanned = 0;
        bool skd = false;
        unsigned long long skbytes = 0;
        if (!p1 && !P.sk_thread && sk_try(P, sda, db, scm)) {
          const int64_t wa = sk_words(sda, P.sk_lk);
          skbytes = 4ull * (unsigned long long)(2 * wa);
          // S_b's level at a's resolution, from its precomputed slot
          skd = sk_rejects_lev(sk_row(P, sa, sda, wa), sk_row(P, b, db, wb) + 2 * (wb - wa), wa,
                               sda, scm, lane);
        }
        const bool res = !skd && scan_survivor<false>(P.adj + soa, sda, scm, nullptr, 0xffffffffu,
                                                      0, C, nstash, nb, db, lane, scanned, first);
        if (res) ++bsim; else ++bdis;
        if (lane == 0) {
          ctr_add(lc, LC_PROBES, (unsigned long long)scanned);
          ctr_add(lc, skd ? LC_SKETCH : LC_INTERS, 1);
          ctr_add(lc, LC_BYTES, 4ull * (unsigned long long)scanned + kBytesRec + skbytes);
        }
        if (lane == src) myres = res;
        src = src2;
        first = first2;
      }
      // the batch's decisions recorded by their own lanes at once (the bound
      // atomics of the a's in flight together, off the survivor loop)
      if (st == 3) record_edge(P, e0 + j, a, (int32_t)b, myres, false, lc);
    }
    if (lane == 0 && (bsim | bdis) && (P.mode == MODE_IDENTIFY || P.mode == MODE_CLEANUP)) {
      apply_bounds(P.bounds, P.role, b, bsim, bdis, P.mu);
      ctr_add(lc, LC_BYTES, 16);
    }
    hot_flush_warp(lc, s_ctr);
    __syncwarp();
  }
  hot_flush_warp(lc, s_ctr);
  shared_ctr_flush(P, s_ctr);
}

// ---------------------------------------------------------------------------
// Identify, stage 1 (k_sk_filter): the sketch bound for every surviving edge
// of the classes deg b >= 64, one thread per edge, before any table of N(b) is
// built.  The CTA-per-b kernels used to run this pass between two barriers
// per chunk of b's survivors -- the CTA then waited for its longest row (30%
// of the medium class's stall samples) at half occupancy.  Here warps are
// independent: a warp takes a work item of up to kP1Chunk candidates of one b
// (rank order, so neighbouring lanes have neighbouring degrees and rows of
// similar length), reads S_a and S_b's level at a's resolution straight from
// their sketch slots (b's level is shared by the warp, L1-resident), records
// the edges it proves dissimilar and marks the rest SIM_PENDING for stage 2
// (the class kernels, which then scan only pending edges and skip every b
// without one).
static constexpr int kP1Chunk = 256;  // candidates per work item

// per b of [rlo, rhi): survivor start (the O(1) bounds' suffix) and work items
__global__ void k_p1_items(SimParams P, int64_t rlo, int64_t rhi, int32_t* __restrict__ j0s,
                           int32_t* __restrict__ nit) {
  unsigned long long bytes = 0;
  for (int64_t b = rlo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < rhi;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t j0 = 0, cnt = 0;
    if (owns(b, P.shard_rank, P.shard_world)) {
      const int64_t ob = P.off[b], db = P.off[b + 1] - ob;
      const int64_t nlow = P.eoff[b + 1] - P.eoff[b];
      bytes += kBytesB + 8;
      j0 = survivor_start(P, P.adj + ob, nlow, P.thr[db], P.dmax, bytes);
      cnt = nlow - j0;
    }
    j0s[b - rlo] = (int32_t)j0;
    nit[b - rlo] = (int32_t)((cnt + kP1Chunk - 1) / kP1Chunk);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
  if ((threadIdx.x & 31) == 0 && bytes) atomicAdd(&P.ctr[CTR_B_SKETCH], bytes);
}

// item -> b (index from rlo); the item count lands in *total
__global__ void k_p1_owner(int64_t nb, const int32_t* __restrict__ nit,
                           const int32_t* __restrict__ ioff, int32_t* __restrict__ owner,
                           int32_t* __restrict__ total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = nit[i], o = ioff[i];
    for (int32_t t = 0; t < k; ++t) owner[o + t] = (int32_t)i;
    if (i == nb - 1) *total = o + k;
  }
}

// the stage-2 classes' slices of the list of b's with a pending edge:
// cls[k] = first list index with b >= bound[k] (k < 4), cls[4] = list size
__global__ void k_p1_bounds(const int32_t* __restrict__ list, const int* __restrict__ nsel,
                            int64_t b1, int64_t b2, int64_t b3, int64_t b4, int* __restrict__ cls) {
  const int t = threadIdx.x;
  const int64_t key = t == 0 ? b1 : t == 1 ? b2 : t == 2 ? b3 : b4;
  const int cnt = *nsel;
  if (t < 4) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int64_t)list[mid] < key) lo = mid + 1; else hi = mid;
    }
    cls[t] = lo;
  }
  if (t == 4) cls[4] = cnt;
}

// union / attach: the b's whose owned edges can need a decision (b_needed)
struct NeedB {
  const uint8_t* role;
  const uint8_t* coreadj;
  int mode, rank, world;
  __device__ bool operator()(int32_t b) const {
    if (!owns(b, rank, world)) return false;
    return role[b] == ROLE_CORE || (mode == MODE_ATTACH && coreadj[b]);
  }
};

struct HasPending {
  const int32_t* pend;
  int64_t lo;
  __device__ bool operator()(int32_t b) const { return pend[b - lo] > 0; }
};

template <int NT, int MINB, int UNROLL, bool NA = true, bool NAB = false>
__global__ void __launch_bounds__(NT, MINB) k_sk_filter(SimParams P, int64_t rlo,
                                                  const int32_t* __restrict__ j0s,
                                                  const int32_t* __restrict__ ioff,
                                                  const int32_t* __restrict__ owner,
                                                  const int32_t* __restrict__ total,
                                                  int32_t* __restrict__ pend) {
  __shared__ unsigned long long s_ctr[LC_N];
  const int lane = threadIdx.x & 31;
  HotCtr lc;
  shared_ctr_init(s_ctr);
  const int32_t T = *total;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(&P.wq[5], 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= T) break;
    const int32_t bi = owner[item];
    const int64_t b = rlo + bi;
    const int64_t ob = P.off[b], db = P.off[b + 1] - ob;
    const int64_t e0 = P.eoff[b], nlow = P.eoff[b + 1] - e0;
    const int64_t jlo = (int64_t)j0s[bi] + (int64_t)(item - ioff[bi]) * kP1Chunk;
    const int64_t jhi = min(nlow, jlo + kP1Chunk);
    const int32_t* __restrict__ nb = P.adj + ob;
    const bool skb = P.sk != nullptr && db >= P.sk_dmin;
    const int64_t wb = skb ? sk_words(db, P.sk_lk) : 0;
    const uint32_t* levb = skb ? sk_row(P, b, db, wb) : nullptr;
    // owner, ioff, j0s, off / eoff pairs of b; b's sketch slot once per b (the
    // warps re-read it from L1 / L2 per edge: not algorithmic traffic)
    const bool first_item = item == ioff[bi];
    if (lane == 0) ctr_add(lc, LC_BYTES, 44ull + (first_item && skb ? 4ull * (2 * wb - 4) : 0ull));
    uint32_t ndis = 0, npend = 0;
    // Software-pipelined over the item's batches of 32: batch i+1's degree and
    // role and batch i+2's a are in flight while batch i walks its rows, and
    // the role decision of a recorded edge (the bound atomic's returned value)
    // is taken one batch later, so neither latency sits on the walk's path.
    constexpr uint64_t kDis = 0ull - (1ull << 32);  // one dissimilar outcome: upper - 1
    int32_t pa = -1;                               // deferred role decision: a, old bounds
    uint64_t pold = 0;
    int32_t a1 = jlo + lane < jhi ? nb[jlo + lane] : -1;
    int32_t a2 = jlo + 32 + lane < jhi ? nb[jlo + 32 + lane] : -1;
    int64_t o1a = 0, o1b = 0;
    uint8_t r1 = 0;
    if (a1 >= 0) { o1a = P.off[a1]; o1b = P.off[a1 + 1]; r1 = ld_role(P.role, a1); }
    for (int64_t jb = jlo; jb < jhi; jb += 32) {
      const int32_t a = a1;
      const int64_t da = o1b - o1a;
      const uint8_t ra = r1;
      a1 = a2;
      if (a1 >= 0) { o1a = P.off[a1]; o1b = P.off[a1 + 1]; r1 = ld_role(P.role, a1); }
      a2 = jb + 64 + lane < jhi ? nb[jb + 64 + lane] : -1;
      if (pa >= 0) {  // the previous batch's record: noncore once upper < mu
        if ((int32_t)(uint32_t)((pold + kDis) >> 32) < P.mu) P.role[pa] = ROLE_NONCORE;
        pa = -1;
      }
      const uint8_t rb = ld_role(P.role, b);
      bool dis = false, pnd = false;
      if (a >= 0) {
        const int64_t e = e0 + jb + lane;
        unsigned long long by = kBytesCand;
        // every j >= j0 survives the O(1) bounds; identify skips an edge whose
        // endpoints both have a role (Alg. 2 line 2)
        if (ra == ROLE_UNKNOWN || rb == ROLE_UNKNOWN) {
          const int32_t cmin = (int32_t)c_min_exact(da, db, da - 1, P.eps);
          if (skb && sk_try(P, da, db, cmin)) {
            const int64_t wa = sk_words(da, P.sk_lk);
            unsigned long long words = 0;
            dis = sk_rejects256<UNROLL, NA, NAB>(sk_row(P, a, da, wa), levb + 2 * (wb - wa), wa,
                                                 da, cmin, words);
            by += 4ull * words;  // S_a's words read (b's level: per b, above)
          }
          if (dis) {  // record_edge(dissimilar), the role decision deferred
            P.sim[e] = SIM_DISSIMILAR;
            pold = atomicAdd(reinterpret_cast<unsigned long long*>(&P.bounds[a]),
                             (unsigned long long)kDis);
            pa = a;
            ctr_add(lc, LC_SKETCH, 1);
            by += kBytesRec;
          } else {
            P.sim[e] = SIM_PENDING;
            pnd = true;
            by += 1;
          }
        }
        ctr_add(lc, LC_BYTES, by);
      }
      ndis += __popc(__ballot_sync(0xffffffffu, dis));
      npend += __popc(__ballot_sync(0xffffffffu, pnd));
    }
    if (pa >= 0 && (int32_t)(uint32_t)((pold + kDis) >> 32) < P.mu) P.role[pa] = ROLE_NONCORE;
    if (lane == 0) {
      if (ndis) {
        apply_bounds(P.bounds, P.role, b, 0u, ndis, P.mu);
        ctr_add(lc, LC_BYTES, 16);
      }
      if (npend) atomicAdd(&pend[bi], (int32_t)npend);
    }
  }
  hot_flush_warp(lc, s_ctr);
  shared_ctr_flush(P, s_ctr);
}

// ---------------------------------------------------------------------------
// host driver

template <int NT, bool GTAB, bool PF = false>
static int launch_hash(gs_engine* e, const SimParams& P, int64_t rlo, int64_t rhi,
                       uint32_t tcap, int qi, int chunk, int64_t dcls, cudaStream_t st) {
  if (rhi <= rlo) return GS_OK;
  size_t smem =
      (size_t)((P.bm_words + 4 + 3) & ~3u) * 4 + (GTAB ? 0 : (size_t)tcap * 16) + (size_t)chunk * 24;
  // b's sketch levels in shared memory when they fit (else folded from global);
  // identify stage 2 needs none (stage 1 applied the sketch bound)
  int64_t skw = 0;
  const bool p1 = P.p1_pend != nullptr;
  if (P.sk != nullptr && !p1) {
    // dcls bounds the class's degrees (no device read, no host sync)
    const int64_t want = 2 * sk_words(dcls, P.sk_lk);
    const int64_t room = ((int64_t)e->smem_optin - 1024 - (int64_t)smem) / 4;  // static smem
    if (want <= room) {
      skw = want;
    } else if (GTAB && room >= 8) {  // one CTA per SM anyway: levels for the b's that fit
      skw = room & ~int64_t(3);
    }
    smem += (size_t)skw * 4;
  }
  // PF: two N(b) buffers for the bulk-copy prefetch -- measured and off by
  // default (GS_TMA=1 enables): the prefetch state costs 118 B of spills at the
  // 64-register cap and the buffers halve the survivor chunk; s24 eps 0.2 medium
  // class 12.8 -> 14.9 ms (eps 0.5: 0.31 -> 0.27 ms), DESIGN 3c
  static const bool tma_on = getenv("GS_TMA") && atoi(getenv("GS_TMA")) == 1;
  const bool pf = PF && p1 && tma_on;
  uint32_t nbuf_words = 0;
  if (pf) {
    nbuf_words = (uint32_t)((dcls + 8 + 3) & ~int64_t(3));
    smem += 2ull * nbuf_words * 4;
    // keep two CTAs per SM: halve the survivor chunk if the buffers do not fit
    static const bool keep_chunk = getenv("GS_TMA_KEEPCHUNK") != nullptr;  // experiments
    if (!keep_chunk && 2 * (smem + 1024) > 228 * 1024 && chunk > 256) {
      smem -= (size_t)chunk * 12;
      chunk /= 2;
    }
  }
  auto kern = pf ? k_sim_hash<NT, GTAB, PF, true>
                 : p1 ? k_sim_hash<NT, GTAB, false, true> : k_sim_hash<NT, GTAB, false, false>;
  GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  GS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)occ * e->sms;
  if (grid > rhi - rlo) grid = rhi - rlo;
  if (GTAB && grid > e->sms * 2) grid = e->sms * 2;
  kern<<<(unsigned)grid, NT, smem, st>>>(P, rlo, rhi, tcap, qi, chunk, P.hub_lo, P.bm_words,
                                         skw, nbuf_words);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

static int launch_warp(gs_engine* e, const SimParams& P, int64_t rlo, int64_t rhi, int qi,
                       cudaStream_t st) {
  if (rhi <= rlo) return GS_OK;
  constexpr int NT = 256;
  const size_t smem = (size_t)(NT / 32) * kWarpWords * 4;
  static const int minb = getenv("GS_WARP_MINB") ? atoi(getenv("GS_WARP_MINB")) : 4;
  const bool s2 = P.p1_pend != nullptr;
  auto kern = s2 ? (minb == 3 ? k_sim_warp<NT, 3, true> : k_sim_warp<NT, 4, true>)
                 : (minb == 3 ? k_sim_warp<NT, 3> : k_sim_warp<NT, 4>);
  GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  GS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)occ * e->sms;
  const int64_t nw = (rhi - rlo + NT / 32 - 1) / (NT / 32);
  if (grid > nw) grid = nw;
  kern<<<(unsigned)grid, NT, smem, st>>>(P, rlo, rhi, qi);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// hub bitmap range: the top 2^18 ranks (32 KB of shared memory per CTA)
static constexpr int64_t kHubBits = 1 << 18;

// Sharded runs split the pre-pass by rank-space rows: each rank folds ALL the
// O(1)-decided edges of its own rows into their bounds (each vertex counted by
// one rank, so the exchanged counts sum exactly), instead of every rank
// reading every arc for the edges it owns.
int run_prepass(gs_engine* e, int32_t mu) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  const int64_t n = g.n;
  if (n == 0) return GS_OK;
  int64_t own_lo = 0, own_hi = n;
  if (e->shard_world > 1)
    GS_TRY(part_rows(e, n, 2 * g.m, e->shard_rank, e->shard_world, &own_lo, &own_hi, nullptr));
  k_prepass_bs<<<(unsigned)std::min<int64_t>(grid_for(n, 256), (int64_t)e->sms * 32), 256, 0,
                 e->stream>>>(n, own_lo, own_hi, g.dmax, g.off, g.eoff, g.adj, s.thr, s.rdeg,
                              s.dxs, mu, s.bounds, s.role, s.ctr);
  e->launches++;
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

// Sketch resolution by epsilon (k bits per neighbour): the bound proves
// dissimilarity when c_min = eps sqrt(d_a d_b) clears the false hits
// ~ d_a d_b / M; lower eps needs finer sketches (sketch.cu).
static constexpr int64_t kSketchDmin = 32;  // below: one scan step decides (measured: 32 < 48 < 64)
static int sketch_lk(const Eps2& eps) {
  const double e = sqrt(eps.ratio);
  return e >= 0.33 ? 2 : 3;  // measured: k = 4 wins from eps 0.35, k = 8 at 0.3
}

int prepare_similarity(gs_engine* e, const Eps2& eps) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  GS_TRY(e->alloc_n(&s.thr, g.dmax + 1));
  k_thresholds<<<grid_for(g.dmax + 1, 256), 256, 0, e->stream>>>(g.dmax, eps, s.thr);
  GS_TRY(e->alloc_n(&s.rdeg, g.dmax + 3));
  GS_TRY(e->alloc_n(&s.dxs, g.dmax + 1));
  k_degree_tables<<<grid_for(g.dmax + 3, 256), 256, 0, e->stream>>>(g.off, g.n, g.dmax, s.thr,
                                                                    s.rdeg, s.dxs);
  e->launches++;
  {
    int lk = sketch_lk(eps);
    int64_t dmin = kSketchDmin;
    if (const char* v = getenv("GS_SKETCH")) {  // bits per neighbour (0: off), experiments
      const int k = atoi(v);
      lk = k <= 0 ? -1 : 31 - __builtin_clz((unsigned)k);
    }
    if (const char* v = getenv("GS_SKETCH_DMIN")) dmin = std::max(1, atoi(v));
    GS_TRY(build_sketch(e, lk, dmin));
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
  P.sim = s.sim;
  P.bounds = s.bounds;
  P.role = s.role;
  P.coreadj = s.coreadj;
  P.parent = s.parent;
  P.ctr = s.ctr;
  P.wq = s.wq;
  P.eps = eps;
  P.mu = mu;
  P.mode = mode;
  P.gtab = nullptr;
  P.gtab_stride = 0;
  P.thr = s.thr;
  P.rdeg = s.rdeg;
  P.dmax = g.dmax;
  P.sk = g.sk;
  P.skbase = g.skbase;
  P.sk_lk = g.sk_lk;
  P.sk_dmin = (int32_t)g.sk_dmin;
  P.sk_gate = 1.0f;
  P.sk_minscan = 0;
  if (const char* v = getenv("GS_SKETCH_GATE")) P.sk_gate = (float)atof(v);
  if (const char* v = getenv("GS_SKETCH_MINSCAN")) P.sk_minscan = atoi(v);
  P.sk_thread = 1;
  if (const char* v = getenv("GS_SKETCH_THREAD")) P.sk_thread = atoi(v);
  P.sk_tmax = 1 << 30;
  if (const char* v = getenv("GS_SKETCH_TMAX")) P.sk_tmax = atoi(v);
  P.shard_rank = e->shard_rank;
  P.shard_world = e->shard_world;
  const bool ident = mode == MODE_IDENTIFY;
  auto slot = [&](int c) { P.bslot = ident ? c : CTR_B_OTHER; };
  if (ident) e->kev_mark(2);
  {
    const int64_t bits = std::min<int64_t>(kHubBits, ((g.n + 31) / 32) * 32);
    P.hub_lo = (uint32_t)std::max<int64_t>(0, g.n - bits);
    P.bm_words = (uint32_t)((g.n - P.hub_lo + 31) / 32);
  }
  GS_CUDA(cudaMemsetAsync(s.wq, 0, 8 * sizeof(int32_t), e->stream));
  const int64_t* rc = g.rclass;
  // largest degree of the large / medium classes (sizes their sketch levels):
  // one host sync here instead of one per launch
  int64_t dcls[2] = {0, 0};
  {
    int64_t o[4] = {0, 0, 0, 0};
    if (rc[4] > rc[3]) GS_CUDA(cudaMemcpyAsync(o, g.off + rc[4] - 1, 16, cudaMemcpyDeviceToHost, e->stream));
    if (rc[3] > rc[2]) GS_CUDA(cudaMemcpyAsync(o + 2, g.off + rc[3] - 1, 16, cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    dcls[0] = o[1] - o[0];
    dcls[1] = o[3] - o[2];
  }
  // The tiny class (deg b < 64) owns edges no other class touches, so it can
  // run on the copy stream concurrently with stages 1 and 2 (GS_TINY_STREAM=1).
  // Measured and off by default: it loses the roles the other classes decide
  // first (pruning: +1.3 M evaluations at eps 0.5) and slows stage 1 down
  // while they share the SMs (21.73 vs 21.89 ms at eps 0.5, 92.4 vs 91.9 at 0.2).
  static const bool tiny_async = getenv("GS_TINY_STREAM") && atoi(getenv("GS_TINY_STREAM")) == 1;
  const bool tiny_on_cs = tiny_async && rc[1] > rc[0];
  cudaEvent_t tev0 = nullptr, tev1 = nullptr;
  auto launch_tiny = [&](cudaStream_t on) -> int {
    SimParams T = P;
    T.bslot = ident ? CTR_B_TINY : CTR_B_OTHER;
    T.p1_pend = nullptr;  // not in stage 1
    T.p1_j0 = nullptr;
    T.p1_list = nullptr;
    T.gtab = nullptr;
    int64_t grid = (rc[1] - rc[0] + 255) / 256;
    if (grid > e->sms * 16) grid = e->sms * 16;
    if (ident) e->kev_mark(9, on);
    k_sim_tiny<<<(unsigned)grid, 256, 0, on>>>(T, rc[0], rc[1]);
    if (ident) e->kev_mark(10, on);
    e->launches++;
    GS_CUDA(cudaGetLastError());
    return GS_OK;
  };
  if (tiny_on_cs) {
    GS_CUDA(cudaEventCreateWithFlags(&tev0, cudaEventDisableTiming));
    GS_CUDA(cudaEventCreateWithFlags(&tev1, cudaEventDisableTiming));
    GS_CUDA(cudaEventRecord(tev0, e->stream));
    GS_CUDA(cudaStreamWaitEvent(e->cstream, tev0, 0));
    GS_TRY(launch_tiny(e->cstream));
    GS_CUDA(cudaEventRecord(tev1, e->cstream));
  }
  // identify stage 1: the sketch filter over every surviving edge of deg b >= 64
  // (GS_P1=0: the class kernels run the sketch bound themselves, as before)
  static const bool p1_on = !(getenv("GS_P1") && atoi(getenv("GS_P1")) == 0);
  int32_t *p1_j0 = nullptr, *p1_nit = nullptr, *p1_ioff = nullptr, *p1_owner = nullptr,
          *p1_pend = nullptr, *p1_list = nullptr;
  int* p1_cls = nullptr;
  if (ident && p1_on && g.sk != nullptr && g.n > rc[1]) {
    const int64_t lo = rc[1], nb = g.n - lo;
    GS_TRY(e->alloc_n(&p1_j0, nb));
    GS_TRY(e->alloc_n(&p1_nit, nb));
    GS_TRY(e->alloc_n(&p1_ioff, nb + 1));  // [nb]: the item count
    GS_TRY(e->alloc_n(&p1_pend, nb));
    GS_TRY(e->alloc_n(&p1_owner, nb + g.m / kP1Chunk + 1));  // >= items
    GS_CUDA(cudaMemsetAsync(p1_pend, 0, sizeof(int32_t) * (size_t)nb, e->stream));
    P.bslot = CTR_B_SKETCH;
    const unsigned gi = (unsigned)std::min<int64_t>(grid_for(nb, 256), (int64_t)e->sms * 16);
    k_p1_items<<<gi, 256, 0, e->stream>>>(P, lo, g.n, p1_j0, p1_nit);
    size_t tb = 0;
    GS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, p1_nit, p1_ioff, nb, e->stream));
    void* tmp = nullptr;
    GS_TRY(e->alloc(&tmp, tb > 0 ? tb : 1));
    GS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, p1_nit, p1_ioff, nb, e->stream));
    e->release(tmp);
    k_p1_owner<<<gi, 256, 0, e->stream>>>(nb, p1_nit, p1_ioff, p1_owner, p1_ioff + nb);
    static const int p1v = getenv("GS_P1_VARIANT") ? atoi(getenv("GS_P1_VARIANT")) : 0;
    // 0: S_a read without L1 allocation (best), 1: with, 2: S_a and b's level
    // without, 3: two 32-byte steps per check
    auto kern = p1v == 1 ? k_sk_filter<256, 4, 1, false> : p1v == 2 ? k_sk_filter<256, 4, 1, true, true>
              : p1v == 3 ? k_sk_filter<256, 4, 2> : p1v == 5 ? k_sk_filter<256, 5, 1>
              : p1v == 6 ? k_sk_filter<256, 6, 1> : k_sk_filter<256, 4, 1>;
    int occ = 0;
    GS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0));
    kern<<<(unsigned)(std::max(occ, 1) * e->sms), 256, 0, e->stream>>>(P, lo, p1_j0, p1_ioff,
                                                                     p1_owner, p1_ioff + nb,
                                                                     p1_pend);
    e->launches += 4;
    GS_CUDA(cudaGetLastError());
    P.p1_pend = p1_pend;
    P.p1_j0 = p1_j0;
    P.p1_lo = lo;
    // the b's with a pending edge, ascending, and each class's slice of them
    // (GS_P1_LIST=0: the stage-2 launches claim every b of their class)
    // (the TMA prefetch variant claims from the class range itself)
    static const bool use_list = !(getenv("GS_P1_LIST") && atoi(getenv("GS_P1_LIST")) == 0) &&
                                 !(getenv("GS_TMA") && atoi(getenv("GS_TMA")) == 1);
    if (use_list) {
      GS_TRY(e->alloc_n(&p1_list, nb));
      GS_TRY(e->alloc_n(&p1_cls, 8));
      size_t tb2 = 0;
      thrust::counting_iterator<int32_t> it((int32_t)lo);
      const HasPending pred{p1_pend, lo};
      GS_CUDA(cub::DeviceSelect::If(nullptr, tb2, it, p1_list, p1_cls + 5, (int)nb, pred, e->stream));
      void* t2 = nullptr;
      GS_TRY(e->alloc(&t2, tb2 > 0 ? tb2 : 1));
      GS_CUDA(cub::DeviceSelect::If(t2, tb2, it, p1_list, p1_cls + 5, (int)nb, pred, e->stream));
      e->release(t2);
      k_p1_bounds<<<1, 32, 0, e->stream>>>(p1_list, p1_cls + 5, rc[1], rc[2], rc[3], rc[4], p1_cls);
      e->launches += 2;
      P.p1_list = p1_list;
    }
  }
  // union / attach: the class launches claim only the b's that can need a
  // decision (cores; for attach also the cores' neighbours), listed
  // ascending and sliced per class like stage 2's list, instead of claiming
  // every b of their class from one work counter (GS_CLUSTER_LIST=0)
  static const bool clu_list = !(getenv("GS_CLUSTER_LIST") && atoi(getenv("GS_CLUSTER_LIST")) == 0);
  if (!ident && clu_list && (mode == MODE_UNION || mode == MODE_ATTACH) && g.n > rc[1]) {
    const int64_t lo = rc[1], nb = g.n - lo;
    GS_TRY(e->alloc_n(&p1_list, nb));
    GS_TRY(e->alloc_n(&p1_cls, 8));
    size_t tb2 = 0;
    thrust::counting_iterator<int32_t> it((int32_t)lo);
    const NeedB pred{s.role, s.coreadj, mode, e->shard_rank, e->shard_world};
    GS_CUDA(cub::DeviceSelect::If(nullptr, tb2, it, p1_list, p1_cls + 5, (int)nb, pred, e->stream));
    void* t2 = nullptr;
    GS_TRY(e->alloc(&t2, tb2 > 0 ? tb2 : 1));
    GS_CUDA(cub::DeviceSelect::If(t2, tb2, it, p1_list, p1_cls + 5, (int)nb, pred, e->stream));
    e->release(t2);
    k_p1_bounds<<<1, 32, 0, e->stream>>>(p1_list, p1_cls + 5, rc[1], rc[2], rc[3], rc[4], p1_cls);
    e->launches += 2;
    P.p1_list = p1_list;
  }
  if (ident) e->kev_mark(3);
  // huge b first (longest work items), with an L2-resident table per CTA
  const int64_t rhuge = rc[4];
  if (g.n > rhuge) {
    const int64_t tcap_g = (g.dmax * 5) / 12 + 1;  // buckets
    const int64_t nblk = (int64_t)e->sms * 2;
    GS_TRY(e->alloc_n(&P.gtab, 4 * tcap_g * nblk));
    P.gtab_stride = 4 * tcap_g;
    slot(CTR_B_HUGE);
    if (P.p1_list) P.p1_rng = p1_cls + 3;
    GS_TRY((launch_hash<1024, true>(e, P, rhuge, g.n, (uint32_t)tcap_g, 4, 1024, g.dmax,
                                     e->stream)));
  }
  if (ident) e->kev_mark(4);
  // shared memory per CTA: hub bitmap (top 2^18 ranks: 32 KB) + cuckoo table
  // for the non-hub part of N(b) (16-byte buckets) + survivor lists (24 B
  // per candidate of a chunk); the small class runs warp-per-b
  slot(CTR_B_LARGE);
  if (P.p1_list) P.p1_rng = p1_cls + 2;
  GS_TRY((launch_hash<1024, false>(e, P, rc[3], rc[4], 8192, 3, 1024, dcls[0], e->stream)));
  if (ident) e->kev_mark(5);
  slot(CTR_B_MED);
  if (P.p1_list) P.p1_rng = p1_cls + 1;
  static const int med_chunk = getenv("GS_MED_CHUNK") ? atoi(getenv("GS_MED_CHUNK")) : 1024;
  GS_TRY((launch_hash<512, false, true>(e, P, rc[2], rc[3], 2048, 2, med_chunk, dcls[1], e->stream)));
  if (ident) e->kev_mark(6);
  slot(CTR_B_SMALL);
  if (P.p1_list) P.p1_rng = p1_cls + 0;
  GS_TRY(launch_warp(e, P, rc[1], rc[2], 1, e->stream));
  if (ident) e->kev_mark(7);
  if (tiny_on_cs) {  // join the tiny class
    GS_CUDA(cudaStreamWaitEvent(e->stream, tev1, 0));
    cudaEventDestroy(tev0);
    cudaEventDestroy(tev1);
  } else if (rc[1] > rc[0]) {
    GS_TRY(launch_tiny(e->stream));
  }
  if (ident) e->kev_mark(8);
  for (int32_t* x : {p1_j0, p1_nit, p1_ioff, p1_owner, p1_pend, p1_list}) e->release(x);
  e->release(p1_cls);
  if (P.gtab) {
    GS_CUDA(cudaStreamSynchronize(e->stream));
    e->release(P.gtab);
  }
  return GS_OK;
}

}  // namespace gs
