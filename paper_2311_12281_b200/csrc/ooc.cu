// ooc.cu -- check_sim batches (scan.py:241-258) and the partitioned,
// out-of-core scan (scan_out_of_core, partition.py:666-757; Alg. 5).
//
// Out-of-core design (B200-first restatement of Alg. 5 / Def. 9):
//   * The graph (reference CSR: offsets i64, adjacency i32) stays in PINNED
//     HOST memory.  Only per-vertex state is resident in HBM -- 13 bytes per
//     vertex in every phase: degree (4) + role (1) + either the Lemma-1
//     bounds (8, identify) or the forest/label pair (4 + 4, cluster/classify).
//   * Partitions are contiguous ranges of high endpoints b whose adjacency
//     slice fits a device buffer; slices are streamed with double-buffered
//     cudaMemcpyAsync on a copy stream while the previous partition computes.
//     The lists of the low endpoints a are gathered zero-copy from the mapped
//     pinned host arrays (Lemma 2: sigma(a, b) needs only N(a) and N(b)), so
//     no edge-extended subgraph is ever materialised (the reference's greedy
//     closure planner replicates R-MAT edges 181-1,993x).
//   * No per-edge status is kept: the union and attach passes re-decide the
//     edges they need with the same exact predicate (deterministic), so the
//     device footprint is independent of m.
//   * Every device allocation is counted against the HBM cap (engine
//     allocator); GS_EBUDGET if the resident state alone cannot fit.
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "simcore.cuh"

namespace gs {

// ---------------------------------------------------------------------------
// check_sim: order endpoints by (degree, id) = rank, verify adjacency, then
// count common neighbours by merge and apply the exact predicate.
__global__ void k_check_sim(int64_t k, const int32_t* __restrict__ U, const int32_t* __restrict__ V,
                            int64_t n, const int32_t* __restrict__ rank,
                            const int64_t* __restrict__ off, const int32_t* __restrict__ adj,
                            Eps2 eps, int8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = U[i], v = V[i];
    if (u < 0 || v < 0 || u >= n || v >= n || u == v) { out[i] = -1; continue; }
    int32_t a = rank[u], b = rank[v];
    if (a > b) { int32_t t = a; a = b; b = t; }
    int64_t lo = off[a], hi = off[a + 1];
    int64_t l = lo, h = hi;
    while (l < h) {
      int64_t mid = (l + h) >> 1;
      if (adj[mid] < b) l = mid + 1; else h = mid;
    }
    if (l >= hi || adj[l] != b) { out[i] = -1; continue; }
    int64_t ia = lo, ib = off[b];
    const int64_t ea = hi, eb = off[b + 1];
    int64_t c = 0;
    while (ia < ea && ib < eb) {
      const int32_t x = adj[ia], y = adj[ib];
      if (x == y) { ++c; ++ia; ++ib; }
      else if (x < y) ++ia;
      else ++ib;
    }
    out[i] = is_similar(c, ea - lo, eb - off[b], eps) ? 1 : 0;
  }
}

int check_sim_batch(gs_engine* e, int64_t k, const int32_t* u, const int32_t* v,
                    const Eps2& eps, int8_t* out) {
  if (k <= 0) return GS_OK;
  if (!e->g.rank) { set_error("no graph loaded"); return GS_EINVAL; }
  int32_t *du = nullptr, *dv = nullptr;
  int8_t* dout = nullptr;
  GS_TRY(e->alloc_n(&du, k));
  GS_TRY(e->alloc_n(&dv, k));
  GS_TRY(e->alloc_n(&dout, k));
  GS_CUDA(cudaMemcpyAsync(du, u, 4 * (size_t)k, cudaMemcpyHostToDevice, e->stream));
  GS_CUDA(cudaMemcpyAsync(dv, v, 4 * (size_t)k, cudaMemcpyHostToDevice, e->stream));
  k_check_sim<<<grid_for(k, 256), 256, 0, e->stream>>>(k, du, dv, e->g.n, e->g.rank, e->g.off,
                                                      e->g.adj, eps, dout);
  GS_CUDA(cudaGetLastError());
  GS_CUDA(cudaMemcpyAsync(out, dout, (size_t)k, cudaMemcpyDeviceToHost, e->stream));
  GS_CUDA(cudaStreamSynchronize(e->stream));
  e->release(du);
  e->release(dv);
  e->release(dout);
  return GS_OK;
}

// ---------------------------------------------------------------------------
// out-of-core kernels (original vertex ids; orientation by (degree, id))

enum OocMode : int { OOC_IDENTIFY = 0, OOC_UNION = 1, OOC_ATTACH = 2 };

struct OocParams {
  const int64_t* hoff;  // mapped host offsets [n+1]
  const int32_t* hadj;  // mapped host adjacency [2m]
  const int32_t* padj;  // device: adjacency slice of the partition
  const int64_t* poff;  // device: offsets slice [lo, hi] of the partition
  int64_t lo, hi, base;  // partition b range and off[lo]
  const uint32_t* deg;   // [n]
  uint64_t* bounds;      // [n] identify
  uint8_t* role;         // [n]
  int32_t* parent;       // [n] union forest; after flatten: min label (lmin)
  int32_t* aux;          // [n] root labels; after flatten: max label (lmax)
  const int2* thr;
  const int32_t* big;    // b ids of the partition with degree > kOocWarpMax
  int nbig;
  Eps2 eps;
  int32_t mu;
  int mode;
  unsigned long long* ctr;
  int32_t* wq;
  uint32_t* gtab;
  int64_t gtab_stride;
  // neighbourhood sketches (sketch.cu) of every vertex, in mapped pinned host
  // memory: vertex v's row starts at 16-byte unit hsk_off[v] (nullptr: none)
  const uint32_t* hsk;
  const uint32_t* hsk_off;
  int sk_lk;
  int32_t sk_dmin;
  float sk_gate;
};

static constexpr int64_t kOocWarpMax = 512;      // deg(b) <= this: warp per b
static constexpr int kOocWarpSk = 256;           // words of b's sketch levels per warp
static constexpr int64_t kOocSmemBuckets = 10240;  // 160 KB cuckoo, deg(b) <= 24576

__device__ __forceinline__ bool ooc_owns(uint32_t da, int32_t a, uint32_t db, int32_t b) {
  return da < db || (da == db && a < b);  // graph.py:226
}

// does (a, b) need a decision in this pass?
__device__ __forceinline__ bool ooc_needed(const OocParams& P, int32_t a, int32_t b) {
  const uint8_t ra = ld_role(P.role, a), rb = ld_role(P.role, b);
  if (P.mode == OOC_IDENTIFY) return ra == ROLE_UNKNOWN || rb == ROLE_UNKNOWN;
  if (P.mode == OOC_UNION) {
    if (ra != ROLE_CORE || rb != ROLE_CORE) return false;
    return uf_find(P.parent, a) != uf_find(P.parent, b);
  }
  return (ra == ROLE_CORE) != (rb == ROLE_CORE);  // attach
}

// Should (a, b) try the sketch bound (as sk_try, sim.cu)?
__device__ __forceinline__ bool ooc_sk_try(const OocParams& P, int64_t da, int64_t db,
                                           int32_t cmin) {
  if (P.hsk == nullptr || da < P.sk_dmin) return false;
  const float ma = 32.f * (float)sk_words(da, P.sk_lk), fa = (float)da;
  const float ef = fa * (1.f - __expf(-(float)db / ma)) + fa * fa / (2.f * ma);
  return ef < P.sk_gate * (float)cmin;
}

__device__ __forceinline__ const uint32_t* ooc_sk_row(const OocParams& P, int64_t v) {
  return P.hsk + 4 * (int64_t)P.hsk_off[v];  // zero-copy
}

// S_b and its folds (the layout of sk_stage_levels) hashed straight from the
// streamed slice N(b) -- the same bits as b's stored sketch, no host read
template <class Sync>
__device__ __forceinline__ void ooc_sk_levels(const int32_t* __restrict__ nb, int64_t db, int lk,
                                              uint32_t* lev, int t, int nt, Sync sync) {
  const int64_t wb = sk_words(db, lk);
  const uint32_t mask = (uint32_t)(wb * 32 - 1);
  for (int64_t i = t; i < wb; i += nt) lev[i] = 0u;
  sync();
  for (int64_t i = t; i < db; i += nt) {
    const uint32_t h = sk_hash((uint32_t)nb[i]) & mask;
    atomicOr(&lev[h >> 5], 1u << (h & 31));
  }
  sync();
  for (int64_t lo = 0, w = wb; w > 4; lo += w, w >>= 1) {
    const int64_t h = w >> 1;
    for (int64_t i = t; i < h; i += nt) lev[lo + w + i] = lev[lo + i] | lev[lo + h + i];
    sync();
  }
}

// record one decided edge; b's identify bounds are aggregated by the caller
__device__ __forceinline__ void ooc_record(const OocParams& P, int32_t a, int32_t b, bool sim,
                                           LocalCtr& lc) {
  lc.evals++;
  if (P.mode == OOC_IDENTIFY) {
    apply_bounds(P.bounds, P.role, a, sim ? 1u : 0u, sim ? 0u : 1u, P.mu);
  } else if (P.mode == OOC_UNION) {
    if (sim) uf_union(P.parent, a, b, lc.retries);
  } else if (sim) {
    const bool ca = ld_role(P.role, a) == ROLE_CORE;
    const int32_t core = ca ? a : b, w = ca ? b : a;
    const int32_t L = P.parent[core];
    atomicMin(&P.parent[w], L);
    atomicMax(&P.aux[w], L);
  }
}

__device__ __forceinline__ void ooc_flush(const OocParams& P, LocalCtr& lc) {
  SimParams S;
  S.ctr = P.ctr;
  S.bslot = CTR_PCIE;  // the out-of-core kernels count their zero-copy bytes
  flush_ctr(S, lc);
}

// small b: one warp per b, private cuckoo of N(b) from the streamed slice
template <int NT>
__global__ void __launch_bounds__(NT, 2048 / NT / 2) k_ooc_warp(OocParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  constexpr int kWB = 256;
  constexpr int kWW = 4 * kWB + kStash + 4 + kOocWarpSk;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* tab = smem + (size_t)wid * kWW;
  uint32_t* lev = tab + 4 * kWB + kStash + 4;  // b's sketch levels (16-byte aligned)
  Cuckoo C;
  C.tab = tab;
  C.stash = tab + 4 * kWB;
  C.nstash = reinterpret_cast<int*>(C.stash + kStash);
  LocalCtr lc;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(&P.wq[0], 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    const int64_t b = P.lo + item;
    if (b >= P.hi) break;
    const uint32_t db = P.deg[b];
    if (db == 0 || db > kOocWarpMax) continue;
    const int32_t* __restrict__ nb = P.padj + (P.poff[b - P.lo] - P.base);
    const int2 th = P.thr[db];
    bool built = false, skb = false;
    uint32_t bsim = 0, bdis = 0;
    const bool bsk = P.hsk != nullptr && 2 * sk_words(db, P.sk_lk) <= kOocWarpSk;
    for (uint32_t base = 0; base < db; base += 32) {
      const uint32_t j = base + lane;
      int st = 0;  // 0 none, 1 dissimilar by bound, 2 similar by bound, 3 survivor, 4 sketch
      int32_t a = 0, cmin = 0;
      uint32_t da = 0;
      bool want = false;
      if (j < db) {
        a = nb[j];
        da = P.deg[a];
        if (ooc_owns(da, a, db, (int32_t)b) && ooc_needed(P, a, (int32_t)b)) {
          if ((int64_t)da + 1 < th.x) st = 1;
          else if ((int64_t)da <= th.y) st = 2;
          else {
            st = 3;
            cmin = (int32_t)c_min_exact(da, db, (int64_t)da - 1, P.eps);
            want = bsk && ooc_sk_try(P, da, db, cmin);
          }
          if (st == 1 || st == 2) {
            lc.bound++;
            ooc_record(P, a, (int32_t)b, st == 2, lc);
          }
        }
      }
      uint32_t sku = 0;  // the candidate's sketch row (16-byte units), read here in parallel
      if (want) {
        sku = P.hsk_off[a];  // zero-copy
        lc.bytes += 4;
      }
      if (__any_sync(0xffffffffu, want) && !skb) {
        ooc_sk_levels(nb, db, P.sk_lk, lev, lane, 32, [] { __syncwarp(); });
        skb = true;
      }
      bdis += __popc(__ballot_sync(0xffffffffu, st == 1));
      bsim += __popc(__ballot_sync(0xffffffffu, st == 2));
      uint32_t smask = __ballot_sync(0xffffffffu, st == 3);
      if (smask && !built) {
        uint32_t T = (uint32_t)((db * 5) / 12 + 1);
        if (T > (uint32_t)kWB) T = kWB;
        C.T = T;
        for (uint32_t i = lane; i < T; i += 32)
          reinterpret_cast<uint4*>(tab)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        if (lane == 0) *C.nstash = 0;
        __syncwarp();
        for (uint32_t i = lane; i < db; i += 32) cuckoo_insert(C, (uint32_t)nb[i]);
        __syncwarp();
        built = true;
      }
      const int nstash = built ? *C.nstash : 0;
      while (smask) {
        const int src = __ffs(smask) - 1;
        smask &= smask - 1;
        const int32_t sa = __shfl_sync(0xffffffffu, a, src);
        const int32_t sda = (int32_t)__shfl_sync(0xffffffffu, da, src);
        const int32_t scm = __shfl_sync(0xffffffffu, cmin, src);
        if (__shfl_sync(0xffffffffu, want, src)) {  // sketch bound: the warp reads a's row
          const uint32_t u = __shfl_sync(0xffffffffu, sku, src);
          const int64_t wa = sk_words(sda, P.sk_lk), wb = sk_words(db, P.sk_lk);
          unsigned long long skb_read = 0;
          const bool rej = sk_rejects_lev4(P.hsk + 4 * (int64_t)u, lev + 2 * (wb - wa), wa, sda,
                                           scm, lane, skb_read);
          if (lane == 0) lc.bytes += skb_read;
          if (rej) {
            if (P.mode == OOC_IDENTIFY) ++bdis;
            if (lane == 0) {
              lc.sketch++;
              ooc_record(P, sa, (int32_t)b, false, lc);
            }
            continue;
          }
        }
        int64_t oa = 0;
        if (lane == 0) oa = P.hoff[sa];  // zero-copy: where N(a) starts in host memory
        oa = __shfl_sync(0xffffffffu, oa, 0);
        int32_t scanned;
        const bool res = scan_survivor<false>(P.hadj + oa, sda, scm, nullptr, 0xffffffffu, 0, C,
                                              nstash, nb, db, lane, scanned,
                                              first_element(P.hadj + oa, sda, lane));
        if (P.mode == OOC_IDENTIFY) { if (res) ++bsim; else ++bdis; }
        if (lane == 0) {
          lc.probes += (unsigned long long)scanned;
          lc.bytes += 8ull + 4ull * (unsigned long long)scanned;  // hoff[a] + N(a), zero-copy
          lc.inters++;
          ooc_record(P, sa, (int32_t)b, res, lc);
        }
      }
    }
    if (lane == 0 && P.mode == OOC_IDENTIFY && (bsim | bdis))
      apply_bounds(P.bounds, P.role, b, bsim, bdis, P.mu);
    __syncwarp();
  }
  ooc_flush(P, lc);
}

// big b: one CTA per b (listed in P.big), cuckoo of N(b) in shared memory or,
// for the largest lists, in an HBM slab per CTA
template <int NT, bool GTAB>
__global__ void __launch_bounds__(NT, 1) k_ooc_cta(OocParams P, uint32_t tcap, int chunk,
                                                  int64_t skw) {
  extern __shared__ __align__(16) uint32_t smem[];
  int64_t* surv_oa = reinterpret_cast<int64_t*>(smem + (GTAB ? 0 : 4 * (size_t)tcap));
  int2* surv_ad = reinterpret_cast<int2*>(surv_oa + chunk);
  int2* surv_jc = surv_ad + chunk;
  uint32_t* surv_sk = reinterpret_cast<uint32_t*>(surv_jc + chunk);  // sketch row or ~0
  uint32_t* lev = surv_sk + chunk;  // b's sketch levels [skw] (16-byte aligned: chunk % 4 == 0)
  __shared__ int s_item, s_nsurv, s_next, s_nstash;
  __shared__ unsigned int s_bsim, s_bdis;
  __shared__ uint32_t s_stash[kStash];
  const int tid = threadIdx.x, lane = tid & 31;
  LocalCtr lc;
  Cuckoo C;
  C.tab = GTAB ? (P.gtab + (int64_t)blockIdx.x * P.gtab_stride) : smem;
  C.nstash = &s_nstash;
  C.stash = s_stash;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(&P.wq[1], 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= P.nbig) break;
    const int32_t b = P.big[item];
    const uint32_t db = P.deg[b];
    const int32_t* __restrict__ nb = P.padj + (P.poff[b - P.lo] - P.base);
    const int2 th = P.thr[db];
    uint32_t T = (uint32_t)(((int64_t)db * 5) / 12 + 1);
    if (T > tcap) T = tcap;
    C.T = T;
    bool built = false, skb = false;
    const bool bsk = P.hsk != nullptr && 2 * sk_words(db, P.sk_lk) <= skw;
    for (uint32_t base = 0; base < db; base += chunk) {
      if (tid == 0) { s_nsurv = 0; s_next = 0; s_bsim = 0; s_bdis = 0; }
      __syncthreads();
      const uint32_t lim = base + chunk < db ? base + chunk : db;
      for (uint32_t j = base + tid; j < lim; j += NT) {
        const int32_t a = nb[j];
        const uint32_t da = P.deg[a];
        if (!ooc_owns(da, a, db, b) || !ooc_needed(P, a, b)) continue;
        if ((int64_t)da + 1 < th.x) {
          lc.bound++;
          ooc_record(P, a, b, false, lc);
          atomicAdd(&s_bdis, 1u);
        } else if ((int64_t)da <= th.y) {
          lc.bound++;
          ooc_record(P, a, b, true, lc);
          atomicAdd(&s_bsim, 1u);
        } else {
          const int slot = atomicAdd(&s_nsurv, 1);
          const int32_t cm = (int32_t)c_min_exact(da, db, (int64_t)da - 1, P.eps);
          surv_oa[slot] = P.hoff[a];  // zero-copy
          surv_ad[slot] = make_int2(a, (int32_t)da);
          surv_jc[slot] = make_int2((int32_t)j, cm);
          const bool tsk = bsk && ooc_sk_try(P, da, db, cm);
          surv_sk[slot] = tsk ? P.hsk_off[a] : 0xFFFFFFFFu;
          lc.bytes += tsk ? 12u : 8u;
        }
      }
      __syncthreads();
      const int ns = s_nsurv;
      int ns_scan = ns;
      if (ns > 0 && bsk && !skb) {  // b's sketch levels, hashed from the slice
        ooc_sk_levels(nb, db, P.sk_lk, lev, tid, NT, [] { __syncthreads(); });
        skb = true;
      }
      if (ns_scan > 0) {
        if (!built) {
          for (uint32_t i = tid; i < T; i += NT)
            reinterpret_cast<uint4*>(C.tab)[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
          if (tid == 0) s_nstash = 0;
          __syncthreads();
          for (uint32_t i = tid; i < db; i += NT) cuckoo_insert(C, (uint32_t)nb[i]);
          __syncthreads();
          built = true;
        }
        const int nstash = s_nstash;
        for (;;) {
          int s = 0;
          if (lane == 0) s = atomicAdd(&s_next, 1);
          s = __shfl_sync(0xffffffffu, s, 0);
          if (s >= ns_scan) break;
          const int2 jc = surv_jc[s];
          const int2 ad = surv_ad[s];
          const uint32_t u = surv_sk[s];
          if (u != 0xFFFFFFFFu) {  // sketch bound: the warp reads a's row
            const int64_t wa = sk_words(ad.y, P.sk_lk), wb = sk_words(db, P.sk_lk);
            unsigned long long skb_read = 0;
            const bool rej = sk_rejects_lev4(P.hsk + 4 * (int64_t)u, lev + 2 * (wb - wa), wa, ad.y,
                                             jc.y, lane, skb_read);
            if (lane == 0) lc.bytes += skb_read;
            if (rej) {
              if (lane == 0) {
                lc.sketch++;
                ooc_record(P, ad.x, b, false, lc);
                atomicAdd(&s_bdis, 1u);
              }
              continue;
            }
          }
          int32_t scanned;
          const bool res = scan_survivor<GTAB>(P.hadj + surv_oa[s], ad.y, jc.y, nullptr,
                                               0xffffffffu, 0, C, nstash, nb, db, lane, scanned,
                                               first_element(P.hadj + surv_oa[s], ad.y, lane));
          if (lane == 0) {
            lc.probes += (unsigned long long)scanned;
            lc.bytes += 4ull * (unsigned long long)scanned;  // N(a), zero-copy
            lc.inters++;
            ooc_record(P, ad.x, b, res, lc);
            atomicAdd(res ? &s_bsim : &s_bdis, 1u);
          }
        }
      }
      __syncthreads();
      if (tid == 0 && P.mode == OOC_IDENTIFY && (s_bsim | s_bdis))
        apply_bounds(P.bounds, P.role, b, s_bsim, s_bdis, P.mu);
      __syncthreads();
    }
  }
  ooc_flush(P, lc);
}

// Sketches of the partition's vertices (sketch.cu layout per vertex) into
// skbuf (16-byte unit u0 = hsk_off[lo]); the host copies them out.
__global__ void __launch_bounds__(256) k_ooc_sk_build(OocParams P, uint32_t* __restrict__ skbuf,
                                                      uint32_t u0) {
  __shared__ uint32_t sm[8][128];
  const int lane = threadIdx.x & 31;
  uint32_t* s = sm[threadIdx.x >> 5];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = P.lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); v < P.hi;
       v += nw) {
    const int64_t d = P.deg[v];
    if (d < P.sk_dmin) continue;
    const int64_t W = sk_words(d, P.sk_lk);
    const uint32_t mask = (uint32_t)(W * 32 - 1);
    const int32_t* __restrict__ nb = P.padj + (P.poff[v - P.lo] - P.base);
    uint32_t* out = skbuf + 4 * (int64_t)(P.hsk_off[v] - u0);
    uint32_t* t = W <= 128 ? s : out;  // long rows: global atomics (zeroed by the host)
    if (W <= 128)
      for (int64_t j = lane; j < W; j += 32) s[j] = 0u;
    __syncwarp();
    for (int64_t i = lane; i < d; i += 32) {
      const uint32_t h = sk_hash((uint32_t)nb[i]) & mask;
      atomicOr(&t[h >> 5], 1u << (h & 31));
    }
    __syncwarp();
    if (W <= 128)
      for (int64_t j = lane; j < W; j += 32) out[j] = s[j];
    __syncwarp();
  }
}

// list the partition's b with deg > kOocWarpMax, split at the smem capacity
__global__ void k_ooc_bigs(const uint32_t* __restrict__ deg, int64_t lo, int64_t hi,
                           int32_t* __restrict__ mid, int32_t* __restrict__ huge,
                           int* __restrict__ counts, int64_t smem_max) {
  for (int64_t b = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < hi;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = deg[b];
    if (d <= kOocWarpMax) continue;
    if (d <= smem_max) mid[atomicAdd(&counts[0], 1)] = (int32_t)b;
    else huge[atomicAdd(&counts[1], 1)] = (int32_t)b;
  }
}

__global__ void k_ooc_degree(const int64_t* __restrict__ hoff, int64_t n, uint32_t* __restrict__ deg,
                             uint64_t* __restrict__ bounds, uint8_t* __restrict__ role, int32_t mu,
                             unsigned long long* __restrict__ dmax) {
  unsigned long long mx = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = hoff[v + 1] - hoff[v];
    deg[v] = (uint32_t)d;
    bounds[v] = 1ull | ((uint64_t)(d + 1) << 32);
    role[v] = d + 1 < mu ? ROLE_NONCORE : ROLE_UNKNOWN;
    mx = (unsigned long long)d > mx ? (unsigned long long)d : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(dmax, mx);
}

__global__ void k_ooc_resolve(int64_t n, int32_t mu, const uint64_t* __restrict__ bounds,
                              uint8_t* __restrict__ role, unsigned long long* __restrict__ ctr) {
  unsigned long long unresolved = 0, cores = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    uint8_t r = role[v];
    if (r == ROLE_UNKNOWN) {
      const uint64_t b = bounds[v];
      const int32_t lower = (int32_t)(uint32_t)b, upper = (int32_t)(uint32_t)(b >> 32);
      if (lower >= mu) r = ROLE_CORE;
      else if (upper < mu) r = ROLE_NONCORE;
      else ++unresolved;
      role[v] = r;
    }
    cores += r == ROLE_CORE;
  }
  if (unresolved) atomicAdd(&ctr[CTR_UNRESOLVED], unresolved);
  if (cores) atomicAdd(&ctr[CTR_CORES_PRE], cores);
}

__global__ void k_ooc_singletons(int64_t n, const uint8_t* __restrict__ role,
                                 int32_t* __restrict__ parent, int32_t* __restrict__ aux) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    parent[v] = role[v] == ROLE_CORE ? (int32_t)v : -1;
    aux[v] = 0x7fffffff;
  }
}

// flatten cores to their root, then the canonical label (min id) per root
__global__ void k_ooc_flatten(int64_t n, const uint8_t* __restrict__ role, int32_t* parent,
                              int32_t* __restrict__ aux, unsigned long long* __restrict__ ctr) {
  unsigned long long roots = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] != ROLE_CORE) continue;
    const volatile int32_t* p = parent;
    int32_t x = (int32_t)v, px = p[x];
    while (px != x) { x = px; px = p[x]; }
    if (x == (int32_t)v) ++roots;
    atomicMin(&aux[x], (int32_t)v);
  }
  if (roots) atomicAdd(&ctr[CTR_N_CLUSTERS], roots);
}

// parent <- root after all roots are known (second pass keeps chases valid)
__global__ void k_ooc_to_root(int64_t n, const uint8_t* __restrict__ role, int32_t* parent) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (role[v] != ROLE_CORE) continue;
    const volatile int32_t* p = parent;
    int32_t x = (int32_t)v, px = p[x];
    while (px != x) { x = px; px = p[x]; }
    parent[v] = x;  // only ever shortens paths to the same root
  }
}

// lmin (in parent) and lmax (in aux) from the root labels held in aux
// lmin_out may be parent itself (in place: each thread reads parent[v] before
// it writes slot v), so neither is __restrict__
__global__ void k_ooc_labels(int64_t n, const uint8_t* __restrict__ role, const int32_t* parent,
                             const int32_t* __restrict__ rootlab, int32_t* lmin_out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    lmin_out[v] = role[v] == ROLE_CORE ? rootlab[parent[v]] : 0x7fffffff;
}

__global__ void k_ooc_lmax(int64_t n, const uint8_t* __restrict__ role, const int32_t* __restrict__ lmin,
                           int32_t* __restrict__ lmax) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    lmax[v] = role[v] == ROLE_CORE ? lmin[v] : -1;
}

// classify over a partition's vertices (their lists are streamed): hubs and
// outliers are written into the device role array
__global__ void k_ooc_classify(OocParams P) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = P.lo + wid; v < P.hi; v += nw) {
    if (P.role[v] == ROLE_CORE || P.aux[v] >= 0) continue;
    const int64_t lo = P.poff[v - P.lo] - P.base, hi = P.poff[v - P.lo + 1] - P.base;
    int cnt = 0;
    int32_t umin = 0x7fffffff, umax = -1;
    for (int64_t i = lo + lane; i < hi; i += 32) {
      const int32_t x = P.padj[i];
      const int32_t hx = P.aux[x];
      if (hx < 0) continue;
      ++cnt;
      umin = min(umin, P.parent[x]);
      umax = max(umax, hx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      umin = min(umin, __shfl_xor_sync(0xffffffffu, umin, o));
      umax = max(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    }
    if (lane == 0) P.role[v] = (cnt >= 2 && umin != umax) ? ROLE_HUB : ROLE_OUTLIER;
  }
}

// final roles / canonical ids, one thread per vertex: coalesced zero-copy
// stores into the caller's (mapped) host arrays
__global__ void k_ooc_output(int64_t n, const uint8_t* __restrict__ role,
                             const int32_t* __restrict__ lmin, const int32_t* __restrict__ lmax,
                             bool any_cluster, uint8_t* __restrict__ role_out,
                             int32_t* __restrict__ cluster_out, unsigned long long* __restrict__ ctr) {
  unsigned long long c[4] = {0, 0, 0, 0};
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    uint8_t f;
    int32_t cl = -1;
    const uint8_t r = role[v];
    if (!any_cluster) f = ROLE_OUTLIER;
    else if (r == ROLE_CORE) { f = ROLE_CORE; cl = lmin[v]; }
    else if (lmax[v] >= 0) { f = ROLE_MEMBER; cl = lmin[v]; }
    else f = r == ROLE_HUB ? ROLE_HUB : ROLE_OUTLIER;
    role_out[v] = f;
    cluster_out[v] = cl;
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
// host driver

// Host arrays are used zero-copy: already-pinned memory directly, otherwise
// registered (cudaHostRegisterMapped).  When registration is refused (small
// arrays sharing a page with another registration, exotic allocators) a pinned
// mapped mirror is used instead, copied in (inputs) or back (outputs).
struct Mapped {
  void* host = nullptr;
  void* dev = nullptr;
  void* mirror = nullptr;
  size_t bytes = 0;
  bool registered = false;
  bool copy_back = false;
};

static int map_host(const void* p, size_t bytes, bool input, Mapped& out) {
  out.host = const_cast<void*>(p);
  out.bytes = bytes;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost &&
      at.devicePointer) {
    out.dev = at.devicePointer;
    return GS_OK;
  }
  cudaGetLastError();
  cudaError_t err = cudaErrorInvalidValue;
  if (bytes >= (1u << 22)) {  // registering pays off for large arrays only
    unsigned flags = cudaHostRegisterMapped | (input ? cudaHostRegisterReadOnly : 0u);
    err = cudaHostRegister(out.host, bytes, flags);
    if (err != cudaSuccess && input) {
      cudaGetLastError();
      err = cudaHostRegister(out.host, bytes, cudaHostRegisterMapped);
    }
  }
  if (err == cudaSuccess) {
    out.registered = true;
    GS_CUDA(cudaHostGetDevicePointer(&out.dev, out.host, 0));
    return GS_OK;
  }
  cudaGetLastError();
  GS_CUDA(cudaHostAlloc(&out.mirror, bytes > 0 ? bytes : 1, cudaHostAllocMapped));
  if (input) memcpy(out.mirror, p, bytes);
  out.copy_back = !input;
  GS_CUDA(cudaHostGetDevicePointer(&out.dev, out.mirror, 0));
  return GS_OK;
}

static void unmap_host(Mapped& m) {
  if (m.registered) cudaHostUnregister(m.host);
  if (m.mirror) {
    if (m.copy_back) memcpy(m.host, m.mirror, m.bytes);
    cudaFreeHost(m.mirror);
  }
  m = Mapped();
}

static void* mapped_ptr(void* host) {
  void* dev = nullptr;
  if (cudaHostGetDevicePointer(&dev, host, 0) != cudaSuccess) {
    cudaGetLastError();
    return host;  // UVA: the host pointer is valid on the device
  }
  return dev;
}

// ---------------------------------------------------------------------------
// Partition plan (host only, no device calls): contiguous ranges of high
// endpoints b whose adjacency slice fits one of the two streaming buffers the
// cap leaves after the resident state.  The resident bytes are computed as the
// engine allocator will count them (512-byte granules), so a plan made by the
// caller (gs_plan_partitions -> PartitionPlan, partition.py:231-333's role)
// runs unchanged on the device; a given plan is validated, never re-cut.
// Per partition the host also counts the b's routed to the CTA kernels, so
// the sweeps launch them without a device round trip.

struct Partition {
  int64_t lo, hi, a0, a1;  // b range and adjacency slice [a0, a1)
  int64_t nmid, nhuge;     // b's with kOocWarpMax < deg <= smem_max / deg > smem_max
};

static constexpr int kOocSlabs = 32;  // CTAs of the L2-table kernel (one HBM slab each)

struct OocPlan {
  int64_t dmax = 0, smem_max = 0, tcap_g = 0, buf_elems = 0, max_verts = 0, vmax = 0;
  int64_t nmid_max = 0, nhuge_max = 0;
  bool sketches = true;
  std::vector<Partition> parts;
};

static size_t r512(size_t b) { return ((b > 0 ? b : 1) + 511) & ~size_t(511); }

static int ooc_plan(int64_t n, const int64_t* off, uint64_t cap, const int64_t* bounds,
                    int64_t nb, OocPlan& pl) {
  pl = OocPlan();
  if (n <= 0) return GS_OK;
  if (off[0] != 0) {
    set_error("invalid graph: vertex_offsets must start at 0");
    return GS_EINVAL;
  }
  const size_t resident = 13 * (size_t)n;
  if (cap && resident + (1u << 20) > cap) {
    char buf[200];
    snprintf(buf, sizeof(buf), "resident vertex state needs %zu bytes against a cap of %llu",
             resident, (unsigned long long)cap);
    set_error(buf);
    return GS_EBUDGET;
  }
  int64_t dmax = 0;
  for (int64_t v = 0; v < n; ++v) {
    const int64_t d = off[v + 1] - off[v];
    if (d < 0) {
      set_error("invalid graph: vertex_offsets must be non-decreasing");
      return GS_EINVAL;
    }
    dmax = std::max(dmax, d);
  }
  pl.dmax = dmax;
  pl.smem_max = kOocSmemBuckets * 4 * 3 / 5;  // keys the smem cuckoo holds
  pl.tcap_g = dmax > pl.smem_max ? (dmax * 5) / 12 + 1 : 0;
  if (const char* v = getenv("GS_SKETCH")) pl.sketches = atoi(v) > 0;
  // what the device allocates before the streaming buffers: deg, role, bounds,
  // counters, work queue, thresholds, the L2 tables of the huge lists
  const size_t fixed = r512(4 * (size_t)n) + r512((size_t)n) + r512(8 * (size_t)n) +
                       r512(8 * (size_t)(CTR_COUNT + 1)) + r512(32) + r512(8 * (size_t)(dmax + 1)) +
                       r512((size_t)kOocSlabs * 16 * (size_t)pl.tcap_g) + (2u << 20);
  const size_t avail = cap ? (cap > fixed ? cap - fixed : 0) : ((size_t)1 << 30);
  // two buffers of adjacency (4 B/elem) + offsets (8 B/vertex) + big lists
  // (+ with sketches, one partition's rows: <= k/4 bytes per element)
  int64_t buf_elems = (int64_t)(avail / 2 / 4 * (pl.sketches ? 1 : 3) / (pl.sketches ? 2 : 4));
  buf_elems = std::min<int64_t>(buf_elems, (int64_t)1 << 28);
  if (buf_elems < dmax || buf_elems < 1024) {
    char buf[200];
    snprintf(buf, sizeof(buf),
             "HBM cap %llu leaves %zu bytes for streaming; the largest list needs %llu",
             (unsigned long long)cap, avail, (unsigned long long)(4 * dmax));
    set_error(buf);
    return GS_EBUDGET;
  }
  pl.buf_elems = buf_elems;
  pl.max_verts = std::max<int64_t>(1, buf_elems / 4);
  if (bounds) {  // the caller's plan: validate, never re-cut
    if (nb < 1 || bounds[0] != 0 || bounds[nb] != n) {
      set_error("partition bounds must run from 0 to n");
      return GS_EINVAL;
    }
    for (int64_t k = 0; k < nb; ++k) {
      const int64_t lo = bounds[k], hi = bounds[k + 1];
      if (hi <= lo) {
        set_error("partition bounds must be strictly increasing");
        return GS_EINVAL;
      }
      if (off[hi] - off[lo] > buf_elems || hi - lo > pl.max_verts) {
        char buf[240];
        snprintf(buf, sizeof(buf),
                 "partition %lld ([%lld, %lld): %lld adjacency elements) exceeds the %lld-element "
                 "streaming buffer this cap allows", (long long)k, (long long)lo, (long long)hi,
                 (long long)(off[hi] - off[lo]), (long long)buf_elems);
        set_error(buf);
        return GS_EBUDGET;
      }
      pl.parts.push_back({lo, hi, off[lo], off[hi], 0, 0});
    }
  } else {
    for (int64_t lo = 0; lo < n;) {
      // largest hi with off[hi] - off[lo] <= buf_elems and hi - lo <= max_verts
      int64_t l = lo + 1, h = std::min<int64_t>(n, lo + pl.max_verts);
      while (l < h) {
        const int64_t mid = (l + h + 1) >> 1;
        if (off[mid] - off[lo] <= buf_elems) l = mid; else h = mid - 1;
      }
      pl.parts.push_back({lo, l, off[lo], off[l], 0, 0});
      lo = l;
    }
  }
  for (auto& p : pl.parts) {
    for (int64_t v = p.lo; v < p.hi; ++v) {
      const int64_t d = off[v + 1] - off[v];
      if (d > kOocWarpMax) ++(d <= pl.smem_max ? p.nmid : p.nhuge);
    }
    pl.vmax = std::max(pl.vmax, p.hi - p.lo);
    pl.nmid_max = std::max(pl.nmid_max, p.nmid);
    pl.nhuge_max = std::max(pl.nhuge_max, p.nhuge);
  }
  return GS_OK;
}

int plan_partitions(int64_t n, const int64_t* off, uint64_t cap, int64_t* bounds_out,
                    int64_t max_parts, int64_t* nparts, int64_t* stream_elems) {
  OocPlan pl;
  GS_TRY(ooc_plan(n, off, cap, nullptr, 0, pl));
  const int64_t np = (int64_t)pl.parts.size();
  if (nparts) *nparts = np;
  if (stream_elems) *stream_elems = pl.buf_elems;
  if (bounds_out && max_parts >= np) {
    for (int64_t k = 0; k < np; ++k) bounds_out[k] = pl.parts[k].lo;
    bounds_out[np] = n;
  }
  return GS_OK;
}

int validate_plan(int64_t n, const int64_t* off, uint64_t cap, const int64_t* bounds,
                  int64_t nb) {
  OocPlan pl;
  return ooc_plan(n, off, cap, bounds, nb, pl);
}

int scan_partitioned(gs_engine* e, int64_t n, int64_t m, const int64_t* off,
                     const int32_t* adj, int32_t mu, const Eps2& eps, uint8_t* role_out,
                     int32_t* cluster_out, gs_stats* st, const int64_t* part_bounds,
                     int64_t nb) {
  cudaStream_t cs = e->stream;
  if (n == 0) return GS_OK;
  if (off[0] != 0 || off[n] != 2 * m) {
    set_error("invalid graph: vertex_offsets must start at 0 and end at 2m");
    return GS_EINVAL;
  }
  // ---- the plan (host): resident state (13 bytes per vertex) + fixed scratch
  OocPlan pl;
  GS_TRY(ooc_plan(n, off, e->cap, part_bounds, nb, pl));
  Mapped moff, madj, mrole, mclus;
  GS_TRY(map_host(off, 8 * (size_t)(n + 1), true, moff));
  int rc = map_host(adj, 4 * (size_t)(2 * m > 0 ? 2 * m : 1), true, madj);
  if (rc == GS_OK) rc = map_host(role_out, (size_t)n, false, mrole);
  if (rc == GS_OK) rc = map_host(cluster_out, 4 * (size_t)n, false, mclus);
  auto cleanup = [&]() {
    unmap_host(moff);
    unmap_host(madj);
    unmap_host(mrole);
    unmap_host(mclus);
  };
  if (rc != GS_OK) { cleanup(); return rc; }
  const int64_t* hoff = static_cast<const int64_t*>(moff.dev);
  const int32_t* hadj = static_cast<const int32_t*>(madj.dev);

  cudaStream_t copy = nullptr;
  cudaEvent_t ev_copied[2], ev_free[2], t0, t1, t2, t3, t4, t5;
  cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking);
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&ev_copied[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming);
  }
  cudaEventCreate(&t0); cudaEventCreate(&t1); cudaEventCreate(&t2);
  cudaEventCreate(&t3); cudaEventCreate(&t4); cudaEventCreate(&t5);
  int result = GS_OK;
  int64_t launches = 0;
  int64_t pcie_host = 0;  // bytes the host moves over PCIe (copies, mapped reads it can count)
  int64_t nsketched = 0;
  uint32_t* hsk = nullptr;      // pinned host sketch rows
  uint32_t* hsk_off = nullptr;  // pinned host row offsets (16-byte units)
  uint32_t* skbuf = nullptr;    // device scratch: one partition's rows
  do {
    uint32_t* deg = nullptr;
    uint8_t* role = nullptr;
    uint64_t* bounds = nullptr;
    unsigned long long* ctr = nullptr;
    int32_t* wq = nullptr;
    if ((result = e->alloc_n(&deg, n)) != GS_OK) break;
    if ((result = e->alloc_n(&role, n)) != GS_OK) break;
    if ((result = e->alloc_n(&bounds, n)) != GS_OK) break;
    if ((result = e->alloc_n(&ctr, CTR_COUNT + 1)) != GS_OK) break;
    if ((result = e->alloc_n(&wq, 8)) != GS_OK) break;
    cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * (CTR_COUNT + 1), cs);
    cudaEventRecord(t0, cs);
    k_ooc_degree<<<e->sms * 8, 256, 0, cs>>>(hoff, n, deg, bounds, role, mu, ctr + CTR_COUNT);
    ++launches;
    pcie_host += 8 * (n + 1);  // the degree pass reads the mapped offsets
    const int64_t dmax = pl.dmax;  // from the host plan: no device round trip
    int2* thr = nullptr;
    if ((result = e->alloc_n(&thr, dmax + 1)) != GS_OK) break;
    GS_TRY(launch_thresholds(dmax, eps, thr, cs));
    ++launches;
    const int64_t smem_max = pl.smem_max;
    const int nslab = kOocSlabs;
    const int64_t tcap_g = pl.tcap_g;
    const int64_t buf_elems = pl.buf_elems;
    // sketch resolution as in sim.cu (k = 2^sk_lk bits per neighbour; -1: off)
    int sk_lk = sqrt(eps.ratio) >= 0.33 ? 2 : 3;
    int64_t sk_dmin = 32;  // as in HBM (measured at s26: 12.1 vs 12.7 s with 48)
    if (const char* v = getenv("GS_SKETCH")) {
      const int k = atoi(v);
      sk_lk = k <= 0 ? -1 : 31 - __builtin_clz((unsigned)k);
    }
    if (const char* v = getenv("GS_SKETCH_DMIN")) sk_dmin = std::max(1, atoi(v));
    const std::vector<Partition>& parts = pl.parts;
    const int64_t vmax = pl.vmax;
    // ---- neighbourhood sketches (sketch.cu) in mapped pinned host memory:
    // per-vertex row offsets (16-byte units) are laid out here, the rows are
    // hashed on the device from the streamed slices in a pre-pass below
    int64_t skbuf_units = 0;
    if (sk_lk >= 0) {
      if (cudaHostAlloc(&hsk_off, 4 * (size_t)(n + 1), cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError();
        hsk_off = nullptr;
      }
      uint64_t acc = 0;
      nsketched = 0;
      for (int64_t v = 0; hsk_off && v < n; ++v) {
        hsk_off[v] = (uint32_t)acc;
        const int64_t d = off[v + 1] - off[v];
        if (d >= sk_dmin) {
          acc += (uint64_t)sk_words(d, sk_lk) / 4;
          ++nsketched;
        }
        if (acc >= 0xFFFFFFFFull) break;
      }
      if (hsk_off && acc < 0xFFFFFFFFull) {
        hsk_off[n] = (uint32_t)acc;
        for (auto& p : parts)
          skbuf_units = std::max<int64_t>(skbuf_units, (int64_t)hsk_off[p.hi] - hsk_off[p.lo]);
        if (cudaHostAlloc(&hsk, 16 * (size_t)std::max<uint64_t>(acc, 1), cudaHostAllocMapped) !=
            cudaSuccess) {
          cudaGetLastError();
          hsk = nullptr;
        }
      }
      if (!hsk) {  // no room on the host: scan without sketches
        if (hsk_off) cudaFreeHost(hsk_off);
        hsk_off = nullptr;
      }
    }
    int32_t* pbuf[2] = {nullptr, nullptr};
    int64_t* obuf[2] = {nullptr, nullptr};
    int32_t *bigmid = nullptr, *bighuge = nullptr;
    int* bigcnt = nullptr;
    uint32_t* gtab = nullptr;
    for (int i = 0; i < 2 && result == GS_OK; ++i) {
      result = e->alloc_n(&pbuf[i], buf_elems);
      if (result == GS_OK) result = e->alloc_n(&obuf[i], vmax + 1);
    }
    if (result != GS_OK) break;
    if ((result = e->alloc_n(&bigmid, pl.nmid_max + 1)) != GS_OK) break;
    if ((result = e->alloc_n(&bighuge, pl.nhuge_max + 1)) != GS_OK) break;
    if ((result = e->alloc_n(&bigcnt, 2)) != GS_OK) break;
    if (tcap_g > 0 && (result = e->alloc_n(&gtab, 4 * tcap_g * nslab)) != GS_OK) break;
    if (hsk && e->alloc_n(&skbuf, 4 * std::max<int64_t>(skbuf_units, 1)) != GS_OK) {
      cudaFreeHost(hsk);  // the partition scratch does not fit the cap: no sketches
      cudaFreeHost(hsk_off);
      hsk = nullptr;
      hsk_off = nullptr;
      skbuf = nullptr;
    }

    OocParams P;
    memset(&P, 0, sizeof(P));
    P.hoff = hoff;
    P.hadj = hadj;
    P.deg = deg;
    P.bounds = bounds;
    P.role = role;
    P.thr = thr;
    P.eps = eps;
    P.mu = mu;
    P.ctr = ctr;
    P.wq = wq;
    P.gtab = gtab;
    P.gtab_stride = 4 * tcap_g;
    if (hsk) {
      P.hsk = static_cast<const uint32_t*>(mapped_ptr(hsk));
      P.hsk_off = static_cast<const uint32_t*>(mapped_ptr(hsk_off));
      P.sk_lk = sk_lk;
      P.sk_dmin = (int32_t)sk_dmin;
      P.sk_gate = 1.0f;
      if (const char* v = getenv("GS_SKETCH_GATE")) P.sk_gate = (float)atof(v);
    }
    const size_t smem_warp = 8 * (4 * 256 + kStash + 4 + kOocWarpSk) * 4;
    const size_t smem_base = (size_t)kOocSmemBuckets * 16 + 1024 * 28;
    const int64_t smem_opt = e->smem_optin - 1024;  // static shared memory
    // b's sketch levels in shared memory, as many words as fit (else no sketch for that b)
    const int64_t skw_cta =
        hsk ? std::min<int64_t>(2 * sk_words(smem_max, sk_lk), (smem_opt - (int64_t)smem_base) / 4) : 0;
    const int64_t skw_gta =
        hsk ? std::min<int64_t>(2 * sk_words((int64_t)dmax, sk_lk), (smem_opt - 1024 * 28) / 4) : 0;
    const size_t smem_cta = smem_base + 4 * (size_t)std::max<int64_t>(skw_cta, 0);
    const size_t smem_gta = 1024 * 28 + 4 * (size_t)std::max<int64_t>(skw_gta, 0);
    {
      const cudaError_t e1 = cudaFuncSetAttribute(
          k_ooc_warp<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_warp);
      const cudaError_t e2 = cudaFuncSetAttribute(
          k_ooc_cta<1024, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cta);
      const cudaError_t e3 = cudaFuncSetAttribute(
          k_ooc_cta<1024, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_gta);
      if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
        char buf[256];
        snprintf(buf, sizeof(buf), "shared memory configuration failed (%zu/%zu/%zu bytes: %s)",
                 smem_warp, smem_cta, smem_gta,
                 cudaGetErrorString(e1 != cudaSuccess ? e1 : e2 != cudaSuccess ? e2 : e3));
        cudaGetLastError();
        set_error(buf);
        result = GS_ECUDA;
        break;
      }
    }
    int occ_w = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_w, k_ooc_warp<256>, 256, smem_warp);
    if (occ_w < 1) occ_w = 1;

    // one sweep over all partitions; `body` launches the pass kernels
    auto sweep = [&](auto&& body) -> int {
      // the streaming buffers may still be read by the previous sweep's kernels
      GS_CUDA(cudaEventRecord(t4, cs));
      GS_CUDA(cudaStreamWaitEvent(copy, t4, 0));
      for (size_t p = 0; p < parts.size(); ++p) {
        const int k = (int)(p & 1);
        const Partition& pt = parts[p];
        // the buffer is free once the kernels of partition p-2 are done
        if (p >= 2) GS_CUDA(cudaStreamWaitEvent(copy, ev_free[k], 0));
        if (pt.a1 > pt.a0)
          GS_CUDA(cudaMemcpyAsync(pbuf[k], adj + pt.a0, 4 * (size_t)(pt.a1 - pt.a0),
                                  cudaMemcpyHostToDevice, copy));
        GS_CUDA(cudaMemcpyAsync(obuf[k], off + pt.lo, 8 * (size_t)(pt.hi - pt.lo + 1),
                                cudaMemcpyHostToDevice, copy));
        pcie_host += 4 * (pt.a1 - pt.a0) + 8 * (pt.hi - pt.lo + 1);
        GS_CUDA(cudaEventRecord(ev_copied[k], copy));
        GS_CUDA(cudaStreamWaitEvent(cs, ev_copied[k], 0));
        P.padj = pbuf[k];
        P.poff = obuf[k];
        P.lo = pt.lo;
        P.hi = pt.hi;
        P.base = pt.a0;
        GS_TRY(body(pt));
        GS_CUDA(cudaEventRecord(ev_free[k], cs));
      }
      return GS_OK;
    };
    auto sim_body = [&](const Partition& pt) -> int {
      GS_CUDA(cudaMemsetAsync(wq, 0, 8 * sizeof(int32_t), cs));
      GS_CUDA(cudaMemsetAsync(bigcnt, 0, 2 * sizeof(int), cs));
      k_ooc_bigs<<<grid_for(pt.hi - pt.lo, 256), 256, 0, cs>>>(deg, pt.lo, pt.hi, bigmid, bighuge,
                                                              bigcnt, smem_max);
      // the plan counted them on the host: no device round trip per partition
      const int64_t h_cnt[2] = {pt.nmid, pt.nhuge};
      const int64_t nw = (pt.hi - pt.lo + 7) / 8;
      k_ooc_warp<256><<<(unsigned)std::min<int64_t>(nw, (int64_t)occ_w * e->sms), 256, smem_warp,
                        cs>>>(P);
      launches += 2;
      if (h_cnt[0] > 0) {
        OocParams Q = P;
        Q.big = bigmid;
        Q.nbig = h_cnt[0];
        k_ooc_cta<1024, false><<<(unsigned)std::min<int64_t>(h_cnt[0], e->sms), 1024, smem_cta, cs>>>(
            Q, (uint32_t)kOocSmemBuckets, 1024, skw_cta);
        ++launches;
      }
      if (h_cnt[1] > 0) {
        GS_CUDA(cudaMemsetAsync(wq + 1, 0, sizeof(int32_t), cs));
        OocParams Q = P;
        Q.big = bighuge;
        Q.nbig = h_cnt[1];
        k_ooc_cta<1024, true><<<(unsigned)std::min<int64_t>(h_cnt[1], nslab), 1024, smem_gta, cs>>>(
            Q, (uint32_t)tcap_g, 1024, skw_gta);
        ++launches;
      }
      GS_CUDA(cudaGetLastError());
      return GS_OK;
    };
    // ---- sketch pre-pass: every vertex's row hashed from its streamed slice
    if (hsk) {
      auto sk_body = [&](const Partition& pt) -> int {
        const uint32_t u0 = hsk_off[pt.lo], u1 = hsk_off[pt.hi];
        if (u1 == u0) return GS_OK;
        GS_CUDA(cudaMemsetAsync(skbuf, 0, 16 * (size_t)(u1 - u0), cs));
        const int64_t nw = (pt.hi - pt.lo + 7) / 8;
        k_ooc_sk_build<<<(unsigned)std::min<int64_t>(nw, (int64_t)e->sms * 8), 256, 0, cs>>>(
            P, skbuf, u0);
        ++launches;
        GS_CUDA(cudaMemcpyAsync(hsk + 4 * (size_t)u0, skbuf, 16 * (size_t)(u1 - u0),
                                cudaMemcpyDeviceToHost, cs));
        pcie_host += 16 * (int64_t)(u1 - u0);
        GS_CUDA(cudaGetLastError());
        return GS_OK;
      };
      if ((result = sweep(sk_body)) != GS_OK) break;
      pcie_host += 4 * nsketched;  // the build reads each sketched vertex's row offset (mapped)
    }
    cudaEventRecord(t5, cs);  // end of the sketch pre-pass (== t0 without sketches)
    // ---- pass 1: identify (Alg. 5 first loop)
    P.mode = OOC_IDENTIFY;
    if ((result = sweep(sim_body)) != GS_OK) break;
    cudaEventRecord(t1, cs);
    k_ooc_resolve<<<e->sms * 8, 256, 0, cs>>>(n, mu, bounds, role, ctr);
    ++launches;
    unsigned long long hc[CTR_COUNT];
    cudaMemcpyAsync(hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, cs);
    if (cudaStreamSynchronize(cs) != cudaSuccess) { set_error("identify pass failed"); result = GS_ECUDA; break; }
    if (hc[CTR_UNRESOLVED]) {
      set_error("role resolution incomplete after full edge sweep");
      result = GS_EINTERNAL;
      break;
    }
    const unsigned long long ncores = hc[CTR_CORES_PRE];
    // ---- pass 2: cluster (Alg. 5 second loop); bounds memory becomes forest + labels
    e->release(bounds);
    bounds = nullptr;
    P.bounds = nullptr;
    int32_t *parent = nullptr, *aux = nullptr;
    if ((result = e->alloc_n(&parent, n)) != GS_OK) break;
    if ((result = e->alloc_n(&aux, n)) != GS_OK) break;
    P.parent = parent;
    P.aux = aux;
    k_ooc_singletons<<<e->sms * 8, 256, 0, cs>>>(n, role, parent, aux);
    ++launches;
    if (ncores > 0) {
      P.mode = OOC_UNION;
      if ((result = sweep(sim_body)) != GS_OK) break;
      k_ooc_flatten<<<e->sms * 8, 256, 0, cs>>>(n, role, parent, aux, ctr);
      k_ooc_to_root<<<e->sms * 8, 256, 0, cs>>>(n, role, parent);
      // lmin over parent's memory: needs the root labels (aux) intact
      k_ooc_labels<<<e->sms * 8, 256, 0, cs>>>(n, role, parent, aux, parent);
      k_ooc_lmax<<<e->sms * 8, 256, 0, cs>>>(n, role, parent, aux);
      launches += 4;
      P.mode = OOC_ATTACH;
      if ((result = sweep(sim_body)) != GS_OK) break;
    }
    cudaEventRecord(t2, cs);
    // ---- pass 3: classify (streamed lists), then results to the mapped host outputs
    auto cls_body = [&](const Partition& pt) -> int {
      const int64_t nw = pt.hi - pt.lo;
      k_ooc_classify<<<(unsigned)std::min<int64_t>(grid_for(nw * 32, 256), (int64_t)e->sms * 32), 256,
                       0, cs>>>(P);
      ++launches;
      GS_CUDA(cudaGetLastError());
      return GS_OK;
    };
    if (ncores > 0 && (result = sweep(cls_body)) != GS_OK) break;
    k_ooc_output<<<e->sms * 8, 256, 0, cs>>>(n, role, parent, aux, ncores > 0,
                                            static_cast<uint8_t*>(mrole.dev),
                                            static_cast<int32_t*>(mclus.dev), ctr);
    ++launches;
    pcie_host += 5 * n;  // roles + cluster ids written zero-copy
    cudaEventRecord(t3, cs);
    cudaMemcpyAsync(hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, cs);
    if (cudaStreamSynchronize(cs) != cudaSuccess) { set_error("classify pass failed"); result = GS_ECUDA; break; }
    if (st) {
      st->n = n;
      st->m = m;
      st->sim_evals = (int64_t)hc[CTR_SIM_EVALS];
      st->adj_probes = (int64_t)hc[CTR_PROBES];
      st->union_retries = (int64_t)hc[CTR_UNION_RETRIES];
      st->sim_decided_by_bound = (int64_t)hc[CTR_BOUND_DECIDED];
      st->sim_intersections = (int64_t)hc[CTR_INTERSECTIONS];
      st->sim_decided_by_sketch = (int64_t)hc[CTR_SKETCH_DECIDED];
      st->n_clusters = (int64_t)hc[CTR_N_CLUSTERS];
      st->n_core = (int64_t)ncores;
      st->partitions = (int64_t)parts.size();
      st->pcie_bytes = (int64_t)hc[CTR_PCIE] + pcie_host;
      st->kernel_launches = launches;
      float ms = 0;
      cudaEventElapsedTime(&ms, t0, t1); st->phase_ms[GS_PH_IDENTIFY] = ms;
      cudaEventElapsedTime(&ms, t1, t2); st->phase_ms[GS_PH_CLUSTER] = ms;
      cudaEventElapsedTime(&ms, t2, t3); st->phase_ms[GS_PH_CLASSIFY] = ms;
      cudaEventElapsedTime(&ms, t0, t3); st->phase_ms[GS_PH_TOTAL] = ms;
      cudaEventElapsedTime(&ms, t0, t5); st->phase_ms[GS_PH_BUILD] = ms;  // sketch pre-pass
    }
    if (st) {
      st->n_member = (int64_t)hc[CTR_N_MEMBER];
      st->n_hub = (int64_t)hc[CTR_N_HUB];
      st->n_outlier = (int64_t)hc[CTR_N_OUTLIER];
    }
  } while (false);
  cudaStreamSynchronize(cs);
  cudaStreamSynchronize(copy);
  cudaStreamDestroy(copy);
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(ev_copied[i]);
    cudaEventDestroy(ev_free[i]);
  }
  cudaEventDestroy(t0); cudaEventDestroy(t1); cudaEventDestroy(t2);
  cudaEventDestroy(t3); cudaEventDestroy(t4); cudaEventDestroy(t5);
  if (hsk) cudaFreeHost(hsk);
  if (hsk_off) cudaFreeHost(hsk_off);
  cleanup();
  return result;
}

}  // namespace gs
