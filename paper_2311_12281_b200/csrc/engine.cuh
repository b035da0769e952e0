// engine.cuh -- device context, resident graph and scan state of libgscan.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace gs {

// Degree-rank space graph (the engine's only internal layout).
//
// Vertices are relabelled by rank = position in (degree, original id) order,
// the order the reference uses to orient edges (graph.py:218-231).  In rank
// space the oriented edge (a, b) -- a the lower-degree endpoint -- is simply
// "a < b", so the edges owned by the higher endpoint b are the prefix of b's
// sorted adjacency run that is smaller than b.  Oriented edge ids are
// e = eoff[b] + j for the j-th prefix element: edges are grouped by their
// HIGH endpoint, which is the endpoint whose list the similarity kernels
// stage in shared memory.
struct DevGraph {
  int64_t n = 0, m = 0;
  int64_t* off = nullptr;   // [n+1] CSR offsets (rank space)
  int32_t* adj = nullptr;   // [2m] sorted neighbour ranks
  int32_t* orig = nullptr;  // [n] rank -> caller vertex id
  int32_t* rank = nullptr;  // [n] caller vertex id -> rank
  int64_t* eoff = nullptr;  // [n+1] oriented-edge offsets (prefix counts)
  int32_t* elo = nullptr;   // [m] low endpoint a of edge e
  int32_t* ehi = nullptr;   // [m] high endpoint b of edge e
  int64_t dmax = 0;
  // rank boundaries of degree classes: first rank with degree >= kDegClass[i]
  static constexpr int kClasses = 6;
  int64_t rclass[kClasses] = {0};
  bool adj_external = false;  // adj is a caller buffer (partitioned build), not ours
  // Neighbourhood sketches (sketch.cu): vertex v of degree d >= sk_dmin owns
  // sk_words(d) words at sk + skbase[d] + (v - rdeg[d]) * sk_words(d), a
  // bitmap of hash(w) mod M over its neighbours w, M = pow2 >= 2^sk_lk * d.
  uint32_t* sk = nullptr;
  int64_t* skbase = nullptr;  // [dmax+2] first word of each degree's block
  int sk_lk = -1;             // log2 of bits per neighbour; -1: not built
  int64_t sk_dmin = 0;
};

// words of a degree-d sketch: M = the smallest power of two >= 2^lk * d
// (at least four words)
__host__ __device__ __forceinline__ int64_t sk_words(int64_t d, int lk) {
  const int64_t x = d << lk;
  if (x <= 128) return 4;  // >= 4 words: every sketch row is 16-byte aligned
#ifdef __CUDA_ARCH__
  return (1ll << (64 - __clzll(x - 1))) >> 5;
#else
  return (1ll << (64 - __builtin_clzll((unsigned long long)(x - 1)))) >> 5;
#endif
}

// degree-class thresholds used to route edges to kernels (by HIGH endpoint):
// [1,64) tiny (thread per edge), [64,512) small, [512,4096) medium,
// [4096,28672) large (CTA + shared-memory table), >= 28672 huge (L2 table)
__host__ __device__ constexpr int64_t deg_class(int c) {
  return c == 0 ? 1 : c == 1 ? 64 : c == 2 ? 512 : c == 3 ? 4096 : c == 4 ? 28672 : (1ll << 40);
}

// Scan working state (ClusterState, scan.py:87-134, re-laid out for atomics).
struct DevState {
  uint8_t* sim = nullptr;       // [m] similarity status per oriented edge
  uint64_t* bounds = nullptr;   // [n] lower | upper << 32 (Lemma 1 counters)
  uint8_t* role = nullptr;      // [n] ROLE_* (write-once during identify)
  int32_t* parent = nullptr;    // [n] union-find forest over cores (ranks)
  int32_t* label = nullptr;     // [n] canonical label (min caller id) per root
  int32_t* lmin = nullptr;      // [n] min cluster label per clustered vertex
  int32_t* lmax = nullptr;      // [n] max cluster label per clustered vertex
  unsigned long long* ctr = nullptr;  // device counters (see Ctr)
  int2* thr = nullptr;          // [dmax+1] per-degree O(1) thresholds for this epsilon
  int32_t* rdeg = nullptr;      // [dmax+3] first rank with degree >= d (degrees ascend with rank)
  int2* dxs = nullptr;          // [dmax+1] per low degree d: {dx, ds} (see sim.cu)
  int32_t* wq = nullptr;        // work-queue heads for persistent kernels
  uint8_t* coreadj = nullptr;   // [n] has a core neighbour (set before attach)
  int32_t* clist = nullptr;     // [ncores] the cores (core-centric cluster phases)
  int* lcnt = nullptr;          // [4] list sizes (cores, clustered, near) + spare
  bool sparse = false;          // this scan's union / attach run core-centric
};

enum Ctr {
  CTR_SIM_EVALS = 0,
  CTR_PROBES,
  CTR_UNION_RETRIES,
  CTR_BOUND_DECIDED,
  CTR_INTERSECTIONS,
  CTR_ALG_BYTES,
  CTR_UNRESOLVED,
  CTR_N_CORE,
  CTR_N_MEMBER,
  CTR_N_HUB,
  CTR_N_OUTLIER,
  CTR_N_CLUSTERS,
  CTR_CORES_PRE,
  CTR_SKETCH_DECIDED,
  // Algorithmic bytes of the identify pass per kernel class (DESIGN 5): every
  // global element the kernels read or write as graph / sketch / state data,
  // at its size (scratch tables excluded).  The roofline's numerator.
  CTR_B_PREP,   // thresholds, degree tables, hub split, sketch build, Lemma-1 pre-pass
  CTR_B_HUGE,   // k_sim_hash<1024, true>
  CTR_B_LARGE,  // k_sim_hash<1024, false>
  CTR_B_MED,    // k_sim_hash<512, false>
  CTR_B_SMALL,  // k_sim_warp
  CTR_B_TINY,   // k_sim_tiny
  CTR_B_SKETCH, // k_sk_filter (identify stage 1: the sketch bound, thread per surviving edge)
  CTR_B_OTHER,  // the same kernels in the cleanup / union / attach passes
  CTR_WSIM,     // SURVEY 8(d) W_sim terms counted on the device (4 min(d) per intersected edge)
  CTR_PCIE,     // out of core: bytes read zero-copy from mapped host memory
  CTR_COUNT
};
static constexpr int kKernelClasses = 7;  // CTR_B_PREP .. CTR_B_SKETCH

enum SimMode : int {
  MODE_IDENTIFY = 0,  // identifyCore (Alg. 2): skip if both roles decided
  MODE_CLEANUP = 1,   // unresolved endpoint, status unknown
  MODE_UNION = 2,     // core-core, unknown, roots differ -> union if similar
  MODE_ATTACH = 3     // core-noncore, unknown
};

struct SimParams {
  const int64_t* off;
  const int32_t* adj;
  const int64_t* eoff;
  uint8_t* sim;
  uint64_t* bounds;
  uint8_t* role;
  const uint8_t* coreadj;  // [n] vertex has a core neighbour (attach pass only)
  int32_t* parent;
  unsigned long long* ctr;
  int32_t* wq;
  uint32_t* gtab;  // global hash scratch for very large lists
  int64_t gtab_stride;
  const int2* thr;      // per degree d of b: {xmin, simmax} O(1) bounds (see sim.cu)
  const int32_t* rdeg;  // [dmax+3] first rank with degree >= d
  int64_t dmax;
  uint32_t hub_lo;      // first rank of the hub bitmap range
  uint32_t bm_words;    // hub bitmap words (range [hub_lo, n))
  const uint32_t* sk;   // neighbourhood sketches (nullptr: none), see DevGraph
  const int64_t* skbase;
  int sk_lk;
  int32_t sk_dmin;
  float sk_gate;        // try the sketch bound iff expected false hits < gate * c_min
  int32_t sk_minscan;   //   and the scan would need at least this many misses
  int sk_thread;        // thread-per-survivor sketch pass before the warp scans
  int32_t sk_tmax;      //   for rows of at most this many words (longer: per warp)
  int bslot;            // counter slot of this launch's algorithmic bytes (CTR_B_*)
  // identify stage 2: the sketch filter (k_sk_filter) ran first; only edges
  // it marked SIM_PENDING are scanned, b's with p1_pend[b - p1_lo] == 0 skipped
  const int32_t* p1_pend = nullptr;
  const int32_t* p1_j0 = nullptr;  // survivor start of b's owned prefix
  int64_t p1_lo = 0;
  // ... and the b's with a pending edge, ascending (p1_list), this launch's slice
  // [p1_rng[0], p1_rng[1]) of it: the stage-2 launches visit only those
  const int32_t* p1_list = nullptr;
  const int* p1_rng = nullptr;
  int shard_rank;       // this process owns the edges whose high endpoint
  int shard_world;      //   b satisfies b % shard_world == shard_rank
  Eps2 eps;
  int32_t mu;
  int mode;
};

}  // namespace gs

struct gs_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cstream = nullptr;  // host->device copies overlapped with the build
  // pinned staging for pageable host inputs (allocated on first use, kept)
  void* hstage = nullptr;
  size_t hstage_bytes = 0;
  uint64_t cap = 0;
  size_t live = 0, peak = 0;  // bytes in use (peak = high-water mark)
  size_t reserved = 0;        // bytes held: in use + cached free blocks
  std::unordered_map<void*, size_t> sizes;   // in-use blocks
  std::multimap<size_t, void*> cache;         // free blocks by size, reused by alloc
  void trim(size_t need);                     // free cached blocks until `need` fits
  gs::DevGraph g;
  gs::DevState s;
  int sms = 148;
  int smem_optin = 227 * 1024;  // max dynamic shared memory per block
  int64_t launches = 0;
  float last_h2d_ms = 0, last_build_ms = 0;
  int shard_rank = 0, shard_world = 1;  // multi-GPU edge ownership (b % world == rank)
  int32_t mu = 0;                       // parameters of the scan in progress
  gs::Eps2 eps{};
  unsigned long long ncores = 0;
  float phase_ms[GS_PH_COUNT] = {0};    // timings of the sharded phase calls
  // partitioned build (gs_engine_load_csr_part) waiting for gs_engine_load_finish
  bool pend_finish = false;
  int64_t pend_n = 0, pend_m = 0;
  int64_t pend_cls[gs::DevGraph::kClasses + 1] = {0};
  int* pend_bad = nullptr;
  // host-side pinned staging for counters
  unsigned long long* h_ctr = nullptr;
  std::vector<cudaEvent_t> ev;
  // identify-pass kernel-class timing: kev[0] / kev[1] around the preparation,
  // kev[2] at the start of the sweep, kev[3] after the sketch filter, kev[3 + c]
  // after class c (huge, large, medium, small, tiny); recorded when kev_on, read into
  // gs_stats.phase_ms[GS_PH_K_PREP ..] (kev_class_ms)
  cudaEvent_t kev[gs::kKernelClasses + 4] = {};  // see kev_class_ms
  bool kev_on = false;
  void kev_mark(int i, cudaStream_t on = nullptr);
  void kev_class_ms(double* out);  // [kKernelClasses], synchronises the events

  int alloc(void** p, size_t bytes);
  void release(void* p);
  template <class T>
  int alloc_n(T** p, int64_t count) {
    return alloc(reinterpret_cast<void**>(p), (size_t)(count > 0 ? count : 1) * sizeof(T));
  }
  void free_graph();
  void free_state();
};

// ingest.cpp: multi-threaded host memcpy (pageable -> pinned staging)
void gs_parallel_copy(void* dst, const void* src, size_t bytes);

namespace gs {
// build.cu
int build_from_edges(gs_engine* e, int64_t n, int64_t m, const int32_t* edges_dev);
// Partitioned builds: with part_world > 1 only the rank-space rows of part
// part_rank (~2m/part_world arcs each) are built, into adj_out (caller-owned,
// 2m) when given; slot_bounds[part_world + 1] receives every part's slot range;
// the engine then waits for finish_build once the caller filled the other parts.
int build_from_csr(gs_engine* e, int64_t n, int64_t m, const int64_t* off_dev,
                   const int32_t* adj_dev, int part_rank = 0, int part_world = 1,
                   int32_t* adj_out = nullptr, int64_t* slot_bounds = nullptr);
// host CSR: adjacency streamed in chunks on cstream, scattered as it lands
int build_from_csr_host(gs_engine* e, int64_t n, int64_t m, const int64_t* off_host,
                        const int32_t* adj_host, int part_rank = 0, int part_world = 1,
                        int32_t* adj_out = nullptr, int64_t* slot_bounds = nullptr);
int finish_build(gs_engine* e);
int ensure_endpoints(gs_engine* e);  // elo / ehi on first use
// rank-space rows [row_lo, row_hi) of part part_rank (~slots/part_world arcs each)
int part_rows(gs_engine* e, int64_t n, int64_t slots, int part_rank, int part_world,
              int64_t* row_lo, int64_t* row_hi, int64_t* slot_bounds);
// sim.cu
int run_similarity(gs_engine* e, int mode, const Eps2& eps, int32_t mu);
int prepare_similarity(gs_engine* e, const Eps2& eps);  // thresholds + hub split
int run_prepass(gs_engine* e, int32_t mu);  // O(1)-decided edges -> initial bounds
// sketch.cu: neighbourhood sketches for the exact dissimilarity bound (needs
// the per-scan rdeg table); lk < 0 releases them
int build_sketch(gs_engine* e, int lk, int64_t dmin);
// sketch rows built while a host CSR streams in (sketch.cu)
int sketch_stream_begin(gs_engine* e, int64_t n, int64_t dmax, int lk, int64_t dmin,
                        int32_t** rdeg_out);
int sketch_stream_rows(gs_engine* e, int64_t dmax, int lk, int64_t dmin, const int32_t* rdeg,
                       const int32_t* adj, const int32_t* lists, int64_t stride,
                       const int* counts, int64_t nlisted);
// cluster.cu: the scan as phases (single GPU: all of them in a row; sharded:
// the host layer runs the collectives between them, see dist.py)
int run_scan(gs_engine* e, int32_t mu, const Eps2& eps, uint8_t* role_out,
             int32_t* cluster_out, int out_on_device, gs_stats* st);
int phase_begin(gs_engine* e, int32_t mu, const Eps2& eps);
int phase_identify(gs_engine* e);
int phase_export_counts(gs_engine* e, int32_t* counts);
int phase_import_counts(gs_engine* e, const int32_t* counts);
int phase_resolve(gs_engine* e, bool allow_cleanup);
int phase_union(gs_engine* e);
int phase_export_pairs(gs_engine* e, int32_t* pairs, int64_t* npairs);
int phase_merge_pairs(gs_engine* e, const int32_t* pairs, int64_t npairs);
int phase_labels(gs_engine* e);
int phase_attach(gs_engine* e);
int phase_export_labels(gs_engine* e, int32_t* labels);
int phase_import_labels(gs_engine* e, const int32_t* labels);
int phase_finish(gs_engine* e, uint8_t* role_out, int32_t* cluster_out, int out_on_device,
                 gs_stats* st);
void fill_counters(gs_stats* st, int64_t n, int64_t m, const unsigned long long* h);
int read_counters(gs_engine* e, gs_stats* st);
int export_state(gs_engine* e, int stage, int32_t* lower, int32_t* upper, uint8_t* role,
                 int32_t* parent, uint8_t* sim, int32_t* pairs);
// owner of the edges of high endpoint b
__host__ __device__ __forceinline__ bool owns(int64_t b, int rank, int world) {
  return world == 1 || (int)(b % world) == rank;
}
// the item-th owned high endpoint from the top of [rlo, rhi) (< rlo: done)
__host__ __device__ __forceinline__ int64_t shard_top(int64_t rlo, int64_t rhi, int64_t item,
                                                      int rank, int world) {
  if (world == 1) return rhi - 1 - item;
  int64_t top = rhi - 1;
  top -= ((top - rank) % world + world) % world;
  return top - item * world;
}
// launch helper: grid for n items
inline unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  return (unsigned)g;
}
}  // namespace gs
