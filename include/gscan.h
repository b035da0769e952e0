/*
 * gscan.h -- C-ABI of libgscan.so, the B200 (sm_100a) structural-clustering
 * engine that replaces the reference's clustering call.
 *
 * The reference (graphscan, pure Python) has no FFI; its drop-in boundary is
 * the pair of Python entry points below.  Each C entry point states which
 * reference interface it replaces; INTEGRATION.md shows the ctypes binding
 * the reference would add.  The Python host package
 * paper_2311_12281_b200 binds exactly these symbols.
 *
 *   gs_scan_csr        scan_in_memory(g, mu, epsilon, workers)   scan.py:965-982
 *   gs_scan_edges      build_graph(el) + scan_in_memory(...)     graph.py:162-259, scan.py:965
 *   gs_build_graph     build_graph(el)                           graph.py:162-259
 *   gs_scan_partitioned scan_out_of_core(meta, plan, mu, eps)    partition.py:666-757
 *   gs_check_sim       check_sim over a batch of edges           scan.py:241-258
 *   gs_plan_closure    partition_graph(g, budget, spill_dir)     partition.py:231-333
 *   gs_engine_*        a reusable device context (stream, memory pool,
 *                      resident graph) behind the one-shot calls
 *
 * Conventions
 *   - Plain pointers and sizes only.  Host pointers unless a flag says device.
 *   - Return 0 (GS_OK) or a GS_E* code; gs_last_error() gives the message of
 *     the calling thread's last failure.  No C++ exception crosses the ABI.
 *   - Error mapping used by the Python host (same taxonomy as the reference):
 *       GS_EINVAL -> ValueError       (scan.py:969-973, graph.py:181-195)
 *       GS_EBUDGET -> InfeasibleBudgetError(ValueError)  (partition.py:79-89)
 *       GS_ENOMEM -> MemoryError, GS_ECUDA/GS_EINTERNAL -> RuntimeError
 *   - The caller owns every buffer it passes; the library owns device memory
 *     and releases per-call temporaries before returning.  Engines are not
 *     shared between threads; one-shot calls are reentrant (no global
 *     mutable state besides the thread-local error string).
 *   - Epsilon enters as its exact square p/q (scan.py:155-158), each as two
 *     64-bit halves; the device threshold test is the integer predicate
 *     (c+2)^2 * q >= p * (da+1)(db+1) (scan.py:232-233) in 192-bit arithmetic.
 *
 * Role codes written to role_out (the reference's byte codes, scan.py:43-52):
 *   1 core, 3 member, 5 hub, 6 outlier.
 * cluster_out: canonical cluster id = minimum core vertex id of the cluster
 *   (for members: the minimum eligible cluster), -1 for hubs and outliers.
 */
#ifndef GSCAN_H
#define GSCAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 3

#define GS_OK 0
#define GS_EINVAL 1
#define GS_EBUDGET 2
#define GS_ECUDA 3
#define GS_ENOMEM 4
#define GS_EINTERNAL 5
#define GS_EPARSE 6 /* input outside the native grammar; err_line says where */

#define GS_ROLE_CORE 1
#define GS_ROLE_MEMBER 3
#define GS_ROLE_HUB 5
#define GS_ROLE_OUTLIER 6

/* epsilon^2 = p / q exactly; both < 2^128. */
typedef struct gs_eps2 {
  uint64_t p_lo, p_hi, q_lo, q_hi;
} gs_eps2;

/* Phase timings in milliseconds (CUDA events on the engine stream). */
enum {
  GS_PH_H2D = 0,      /* host -> device copy of the graph */
  GS_PH_BUILD = 1,    /* degree-rank relabel + CSR build on the device */
  GS_PH_IDENTIFY = 2, /* phase 1 similarity sweep (identify_core) */
  GS_PH_CLEANUP = 3,  /* role resolution (+ rare re-evaluation) */
  GS_PH_CLUSTER = 4,  /* phase 2: union-find, flatten, labels, attach */
  GS_PH_CLASSIFY = 5, /* phase 3: hub / outlier */
  GS_PH_D2H = 6,      /* result copy back */
  GS_PH_TOTAL = 7,
  GS_PH_SIM_KERNELS = 8, /* summed duration of the similarity kernels */
  /* identify pass by kernel class (CUDA events between the launches): */
  GS_PH_K_PREP = 9,    /* thresholds, degree tables, hub split, sketch build, Lemma-1 pre-pass */
  GS_PH_K_HUGE = 10,   /* k_sim_hash<1024, L2 table>  (deg b >= 28672) */
  GS_PH_K_LARGE = 11,  /* k_sim_hash<1024>            (4096 <= deg b < 28672) */
  GS_PH_K_MEDIUM = 12, /* k_sim_hash<512>             (512 <= deg b < 4096) */
  GS_PH_K_SMALL = 13,  /* k_sim_warp                  (64 <= deg b < 512) */
  GS_PH_K_TINY = 14,   /* k_sim_tiny                  (deg b < 64) */
  GS_PH_K_SKETCH = 15, /* k_sk_filter: sketch bound, thread per surviving edge (deg b >= 64) */
  GS_PH_COUNT = 16
};

/* StatsReport counters (scan.py:911-947) plus engine extras. */
typedef struct gs_stats {
  int64_t n, m;
  int64_t sim_evals;              /* edges whose similarity was decided */
  int64_t adj_probes;             /* adjacency elements probed */
  int64_t union_retries;          /* failed CAS hooks in union-find */
  int64_t probe_bound_violations; /* always 0: probes <= min degree */
  int64_t sim_decided_by_bound;   /* decided by the O(1) degree bounds */
  int64_t sim_intersections;      /* edges that ran a set intersection */
  int64_t alg_bytes_sim;          /* SURVEY 8(d) W_sim of the similarity pass */
  int64_t n_core, n_member, n_hub, n_outlier, n_clusters;
  int64_t partitions;             /* out-of-core / sharded passes */
  int64_t kernel_launches;        /* kernels launched (gs_engine_scan: load + scan) */
  int64_t peak_device_bytes;      /* high-water mark of engine allocations */
  int64_t sim_decided_by_sketch;  /* decided dissimilar by the sketch bound (no scan) */
  double phase_ms[GS_PH_COUNT];
  /* (ABI 2) algorithmic bytes of the identify pass per kernel class, in the
   * order of GS_PH_K_PREP .. GS_PH_K_SKETCH (ABI 3: + the sketch filter): every global element of graph,
   * sketch and state data the kernels read or write, at its size (early
   * exits counted where they stop; scratch tables excluded).  Divided by the
   * class's phase_ms this is the roofline's achieved bandwidth. */
  int64_t kernel_bytes[7];
  int64_t wsim_bytes;    /* SURVEY 8(d) W_sim: 4 min(d) per edge left by the O(1)
                          * bounds + 4 d_b per staged b (the accounting of
                          * round 1, reported for comparison only) */
  int64_t pcie_bytes;    /* out of core: bytes moved over PCIe (slices + zero-copy) */
} gs_stats;

typedef struct gs_engine gs_engine;

/* device < 0 selects the current device.  hbm_cap_bytes = 0: no cap.  With
 * a cap, every device allocation of the engine is counted against it and a
 * call that cannot fit returns GS_EBUDGET (the partitioned path is chosen
 * automatically by gs_scan_partitioned). */
int gs_engine_create(int device, uint64_t hbm_cap_bytes, gs_engine** out);
void gs_engine_destroy(gs_engine* e);
/* cudaStream_t the engine launches on (for callers timing with events). */
void* gs_engine_stream(gs_engine* e);

/* Load a graph into the engine.  `on_device` = 1 means the pointers are
 * device pointers (e.g. torch CUDA tensors); 0 means host memory (pinned or
 * pageable).  The CSR form is the reference Graph layout (vertex_offsets i64
 * [n+1], adjacency i32 [2m], sorted runs); the edge form is a normalised
 * EdgeList (pairs u<v, unique, interleaved i32 [2m]). */
int gs_engine_load_csr(gs_engine* e, int64_t n, int64_t m, const int64_t* offsets,
                       const int32_t* adjacency, int on_device);
int gs_engine_load_edges(gs_engine* e, int64_t n, int64_t m, const int32_t* edges_uv,
                         int on_device);

/* Partitioned load for the sharded scan: every rank computes the
 * degree-rank relabel, but relabels and sorts only the rank-space rows of its
 * part (~2m/part_world arcs) into adj_out (caller-owned device buffer, 2m
 * int32).  slot_bounds[part_world + 1] receives every part's slot range; the
 * caller fills the other parts' slices of adj_out (e.g. NCCL broadcast from
 * each owner, paper_2311_12281_b200/dist.py) and then calls
 * gs_engine_load_finish.  part_world = 1 is gs_engine_load_csr. */
int gs_engine_load_csr_part(gs_engine* e, int64_t n, int64_t m, const int64_t* offsets,
                            const int32_t* adjacency, int on_device, int part_rank,
                            int part_world, int32_t* adj_out, int64_t* slot_bounds);
int gs_engine_load_finish(gs_engine* e);

/* Run the three phases on the loaded graph.  Outputs are written to host
 * buffers (out_on_device = 0) or device buffers (1), indexed by the caller's
 * vertex ids.  role_out / cluster_out may be NULL to skip the copy. */
int gs_engine_scan(gs_engine* e, int32_t mu, const gs_eps2* eps2, uint8_t* role_out,
                   int32_t* cluster_out, int out_on_device, gs_stats* stats);

/* Sharded (multi-GPU) scan, SURVEY 8(e).  Every rank loads the same graph
 * into its engine and owns the oriented edges whose high endpoint b (in the
 * engine's degree-rank order) satisfies b % world == rank.  The phases below
 * are the single-GPU scan cut where a collective is needed; the host runs,
 * between them (paper_2311_12281_b200/dist.py, NCCL via torch.distributed):
 *   counts  [2n] i32 (similar | dissimilar per vertex)  -> all-reduce SUM
 *   pairs   [2*npairs] i32 (core, local root)            -> all-gather (merge forests)
 *   labels  [2n] i32 (min | max member label)            -> all-reduce MIN | MAX
 * Device buffers are caller-owned (capacity 2n).  With world = 1 and NULL
 * buffers the phases reproduce gs_engine_scan exactly. */
int gs_engine_set_shard(gs_engine* e, int rank, int world);
int gs_engine_phase_begin(gs_engine* e, int32_t mu, const gs_eps2* eps2);
int gs_engine_phase_identify(gs_engine* e, int32_t* counts_dev);
int gs_engine_phase_resolve(gs_engine* e, const int32_t* counts_dev, int64_t* ncores);
int gs_engine_phase_union(gs_engine* e, int32_t* pairs_dev, int64_t* npairs);
int gs_engine_phase_merge(gs_engine* e, const int32_t* pairs_dev, int64_t npairs);
int gs_engine_phase_attach(gs_engine* e, int32_t* labels_dev);
int gs_engine_phase_finish(gs_engine* e, const int32_t* labels_dev, uint8_t* role_out,
                           int32_t* cluster_out, int out_on_device, gs_stats* stats);

/* The engine's scan state in the reference ClusterState layout (scan.py:87-134),
 * host buffers indexed by caller ids (any may be NULL): lower/upper [n] i32
 * (Lemma-1 bounds incl. the vertex itself), role [n] u8 (internal codes
 * 0..6), parent [n] i32 (canonical cluster label, -1 hub, -2 none), and per
 * oriented edge sim [m] u8 (SIM_*) with its caller-id pair edge_pairs [2m]
 * (low-(degree, id) endpoint first; the host maps them onto the reference
 * edge_list order).  stage: 0 after the identify phase (gs_engine_phase_
 * resolve), 1 after the cluster phases (gs_engine_phase_attach), 2 after
 * gs_engine_phase_finish.  Replaces direct access to ClusterState fields
 * (scan.py:87-107) for callers of identify_core / detect_clusters /
 * classify_hub_outlier (scan.py:452, 701, 832). */
int gs_engine_export_state(gs_engine* e, int stage, int32_t* lower, int32_t* upper,
                           uint8_t* role, int32_t* parent, uint8_t* sim, int32_t* edge_pairs);
/* Counters and per-phase device times of the engine's scan so far (the
 * StatsReport of identify_core / detect_clusters / classify_hub_outlier
 * called one at a time, scan.py:488-492). */
int gs_engine_phase_stats(gs_engine* e, gs_stats* stats);

/* One-shot calls (temporary engine on the current device). */
int gs_scan_csr(int64_t n, int64_t m, const int64_t* offsets, const int32_t* adjacency,
                int32_t mu, const gs_eps2* eps2, uint8_t* role_out,
                int32_t* cluster_out, gs_stats* stats);
int gs_scan_edges(int64_t n, int64_t m, const int32_t* edges_uv, int32_t mu,
                  const gs_eps2* eps2, uint8_t* role_out, int32_t* cluster_out,
                  gs_stats* stats);

/* build_graph on the device, reference layout, host in / host out. */
int gs_build_graph(int64_t n, int64_t m, const int32_t* edges_uv, int64_t* offsets,
                   int32_t* adjacency, int32_t* edge_ids, int32_t* edge_list);

/* build_graph's CSR part (vertex_offsets, sorted adjacency) on the device,
 * device in / device out: edges_dev = normalised pairs, off_dev [n+1] i64,
 * adj_dev [2m] i32.  Used to prepare very large inputs for the partitioned
 * scan (the CSR is then copied to pinned host memory). */
int gs_build_csr_device(int64_t n, int64_t m, const int32_t* edges_dev, int64_t* off_dev,
                        int32_t* adj_dev, void* stream);

/* check_sim for k edges (u_i, v_i) of the loaded graph: out[i] = 1 similar,
 * 0 dissimilar, -1 not an edge. */
int gs_engine_check_sim(gs_engine* e, int64_t k, const int32_t* u, const int32_t* v,
                        const gs_eps2* eps2, int8_t* out);

/* Partitioned (out-of-core) scan: the graph stays in HOST memory (the CSR
 * arrays, ideally pinned); only per-vertex state plus one streamed partition
 * of adjacency live in HBM, under hbm_cap_bytes.  Returns GS_EBUDGET if the
 * resident state alone cannot fit. */
int gs_scan_partitioned(int64_t n, int64_t m, const int64_t* offsets,
                        const int32_t* adjacency, int32_t mu, const gs_eps2* eps2,
                        uint64_t hbm_cap_bytes, uint8_t* role_out, int32_t* cluster_out,
                        gs_stats* stats);

/* The partition plan (scan_out_of_core's PartitionPlan, partition.py:231-333):
 * host only, no device needed.  Contiguous ranges of b (vertex ids) whose
 * adjacency slice fits one of the two streaming buffers the cap leaves after
 * the resident state; part_bounds [nparts + 1] receives the range starts and n
 * (when max_parts >= nparts; call with NULL first to size it), stream_elems the
 * buffer size in adjacency elements.  GS_EBUDGET if the state or the largest
 * list cannot fit (InfeasibleBudgetError, partition.py:79-89). */
int gs_plan_partitions(int64_t n, const int64_t* offsets, uint64_t hbm_cap_bytes,
                       int64_t* part_bounds, int64_t max_parts, int64_t* nparts,
                       int64_t* stream_elems);
/* gs_scan_partitioned executing the caller's plan (partition.py:666-757 iterates
 * plan.partitions): part_bounds [nparts + 1] from gs_plan_partitions or any
 * cut whose slices fit the buffers (GS_EBUDGET names the partition that does
 * not).  gs_scan_partitioned = this call with the plan gs_plan_partitions makes. */
int gs_scan_partitioned_plan(int64_t n, int64_t m, const int64_t* offsets,
                             const int32_t* adjacency, int32_t mu, const gs_eps2* eps2,
                             uint64_t hbm_cap_bytes, int64_t nparts, const int64_t* part_bounds,
                             uint8_t* role_out, int32_t* cluster_out, gs_stats* stats);

/* The reference's closure planner (partition_graph, partition.py:231-333), host
 * only, for spill files in its GSCP format (partition.py:336-446): edges in
 * edge_list order, each adding its closure (every edge at either endpoint);
 * a partition is sealed when 25*|E_s| + 4*|V_s| + state_bytes would exceed
 * budget_bytes.  Partition p owns edge ids [owned_bounds[p], owned_bounds[p+1])
 * and its closure has n_local[p] vertices and m_local[p] edges.  Arrays hold
 * `cap` partitions (owned_bounds cap + 1); *nparts is the full count, so a
 * call with *nparts > cap is repeated with a larger cap.  GS_EBUDGET: one
 * edge's closure cannot fit; bad_edge[3] = (u, v, required bytes). */
int gs_plan_closure(int64_t n, int64_t m, const int64_t* offsets, const int32_t* adjacency,
                    const int32_t* edge_ids, const int32_t* edge_list, uint64_t budget_bytes,
                    int64_t state_bytes, int64_t* owned_bounds, int64_t* n_local,
                    int64_t* m_local, int64_t cap, int64_t* nparts, int64_t* bad_edge);

/* Deterministic R-MAT workload generator (bench/test input; same stream as
 * the CPU generator in oracle/): raw samples, device pointers. */
int gs_rmat_generate(int scale, int edgefactor, uint64_t seed, int32_t* src_dev,
                     int32_t* dst_dev, void* stream);
/* Chung-Lu (expected-degree power law, exponent gamma) workload: `count` raw
 * samples over 2^logn vertices, the largest expected degree ~max_degree;
 * device pointers, deterministic in seed. */
int gs_chunglu_generate(int logn, double gamma, double max_degree, int64_t count,
                        uint64_t seed, int32_t* src_dev, int32_t* dst_dev, void* stream);
/* Normalise raw device samples in place (drop loops, orient, sort, dedupe);
 * writes the unique count to *m_out and interleaved pairs to edges_dev. */
int gs_normalize_edges(int64_t count, int32_t* src_dev, int32_t* dst_dev,
                       int32_t* edges_dev, int64_t* m_out, void* stream);

/* Native ingest (parse_edge_list, graph.py:63-118), host memory in and out.
 * gs_parse_edge_text: ASCII edge-list text -> raw (u, v) pairs in input order
 * (self-loops kept), multi-threaded; u_out/v_out hold `cap` pairs (one per
 * line at most).  GS_EPARSE + *err_line for anything outside the native
 * grammar (the caller then applies the reference parser to report or accept).
 * gs_normalize_sparse (device): dense ids = rank of the sorted distinct
 * endpoint ids (ids_out [n], capacity 2*count), self-loops dropped, pairs
 * oriented u < v, sorted, deduplicated (edges_out [2m], capacity 2*count). */
int gs_parse_edge_text(const char* buf, int64_t len, int threads, uint32_t* u_out,
                       uint32_t* v_out, int64_t cap, int64_t* count, int64_t* err_line);
int gs_normalize_sparse(int64_t count, const uint32_t* u, const uint32_t* v, uint32_t* ids_out,
                        int64_t* n_out, int32_t* edges_out, int64_t* m_out);

/* ClusteringResult.to_text (scan.py:892-904), host, multi-threaded: n lines
 * "orig[v]\t{C|M|H|O}\t orig[cluster[v]] or -1\n" into out (capacity cap;
 * 25 bytes per vertex always suffice); *len = bytes written. */
int gs_format_result(int64_t n, const uint8_t* role, const int32_t* cluster,
                     const uint32_t* orig, int threads, char* out, int64_t cap, int64_t* len);

/* Number of visible CUDA devices (0 when there is no usable driver/device). */
int gs_device_count(void);

/* Pay the one-time costs of a process's first scan ahead of it: CUDA context
 * creation on `device` (< 0: current), the stream-ordered memory pool and
 * the lazy loading of the scan kernels (one scan of a 4-vertex graph).  The
 * Python package calls it from a background thread at import (opt out with
 * GS_NO_WARMUP=1), so a cold process's first scan_in_memory does not wait
 * ~1 s for the driver.  Thread-safe; GS_ECUDA without a usable device. */
int gs_warmup(int device);

const char* gs_last_error(void);
int gs_version(void);

#ifdef __cplusplus
}
#endif
#endif
