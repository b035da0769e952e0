// api.cu -- the C-ABI of libgscan.so (include/gscan.h) and the engine
// context.  No C++ exception crosses this boundary; every entry point
// returns a GS_* code and leaves a message in gs_last_error().
#include <cstdio>
#include <cstring>
#include <exception>
#include <new>
#include <string>

#include "engine.cuh"

namespace gs {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
std::string cuda_msg(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
           cudaGetErrorString(e), what, file, line);
  return buf;
}
int build_reference_layout(gs_engine* e, int64_t n, int64_t m, const int32_t* uv_dev,
                           int64_t* off_dev, int32_t* adj_dev, int32_t* eids_dev,
                           int32_t* elist_dev, bool csr_only);
int rmat_generate(int scale, uint64_t seed, int64_t count, int32_t* src, int32_t* dst,
                  cudaStream_t st);
int chunglu_generate(int logn, double gamma, double wmax, int64_t count, uint64_t seed,
                     int32_t* src, int32_t* dst, cudaStream_t st);
int normalize_sparse(gs_engine* e, int64_t count, uint32_t* src, uint32_t* dst, uint32_t* ids,
                     int64_t* n_out, int32_t* uv, int64_t* m_out);
int normalize_edges(gs_engine* e, int64_t count, const int32_t* src, const int32_t* dst,
                    int32_t* uv, int64_t* m_out);
int scan_partitioned(gs_engine* e, int64_t n, int64_t m, const int64_t* off,
                     const int32_t* adj, int32_t mu, const Eps2& eps, uint8_t* role_out,
                     int32_t* cluster_out, gs_stats* st, const int64_t* bounds, int64_t nb);
int plan_partitions(int64_t n, const int64_t* off, uint64_t cap, int64_t* bounds_out,
                    int64_t max_parts, int64_t* nparts, int64_t* stream_elems);
int validate_plan(int64_t n, const int64_t* off, uint64_t cap, const int64_t* bounds,
                  int64_t nb);
int check_sim_batch(gs_engine* e, int64_t k, const int32_t* u, const int32_t* v,
                    const Eps2& eps, int8_t* out);

static Eps2 to_eps(const gs_eps2* p) {
  Eps2 e;
  e.p_lo = p->p_lo;
  e.p_hi = p->p_hi;
  e.q_lo = p->q_lo;
  e.q_hi = p->q_hi;
  const double two64 = 18446744073709551616.0;
  const double pd = (double)p->p_hi * two64 + (double)p->p_lo;
  const double qd = (double)p->q_hi * two64 + (double)p->q_lo;
  e.ratio = pd / qd;
  return e;
}

static int check_eps(const gs_eps2* p) {
  if (!p) { set_error("epsilon is NULL"); return GS_EINVAL; }
  if ((p->q_lo | p->q_hi) == 0) { set_error("epsilon^2 denominator is 0"); return GS_EINVAL; }
  if ((p->p_lo | p->p_hi) == 0) { set_error("epsilon must be in (0, 1]"); return GS_EINVAL; }
  if (p->p_hi > p->q_hi || (p->p_hi == p->q_hi && p->p_lo > p->q_lo)) {
    set_error("epsilon must be in (0, 1]");
    return GS_EINVAL;
  }
  return GS_OK;
}
}  // namespace gs

using namespace gs;

// event-timed phase call (sharded path): adds the device time to e->phase_ms[ph]
template <class F>
static int timed(gs_engine* e, int ph, F&& f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, e->stream);
  int rc = f();
  cudaEventRecord(b, e->stream);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  e->phase_ms[ph] += ms;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return rc;
}


// Engine allocations are cached: a released block goes to a size-keyed free
// list and the next request of a similar size reuses it, so repeated calls
// (the same build + scan sequence every time) never touch the driver
// allocator.  With an HBM cap the cached blocks count against it and are
// trimmed first when a request would exceed it.
int gs_engine::alloc(void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 1;
  bytes = (bytes + 511) & ~size_t(511);
  auto it = cache.lower_bound(bytes);
  if (it != cache.end() && it->first <= bytes + bytes / 4 + (1u << 20)) {
    *p = it->second;
    const size_t sz = it->first;
    cache.erase(it);
    sizes[*p] = sz;
    live += sz;
    if (live > peak) peak = live;
    return GS_OK;
  }
  if (cap && reserved + bytes > cap) trim(bytes);
  if (cap && reserved + bytes > cap) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "device allocation of %zu bytes exceeds the HBM cap (%llu in use of %llu)", bytes,
             (unsigned long long)live, (unsigned long long)cap);
    set_error(buf);
    return GS_EBUDGET;
  }
  cudaError_t err = cudaMallocAsync(p, bytes, stream);
  if (err == cudaErrorMemoryAllocation && !cache.empty()) {
    cudaGetLastError();
    trim(SIZE_MAX);
    err = cudaMallocAsync(p, bytes, stream);
  }
  if (err != cudaSuccess) {
    set_error(cuda_msg(err, "cudaMallocAsync", __FILE__, __LINE__));
    *p = nullptr;
    return err == cudaErrorMemoryAllocation ? GS_ENOMEM : GS_ECUDA;
  }
  sizes[*p] = bytes;
  live += bytes;
  reserved += bytes;
  if (live > peak) peak = live;
  return GS_OK;
}

void gs_engine::kev_mark(int i, cudaStream_t on) {
  if (!kev_on) return;
  if (kev[i] == nullptr && cudaEventCreate(&kev[i]) != cudaSuccess) {
    kev[i] = nullptr;
    return;
  }
  cudaEventRecord(kev[i], on ? on : stream);
}

void gs_engine::kev_class_ms(double* out) {
  // class c runs between events from[c] and to[c] (the sketch filter first)
  // (the tiny class runs on the copy stream, concurrently: events 9 / 10)
  static const int from[kKernelClasses] = {0, 3, 4, 5, 6, 9, 2};
  static const int to[kKernelClasses] = {1, 4, 5, 6, 7, 10, 3};
  for (int c = 0; c < kKernelClasses; ++c) {
    const int a = from[c], b = to[c];
    float t = 0;
    if (g.m > 0 && kev[a] && kev[b] && cudaEventSynchronize(kev[b]) == cudaSuccess &&
        cudaEventElapsedTime(&t, kev[a], kev[b]) != cudaSuccess) {
      cudaGetLastError();  // an event of this class was not recorded in this scan
      t = 0;
    }
    out[c] = t;
  }
}

void gs_engine::release(void* p) {
  if (!p) return;
  auto it = sizes.find(p);
  if (it == sizes.end()) return;
  live -= it->second;
  cache.emplace(it->second, p);
  sizes.erase(it);
}

void gs_engine::trim(size_t need) {
  size_t freed = 0;
  while (!cache.empty() && (need == SIZE_MAX || freed < need || (cap && reserved + need > cap))) {
    auto it = std::prev(cache.end());  // largest first
    cudaFreeAsync(it->second, stream);
    reserved -= it->first;
    freed += it->first;
    cache.erase(it);
  }
  cudaStreamSynchronize(stream);
}

void gs_engine::free_graph() {
  release(g.off);
  if (!g.adj_external) release(g.adj);
  if (pend_bad) { release(pend_bad); pend_bad = nullptr; }
  pend_finish = false;
  release(g.orig);
  release(g.rank);
  release(g.eoff);
  release(g.elo);
  release(g.ehi);
  release(g.sk);
  release(g.skbase);
  g = DevGraph();
}

void gs_engine::free_state() {
  release(s.sim);
  release(s.bounds);
  release(s.role);
  release(s.parent);
  release(s.label);
  release(s.lmin);
  release(s.lmax);
  release(s.ctr);
  release(s.wq);
  release(s.coreadj);
  release(s.clist);
  release(s.lcnt);
  release(s.thr);
  release(s.rdeg);
  release(s.dxs);
  s = DevState();
}

// Every entry point that allocates host memory runs its body through this:
// no C++ exception crosses the C-ABI (std::bad_alloc -> GS_ENOMEM, anything
// else -> GS_EINTERNAL, the message in gs_last_error()).
template <class F>
static int guarded(F&& body) {
  try {
    return body();
  } catch (const std::bad_alloc&) {
    set_error("host memory exhausted");
    return GS_ENOMEM;
  } catch (const std::exception& x) {
    set_error(std::string("internal error: ") + x.what());
    return GS_EINTERNAL;
  } catch (...) {
    set_error("internal error (unknown exception)");
    return GS_EINTERNAL;
  }
}

extern "C" {

int gs_version(void) { return GS_ABI_VERSION; }

int gs_warmup(int device) {
  return guarded([&]() -> int {
    gs_engine* e = nullptr;
    GS_TRY(gs_engine_create(device, 0, &e));
    // triangle 0-1-2 plus the pendant edge 2-3 (reference CSR), eps 0.5, mu 2
    static const int64_t off[5] = {0, 2, 4, 7, 8};
    static const int32_t adj[8] = {1, 2, 0, 2, 0, 1, 3, 2};
    uint8_t role[4];
    int32_t cl[4];
    gs_eps2 eps{1, 0, 4, 0};
    int rc = gs_engine_load_csr(e, 4, 4, off, adj, 0);
    if (rc == GS_OK) rc = gs_engine_scan(e, 2, &eps, role, cl, 0, nullptr);
    gs_engine_destroy(e);
    return rc;
  });
}
int gs_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n;
}
const char* gs_last_error(void) { return g_err.c_str(); }

int gs_engine_create(int device, uint64_t hbm_cap_bytes, gs_engine** out) {
  return guarded([&]() -> int {
    if (!out) { set_error("out is NULL"); return GS_EINVAL; }
    *out = nullptr;
    int dev = device;
    if (dev < 0) GS_CUDA(cudaGetDevice(&dev));
    GS_CUDA(cudaSetDevice(dev));
    gs_engine* e = new gs_engine();
    e->device = dev;
    e->cap = hbm_cap_bytes;
    cudaError_t err = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking);
    if (err != cudaSuccess) {
      delete e;
      set_error(cuda_msg(err, "cudaStreamCreate", __FILE__, __LINE__));
      return GS_ECUDA;
    }
    err = cudaStreamCreateWithFlags(&e->cstream, cudaStreamNonBlocking);
    if (err != cudaSuccess) {
      cudaStreamDestroy(e->stream);
      delete e;
      set_error(cuda_msg(err, "cudaStreamCreate", __FILE__, __LINE__));
      return GS_ECUDA;
    }
    cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&e->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;  // keep freed blocks for the next call
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = e;
    return GS_OK;
  });
}

void gs_engine_destroy(gs_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  e->free_state();
  e->free_graph();
  for (auto& kv : e->sizes) cudaFreeAsync(kv.first, e->stream);
  for (auto& kv : e->cache) cudaFreeAsync(kv.second, e->stream);
  cudaStreamSynchronize(e->stream);
  cudaStreamSynchronize(e->cstream);
  if (e->hstage) cudaFreeHost(e->hstage);
  for (auto& x : e->kev)
    if (x) cudaEventDestroy(x);
  cudaStreamDestroy(e->cstream);
  cudaStreamDestroy(e->stream);
  // hand the pool's reserved memory back (the release threshold keeps it
  // across calls of a live engine, not beyond its lifetime)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, e->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  delete e;
}

void* gs_engine_stream(gs_engine* e) { return e ? (void*)e->stream : nullptr; }

static int load_common(gs_engine* e, int64_t n, int64_t m) {
  if (!e) { set_error("engine is NULL"); return GS_EINVAL; }
  if (n < 0 || m < 0) { set_error("negative n or m"); return GS_EINVAL; }
  if (n > 0x7fffffffLL) { set_error("vertex count exceeds the 4-byte id range"); return GS_EINVAL; }
  GS_CUDA(cudaSetDevice(e->device));
  e->launches = 0;
  return GS_OK;
}

int gs_engine_load_csr(gs_engine* e, int64_t n, int64_t m, const int64_t* offsets,
                       const int32_t* adjacency, int on_device) {
  return guarded([&]() -> int {
    GS_TRY(load_common(e, n, m));
    int64_t h_ends[2] = {0, 0};
    if (on_device) {
      GS_CUDA(cudaMemcpyAsync(&h_ends[0], offsets, sizeof(int64_t), cudaMemcpyDeviceToHost, e->stream));
      GS_CUDA(cudaMemcpyAsync(&h_ends[1], offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                              e->stream));
      GS_CUDA(cudaStreamSynchronize(e->stream));
    } else {
      h_ends[0] = offsets[0];
      h_ends[1] = offsets[n];
    }
    if (h_ends[0] != 0 || h_ends[1] != 2 * m) {
      set_error("invalid graph: vertex_offsets must start at 0 and end at 2m");
      return GS_EINVAL;
    }
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0); cudaEventCreate(&t1);
    cudaEventRecord(t0, e->stream);
    // host input: the adjacency is streamed chunk by chunk and scattered into
    // its rank-space runs as it lands (the copy overlaps the relabel)
    int rc = on_device ? build_from_csr(e, n, m, offsets, adjacency)
                       : build_from_csr_host(e, n, m, offsets, adjacency);
    cudaEventRecord(t1, e->stream);
    cudaStreamSynchronize(e->stream);
    e->last_h2d_ms = 0;  // inside the build (overlapped)
    cudaEventElapsedTime(&e->last_build_ms, t0, t1);
    cudaEventDestroy(t0); cudaEventDestroy(t1);
    return rc;
  });
}

int gs_engine_load_csr_part(gs_engine* e, int64_t n, int64_t m, const int64_t* offsets,
                            const int32_t* adjacency, int on_device, int part_rank,
                            int part_world, int32_t* adj_out, int64_t* slot_bounds) {
  return guarded([&]() -> int {
    GS_TRY(load_common(e, n, m));
    if (part_world < 1 || part_rank < 0 || part_rank >= part_world) {
      set_error("invalid part");
      return GS_EINVAL;
    }
    if (part_world > 1 && !adj_out) {
      set_error("a partitioned build needs the caller's adjacency buffer (2m int32)");
      return GS_EINVAL;
    }
    int64_t h_ends[2] = {0, 0};
    if (on_device) {
      GS_CUDA(cudaMemcpyAsync(&h_ends[0], offsets, sizeof(int64_t), cudaMemcpyDeviceToHost, e->stream));
      GS_CUDA(cudaMemcpyAsync(&h_ends[1], offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                              e->stream));
      GS_CUDA(cudaStreamSynchronize(e->stream));
    } else {
      h_ends[0] = offsets[0];
      h_ends[1] = offsets[n];
    }
    if (h_ends[0] != 0 || h_ends[1] != 2 * m) {
      set_error("invalid graph: vertex_offsets must start at 0 and end at 2m");
      return GS_EINVAL;
    }
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0); cudaEventCreate(&t1);
    cudaEventRecord(t0, e->stream);
    int rc = on_device ? build_from_csr(e, n, m, offsets, adjacency, part_rank, part_world, adj_out,
                                        slot_bounds)
                       : build_from_csr_host(e, n, m, offsets, adjacency, part_rank, part_world,
                                             adj_out, slot_bounds);
    cudaEventRecord(t1, e->stream);
    cudaStreamSynchronize(e->stream);
    e->last_h2d_ms = 0;
    cudaEventElapsedTime(&e->last_build_ms, t0, t1);
    cudaEventDestroy(t0); cudaEventDestroy(t1);
    return rc;
  });
}

int gs_engine_load_finish(gs_engine* e) {
  return guarded([&]() -> int {
    if (!e) { set_error("engine is NULL"); return GS_EINVAL; }
    GS_CUDA(cudaSetDevice(e->device));
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0); cudaEventCreate(&t1);
    cudaEventRecord(t0, e->stream);
    int rc = finish_build(e);
    cudaEventRecord(t1, e->stream);
    cudaStreamSynchronize(e->stream);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    e->last_build_ms += ms;
    cudaEventDestroy(t0); cudaEventDestroy(t1);
    return rc;
  });
}

int gs_engine_load_edges(gs_engine* e, int64_t n, int64_t m, const int32_t* edges_uv,
                         int on_device) {
  return guarded([&]() -> int {
    GS_TRY(load_common(e, n, m));
    cudaEvent_t t0, t1, t2;
    cudaEventCreate(&t0); cudaEventCreate(&t1); cudaEventCreate(&t2);
    cudaEventRecord(t0, e->stream);
    const int32_t* uv = edges_uv;
    int32_t* d_uv = nullptr;
    if (!on_device && m > 0) {
      GS_TRY(e->alloc_n(&d_uv, 2 * m));
      GS_CUDA(cudaMemcpyAsync(d_uv, edges_uv, sizeof(int32_t) * (size_t)(2 * m),
                              cudaMemcpyHostToDevice, e->stream));
      uv = d_uv;
    }
    cudaEventRecord(t1, e->stream);
    int rc = build_from_edges(e, n, m, uv);
    cudaEventRecord(t2, e->stream);
    cudaStreamSynchronize(e->stream);
    e->release(d_uv);
    cudaEventElapsedTime(&e->last_h2d_ms, t0, t1);
    cudaEventElapsedTime(&e->last_build_ms, t1, t2);
    cudaEventDestroy(t0); cudaEventDestroy(t1); cudaEventDestroy(t2);
    return rc;
  });
}

int gs_engine_scan(gs_engine* e, int32_t mu, const gs_eps2* eps2, uint8_t* role_out,
                   int32_t* cluster_out, int out_on_device, gs_stats* stats) {
  return guarded([&]() -> int {
    if (!e) { set_error("engine is NULL"); return GS_EINVAL; }
    if (mu < 2) { set_error("mu must be >= 2"); return GS_EINVAL; }
    GS_TRY(check_eps(eps2));
    GS_CUDA(cudaSetDevice(e->device));
    if (stats) memset(stats, 0, sizeof(*stats));
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0); cudaEventCreate(&t1);
    cudaEventRecord(t0, e->stream);
    int rc = run_scan(e, mu, to_eps(eps2), role_out, cluster_out, out_on_device, stats);
    cudaEventRecord(t1, e->stream);
    cudaStreamSynchronize(e->stream);
    if (stats) {
      float ms = 0;
      cudaEventElapsedTime(&ms, t0, t1);
      stats->phase_ms[GS_PH_TOTAL] = ms;
      stats->phase_ms[GS_PH_H2D] = e->last_h2d_ms;
      stats->phase_ms[GS_PH_BUILD] = e->last_build_ms;
      stats->kernel_launches = e->launches;  // since the last load: build + scan
      stats->peak_device_bytes = (int64_t)e->peak;
    }
    cudaEventDestroy(t0); cudaEventDestroy(t1);
    return rc;
  });
}

// ---- sharded (multi-GPU) scan: phases with the collectives in between
static int phase_guard(gs_engine* e) {
  if (!e) { set_error("engine is NULL"); return GS_EINVAL; }
  if (!e->g.off && e->g.n > 0) { set_error("no graph loaded"); return GS_EINVAL; }
  GS_CUDA(cudaSetDevice(e->device));
  return GS_OK;
}

int gs_engine_set_shard(gs_engine* e, int rank, int world) {
  if (!e || world < 1 || rank < 0 || rank >= world) { set_error("invalid shard"); return GS_EINVAL; }
  e->shard_rank = rank;
  e->shard_world = world;
  return GS_OK;
}

int gs_engine_phase_begin(gs_engine* e, int32_t mu, const gs_eps2* eps2) {
  return guarded([&]() -> int {
    GS_TRY(phase_guard(e));
    if (mu < 2) { set_error("mu must be >= 2"); return GS_EINVAL; }
    GS_TRY(check_eps(eps2));
    e->launches = 0;
    for (auto& x : e->phase_ms) x = 0;
    e->kev_on = true;  // per-class identify timing, read at gs_engine_phase_finish
    return timed(e, GS_PH_IDENTIFY, [&] { return phase_begin(e, mu, to_eps(eps2)); });
  });
}

int gs_engine_phase_identify(gs_engine* e, int32_t* counts_dev) {
  return guarded([&]() -> int {
    GS_TRY(phase_guard(e));
    GS_TRY(timed(e, GS_PH_IDENTIFY, [&] { return phase_identify(e); }));
    if (counts_dev) GS_TRY(phase_export_counts(e, counts_dev));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    return GS_OK;
  });
}

int gs_engine_phase_resolve(gs_engine* e, const int32_t* counts_dev, int64_t* ncores) {
  return guarded([&]() -> int {
    GS_TRY(phase_guard(e));
    if (counts_dev) GS_TRY(phase_import_counts(e, counts_dev));
    GS_TRY(timed(e, GS_PH_CLEANUP, [&] {
      return phase_resolve(e, counts_dev == nullptr && e->shard_world == 1);
    }));
    if (ncores) *ncores = (int64_t)e->ncores;
    return GS_OK;
  });
}

int gs_engine_phase_union(gs_engine* e, int32_t* pairs_dev, int64_t* npairs) {
  return guarded([&]() -> int {
    GS_TRY(phase_guard(e));
    GS_TRY(timed(e, GS_PH_CLUSTER, [&] { return phase_union(e); }));
    int64_t np = 0;
    if (pairs_dev) GS_TRY(phase_export_pairs(e, pairs_dev, &np));
    if (npairs) *npairs = np;
    GS_CUDA(cudaStreamSynchronize(e->stream));
    return GS_OK;
  });
}

int gs_engine_phase_merge(gs_engine* e, const int32_t* pairs_dev, int64_t npairs) {
  return guarded([&]() -> int {
    GS_TRY(phase_guard(e));
    GS_TRY(timed(e, GS_PH_CLUSTER, [&] {
      int rc = pairs_dev ? phase_merge_pairs(e, pairs_dev, npairs) : GS_OK;
      return rc == GS_OK ? phase_labels(e) : rc;
    }));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    return GS_OK;
  });
}

int gs_engine_phase_attach(gs_engine* e, int32_t* labels_dev) {
  return guarded([&]() -> int {
    GS_TRY(phase_guard(e));
    GS_TRY(timed(e, GS_PH_CLUSTER, [&] { return phase_attach(e); }));
    if (labels_dev) GS_TRY(phase_export_labels(e, labels_dev));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    return GS_OK;
  });
}

int gs_engine_phase_finish(gs_engine* e, const int32_t* labels_dev, uint8_t* role_out,
                           int32_t* cluster_out, int out_on_device, gs_stats* stats) {
  return guarded([&]() -> int {
    struct KevOff {  // class timing ends with the scan, whichever way this returns
      gs_engine* e;
      ~KevOff() { if (e) e->kev_on = false; }
    } kev_off{e};
    GS_TRY(phase_guard(e));
    if (stats) memset(stats, 0, sizeof(*stats));
    if (labels_dev) GS_TRY(phase_import_labels(e, labels_dev));
    GS_TRY(timed(e, GS_PH_CLASSIFY, [&] {
      return phase_finish(e, role_out, cluster_out, out_on_device, stats);
    }));
    if (stats) {
      stats->kernel_launches = e->launches;
      stats->peak_device_bytes = (int64_t)e->peak;
      const double d2h = stats->phase_ms[GS_PH_D2H];
      for (int i = 0; i < GS_PH_COUNT; ++i) stats->phase_ms[i] = e->phase_ms[i];
      stats->phase_ms[GS_PH_D2H] = d2h;
      if (e->kev_on) e->kev_class_ms(stats->phase_ms + GS_PH_K_PREP);
      stats->phase_ms[GS_PH_CLASSIFY] -= d2h;
      stats->phase_ms[GS_PH_H2D] = e->last_h2d_ms;
      stats->phase_ms[GS_PH_BUILD] = e->last_build_ms;
      stats->phase_ms[GS_PH_TOTAL] = e->phase_ms[GS_PH_IDENTIFY] + e->phase_ms[GS_PH_CLEANUP] +
                                     e->phase_ms[GS_PH_CLUSTER] + e->phase_ms[GS_PH_CLASSIFY];
    }
    return GS_OK;
  });
}

int gs_scan_csr(int64_t n, int64_t m, const int64_t* offsets, const int32_t* adjacency,
                int32_t mu, const gs_eps2* eps2, uint8_t* role_out, int32_t* cluster_out,
                gs_stats* stats) {
  return guarded([&]() -> int {
    if (mu < 2) { set_error("mu must be >= 2"); return GS_EINVAL; }
    GS_TRY(check_eps(eps2));
    gs_engine* e = nullptr;
    GS_TRY(gs_engine_create(-1, 0, &e));
    int rc = gs_engine_load_csr(e, n, m, offsets, adjacency, 0);
    int64_t build_launches = e->launches;
    if (rc == GS_OK) rc = gs_engine_scan(e, mu, eps2, role_out, cluster_out, 0, stats);
    if (rc == GS_OK && stats) {
      stats->kernel_launches += build_launches;
      stats->phase_ms[GS_PH_TOTAL] += stats->phase_ms[GS_PH_H2D] + stats->phase_ms[GS_PH_BUILD];
    }
    gs_engine_destroy(e);
    return rc;
  });
}

int gs_scan_edges(int64_t n, int64_t m, const int32_t* edges_uv, int32_t mu,
                  const gs_eps2* eps2, uint8_t* role_out, int32_t* cluster_out,
                  gs_stats* stats) {
  return guarded([&]() -> int {
    if (mu < 2) { set_error("mu must be >= 2"); return GS_EINVAL; }
    GS_TRY(check_eps(eps2));
    gs_engine* e = nullptr;
    GS_TRY(gs_engine_create(-1, 0, &e));
    int rc = gs_engine_load_edges(e, n, m, edges_uv, 0);
    int64_t build_launches = e->launches;
    if (rc == GS_OK) rc = gs_engine_scan(e, mu, eps2, role_out, cluster_out, 0, stats);
    if (rc == GS_OK && stats) {
      stats->kernel_launches += build_launches;
      stats->phase_ms[GS_PH_TOTAL] += stats->phase_ms[GS_PH_H2D] + stats->phase_ms[GS_PH_BUILD];
    }
    gs_engine_destroy(e);
    return rc;
  });
}

int gs_build_graph(int64_t n, int64_t m, const int32_t* edges_uv, int64_t* offsets,
                   int32_t* adjacency, int32_t* edge_ids, int32_t* edge_list) {
  return guarded([&]() -> int {
    gs_engine* e = nullptr;
    GS_TRY(gs_engine_create(-1, 0, &e));
    int rc = load_common(e, n, m);
    int32_t *d_uv = nullptr, *d_adj = nullptr, *d_eids = nullptr, *d_el = nullptr;
    int64_t* d_off = nullptr;
    if (rc == GS_OK) rc = e->alloc_n(&d_uv, 2 * m);
    if (rc == GS_OK) rc = e->alloc_n(&d_off, n + 1);
    if (rc == GS_OK) rc = e->alloc_n(&d_adj, 2 * m);
    if (rc == GS_OK) rc = e->alloc_n(&d_eids, 2 * m);
    if (rc == GS_OK) rc = e->alloc_n(&d_el, 2 * m);
    if (rc == GS_OK && m > 0 &&
        cudaMemcpyAsync(d_uv, edges_uv, 8 * (size_t)m, cudaMemcpyHostToDevice, e->stream) !=
            cudaSuccess) {
      set_error("host to device copy failed");
      rc = GS_ECUDA;
    }
    if (rc == GS_OK) rc = build_reference_layout(e, n, m, d_uv, d_off, d_adj, d_eids, d_el, false);
    if (rc == GS_OK) {
      cudaMemcpyAsync(offsets, d_off, 8 * (size_t)(n + 1), cudaMemcpyDeviceToHost, e->stream);
      if (m > 0) {
        cudaMemcpyAsync(adjacency, d_adj, 8 * (size_t)m, cudaMemcpyDeviceToHost, e->stream);
        cudaMemcpyAsync(edge_ids, d_eids, 8 * (size_t)m, cudaMemcpyDeviceToHost, e->stream);
        cudaMemcpyAsync(edge_list, d_el, 8 * (size_t)m, cudaMemcpyDeviceToHost, e->stream);
      }
      cudaError_t err = cudaStreamSynchronize(e->stream);
      if (err != cudaSuccess) {
        set_error(cuda_msg(err, "gs_build_graph copy-back", __FILE__, __LINE__));
        rc = GS_ECUDA;
      }
    }
    gs_engine_destroy(e);
    return rc;
  });
}

int gs_build_csr_device(int64_t n, int64_t m, const int32_t* edges_dev, int64_t* off_dev,
                        int32_t* adj_dev, void* stream) {
  return guarded([&]() -> int {
    gs_engine* e = nullptr;
    GS_TRY(gs_engine_create(-1, 0, &e));
    if (stream) cudaStreamSynchronize((cudaStream_t)stream);
    int rc = load_common(e, n, m);
    if (rc == GS_OK)
      rc = build_reference_layout(e, n, m, edges_dev, off_dev, adj_dev, nullptr, nullptr, true);
    gs_engine_destroy(e);
    return rc;
  });
}

int gs_engine_phase_stats(gs_engine* e, gs_stats* stats) {
  return guarded([&]() -> int {
    GS_TRY(phase_guard(e));
    if (!stats) return GS_OK;
    memset(stats, 0, sizeof(*stats));
    GS_TRY(read_counters(e, stats));
    stats->kernel_launches = e->launches;
    stats->peak_device_bytes = (int64_t)e->peak;
    for (int i = 0; i < GS_PH_COUNT; ++i) stats->phase_ms[i] = e->phase_ms[i];
    stats->phase_ms[GS_PH_H2D] = e->last_h2d_ms;
    stats->phase_ms[GS_PH_BUILD] = e->last_build_ms;
    return GS_OK;
  });
}

int gs_engine_export_state(gs_engine* e, int stage, int32_t* lower, int32_t* upper,
                           uint8_t* role, int32_t* parent, uint8_t* sim, int32_t* edge_pairs) {
  return guarded([&]() -> int {
    GS_TRY(phase_guard(e));
    if (stage < 0 || stage > 2) { set_error("stage must be 0, 1 or 2"); return GS_EINVAL; }
    return export_state(e, stage, lower, upper, role, parent, sim, edge_pairs);
  });
}

int gs_engine_check_sim(gs_engine* e, int64_t k, const int32_t* u, const int32_t* v,
                        const gs_eps2* eps2, int8_t* out) {
  return guarded([&]() -> int {
    if (!e) { set_error("engine is NULL"); return GS_EINVAL; }
    GS_TRY(check_eps(eps2));
    GS_CUDA(cudaSetDevice(e->device));
    return check_sim_batch(e, k, u, v, to_eps(eps2), out);
  });
}

int gs_scan_partitioned_plan(int64_t n, int64_t m, const int64_t* offsets,
                             const int32_t* adjacency, int32_t mu, const gs_eps2* eps2,
                             uint64_t hbm_cap_bytes, int64_t nparts, const int64_t* part_bounds,
                             uint8_t* role_out, int32_t* cluster_out, gs_stats* stats) {
  if (mu < 2) { set_error("mu must be >= 2"); return GS_EINVAL; }
  GS_TRY(check_eps(eps2));
  if (part_bounds && nparts < 1) { set_error("a plan needs at least one partition"); return GS_EINVAL; }
  if (n < 0 || m < 0 || (n > 0 && (!offsets || offsets[n] != 2 * m))) {
    set_error("invalid graph: vertex_offsets must end at 2m");
    return GS_EINVAL;
  }
  if (n > 0 && part_bounds) {  // a plan that cannot run fails before any device work
    try {
      GS_TRY(validate_plan(n, offsets, hbm_cap_bytes, part_bounds, nparts));
    } catch (const std::bad_alloc&) {
      set_error("host memory exhausted while validating the plan");
      return GS_ENOMEM;
    }
  }
  gs_engine* e = nullptr;
  GS_TRY(gs_engine_create(-1, hbm_cap_bytes, &e));
  int rc = load_common(e, n, m);
  if (stats) memset(stats, 0, sizeof(*stats));
  if (rc == GS_OK) {
    try {
      rc = scan_partitioned(e, n, m, offsets, adjacency, mu, to_eps(eps2), role_out, cluster_out,
                            stats, part_bounds, part_bounds ? nparts : 0);
    } catch (const std::bad_alloc&) {
      set_error("host memory exhausted in the partitioned scan");
      rc = GS_ENOMEM;
    }
  }
  if (stats) stats->peak_device_bytes = (int64_t)e->peak;
  gs_engine_destroy(e);
  return rc;
}

int gs_scan_partitioned(int64_t n, int64_t m, const int64_t* offsets, const int32_t* adjacency,
                        int32_t mu, const gs_eps2* eps2, uint64_t hbm_cap_bytes,
                        uint8_t* role_out, int32_t* cluster_out, gs_stats* stats) {
  return gs_scan_partitioned_plan(n, m, offsets, adjacency, mu, eps2, hbm_cap_bytes, 0, nullptr,
                                  role_out, cluster_out, stats);
}

int gs_plan_partitions(int64_t n, const int64_t* offsets, uint64_t hbm_cap_bytes,
                       int64_t* part_bounds, int64_t max_parts, int64_t* nparts,
                       int64_t* stream_elems) {
  if (n < 0 || (n > 0 && !offsets)) { set_error("invalid graph"); return GS_EINVAL; }
  try {
    return plan_partitions(n, offsets, hbm_cap_bytes, part_bounds, max_parts, nparts,
                           stream_elems);
  } catch (const std::bad_alloc&) {
    set_error("host memory exhausted while planning");
    return GS_ENOMEM;
  }
}

int gs_rmat_generate(int scale, int edgefactor, uint64_t seed, int32_t* src_dev,
                     int32_t* dst_dev, void* stream) {
  return guarded([&]() -> int {
    if (scale < 1 || scale > 31 || edgefactor < 1) {
      set_error("invalid R-MAT scale / edgefactor");
      return GS_EINVAL;
    }
    return rmat_generate(scale, seed, (int64_t)edgefactor << scale, src_dev, dst_dev,
                         (cudaStream_t)stream);
  });
}

int gs_chunglu_generate(int logn, double gamma, double max_degree, int64_t count,
                        uint64_t seed, int32_t* src_dev, int32_t* dst_dev, void* stream) {
  return guarded([&]() -> int {
    if (logn < 1 || logn > 31 || gamma <= 1.5 || max_degree <= 1 || count < 0) {
      set_error("invalid Chung-Lu parameters");
      return GS_EINVAL;
    }
    return chunglu_generate(logn, gamma, max_degree, count, seed, src_dev, dst_dev,
                            (cudaStream_t)stream);
  });
}

int gs_normalize_edges(int64_t count, int32_t* src_dev, int32_t* dst_dev, int32_t* edges_dev,
                       int64_t* m_out, void* stream) {
  return guarded([&]() -> int {
    gs_engine* e = nullptr;
    GS_TRY(gs_engine_create(-1, 0, &e));
    if (stream) GS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    int rc = normalize_edges(e, count, src_dev, dst_dev, edges_dev, m_out);
    gs_engine_destroy(e);
    return rc;
  });
}

int gs_normalize_sparse(int64_t count, const uint32_t* u, const uint32_t* v, uint32_t* ids_out,
                        int64_t* n_out, int32_t* edges_out, int64_t* m_out) {
  return guarded([&]() -> int {
    if (count < 0 || !n_out || !m_out) { set_error("invalid arguments"); return GS_EINVAL; }
    *n_out = 0;
    *m_out = 0;
    if (count == 0) return GS_OK;
    gs_engine* e = nullptr;
    GS_TRY(gs_engine_create(-1, 0, &e));
    struct Guard { gs_engine* e; ~Guard() { gs_engine_destroy(e); } } guard{e};
    uint32_t *du = nullptr, *dv = nullptr, *dids = nullptr;
    int32_t* duv = nullptr;
    GS_TRY(e->alloc_n(&du, count));
    GS_TRY(e->alloc_n(&dv, count));
    GS_TRY(e->alloc_n(&dids, 2 * count));
    GS_TRY(e->alloc_n(&duv, 2 * count));
    GS_CUDA(cudaMemcpyAsync(du, u, 4 * (size_t)count, cudaMemcpyHostToDevice, e->stream));
    GS_CUDA(cudaMemcpyAsync(dv, v, 4 * (size_t)count, cudaMemcpyHostToDevice, e->stream));
    GS_TRY(normalize_sparse(e, count, du, dv, dids, n_out, duv, m_out));
    if (*n_out > 0)
      GS_CUDA(cudaMemcpyAsync(ids_out, dids, 4 * (size_t)*n_out, cudaMemcpyDeviceToHost, e->stream));
    if (*m_out > 0)
      GS_CUDA(cudaMemcpyAsync(edges_out, duv, 8 * (size_t)*m_out, cudaMemcpyDeviceToHost, e->stream));
    GS_CUDA(cudaStreamSynchronize(e->stream));
    return GS_OK;
  });
}

}  // extern "C"
