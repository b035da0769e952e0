// ooc.cu -- check_sim batches (scan.py:241-258) and the partitioned
// (out-of-core) scan (partition.py:666-757).
#include "engine.cuh"

namespace gs {

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

int scan_partitioned(gs_engine* e, int64_t n, int64_t m, const int64_t* off,
                     const int32_t* adj, int32_t mu, const Eps2& eps, uint8_t* role_out,
                     int32_t* cluster_out, gs_stats* st) {
  (void)e; (void)n; (void)m; (void)off; (void)adj; (void)mu; (void)eps;
  (void)role_out; (void)cluster_out; (void)st;
  set_error("partitioned scan: not built yet");
  return GS_EINTERNAL;
}

}  // namespace gs
