// sketch.cu -- neighbourhood sketches: an exact upper bound on |N(a) ∩ N(b)|
// that decides most surviving edges "dissimilar" without walking N(a).
//
// Vertex v of degree d keeps a bitmap S_v of M(d) bits, M(d) = the smallest
// power of two >= k*d (k = 2^lk bits per neighbour), bit h(w) mod M(d) set
// for every neighbour w (h = a 32-bit mixer).  For an edge (a, b), d_a <= d_b
// so M(d_a) <= M(d_b), and S_b folded to M(d_a) bits (OR of the M(d_b)/M(d_a)
// slices; h mod M(d_a) = (h mod M(d_b)) mod M(d_a)) is the bitmap of N(b) at
// a's resolution.  Every common neighbour sets a bit in both maps, and the
// neighbours of a that share a bit of S_a with another neighbour of a number
// d_a - |S_a|, so
//
//     c = |N(a) ∩ N(b)|  <=  |S_a & fold(S_b)| + (d_a - |S_a|)  =: U.
//
// U < c_min proves sigma(a, b) < eps with the same exact integer c_min the
// scan uses (sim.cu), so the decision is exact; U >= c_min decides nothing
// and the edge is scanned as before.  The bound pays off when the edge is
// far from the threshold -- on R-MAT graphs almost every surviving edge has
// few common neighbours (the s24 eps 0.5 sweep ends with no core)
// -- and it reads k*d_a/8 bytes of a's sketch in one coalesced burst instead
// of a dependent chain of adjacency steps.  The similar side is never decided
// by the sketch (no lower bound), so results are unchanged bit for bit.
//
// Layout: every row carries its folds ("levels"): S_v (w words), S_v folded to
// w/2, w/4, ... 4 words, back to back in a 2w-word slot -- level L (w >> L
// words) at word 2 (w - (w >> L)).  So S_b at a's resolution (w_a words) is a
// plain read of w_a words at 2 (w_b - w_a), by any kernel, without folding.
#include <algorithm>

#include <cub/cub.cuh>

#include "simcore.cuh"

namespace gs {

// per degree: words of all sketches of that degree (0 below dmin)
__global__ void k_sk_sizes(int64_t dmax, int64_t dmin, int lk, const int32_t* __restrict__ rdeg,
                           int64_t* __restrict__ sizes) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d <= dmax + 1;
       d += (int64_t)gridDim.x * blockDim.x)
    sizes[d] = (d >= dmin && d <= dmax) ? (int64_t)(rdeg[d + 1] - rdeg[d]) * 2 * sk_words(d, lk) : 0;
}

// hash a run's neighbours into the bitmap t (threads i0, i0 + step, ...): with
// UNR 4, four loads in flight per thread before their atomics
template <int UNR>
__device__ __forceinline__ void sk_hash_run(const int32_t* __restrict__ a, int64_t d, int i0,
                                            int step, uint32_t mask, uint32_t* t) {
  int64_t i = i0;
  if (UNR > 1) {
    for (; i + (UNR - 1) * step < d; i += UNR * step) {
      uint32_t x[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) x[u] = (uint32_t)__ldg(a + i + u * step);
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint32_t h = sk_hash(x[u]) & mask;
        atomicOr(&t[h >> 5], 1u << (h & 31));
      }
    }
  }
  for (; i < d; i += step) {
    const uint32_t h = sk_hash((uint32_t)__ldg(a + i)) & mask;
    atomicOr(&t[h >> 5], 1u << (h & 31));
  }
}

// warp per vertex, sketch of <= WMAX words built in shared memory
template <int NT, int WMAX, int UNR = 1>
__global__ void __launch_bounds__(NT) k_sk_warp(const int64_t* __restrict__ off,
                                                const int32_t* __restrict__ adj, int64_t r0,
                                                int64_t r1, const int32_t* __restrict__ rdeg,
                                                const int64_t* __restrict__ skbase, int lk,
                                                uint32_t* __restrict__ sk) {
  __shared__ uint32_t sm[NT / 32][2 * WMAX];
  const int lane = threadIdx.x & 31;
  uint32_t* s = sm[threadIdx.x >> 5];
  const int64_t nw = ((int64_t)gridDim.x * NT) >> 5;
  // two neighbouring ranks per round (similar degrees): rows of <= WMAX/2
  // words are built by the two half-warps side by side, longer ones in turn
  for (int64_t v0 = r0 + 2 * ((blockIdx.x * (int64_t)NT + threadIdx.x) >> 5); v0 < r1;
       v0 += 2 * nw) {
    const bool two = v0 + 1 < r1;
    const int64_t dlast = two ? off[v0 + 2] - off[v0 + 1] : off[v0 + 1] - off[v0];
    if (two && sk_words(dlast, lk) <= WMAX / 2) {  // degrees ascend: both rows fit
      const int hf = lane >> 4, hl = lane & 15;
      const int64_t v = v0 + hf;
      const int64_t o = off[v], d = off[v + 1] - o;
      const int64_t W = sk_words(d, lk);
      const uint32_t mask = (uint32_t)(W * 32 - 1);
      uint32_t* t = s + hf * WMAX;
      for (int64_t j = hl; j < W; j += 16) t[j] = 0u;
      __syncwarp();
      sk_hash_run<UNR>(adj + o, d, hl, 16, mask, t);
      __syncwarp();
      sk_fold_levels(t, W, hl, 16);
      uint32_t* out = sk + skbase[d] + (v - rdeg[d]) * 2 * W;
      for (int64_t j = hl; j < 2 * W - 4; j += 16) out[j] = t[j];
      __syncwarp();
      continue;
    }
    for (int64_t v = v0; v < v0 + 2 && v < r1; ++v) {
      const int64_t o = off[v], d = off[v + 1] - o;
      const int64_t W = sk_words(d, lk);
      const uint32_t mask = (uint32_t)(W * 32 - 1);
      for (int64_t j = lane; j < W; j += 32) s[j] = 0u;
      __syncwarp();
      sk_hash_run<UNR>(adj + o, d, lane, 32, mask, s);
      __syncwarp();
      sk_fold_levels(s, W, lane, 32);
      uint32_t* out = sk + skbase[d] + (v - rdeg[d]) * 2 * W;
      for (int64_t j = lane; j < 2 * W - 4; j += 32) out[j] = s[j];
      __syncwarp();
    }
  }
}

// the row of vertex v by a CTA: shared memory up to smem_words, global atomics beyond
__device__ __forceinline__ void sk_cta_row(const int64_t* __restrict__ off,
                                           const int32_t* __restrict__ adj, int64_t v,
                                           const int32_t* __restrict__ rdeg,
                                           const int64_t* __restrict__ skbase, int lk,
                                           uint32_t* __restrict__ sk, uint32_t* s,
                                           int64_t smem_words) {
  const int64_t o = off[v], d = off[v + 1] - o;
  const int64_t W = sk_words(d, lk);
  const uint32_t mask = (uint32_t)(W * 32 - 1);
  uint32_t* out = sk + skbase[d] + (v - rdeg[d]) * 2 * W;
  const bool in_smem = W <= smem_words;
  uint32_t* t = in_smem ? s : out;
  for (int64_t j = threadIdx.x; j < W; j += blockDim.x) t[j] = 0u;
  __syncthreads();
  sk_hash_run<4>(adj + o, d, threadIdx.x, blockDim.x, mask, t);
  __syncthreads();
  if (in_smem) {
    sk_fold_levels(s, W, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    for (int64_t j = threadIdx.x; j < 2 * W - 4; j += blockDim.x) out[j] = s[j];
  } else {  // level 0 was built with global atomics (at L2): fold through L2
    for (int64_t lo = 0, w = W; w > 4; lo += w, w >>= 1) {
      const int64_t h = w >> 1;
      for (int64_t i = threadIdx.x; i < h; i += blockDim.x)
        out[lo + w + i] = __ldcg(out + lo + i) | __ldcg(out + lo + h + i);
      __syncthreads();
    }
  }
  __syncthreads();
}

// CTA per vertex of the rank range [r0, r1)
__global__ void __launch_bounds__(512) k_sk_cta(const int64_t* __restrict__ off,
                                                const int32_t* __restrict__ adj, int64_t r0,
                                                int64_t r1, const int32_t* __restrict__ rdeg,
                                                const int64_t* __restrict__ skbase, int lk,
                                                uint32_t* __restrict__ sk, int64_t smem_words) {
  extern __shared__ uint32_t s[];  // [2 * smem_words]
  for (int64_t v = r0 + blockIdx.x; v < r1; v += gridDim.x)
    sk_cta_row(off, adj, v, rdeg, skbase, lk, sk, s, smem_words);
}

// Rows of listed ranks (the host-CSR chunk pipeline: the runs a chunk
// completed, in its sort-class lists [c0, c1), stride apart), those of degree
// in [dlo, dhi]: a warp per row (WARP, rows of <= 2 * WMAX words with the
// levels) or a CTA per row
template <bool WARP, int NT, int WMAX>
__global__ void __launch_bounds__(NT) k_sk_list(const int64_t* __restrict__ off,
                                                const int32_t* __restrict__ adj,
                                                const int32_t* __restrict__ lists, int64_t stride,
                                                const int* __restrict__ counts, int c0, int c1,
                                                int64_t dlo, int64_t dhi,
                                                const int32_t* __restrict__ rdeg,
                                                const int64_t* __restrict__ skbase, int lk,
                                                uint32_t* __restrict__ sk, int64_t smem_words) {
  extern __shared__ uint32_t dyn[];
  const int64_t g0 = WARP ? (blockIdx.x * (int64_t)NT + threadIdx.x) >> 5 : blockIdx.x;
  const int64_t ng = WARP ? ((int64_t)gridDim.x * NT) >> 5 : gridDim.x;
  const int lane = threadIdx.x & 31;
  uint32_t* s = WARP ? dyn + (threadIdx.x >> 5) * 2 * WMAX : dyn;
  for (int c = c0; c < c1; ++c) {
    const int64_t cnt = counts[c];
    for (int64_t j = g0; j < cnt; j += ng) {
      const int64_t v = lists[c * stride + j];
      const int64_t o = off[v], d = off[v + 1] - o;
      if (d < dlo || d > dhi) continue;  // uniform over the warp / CTA
      if (!WARP) {
        sk_cta_row(off, adj, v, rdeg, skbase, lk, sk, s, smem_words);
        continue;
      }
      const int64_t W = sk_words(d, lk);
      const uint32_t mask = (uint32_t)(W * 32 - 1);
      for (int64_t k = lane; k < W; k += 32) s[k] = 0u;
      __syncwarp();
      sk_hash_run<4>(adj + o, d, lane, 32, mask, s);
      __syncwarp();
      sk_fold_levels(s, W, lane, 32);
      uint32_t* out = sk + skbase[d] + (v - rdeg[d]) * 2 * W;
      for (int64_t k = lane; k < 2 * W - 4; k += 32) out[k] = s[k];
      __syncwarp();
    }
  }
}

// rdeg[d] = first rank of degree >= d (d in [0, dmax + 2]), as k_degree_tables
__global__ void k_sk_rdeg(const int64_t* __restrict__ off, int64_t n, int64_t dmax,
                          int32_t* __restrict__ rdeg) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d <= dmax + 2;
       d += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid + 1] - off[mid] < d) lo = mid + 1; else hi = mid;
    }
    rdeg[d] = (int32_t)lo;
  }
}

// algorithmic bytes of the build (CTR_B_PREP): the arcs of every sketched
// vertex read once, its row written once, its offsets read
__global__ void k_sk_bytes(const int64_t* __restrict__ off, int64_t n, int64_t r0,
                           const int64_t* __restrict__ skbase, int64_t dmax,
                           unsigned long long* __restrict__ ctr) {
  const int64_t arcs = off[n] - off[r0];
  // skbase[dmax + 1] counts the 2w-word slots; the levels fill 2w - 4 of each
  atomicAdd(&ctr[CTR_B_PREP], (unsigned long long)(4 * arcs + 4 * skbase[dmax + 1] + 16 * (n - r0)));
}

int build_sketch(gs_engine* e, int lk, int64_t dmin) {
  DevGraph& g = e->g;
  DevState& s = e->s;
  cudaStream_t st = e->stream;
  if (lk < 0 || g.n == 0 || g.dmax < dmin) {
    e->release(g.sk);
    e->release(g.skbase);
    g.sk = nullptr;
    g.skbase = nullptr;
    g.sk_lk = -1;
    return GS_OK;
  }
  if (g.sk && g.sk_lk == lk && g.sk_dmin == dmin) return GS_OK;  // cached with the graph
  e->release(g.sk);
  e->release(g.skbase);
  g.sk = nullptr;
  g.skbase = nullptr;
  g.sk_lk = -1;
  int64_t* sizes = nullptr;
  GS_TRY(e->alloc_n(&sizes, g.dmax + 2));
  GS_TRY(e->alloc_n(&g.skbase, g.dmax + 2));
  k_sk_sizes<<<grid_for(g.dmax + 2, 256), 256, 0, st>>>(g.dmax, dmin, lk, s.rdeg, sizes);
  e->launches++;
  size_t tb = 0;
  GS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, sizes, g.skbase, g.dmax + 2, st));
  void* tmp = nullptr;
  GS_TRY(e->alloc(&tmp, tb > 0 ? tb : 1));
  GS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, sizes, g.skbase, g.dmax + 2, st));
  e->launches++;
  e->release(tmp);
  e->release(sizes);
  int64_t total = 0;
  int32_t r[3] = {0, 0, 0};
  // rank ranges by sketch size: <= 128 words (warp per vertex), <= 2048
  // words (8 KB CTA), larger (one big CTA per vertex)
  // rows of <= 256 words by a warp (measured: 128 / 256 / 512 words -> prep 2.33 / 2.21 / 2.64 ms)
  static const int wmax = getenv("GS_SK_WMAX") ? atoi(getenv("GS_SK_WMAX")) : 256;
  // four neighbour loads in flight per lane before their shared atomics
  // (measured: prep 2.22 -> 2.00 ms at s24 eps 0.5, step 21.11 -> 20.89; GS_SK_UNROLL=1: one)
  static const int sk_unr = getenv("GS_SK_UNROLL") ? atoi(getenv("GS_SK_UNROLL")) : 4;
  const int64_t dsplit = (int64_t)wmax * 32 >> lk, dsplit2 = 2048 * 32 >> lk;
  GS_CUDA(cudaMemcpyAsync(&total, g.skbase + g.dmax + 1, sizeof(total), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaMemcpyAsync(&r[0], s.rdeg + dmin, 4, cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaMemcpyAsync(&r[1], s.rdeg + std::min<int64_t>(dsplit + 1, g.dmax + 2), 4,
                          cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaMemcpyAsync(&r[2], s.rdeg + std::min<int64_t>(dsplit2 + 1, g.dmax + 2), 4,
                          cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  if (e->alloc_n(&g.sk, total) != GS_OK) {  // no room (HBM cap): scan without sketches
    e->release(g.skbase);
    g.skbase = nullptr;
    g.sk = nullptr;
    return GS_OK;
  }
  const int64_t r0 = r[0], r1 = std::max<int64_t>(r[0], r[1]), n = g.n;
  const int64_t r2 = std::max<int64_t>(r1, r[2]);
  if (r1 > r0) {
    constexpr int NT = 256;
    int64_t grid = (r1 - r0 + NT / 32 - 1) / (NT / 32);
    grid = std::min<int64_t>(grid, (int64_t)e->sms * 8);
    if (wmax >= 512)
      k_sk_warp<NT, 512><<<(unsigned)grid, NT, 0, st>>>(g.off, g.adj, r0, r1, s.rdeg, g.skbase, lk,
                                                        g.sk);
    else if (wmax >= 256 && sk_unr == 4)
      k_sk_warp<NT, 256, 4><<<(unsigned)grid, NT, 0, st>>>(g.off, g.adj, r0, r1, s.rdeg, g.skbase,
                                                           lk, g.sk);
    else if (wmax >= 256)
      k_sk_warp<NT, 256><<<(unsigned)grid, NT, 0, st>>>(g.off, g.adj, r0, r1, s.rdeg, g.skbase, lk,
                                                        g.sk);
    else
      k_sk_warp<NT, 128><<<(unsigned)grid, NT, 0, st>>>(g.off, g.adj, r0, r1, s.rdeg, g.skbase, lk,
                                                        g.sk);
    e->launches++;
  }
  if (r2 > r1) {
    const int64_t smem_words = 2048;  // 16 KB with the levels: many CTAs per SM
    const int64_t grid = std::min<int64_t>(r2 - r1, (int64_t)e->sms * 8);
    k_sk_cta<<<(unsigned)grid, 256, smem_words * 8, st>>>(g.off, g.adj, r1, r2, s.rdeg, g.skbase,
                                                          lk, g.sk, smem_words);
    e->launches++;
  }
  if (n > r2) {
    const int64_t smem_words =
        std::min<int64_t>(16384, sk_words(g.dmax, lk));  // <= 128 KB with the levels
    auto kern = k_sk_cta;
    GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(smem_words * 8)));
    const int64_t grid = std::min<int64_t>(n - r2, (int64_t)e->sms * 2);
    kern<<<(unsigned)grid, 512, smem_words * 8, st>>>(g.off, g.adj, r2, n, s.rdeg, g.skbase, lk,
                                                      g.sk, smem_words);
    e->launches++;
  }
  if (s.ctr && n > r0) {
    k_sk_bytes<<<1, 1, 0, st>>>(g.off, n, r0, g.skbase, g.dmax, s.ctr);
    e->launches++;
  }
  GS_CUDA(cudaGetLastError());
  g.sk_lk = lk;
  g.sk_dmin = dmin;
  return GS_OK;
}

// --- rows built while the graph streams in (host-CSR chunk pipeline) -------
// The layout of build_sketch at resolution lk (the rank-space offsets exist,
// the runs do not yet): rdeg (returned, the caller releases it), skbase and
// the rows' buffer.  Leaves g.sk null when there is no room (HBM cap).
int sketch_stream_begin(gs_engine* e, int64_t n, int64_t dmax, int lk, int64_t dmin,
                        int32_t** rdeg_out) {
  DevGraph& g = e->g;
  cudaStream_t st = e->stream;
  *rdeg_out = nullptr;
  if (n == 0 || dmax < dmin) return GS_OK;
  int32_t* rdeg = nullptr;
  int64_t* sizes = nullptr;
  GS_TRY(e->alloc_n(&rdeg, dmax + 3));
  GS_TRY(e->alloc_n(&sizes, dmax + 2));
  GS_TRY(e->alloc_n(&g.skbase, dmax + 2));
  k_sk_rdeg<<<grid_for(dmax + 3, 256), 256, 0, st>>>(g.off, n, dmax, rdeg);
  k_sk_sizes<<<grid_for(dmax + 2, 256), 256, 0, st>>>(dmax, dmin, lk, rdeg, sizes);
  size_t tb = 0;
  GS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, sizes, g.skbase, dmax + 2, st));
  void* tmp = nullptr;
  GS_TRY(e->alloc(&tmp, tb > 0 ? tb : 1));
  GS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, sizes, g.skbase, dmax + 2, st));
  e->launches += 3;
  e->release(tmp);
  e->release(sizes);
  int64_t total = 0;
  GS_CUDA(cudaMemcpyAsync(&total, g.skbase + dmax + 1, sizeof(total), cudaMemcpyDeviceToHost, st));
  GS_CUDA(cudaStreamSynchronize(st));
  if (e->alloc_n(&g.sk, std::max<int64_t>(total, 1)) != GS_OK) {
    cudaGetLastError();
    e->release(g.skbase);
    g.skbase = nullptr;
    e->release(rdeg);
    return GS_OK;
  }
  *rdeg_out = rdeg;
  return GS_OK;
}

// rows of the runs listed in [c0, c1) of a chunk's class lists (runs complete,
// in any order: a row is a set)
//
// The chunk's lists are its sort classes (build.cu k_chunk_classes: <= 32,
// <= 256, <= 512, <= 1024, <= 2048, < 4096, <= 16384, longer); at k = 4 the
// warp rows (<= 2048 neighbours) are classes 0-4, the 2048-word CTA rows
// classes 5-6 and the long rows class 7, so each kernel walks only its own
// lists (every kernel still filters by degree).
int sketch_stream_rows(gs_engine* e, int64_t dmax, int lk, int64_t dmin, const int32_t* rdeg,
                       const int32_t* adj, const int32_t* lists, int64_t stride,
                       const int* counts, int64_t nlisted) {
  DevGraph& g = e->g;
  cudaStream_t st = e->stream;
  if (!g.sk || nlisted == 0) return GS_OK;
  if (lk != 2) { set_error("streamed sketch rows are built at k = 4 only"); return GS_EINVAL; }
  constexpr int NT = 256, WMAX = 256;
  const int64_t dsplit = (int64_t)WMAX * 32 >> lk, dsplit2 = (int64_t)2048 * 32 >> lk;
  const unsigned wg = (unsigned)std::min<int64_t>((nlisted + 7) / 8, (int64_t)e->sms * 8);
  k_sk_list<true, NT, WMAX><<<wg, NT, (NT / 32) * 2 * WMAX * 4, st>>>(
      g.off, adj, lists, stride, counts, 0, 5, dmin, dsplit, rdeg, g.skbase, lk, g.sk, 0);
  k_sk_list<false, NT, WMAX><<<(unsigned)e->sms * 2, NT, 2048 * 8, st>>>(
      g.off, adj, lists, stride, counts, 5, 7, std::max(dmin, dsplit + 1), dsplit2, rdeg,
      g.skbase, lk, g.sk, 2048);
  e->launches += 2;
  if (dmax > dsplit2) {
    const int64_t smem_words = std::min<int64_t>(16384, sk_words(dmax, lk));
    auto kern = k_sk_list<false, 512, WMAX>;
    GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(smem_words * 8)));
    kern<<<(unsigned)e->sms, 512, smem_words * 8, st>>>(
        g.off, adj, lists, stride, counts, 7, 8, std::max(dmin, dsplit2 + 1), dmax, rdeg,
        g.skbase, lk, g.sk, smem_words);
    e->launches++;
  }
  GS_CUDA(cudaGetLastError());
  return GS_OK;
}

}  // namespace gs
