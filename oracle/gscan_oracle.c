/*
 * gscan_oracle.c -- CPU restatement of the reference clustering path.
 * TEST INFRASTRUCTURE ONLY (see gscan_oracle.h): the checker and the timed
 * CPU baseline, never part of the shipped product path.
 */
#include "gscan_oracle.h"

#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

/* ------------------------------------------------------------------------ */
/* minimal pthread parallel-for with dynamic chunks (no OpenMP dependency)   */

typedef void (*par_body)(int64_t lo, int64_t hi, void* ctx, int tid);
typedef struct par_job {
  par_body fn; void* ctx; int64_t n, chunk; _Atomic int64_t next; int tid;
} par_job;
typedef struct par_arg { par_job* job; int tid; } par_arg;

static void* par_worker(void* p) {
  par_arg* a = (par_arg*)p;
  par_job* j = a->job;
  for (;;) {
    int64_t lo = atomic_fetch_add(&j->next, j->chunk);
    if (lo >= j->n) break;
    int64_t hi = lo + j->chunk < j->n ? lo + j->chunk : j->n;
    j->fn(lo, hi, j->ctx, a->tid);
  }
  return NULL;
}

static int g_threads = 0;
int orc_max_threads(void) {
  if (g_threads > 0) return g_threads;
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}

static void par_for(int64_t n, int64_t chunk, int threads, par_body fn, void* ctx) {
  if (threads <= 0) threads = orc_max_threads();
  if (threads > 256) threads = 256;
  if (n <= chunk || threads == 1) { if (n > 0) fn(0, n, ctx, 0); return; }
  par_job job; job.fn = fn; job.ctx = ctx; job.n = n; job.chunk = chunk;
  atomic_init(&job.next, 0);
  pthread_t th[256]; par_arg args[256];
  for (int t = 0; t < threads; ++t) {
    args[t].job = &job; args[t].tid = t;
    pthread_create(&th[t], NULL, par_worker, &args[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* synthetic workload: R-MAT with a counter-based hash (bit-identical to the
 * CUDA generator gs_rmat_generate in paper_2311_12281_b200/csrc/ingest.cu)  */

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* Graph500 initiator (0.57, 0.19, 0.19, 0.05) as 32-bit thresholds. */
#define RMAT_TA 2448131358u   /* floor(0.57 * 2^32) */
#define RMAT_TAB 3264175144u  /* floor(0.76 * 2^32) */
#define RMAT_TABC 4080218931u /* floor(0.95 * 2^32) */

static inline uint32_t rmat_scramble(uint32_t x, int scale, uint64_t sm) {
  const uint64_t mask = (scale >= 32) ? 0xFFFFFFFFull : ((1ull << scale) - 1);
  const int h = (scale + 1) / 2;
  uint64_t y = x;
  y = (y * 0x9E3779B97F4A7C15ULL + (sm & mask)) & mask;
  y ^= y >> h;
  y = (y * 0xD6E8FEB86659FD93ULL) & mask;
  y ^= y >> h;
  return (uint32_t)y;
}

typedef struct rmat_ctx {
  int scale; uint64_t sm; int64_t first; int32_t *src, *dst;
} rmat_ctx;

static void rmat_body(int64_t lo, int64_t hi, void* p, int tid) {
  (void)tid;
  rmat_ctx* c = (rmat_ctx*)p;
  const int scale = c->scale;
  const uint64_t sm = c->sm;
  int32_t* src = c->src;
  int32_t* dst = c->dst;
  for (int64_t t = lo; t < hi; ++t) {
    const uint64_t i = (uint64_t)(c->first + t);
    uint32_t u = 0, v = 0;
    uint64_t r = 0;
    for (int l = 0; l < scale; ++l) {
      uint32_t x;
      if ((l & 1) == 0) {
        r = mix64(sm ^ (i * 32u + (uint64_t)(l >> 1)));
        x = (uint32_t)(r >> 32);
      } else {
        x = (uint32_t)r;
      }
      const uint32_t qd = x < RMAT_TA ? 0u : x < RMAT_TAB ? 1u : x < RMAT_TABC ? 2u : 3u;
      u = (u << 1) | (qd >> 1);
      v = (v << 1) | (qd & 1u);
    }
    src[t] = (int32_t)rmat_scramble(u, scale, sm);
    dst[t] = (int32_t)rmat_scramble(v, scale, sm ^ 0x5bd1e995u);
  }
}

void orc_rmat_edges(int scale, int ef, uint64_t seed, int64_t first,
                    int64_t count, int32_t* src, int32_t* dst) {
  (void)ef;
  rmat_ctx c = {scale, mix64(seed), first, src, dst};
  par_for(count, 1 << 16, 0, rmat_body, &c);
}

/* LSD radix sort of 64-bit keys, 16-bit digits, skipping constant digits. */
static void radix_sort_u64(uint64_t* keys, int64_t n) {
  if (n < 2) return;
  uint64_t* tmp = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
  size_t* cnt = (size_t*)malloc(65536 * sizeof(size_t));
  uint64_t* a = keys;
  uint64_t* b = tmp;
  for (int shift = 0; shift < 64; shift += 16) {
    memset(cnt, 0, 65536 * sizeof(size_t));
    for (int64_t i = 0; i < n; ++i) cnt[(a[i] >> shift) & 0xFFFF]++;
    int constant = 0;
    for (int d = 0; d < 65536; ++d)
      if (cnt[d] == (size_t)n) { constant = 1; break; }
    if (constant) continue;
    size_t s = 0;
    for (int d = 0; d < 65536; ++d) { size_t c = cnt[d]; cnt[d] = s; s += c; }
    for (int64_t i = 0; i < n; ++i) b[cnt[(a[i] >> shift) & 0xFFFF]++] = a[i];
    uint64_t* t = a; a = b; b = t;
  }
  if (a != keys) memcpy(keys, a, (size_t)n * sizeof(uint64_t));
  free(tmp);
  free(cnt);
}

/* parse_edge_list normalisation (graph.py:96-117): self-loops dropped,
 * (min,max) orientation, duplicates merged, sorted. */
int64_t orc_normalize(int64_t count, int32_t* src, int32_t* dst) {
  uint64_t* k = (uint64_t*)malloc((size_t)(count > 0 ? count : 1) * sizeof(uint64_t));
  int64_t c = 0;
  for (int64_t i = 0; i < count; ++i) {
    uint32_t u = (uint32_t)src[i], v = (uint32_t)dst[i];
    if (u == v) continue;
    if (u > v) { uint32_t t = u; u = v; v = t; }
    k[c++] = ((uint64_t)u << 32) | v;
  }
  radix_sort_u64(k, c);
  int64_t w = 0;
  for (int64_t i = 0; i < c; ++i) {
    if (i > 0 && k[i] == k[i - 1]) continue;
    src[w] = (int32_t)(k[i] >> 32);
    dst[w] = (int32_t)(uint32_t)k[i];
    ++w;
  }
  free(k);
  return w;
}

/* ------------------------------------------------------------------------ */
/* build_graph (graph.py:162-259)                                           */

static int64_t lower_bound_i32(const int32_t* a, int64_t lo, int64_t hi, int32_t x) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

typedef struct eid_ctx {
  const int64_t* off; const int32_t* adj; const int32_t* el; int32_t* eid;
} eid_ctx;

/* Eid by binary search of each endpoint in the other's run (graph.py:233-240);
 * every slot is written by exactly one edge, so edges run in parallel. */
static void eid_body(int64_t lo, int64_t hi, void* p, int tid) {
  (void)tid;
  eid_ctx* c = (eid_ctx*)p;
  for (int64_t e = lo; e < hi; ++e) {
    int32_t a = c->el[2 * e], b = c->el[2 * e + 1];
    int64_t sa = lower_bound_i32(c->adj, c->off[a], c->off[a + 1], b);
    int64_t sb = lower_bound_i32(c->adj, c->off[b], c->off[b + 1], a);
    c->eid[sa] = (int32_t)e;
    c->eid[sb] = (int32_t)e;
  }
}

int orc_build_graph(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev,
                    int64_t* offsets, int32_t* adjacency, int32_t* edge_ids,
                    int32_t* edge_list) {
  int64_t* deg = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
  for (int64_t k = 0; k < m; ++k) {  /* graph.py:184-196 */
    int32_t u = eu[k], v = ev[k];
    if (u < 0 || v < 0 || u >= n || v >= n || u == v) { free(deg); return -1; }
    deg[u]++; deg[v]++;
  }
  int64_t tot = 0;                    /* graph.py:198-203 */
  for (int64_t u = 0; u < n; ++u) { offsets[u] = tot; tot += deg[u]; }
  offsets[n] = tot;
  int64_t* cur = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  memcpy(cur, offsets, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t k = 0; k < m; ++k) {  /* graph.py:205-211 */
    adjacency[cur[eu[k]]++] = ev[k];
    adjacency[cur[ev[k]]++] = eu[k];
  }
  free(cur);
  int bad = 0;
  for (int64_t u = 0; u < n && !bad; ++u) { /* graph.py:212-216 sort runs */
    int64_t lo = offsets[u], hi = offsets[u + 1];
    for (int64_t i = lo + 1; i < hi; ++i) {
      int32_t x = adjacency[i];
      int64_t j = i - 1;
      while (j >= lo && adjacency[j] > x) { adjacency[j + 1] = adjacency[j]; --j; }
      adjacency[j + 1] = x;
    }
    for (int64_t i = lo + 1; i < hi; ++i)
      if (adjacency[i] == adjacency[i - 1]) bad = 1; /* duplicate edge */
  }
  if (bad) { free(deg); return -1; }
  int64_t k = 0;                      /* graph.py:218-231 */
  for (int64_t a = 0; a < n; ++a) {
    int64_t da = deg[a];
    for (int64_t s = offsets[a]; s < offsets[a + 1]; ++s) {
      int32_t b = adjacency[s];
      int64_t db = deg[b];
      if (da < db || (da == db && a < b)) {
        edge_list[2 * k] = (int32_t)a;
        edge_list[2 * k + 1] = b;
        ++k;
      }
    }
  }
  eid_ctx ec = {offsets, adjacency, edge_list, edge_ids};  /* graph.py:233-240 */
  par_for(m, 4096, 0, eid_body, &ec);
  free(deg);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* exact threshold (scan.py:232-233, oracle.py:58-60):                      */
/*   (c+2)^2 * q >= p * (da+1)(db+1), in 192-bit integer arithmetic.         */

static inline int ge192(uint64_t x, uint64_t d, orc_eps2 e) {
  u128 l0 = (u128)x * e.q_lo;
  u128 l1 = (u128)x * e.q_hi + (uint64_t)(l0 >> 64);
  u128 r0 = (u128)d * e.p_lo;
  u128 r1 = (u128)d * e.p_hi + (uint64_t)(r0 >> 64);
  uint64_t a2 = (uint64_t)(l1 >> 64), a1 = (uint64_t)l1, a0 = (uint64_t)l0;
  uint64_t b2 = (uint64_t)(r1 >> 64), b1 = (uint64_t)r1, b0 = (uint64_t)r0;
  if (a2 != b2) return a2 > b2;
  if (a1 != b1) return a1 > b1;
  return a0 >= b0;
}

static inline int is_similar(int64_t common, int64_t da, int64_t db, orc_eps2 e) {
  uint64_t s = (uint64_t)(common + 2);
  return ge192(s * s, (uint64_t)(da + 1) * (uint64_t)(db + 1), e);
}

/* common_neighbors by sorted-run merge (oracle.py:27-44) */
static int64_t merge_common(const int64_t* off, const int32_t* adj, int32_t u, int32_t v) {
  int64_t i = off[u], ihi = off[u + 1], j = off[v], jhi = off[v + 1], c = 0;
  while (i < ihi && j < jhi) {
    int32_t x = adj[i], y = adj[j];
    if (x == y) { ++c; ++i; ++j; }
    else if (x < y) ++i;
    else ++j;
  }
  return c;
}

typedef struct commons_ctx {
  const int64_t* off; const int32_t* adj; const int32_t* el; int32_t* out;
  uint8_t* sim; orc_eps2 e;
} commons_ctx;

static void commons_body(int64_t lo, int64_t hi, void* p, int tid) {
  (void)tid;
  commons_ctx* c = (commons_ctx*)p;
  for (int64_t k = lo; k < hi; ++k) {
    int32_t u = c->el[2 * k], v = c->el[2 * k + 1];
    int64_t cm = merge_common(c->off, c->adj, u, v);
    if (c->out) c->out[k] = (int32_t)cm;
    if (c->sim)
      c->sim[k] = (uint8_t)is_similar(cm, c->off[u + 1] - c->off[u],
                                      c->off[v + 1] - c->off[v], c->e);
  }
}

void orc_edge_commons(int64_t n, int64_t m, const int64_t* offsets,
                      const int32_t* adjacency, const int32_t* edge_list,
                      int32_t* commons) {
  (void)n;
  commons_ctx c = {offsets, adjacency, edge_list, commons, NULL, {0, 0, 1, 0}};
  par_for(m, 1024, 0, commons_body, &c);
}

/* ------------------------------------------------------------------------ */
/* serial_scan (oracle.py:97-206), canonical output.           */

static int32_t uf_find(int32_t* p, int32_t x) {
  while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
  return x;
}

/* Common-neighbour counts of every edge (edge_list order) by marking instead
 * of merging: per high endpoint b (the larger (degree, id) side, graph.py:226)
 * N(b) is set in a thread-private bitmap of n bits and every lower neighbour
 * a counts N(a) against it.  Same numbers as merge_common (checked against it
 * in tests/test_oracle_golden.py); sum_k min(d) work instead of sum_k (da+db),
 * which is what makes R-MAT s24 (sum d^2 = 3.6e12) a minutes-long check. */
typedef struct marks_ctx {
  const int64_t* off; const int32_t* adj; const int32_t* eid; int32_t* out;
  uint64_t** bits;
} marks_ctx;

static void marks_body(int64_t lo, int64_t hi, void* p, int tid) {
  marks_ctx* c = (marks_ctx*)p;
  uint64_t* bm = c->bits[tid];
  for (int64_t b = lo; b < hi; ++b) {
    int64_t b0 = c->off[b], b1 = c->off[b + 1], db = b1 - b0;
    int any = 0;
    for (int64_t s = b0; s < b1; ++s) {
      int32_t a = c->adj[s];
      int64_t da = c->off[a + 1] - c->off[a];
      if (da < db || (da == db && a < b)) { any = 1; break; }
    }
    if (!any) continue;
    for (int64_t s = b0; s < b1; ++s) { uint32_t w = (uint32_t)c->adj[s]; bm[w >> 6] |= 1ull << (w & 63); }
    for (int64_t s = b0; s < b1; ++s) {
      int32_t a = c->adj[s];
      int64_t a0 = c->off[a], a1 = c->off[a + 1], da = a1 - a0;
      if (!(da < db || (da == db && a < b))) continue;
      int64_t cm = 0;
      for (int64_t i = a0; i < a1; ++i) {
        uint32_t w = (uint32_t)c->adj[i];
        cm += (int64_t)((bm[w >> 6] >> (w & 63)) & 1u);
      }
      c->out[c->eid[s]] = (int32_t)cm;
    }
    for (int64_t s = b0; s < b1; ++s) { uint32_t w = (uint32_t)c->adj[s]; bm[w >> 6] = 0; }
  }
}

void orc_edge_commons_marked(int64_t n, int64_t m, const int64_t* offsets,
                             const int32_t* adjacency, const int32_t* edge_ids,
                             int32_t* commons) {
  (void)m;
  int threads = orc_max_threads();
  if (threads > 256) threads = 256;
  uint64_t* bits[256];
  size_t words = (size_t)((n + 63) / 64 + 1);
  for (int t = 0; t < threads; ++t) bits[t] = (uint64_t*)calloc(words, sizeof(uint64_t));
  marks_ctx c = {offsets, adjacency, edge_ids, commons, bits};
  par_for(n, 256, threads, marks_body, &c);
  for (int t = 0; t < threads; ++t) free(bits[t]);
}

typedef struct thr_ctx {
  const int64_t* off; const int32_t* el; const int32_t* cm; uint8_t* sim; orc_eps2 e;
} thr_ctx;

static void thr_body(int64_t lo, int64_t hi, void* p, int tid) {
  (void)tid;
  thr_ctx* c = (thr_ctx*)p;
  for (int64_t k = lo; k < hi; ++k) {
    int32_t u = c->el[2 * k], v = c->el[2 * k + 1];
    c->sim[k] = (uint8_t)is_similar(c->cm[k], c->off[u + 1] - c->off[u],
                                    c->off[v + 1] - c->off[v], c->e);
  }
}

static int serial_scan_core(int64_t n, int64_t m, const int64_t* off, const int32_t* adj,
                            const int32_t* el, int32_t mu, uint8_t* similar,
                            uint8_t* role_out, int32_t* cluster_out);

int orc_serial_scan(int64_t n, int64_t m, const int64_t* off,
                    const int32_t* adj, const int32_t* el, int32_t mu,
                    orc_eps2 eps2, uint8_t* role_out, int32_t* cluster_out) {
  if (mu < 2) return -1;
  uint8_t* similar = (uint8_t*)malloc((size_t)(m > 0 ? m : 1));
  {                                               /* oracle.py:118-127 */
    commons_ctx cc = {off, adj, el, NULL, similar, eps2};
    par_for(m, 1024, 0, commons_body, &cc);
  }
  return serial_scan_core(n, m, off, adj, el, mu, similar, role_out, cluster_out);
}

/* serial_scan with the common-neighbour counts given (one count pass serves
 * every (eps, mu) of a sweep); identical output to orc_serial_scan. */
int orc_serial_scan_commons(int64_t n, int64_t m, const int64_t* off,
                            const int32_t* adj, const int32_t* el, const int32_t* commons,
                            int32_t mu, orc_eps2 eps2, uint8_t* role_out,
                            int32_t* cluster_out) {
  if (mu < 2) return -1;
  uint8_t* similar = (uint8_t*)malloc((size_t)(m > 0 ? m : 1));
  thr_ctx tc = {off, el, commons, similar, eps2};
  par_for(m, 4096, 0, thr_body, &tc);
  return serial_scan_core(n, m, off, adj, el, mu, similar, role_out, cluster_out);
}

static int serial_scan_core(int64_t n, int64_t m, const int64_t* off, const int32_t* adj,
                            const int32_t* el, int32_t mu, uint8_t* similar,
                            uint8_t* role_out, int32_t* cluster_out) {
  int64_t* simcnt = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  for (int64_t k = 0; k < m; ++k)
    if (similar[k]) { simcnt[el[2 * k]]++; simcnt[el[2 * k + 1]]++; }
  uint8_t* core = (uint8_t*)malloc((size_t)(n > 0 ? n : 1));
  for (int64_t v = 0; v < n; ++v) core[v] = (uint8_t)(simcnt[v] + 1 >= mu); /* :129 */
  /* clusters = components of the similar core-core graph, label = min id
   * (oracle.py:131-160); union-find with min-root is the same partition. */
  int32_t* p = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
  for (int64_t v = 0; v < n; ++v) p[v] = (int32_t)v;
  for (int64_t k = 0; k < m; ++k) {
    if (!similar[k]) continue;
    int32_t u = el[2 * k], v = el[2 * k + 1];
    if (!core[u] || !core[v]) continue;
    int32_t ru = uf_find(p, u), rv = uf_find(p, v);
    if (ru == rv) continue;
    if (ru < rv) p[rv] = ru; else p[ru] = rv;
  }
  /* memberships as (min,max) label per vertex (oracle.py:162-171); a set of
   * labels has >=2 elements iff min != max, which is all _oracle_is_hub needs */
  int32_t* lmin = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
  int32_t* lmax = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
  for (int64_t v = 0; v < n; ++v) {
    if (core[v]) { int32_t r = uf_find(p, (int32_t)v); lmin[v] = lmax[v] = r; }
    else { lmin[v] = INT32_MAX; lmax[v] = -1; }
  }
  for (int64_t k = 0; k < m; ++k) {
    if (!similar[k]) continue;
    int32_t u = el[2 * k], v = el[2 * k + 1];
    for (int side = 0; side < 2; ++side) {
      int32_t c = side ? v : u, w = side ? u : v;
      if (core[c] && !core[w]) {
        int32_t L = lmin[c];
        if (L < lmin[w]) lmin[w] = L;
        if (L > lmax[w]) lmax[w] = L;
      }
    }
  }
  for (int64_t v = 0; v < n; ++v) {               /* oracle.py:173-181 */
    if (core[v]) { role_out[v] = ORC_ROLE_CORE; cluster_out[v] = lmin[v]; continue; }
    if (lmax[v] >= 0) { role_out[v] = ORC_ROLE_MEMBER; cluster_out[v] = lmin[v]; continue; }
    /* _oracle_is_hub (oracle.py:193-206) */
    int64_t clustered = 0;
    int32_t umin = INT32_MAX, umax = -1;
    int hub = 0;
    for (int64_t i = off[v]; i < off[v + 1] && !hub; ++i) {
      int32_t x = adj[i];
      if (lmax[x] < 0) continue;
      clustered++;
      if (lmin[x] < umin) umin = lmin[x];
      if (lmax[x] > umax) umax = lmax[x];
      if (clustered >= 2 && umin != umax) hub = 1;
    }
    role_out[v] = hub ? ORC_ROLE_HUB : ORC_ROLE_OUTLIER;
    cluster_out[v] = -1;
  }
  free(similar); free(simcnt); free(core); free(p); free(lmin); free(lmax);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* scan_in_memory, workers=1 (scan.py:110-982), sequential restatement.     */

/* _eval_edge (scan.py:203-233): binary-search probing, probe count. */
static inline int eval_edge(const int32_t* adj, int64_t alo, int64_t ahi,
                            int64_t blo, int64_t bhi, orc_eps2 e, int64_t* probes) {
  int64_t count = 0, pr = 0;
  for (int64_t i = alo; i < ahi; ++i) {
    int32_t w = adj[i];
    int64_t lo = blo, hi = bhi;
    while (lo < hi) {
      ++pr;
      int64_t mid = (lo + hi) >> 1;
      int32_t x = adj[mid];
      if (x < w) lo = mid + 1;
      else if (x > w) hi = mid;
      else { ++count; break; }
    }
  }
  *probes = pr;
  return is_similar(count, ahi - alo, bhi - blo, e);
}

/* _probe_cap (scan.py:236-238): da * (ceil(log2 db) + 1) */
static inline int64_t probe_cap(int64_t da, int64_t db) {
  int64_t bits = 0, x = db - 1;
  while (x > 0) { ++bits; x >>= 1; }
  return da * (bits + 1);
}

typedef struct ref_state {
  int32_t *lower, *upper, *parent, *height;
  uint8_t *role, *sim;
} ref_state;

static void record_similarity(ref_state* st, int32_t u, int32_t v, int similar, int32_t mu) {
  int32_t xs[2] = {u, v};                          /* scan.py:302-345 */
  for (int i = 0; i < 2; ++i) {
    int32_t x = xs[i];
    if (similar) {
      int32_t lv = ++st->lower[x];
      if (lv >= mu && st->role[x] == ORC_ROLE_UNKNOWN) st->role[x] = ORC_ROLE_CORE;
    } else {
      int32_t uv = --st->upper[x];
      if (uv < mu && st->role[x] == ORC_ROLE_UNKNOWN) st->role[x] = ORC_ROLE_NONCORE;
    }
  }
}

static int32_t chase(const int32_t* parent, int32_t u) {  /* scan.py:498-504 */
  int32_t r = u, nxt = parent[r];
  while (nxt != r) { r = nxt; nxt = parent[r]; }
  return r;
}

static void union_roots(ref_state* st, int32_t u, int32_t v) { /* scan.py:514-548 */
  int32_t ru = chase(st->parent, u), rv = chase(st->parent, v);
  if (ru == rv) return;
  int32_t hu = st->height[ru], hv = st->height[rv];
  if (hu < hv) st->parent[ru] = rv;
  else if (hv < hu) st->parent[rv] = ru;
  else { st->parent[rv] = ru; st->height[ru] = hu + 1; }
}

#define EVAL_COUNTED(a, b, out_sim)                                              \
  do {                                                                           \
    int64_t _pr;                                                                 \
    int64_t _alo = off[a], _ahi = off[(a) + 1], _blo = off[b], _bhi = off[(b) + 1]; \
    out_sim = eval_edge(adj, _alo, _ahi, _blo, _bhi, eps2, &_pr);                \
    c->sim_evals++;                                                              \
    c->adj_probes += _pr;                                                        \
    if (_pr > probe_cap(_ahi - _alo, _bhi - _blo)) c->probe_bound_violations++;  \
  } while (0)

int orc_ref_scan(int64_t n, int64_t m, const int64_t* off, const int32_t* adj,
                 const int32_t* el, int32_t mu, orc_eps2 eps2, uint8_t* role_out,
                 int32_t* cluster_out, orc_counters* c) {
  if (mu < 2) return -1;
  memset(c, 0, sizeof(*c));
  size_t nn = (size_t)(n > 0 ? n : 1), mm = (size_t)(m > 0 ? m : 1);
  ref_state s;
  s.lower = (int32_t*)malloc(nn * 4); s.upper = (int32_t*)malloc(nn * 4);
  s.parent = (int32_t*)malloc(nn * 4); s.height = (int32_t*)malloc(nn * 4);
  s.role = (uint8_t*)calloc(nn, 1); s.sim = (uint8_t*)calloc(mm, 1);
  for (int64_t v = 0; v < n; ++v) {                /* init_vertex_state 117-134 */
    s.lower[v] = 1; s.upper[v] = (int32_t)(off[v + 1] - off[v] + 1);
    s.parent[v] = -2; s.height[v] = 1;
  }
  /* identify_core: _identify_range(0, m) (scan.py:351-387) */
  for (int64_t k = 0; k < m; ++k) {
    int32_t a = el[2 * k], b = el[2 * k + 1];
    if (s.role[a] && s.role[b]) continue;
    int sm;
    EVAL_COUNTED(a, b, sm);
    s.sim[k] = sm ? 1 : 2;
    record_similarity(&s, a, b, sm, mu);
  }
  /* _cleanup_unknown_roles (scan.py:415-449) */
  int unresolved = 0;
  for (int64_t v = 0; v < n; ++v) {                /* resolve_roles_from_bounds */
    if (s.role[v] == 0) {
      if (s.lower[v] >= mu) s.role[v] = ORC_ROLE_CORE;
      else if (s.upper[v] < mu) s.role[v] = ORC_ROLE_NONCORE;
      else unresolved = 1;
    }
  }
  if (unresolved) {
    for (int64_t k = 0; k < m; ++k) {
      if (s.sim[k] != 0) continue;
      int32_t a = el[2 * k], b = el[2 * k + 1];
      if (s.role[a] && s.role[b]) continue;
      int sm;
      EVAL_COUNTED(a, b, sm);
      s.sim[k] = sm ? 1 : 2;
      record_similarity(&s, a, b, sm, mu);
    }
    for (int64_t v = 0; v < n; ++v) {
      if (s.role[v] == 0) {
        if (s.lower[v] >= mu) s.role[v] = ORC_ROLE_CORE;
        else if (s.upper[v] < mu) s.role[v] = ORC_ROLE_NONCORE;
        else { unresolved = 2; }
      }
    }
    if (unresolved == 2) goto fail;
  }
  /* detect_clusters, workers=1 (scan.py:724-733) */
  for (int64_t v = 0; v < n; ++v)
    if (s.role[v] == ORC_ROLE_CORE && s.parent[v] == -2) s.parent[v] = (int32_t)v;
  for (int64_t k = 0; k < m; ++k) {                /* _union_known_range */
    if (s.sim[k] != 1) continue;
    int32_t a = el[2 * k], b = el[2 * k + 1];
    if (s.role[a] == ORC_ROLE_CORE && s.role[b] == ORC_ROLE_CORE) union_roots(&s, a, b);
  }
  for (int64_t k = 0; k < m; ++k) {                /* _union_unknown_range */
    if (s.sim[k] != 0) continue;
    int32_t a = el[2 * k], b = el[2 * k + 1];
    if (s.role[a] != ORC_ROLE_CORE || s.role[b] != ORC_ROLE_CORE) continue;
    int32_t ra = chase(s.parent, a), rb = chase(s.parent, b);
    if (ra == rb) continue;
    int sm;
    EVAL_COUNTED(a, b, sm);
    s.sim[k] = sm ? 1 : 2;
    if (sm) union_roots(&s, ra, rb);
  }
  for (int64_t v = 0; v < n; ++v)                  /* flatten */
    if (s.role[v] == ORC_ROLE_CORE) s.parent[v] = chase(s.parent, (int32_t)v);
  for (int64_t k = 0; k < m; ++k) {                /* _attach_range */
    int32_t a = el[2 * k], b = el[2 * k + 1];
    int ca = s.role[a] == ORC_ROLE_CORE;
    if (ca == (s.role[b] == ORC_ROLE_CORE)) continue;
    int32_t core = ca ? a : b, w = ca ? b : a;
    int sv = s.sim[k];
    if (sv == 0) {
      int sm;
      EVAL_COUNTED(a, b, sm);
      sv = sm ? 1 : 2;
      s.sim[k] = (uint8_t)sv;
    }
    if (sv == 1) {                                 /* _attach_member 570-590 */
      int32_t root = chase(s.parent, core);
      int32_t cur = s.parent[w];
      if (cur < 0) { s.parent[w] = root; s.role[w] = ORC_ROLE_MEMBER; }
      else if (cur != root) {
        s.role[w] = ORC_ROLE_MEMBER_SHARED;
        if (root < cur) s.parent[w] = root;
      }
    }
  }
  /* classify_hub_outlier (scan.py:779-829) */
  for (int64_t v = 0; v < n; ++v) {
    if (s.parent[v] >= 0) continue;
    int64_t deg = off[v + 1] - off[v];
    int hub = 0;
    if (deg > 1) {
      int32_t first = -1;
      int first_shared = 0;
      for (int64_t i = off[v]; i < off[v + 1]; ++i) {
        int32_t x = adj[i];
        int32_t px = s.parent[x];
        if (px < 0) continue;
        int shared = s.role[x] == ORC_ROLE_MEMBER_SHARED;
        if (first < 0) { first = px; first_shared = shared; }
        else if (first_shared || shared || px != first) { hub = 1; break; }
      }
    }
    if (hub) { s.parent[v] = -1; s.role[v] = ORC_ROLE_HUB; }
    else { s.parent[v] = -2; s.role[v] = ORC_ROLE_OUTLIER; }
  }
  for (int64_t v = 0; v < n; ++v) {                /* build_result 950-962 */
    role_out[v] = s.role[v];
    cluster_out[v] = s.parent[v] >= 0 ? s.parent[v] : -1;
  }
  free(s.lower); free(s.upper); free(s.parent); free(s.height); free(s.role); free(s.sim);
  return 0;
fail:
  free(s.lower); free(s.upper); free(s.parent); free(s.height); free(s.role); free(s.sim);
  return -2;
}

/* ------------------------------------------------------------------------ */
/* CPU baseline: the hot loop (_eval_edge) over a bounded edge sample.       */

typedef struct sample_ctx {
  const int64_t* off; const int32_t* adj; const int32_t* el; orc_eps2 e;
  const int64_t* sample; int64_t probes[256], similar[256];
} sample_ctx;

static void sample_body(int64_t lo, int64_t hi, void* p, int tid) {
  sample_ctx* c = (sample_ctx*)p;
  int64_t pr_tot = 0, sim_tot = 0;
  for (int64_t i = lo; i < hi; ++i) {
    int64_t k = c->sample[i];
    int32_t a = c->el[2 * k], b = c->el[2 * k + 1];
    int64_t pr;
    sim_tot += eval_edge(c->adj, c->off[a], c->off[a + 1], c->off[b], c->off[b + 1], c->e, &pr);
    pr_tot += pr;
  }
  c->probes[tid] += pr_tot;
  c->similar[tid] += sim_tot;
}

double orc_sample_eval(int64_t n, int64_t m, const int64_t* off,
                       const int32_t* adj, const int32_t* el, orc_eps2 eps2,
                       const int64_t* sample, int64_t count, int threads,
                       int64_t* probes, int64_t* similar) {
  (void)n; (void)m;
  sample_ctx* c = (sample_ctx*)calloc(1, sizeof(sample_ctx));
  c->off = off; c->adj = adj; c->el = el; c->e = eps2; c->sample = sample;
  double t0 = now_s();
  par_for(count, 64, threads, sample_body, c);
  double t1 = now_s();
  int64_t pr = 0, sm = 0;
  for (int t = 0; t < 256; ++t) { pr += c->probes[t]; sm += c->similar[t]; }
  *probes = pr;
  *similar = sm;
  free(c);
  return t1 - t0;
}

void orc_set_threads(int threads) { g_threads = threads; }

/* ------------------------------------------------------------------------ */
/* Parallel CSR-only build (offsets + sorted runs) for large CPU baselines.  */
/* Same arrays as orc_build_graph's first two outputs (graph.py:184-216).   */

typedef struct csr_ctx {
  const int32_t *eu, *ev; int64_t* deg; int64_t* cur; int32_t* adj; const int64_t* off;
} csr_ctx;

static void csr_count_body(int64_t lo, int64_t hi, void* p, int tid) {
  (void)tid;
  csr_ctx* c = (csr_ctx*)p;
  for (int64_t k = lo; k < hi; ++k) {
    __atomic_fetch_add(&c->deg[c->eu[k]], 1, __ATOMIC_RELAXED);
    __atomic_fetch_add(&c->deg[c->ev[k]], 1, __ATOMIC_RELAXED);
  }
}

static void csr_fill_body(int64_t lo, int64_t hi, void* p, int tid) {
  (void)tid;
  csr_ctx* c = (csr_ctx*)p;
  for (int64_t k = lo; k < hi; ++k) {
    int32_t u = c->eu[k], v = c->ev[k];
    c->adj[__atomic_fetch_add(&c->cur[u], 1, __ATOMIC_RELAXED)] = v;
    c->adj[__atomic_fetch_add(&c->cur[v], 1, __ATOMIC_RELAXED)] = u;
  }
}

static int cmp_i32(const void* x, const void* y) {
  int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
  return (a > b) - (a < b);
}

static void csr_sort_body(int64_t lo, int64_t hi, void* p, int tid) {
  (void)tid;
  csr_ctx* c = (csr_ctx*)p;
  for (int64_t u = lo; u < hi; ++u) {
    int64_t a = c->off[u], b = c->off[u + 1];
    if (b - a > 1) qsort(c->adj + a, (size_t)(b - a), sizeof(int32_t), cmp_i32);
  }
}

int orc_build_csr(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev,
                  int64_t* offsets, int32_t* adjacency) {
  csr_ctx c;
  c.eu = eu; c.ev = ev; c.adj = adjacency; c.off = offsets;
  c.deg = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
  c.cur = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  for (int64_t k = 0; k < m; ++k)
    if (eu[k] < 0 || ev[k] < 0 || eu[k] >= n || ev[k] >= n || eu[k] == ev[k]) {
      free(c.deg); free(c.cur); return -1;
    }
  par_for(m, 1 << 16, 0, csr_count_body, &c);
  int64_t tot = 0;
  for (int64_t u = 0; u < n; ++u) { offsets[u] = tot; c.cur[u] = tot; tot += c.deg[u]; }
  offsets[n] = tot;
  par_for(m, 1 << 16, 0, csr_fill_body, &c);
  par_for(n, 4096, 0, csr_sort_body, &c);
  free(c.deg); free(c.cur);
  return 0;
}

/* _eval_edge over edges sampled as uniform adjacency slots, oriented by
 * (degree, id) like build_graph's edge array (graph.py:226). */
typedef struct slot_ctx {
  int64_t n; const int64_t* off; const int32_t* adj; orc_eps2 e; const int64_t* slots;
  int64_t probes[256], similar[256];
} slot_ctx;

static void slot_body(int64_t lo, int64_t hi, void* p, int tid) {
  slot_ctx* c = (slot_ctx*)p;
  int64_t pr_tot = 0, sim_tot = 0;
  for (int64_t i = lo; i < hi; ++i) {
    int64_t s = c->slots[i];
    int64_t l = 0, h = c->n;           /* owner: last u with off[u] <= s */
    while (h - l > 1) { int64_t mid = (l + h) >> 1; if (c->off[mid] <= s) l = mid; else h = mid; }
    int32_t a = (int32_t)l, b = c->adj[s];
    int64_t da = c->off[a + 1] - c->off[a], db = c->off[b + 1] - c->off[b];
    if (db < da || (db == da && b < a)) { int32_t t = a; a = b; b = t; }
    int64_t pr;
    sim_tot += eval_edge(c->adj, c->off[a], c->off[a + 1], c->off[b], c->off[b + 1], c->e, &pr);
    pr_tot += pr;
  }
  c->probes[tid] += pr_tot;
  c->similar[tid] += sim_tot;
}

double orc_sample_eval_slots(int64_t n, const int64_t* off, const int32_t* adj, orc_eps2 eps2,
                             const int64_t* slots, int64_t count, int threads, int64_t* probes,
                             int64_t* similar) {
  slot_ctx* c = (slot_ctx*)calloc(1, sizeof(slot_ctx));
  c->n = n; c->off = off; c->adj = adj; c->e = eps2; c->slots = slots;
  double t0 = now_s();
  par_for(count, 64, threads, slot_body, c);
  double t1 = now_s();
  int64_t pr = 0, sm = 0;
  for (int t = 0; t < 256; ++t) { pr += c->probes[t]; sm += c->similar[t]; }
  *probes = pr; *similar = sm;
  free(c);
  return t1 - t0;
}
