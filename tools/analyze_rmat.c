// Workload analysis for kernel design (not part of the product or tests).
// Usage: analyze_rmat <scale> [seed] [samples]
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <stdint.h>
#include "../oracle/gscan_oracle.h"

static int64_t* g_deg;
static int cmp_rank(const void* x, const void* y) {
  int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
  if (g_deg[a] != g_deg[b]) return g_deg[a] < g_deg[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}
static int cmp_i32(const void* x, const void* y) {
  int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
  return a < b ? -1 : (a > b);
}
static uint64_t rng = 88172645463325252ull;
static uint64_t xr(void) { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; }

int main(int argc, char** argv) {
  int s = argc > 1 ? atoi(argv[1]) : 20;
  uint64_t seed = argc > 2 ? strtoull(argv[2], 0, 10) : 1;
  int64_t nsamp = argc > 3 ? atoll(argv[3]) : 200000;
  int64_t n = 1ll << s, cnt = 16ll << s;
  int32_t* su = malloc(cnt * 4); int32_t* sv = malloc(cnt * 4);
  orc_rmat_edges(s, 16, seed, 0, cnt, su, sv);
  int64_t m = orc_normalize(cnt, su, sv);
  int64_t* deg = calloc(n, 8);
  for (int64_t k = 0; k < m; ++k) { deg[su[k]]++; deg[sv[k]]++; }
  int64_t dmax = 0, iso = 0;
  for (int64_t v = 0; v < n; ++v) { if (deg[v] > dmax) dmax = deg[v]; if (!deg[v]) iso++; }
  printf("scale %d n %lld m %lld dmax %lld isolated %lld\n", s, (long long)n, (long long)m, (long long)dmax, (long long)iso);
  // rank relabel
  int32_t* perm = malloc(n * 4); for (int64_t v = 0; v < n; ++v) perm[v] = v;
  g_deg = deg; qsort(perm, n, 4, cmp_rank);
  int32_t* rk = malloc(n * 4); for (int64_t r = 0; r < n; ++r) rk[perm[r]] = r;
  int64_t* off = calloc(n + 1, 8);
  for (int64_t r = 0; r < n; ++r) off[r + 1] = off[r] + deg[perm[r]];
  int32_t* adj = malloc(2 * m * 4); int64_t* cur = malloc(n * 8); memcpy(cur, off, n * 8);
  for (int64_t k = 0; k < m; ++k) { int32_t a = rk[su[k]], b = rk[sv[k]]; adj[cur[a]++] = b; adj[cur[b]++] = a; }
  for (int64_t r = 0; r < n; ++r) qsort(adj + off[r], off[r + 1] - off[r], 4, cmp_i32);
  free(su); free(sv);
  // classes of big side
  const int64_t th[] = {0, 32, 256, 1024, 4096, 16384, 28000, 65536, 1ll << 40};
  const int NT = 8;
  double wk[16] = {0}, ec[16] = {0}; int64_t vc[16] = {0};
  double sum_min = 0, sum_plus = 0;
  int64_t* dplus = calloc(n, 8);
  for (int64_t b = 0; b < n; ++b) {
    int64_t db = off[b + 1] - off[b];
    int cls = 0; while (cls < NT - 1 && db >= th[cls + 1]) cls++;
    vc[cls]++;
    for (int64_t i = off[b]; i < off[b + 1]; ++i) {
      int32_t a = adj[i];
      if (a >= b) break;
      int64_t da = off[a + 1] - off[a];
      wk[cls] += da; ec[cls] += 1; sum_min += da; dplus[a]++;
    }
  }
  for (int c = 0; c < NT; ++c)
    printf("  big-side d in [%lld,%lld): vertices %lld  edges %.3g (%.1f%%)  sum min(d) %.3g (%.1f%%)\n",
           (long long)th[c], (long long)th[c + 1], (long long)vc[c], ec[c], 100 * ec[c] / m, wk[c], 100 * wk[c] / sum_min);
  printf("sum min(d) = %.4g  (x4B = %.3f TB)\n", sum_min, 4 * sum_min / 1e12);
  // triangle-listing work
  double wtri = 0, wtri2 = 0; int64_t dpmax = 0;
  for (int64_t b = 0; b < n; ++b) if (dplus[b] > dpmax) dpmax = dplus[b];
  for (int64_t b = 0; b < n; ++b)
    for (int64_t i = off[b]; i < off[b + 1]; ++i) {
      int32_t a = adj[i]; if (a >= b) break;
      wtri += dplus[a] < dplus[b] ? dplus[a] : dplus[b];
      wtri2 += dplus[a] + dplus[b];
    }
  printf("oriented out-degree max %lld; triangle work sum min(d+) %.4g, merge sum(d+) %.4g\n", (long long)dpmax, wtri, wtri2);
  // O(1) bounds and sampled intersection statistics per eps
  double epss[] = {0.2, 0.3, 0.4, 0.5, 0.6, 0.8};
  for (int ie = 0; ie < 6; ++ie) {
    double e2 = epss[ie] * epss[ie];
    double dec_dis = 0, dec_sim = 0, wint = 0;
    for (int64_t b = 0; b < n; ++b) {
      int64_t db = off[b + 1] - off[b];
      for (int64_t i = off[b]; i < off[b + 1]; ++i) {
        int32_t a = adj[i]; if (a >= b) break;
        int64_t da = off[a + 1] - off[a];
        double D = (double)(da + 1) * (db + 1);
        double cmax = da - 1;   // |N(a) ∩ N(b)| <= da-1
        if ((cmax + 2) * (cmax + 2) < e2 * D) dec_dis++;
        else if (4.0 >= e2 * D) dec_sim++;
        else wint += da;
      }
    }
    printf("eps %.1f: O(1)-dissimilar %.1f%%  O(1)-similar %.1f%%  needs-intersection sum min(d) %.3g (%.1f%%)\n",
           epss[ie], 100 * dec_dis / m, 100 * dec_sim / m, wint, 100 * wint / sum_min);
  }
  // sample edges uniformly among those needing intersection at eps=.5: early-exit work
  for (int ie = 0; ie < 6; ie += 3) {
    double e2 = epss[ie] * epss[ie];
    double full = 0, asc = 0, desc = 0, sims = 0, tot = 0;
    double hubfrac[4] = {0}, hubscan[4] = {0};
    for (int64_t t = 0; t < nsamp; ) {
      int64_t slot = xr() % (2 * m);
      int64_t lo = 0, hi = n;  // owner of slot: last v with off[v] <= slot
      while (hi - lo > 1) { int64_t mid = (lo + hi) / 2; if (off[mid] <= slot) lo = mid; else hi = mid; }
      int64_t b = lo; int32_t a = adj[slot];
      if (a > b) { int64_t t2 = a; a = (int32_t)b; b = t2; }
      int64_t db = off[b + 1] - off[b];
      int64_t da = off[a + 1] - off[a];
      double D = (double)(da + 1) * (db + 1);
      if ((da + 1.0) * (da + 1.0) < e2 * D) continue;
      if (4.0 >= e2 * D) continue;
      ++t;
      // need c >= cmin
      int64_t cmin = (int64_t)ceil(sqrt(e2 * D) - 2.0 - 1e-9); if (cmin < 0) cmin = 0;
      // exact membership flags
      int64_t c = 0, j = off[b];
      char* hit = malloc(da);
      for (int64_t i = 0; i < da; ++i) {
        int32_t w = adj[off[a] + i];
        while (j < off[b + 1] && adj[j] < w) ++j;
        hit[i] = (j < off[b + 1] && adj[j] == w);
        c += hit[i];
      }
      int similar = c >= cmin;
      sims += similar; full += da; tot++;
      // ascending scan with early exit
      int64_t cc = 0, i;
      for (i = 0; i < da; ++i) { cc += hit[i]; if (cc >= cmin || cc + (da - 1 - i) < cmin) { ++i; break; } }
      asc += i;
      cc = 0;
      for (i = 0; i < da; ++i) { cc += hit[da - 1 - i]; if (cc >= cmin || cc + (da - 1 - i) < cmin) { ++i; break; } }
      desc += i;
      for (int r = 0; r < 4; ++r) {
        int64_t lo_rank = n - (n >> (5 + r));   /* top n/32, n/64, n/128, n/256 */
        int64_t inreg = 0, sc = 0; cc = 0;
        for (i = 0; i < da; ++i) {
          int32_t w = adj[off[a] + da - 1 - i];
          inreg += (w >= lo_rank); ++sc;
          cc += hit[da - 1 - i];
          if (cc >= cmin || cc + (da - 1 - i) < cmin) break;
        }
        hubfrac[r] += inreg; hubscan[r] += sc;
      }
      free(hit);
    }
    printf("eps %.1f sampled %lld intersect-edges: similar %.1f%%, mean da %.1f, early-exit asc %.1f%% desc %.1f%% of elements\n",
           epss[ie], (long long)nsamp, 100 * sims / tot, full / tot, 100 * asc / full, 100 * desc / full);
    for (int r = 0; r < 4; ++r)
      printf("   scanned elements (desc) inside top n/%d ranks: %.1f%%\n", 32 << r, 100 * hubfrac[r] / hubscan[r]);
  }
  return 0;
}
