// spill.cpp -- the reference's closure planner (partition.py:231-333), native.
//
// Used only when a caller asks for spill files (partition_graph(..., spill_dir)):
// the device's own out-of-core mode streams b-range slices from pinned host
// memory (ooc.cu) and never needs these partitions.  The spill files are the
// reference's GSCP format (partition.py:336-446) so the reference's
// load_partition / scan_out_of_core can read them, and so a plan's owned
// ranges, local sizes and estimates are the ones the reference computes: this
// is the same greedy, edge by edge in edge_list order, sealing when the next
// closure would overflow 25*|E_s| + 4*|V_s| + state_bytes.
//
// The one change is a shortcut that does not alter any decision: a vertex x
// whose whole closure (x, N(x), every edge at x) is already in the open
// partition adds nothing, so its list is not walked again (the reference
// walks it for every edge of x; closure(), partition.py:258-275).  Edges are
// grouped by their low endpoint, so each list is walked about once per
// partition that touches it instead of once per incident edge.
#include <stdint.h>
#include <string.h>

#include <new>
#include <vector>

#include "../../include/gscan.h"

namespace {

constexpr int64_t kEdgeBytes = 25;   // partition.py:71 EDGE_BYTES
constexpr int64_t kVertexBytes = 4;  // partition.py:72 VERTEX_BYTES

int plan_closure(int64_t n, int64_t m, const int64_t* off, const int32_t* adj,
                 const int32_t* eids, const int32_t* pairs, uint64_t budget,
                 int64_t state_bytes, int64_t* bounds, int64_t* n_local, int64_t* m_local,
                 int64_t cap, int64_t* nparts, int64_t* bad) {
  *nparts = 0;
  if (n < 0 || m < 0 || (m && (!off || !adj || !eids || !pairs))) return GS_EINVAL;
  const int64_t B = (int64_t)(budget > (uint64_t)INT64_MAX ? INT64_MAX : budget);
  std::vector<int32_t> in_v(n, -1), closed(n, -1);
  std::vector<int32_t> in_e(m, -1);
  std::vector<int64_t> tv(n, -1), te(m, -1);  // per-call "seen" stamps
  std::vector<int32_t> new_v, new_e;
  int32_t index = 0;
  int64_t call = 0, owned_lo = 0, cur_cost = 0, cur_nv = 0, cur_ne = 0, np = 0;

  auto closure = [&](int32_t u, int32_t v) {
    ++call;
    new_v.clear();
    new_e.clear();
    for (int32_t x : {u, v}) {
      if (closed[x] == index) continue;  // nothing of x's closure is new
      if (in_v[x] != index && tv[x] != call) { tv[x] = call; new_v.push_back(x); }
      for (int64_t i = off[x]; i < off[x + 1]; ++i) {
        const int32_t w = adj[i], e = eids[i];
        if (in_v[w] != index && tv[w] != call) { tv[w] = call; new_v.push_back(w); }
        if (in_e[e] != index && te[e] != call) { te[e] = call; new_e.push_back(e); }
      }
    }
    return kEdgeBytes * (int64_t)new_e.size() + kVertexBytes * (int64_t)new_v.size();
  };
  auto seal = [&](int64_t owned_hi) {
    if (np < cap) {
      bounds[np] = owned_lo;
      bounds[np + 1] = owned_hi;
      n_local[np] = cur_nv;
      m_local[np] = cur_ne;
    }
    ++np;
  };

  for (int64_t k = 0; k < m; ++k) {
    const int32_t u = pairs[2 * k], v = pairs[2 * k + 1];
    if (u < 0 || v < 0 || u >= n || v >= n || u == v) return GS_EINVAL;
    int64_t add = closure(u, v);
    if (cur_ne && cur_cost + add + state_bytes > B) {  // partition.py:282-296
      seal(k);
      ++index;
      owned_lo = k;
      cur_cost = cur_nv = cur_ne = 0;
      add = closure(u, v);
    }
    if (cur_cost + add + state_bytes > B) {  // partition.py:297-298
      bad[0] = u;
      bad[1] = v;
      bad[2] = cur_cost + add + state_bytes;
      *nparts = np;
      return GS_EBUDGET;
    }
    for (int32_t x : new_v) in_v[x] = index;
    for (int32_t e : new_e) in_e[e] = index;
    closed[u] = closed[v] = index;
    cur_nv += (int64_t)new_v.size();
    cur_ne += (int64_t)new_e.size();
    cur_cost += add;
  }
  if (cur_ne) seal(m);
  *nparts = np;
  return GS_OK;
}

}  // namespace

extern "C" int gs_plan_closure(int64_t n, int64_t m, const int64_t* offsets,
                               const int32_t* adjacency, const int32_t* edge_ids,
                               const int32_t* edge_list, uint64_t budget_bytes,
                               int64_t state_bytes, int64_t* owned_bounds, int64_t* n_local,
                               int64_t* m_local, int64_t cap, int64_t* nparts,
                               int64_t* bad_edge) {
  try {
    return plan_closure(n, m, offsets, adjacency, edge_ids, edge_list, budget_bytes,
                        state_bytes, owned_bounds, n_local, m_local, cap, nparts, bad_edge);
  } catch (const std::bad_alloc&) {
    return GS_ENOMEM;
  } catch (...) {
    return GS_EINTERNAL;
  }
}
