// Integer preprocessing of the HongTu path, native and bit-exact with the
// reference (graph.py / partition.py / planner.py of chunktrain).
//
// Everything here is deterministic sequential or order-preserving code:
// counting sorts instead of comparison sorts (stable, so duplicate edges
// keep input order exactly like numpy's lexsort), merge-based set algebra,
// and the LDG scores evaluated with the same IEEE double operations as the
// numpy expression they restate.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include <omp.h>

#include "ht_common.h"

namespace ht {
std::string& last_error() {
  static thread_local std::string s;
  return s;
}
}  // namespace ht

using ht::fail;

extern "C" const char* ht_last_error(void) { return ht::last_error().c_str(); }
extern "C" int ht_version(void) { return 1; }

namespace {

// Edge positions grouped by key (stable, original order inside a group):
// one counting scatter.  Returns the group offsets.
void group_by(const int64_t* key, int64_t E, int64_t K, std::vector<int64_t>& out,
              std::vector<int64_t>& off) {
  off.assign(K + 1, 0);
  for (int64_t e = 0; e < E; ++e) off[key[e] + 1]++;
  for (int64_t k = 0; k < K; ++k) off[k + 1] += off[k];
  std::vector<int64_t> cur(off.begin(), off.end() - 1);
  out.resize(E);
  for (int64_t e = 0; e < E; ++e) out[cur[key[e]]++] = e;
}

// Inside every group, order positions by (key2, position): a stable sort
// on key2.  Groups are small (degrees), so this is cache friendly and runs
// group-parallel.
void sort_groups(std::vector<int64_t>& pos, const std::vector<int64_t>& off, const int64_t* key2) {
  const int64_t G = (int64_t)off.size() - 1;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t g = 0; g < G; ++g) {
    int64_t* b = pos.data() + off[g];
    int64_t* e = pos.data() + off[g + 1];
    if (e - b < 2) continue;
    bool sorted = true;
    for (int64_t* q = b + 1; q < e; ++q)
      if (key2[*(q - 1)] > key2[*q]) { sorted = false; break; }
    if (!sorted) std::stable_sort(b, e, [&](int64_t x, int64_t y) { return key2[x] < key2[y]; });
  }
}

}  // namespace

// graph.py:91-150 (from_edges + gcn_edge_weights)
extern "C" int ht_build_graph(const int64_t* src, const int64_t* dst, int64_t E, int64_t V,
                              int64_t* csc_offsets, int64_t* csc_sources, int64_t* csr_offsets,
                              int64_t* csr_targets, int64_t* csr_edge_perm, double* weights) {
  if (E < 0 || V < 0) return fail(HT_EINVAL, "negative graph size");
  int bad = 0;
#pragma omp parallel for reduction(| : bad)
  for (int64_t e = 0; e < E; ++e)
    bad |= (src[e] < 0 || dst[e] < 0 || src[e] >= V || dst[e] >= V);
  if (bad) return fail(HT_EINVAL, "an edge references a vertex outside [0, %lld)", (long long)V);
  // canonical order: by (dst, src), ties by input position
  bool canonical = true;
  for (int64_t e = 1; e < E && canonical; ++e)
    canonical = dst[e - 1] < dst[e] || (dst[e - 1] == dst[e] && src[e - 1] <= src[e]);
  std::vector<int64_t> a, off;
  if (canonical) {
    a.resize(E);
    std::iota(a.begin(), a.end(), 0);
    off.assign(V + 1, 0);
    for (int64_t e = 0; e < E; ++e) off[dst[e] + 1]++;
    for (int64_t v = 0; v < V; ++v) off[v + 1] += off[v];
  } else {
    group_by(dst, E, V, a, off);
    sort_groups(a, off, src);
  }
  std::memcpy(csc_offsets, off.data(), (V + 1) * sizeof(int64_t));
  std::vector<int64_t> canon_rank(E);
#pragma omp parallel for
  for (int64_t p = 0; p < E; ++p) {
    csc_sources[p] = src[a[p]];
    canon_rank[a[p]] = p;
  }
  std::vector<double> inv(V);
#pragma omp parallel for
  for (int64_t v = 0; v < V; ++v) inv[v] = 1.0 / std::sqrt(1.0 + (double)(off[v + 1] - off[v]));
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < V; ++v)
    for (int64_t p = off[v]; p < off[v + 1]; ++p) weights[p] = inv[csc_sources[p]] * inv[v];
  // CSR: canonical positions grouped by source keep (dst, position) order
  std::vector<int64_t> cnt(V + 1, 0);
  for (int64_t p = 0; p < E; ++p) cnt[csc_sources[p] + 1]++;
  for (int64_t v = 0; v < V; ++v) cnt[v + 1] += cnt[v];
  std::memcpy(csr_offsets, cnt.data(), (V + 1) * sizeof(int64_t));
  for (int64_t v = 0; v < V; ++v)
    for (int64_t p = off[v]; p < off[v + 1]; ++p) {
      const int64_t q = cnt[csc_sources[p]]++;
      csr_targets[q] = v;
      csr_edge_perm[q] = p;
    }
  return HT_OK;
}

// ---------------------------------------------------------------------------
// partition.py:102-209  LDG streaming partition + refinement + repair
// ---------------------------------------------------------------------------
namespace {

struct Adj {
  const int64_t *co, *cs, *ro, *rt;
  // visit every undirected neighbour of v (in-edges then out-edges, self
  // loops dropped; duplicates kept, partition.py:102-120)
  template <class F>
  void each(int64_t v, F&& f) const {
    for (int64_t p = co[v]; p < co[v + 1]; ++p)
      if (cs[p] != v) f(cs[p]);
    for (int64_t p = ro[v]; p < ro[v + 1]; ++p)
      if (rt[p] != v) f(rt[p]);
  }
};

void repair_empty(std::vector<int64_t>& sizes, int64_t* owner, int64_t V,
                  const std::vector<int64_t>& adeg) {
  const int64_t m = (int64_t)sizes.size();
  for (;;) {
    int64_t empty = -1;
    for (int64_t p = 0; p < m; ++p)
      if (sizes[p] == 0) { empty = p; break; }
    if (empty < 0) return;
    int64_t donor = 0;
    for (int64_t p = 1; p < m; ++p)
      if (sizes[p] > sizes[donor]) donor = p;
    int64_t best = -1;
    for (int64_t v = 0; v < V; ++v)
      if (owner[v] == donor && (best < 0 || adeg[v] < adeg[best])) best = v;
    owner[best] = empty;
    sizes[donor]--;
    sizes[empty]++;
  }
}

}  // namespace

// CSR -> canonical permutation of a graph given by its CSC (sorted by
// (dst, src)): CSR position k holds canonical edge perm[k], the CSR order
// being by (src, dst) with ties in canonical order - what
// np.lexsort((dst, csc_sources)) gives (graph.py:117).  One counting pass
// over the canonical edges (O(E), no sort): used when an HTG1 cache is
// loaded (graph.py:224-266).
extern "C" int ht_csr_perm(int64_t V, int64_t E, const int64_t* csc_offsets,
                           const int64_t* csc_sources, const int64_t* csr_offsets,
                           int64_t* perm) {
  if (V < 0 || E < 0) return ht::fail(HT_EINVAL, "negative sizes");
  if (csc_offsets[V] != E || csr_offsets[V] != E)
    return ht::fail(HT_EINVAL, "offsets do not end at the edge count");
  std::vector<int64_t> cur(csr_offsets, csr_offsets + V);
  for (int64_t v = 0; v < V; ++v)
    for (int64_t e = csc_offsets[v]; e < csc_offsets[v + 1]; ++e) {
      const int64_t u = csc_sources[e];
      if (u < 0 || u >= V) return ht::fail(HT_EINVAL, "source id out of range");
      const int64_t k = cur[u]++;
      if (k >= csr_offsets[u + 1]) return ht::fail(HT_EINVAL, "CSR offsets inconsistent with CSC");
      perm[k] = e;
    }
  return HT_OK;
}

extern "C" int ht_ldg_partition(int64_t V, const int64_t* csc_offsets, const int64_t* csc_sources,
                                const int64_t* csr_offsets, const int64_t* csr_targets,
                                const int64_t* arrival, int64_t m, int64_t cap, int64_t* owner) {
  if (m < 1 || m > V) return fail(HT_EINVAL, "m=%lld outside [1, V]", (long long)m);
  if (m == 1) {  // every choice is partition 0; refinement and repair are no-ops
    std::fill(owner, owner + V, (int64_t)0);
    return HT_OK;
  }
  Adj adj{csc_offsets, csc_sources, csr_offsets, csr_targets};
  std::vector<int64_t> adeg(V, 0);
  for (int64_t v = 0; v < V; ++v) adj.each(v, [&](int64_t) { adeg[v]++; });
  std::fill(owner, owner + V, (int64_t)-1);
  std::vector<int64_t> sizes(m, 0), cnt(m);
  const double dcap = (double)cap;
  for (int64_t t = 0; t < V; ++t) {
    const int64_t v = arrival[t];
    std::fill(cnt.begin(), cnt.end(), 0);
    adj.each(v, [&](int64_t u) {
      if (owner[u] >= 0) cnt[owner[u]]++;
    });
    // pick the eligible partition minimising (-score, size, id)
    int64_t pick = -1;
    double best_neg = 0.0;
    for (int64_t p = 0; p < m; ++p) {
      if (sizes[p] >= cap) continue;
      const double score = (double)cnt[p] * (1.0 - (double)sizes[p] / dcap);
      const double neg = -score;
      if (pick < 0 || neg < best_neg || (neg == best_neg && sizes[p] < sizes[pick])) {
        pick = p;
        best_neg = neg;
      }
    }
    if (pick < 0) return fail(HT_EINVAL, "no partition below capacity");
    owner[v] = pick;
    sizes[pick]++;
  }
  repair_empty(sizes, owner, V, adeg);
  // one refinement sweep, ascending vertex id
  for (int64_t v = 0; v < V; ++v) {
    if (adeg[v] == 0) continue;
    const int64_t cur = owner[v];
    if (sizes[cur] <= 1) continue;
    std::fill(cnt.begin(), cnt.end(), 0);
    adj.each(v, [&](int64_t u) { cnt[owner[u]]++; });
    int64_t best = 0, best_val = 0;
    for (int64_t p = 0; p < m; ++p) {
      const int64_t val = (p == cur || sizes[p] < cap) ? cnt[p] : -1;
      if (p == 0 || val > best_val) {
        best = p;
        best_val = val;
      }
    }
    if (best != cur && best_val > cnt[cur]) {
      owner[v] = best;
      sizes[cur]--;
      sizes[best]++;
    }
  }
  repair_empty(sizes, owner, V, adeg);
  return HT_OK;
}

// partition.py:235-267
extern "C" int ht_chunk_fill(const int64_t* csc_offsets, const int64_t* csc_sources,
                             const double* weights, const int64_t* verts, int64_t nv,
                             int64_t* sources, int64_t* n_sources, int64_t* csc_off,
                             int64_t* csc_local_src, double* edge_w, int64_t* csr_off,
                             int64_t* csr_local_dst, int64_t* csr_perm) {
  csc_off[0] = 0;
  for (int64_t k = 0; k < nv; ++k) {
    const int64_t v = verts[k];
    csc_off[k + 1] = csc_off[k] + (csc_offsets[v + 1] - csc_offsets[v]);
  }
  const int64_t ne = csc_off[nv];
  int64_t vmax = -1;
#pragma omp parallel for reduction(max : vmax) schedule(dynamic, 1024)
  for (int64_t k = 0; k < nv; ++k) {
    const int64_t v = verts[k], base = csc_offsets[v];
    for (int64_t q = csc_off[k]; q < csc_off[k + 1]; ++q) {
      const int64_t u = csc_sources[base + (q - csc_off[k])];
      csc_local_src[q] = u;  // global id for now
      edge_w[q] = weights[base + (q - csc_off[k])];
      vmax = std::max(vmax, u);
    }
  }
  int64_t nn = 0;
  if (ne > 0 && vmax + 1 <= 8 * ne) {
    // dense id map: mark, prefix-sum, translate
    std::vector<int32_t> map(vmax + 1, 0);
#pragma omp parallel for
    for (int64_t q = 0; q < ne; ++q) map[csc_local_src[q]] = 1;
    for (int64_t u = 0; u <= vmax; ++u)
      if (map[u]) { sources[nn] = u; map[u] = (int32_t)nn++; }
#pragma omp parallel for
    for (int64_t q = 0; q < ne; ++q) csc_local_src[q] = map[csc_local_src[q]];
  } else if (ne > 0) {
    std::vector<int64_t> uniq(csc_local_src, csc_local_src + ne);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    nn = (int64_t)uniq.size();
    std::memcpy(sources, uniq.data(), nn * sizeof(int64_t));
#pragma omp parallel for
    for (int64_t q = 0; q < ne; ++q)
      csc_local_src[q] = std::lower_bound(uniq.begin(), uniq.end(), csc_local_src[q]) - uniq.begin();
  }
  *n_sources = nn;
  std::vector<int64_t> cnt(nn + 1, 0);
  for (int64_t q = 0; q < ne; ++q) cnt[csc_local_src[q] + 1]++;
  for (int64_t u = 0; u < nn; ++u) cnt[u + 1] += cnt[u];
  std::memcpy(csr_off, cnt.data(), (nn + 1) * sizeof(int64_t));
  // stable by local source over canonical order == lexsort((dst, src))
  for (int64_t k = 0; k < nv; ++k)
    for (int64_t q = csc_off[k]; q < csc_off[k + 1]; ++q) {
      const int64_t pos = cnt[csc_local_src[q]]++;
      csr_perm[pos] = q;
      csr_local_dst[pos] = k;
    }
  return HT_OK;
}

// ---------------------------------------------------------------------------
// planner.py:45-63 sorted-set primitives, 252-284 layout, 386-450 reorganize
// ---------------------------------------------------------------------------

extern "C" int ht_set_op(int op, const int64_t* a, int64_t na, const int64_t* b, int64_t nb,
                         int64_t* out, int64_t* n_out) {
  int64_t* e;
  switch (op) {
    case 0: e = std::set_intersection(a, a + na, b, b + nb, out); break;
    case 1: e = std::set_difference(a, a + na, b, b + nb, out); break;
    case 2: e = std::set_union(a, a + na, b, b + nb, out); break;
    default: return fail(HT_EINVAL, "unknown set op %d", op);
  }
  *n_out = e - out;
  return HT_OK;
}

extern "C" int64_t ht_intersect_count(const int64_t* a, int64_t na, const int64_t* b,
                                      int64_t nb) {
  int64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (b[j] < a[i]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

// Stable slots: rows live in consecutive batches keep their slot; new rows
// (ascending id) take the free slots in ascending order, then fresh ones.
// The reference's min-heap of evicted slots always holds exactly the slots
// below the high-water mark not held by a carried row, so rank/select over
// that complement reproduces it.
extern "C" int ht_slot_layout(int64_t n, const int64_t* live, const int64_t* off,
                              int64_t* slots, int64_t* capacity) {
  int64_t top = 0;
  std::vector<char> held;
  for (int64_t j = 0; j < n; ++j) {
    const int64_t lo = off[j], hi = off[j + 1];
    held.assign(top, 0);
    int64_t fresh = 0;
    if (j > 0) {
      const int64_t plo = off[j - 1], phi = off[j];
      int64_t p = plo;
      for (int64_t q = lo; q < hi; ++q) {
        while (p < phi && live[p] < live[q]) ++p;
        if (p < phi && live[p] == live[q]) {
          slots[q] = slots[p];
          held[slots[q]] = 1;
        } else {
          slots[q] = -1;
          ++fresh;
        }
      }
    } else {
      for (int64_t q = lo; q < hi; ++q) slots[q] = -1;
      fresh = hi - lo;
    }
    int64_t scan = 0;
    for (int64_t q = lo; q < hi; ++q) {
      if (slots[q] >= 0) continue;
      while (scan < top && held[scan]) ++scan;
      if (scan < top) {
        slots[q] = scan++;
      } else {
        slots[q] = top++;
        scan = top;
      }
    }
    (void)fresh;
  }
  *capacity = top;
  return HT_OK;
}

extern "C" int ht_reorganize(int64_t m, int64_t n, const int64_t* nbr, const int64_t* off,
                             int move_all_rows, int64_t* chunk_orders, int64_t* batch_order) {
  auto set = [&](int64_t i, int64_t j) {
    const int64_t id = i * n + j;
    return std::make_pair(nbr + off[id], off[id + 1] - off[id]);
  };
  std::vector<std::vector<int64_t>> acc(n);
  for (int64_t j = 0; j < n; ++j) {
    auto s = set(0, j);
    acc[j].assign(s.first, s.first + s.second);
    chunk_orders[j] = j;
  }
  std::vector<int64_t> tmp;
  for (int64_t i = 1; i < m; ++i) {
    std::vector<int64_t> left(n);
    std::iota(left.begin(), left.end(), 0);
    for (int64_t j = 0; j < n; ++j) {
      int64_t best = 0, best_score = -1;
      for (size_t t = 0; t < left.size(); ++t) {
        auto s = set(i, left[t]);
        const int64_t sc = ht_intersect_count(s.first, s.second, acc[j].data(), acc[j].size());
        if (sc > best_score) { best_score = sc; best = (int64_t)t; }
      }
      const int64_t k = left[best];
      left.erase(left.begin() + best);
      chunk_orders[i * n + j] = k;
      auto s = set(i, k);
      tmp.resize(acc[j].size() + s.second);
      tmp.resize(std::set_union(acc[j].begin(), acc[j].end(), s.first, s.first + s.second,
                                tmp.begin()) - tmp.begin());
      acc[j].swap(tmp);
    }
  }
  std::vector<int64_t> left(n > 0 ? n - 1 : 0);
  std::iota(left.begin(), left.end(), 1);
  if (n > 0) batch_order[0] = 0;
  for (int64_t pos = 1; pos < n; ++pos) {
    const auto& prev = acc[batch_order[pos - 1]];
    int64_t best = 0, best_score = -1;
    for (size_t t = 0; t < left.size(); ++t) {
      const auto& u = acc[left[t]];
      const int64_t sc = ht_intersect_count(u.data(), u.size(), prev.data(), prev.size());
      if (sc > best_score) { best_score = sc; best = (int64_t)t; }
    }
    batch_order[pos] = left[best];
    left.erase(left.begin() + best);
  }
  // rows are emitted in batch order (row 0 optionally kept in place)
  std::vector<int64_t> row(n);
  for (int64_t i = 0; i < m; ++i) {
    if (i == 0 && !move_all_rows) continue;
    for (int64_t b = 0; b < n; ++b) row[b] = chunk_orders[i * n + batch_order[b]];
    std::copy(row.begin(), row.end(), chunk_orders + i * n);
  }
  return HT_OK;
}

// synth.py:154-157: indices of the first occurrence of every distinct
// (dst, src) pair, in ascending (dst, src) order - np.unique(dst*V+src,
// return_index=True) without the 64-bit comparison sort.
extern "C" int ht_dedup_edges(const int64_t* src, const int64_t* dst, int64_t E, int64_t V,
                              int64_t* keep, int64_t* n_keep) {
  int bad = 0;
#pragma omp parallel for reduction(| : bad)
  for (int64_t e = 0; e < E; ++e)
    bad |= (src[e] < 0 || dst[e] < 0 || src[e] >= V || dst[e] >= V);
  if (bad) return fail(HT_EINVAL, "an edge lies outside [0, %lld)", (long long)V);
  std::vector<int64_t> a, off;
  group_by(dst, E, V, a, off);
  sort_groups(a, off, src);
  int64_t k = 0;
  for (int64_t p = 0; p < E; ++p) {
    const int64_t e = a[p];
    if (p > 0) {
      const int64_t q = a[p - 1];
      if (src[q] == src[e] && dst[q] == dst[e]) continue;
    }
    keep[k++] = e;
  }
  *n_keep = k;
  return HT_OK;
}

// ---------------------------------------------------------------------------
// Lean graph build for 10^9-edge synthetic graphs (synth.synth_graph_streaming):
// 32-bit (src, dst) pairs in, parallel edges removed, canonical CSC / CSR /
// weights out - the same arrays as ht_dedup_edges + ht_build_graph
// (graph.py:91-150, synth.py:154-157) without their 64-bit temporaries:
// one counting sort by destination straight into csc_sources, a sort +
// unique per destination, one counting sort by source for the CSR.  Peak
// memory ~ the 8-byte inputs + the 32-byte/edge outputs.  Outputs are sized
// for E edges; *e_out receives the edge count after deduplication.
// ---------------------------------------------------------------------------
extern "C" int ht_build_graph_dedup32(const int32_t* src, const int32_t* dst, int64_t E, int64_t V,
                                      int64_t* csc_offsets, int64_t* csc_sources,
                                      int64_t* csr_offsets, int64_t* csr_targets,
                                      int64_t* csr_edge_perm, double* weights, int64_t* e_out) {
  if (E < 0 || V < 0 || V >= ((int64_t)1 << 31)) return fail(HT_EINVAL, "bad graph size");
  int bad = 0;
#pragma omp parallel for reduction(| : bad)
  for (int64_t e = 0; e < E; ++e)
    bad |= (src[e] < 0 || dst[e] < 0 || src[e] >= V || dst[e] >= V);
  if (bad) return fail(HT_EINVAL, "an edge lies outside [0, %lld)", (long long)V);
  // counting sort by destination: csc_offsets = bucket starts
  std::vector<int64_t> pos(V + 1, 0);
  for (int64_t e = 0; e < E; ++e) pos[dst[e] + 1]++;
  for (int64_t v = 0; v < V; ++v) pos[v + 1] += pos[v];
  std::vector<int64_t> start(pos.begin(), pos.end());
  for (int64_t e = 0; e < E; ++e) csc_sources[pos[dst[e]]++] = src[e];
  // sort + unique each destination's sources, compact in place
  std::vector<int64_t> cnt(V, 0);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < V; ++v) {
    int64_t* b = csc_sources + start[v];
    const int64_t n = start[v + 1] - start[v];
    std::sort(b, b + n);
    cnt[v] = std::unique(b, b + n) - b;
  }
  int64_t k = 0;
  csc_offsets[0] = 0;
  for (int64_t v = 0; v < V; ++v) {  // (sequential compaction: ranges move left only)
    if (k != start[v]) std::memmove(csc_sources + k, csc_sources + start[v], cnt[v] * sizeof(int64_t));
    k += cnt[v];
    csc_offsets[v + 1] = k;
  }
  const int64_t Ed = k;
  std::vector<double> inv(V);
#pragma omp parallel for
  for (int64_t v = 0; v < V; ++v)
    inv[v] = 1.0 / std::sqrt(1.0 + (double)(csc_offsets[v + 1] - csc_offsets[v]));
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < V; ++v)
    for (int64_t p = csc_offsets[v]; p < csc_offsets[v + 1]; ++p)
      weights[p] = inv[csc_sources[p]] * inv[v];
  // CSR by (src, dst): canonical positions grouped by source, in position order
  std::fill(pos.begin(), pos.end(), 0);
  for (int64_t p = 0; p < Ed; ++p) pos[csc_sources[p] + 1]++;
  for (int64_t v = 0; v < V; ++v) pos[v + 1] += pos[v];
  std::memcpy(csr_offsets, pos.data(), (V + 1) * sizeof(int64_t));
  for (int64_t v = 0; v < V; ++v)
    for (int64_t p = csc_offsets[v]; p < csc_offsets[v + 1]; ++p) {
      const int64_t q = pos[csc_sources[p]]++;
      csr_targets[q] = v;
      csr_edge_perm[q] = p;
    }
  *e_out = Ed;
  return HT_OK;
}
