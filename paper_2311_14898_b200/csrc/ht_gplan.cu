// GPU dedup planner: the DedupPlan of planner.py:292-315
// computed on the device from the raw neighbour ids of every chunk.
//
//   N_ij      = unique(edge source ids of chunk (i,j))      sort + unique
//   U_j       = union_i N_ij                                  sort + unique
//   T_ij      = U_j restricted to owner i                     stable owner sort
//   carry_ij  = T_ij ^ T_i,j-1 ; load_ij = T_ij \ T_i,j-1    membership + select
//   fetch_ijk = N_ij restricted to owner k (k != i)           stable owner sort
//               (== N_ij ^ T_kj because N_ij c U_j)
//   nbrc_ij   = N_ij ^ N_i,j-1
//   live_ij   = T_ij u N_ij, slots: carried rows keep their slot, the k-th
//               new row (ascending id) takes the k-th smallest slot not held
//               by a carried row (the min-heap of planner.py:264-277 as a
//               bitmap + exclusive scan)
//
// Every set is a sorted unique int64 array in device memory; the results are
// bit-identical with the host planner (tests/test_gpu_plan.py).  Sorting is
// CUB's LSD radix sort restricted to the bits of the vertex-id range
// (stable, so owner partitions keep ascending ids).

#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "ht_common.h"

using ht::fail;

#define CUP(expr)                                                                   \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return fail(HT_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                              \
  } while (0)

namespace {

__global__ void k_member(const int64_t* __restrict__ a, int64_t na, const int64_t* __restrict__ b,
                         int64_t nb, uint8_t* __restrict__ flag, int invert) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < na;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = a[q];
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (b[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    const bool in = lo < nb && b[lo] == x;
    flag[q] = (uint8_t)(in != (invert != 0));
  }
}

__global__ void k_owner_keys(const int64_t* __restrict__ s, int64_t n, const int64_t* __restrict__ owner,
                             int32_t* __restrict__ key, int32_t* __restrict__ count) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = (int32_t)owner[s[q]];
    key[q] = o;
    atomicAdd(&count[o], 1);
  }
}

// carried rows keep their slot; fresh rows are marked -1
__global__ void k_carry_slots(const int64_t* __restrict__ live, int64_t n, const int64_t* __restrict__ prev,
                              const int64_t* __restrict__ pslot, int64_t np, int64_t* __restrict__ slot,
                              uint8_t* __restrict__ held, int32_t* __restrict__ fresh) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = live[q];
    int64_t lo = 0, hi = np;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (prev[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    if (lo < np && prev[lo] == x) {
      const int64_t s = pslot[lo];
      slot[q] = s;
      held[s] = 1;
      fresh[q] = 0;
    } else {
      slot[q] = -1;
      fresh[q] = 1;
    }
  }
}

__global__ void k_free_flags(const uint8_t* __restrict__ held, int64_t top, int64_t range,
                             int32_t* __restrict__ freef) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < range;
       s += (int64_t)gridDim.x * blockDim.x)
    freef[s] = (s >= top || !held[s]) ? 1 : 0;
}

// free slot s with exclusive rank r < nfresh becomes the r-th fresh row's slot
__global__ void k_take_free(const int32_t* __restrict__ freef, const int32_t* __restrict__ frank,
                            int64_t range, int64_t nfresh, int64_t* __restrict__ freeslot) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < range;
       s += (int64_t)gridDim.x * blockDim.x)
    if (freef[s] && frank[s] < nfresh) freeslot[frank[s]] = s;
}

__global__ void k_fill_fresh(int64_t* __restrict__ slot, const int32_t* __restrict__ fresh,
                             const int32_t* __restrict__ qrank, int64_t n,
                             const int64_t* __restrict__ freeslot) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    if (fresh[q]) slot[q] = freeslot[qrank[q]];
}

__global__ void k_iota(int64_t* __restrict__ x, int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    x[q] = q;
}

inline int grid(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

struct Set {
  int64_t* p = nullptr;
  int64_t n = 0;
};

}  // namespace

struct ht_gplan {
  int device = 0;
  int m = 0, n = 0;
  int64_t V = 0;
  cudaStream_t s = nullptr;
  int bits = 1;
  std::vector<void*> allocs;
  // scratch
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int64_t* nsel = nullptr;  // device counter for CUB select
  std::vector<Set> sets;    // in the order of ht_gplan_sizes
  std::vector<int64_t> caps;
  int64_t vol[3] = {0, 0, 0};

  ~ht_gplan() {
    cudaSetDevice(device);
    for (void* p : allocs) cudaFree(p);
    if (tmp) cudaFree(tmp);
    if (nsel) cudaFree(nsel);
    if (s) cudaStreamDestroy(s);
  }
  int alloc(void** p, int64_t bytes) {
    *p = nullptr;
    if (bytes <= 0) bytes = 8;
    CUP(cudaMalloc(p, bytes));
    allocs.push_back(*p);
    return HT_OK;
  }
  int scratch(size_t bytes) {
    if (bytes <= tmp_bytes) return HT_OK;
    if (tmp) cudaFree(tmp);
    tmp = nullptr;
    tmp_bytes = 0;
    CUP(cudaMalloc(&tmp, bytes));
    tmp_bytes = bytes;
    return HT_OK;
  }
  int64_t read_count() {
    int64_t c = 0;
    cudaMemcpyAsync(&c, nsel, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return c;
  }
  // sorted unique copy of in[0..n)
  int sort_unique(const int64_t* in, int64_t n, Set* out) {
    out->n = 0;
    HT_TRY(alloc((void**)&out->p, n * 8));
    if (n == 0) return HT_OK;
    int64_t* sorted;
    CUP(cudaMallocAsync((void**)&sorted, n * 8, s));
    size_t b1 = 0, b2 = 0;
    CUP(cub::DeviceRadixSort::SortKeys(nullptr, b1, in, sorted, n, 0, bits, s));
    CUP(cub::DeviceSelect::Unique(nullptr, b2, sorted, out->p, nsel, n, s));
    HT_TRY(scratch(std::max(b1, b2)));
    CUP(cub::DeviceRadixSort::SortKeys(tmp, b1, in, sorted, n, 0, bits, s));
    CUP(cub::DeviceSelect::Unique(tmp, b2, sorted, out->p, nsel, n, s));
    out->n = read_count();
    CUP(cudaFreeAsync(sorted, s));
    return HT_OK;
  }
  // a ^ b (invert = 0) or a \ b (invert = 1)
  int select(const Set& a, const Set& b, int invert, Set* out) {
    out->n = 0;
    HT_TRY(alloc((void**)&out->p, a.n * 8));
    if (a.n == 0) return HT_OK;
    if (b.n == 0 && invert) {
      CUP(cudaMemcpyAsync(out->p, a.p, a.n * 8, cudaMemcpyDeviceToDevice, s));
      out->n = a.n;
      return HT_OK;
    }
    uint8_t* flag;
    CUP(cudaMallocAsync((void**)&flag, a.n, s));
    k_member<<<grid(a.n), 256, 0, s>>>(a.p, a.n, b.p, b.n, flag, invert);
    CUP(cudaGetLastError());
    size_t b1 = 0;
    CUP(cub::DeviceSelect::Flagged(nullptr, b1, a.p, flag, out->p, nsel, a.n, s));
    HT_TRY(scratch(b1));
    CUP(cub::DeviceSelect::Flagged(tmp, b1, a.p, flag, out->p, nsel, a.n, s));
    out->n = read_count();
    CUP(cudaFreeAsync(flag, s));
    return HT_OK;
  }
  int unite(const Set& a, const Set& b, Set* out) {
    int64_t* cat;
    CUP(cudaMallocAsync((void**)&cat, (a.n + b.n) * 8 + 8, s));
    if (a.n) CUP(cudaMemcpyAsync(cat, a.p, a.n * 8, cudaMemcpyDeviceToDevice, s));
    if (b.n) CUP(cudaMemcpyAsync(cat + a.n, b.p, b.n * 8, cudaMemcpyDeviceToDevice, s));
    HT_TRY(sort_unique(cat, a.n + b.n, out));
    CUP(cudaFreeAsync(cat, s));
    return HT_OK;
  }
  // stable split of a sorted set by owner: parts[k] (ascending ids each)
  int by_owner(const Set& a, const int64_t* owner, std::vector<Set>& parts) {
    parts.assign(m, Set{});
    int64_t* vals;
    HT_TRY(alloc((void**)&vals, a.n * 8));
    int32_t *key, *key2, *cnt;
    CUP(cudaMallocAsync((void**)&key, a.n * 4 + 4, s));
    CUP(cudaMallocAsync((void**)&key2, a.n * 4 + 4, s));
    CUP(cudaMallocAsync((void**)&cnt, m * 4, s));
    CUP(cudaMemsetAsync(cnt, 0, m * 4, s));
    std::vector<int32_t> hc(m, 0);
    if (a.n) {
      k_owner_keys<<<grid(a.n), 256, 0, s>>>(a.p, a.n, owner, key, cnt);
      CUP(cudaGetLastError());
      int obits = 1;
      while ((1 << obits) < m) ++obits;
      size_t b1 = 0;
      CUP(cub::DeviceRadixSort::SortPairs(nullptr, b1, key, key2, a.p, vals, a.n, 0, obits, s));
      HT_TRY(scratch(b1));
      CUP(cub::DeviceRadixSort::SortPairs(tmp, b1, key, key2, a.p, vals, a.n, 0, obits, s));
      CUP(cudaMemcpyAsync(hc.data(), cnt, m * 4, cudaMemcpyDeviceToHost, s));
      CUP(cudaStreamSynchronize(s));
    }
    int64_t off = 0;
    for (int k = 0; k < m; ++k) {
      parts[k].p = vals + off;
      parts[k].n = hc[k];
      off += hc[k];
    }
    CUP(cudaFreeAsync(key, s));
    CUP(cudaFreeAsync(key2, s));
    CUP(cudaFreeAsync(cnt, s));
    return HT_OK;
  }
  // slots of live set `cur` given the previous batch's live set and slots
  int slots(const Set& cur, const Set* prev, const int64_t* pslot, int64_t* top, int64_t* out) {
    if (cur.n == 0) return HT_OK;
    if (!prev) {
      k_iota<<<grid(cur.n), 256, 0, s>>>(out, cur.n);
      CUP(cudaGetLastError());
      *top = std::max<int64_t>(*top, cur.n);
      return HT_OK;
    }
    const int64_t range = *top + cur.n;
    uint8_t* held;
    int32_t *fresh, *qrank, *freef, *frank;
    int64_t* freeslot;
    CUP(cudaMallocAsync((void**)&held, range, s));
    CUP(cudaMallocAsync((void**)&fresh, cur.n * 4, s));
    CUP(cudaMallocAsync((void**)&qrank, cur.n * 4, s));
    CUP(cudaMallocAsync((void**)&freef, range * 4, s));
    CUP(cudaMallocAsync((void**)&frank, range * 4, s));
    CUP(cudaMallocAsync((void**)&freeslot, cur.n * 8, s));
    CUP(cudaMemsetAsync(held, 0, range, s));
    k_carry_slots<<<grid(cur.n), 256, 0, s>>>(cur.p, cur.n, prev->p, pslot, prev->n, out, held, fresh);
    CUP(cudaGetLastError());
    k_free_flags<<<grid(range), 256, 0, s>>>(held, *top, range, freef);
    CUP(cudaGetLastError());
    size_t b1 = 0, b2 = 0;
    CUP(cub::DeviceScan::ExclusiveSum(nullptr, b1, fresh, qrank, cur.n, s));
    CUP(cub::DeviceScan::ExclusiveSum(nullptr, b2, freef, frank, range, s));
    HT_TRY(scratch(std::max(b1, b2)));
    CUP(cub::DeviceScan::ExclusiveSum(tmp, b1, fresh, qrank, cur.n, s));
    int32_t lastq = 0, lastf = 0;
    CUP(cudaMemcpyAsync(&lastq, qrank + cur.n - 1, 4, cudaMemcpyDeviceToHost, s));
    CUP(cudaMemcpyAsync(&lastf, fresh + cur.n - 1, 4, cudaMemcpyDeviceToHost, s));
    CUP(cub::DeviceScan::ExclusiveSum(tmp, b2, freef, frank, range, s));
    CUP(cudaStreamSynchronize(s));
    const int64_t nfresh = (int64_t)lastq + lastf;
    if (nfresh > 0) {
      k_take_free<<<grid(range), 256, 0, s>>>(freef, frank, range, nfresh, freeslot);
      CUP(cudaGetLastError());
      k_fill_fresh<<<grid(cur.n), 256, 0, s>>>(out, fresh, qrank, cur.n, freeslot);
      CUP(cudaGetLastError());
      int64_t last = 0;
      CUP(cudaMemcpyAsync(&last, freeslot + nfresh - 1, 8, cudaMemcpyDeviceToHost, s));
      CUP(cudaStreamSynchronize(s));
      *top = std::max(*top, last + 1);
    }
    for (void* p : {(void*)held, (void*)fresh, (void*)qrank, (void*)freef, (void*)frank, (void*)freeslot})
      CUP(cudaFreeAsync(p, s));
    return HT_OK;
  }
};

namespace {

int build(ht_gplan* g, const int64_t* owner_h, const int64_t* src_h, const int64_t* off_h) {
  const int m = g->m, n = g->n;
  cudaStream_t s = g->s;
  while ((int64_t(1) << g->bits) < g->V) ++g->bits;
  int64_t *owner, *src;
  const int64_t E = off_h[(int64_t)m * n];
  CUP(cudaMallocAsync((void**)&owner, g->V * 8 + 8, s));
  CUP(cudaMallocAsync((void**)&src, E * 8 + 8, s));
  CUP(cudaMemcpyAsync(owner, owner_h, g->V * 8, cudaMemcpyHostToDevice, s));
  CUP(cudaMemcpyAsync(src, src_h, E * 8, cudaMemcpyHostToDevice, s));
  auto at = [n](int i, int j) { return (int64_t)i * n + j; };
  // N_ij
  std::vector<Set> N(m * n), U(n), T(m * n), carry(m * n), load(m * n), nbrc(m * n), live(m * n);
  std::vector<Set> fetch((int64_t)m * n * std::max(1, m - 1));
  std::vector<int64_t*> slot(m * n, nullptr);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      const int64_t a = off_h[at(i, j)], b = off_h[at(i, j) + 1];
      if (b < a) return fail(HT_EINVAL, "chunk offsets must be non-decreasing");
      HT_TRY(g->sort_unique(src + a, b - a, &N[at(i, j)]));
    }
  // range checks (the host planner raises PlanError for these)
  for (auto& x : N)
    if (x.n) {
      int64_t lo = 0, hi = 0;
      CUP(cudaMemcpyAsync(&lo, x.p, 8, cudaMemcpyDeviceToHost, s));
      CUP(cudaMemcpyAsync(&hi, x.p + x.n - 1, 8, cudaMemcpyDeviceToHost, s));
      CUP(cudaStreamSynchronize(s));
      if (lo < 0 || hi >= g->V)
        return fail(HT_EINVAL, "neighbour id %lld outside the owner map (size %lld)",
                    (long long)(lo < 0 ? lo : hi), (long long)g->V);
    }
  // U_j, then T_ij by a stable owner split
  for (int j = 0; j < n; ++j) {
    int64_t tot = 0;
    for (int i = 0; i < m; ++i) tot += N[at(i, j)].n;
    int64_t* cat;
    CUP(cudaMallocAsync((void**)&cat, tot * 8 + 8, s));
    int64_t o = 0;
    for (int i = 0; i < m; ++i) {
      const Set& x = N[at(i, j)];
      if (x.n) CUP(cudaMemcpyAsync(cat + o, x.p, x.n * 8, cudaMemcpyDeviceToDevice, s));
      o += x.n;
    }
    HT_TRY(g->sort_unique(cat, tot, &U[j]));
    CUP(cudaFreeAsync(cat, s));
    std::vector<Set> parts;
    HT_TRY(g->by_owner(U[j], owner, parts));
    for (int i = 0; i < m; ++i) T[at(i, j)] = parts[i];
  }
  // carry/load, neighbour carry, fetch sets
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      if (j == 0) {
        HT_TRY(g->alloc((void**)&carry[at(i, j)].p, 8));
        load[at(i, j)] = T[at(i, j)];
        HT_TRY(g->alloc((void**)&nbrc[at(i, j)].p, 8));
      } else {
        HT_TRY(g->select(T[at(i, j)], T[at(i, j - 1)], 0, &carry[at(i, j)]));
        HT_TRY(g->select(T[at(i, j)], T[at(i, j - 1)], 1, &load[at(i, j)]));
        HT_TRY(g->select(N[at(i, j)], N[at(i, j - 1)], 0, &nbrc[at(i, j)]));
      }
      std::vector<Set> parts;
      HT_TRY(g->by_owner(N[at(i, j)], owner, parts));
      int q = 0;
      for (int k = 0; k < m; ++k)
        if (k != i) fetch[at(i, j) * (m - 1) + q++] = parts[k];
    }
  // live sets and slots
  g->caps.assign(m, 0);
  for (int i = 0; i < m; ++i) {
    int64_t top = 0;
    for (int j = 0; j < n; ++j) {
      HT_TRY(g->unite(T[at(i, j)], N[at(i, j)], &live[at(i, j)]));
      HT_TRY(g->alloc((void**)&slot[at(i, j)], live[at(i, j)].n * 8));
      HT_TRY(g->slots(live[at(i, j)], j ? &live[at(i, j - 1)] : nullptr, j ? slot[at(i, j - 1)] : nullptr,
                      &top, slot[at(i, j)]));
    }
    g->caps[i] = top;
  }
  // volumes (planner.py:221-227)
  g->vol[0] = g->vol[1] = 0;
  for (auto& x : N) g->vol[0] += x.n;
  for (auto& u : U) g->vol[1] += u.n;
  g->vol[2] = n ? U[0].n : 0;
  for (int j = 1; j < n; ++j) {
    Set d;
    HT_TRY(g->select(U[j], U[j - 1], 1, &d));
    g->vol[2] += d.n;
  }
  CUP(cudaFreeAsync(owner, s));
  CUP(cudaFreeAsync(src, s));
  // the output order of ht_gplan_sizes
  auto& S = g->sets;
  S.clear();
  S.insert(S.end(), N.begin(), N.end());
  S.insert(S.end(), U.begin(), U.end());
  S.insert(S.end(), T.begin(), T.end());
  S.insert(S.end(), carry.begin(), carry.end());
  S.insert(S.end(), load.begin(), load.end());
  S.insert(S.end(), nbrc.begin(), nbrc.end());
  if (m > 1) S.insert(S.end(), fetch.begin(), fetch.end());
  S.insert(S.end(), live.begin(), live.end());
  for (int q = 0; q < m * n; ++q) S.push_back(Set{slot[q], live[q].n});
  CUP(cudaStreamSynchronize(s));
  return HT_OK;
}

}  // namespace

extern "C" int ht_gplan_build(int device, int m, int n, int64_t V, const int64_t* owner,
                              const int64_t* src_concat, const int64_t* src_offsets,
                              ht_gplan** out) {
  *out = nullptr;
  if (m < 1 || n < 1 || V < 0) return fail(HT_EINVAL, "bad plan grid m=%d n=%d V=%lld", m, n, (long long)V);
  for (int64_t v = 0; v < V; ++v)
    if (owner[v] < 0 || owner[v] >= m)
      return fail(HT_EINVAL, "vertex %lld has owner %lld, outside [0, %d)", (long long)v,
                  (long long)owner[v], m);
  CUP(cudaSetDevice(device));
  ht_gplan* g = new ht_gplan();
  g->device = device;
  g->m = m;
  g->n = n;
  g->V = V;
  int rc = HT_OK;
  if (cudaStreamCreateWithFlags(&g->s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc((void**)&g->nsel, 8) != cudaSuccess)
    rc = fail(HT_ECUDA, "gplan: stream/counter allocation failed");
  if (rc == HT_OK) rc = build(g, owner, src_concat, src_offsets);
  if (rc != HT_OK) {
    delete g;
    return rc;
  }
  *out = g;
  return HT_OK;
}

extern "C" int ht_gplan_count(ht_gplan* g, int64_t* nsets) {
  *nsets = (int64_t)g->sets.size();
  return HT_OK;
}

extern "C" int ht_gplan_sizes(ht_gplan* g, int64_t* sizes, int64_t* caps, int64_t* volumes) {
  for (size_t q = 0; q < g->sets.size(); ++q) sizes[q] = g->sets[q].n;
  for (int i = 0; i < g->m; ++i) caps[i] = g->caps[i];
  for (int k = 0; k < 3; ++k) volumes[k] = g->vol[k];
  return HT_OK;
}

extern "C" int ht_gplan_fetch(ht_gplan* g, int64_t* concat) {
  CUP(cudaSetDevice(g->device));
  int64_t o = 0;
  for (auto& x : g->sets) {
    if (x.n) CUP(cudaMemcpyAsync(concat + o, x.p, x.n * 8, cudaMemcpyDeviceToHost, g->s));
    o += x.n;
  }
  CUP(cudaStreamSynchronize(g->s));
  return HT_OK;
}

extern "C" int ht_gplan_free(ht_gplan* g) {
  delete g;
  return HT_OK;
}
