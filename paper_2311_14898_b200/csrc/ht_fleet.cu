// Fleet runtime: m virtual devices executing one DedupPlan, and the GCN
// epoch layer drivers (devices.py / engine.py of the reference, re-designed
// for B200: slot buffers in HBM, zero-copy pinned host rows, peer-pointer
// fetches, per-device streams with event barriers at the Alg. 2/3 sync
// points).

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include "ht_common.h"
#include "ht_gat.cuh"
#include "ht_kernels.cuh"
#include "ht_tc.cuh"

using ht::fail;

#define CU(expr)                                                                    \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return fail(HT_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                              \
  } while (0)

namespace {

// long-segment piece length (edges); HT_SPLIT overrides it for tuning runs
const int64_t kSplit = [] {
  const char* e = getenv("HT_SPLIT");
  const long long v = e ? atoll(e) : 0;
  return (int64_t)(v >= 64 ? v : 1024);  // r1 sweep: 4096 -> 1024 saved 3 ms (GCN), 6 ms (GAT)
}();
constexpr int kThreads = 256;
constexpr int kMarks = 16;
std::atomic<int64_t> g_launches{0};  // kernels launched by this library
inline void count_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// Grow-only device allocation.
struct DBuf {
  void* p = nullptr;
  int64_t bytes = 0;
  int dev = 0;
  bool owned = true;  // false: a peer process's buffer mapped through CUDA IPC
  bool alias = false; // true: a caller-owned device array (an HBM host store)
  int ensure(int64_t want) {
    if (alias) p = nullptr, bytes = 0, alias = false;
    if (want <= bytes) return HT_OK;
    if (!owned) return fail(HT_ESTATE, "cannot grow a buffer shared with peer processes");
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (want <= 0) return HT_OK;
    CU(cudaMalloc(&p, want));
    bytes = want;
    return HT_OK;
  }
  void release() {
    if (p && !alias) {
      if (owned) cudaFree(p);
      else cudaIpcCloseMemHandle(p);
    }
    p = nullptr;
    bytes = 0;
    owned = true;
    alias = false;
  }
  void set_alias(void* q) {
    release();
    p = q;
    alias = true;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

template <class T>
int upload(DBuf& b, const std::vector<T>& v, cudaStream_t s) {
  HT_TRY(b.ensure((int64_t)(v.size() * sizeof(T))));
  if (!v.empty()) CU(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return HT_OK;
}

struct CopyList {
  int64_t n = 0;
  DBuf src, dst, flag;  // int64 src rows, int64 dst rows, uint8 flags
  // maximal runs of consecutive (host row, device row) pairs, sorted by
  // host row; when there are few of them the copy engines move the list
  // (no SMs, full PCIe duplex) instead of the zero-copy kernel
  std::vector<int64_t> run_host, run_dev, run_len;
  bool dma = false;
};

constexpr int64_t kMaxDmaRuns = 512;
constexpr int kChunks = 8;  // host-row chunks for store -> load streaming

// runs of a list whose host-side rows are `host` and device-side rows `dev`
void make_runs(CopyList& cl, const std::vector<int64_t>& host, const std::vector<int64_t>& dev,
               const std::vector<uint8_t>* flag) {
  cl.run_host.clear();
  cl.run_dev.clear();
  cl.run_len.clear();
  bool sorted = true;
  for (size_t q = 0; q < host.size(); ++q) {
    if (q > 0 && host[q] < host[q - 1]) sorted = false;
    if (q > 0 && host[q] == host[q - 1] + 1 && dev[q] == dev[q - 1] + 1 &&
        (!flag || (*flag)[q] == (*flag)[q - 1])) {
      cl.run_len.back()++;
    } else {
      cl.run_host.push_back(host[q]);
      cl.run_dev.push_back(dev[q]);
      cl.run_len.push_back(1);
    }
    if ((int64_t)cl.run_len.size() > kMaxDmaRuns) break;
  }
  bool first_only = true;
  if (flag)
    for (uint8_t v : *flag) first_only &= v != 0;
  cl.dma = sorted && (int64_t)cl.run_len.size() <= kMaxDmaRuns && first_only;
  if (!cl.dma) cl.run_host.clear(), cl.run_dev.clear(), cl.run_len.clear();
}

// Host-side plan sets of one chunk (i, j)
struct HostSets {
  std::vector<int64_t> nbr, owned, load, nbr_carry, live, slots, dest;
  bool has_dest = false;
  std::vector<std::vector<int64_t>> fetch;  // [k]
  // chunk structure
  bool has_chunk = false;
  int64_t nv = 0, nn = 0, ne = 0;
  std::vector<int64_t> csc_off, csc_src, csr_off, csr_dst, csr_perm;
  std::vector<double> w;
};

struct DevChunk {
  int64_t nv = 0, nn = 0, ne = 0, nlive = 0;
  DBuf nbr_slot;   // int64 [nn]
  DBuf dest_rows;  // int64 [nv]
  CopyList dest;   // runs of (host row = dest_rows[r], staging row r)
  std::vector<int64_t> dest_pos;  // [kChunks+1]: first staging row of each host-row chunk
  CopyList h2d;    // host row -> slot
  std::vector<CopyList> d2d;   // [step 1..m-1] peer slot -> own slot
  std::vector<CopyList> push;  // [source device i] pos in N_ij(i) -> own slot (owner = this device)
  CopyList flush;              // slot -> host row (+first flag)
  CopyList base_bwd;           // baseline: pos -> host row
  // graph
  DBuf csc_off, csc_slot, csc_w;     // int64 [nv+1], int32 [ne], float [ne]
  DBuf csr_off, csr_dst, csr_w;      // int64 [nn+1], int32 [ne], float [ne]
  int64_t fw_np = 0, fw_nf = 0, bw_np = 0, bw_nf = 0;
  DBuf fw_lo, fw_hi, fw_seg, fw_first, fw_cnt;  // long-segment pieces (forward)
  DBuf bw_lo, bw_hi, bw_seg, bw_first, bw_cnt;  // (backward)
  // one device, one batch: the CSR offsets expanded to every host row
  // (empty segments for rows without out-edges) so the transposed
  // aggregation writes the dense grad mirror directly; pieces re-indexed
  DBuf bx_off, bx_lo, bx_hi, bx_seg, bx_first, bx_cnt;
  int64_t bx_np = 0, bx_nf = 0, bx_rows = -1;
  // GAT: chunk-local CSC sources (rows of q) and the CSC edge id of each
  // CSR edge; uploaded by the first GAT epoch
  DBuf csc_loc, csr_perm;            // int32 [ne], int32 [ne]
  bool gat_ready = false;
  // HBM owner cache: the destination rows are the contiguous mirror rows
  // [dest_m0, dest_m0 + nv); h2d / flush rows as mirror positions
  int64_t dest_m0 = -1;
  DBuf h2d_m, flush_m;               // int64 [h2d.n], int64 [flush.n]
  // single device (m = 1): sources by global row, so the gathers read an
  // HBM-resident h^l (mirror or HBM store) in place, without slot loads
  DBuf csc_gid;                      // int32 [ne]: global row of each CSC source
  DBuf nbr_gid;                      // int64 [nn]: global row of each neighbour
};

struct LayerW {
  DBuf W, Wt, Wp, Wt_hi, Wt_lo, Wp_hi, Wp_lo;
  DBuf A;  // GAT attention vector [a_dst | a_src] (2 d_out)
  bool valid = false;
};

constexpr int kHostGrid = 128;    // CTAs of a zero-copy host transfer kernel
constexpr int kSplitsMax = 148;   // row slices of the weight-gradient GEMM (one per SM)

struct TimerRec {
  cudaEvent_t a, b;
  int which;
  double bytes;
};

struct Device {
  int ordinal = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev = nullptr;
  int64_t cap = 0;
  DBuf value, grad;                    // cap x dim slot buffers
  DBuf sa, sb, sc, sd, se, partial;    // staging
  DBuf tT;                             // A^T gz in d_out space (narrow-side backward)
  DBuf pf_p, pf_z;                     // project-first layers: h.W and A.(h.W), pad4(d_out) wide
  DBuf gemm_ws;
  DBuf W, Wt, Wp;                      // current layer weights, transpose, padded
  DBuf Wt_hi, Wt_lo, Wp_hi, Wp_lo;     // TF32 hi/lo halves for tcgen05
  DBuf gWall;                          // weight-gradient accumulators, all layers
  std::vector<int64_t> gW_off;         // float offset of layer l inside gWall
  DBuf flags;                          // cross-process barrier counter (rank mode)
  bool local = true;                   // false: a peer rank's device (IPC views only)
  DBuf hL;                             // last-layer outputs (concat over batches)
  std::vector<int64_t> hL_off;         // row offset of batch j inside hL
  DBuf labels, mask, loss_part;
  std::vector<DevChunk> chunks;
  cudaEvent_t mark[kMarks] = {};  // ht_fleet_mark slots (compute stream)
  // epoch pipeline: transfer streams, double-buffered staging, events
  cudaStream_t tin = nullptr, tout = nullptr;
  // checkpoint prefetch: agg rows of layer l come back from the host as
  // soon as they are stored (same bytes, moved while the link is idle)
  cudaStream_t tpre = nullptr;
  std::vector<DBuf> ck;
  std::vector<cudaEvent_t> e_ck;
  DBuf fa[2], fb[2], ba[2], bb[2];
  cudaEvent_t e_in = nullptr, e_fetch = nullptr, e_agg = nullptr, e_comp = nullptr;
  cudaEvent_t e_out[2] = {nullptr, nullptr}, e_hst = nullptr, e_loss = nullptr;
  cudaEvent_t e_bin = nullptr, e_bcomp[2] = {nullptr, nullptr}, e_flush = nullptr;
  cudaEvent_t e_hchunk[kChunks] = {}, e_fchunk[kChunks] = {};  // stores / flushes per host-row chunk
  cudaEvent_t e_gchunk[kChunks] = {}, e_gin[kChunks] = {};     // GEMM / gradient-load chunks
  std::vector<cudaEvent_t> e_aggst;  // [layer * kChunks + chunk]: checkpoint rows stored
  int64_t fwd_count = 0, bwd_count = 0;
  std::vector<LayerW> lw;            // per-layer weights (valid until the SGD step)
  float* wpin = nullptr;             // pinned scratch for weight uploads
  std::vector<int64_t> wpin_off;
  int64_t wpin_cap = 0;
  uint8_t* lpin = nullptr;           // pinned labels + mask
  int64_t lpin_cap = 0;
  DBuf sgd_p, sgd_w, sgd_t;          // SGD: pointer table, parameters, summed gradients
  uint8_t* sgd_pin = nullptr;        // pinned staging of the SGD step
  int64_t sgd_pin_cap = 0;
  // GAT staging (sized by ht_gat_epoch_begin): neighbour / destination
  // inputs, projections q / p, scores, backward rows and per-edge values
  DBuf g_hn, g_hd[2], g_q, g_p, g_els, g_gs, g_gp, g_al, g_gt, g_sgt, g_gq, g_gts, g_ghd, g_gin[2];
  // gat_direct: each layer's projection p = h.W and el_src = p.a_src kept
  // from the forward for the backward (the recompute-cache hybrid sized to
  // HBM: the backward skips the recompute GEMM, bitwise the same values)
  std::vector<DBuf> g_pl, g_elsl;
  DBuf g_pgts;                         // per-piece g_t sums of split source segments
  DBuf g_cpart;                        // column partials of the attention gradients
  std::vector<int64_t> gA_off;         // attention gradients: gWall + gW_off[L] + gA_off[l]
  cudaEvent_t e_gcomp[2] = {nullptr, nullptr};
  // HBM owner cache: HBM mirrors of the host rows this
  // device owns - h^l (l < L), agg^l (GCN), grad_h^l (l <= L) - read by the
  // layer drivers instead of the host; every row produced is written
  // through to the host store, which stays the reference's complete copy.
  bool cache = false;
  int64_t mcount = 0;                  // owned rows (mirror rows)
  std::vector<int64_t> mrows;          // host row of each mirror position, ascending
  DBuf mrows_d;                        // same, on the device
  CopyList own;                        // runs of (host row, mirror position)
  std::vector<DBuf> mh, ma, mg;
  cudaEvent_t e_up = nullptr, e_mg = nullptr;
};

}  // namespace

struct ht_fleet {
  int m = 0, n = 0, mode = HT_MODE_FULL, flush = HT_FLUSH_ON_EVICTION;
  std::vector<Device> dev;
  std::vector<std::vector<HostSets>> sets;  // [i][j]
  bool finalized = false;
  int dim = 0, elem = 4;
  int hL_dim = 0;
  bool timing = false;
  std::vector<TimerRec> timers;
  int64_t t_launch[4] = {0, 0, 0, 0};
  double t_ms[4] = {0, 0, 0, 0}, t_bytes[4] = {0, 0, 0, 0};
  int L = 0;
  std::vector<int> dims;
  // h^l arrays passed to the forward layers (device-usable) and whether they
  // are HBM: the backward takes ReLU' from h^{l+1} when it is device-resident
  std::vector<void*> hptr;
  std::vector<char> hdev;
  int64_t loss_count = 0;
  bool prefetch = true;  // checkpoint prefetch (HT_CKPT_PREFETCH=0 disables)
  bool gat = false;      // buffers sized by ht_gat_epoch_begin
  int cache_req = 0;     // HBM owner cache: 0 off, 1 on (fail if impossible), 2 auto
  bool host_compact = false;  // host arrays hold only the local device's owned rows
  // lean epoch (opt-in): no grad_h^0 (never consumed,
  // engine.py:449/477) and no host copies of h^L / grad_h^L with the cache
  bool lean = false;
  // checkpoint tier (the recompute-cache hybrid sized to HBM): with the owner
  // cache active, the GCN agg checkpoints stay in their HBM mirrors and are
  // not written through to host.agg; ht_fleet_checkpoint_read materializes
  // them on demand
  bool ckpt_hbm = false;
  // project-first layers of this epoch (one device, one batch, d_out < d_in,
  // HBM checkpoints): agg^l was never formed; ht_fleet_checkpoint_read
  // aggregates it on demand
  std::vector<char> agg_deferred;
  // HBM store (placement "device") on a single device: its arrays serve as
  // the owner-cache mirrors directly (h[0..L], agg[0..L-1], grad[0..L])
  std::vector<void*> alias_h, alias_a, alias_g;
  bool cache_ok = false; // the plan admits the cache (p2p/full, contiguous dest rows)
  int64_t nrows = 0;  // host rows addressed by the plan (max vertex id + 1)
  // rank mode (one process per GPU): index of the local device, barrier
  // sequence, device array of every rank's barrier counter
  int rank = -1;
  int64_t seq = 0;
  DBuf flag_ptrs;
  int imported = 0;
};

namespace {

int set_dev(const Device& d) {
  CU(cudaSetDevice(d.ordinal));
  return HT_OK;
}

// all-to-all event barrier across the per-device streams
// Cross-process barrier of rank mode, on the local compute stream: publish
// the next sequence number in the local counter, wait (device-side) until
// every rank's counter reached it.  Every rank issues the same barriers.
int xbarrier(ht_fleet* f) {
  Device& d = f->dev[f->rank];
  HT_TRY(set_dev(d));
  if (f->imported != f->m - 1) return fail(HT_ESTATE, "rank mode: peer buffers not imported");
  if (!f->flag_ptrs.p) {
    std::vector<uint32_t*> ptrs(f->m);
    for (int k = 0; k < f->m; ++k) ptrs[k] = f->dev[k].flags.as<uint32_t>();
    HT_TRY(f->flag_ptrs.ensure(f->m * sizeof(uint32_t*)));
    CU(cudaMemcpy(f->flag_ptrs.p, ptrs.data(), f->m * sizeof(uint32_t*), cudaMemcpyHostToDevice));
  }
  f->seq++;
  count_launch();
  ht::k_xbarrier<<<1, 32, 0, d.stream>>>(d.flags.as<uint32_t>(), f->flag_ptrs.as<uint32_t*>(), f->m,
                                         (uint32_t)f->seq);
  CU(cudaGetLastError());
  return HT_OK;
}

int barrier(ht_fleet* f) {
  if (f->rank >= 0) return xbarrier(f);
  for (auto& d : f->dev) {
    HT_TRY(set_dev(d));
    CU(cudaEventRecord(d.ev, d.stream));
  }
  for (auto& d : f->dev) {
    HT_TRY(set_dev(d));
    for (auto& o : f->dev)
      if (&o != &d) CU(cudaStreamWaitEvent(d.stream, o.ev, 0));
  }
  return HT_OK;
}

int sync_all(ht_fleet* f) {
  for (auto& d : f->dev) {
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    CU(cudaStreamSynchronize(d.stream));
    if (d.tin) CU(cudaStreamSynchronize(d.tin));
    if (d.tout) CU(cudaStreamSynchronize(d.tout));
    if (d.tpre) CU(cudaStreamSynchronize(d.tpre));
  }
  return HT_OK;
}

int ev_rec(cudaEvent_t& e, cudaStream_t s) {
  if (!e) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CU(cudaEventRecord(e, s));
  return HT_OK;
}

int ev_wait(cudaStream_t s, cudaEvent_t e) {
  if (e) CU(cudaStreamWaitEvent(s, e, 0));
  return HT_OK;
}

int grid_for(int64_t warps_needed) {
  int64_t blocks = (warps_needed * 32 + kThreads - 1) / kThreads;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 16));
  return (int)blocks;
}

// pinned host / device pointer -> device-usable pointer
int dev_ptr(const void* p, void** out) {
  if (!p) { *out = nullptr; return HT_OK; }
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(HT_EINVAL, "array at %p is not pinned or device memory", p);
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    *out = const_cast<void*>(p);
    return HT_OK;
  }
  if (a.type == cudaMemoryTypeHost) {
    *out = a.devicePointer ? a.devicePointer : const_cast<void*>(p);
    return HT_OK;
  }
  return fail(HT_EINVAL, "array at %p is pageable host memory; pin it first", p);
}

bool is_dev_mem(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice;
}

// Row copy with the widest vector the row size and alignment permit.
int launch_copy(cudaStream_t s, void* dst, const void* src, const int64_t* didx,
                const int64_t* sidx, int64_t rows, int64_t row_bytes, int64_t dstride,
                int64_t sstride, int64_t dbase = 0, int max_grid = 0) {
  if (rows <= 0 || row_bytes <= 0) return HT_OK;
  const uintptr_t al = (uintptr_t)dst | (uintptr_t)src | (uintptr_t)row_bytes |
                       (uintptr_t)dstride | (uintptr_t)sstride;
  int g = grid_for(rows);
  if (max_grid > 0) g = std::min(g, max_grid);
  count_launch();
  if ((al & 15) == 0)
    ht::k_copy_rows<int4><<<g, kThreads, 0, s>>>((char*)dst, (const char*)src, didx, sidx, rows,
                                                (int)(row_bytes / 16), dstride, sstride, dbase);
  else if ((al & 7) == 0)
    ht::k_copy_rows<int2><<<g, kThreads, 0, s>>>((char*)dst, (const char*)src, didx, sidx, rows,
                                                (int)(row_bytes / 8), dstride, sstride, dbase);
  else
    ht::k_copy_rows<int><<<g, kThreads, 0, s>>>((char*)dst, (const char*)src, didx, sidx, rows,
                                               (int)(row_bytes / 4), dstride, sstride, dbase);
  CU(cudaGetLastError());
  return HT_OK;
}

// Copy-engine transfer of the rows of a DMA-eligible list whose host row
// lies in [lo, hi): to_host moves device rows -> host rows, else host ->
// device.  Row strides may differ from the row size (2-D copies).
int xfer(cudaStream_t s, const CopyList& cl, bool to_host, void* host_v, int64_t hld, void* dev_v,
         int64_t dld, int64_t rb, int64_t lo, int64_t hi) {
  char* host = static_cast<char*>(host_v);
  char* dev = static_cast<char*>(dev_v);
  for (size_t r = 0; r < cl.run_len.size(); ++r) {
    const int64_t a = cl.run_host[r], len = cl.run_len[r];
    const int64_t a0 = std::max(a, lo), a1 = std::min(a + len, hi);
    if (a0 >= a1) continue;
    char* hp = host + a0 * hld;
    char* dp = dev + (cl.run_dev[r] + (a0 - a)) * dld;
    const int64_t rows = a1 - a0;
    if (hld == rb && dld == rb) {
      CU(cudaMemcpyAsync(to_host ? hp : dp, to_host ? dp : hp, rows * rb, cudaMemcpyDefault, s));
    } else {
      CU(cudaMemcpy2DAsync(to_host ? hp : dp, to_host ? hld : dld, to_host ? dp : hp,
                           to_host ? dld : hld, rb, rows, cudaMemcpyDefault, s));
    }
  }
  return HT_OK;
}

inline int64_t chunk_bound(int64_t V, int g) { return V * g / kChunks; }

int launch_acc(cudaStream_t s, int elem, void* dst, void* src, const int64_t* didx,
               const int64_t* sidx, const uint8_t* first, int64_t rows, int d, int zero_src,
               int64_t sbase = 0) {
  if (rows <= 0) return HT_OK;
  const int g = grid_for(rows);
  count_launch();
  const uintptr_t al = (uintptr_t)dst | (uintptr_t)src;
  if (elem == 4 && d % 4 == 0 && (al & 15) == 0)
    ht::k_acc_rows4<<<grid_for((rows + 1) / 2), kThreads, 0, s>>>(
        (float*)dst, (float*)src, didx, sidx, first, rows, d, zero_src, sbase);
  else if (elem == 4)
    ht::k_acc_rows<float><<<g, kThreads, 0, s>>>((float*)dst, (float*)src, didx, sidx, first, rows,
                                                d, zero_src, sbase);
  else
    ht::k_acc_rows<double><<<g, kThreads, 0, s>>>((double*)dst, (double*)src, didx, sidx, first,
                                                 rows, d, zero_src, sbase);
  CU(cudaGetLastError());
  return HT_OK;
}

void timer_begin(ht_fleet* f, Device& d, TimerRec& r, cudaStream_t s = nullptr) {
  if (!f->timing) return;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s ? s : d.stream);
}
void timer_end(ht_fleet* f, Device& d, TimerRec& r, int which, double bytes,
               cudaStream_t s = nullptr) {
  if (!f->timing) return;
  cudaEventRecord(r.b, s ? s : d.stream);
  r.which = which;
  r.bytes = bytes;
  f->timers.push_back(r);
}
void timers_collect(ht_fleet* f) {
  for (auto& r : f->timers) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    f->t_launch[r.which]++;
    f->t_ms[r.which] += ms;
    f->t_bytes[r.which] += r.bytes;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  f->timers.clear();
}

// Aggregation kernel variant: edges in flight per warp (U) and the
// register cap (MINB resident CTAs per SM); HT_SEG_VARIANT selects one for
// tuning runs, the default is the measured best.
template <int NV>
void seg_variant(int g, cudaStream_t s, float* out, const float* X, int64_t ldx, int d,
                 const int64_t* off, const int32_t* idx, const float* w, int64_t nseg) {
  static int v = [] {
    const char* e = getenv("HT_SEG_VARIANT");
    return e ? atoi(e) : 0;
  }();
  static int v1 = [] {  // narrow rows (<= 128 floats): separate tuning knob
    const char* e = getenv("HT_SEG_VARIANT1");
    return e ? atoi(e) : 0;
  }();
  if (NV == 1) {
    switch (v1) {
      case 1: ht::k_seg_gather_v4<NV, 4, 4><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); return;
      case 2: ht::k_seg_gather_v4<NV, 8, 4><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); return;
      case 3: ht::k_seg_gather_v4<NV, 8, 6><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); return;
      case 4: ht::k_seg_gather_v4<NV, 16, 4><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); return;
      case 5: ht::k_seg_gather_v4<NV, 4, 8><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); return;
      case 6: ht::k_seg_gather_v4<NV, 8, 8><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); return;
      case 7: ht::k_seg_gather_v4<NV, 2, 8><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); return;
      default: ht::k_seg_gather_v4<NV, 8, 4><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); return;  // measured best (sweep, r1)
    }
  }
  switch (v) {
    case 1: ht::k_seg_gather_v4<NV, 4, 4><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); break;
    case 2: ht::k_seg_gather_v4<NV, 8, 2><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); break;
    case 3: ht::k_seg_gather_v4<NV, 8, 3><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); break;
    case 4: ht::k_seg_gather_v4<NV, 4, 1><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); break;
    case 5: ht::k_seg_gather_v4<NV, 2, 6><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); break;
    case 6: ht::k_seg_gather_v4<NV, 1, 8><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); break;
    case 7: ht::k_seg_gather_v4<NV, 4, 5><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); break;
    default: ht::k_seg_gather_v4<NV, 2, 4><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); break;
  }
}

// Segment gather-sum over a chunk's CSC (forward) or CSR (backward) view.
int launch_seg(cudaStream_t s, float* out, const float* X, int64_t ldx, int d, const int64_t* off,
               const int32_t* idx, const float* w, int64_t nseg, int64_t np, const DBuf& lo,
               const DBuf& hi, int64_t nf, const DBuf& seg, const DBuf& first, const DBuf& cnt,
               float* partial) {
  if (nseg <= 0) return HT_OK;
  const int g = grid_for(nseg);
  count_launch(1 + (np ? 1 : 0) + (nf ? 1 : 0));
  static const bool sub_ok = [] {  // HT_NO_SUBWARP=1: narrow rows on the warp kernels
    const char* e = getenv("HT_NO_SUBWARP");
    return !(e && atoi(e));
  }();
  if (d % 4 == 0 && d <= 64 && sub_ok) {  // narrow rows: 2 or 4 segments per warp
    static const int sv = [] {
      const char* e = getenv("HT_SUB_VARIANT");
      return e ? atoi(e) : 0;
    }();
    if (d <= 32) {
      ht::k_seg_gather_sub<8><<<grid_for((nseg + 3) / 4), kThreads, 0, s>>>(out, X, ldx, d, off, idx,
                                                                           w, nseg, kSplit);
      if (np) ht::k_seg_pieces_sub<8><<<grid_for((np + 3) / 4), kThreads, 0, s>>>(
          partial, X, ldx, d, lo.as<int64_t>(), hi.as<int64_t>(), idx, w, np);
    } else {
      const int g2 = grid_for((nseg + 1) / 2);
      if (sv == 1)
        ht::k_seg_gather_sub<16, 4, 4><<<g2, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit);
      else if (sv == 2)
        ht::k_seg_gather_sub<16, 8, 3><<<g2, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit);
      else if (sv == 3)
        ht::k_seg_gather_sub<16, 16, 2><<<g2, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit);
      else
        ht::k_seg_gather_sub<16, 8, 4><<<g2, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit);
      if (np) ht::k_seg_pieces_sub<16><<<grid_for((np + 1) / 2), kThreads, 0, s>>>(
          partial, X, ldx, d, lo.as<int64_t>(), hi.as<int64_t>(), idx, w, np);
    }
  } else if (d % 4 == 0 && d <= 512) {
    const int nv = (d / 4 + 31) / 32;
#define SEGV(NV)                                                                               \
  seg_variant<NV>(g, s, out, X, ldx, d, off, idx, w, nseg);                                \
  if (np) ht::k_seg_pieces_v4<NV><<<grid_for(np), kThreads, 0, s>>>(                           \
      partial, X, ldx, d, lo.as<int64_t>(), hi.as<int64_t>(), idx, w, np);
    switch (nv) {
      case 1: SEGV(1); break;
      case 2: SEGV(2); break;
      case 3: SEGV(3); break;
      default: SEGV(4); break;
    }
#undef SEGV
  } else {
    const int ns = (d + 31) / 32;
    if (ns > 16) return fail(HT_EINVAL, "feature width %d too large", d);
#define SEGS(NS)                                                                              \
  ht::k_seg_gather_s<NS><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, w, nseg, kSplit); \
  if (np) ht::k_seg_pieces_s<NS><<<grid_for(np), kThreads, 0, s>>>(                           \
      partial, X, ldx, d, lo.as<int64_t>(), hi.as<int64_t>(), idx, w, np);
    if (ns <= 1) { SEGS(1); }
    else if (ns <= 2) { SEGS(2); }
    else if (ns <= 4) { SEGS(4); }
    else if (ns <= 8) { SEGS(8); }
    else { SEGS(16); }
#undef SEGS
  }
  CU(cudaGetLastError());
  if (nf) {
    ht::k_seg_fixup<<<grid_for(nf), kThreads, 0, s>>>(out, partial, d, seg.as<int64_t>(),
                                                       first.as<int64_t>(), cnt.as<int64_t>(), nf);
    CU(cudaGetLastError());
  }
  return HT_OK;
}

template <bool TA, bool TB, int EPI>
int gemm(cudaStream_t s, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
         int64_t ldc, const float* G, int64_t ldg, int64_t M, int64_t N, int64_t K, int splits,
         int64_t kps) {
  if (M <= 0 || N <= 0) return HT_OK;
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64), (unsigned)splits);
  count_launch();
  ht::k_gemm<TA, TB, EPI><<<grid, 256, 0, s>>>(A, lda, B, ldb, C, ldc, G, ldg, M, N, K, kps);
  CU(cudaGetLastError());
  return HT_OK;
}

inline int pad4(int d) { return (d + 3) & ~3; }

// Layer weights on the device: W (d_in x d_out) for the SIMT path, and for
// the tensor-core path the TF32 hi/lo halves of W^T (d_out x d_in, the
// K-major operand of z = agg.W) and of W padded to pad4(d_out) columns (the
// K-major operand of gagg = gz.W^T).
int upload_weights(Device& d, const float* W, int d_in, int d_out) {
  const int64_t nw = (int64_t)d_in * d_out;
  const int ldo = pad4(d_out);
  const int64_t np = (int64_t)d_in * ldo;
  HT_TRY(d.W.ensure(nw * 4));
  HT_TRY(d.Wt.ensure(nw * 4));
  HT_TRY(d.Wp.ensure(np * 4));
  for (DBuf* b : {&d.Wt_hi, &d.Wt_lo}) HT_TRY(b->ensure(nw * 4));
  for (DBuf* b : {&d.Wp_hi, &d.Wp_lo}) HT_TRY(b->ensure(np * 4));
  std::vector<float> wt(nw), wp(np, 0.f);
  for (int a = 0; a < d_in; ++a)
    for (int b = 0; b < d_out; ++b) {
      wt[(int64_t)b * d_in + a] = W[(int64_t)a * d_out + b];
      wp[(int64_t)a * ldo + b] = W[(int64_t)a * d_out + b];
    }
  CU(cudaMemcpyAsync(d.W.p, W, nw * 4, cudaMemcpyHostToDevice, d.stream));
  CU(cudaMemcpyAsync(d.Wt.p, wt.data(), nw * 4, cudaMemcpyHostToDevice, d.stream));
  CU(cudaMemcpyAsync(d.Wp.p, wp.data(), np * 4, cudaMemcpyHostToDevice, d.stream));
  HT_TRY(ht::tc::split_weights(d.stream, d.Wt.as<float>(), d.Wt_hi.as<float>(), d.Wt_lo.as<float>(), nw));
  HT_TRY(ht::tc::split_weights(d.stream, d.Wp.as<float>(), d.Wp_hi.as<float>(), d.Wp_lo.as<float>(), np));
  count_launch(2);
  CU(cudaStreamSynchronize(d.stream));
  return HT_OK;
}

// long-segment pieces of an offsets array
void make_pieces(const std::vector<int64_t>& off, std::vector<int64_t>& lo, std::vector<int64_t>& hi,
                 std::vector<int64_t>& seg, std::vector<int64_t>& first, std::vector<int64_t>& cnt) {
  for (size_t sg = 0; sg + 1 < off.size(); ++sg) {
    const int64_t a = off[sg], b = off[sg + 1];
    if (b - a <= kSplit) continue;
    seg.push_back((int64_t)sg);
    first.push_back((int64_t)lo.size());
    int64_t c = 0;
    for (int64_t x = a; x < b; x += kSplit, ++c) {
      lo.push_back(x);
      hi.push_back(std::min(b, x + kSplit));
    }
    cnt.push_back(c);
  }
}

int lookup_slots(const HostSets& hs, const std::vector<int64_t>& rows, std::vector<int64_t>& out,
                 int i, int j) {
  out.resize(rows.size());
  for (size_t q = 0; q < rows.size(); ++q) {
    auto it = std::lower_bound(hs.live.begin(), hs.live.end(), rows[q]);
    if (it == hs.live.end() || *it != rows[q])
      return fail(HT_ELIVE, "device %d batch %d: rows requested outside the live set", i, j);
    out[q] = hs.slots[it - hs.live.begin()];
  }
  return HT_OK;
}

std::vector<int64_t> vdiff(const std::vector<int64_t>& a, const std::vector<int64_t>& b) {
  std::vector<int64_t> o;
  std::set_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
  return o;
}
std::vector<int64_t> visect(const std::vector<int64_t>& a, const std::vector<int64_t>& b) {
  std::vector<int64_t> o;
  std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
  return o;
}

int upload_list(CopyList& cl, const std::vector<int64_t>& src, const std::vector<int64_t>& dst,
                cudaStream_t s, const std::vector<uint8_t>* flag = nullptr) {
  cl.n = (int64_t)src.size();
  HT_TRY(upload(cl.src, src, s));
  HT_TRY(upload(cl.dst, dst, s));
  if (flag) HT_TRY(upload(cl.flag, *flag, s));
  return HT_OK;
}

}  // namespace

// ===========================================================================
// runtime / memory
// ===========================================================================

extern "C" int ht_device_count(int* count) {
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
  }
  return HT_OK;
}

extern "C" int ht_host_alloc(int64_t bytes, void** out) {
  CU(cudaHostAlloc(out, std::max<int64_t>(bytes, 16),
                   cudaHostAllocPortable | cudaHostAllocMapped));
  return HT_OK;
}
extern "C" int ht_host_free(void* p) {
  CU(cudaFreeHost(p));
  return HT_OK;
}
extern "C" int ht_host_register(void* p, int64_t bytes) {
  CU(cudaHostRegister(p, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  return HT_OK;
}
extern "C" int ht_host_unregister(void* p) {
  CU(cudaHostUnregister(p));
  return HT_OK;
}
extern "C" int ht_dev_alloc(int device, int64_t bytes, void** out) {
  CU(cudaSetDevice(device));
  CU(cudaMalloc(out, std::max<int64_t>(bytes, 16)));
  return HT_OK;
}
extern "C" int ht_dev_free(int device, void* p) {
  CU(cudaSetDevice(device));
  CU(cudaFree(p));
  return HT_OK;
}
extern "C" int ht_memcpy(void* dst, const void* src, int64_t bytes) {
  CU(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
  return HT_OK;
}
extern "C" int ht_memset(void* dst, int value, int64_t bytes) {
  CU(cudaMemset(dst, value, bytes));
  CU(cudaDeviceSynchronize());
  return HT_OK;
}

// ===========================================================================
// fleet construction
// ===========================================================================

extern "C" int ht_fleet_create(int m, int n, const int* ordinals, int mode, int flush_policy,
                               ht_fleet** out) {
  if (m < 1 || n < 1) return fail(HT_EINVAL, "fleet needs m >= 1 and n >= 1");
  if (mode < 0 || mode > 2) return fail(HT_EINVAL, "unknown mode %d", mode);
  if (flush_policy < 0 || flush_policy > 1) return fail(HT_EINVAL, "unknown flush policy");
  int ndev = 0;
  ht_device_count(&ndev);
  if (ndev < 1) return fail(HT_ECUDA, "no CUDA device visible");
  std::unique_ptr<ht_fleet> f(new ht_fleet);
  f->m = m;
  f->n = n;
  f->mode = mode;
  f->flush = flush_policy;
  {
    const char* e = getenv("HT_CKPT_PREFETCH");
    f->prefetch = !(e && e[0] == '0');
  }
  f->dev.resize(m);
  f->sets.assign(m, std::vector<HostSets>(n));
  for (int i = 0; i < m; ++i) {
    Device& d = f->dev[i];
    d.ordinal = ordinals ? ordinals[i] : 0;
    if (d.ordinal < 0 || d.ordinal >= ndev) return fail(HT_EINVAL, "bad device ordinal %d", d.ordinal);
    CU(cudaSetDevice(d.ordinal));
    CU(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&d.tin, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&d.tout, cudaStreamNonBlocking));
    {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      CU(cudaStreamCreateWithPriority(&d.tpre, cudaStreamNonBlocking, lo));
    }
    CU(cudaEventCreateWithFlags(&d.ev, cudaEventDisableTiming));
    d.chunks.resize(n);
    for (auto& c : d.chunks) c.csc_gid.release(), c.nbr_gid.release();
    for (auto* b : {&d.value, &d.grad, &d.sa, &d.sb, &d.sc, &d.sd, &d.se, &d.tT, &d.partial, &d.gemm_ws,
                    &d.W, &d.Wt, &d.Wp, &d.Wt_hi, &d.Wt_lo, &d.Wp_hi, &d.Wp_lo, &d.hL,
                    &d.labels, &d.mask, &d.loss_part})
      b->dev = d.ordinal;
    for (int k = 0; k < m; ++k) {
      const int ok = ordinals ? ordinals[k] : 0;
      if (ok == d.ordinal) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, d.ordinal, ok);
      if (!can) return fail(HT_ECUDA, "device %d cannot access peer %d", d.ordinal, ok);
      cudaError_t e = cudaDeviceEnablePeerAccess(ok, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(HT_ECUDA, "peer access %d->%d: %s", d.ordinal, ok, cudaGetErrorString(e));
      cudaGetLastError();
    }
    for (int j = 0; j < n; ++j) f->sets[i][j].fetch.resize(m);
  }
  *out = f.release();
  return HT_OK;
}

// Rank mode: this process drives virtual device `rank` on CUDA device
// `ordinal`; the other m-1 devices belong to peer processes and are reached
// through CUDA IPC (ht_fleet_ipc_export / _import).  p2p/full modes only:
// in those every host row a device touches is owned by it, so each process
// needs only its own host store rows.
extern "C" int ht_fleet_create_rank(int m, int n, int rank, int ordinal, int mode,
                                    int flush_policy, ht_fleet** out) {
  if (m < 1 || n < 1 || rank < 0 || rank >= m) return fail(HT_EINVAL, "bad rank fleet shape");
  if (mode == HT_MODE_BASELINE)
    return fail(HT_EINVAL, "rank mode needs mode p2p or full (baseline touches peers' host rows)");
  std::vector<int> ords(m, ordinal);
  HT_TRY(ht_fleet_create(1, n, &ordinal, mode, flush_policy, out));
  ht_fleet* f = *out;
  // re-shape: m devices, only `rank` local (it takes the device created above)
  Device local = std::move(f->dev[0]);
  f->dev.clear();
  f->dev.resize(m);
  for (int k = 0; k < m; ++k) {
    f->dev[k].ordinal = ordinal;
    f->dev[k].local = false;
    f->dev[k].chunks.resize(n);
  }
  f->dev[rank] = std::move(local);
  f->dev[rank].local = true;
  f->m = m;
  f->rank = rank;
  f->sets.assign(m, std::vector<HostSets>(n));
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) f->sets[i][j].fetch.resize(m);
  return HT_OK;
}

// IPC handles of the local buffers peers read: slot values, neighbour
// gradient views, weight-gradient accumulators, barrier counter.  Call after
// ht_epoch_begin (which sizes them once for the run).
extern "C" int ht_fleet_ipc_export(ht_fleet* f, void* out) {
  if (f->rank < 0) return fail(HT_ESTATE, "not a rank-mode fleet");
  Device& d = f->dev[f->rank];
  HT_TRY(set_dev(d));
  cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(out);
  DBuf* bufs[4] = {&d.value, &d.se, &d.gWall, &d.flags};
  for (int q = 0; q < 4; ++q) {
    if (!bufs[q]->p) return fail(HT_ESTATE, "export before ht_epoch_begin");
    CU(cudaIpcGetMemHandle(&h[q], bufs[q]->p));
  }
  return HT_OK;
}

extern "C" int ht_fleet_ipc_import(ht_fleet* f, int peer, const void* in) {
  if (f->rank < 0 || peer < 0 || peer >= f->m || peer == f->rank)
    return fail(HT_EINVAL, "bad peer %d", peer);
  Device& me = f->dev[f->rank];
  HT_TRY(set_dev(me));
  Device& d = f->dev[peer];
  const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(in);
  DBuf* bufs[4] = {&d.value, &d.se, &d.gWall, &d.flags};
  for (int q = 0; q < 4; ++q) {
    if (bufs[q]->p) continue;  // already imported
    void* p = nullptr;
    CU(cudaIpcOpenMemHandle(&p, h[q], cudaIpcMemLazyEnablePeerAccess));
    bufs[q]->p = p;
    bufs[q]->owned = false;
  }
  d.gW_off = me.gW_off;
  f->imported++;
  f->flag_ptrs.release();
  return HT_OK;
}

extern "C" int ht_fleet_destroy(ht_fleet* f) {
  if (!f) return HT_OK;
  sync_all(f);
  timers_collect(f);
  for (auto& d : f->dev) {
    cudaSetDevice(d.ordinal);
    for (auto* b : {&d.value, &d.grad, &d.sa, &d.sb, &d.sc, &d.sd, &d.se, &d.partial, &d.gemm_ws,
                    &d.W, &d.Wt, &d.Wp, &d.Wt_hi, &d.Wt_lo, &d.Wp_hi, &d.Wp_lo, &d.hL,
                    &d.labels, &d.mask, &d.loss_part, &d.gWall, &d.flags})
      b->release();
    for (auto& c : d.chunks) {
      for (auto* b : {&c.nbr_slot, &c.dest_rows, &c.csc_off, &c.csc_slot, &c.csc_w, &c.csr_off,
                      &c.csr_dst, &c.csr_w, &c.fw_lo, &c.fw_hi, &c.fw_seg, &c.fw_first, &c.fw_cnt,
                      &c.bw_lo, &c.bw_hi, &c.bw_seg, &c.bw_first, &c.bw_cnt, &c.bx_off, &c.bx_lo,
                      &c.bx_hi, &c.bx_seg, &c.bx_first, &c.bx_cnt, &c.csc_loc,
                      &c.csr_perm, &c.h2d_m, &c.flush_m})
        b->release();
      for (CopyList* cl : {&c.h2d, &c.flush, &c.base_bwd})
        cl->src.release(), cl->dst.release(), cl->flag.release();
      for (auto& cl : c.d2d) cl.src.release(), cl.dst.release();
      for (auto& cl : c.push) cl.src.release(), cl.dst.release();
    }
    if (d.ev) cudaEventDestroy(d.ev);
    for (auto& e : d.mark)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {d.e_in, d.e_fetch, d.e_agg, d.e_comp, d.e_out[0], d.e_out[1], d.e_hst,
                          d.e_loss, d.e_bin, d.e_bcomp[0], d.e_bcomp[1], d.e_flush})
      if (e) cudaEventDestroy(e);
    for (int g = 0; g < kChunks; ++g)
      for (cudaEvent_t e : {d.e_hchunk[g], d.e_fchunk[g], d.e_gchunk[g], d.e_gin[g]})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : d.e_aggst)
      if (e) cudaEventDestroy(e);
    for (int s = 0; s < 2; ++s)
      for (DBuf* b : {&d.fa[s], &d.fb[s], &d.ba[s], &d.bb[s]}) b->release();
    for (auto& w : d.lw)
      for (DBuf* b : {&w.W, &w.Wt, &w.Wp, &w.Wt_hi, &w.Wt_lo, &w.Wp_hi, &w.Wp_lo, &w.A}) b->release();
    for (DBuf* b : {&d.g_hn, &d.g_hd[0], &d.g_hd[1], &d.g_q, &d.g_p, &d.g_els, &d.g_gs, &d.g_gp,
                    &d.g_al, &d.g_gt, &d.g_sgt, &d.g_gq, &d.g_gts, &d.g_ghd, &d.g_gin[0],
                    &d.g_gin[1], &d.g_cpart, &d.g_pgts})
      b->release();
    for (auto* v : {&d.g_pl, &d.g_elsl})
      for (auto& b : *v) b.release();
    for (cudaEvent_t e : {d.e_gcomp[0], d.e_gcomp[1], d.e_up, d.e_mg})
      if (e) cudaEventDestroy(e);
    for (auto* v : {&d.mh, &d.ma, &d.mg})
      for (auto& b : *v) b.release();
    d.mrows_d.release();
    for (DBuf* b : {&d.sgd_p, &d.sgd_w, &d.sgd_t, &d.pf_p, &d.pf_z}) b->release();
    if (d.wpin) cudaFreeHost(d.wpin);
    if (d.lpin) cudaFreeHost(d.lpin);
    if (d.sgd_pin) cudaFreeHost(d.sgd_pin);
    if (d.stream) cudaStreamDestroy(d.stream);
    if (d.tin) cudaStreamDestroy(d.tin);
    if (d.tout) cudaStreamDestroy(d.tout);
    if (d.tpre) cudaStreamDestroy(d.tpre);
    for (auto& b : d.ck) b.release();
    for (cudaEvent_t e : d.e_ck)
      if (e) cudaEventDestroy(e);
  }
  delete f;
  return HT_OK;
}

static std::vector<int64_t> vec(const int64_t* p, int64_t n) {
  return n > 0 ? std::vector<int64_t>(p, p + n) : std::vector<int64_t>();
}

extern "C" int ht_fleet_set_sets(ht_fleet* f, int i, int j, const int64_t* nbr, int64_t n_nbr,
                                 const int64_t* owned, int64_t n_owned, const int64_t* load,
                                 int64_t n_load, const int64_t* nbr_carry, int64_t n_nbr_carry,
                                 const int64_t* live, const int64_t* slots, int64_t n_live,
                                 const int64_t* dest, int64_t n_dest) {
  if (i < 0 || i >= f->m || j < 0 || j >= f->n) return fail(HT_EINVAL, "chunk index out of range");
  HostSets& h = f->sets[i][j];
  h.nbr = vec(nbr, n_nbr);
  h.owned = vec(owned, n_owned);
  h.load = vec(load, n_load);
  h.nbr_carry = vec(nbr_carry, n_nbr_carry);
  h.live = vec(live, n_live);
  h.slots = vec(slots, n_live);
  h.has_dest = n_dest >= 0;
  h.dest = vec(dest, n_dest);
  f->finalized = false;
  return HT_OK;
}

extern "C" int ht_fleet_set_fetch(ht_fleet* f, int i, int j, int k, const int64_t* rows, int64_t n) {
  if (i < 0 || i >= f->m || j < 0 || j >= f->n || k < 0 || k >= f->m)
    return fail(HT_EINVAL, "fetch index out of range");
  f->sets[i][j].fetch[k] = vec(rows, n);
  f->finalized = false;
  return HT_OK;
}

extern "C" int ht_fleet_set_chunk(ht_fleet* f, int i, int j, int64_t nv, int64_t nn, int64_t ne,
                                  const int64_t* csc_off, const int64_t* csc_local_src,
                                  const double* edge_w, const int64_t* csr_off,
                                  const int64_t* csr_local_dst, const int64_t* csr_perm) {
  if (i < 0 || i >= f->m || j < 0 || j >= f->n) return fail(HT_EINVAL, "chunk index out of range");
  if (ne >= ((int64_t)1 << 31) || nn >= ((int64_t)1 << 31))
    return fail(HT_EINVAL, "chunk too large for 32-bit local indices");
  HostSets& h = f->sets[i][j];
  h.has_chunk = true;
  h.nv = nv;
  h.nn = nn;
  h.ne = ne;
  h.csc_off = vec(csc_off, nv + 1);
  h.csc_src = vec(csc_local_src, ne);
  h.csr_off = vec(csr_off, nn + 1);
  h.csr_dst = vec(csr_local_dst, ne);
  h.csr_perm = vec(csr_perm, ne);
  h.w.assign(edge_w, edge_w + ne);
  f->finalized = false;
  return HT_OK;
}

extern "C" int ht_fleet_finalize(ht_fleet* f) {
  const int m = f->m, n = f->n;
  const bool base = f->mode == HT_MODE_BASELINE;
  f->nrows = 0;
  for (auto& row : f->sets)
    for (auto& h : row) {
      if (!h.nbr.empty()) f->nrows = std::max(f->nrows, h.nbr.back() + 1);
      if (!h.dest.empty()) f->nrows = std::max(f->nrows, h.dest.back() + 1);
    }
  for (int i = 0; i < m; ++i) {
    Device& d = f->dev[i];
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    cudaStream_t s = d.stream;
    d.cap = 0;
    for (int j = 0; j < n; ++j) {
      HostSets& h = f->sets[i][j];
      if (base) d.cap = std::max<int64_t>(d.cap, (int64_t)h.nbr.size());
      else
        for (int64_t sl : h.slots) d.cap = std::max<int64_t>(d.cap, sl + 1);
    }
    for (int j = 0; j < n; ++j) {
      HostSets& h = f->sets[i][j];
      DevChunk& c = d.chunks[j];
      c.gat_ready = false;
      c.nn = (int64_t)h.nbr.size();
      c.nlive = base ? c.nn : (int64_t)h.live.size();
      c.nv = h.has_dest ? (int64_t)h.dest.size() : 0;
      std::vector<int64_t> nbr_slot, a, b;
      if (base) {
        nbr_slot.resize(h.nbr.size());
        std::iota(nbr_slot.begin(), nbr_slot.end(), 0);
        HT_TRY(upload_list(c.h2d, h.nbr, nbr_slot, s));
        make_runs(c.h2d, h.nbr, nbr_slot, nullptr);
      } else {
        HT_TRY(lookup_slots(h, h.nbr, nbr_slot, i, j));
        const auto& rows = f->mode == HT_MODE_FULL ? h.load : h.owned;
        HT_TRY(lookup_slots(h, rows, b, i, j));
        HT_TRY(upload_list(c.h2d, rows, b, s));
        make_runs(c.h2d, rows, b, nullptr);
        c.d2d.assign(m, CopyList());
        for (int st = 1; st < m; ++st) {
          const int k = (i + st) % m;
          std::vector<int64_t> rows_k = h.fetch[k];
          if (f->mode == HT_MODE_FULL && !h.nbr_carry.empty()) rows_k = vdiff(rows_k, h.nbr_carry);
          std::vector<int64_t> src_slot, dst_slot;
          HT_TRY(lookup_slots(f->sets[k][j], rows_k, src_slot, k, j));
          HT_TRY(lookup_slots(h, rows_k, dst_slot, i, j));
          HT_TRY(upload_list(c.d2d[st], src_slot, dst_slot, s));
        }
      }
      HT_TRY(upload(c.nbr_slot, nbr_slot, s));
      if (h.has_dest) {
        HT_TRY(upload(c.dest_rows, h.dest, s));
        std::vector<int64_t> pos(h.dest.size());
        std::iota(pos.begin(), pos.end(), 0);
        make_runs(c.dest, h.dest, pos, nullptr);
        c.dest_pos.clear();
        if (c.dest.dma && std::is_sorted(h.dest.begin(), h.dest.end())) {
          for (int g = 0; g <= kChunks; ++g)
            c.dest_pos.push_back(std::lower_bound(h.dest.begin(), h.dest.end(),
                                                  chunk_bound(f->nrows, g)) - h.dest.begin());
        }
      }
      if (h.has_chunk) {
        if (h.nn != c.nn || (h.has_dest && h.nv != c.nv))
          return fail(HT_EINVAL, "chunk (%d,%d) structure does not match its plan sets", i, j);
        std::vector<int32_t> slot32(h.ne), dst32(h.ne);
        std::vector<float> w32(h.ne), wcsr(h.ne);
        for (int64_t e = 0; e < h.ne; ++e) {
          slot32[e] = (int32_t)nbr_slot[h.csc_src[e]];
          w32[e] = (float)h.w[e];
          dst32[e] = (int32_t)h.csr_dst[e];
          wcsr[e] = (float)h.w[h.csr_perm[e]];
        }
        HT_TRY(upload(c.csc_off, h.csc_off, s));
        HT_TRY(upload(c.csc_slot, slot32, s));
        if (m == 1 && f->nrows < ((int64_t)1 << 31)) {
          std::vector<int32_t> gid(h.ne);
          for (int64_t e = 0; e < h.ne; ++e) gid[e] = (int32_t)h.nbr[h.csc_src[e]];
          HT_TRY(upload(c.csc_gid, gid, s));
          HT_TRY(upload(c.nbr_gid, h.nbr, s));
        }
        HT_TRY(upload(c.csc_w, w32, s));
        HT_TRY(upload(c.csr_off, h.csr_off, s));
        HT_TRY(upload(c.csr_dst, dst32, s));
        HT_TRY(upload(c.csr_w, wcsr, s));
        c.ne = h.ne;
        std::vector<int64_t> lo, hi, sg, fi, cn;
        make_pieces(h.csc_off, lo, hi, sg, fi, cn);
        c.fw_np = (int64_t)lo.size();
        c.fw_nf = (int64_t)sg.size();
        HT_TRY(upload(c.fw_lo, lo, s)); HT_TRY(upload(c.fw_hi, hi, s));
        HT_TRY(upload(c.fw_seg, sg, s)); HT_TRY(upload(c.fw_first, fi, s)); HT_TRY(upload(c.fw_cnt, cn, s));
        lo.clear(); hi.clear(); sg.clear(); fi.clear(); cn.clear();
        make_pieces(h.csr_off, lo, hi, sg, fi, cn);
        c.bw_np = (int64_t)lo.size();
        c.bw_nf = (int64_t)sg.size();
        HT_TRY(upload(c.bw_lo, lo, s)); HT_TRY(upload(c.bw_hi, hi, s));
        HT_TRY(upload(c.bw_seg, sg, s)); HT_TRY(upload(c.bw_first, fi, s)); HT_TRY(upload(c.bw_cnt, cn, s));
        c.bx_rows = -1;
        if (m == 1 && n == 1 && f->nrows < ((int64_t)1 << 31)) {
          std::vector<int64_t> offx(f->nrows + 1);
          int64_t q = 0;
          for (int64_t g = 0; g <= f->nrows; ++g) {
            while (q < h.nn && h.nbr[q] < g) ++q;
            offx[g] = h.csr_off[q];
          }
          lo.clear(); hi.clear(); sg.clear(); fi.clear(); cn.clear();
          make_pieces(offx, lo, hi, sg, fi, cn);
          c.bx_np = (int64_t)lo.size();
          c.bx_nf = (int64_t)sg.size();
          HT_TRY(upload(c.bx_off, offx, s));
          HT_TRY(upload(c.bx_lo, lo, s)); HT_TRY(upload(c.bx_hi, hi, s));
          HT_TRY(upload(c.bx_seg, sg, s)); HT_TRY(upload(c.bx_first, fi, s)); HT_TRY(upload(c.bx_cnt, cn, s));
          c.bx_rows = f->nrows;
        }
      }
      if (base) {
        std::vector<int64_t> pos(h.nbr.size());
        std::iota(pos.begin(), pos.end(), 0);
        HT_TRY(upload_list(c.base_bwd, pos, h.nbr, s));
      }
    }
  }
  // HBM owner cache structure: mirror rows = the owned rows (the union of
  // the destination sets, ascending); every destination set must be a
  // contiguous mirror range and every host-loaded row an owned row
  f->cache_ok = !base;
  for (int i = 0; i < m && f->cache_ok; ++i) {
    Device& d = f->dev[i];
    if (!d.local) continue;
    d.mrows.clear();
    for (int j = 0; j < n; ++j) {
      if (!f->sets[i][j].has_dest) { f->cache_ok = false; break; }
      d.mrows.insert(d.mrows.end(), f->sets[i][j].dest.begin(), f->sets[i][j].dest.end());
    }
    std::sort(d.mrows.begin(), d.mrows.end());
    d.mrows.erase(std::unique(d.mrows.begin(), d.mrows.end()), d.mrows.end());
    d.mcount = (int64_t)d.mrows.size();
    auto pos_of = [&](int64_t v, int64_t* out) {
      auto it = std::lower_bound(d.mrows.begin(), d.mrows.end(), v);
      if (it == d.mrows.end() || *it != v) return false;
      *out = it - d.mrows.begin();
      return true;
    };
    for (int j = 0; j < n && f->cache_ok; ++j) {
      HostSets& h = f->sets[i][j];
      DevChunk& c = d.chunks[j];
      c.dest_m0 = -1;
      if (!h.dest.empty()) {
        int64_t p0;
        if (!pos_of(h.dest[0], &p0) || p0 + (int64_t)h.dest.size() > d.mcount ||
            !std::equal(h.dest.begin(), h.dest.end(), d.mrows.begin() + p0)) {
          f->cache_ok = false;
          break;
        }
        c.dest_m0 = p0;
      } else {
        c.dest_m0 = 0;
      }
      const auto& rows = f->mode == HT_MODE_FULL ? h.load : h.owned;
      std::vector<int64_t> pm(rows.size());
      for (size_t q = 0; q < rows.size(); ++q)
        if (!pos_of(rows[q], &pm[q])) { f->cache_ok = false; break; }
      if (f->cache_ok) HT_TRY(upload(c.h2d_m, pm, d.stream));
    }
    if (!f->cache_ok) break;
    HT_TRY(upload(d.mrows_d, d.mrows, d.stream));
    std::vector<int64_t> pos(d.mcount);
    std::iota(pos.begin(), pos.end(), 0);
    make_runs(d.own, d.mrows, pos, nullptr);
  }

  // owner-side push and flush lists
  if (!base) {
    std::vector<uint8_t> flushed;
    for (int j = 0; j < n; ++j) {
      for (int k = 0; k < m; ++k) {
        Device& d = f->dev[k];
        if (!d.local) continue;  // rank mode: a peer process drives it
        HT_TRY(set_dev(d));
        cudaStream_t s = d.stream;
        DevChunk& c = d.chunks[j];
        HostSets& hk = f->sets[k][j];
        c.push.assign(m, CopyList());
        for (int i = 0; i < m; ++i) {
          HostSets& hi = f->sets[i][j];
          std::vector<int64_t> rows = (i == k) ? visect(hk.nbr, hk.owned) : hi.fetch[k];
          std::vector<int64_t> pos(rows.size()), slot;
          for (size_t q = 0; q < rows.size(); ++q) {
            auto it = std::lower_bound(hi.nbr.begin(), hi.nbr.end(), rows[q]);
            if (it == hi.nbr.end() || *it != rows[q])
              return fail(HT_EINVAL, "fetch row %lld not in N_%d%d", (long long)rows[q], i, j);
            pos[q] = it - hi.nbr.begin();
          }
          HT_TRY(lookup_slots(hk, rows, slot, k, j));
          HT_TRY(upload_list(c.push[i], pos, slot, s));
        }
        std::vector<int64_t> fl;
        if (f->mode == HT_MODE_P2P || f->flush == HT_FLUSH_EVERY_BATCH || j + 1 == n) fl = hk.owned;
        else fl = vdiff(hk.owned, f->sets[k][j + 1].owned);
        std::vector<int64_t> slot;
        HT_TRY(lookup_slots(hk, fl, slot, k, j));
        std::vector<uint8_t> first(fl.size());
        for (size_t q = 0; q < fl.size(); ++q) {
          const int64_t v = fl[q];
          if ((int64_t)flushed.size() <= v) flushed.resize(v + 1, 0);
          first[q] = flushed[v] ? 0 : 1;
          flushed[v] = 1;
        }
        HT_TRY(upload_list(c.flush, slot, fl, s, &first));
        make_runs(c.flush, fl, slot, &first);
        if (f->cache_ok) {  // flush rows as mirror positions
          std::vector<int64_t> fm(fl.size());
          for (size_t q = 0; q < fl.size(); ++q) {
            auto it = std::lower_bound(d.mrows.begin(), d.mrows.end(), fl[q]);
            if (it == d.mrows.end() || *it != fl[q]) { f->cache_ok = false; break; }
            fm[q] = it - d.mrows.begin();
          }
          HT_TRY(upload(c.flush_m, fm, s));
        }
      }
    }
  }
  HT_TRY(sync_all(f));
  f->finalized = true;
  return HT_OK;
}

extern "C" int ht_fleet_capacity(ht_fleet* f, int i, int64_t* cap) {
  if (i < 0 || i >= f->m) return fail(HT_EINVAL, "device index out of range");
  *cap = f->dev[i].cap;
  return HT_OK;
}

extern "C" int ht_fleet_sync(ht_fleet* f) {
  HT_TRY(sync_all(f));
  timers_collect(f);
  return HT_OK;
}

extern "C" int ht_begin_layer(ht_fleet* f, int dim, int elem_size, int backward) {
  if (!f->finalized) return fail(HT_ESTATE, "fleet not finalized");
  if (elem_size != 4 && elem_size != 8) return fail(HT_EINVAL, "element size must be 4 or 8");
  f->dim = dim;
  f->elem = elem_size;
  for (auto& d : f->dev) {
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    const int64_t bytes = d.cap * (int64_t)dim * elem_size;
    HT_TRY(d.value.ensure(bytes));
    if (backward && f->mode != HT_MODE_BASELINE) {
      HT_TRY(d.grad.ensure(bytes));
      if (bytes) CU(cudaMemsetAsync(d.grad.p, 0, bytes, d.stream));
    }
  }
  return HT_OK;
}

// ===========================================================================
// communication steps (Alg. 2 / Alg. 3)
// ===========================================================================
namespace {

// step 1 + barrier + step 2 + barrier of dedup_comm_fwd for batch j
int stage_batch(ht_fleet* f, int j, const void* host_rows_dev) {
  const int64_t rb = (int64_t)f->dim * f->elem;
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    HT_TRY(set_dev(d));
    DevChunk& c = d.chunks[j];
    TimerRec tr;
    timer_begin(f, d, tr);
    HT_TRY(launch_copy(d.stream, d.value.p, host_rows_dev, c.h2d.dst.as<int64_t>(),
                       c.h2d.src.as<int64_t>(), c.h2d.n, rb, rb, rb));
    timer_end(f, d, tr, 3, (double)c.h2d.n * rb);
  }
  if (f->mode == HT_MODE_BASELINE || f->m == 1) return HT_OK;
  HT_TRY(barrier(f));
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    HT_TRY(set_dev(d));
    DevChunk& c = d.chunks[j];
    for (int st = 1; st < f->m; ++st) {
      const int k = (i + st) % f->m;
      const CopyList& cl = c.d2d[st];
      HT_TRY(launch_copy(d.stream, d.value.p, f->dev[k].value.p, cl.dst.as<int64_t>(),
                         cl.src.as<int64_t>(), cl.n, rb, rb, rb));
    }
  }
  return barrier(f);
}

// push views (device-resident, per device in d.se at row stride dim) to the
// owners, then flush.  assume_zero: first flush of a row stores.
// layer >= 0 and the device caches: flush into its grad mirror of `layer`
int push_flush(ht_fleet* f, int j, void* host_grad_dev, bool assume_zero, int layer = -1) {
  const int dim = f->dim;
  if (f->mode == HT_MODE_BASELINE) {
    // host_grad[N_ij] += view_i in ascending device order
    for (int i = 0; i < f->m; ++i) {
      Device& d = f->dev[i];
      HT_TRY(set_dev(d));
      if (i > 0) CU(cudaStreamWaitEvent(d.stream, f->dev[i - 1].ev, 0));
      const CopyList& cl = d.chunks[j].base_bwd;
      HT_TRY(launch_acc(d.stream, f->elem, host_grad_dev, d.se.p, cl.dst.as<int64_t>(),
                        cl.src.as<int64_t>(), nullptr, cl.n, dim, 0));
      CU(cudaEventRecord(d.ev, d.stream));
    }
    HT_TRY(barrier(f));
    if (j == f->n - 1)
      for (auto& d : f->dev) {
        HT_TRY(set_dev(d));
        for (int g = 0; g < kChunks; ++g) HT_TRY(ev_rec(d.e_fchunk[g], d.stream));
      }
    return HT_OK;
  }
  HT_TRY(barrier(f));
  for (int k = 0; k < f->m; ++k) {
    Device& d = f->dev[k];
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    DevChunk& c = d.chunks[j];
    for (int i = 0; i < f->m; ++i) {  // ascending source device
      const CopyList& cl = c.push[i];
      HT_TRY(launch_acc(d.stream, f->elem, d.grad.p, f->dev[i].se.p, cl.dst.as<int64_t>(),
                        cl.src.as<int64_t>(), nullptr, cl.n, dim, 0));
    }
    const CopyList& fl = c.flush;
    const int64_t rb = (int64_t)dim * f->elem;
    const bool lastb = j == f->n - 1;
    if (layer >= 0 && d.cache) {
      // mirror zeroed at layer start: first flushes store, re-flushes add;
      // the host copy is written through once per layer
      HT_TRY(launch_acc(d.stream, f->elem, d.mg[layer].p, d.grad.p, c.flush_m.as<int64_t>(),
                        fl.src.as<int64_t>(), assume_zero ? fl.flag.as<uint8_t>() : nullptr, fl.n,
                        dim, 1));
    } else if (assume_zero && fl.dma) {
      // every row is a first flush (a store): copy engines, chunked so the
      // next layer can start loading finished chunks
      for (int g = 0; g < kChunks; ++g) {
        HT_TRY(xfer(d.stream, fl, true, host_grad_dev, rb, d.grad.p, rb, rb,
                    chunk_bound(f->nrows, g), chunk_bound(f->nrows, g + 1)));
        if (lastb) HT_TRY(ev_rec(d.e_fchunk[g], d.stream));
      }
      if (!lastb)  // flushed slots restart from zero (devices.py:339)
        for (size_t r = 0; r < fl.run_len.size(); ++r)
          CU(cudaMemsetAsync(static_cast<char*>(d.grad.p) + fl.run_dev[r] * rb, 0,
                             fl.run_len[r] * rb, d.stream));
    } else {
      HT_TRY(launch_acc(d.stream, f->elem, host_grad_dev, d.grad.p, fl.dst.as<int64_t>(),
                        fl.src.as<int64_t>(), assume_zero ? fl.flag.as<uint8_t>() : nullptr, fl.n,
                        dim, 1));
      if (lastb)
        for (int g = 0; g < kChunks; ++g) HT_TRY(ev_rec(d.e_fchunk[g], d.stream));
    }
  }
  return barrier(f);
}

}  // namespace

extern "C" int ht_comm_fwd(ht_fleet* f, int batch, const void* host_rows, void* views_out) {
  if (batch < 0 || batch >= f->n) return fail(HT_EINVAL, "batch out of range");
  if (f->rank >= 0) return fail(HT_ESTATE, "per-batch fleet calls need a single-process fleet");
  void *hsrc, *vout;
  HT_TRY(dev_ptr(host_rows, &hsrc));
  HT_TRY(dev_ptr(views_out, &vout));
  HT_TRY(stage_batch(f, batch, hsrc));
  const int64_t rb = (int64_t)f->dim * f->elem;
  int64_t base = 0;
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    HT_TRY(set_dev(d));
    DevChunk& c = d.chunks[batch];
    HT_TRY(launch_copy(d.stream, vout, d.value.p, nullptr, c.nbr_slot.as<int64_t>(), c.nn, rb, rb,
                       rb, base));
    base += c.nn;
  }
  return sync_all(f);
}

extern "C" int ht_comm_bwd(ht_fleet* f, int batch, const void* views_in, void* host_grad) {
  if (batch < 0 || batch >= f->n) return fail(HT_EINVAL, "batch out of range");
  if (f->rank >= 0) return fail(HT_ESTATE, "per-batch fleet calls need a single-process fleet");
  void *vin, *hg;
  HT_TRY(dev_ptr(views_in, &vin));
  HT_TRY(dev_ptr(host_grad, &hg));
  const int64_t rb = (int64_t)f->dim * f->elem;
  int64_t base = 0;
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    HT_TRY(set_dev(d));
    DevChunk& c = d.chunks[batch];
    HT_TRY(d.se.ensure(std::max<int64_t>(1, c.nn) * rb));
    if (c.nn)
      CU(cudaMemcpyAsync(d.se.p, (const char*)vin + base * rb, c.nn * rb, cudaMemcpyDefault,
                         d.stream));
    base += c.nn;
  }
  HT_TRY(push_flush(f, batch, hg, false));
  return sync_all(f);
}

extern "C" int ht_dest_rows(ht_fleet* f, int op, int batch, int dim, int elem_size, void* host_rows,
                            void* rows_concat) {
  if (batch < 0 || batch >= f->n) return fail(HT_EINVAL, "batch out of range");
  if (f->rank >= 0) return fail(HT_ESTATE, "per-batch fleet calls need a single-process fleet");
  void *hp, *rp;
  HT_TRY(dev_ptr(host_rows, &hp));
  HT_TRY(dev_ptr(rows_concat, &rp));
  const int64_t rb = (int64_t)dim * elem_size;
  int64_t base = 0;
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    HT_TRY(set_dev(d));
    DevChunk& c = d.chunks[batch];
    if (!f->sets[i][batch].has_dest)
      return fail(HT_EINVAL, "plan carries no destination sets; build it from a partition");
    const int64_t* rows = c.dest_rows.as<int64_t>();
    if (op == 0)
      HT_TRY(launch_copy(d.stream, rp, hp, nullptr, rows, c.nv, rb, rb, rb, base));
    else if (op == 1)
      HT_TRY(launch_copy(d.stream, (char*)hp, (char*)rp + base * rb, rows, nullptr, c.nv, rb, rb, rb));
    else {
      // ascending device order on one stream chain
      if (i > 0) CU(cudaStreamWaitEvent(d.stream, f->dev[i - 1].ev, 0));
      HT_TRY(launch_acc(d.stream, elem_size, hp, rp, rows, nullptr, nullptr, c.nv, dim, 0, base));
      CU(cudaEventRecord(d.ev, d.stream));
    }
    base += c.nv;
  }
  return sync_all(f);
}

// ===========================================================================
// GCN epoch
//
// Three streams per device: `stream` (compute + peer traffic), `tin`
// (host -> device rows) and `tout` (device -> host rows).  Events order
// them; nothing in a layer call synchronizes the host, so host loads of the
// next batch / layer, device compute and host stores of the previous batch
// overlap (PCIe is full duplex).  Staging buffers alternate between two sets
// by an epoch-wide batch counter.
// ===========================================================================
namespace {

// weights of layer l into the per-layer device buffers (async, from a
// pinned host scratch): W, W^T and W padded, plus the TF32 hi/lo halves
int upload_layer_weights(Device& d, int l, const float* W, int d_in, int d_out) {
  LayerW& w = d.lw[l];
  const int64_t nw = (int64_t)d_in * d_out;
  const int ldo = pad4(d_out);
  const int64_t np = (int64_t)d_in * ldo;
  float* wt = d.wpin + d.wpin_off[l];
  float* wn = wt + nw;
  float* wp = wn + nw;
  std::memcpy(wn, W, nw * 4);
  for (int a = 0; a < d_in; ++a)
    for (int b = 0; b < ldo; ++b) {
      if (b < d_out) wt[(int64_t)b * d_in + a] = W[(int64_t)a * d_out + b];
      wp[(int64_t)a * ldo + b] = b < d_out ? W[(int64_t)a * d_out + b] : 0.f;
    }
  for (DBuf* b : {&w.W, &w.Wt, &w.Wt_hi, &w.Wt_lo}) HT_TRY(b->ensure(nw * 4));
  for (DBuf* b : {&w.Wp, &w.Wp_hi, &w.Wp_lo}) HT_TRY(b->ensure(np * 4));
  CU(cudaMemcpyAsync(w.W.p, wn, nw * 4, cudaMemcpyHostToDevice, d.stream));
  CU(cudaMemcpyAsync(w.Wt.p, wt, nw * 4, cudaMemcpyHostToDevice, d.stream));
  CU(cudaMemcpyAsync(w.Wp.p, wp, np * 4, cudaMemcpyHostToDevice, d.stream));
  HT_TRY(ht::tc::split_weights(d.stream, w.Wt.as<float>(), w.Wt_hi.as<float>(), w.Wt_lo.as<float>(), nw));
  HT_TRY(ht::tc::split_weights(d.stream, w.Wp.as<float>(), w.Wp_hi.as<float>(), w.Wp_lo.as<float>(), np));
  count_launch(2);
  w.valid = true;
  return HT_OK;
}

int check_chunks(ht_fleet* f) {
  for (int i = 0; i < f->m; ++i)
    for (int j = 0; j < f->n; ++j)
      if (!f->sets[i][j].has_chunk || !f->sets[i][j].has_dest)
        return fail(HT_ESTATE, "chunk (%d,%d) has no graph structure uploaded", i, j);
  return HT_OK;
}

// The output rows h^{layer+1} of chunk j as they sit in HBM (the last
// layer's device copy, the owner-cache mirror, or an HBM host store), or
// nullptr when only pinned host memory holds them.  *rows: row indices
// into the returned array (nullptr = consecutive).
const float* hbm_outputs(ht_fleet* f, Device& d, int j, int layer, int d_out,
                         const int64_t** rows) {
  *rows = nullptr;
  DevChunk& c = d.chunks[j];
  if (layer + 1 == f->L) return d.hL.as<float>() + d.hL_off[j] * d_out;
  if (d.cache) return d.mh[layer + 1].as<float>() + c.dest_m0 * d_out;
  if ((int)f->hdev.size() > layer + 1 && f->hdev[layer + 1]) {
    *rows = c.dest_rows.as<int64_t>();
    return static_cast<const float*>(f->hptr[layer + 1]);
  }
  return nullptr;
}

// m = 1: the layer input h^l as an HBM array indexed by global row (the
// owner-cache mirror when it is the identity map, or an HBM host store),
// or nullptr.  The gathers then read it in place: no slot loads.
const float* hbm_inputs(ht_fleet* f, Device& d, int layer, const void* hin) {
  if (f->m != 1 || !d.chunks[0].csc_gid.p || getenv("HT_NO_DIRECT_READ")) return nullptr;
  if (d.cache && d.mcount == f->nrows && (d.mrows.empty() || d.mrows.back() == d.mcount - 1))
    return d.mh[layer].as<float>();
  if (is_dev_mem(hin)) return static_cast<const float*>(hin);
  return nullptr;
}

// One device, one batch, identity-mapped mirror: the neighbour-gradient
// views go straight to their grad mirror rows (scatter by global row) - the
// owner push into the slot buffer and the flush out of it would move the
// same rows twice.  Bitwise the reference's order: each row's first flush
// is a store (GCN), or follows the destination-gradient add (GAT).
bool direct_bwd(ht_fleet* f, Device& d) {
  return f->m == 1 && f->n == 1 && d.cache && d.chunks[0].nbr_gid.p && d.mcount == f->nrows &&
         (d.mrows.empty() || d.mrows.back() == d.mcount - 1) && !getenv("HT_NO_DIRECT_BWD");
}

// GAT with one device, one batch and the identity-mapped mirror: N_ij is a
// subset of V_ij = every host row, so q = h_nbr.W is p = h.W row for row
// (bitwise: the same input row times the same W).  The projections run once
// over all rows, the edge kernels index p by global row, the CSR pass runs
// over the expanded offsets (gq / gts in global row order, zero rows for
// rows without out-edges) and the input gradients land in the grad mirror
// directly.  ∇W and ∇a sum over all rows (rows without out-edges add zeros):
// the same sums in a different association than the staged path.
bool gat_direct(ht_fleet* f, Device& d) {
  const DevChunk& c = d.chunks[0];
  return !getenv("HT_NO_GAT_DIRECT") && direct_bwd(f, d) && c.bx_rows == d.mcount && c.nv == d.mcount && c.dest_m0 == 0;
}

// Project-first GCN layer (d_out < d_in, one device, one batch, identity
// mirror, HBM checkpoints): z = A.(h.W) instead of (A.h).W - the gather
// moves pad4(d_out)-wide rows instead of d_in-wide ones (47 vs 256 floats
// for the last cfg-2 layer).  The same product reassociated (TF32 3x GEMM,
// FP32 sums); the backward then takes dW = h^T (A^T gz) (rows the narrow-side
// pass computes anyway) and agg^l is only formed if host.agg[l] is read.
bool project_first(ht_fleet* f, Device& d, int d_in, int d_out, int precision) {
  const DevChunk& c = d.chunks[0];
  return precision == HT_PREC_TF32 && d_out < d_in && f->ckpt_hbm && !f->gat &&
         direct_bwd(f, d) && c.bx_rows == d.mcount && c.nv == d.mcount && c.dest_m0 == 0 &&
         !getenv("HT_NO_PROJECT_FIRST");
}

// HBM owner cache: owned rows of a host array -> mirror (on `s`)
int cache_upload(ht_fleet* f, Device& d, cudaStream_t s, const void* host, float* mirror,
                 int64_t rb) {
  if (host == mirror) return HT_OK;  // an aliased HBM store is its own mirror
  if (f->host_compact) {  // host array = owned rows in mirror order
    if (d.mcount) CU(cudaMemcpyAsync(mirror, host, d.mcount * rb, cudaMemcpyDefault, s));
    return HT_OK;
  }
  if (d.own.dma)
    return xfer(s, d.own, false, const_cast<void*>(host), rb, mirror, rb, rb, 0, f->nrows);
  return launch_copy(s, mirror, host, nullptr, d.mrows_d.as<int64_t>(), d.mcount, rb, rb, rb, 0,
                     kHostGrid);
}

// HBM owner cache: write a mirror through to the host rows (on tout, after
// everything enqueued so far on the compute stream)
int cache_writeback(ht_fleet* f, Device& d, void* host, const float* mirror, int64_t rb) {
  if (host == mirror) return HT_OK;  // aliased HBM store
  HT_TRY(ev_rec(d.e_mg, d.stream));
  HT_TRY(ev_wait(d.tout, d.e_mg));
  if (f->host_compact) {
    if (d.mcount) CU(cudaMemcpyAsync(host, mirror, d.mcount * rb, cudaMemcpyDefault, d.tout));
    return HT_OK;
  }
  if (d.own.dma)
    return xfer(d.tout, d.own, true, host, rb, const_cast<float*>(mirror), rb, rb, 0, f->nrows);
  return launch_copy(d.tout, host, mirror, d.mrows_d.as<int64_t>(), nullptr, d.mcount, rb, rb, rb,
                     0, kHostGrid);
}

// Destination rows of chunk c (in destination order at `dev`) -> the host
// array: host-row chunk g (the GEMM / store pipelining unit), or all rows
// for g < 0.  Copy-engine runs, the zero-copy kernel (all rows at g <= 0),
// or - compact host arrays - one contiguous copy at the mirror position.
int put_dest(ht_fleet* f, DevChunk& c, cudaStream_t s, void* host, const float* dev, int64_t rb,
             int g) {
  // rows already in place (an aliased HBM store written directly)
  if (c.dest_m0 >= 0 && reinterpret_cast<const char*>(dev) == static_cast<char*>(host) + c.dest_m0 * rb)
    return HT_OK;
  if (f->host_compact) {
    int64_t r0 = 0, r1 = c.nv;
    if (g >= 0) {
      if (c.dest_pos.empty()) {
        if (g > 0) return HT_OK;
      } else {
        r0 = c.dest_pos[g];
        r1 = c.dest_pos[g + 1];
      }
    }
    if (r1 > r0)
      CU(cudaMemcpyAsync(static_cast<char*>(host) + (c.dest_m0 + r0) * rb,
                         reinterpret_cast<const char*>(dev) + r0 * rb, (r1 - r0) * rb,
                         cudaMemcpyDefault, s));
    return HT_OK;
  }
  if (c.dest.dma) {
    for (int gg = g < 0 ? 0 : g; gg < (g < 0 ? kChunks : g + 1); ++gg)
      HT_TRY(xfer(s, c.dest, true, host, rb, const_cast<float*>(dev), rb, rb,
                  chunk_bound(f->nrows, gg), chunk_bound(f->nrows, gg + 1)));
    return HT_OK;
  }
  if (g > 0) return HT_OK;
  return launch_copy(s, host, dev, c.dest_rows.as<int64_t>(), nullptr, c.nv, rb, rb, rb, 0,
                     kHostGrid);
}

// K6, early: reload the checkpoint rows of `layer` into their per-layer
// device buffer on the low-priority prefetch stream, chunk by chunk as the
// stores land.  The backward then reads them from HBM.
int prefetch_checkpoints(ht_fleet* f, Device& d, int layer, void* aout, int64_t rbi) {
  float* ck = d.ck[layer].as<float>();
  const int dl = f->dims[layer];
  for (int j = 0; j < f->n; ++j) {
    DevChunk& c = d.chunks[j];
    float* dst = ck + d.hL_off[j] * dl;
    if (c.dest.dma) {
      for (int g = 0; g < kChunks; ++g) {
        if (j == 0) HT_TRY(ev_wait(d.tpre, d.e_aggst[layer * kChunks + g]));
        HT_TRY(xfer(d.tpre, c.dest, false, aout, rbi, dst, rbi, rbi, chunk_bound(f->nrows, g),
                    chunk_bound(f->nrows, g + 1)));
      }
    } else {
      if (j == 0) HT_TRY(ev_wait(d.tpre, d.e_aggst[layer * kChunks + kChunks - 1]));
      HT_TRY(launch_copy(d.tpre, dst, aout, nullptr, c.dest_rows.as<int64_t>(), c.nv, rbi, rbi,
                         rbi, 0, kHostGrid));
    }
  }
  return ev_rec(d.e_ck[layer], d.tpre);
}

// extra_grad: floats of further parameter gradients kept behind the weight
// gradients in the (IPC-shared) accumulator (GAT attention vectors)
int epoch_begin_impl(ht_fleet* f, int L, const int* dims, int64_t extra_grad, bool gat) {
  if (!f->finalized) return fail(HT_ESTATE, "fleet not finalized");
  HT_TRY(check_chunks(f));
  HT_TRY(sync_all(f));
  f->L = L;
  f->dims.assign(dims, dims + L + 1);
  f->hptr.assign(L + 1, nullptr);
  f->hdev.assign(L + 1, 0);
  f->agg_deferred.assign(L, 0);
  int dmax = 0;
  for (int l = 0; l <= L; ++l) dmax = std::max(dmax, pad4(dims[l]));
  for (auto& d : f->dev) {
    d.gW_off.assign(L + 1, 0);
    for (int l = 0; l < L; ++l) d.gW_off[l + 1] = d.gW_off[l] + (int64_t)dims[l] * dims[l + 1];
    if (!d.local) continue;  // a peer rank sizes and zeroes its own buffers
    HT_TRY(set_dev(d));
    HT_TRY(d.gWall.ensure((d.gW_off[L] + extra_grad) * 4));
    CU(cudaMemsetAsync(d.gWall.p, 0, (d.gW_off[L] + extra_grad) * 4, d.stream));
    if (f->rank >= 0 && !d.flags.p) {  // barrier counter: zeroed once, monotonic afterwards
      HT_TRY(d.flags.ensure(64));
      CU(cudaMemset(d.flags.p, 0, 64));
    }
    // every buffer of the epoch is sized here, once: no allocation (and no
    // implicit device synchronization) inside the layer calls
    int64_t mv = 1, mn = 1, np = 1;
    d.hL_off.assign(f->n + 1, 0);
    for (int j = 0; j < f->n; ++j) {
      mv = std::max(mv, d.chunks[j].nv);
      mn = std::max(mn, d.chunks[j].nn);
      np = std::max({np, d.chunks[j].fw_np, d.chunks[j].bw_np});
      d.hL_off[j + 1] = d.hL_off[j] + d.chunks[j].nv;
    }
    // sized for 180 GB of HBM: the buffers every path needs first, then
    // either the owner-cache mirrors or the host-path staging sets
    HT_TRY(d.grad.ensure(std::max<int64_t>(1, d.cap) * dmax * 4));
    HT_TRY(d.sc.ensure(mv * dmax * 4));
    HT_TRY(d.sd.ensure(mv * dmax * 4));
    HT_TRY(d.se.ensure(mn * dmax * 4));
    int narrow_w = 0;  // widest d_out of the layers whose backward runs narrow-side
    for (int l = 0; l < L; ++l)
      if (dims[l + 1] < dims[l]) narrow_w = std::max(narrow_w, pad4(dims[l + 1]));
    if (narrow_w)  // (the expanded CSR of one device / one batch has a row per host row)
      HT_TRY(d.tT.ensure(std::max<int64_t>(mn, f->m == 1 && f->n == 1 ? f->nrows : 0) * narrow_w * 4));
    HT_TRY(d.partial.ensure(np * dmax * 4));
    HT_TRY(d.gemm_ws.ensure((int64_t)kSplitsMax * dmax * dmax * 4));
    HT_TRY(d.hL.ensure(std::max<int64_t>(1, d.hL_off[f->n]) * pad4(dims[L]) * 4));
    // HBM owner cache: decided per epoch (requested mode, plan, free HBM).
    // An HBM store on one device with the identity row map *is* the mirror.
    d.cache = false;
    const bool alias = !f->alias_h.empty() && (int)f->alias_h.size() == L + 1 && f->cache_ok &&
                       f->m == 1 && d.mcount == f->nrows &&
                       (gat || (int)f->alias_a.size() == L);
    if (alias) {
      d.cache = true;
      d.mh.resize(L);
      d.ma.resize(gat ? 0 : L);
      d.mg.resize(L + 1);
      for (int l = 0; l < L; ++l) d.mh[l].set_alias(f->alias_h[l]);
      for (int l = 0; l < (gat ? 0 : L); ++l) d.ma[l].set_alias(f->alias_a[l]);
      for (int l = 0; l <= L; ++l) d.mg[l].set_alias(f->alias_g[l]);
    } else if (f->alias_h.empty() && f->cache_req != 0) {  // (an HBM store needs no mirror)
      if (!f->cache_ok) {
        if (f->cache_req == 1)
          return fail(HT_EINVAL, "HBM owner cache needs mode p2p/full and destination sets that "
                                 "are contiguous ranges of each device's owned rows");
      } else {
        int64_t per_row = 0;
        for (int l = 0; l < L; ++l) per_row += dims[l] * (gat ? 1 : 2);  // h (+ agg)
        for (int l = 0; l <= L; ++l) per_row += dims[l];                // grad
        int64_t need = d.mcount * per_row * 4;
        if (gat) {  // GAT staging allocated after this decision (ht_gat_epoch_begin)
          int64_t me = 1;
          for (int j = 0; j < f->n; ++j) me = std::max(me, d.chunks[j].ne);
          need += (3 * mn + 4 * mv) * (int64_t)dmax * 4 + 2 * me * 4 + 2 * me * 4;
        }
        size_t fr = 0, tot = 0;
        CU(cudaMemGetInfo(&fr, &tot));
        const bool fits = need + ((int64_t)4 << 30) <= (int64_t)fr;
        if (!fits && f->cache_req == 1)
          return fail(HT_ENOMEM, "HBM owner cache needs %lld bytes, %lld free", (long long)need,
                      (long long)fr);
        d.cache = fits;
      }
    }
    // the slot value buffer: not needed when a single device's gathers read
    // the identity-mapped mirror in place (hbm_inputs)
    const bool direct = d.cache && f->m == 1 && d.chunks[0].csc_gid.p &&
                        d.mcount == f->nrows && !getenv("HT_NO_DIRECT_READ");
    if (!direct) HT_TRY(d.value.ensure(std::max<int64_t>(1, d.cap) * dmax * 4));
    if (!d.cache)
      for (int s = 0; s < 2; ++s) {
        HT_TRY(d.fa[s].ensure(mv * dmax * 4));
        HT_TRY(d.fb[s].ensure(mv * dmax * 4));
        HT_TRY(d.ba[s].ensure(mv * dmax * 4));
        HT_TRY(d.bb[s].ensure(mv * dmax * 4));
      }
    if (f->host_compact && !d.cache)
      return fail(HT_EINVAL, "compact host arrays need the HBM owner cache (mode on/auto, and "
                             "enough free HBM for the mirrors)");
    if (d.cache && !alias) {
      d.mh.resize(L);
      d.ma.resize(gat ? 0 : L);
      d.mg.resize(L + 1);
      for (int l = 0; l < L; ++l) HT_TRY(d.mh[l].ensure(std::max<int64_t>(1, d.mcount) * dims[l] * 4));
      for (int l = 0; l < (gat ? 0 : L); ++l)
        HT_TRY(d.ma[l].ensure(std::max<int64_t>(1, d.mcount) * dims[l] * 4));
      for (int l = 0; l <= L; ++l) HT_TRY(d.mg[l].ensure(std::max<int64_t>(1, d.mcount) * dims[l] * 4));
    }
    if (f->prefetch && !d.cache) {
      if ((int)d.ck.size() < L) d.ck.resize(L);
      if ((int)d.e_ck.size() < L) d.e_ck.resize(L, nullptr);
      for (int l = 0; l < L; ++l)
        HT_TRY(d.ck[l].ensure(std::max<int64_t>(1, d.hL_off[f->n]) * dims[l] * 4));
    }
    // pinned scratch for weight uploads, one slot per layer
    d.wpin_off.assign(L + 1, 0);
    for (int l = 0; l < L; ++l)
      d.wpin_off[l + 1] = d.wpin_off[l] + 2 * (int64_t)dims[l] * dims[l + 1] +
                          (int64_t)dims[l] * pad4(dims[l + 1]);
    if (d.wpin_cap < d.wpin_off[L]) {
      if (d.wpin) cudaFreeHost(d.wpin);
      CU(cudaHostAlloc(reinterpret_cast<void**>(&d.wpin), d.wpin_off[L] * 4, cudaHostAllocPortable));
      d.wpin_cap = d.wpin_off[L];
    }
    d.lw.resize(L);
    for (auto& w : d.lw) w.valid = false;
    d.fwd_count = d.bwd_count = 0;
    if ((int)d.e_aggst.size() < L * kChunks) d.e_aggst.resize(L * kChunks, nullptr);
  }
  return HT_OK;
}

}  // namespace

extern "C" int ht_fleet_set_cache(ht_fleet* f, int mode) {
  if (mode < 0 || mode > 2) return fail(HT_EINVAL, "cache mode must be 0 (off), 1 (on) or 2 (auto)");
  f->cache_req = mode;
  return HT_OK;
}

extern "C" int ht_fleet_set_host_rows(ht_fleet* f, const int64_t* rows, int64_t n) {
  if (!rows || n <= 0) {
    f->host_compact = false;
    return HT_OK;
  }
  if (!f->finalized) return fail(HT_ESTATE, "fleet not finalized");
  int local = 0;
  for (auto& d : f->dev) local += d.local ? 1 : 0;
  if (local != 1) return fail(HT_EINVAL, "compact host arrays need a fleet with one local device");
  for (auto& d : f->dev)
    if (d.local) {
      if (!f->cache_ok || (int64_t)d.mrows.size() != n || !std::equal(rows, rows + n, d.mrows.begin()))
        return fail(HT_EINVAL, "compact host arrays must hold exactly the owned rows of the "
                               "fleet's device (ascending), and the plan must admit the cache");
    }
  f->host_compact = true;
  return HT_OK;
}

extern "C" int ht_fleet_alias_store(ht_fleet* f, int L, void* const* h, void* const* agg,
                                    void* const* grad) {
  f->alias_h.clear();
  f->alias_a.clear();
  f->alias_g.clear();
  if (!h) return HT_OK;
  for (int l = 0; l <= L; ++l) {
    if (!is_dev_mem(h[l]) || !is_dev_mem(grad[l]) || (agg && l < L && !is_dev_mem(agg[l])))
      return fail(HT_EINVAL, "aliased store arrays must be device memory");
  }
  f->alias_h.assign(h, h + L + 1);
  f->alias_g.assign(grad, grad + L + 1);
  if (agg) f->alias_a.assign(agg, agg + L);
  return HT_OK;
}

extern "C" int ht_fleet_set_lean(ht_fleet* f, int lean) {
  f->lean = lean != 0;
  return HT_OK;
}

extern "C" int ht_fleet_set_checkpoints(ht_fleet* f, int hbm) {
  f->ckpt_hbm = hbm != 0;
  return HT_OK;
}

extern "C" int ht_fleet_checkpoint_read(ht_fleet* f, int layer, void* host_agg) {
  if (layer < 0 || layer >= f->L || f->gat) return fail(HT_EINVAL, "no GCN checkpoint for that layer");
  void* hp;
  HT_TRY(dev_ptr(host_agg, &hp));
  const int64_t rb = (int64_t)f->dims[layer] * 4;
  const bool deferred = layer < (int)f->agg_deferred.size() && f->agg_deferred[layer];
  for (auto& d : f->dev) {
    if (!d.local) continue;
    if (!d.cache || (int)d.ma.size() <= layer || !d.ma[layer].p)
      return fail(HT_ESTATE, "checkpoints are not held in HBM mirrors");
    HT_TRY(set_dev(d));
    if (deferred) {  // project-first layer: agg^l = A.h^l now, the forward's gather
      const DevChunk& c = d.chunks[0];
      const int din = f->dims[layer];
      HT_TRY(launch_seg(d.stream, d.ma[layer].as<float>(), d.mh[layer].as<float>(), din, din,
                        c.csc_off.as<int64_t>(), c.csc_gid.as<int32_t>(), c.csc_w.as<float>(), c.nv,
                        c.fw_np, c.fw_lo, c.fw_hi, c.fw_nf, c.fw_seg, c.fw_first, c.fw_cnt,
                        d.partial.as<float>()));
    }
    HT_TRY(cache_writeback(f, d, hp, d.ma[layer].as<float>(), rb));
  }
  if (deferred) f->agg_deferred[layer] = 0;
  for (auto& d : f->dev)
    if (d.local) {
      HT_TRY(set_dev(d));
      CU(cudaStreamSynchronize(d.stream));
      CU(cudaStreamSynchronize(d.tout));
    }
  return HT_OK;
}

extern "C" int ht_fleet_cache_state(ht_fleet* f, int* on) {
  *on = 1;
  int any = 0;
  for (auto& d : f->dev)
    if (d.local) {
      any = 1;
      if (!d.cache) *on = 0;
    }
  if (!any) *on = 0;
  return HT_OK;
}

extern "C" int ht_epoch_begin(ht_fleet* f, int L, const int* dims) {
  HT_TRY(epoch_begin_impl(f, L, dims, 0, false));
  f->gat = false;
  return HT_OK;
}

extern "C" int ht_forward_layer(ht_fleet* f, int layer, int d_in, int d_out, const float* W,
                                const void* h_in, void* h_out, void* agg_out, int precision) {
  if (layer < 0 || layer >= f->L || f->dims[layer] != d_in || f->dims[layer + 1] != d_out)
    return fail(HT_EINVAL, "layer %d shape does not match ht_epoch_begin", layer);
  void *hin, *hout, *aout;
  HT_TRY(dev_ptr(h_in, &hin));
  HT_TRY(dev_ptr(h_out, &hout));
  HT_TRY(dev_ptr(agg_out, &aout));
  if (precision == HT_PREC_TF32 && (d_in & 3))
    return fail(HT_EINVAL, "tf32 path needs layer input widths divisible by 4 (got %d)", d_in);
  f->dim = d_in;
  f->elem = 4;
  const bool last = layer == f->L - 1;
  const int64_t rbi = (int64_t)d_in * 4, rbo = (int64_t)d_out * 4;
  f->hptr[layer + 1] = hout;
  f->hdev[layer + 1] = is_dev_mem(hout);
  for (auto& d : f->dev) {
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    HT_TRY(upload_layer_weights(d, layer, W, d_in, d_out));
  }
  if (last) f->hL_dim = d_out;
  for (int j = 0; j < f->n; ++j) {
    // ---- step 1: host loads into slots (tin) ----
    for (int i = 0; i < f->m; ++i) {
      Device& d = f->dev[i];
      if (!d.local) continue;  // rank mode: a peer process drives it
      HT_TRY(set_dev(d));
      DevChunk& c = d.chunks[j];
      if (d.cache) {  // owned rows come from the HBM mirror (compute stream)
        if (layer == 0 && j == 0) {
          HT_TRY(cache_upload(f, d, d.tin, hin, d.mh[0].as<float>(), rbi));
          HT_TRY(ev_rec(d.e_up, d.tin));
          HT_TRY(ev_wait(d.stream, d.e_up));
        }
        for (auto& o : f->dev) HT_TRY(ev_wait(d.stream, o.e_fetch));  // peers done with our slots
        if (!hbm_inputs(f, d, layer, hin))  // else K3 reads the mirror in place
          HT_TRY(launch_copy(d.stream, d.value.p, d.mh[layer].p, c.h2d.dst.as<int64_t>(),
                             c.h2d_m.as<int64_t>(), c.h2d.n, rbi, rbi, rbi));
        HT_TRY(ev_rec(d.e_in, d.stream));
        continue;
      }
      if (hbm_inputs(f, d, layer, hin)) {  // HBM store, one device: K3 reads it in place
        HT_TRY(ev_rec(d.e_in, d.stream));
        continue;
      }
      if (d.fwd_count > 0) {  // slots of the previous batch no longer read
        HT_TRY(ev_wait(d.tin, d.e_agg));
        for (auto& o : f->dev) HT_TRY(ev_wait(d.tin, o.e_fetch));
      }
      // h^l rows come from the previous layer's stores (every owner's in
      // baseline mode); with copy-engine lists each host-row chunk is
      // loaded as soon as it has been stored (D2H and H2D overlap)
      const bool after = j == 0 && layer > 0;
      TimerRec tr;
      timer_begin(f, d, tr, d.tin);
      if (c.h2d.dma) {
        for (int g = 0; g < kChunks; ++g) {
          if (after)
            for (auto& o : f->dev) HT_TRY(ev_wait(d.tin, o.e_hchunk[g]));
          HT_TRY(xfer(d.tin, c.h2d, false, hin, rbi, d.value.p, rbi, rbi,
                      chunk_bound(f->nrows, g), chunk_bound(f->nrows, g + 1)));
        }
      } else {
        if (after)
          for (auto& o : f->dev) HT_TRY(ev_wait(d.tin, o.e_hchunk[kChunks - 1]));
        HT_TRY(launch_copy(d.tin, d.value.p, hin, c.h2d.dst.as<int64_t>(), c.h2d.src.as<int64_t>(),
                           c.h2d.n, rbi, rbi, rbi, 0, kHostGrid));
      }
      timer_end(f, d, tr, 3, (double)c.h2d.n * rbi, d.tin);
      HT_TRY(ev_rec(d.e_in, d.tin));
    }
    // ---- barrier + step 2: staggered peer fetches (compute stream) ----
    for (int i = 0; i < f->m; ++i) {
      Device& d = f->dev[i];
      if (!d.local) continue;  // rank mode: a peer process drives it
      HT_TRY(set_dev(d));
      DevChunk& c = d.chunks[j];
      for (auto& o : f->dev) HT_TRY(ev_wait(d.stream, o.e_in));
      if (f->rank >= 0 && f->m > 1) HT_TRY(xbarrier(f));  // every rank's hosted rows staged
      if (f->mode != HT_MODE_BASELINE)
        for (int st = 1; st < f->m; ++st) {
          const int k = (i + st) % f->m;
          const CopyList& cl = c.d2d[st];
          HT_TRY(launch_copy(d.stream, d.value.p, f->dev[k].value.p, cl.dst.as<int64_t>(),
                             cl.src.as<int64_t>(), cl.n, rbi, rbi, rbi));
        }
      if (f->rank >= 0 && f->m > 1) HT_TRY(xbarrier(f));  // peers done reading our slots
      HT_TRY(ev_rec(d.e_fetch, d.stream));
    }
    // ---- aggregation, dense transform, stores (tout) ----
    for (int i = 0; i < f->m; ++i) {
      Device& d = f->dev[i];
      if (!d.local) continue;  // rank mode: a peer process drives it
      HT_TRY(set_dev(d));
      DevChunk& c = d.chunks[j];
      const int s = (int)(d.fwd_count & 1);
      if (d.fwd_count >= 2 && !d.cache) HT_TRY(ev_wait(d.stream, d.e_out[s]));  // staging set s drained
      const bool lastb = j == f->n - 1;
      if (hbm_inputs(f, d, layer, hin) && project_first(f, d, d_in, d_out, precision)) {
        // z = A.(h.W): the narrow projection of every row first, then the
        // CSC gather over pad4(d_out)-wide rows, then ReLU into h^{l+1}
        const int ldp = pad4(d_out);
        const int64_t rows = d.mcount;
        HT_TRY(d.pf_p.ensure(rows * ldp * 4));
        HT_TRY(d.pf_z.ensure(rows * ldp * 4));
        if (ldp != d_out) CU(cudaMemsetAsync(d.pf_p.p, 0, rows * ldp * 4, d.stream));  // pad column
        LayerW& w = d.lw[layer];
        TimerRec tg;
        timer_begin(f, d, tg, d.stream);
        HT_TRY(ht::tc::rows<ht::tc::TC_STORE>(d.stream, true, hbm_inputs(f, d, layer, hin), d_in,
                                              rows, d_in, w.Wt_hi.as<float>(), w.Wt_lo.as<float>(),
                                              d_in, d_out, d.pf_p.as<float>(), ldp, nullptr, 0));
        timer_end(f, d, tg, 2, 2.0 * rows * d_in * d_out, d.stream);
        TimerRec tr;
        timer_begin(f, d, tr, d.stream);
        HT_TRY(launch_seg(d.stream, d.pf_z.as<float>(), d.pf_p.as<float>(), ldp, ldp,
                          c.csc_off.as<int64_t>(), c.csc_gid.as<int32_t>(), c.csc_w.as<float>(),
                          c.nv, c.fw_np, c.fw_lo, c.fw_hi, c.fw_nf, c.fw_seg, c.fw_first, c.fw_cnt,
                          d.partial.as<float>()));
        timer_end(f, d, tr, 0, (double)c.ne * (8.0 + 4.0 * ldp) + (double)c.nv * (4.0 * ldp + 4.0),
                  d.stream);
        HT_TRY(ev_rec(d.e_agg, d.stream));
        float* hdst = last ? d.hL.as<float>() + d.hL_off[j] * d_out
                           : d.mh[layer + 1].as<float>() + c.dest_m0 * d_out;
        count_launch(3);
        ht::k_relu_rows<<<grid_for(c.nv * (int64_t)d_out / 32 + 1), kThreads, 0, d.stream>>>(
            hdst, d_out, d.pf_z.as<float>(), ldp, c.nv, d_out);
        CU(cudaGetLastError());
        HT_TRY(ev_rec(d.e_comp, d.stream));
        HT_TRY(ev_wait(d.tout, d.e_comp));
        if (!(last && f->lean && d.cache)) HT_TRY(put_dest(f, c, d.tout, hout, hdst, rbo, -1));
        if (lastb)
          for (int g = 0; g < kChunks; ++g) {
            HT_TRY(ev_rec(d.e_hchunk[g], d.tout));
            HT_TRY(ev_rec(d.e_aggst[layer * kChunks + g], d.tout));
          }
        HT_TRY(ev_rec(d.e_out[s], d.tout));
        f->agg_deferred[layer] = 1;  // agg^l formed only if host.agg[l] is read
        d.fwd_count++;
        continue;
      }
      // cache: the aggregation and h rows land in their mirrors directly
      float* agg = d.cache ? d.ma[layer].as<float>() + c.dest_m0 * d_in : d.fa[s].as<float>();
      TimerRec tr;
      timer_begin(f, d, tr, d.stream);
      const float* Xd = hbm_inputs(f, d, layer, hin);
      HT_TRY(launch_seg(d.stream, agg, Xd ? Xd : d.value.as<float>(), d_in, d_in,
                        c.csc_off.as<int64_t>(),
                        Xd ? c.csc_gid.as<int32_t>() : c.csc_slot.as<int32_t>(), c.csc_w.as<float>(),
                        c.nv, c.fw_np, c.fw_lo,
                        c.fw_hi, c.fw_nf, c.fw_seg, c.fw_first, c.fw_cnt, d.partial.as<float>()));
      timer_end(f, d, tr, 0, (double)c.ne * (8.0 + 4.0 * d_in) + (double)c.nv * (4.0 * d_in + 4.0),
                d.stream);
      HT_TRY(ev_rec(d.e_agg, d.stream));
      float* hdst = last     ? d.hL.as<float>() + d.hL_off[j] * d_out
                    : d.cache ? d.mh[layer + 1].as<float>() + c.dest_m0 * d_out
                              : d.fb[s].as<float>();
      LayerW& w = d.lw[layer];
      const int64_t* rows = c.dest_rows.as<int64_t>();
      // K4 in host-row chunks when the destination rows are copy-engine
      // runs: chunk g's h rows go to the host (K5) while chunk g+1 computes
      const int nck = c.dest_pos.empty() ? 1 : kChunks;
      for (int g = 0; g < nck; ++g) {
        const int64_t r0 = nck > 1 ? c.dest_pos[g] : 0, r1 = nck > 1 ? c.dest_pos[g + 1] : c.nv;
        if (r1 > r0) {
          TimerRec tg;
          timer_begin(f, d, tg, d.stream);
          if (precision == HT_PREC_TF32) {
            HT_TRY(ht::tc::rows<ht::tc::TC_RELU>(d.stream, true, agg + r0 * d_in, d_in, r1 - r0,
                                                 d_in, w.Wt_hi.as<float>(), w.Wt_lo.as<float>(),
                                                 d_in, d_out, hdst + r0 * d_out, d_out, nullptr, 0));
          } else {
            HT_TRY((gemm<false, false, ht::EPI_RELU>(d.stream, agg + r0 * d_in, d_in,
                                                     w.W.as<float>(), d_out, hdst + r0 * d_out,
                                                     d_out, nullptr, 0, r1 - r0, d_out, d_in, 1,
                                                     d_in)));
          }
          timer_end(f, d, tg, 2, 2.0 * (r1 - r0) * d_in * d_out, d.stream);
        }
        if (nck > 1) {
          HT_TRY(ev_rec(d.e_gchunk[g], d.stream));
          HT_TRY(ev_wait(d.tout, d.e_gchunk[g]));
          if (!(last && f->lean && d.cache)) HT_TRY(put_dest(f, c, d.tout, hout, hdst, rbo, g));
          if (lastb) HT_TRY(ev_rec(d.e_hchunk[g], d.tout));
        }
      }
      HT_TRY(ev_rec(d.e_comp, d.stream));
      // K5: (remaining) destination rows, then checkpoint rows, to the host store
      HT_TRY(ev_wait(d.tout, d.e_comp));
      if (nck == 1)
        for (int g = 0; g < kChunks; ++g) {
          if (!(last && f->lean && d.cache)) HT_TRY(put_dest(f, c, d.tout, hout, hdst, rbo, g));
          if (lastb) HT_TRY(ev_rec(d.e_hchunk[g], d.tout));
        }
      // checkpoint rows, chunked: the first backward layer reloads the last
      // forward layer's checkpoints chunk by chunk as they land
      for (int g = 0; g < kChunks; ++g) {
        if (!(d.cache && f->ckpt_hbm)) HT_TRY(put_dest(f, c, d.tout, aout, agg, rbi, g));
        if (lastb) HT_TRY(ev_rec(d.e_aggst[layer * kChunks + g], d.tout));
      }
      (void)rows;
      HT_TRY(ev_rec(d.e_out[s], d.tout));
      if (lastb && f->prefetch && !d.cache) HT_TRY(prefetch_checkpoints(f, d, layer, aout, rbi));
      d.fwd_count++;
    }
  }
  return HT_OK;
}

extern "C" int ht_loss(ht_fleet* f, int d_last, const int64_t* labels, const uint8_t* mask,
                       int64_t V, int64_t count, void* grad_out, double* loss) {
  if (f->hL_dim != d_last) return fail(HT_ESTATE, "loss before the last forward layer");
  void* gout;
  HT_TRY(dev_ptr(grad_out, &gout));
  f->loss_count = count;
  const int blocks = 148 * 8;  // one full wave of 8 resident 256-thread blocks per SM
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    // labels/mask through a pinned copy so the upload does not block the host
    if (d.lpin_cap < V * 9) {
      if (d.lpin) cudaFreeHost(d.lpin);
      CU(cudaHostAlloc(reinterpret_cast<void**>(&d.lpin), V * 9, cudaHostAllocPortable));
      d.lpin_cap = V * 9;
    }
    std::memcpy(d.lpin, labels, V * 8);
    std::memcpy(d.lpin + V * 8, mask, V);
    HT_TRY(d.labels.ensure(V * 8));
    HT_TRY(d.mask.ensure(V));
    HT_TRY(d.loss_part.ensure((int64_t)blocks * f->n * 8));
    CU(cudaMemcpyAsync(d.labels.p, d.lpin, V * 8, cudaMemcpyHostToDevice, d.stream));
    CU(cudaMemcpyAsync(d.mask.p, d.lpin + V * 8, V, cudaMemcpyHostToDevice, d.stream));
    CU(cudaMemsetAsync(d.loss_part.p, 0, (int64_t)blocks * f->n * 8, d.stream));
    if (count > 0)
      for (int j = 0; j < f->n; ++j) {
        DevChunk& c = d.chunks[j];
        count_launch();
        ht::k_loss<<<blocks, 256, 0, d.stream>>>(
            d.hL.as<float>() + d.hL_off[j] * d_last, c.nv, d_last, d.labels.as<int64_t>(),
            d.mask.as<uint8_t>(), c.dest_rows.as<int64_t>(),
            d.cache ? d.mg[f->L].as<float>() : (float*)gout, d.cache ? c.dest_m0 : -1,
            (float)count, d.loss_part.as<double>() + (int64_t)j * blocks);
        CU(cudaGetLastError());
      }
    if (d.cache) {  // grad_h[L] rows live in the mirror; write them through
      if (count <= 0) CU(cudaMemsetAsync(d.mg[f->L].p, 0, d.mcount * (int64_t)d_last * 4, d.stream));
      if (!f->lean) HT_TRY(cache_writeback(f, d, gout, d.mg[f->L].as<float>(), (int64_t)d_last * 4));
    }
    HT_TRY(ev_rec(d.e_loss, d.stream));
  }
  if (loss) return ht_loss_value(f, loss);
  return HT_OK;
}

extern "C" int ht_loss_value(ht_fleet* f, double* loss) {
  *loss = 0.0;
  if (f->loss_count <= 0) return HT_OK;
  double tot = 0.0;
  for (auto& d : f->dev) {
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    std::vector<double> parts(d.loss_part.bytes / 8);
    CU(cudaMemcpyAsync(parts.data(), d.loss_part.p, parts.size() * 8, cudaMemcpyDeviceToHost,
                       d.stream));
    CU(cudaStreamSynchronize(d.stream));
    for (double p : parts) tot += p;
  }
  *loss = tot / (double)f->loss_count;
  return HT_OK;
}

extern "C" int ht_backward_layer(ht_fleet* f, int layer, int d_in, int d_out, const float* W,
                                 const void* agg_in, const void* grad_out, void* grad_in,
                                 int precision) {
  if (layer < 0 || layer >= f->L || f->dims[layer] != d_in || f->dims[layer + 1] != d_out)
    return fail(HT_EINVAL, "layer %d shape does not match ht_epoch_begin", layer);
  void *ain, *gout, *gin;
  HT_TRY(dev_ptr(agg_in, &ain));
  HT_TRY(dev_ptr(grad_out, &gout));
  HT_TRY(dev_ptr(grad_in, &gin));
  f->dim = d_in;
  f->elem = 4;
  const int64_t rbi = (int64_t)d_in * 4, rbo = (int64_t)d_out * 4;
  const int ldz = precision == HT_PREC_TF32 ? pad4(d_out) : d_out;
  for (auto& d : f->dev) {
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    if (!d.lw[layer].valid) HT_TRY(upload_layer_weights(d, layer, W, d_in, d_out));
    if (f->mode != HT_MODE_BASELINE && !direct_bwd(f, d))  // zeroed gradient slots
      CU(cudaMemsetAsync(d.grad.p, 0, d.cap * rbi, d.stream));
    if (d.cache) CU(cudaMemsetAsync(d.mg[layer].p, 0, d.mcount * rbi, d.stream));
  }
  for (int j = 0; j < f->n; ++j) {
    for (int i = 0; i < f->m; ++i) {
      Device& d = f->dev[i];
      if (!d.local) continue;  // rank mode: a peer process drives it
      HT_TRY(set_dev(d));
      DevChunk& c = d.chunks[j];
      const int s = (int)(d.bwd_count & 1);
      const int64_t* rows = c.dest_rows.as<int64_t>();
      float *A = d.ba[s].as<float>(), *G = d.bb[s].as<float>();
      if (d.cache) {  // checkpoint and gradient rows straight from the mirrors
        A = d.ma[layer].as<float>() + c.dest_m0 * d_in;
        G = d.mg[layer + 1].as<float>() + c.dest_m0 * d_out;
      } else {
      // K6 on tin: checkpoint rows (ready since the forward), then the
      // destination gradients (ready once the layer above has flushed)
      if (d.bwd_count >= 2) HT_TRY(ev_wait(d.tin, d.e_bcomp[s]));
      if (f->prefetch) {
        A = d.ck[layer].as<float>() + d.hL_off[j] * d_in;  // reloaded during the forward
      } else if (c.dest.dma) {
        for (int g = 0; g < kChunks; ++g) {
          if (j == 0) HT_TRY(ev_wait(d.tin, d.e_aggst[layer * kChunks + g]));
          HT_TRY(xfer(d.tin, c.dest, false, ain, rbi, A, rbi, rbi, chunk_bound(f->nrows, g),
                      chunk_bound(f->nrows, g + 1)));
        }
      } else {
        if (j == 0) HT_TRY(ev_wait(d.tin, d.e_aggst[layer * kChunks + kChunks - 1]));
        HT_TRY(launch_copy(d.tin, A, ain, nullptr, rows, c.nv, rbi, rbi, rbi, 0, kHostGrid));
      }
      // gradient rows of the layer above: written by the loss, or by the
      // flushes of the previous backward layer (of every device in baseline
      // mode); streamed per host-row chunk when both sides use copy engines
      const bool top = layer == f->L - 1;
      if (j == 0 && top) HT_TRY(ev_wait(d.tin, d.e_loss));
      if (c.dest.dma) {
        for (int g = 0; g < kChunks; ++g) {
          if (j == 0 && !top) {
            if (f->mode == HT_MODE_BASELINE)
              for (auto& o : f->dev) HT_TRY(ev_wait(d.tin, o.e_fchunk[g]));
            else
              HT_TRY(ev_wait(d.tin, d.e_fchunk[g]));
          }
          HT_TRY(xfer(d.tin, c.dest, false, gout, rbo, G, rbo, rbo, chunk_bound(f->nrows, g),
                      chunk_bound(f->nrows, g + 1)));
        }
      } else {
        if (j == 0 && !top) {
          if (f->mode == HT_MODE_BASELINE)
            for (auto& o : f->dev) HT_TRY(ev_wait(d.tin, o.e_fchunk[kChunks - 1]));
          else
            HT_TRY(ev_wait(d.tin, d.e_fchunk[kChunks - 1]));
        }
        HT_TRY(launch_copy(d.tin, G, gout, nullptr, rows, c.nv, rbo, rbo, rbo, 0, kHostGrid));
      }
      HT_TRY(ev_rec(d.e_bin, d.tin));
      // K7 on the compute stream
      HT_TRY(ev_wait(d.stream, d.e_bin));
      if (f->prefetch && j == 0) HT_TRY(ev_wait(d.stream, d.e_ck[layer]));
      }
      float *GZ = d.sc.as<float>(), *GA = d.sd.as<float>();
      LayerW& w = d.lw[layer];
      TimerRec tg;
      timer_begin(f, d, tg, d.stream);
      const int64_t M = c.nv;
      const int64_t nw = (int64_t)d_in * d_out;
      const int64_t* hrows = nullptr;
      const float* HO = hbm_outputs(f, d, j, layer, d_out, &hrows);
      // narrow-side transposed aggregation: grad_h_nbr = (A^T gz) W^T when
      // d_out < d_in (K8 gathers d_out-wide rows instead of d_in-wide ones;
      // same product, reassociated).  Needs gz with zeroed pad columns.
      const bool no_in = f->lean && layer == 0;  // lean: grad_h^0 is not produced
      const bool narrow = !no_in && HO && d_out < d_in && !getenv("HT_NO_NARROW_BWD");
      // project-first forward (agg^l never formed): the narrow-side rows
      // A^T gz give dW = h^T (A^T gz); needs them in row order (expanded CSR)
      const bool pfl = layer < (int)f->agg_deferred.size() && f->agg_deferred[layer] &&
                       precision == HT_PREC_TF32;
      if (HO && M > 0) {  // gz = g * (h > 0): z need not be recomputed
        count_launch();
        ht::k_relu_mask<<<grid_for(M), kThreads, 0, d.stream>>>(GZ, ldz, G, HO, hrows, M, d_out);
        CU(cudaGetLastError());
      }
      if (precision == HT_PREC_TF32) {
        if (!HO)
          HT_TRY(ht::tc::rows<ht::tc::TC_MASK>(d.stream, true, A, d_in, M, d_in, w.Wt_hi.as<float>(),
                                               w.Wt_lo.as<float>(), d_in, d_out, GZ, ldz, G, d_out));
        if (!narrow && !no_in)
          HT_TRY(ht::tc::rows<ht::tc::TC_STORE>(d.stream, false, GZ, ldz, M, d_out,
                                                w.Wp_hi.as<float>(), nullptr, ldz, d_in, GA, d_in,
                                                nullptr, 0));
        if (M > 0 && !pfl) {  // (project-first layer: dW = h^T (A^T gz) after K8)
          int used = 1;
          HT_TRY(ht::tc::wgrad(d.stream, A, d_in, d_in, GZ, ldz, d_out, M, kSplitsMax,
                               d.gemm_ws.as<float>(), &used));
          count_launch(4);
          ht::k_reduce_splits<<<grid_for(nw / 32 + 1), 256, 0, d.stream>>>(
              d.gWall.as<float>() + d.gW_off[layer], d.gemm_ws.as<float>(), nw, used);
          CU(cudaGetLastError());
        }
      } else {
        int splits = (int)std::min<int64_t>(kSplitsMax, std::max<int64_t>(1, M / 2048));
        int64_t kps = ((M + splits - 1) / splits + 15) / 16 * 16;
        splits = (int)std::max<int64_t>(1, (M + kps - 1) / kps);
        if (!HO)
          HT_TRY((gemm<false, false, ht::EPI_MASK>(d.stream, A, d_in, w.W.as<float>(), d_out, GZ,
                                                   ldz, G, d_out, M, d_out, d_in, 1, d_in)));
        if (M > 0) {
          HT_TRY((gemm<true, false, ht::EPI_STORE>(d.stream, A, d_in, GZ, ldz,
                                                   d.gemm_ws.as<float>(), d_out, nullptr, 0, d_in,
                                                   d_out, M, splits, kps)));
          count_launch();
          ht::k_reduce_splits<<<grid_for(nw / 32 + 1), 256, 0, d.stream>>>(
              d.gWall.as<float>() + d.gW_off[layer], d.gemm_ws.as<float>(), nw, splits);
          CU(cudaGetLastError());
        }
        if (!narrow && !no_in)
          HT_TRY((gemm<false, true, ht::EPI_STORE>(d.stream, GZ, ldz, w.W.as<float>(), d_out, GA,
                                                   d_in, nullptr, 0, M, d_in, d_out, 1, d_out)));
      }
      timer_end(f, d, tg, 2, 6.0 * c.nv * d_in * d_out, d.stream);
      HT_TRY(ev_rec(d.e_bcomp[s], d.stream));
      if (no_in && !pfl) {
        d.bwd_count++;
        continue;
      }
      // K8: transposed aggregation over the CSR view -> neighbour-row grads
      TimerRec tr;
      timer_begin(f, d, tr, d.stream);
      const int kw = narrow ? ldz : d_in;  // width of the gathered rows
      // one device, one batch: the expanded CSR writes the grad mirror rows
      // (every host row; zero rows for sources without out-edges) in place
      // of the views - the only flush of each row, a store
      const bool dx = direct_bwd(f, d) && c.bx_rows == d.mcount;
      if (pfl && !(dx && HO && (narrow || no_in)))
        return fail(HT_ESTATE, "project-first layer %d needs the one-device narrow backward", layer);
      const int64_t nseg = dx ? c.bx_rows : c.nn;
      float* views = dx ? d.mg[layer].as<float>() : d.se.as<float>();
      HT_TRY(launch_seg(d.stream, (narrow || pfl) ? d.tT.as<float>() : views,
                        (narrow || pfl) ? GZ : GA, (narrow || pfl) ? ldz : kw,
                        (narrow || pfl) ? ldz : kw,
                        dx ? c.bx_off.as<int64_t>() : c.csr_off.as<int64_t>(),
                        c.csr_dst.as<int32_t>(), c.csr_w.as<float>(), nseg,
                        dx ? c.bx_np : c.bw_np, dx ? c.bx_lo : c.bw_lo, dx ? c.bx_hi : c.bw_hi,
                        dx ? c.bx_nf : c.bw_nf, dx ? c.bx_seg : c.bw_seg,
                        dx ? c.bx_first : c.bw_first, dx ? c.bx_cnt : c.bw_cnt,
                        d.partial.as<float>()));
      timer_end(f, d, tr, 1, (double)c.ne * (8.0 + 4.0 * kw) + (double)c.nn * (4.0 * kw + 4.0),
                d.stream);
      if (pfl && nseg > 0) {  // dW = h^T (A^T gz), rows in row order
        int used = 1;
        const int64_t nwl = (int64_t)d_in * d_out;
        HT_TRY(ht::tc::wgrad(d.stream, d.mh[layer].as<float>(), d_in, d_in, d.tT.as<float>(), ldz,
                             d_out, nseg, kSplitsMax, d.gemm_ws.as<float>(), &used));
        count_launch(2);
        ht::k_reduce_splits<<<grid_for(nwl / 32 + 1), 256, 0, d.stream>>>(
            d.gWall.as<float>() + d.gW_off[layer], d.gemm_ws.as<float>(), nwl, used);
        CU(cudaGetLastError());
      }
      if (no_in) {  // (lean, layer 0: grad_h^0 is not produced)
        d.bwd_count++;
        continue;
      }
      if (narrow && nseg > 0) {  // views = (A^T gz) W^T
        if (precision == HT_PREC_TF32)
          HT_TRY(ht::tc::rows<ht::tc::TC_STORE>(d.stream, false, d.tT.as<float>(), ldz, nseg, d_out,
                                                w.Wp_hi.as<float>(), nullptr, ldz, d_in, views,
                                                d_in, nullptr, 0));
        else
          HT_TRY((gemm<false, true, ht::EPI_STORE>(d.stream, d.tT.as<float>(), ldz, w.W.as<float>(),
                                                   d_out, views, d_in, nullptr, 0, nseg, d_in,
                                                   d_out, 1, d_out)));
      }
      if (direct_bwd(f, d) && !dx)  // views -> grad mirror rows (the only, first flush: a store)
        HT_TRY(launch_copy(d.stream, d.mg[layer].p, d.se.p, c.nbr_gid.as<int64_t>(), nullptr, c.nn,
                           rbi, rbi, rbi));
      d.bwd_count++;
    }
    // K9/K10: owner push (ascending source device) + flush into host grads
    // (into the mirror with the cache)
    if (!(f->lean && layer == 0) && !direct_bwd(f, f->dev[f->rank >= 0 ? f->rank : 0]))
      HT_TRY(push_flush(f, j, gin, true, layer));
  }
  for (auto& d : f->dev) {
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    if (d.cache && !(f->lean && layer == 0))
      HT_TRY(cache_writeback(f, d, gin, d.mg[layer].as<float>(), rbi));
    HT_TRY(ev_rec(d.e_flush, d.stream));
  }
  return HT_OK;
}

// ===========================================================================
// GAT epoch: src/engine.py:196-289 (layer math),
// src/engine.py:411-476 (epoch), src/devices.py:376-385 / 427-432 (dest
// gradient adds, input re-staging for the recompute backward).
//
// Per batch and device: neighbour rows staged into the slot buffer through
// the same dedup machinery as GCN (host loads, barrier, staggered peer
// fetches, barrier), then gathered into N_ij order (the reference's views);
// destination input rows come from the host; q = h_nbr.W and p = h_dst.W on
// the tensor cores (3xTF32, like z), attention and aggregation in
// k_gat_dst.  The backward re-stages the inputs, recomputes, and produces
// the neighbour-gradient views (pushed to owners and flushed exactly like
// GCN) plus destination-input gradients added into the host rows.  Every
// host gradient write is a read-modify-write (dest adds and flushes both
// touch grad_h[l]); the host gradient arrays are zeroed at epoch start.
// ===========================================================================
namespace {

constexpr int kColBlocks = 1184;  // 148 SMs x 8

int gat_width_ok(int d) {
  if (d % 4 == 0 && d >= 4 && d <= 512) return HT_OK;
  return fail(HT_EINVAL, "GAT path needs feature widths that are multiples of 4 in [4, 512] (got %d)", d);
}

inline int nv_of(int d) { return std::max(1, std::min(4, (d / 4 + 31) / 32)); }

int launch_rowdot(cudaStream_t s, float* out, const float* X, const float* a, int d, int64_t rows) {
  if (rows <= 0) return HT_OK;
  const int g = grid_for(rows);
  count_launch();
  switch (nv_of(d)) {
    case 1: ht::gat::k_rowdot<1><<<g, kThreads, 0, s>>>(out, X, d, a, d, rows); break;
    case 2: ht::gat::k_rowdot<2><<<g, kThreads, 0, s>>>(out, X, d, a, d, rows); break;
    case 3: ht::gat::k_rowdot<3><<<g, kThreads, 0, s>>>(out, X, d, a, d, rows); break;
    default: ht::gat::k_rowdot<4><<<g, kThreads, 0, s>>>(out, X, d, a, d, rows); break;
  }
  CU(cudaGetLastError());
  return HT_OK;
}

template <bool BWD>
int launch_gat_dst(cudaStream_t s, const DevChunk& c, const float* Q, const float* P,
                   const float* els, const float* a_dst, int d, float slope, float* H,
                   const float* G, float* GS, float* GP, float* AL, float* GT, float* SGT,
                   const float* HO = nullptr, const int64_t* ho_rows = nullptr,
                   bool global_src = false) {
  if (c.nv <= 0) return HT_OK;
  const int g = grid_for(c.nv);
  const int64_t* off = c.csc_off.as<int64_t>();
  // sources as chunk-local rows of Q, or (direct) as global rows of P
  const int32_t* idx = global_src ? c.csc_gid.as<int32_t>() : c.csc_loc.as<int32_t>();
  count_launch();
#define GATD(NV)                                                                              \
  ht::gat::k_gat_dst<NV, BWD><<<g, kThreads, 0, s>>>(off, idx, c.nv, Q, P, els, a_dst, d, slope, \
                                                     H, G, GS, GP, AL, GT, SGT, HO, ho_rows)
  switch (nv_of(d)) {
    case 1: GATD(1); break;
    case 2: GATD(2); break;
    case 3: GATD(3); break;
    default: GATD(4); break;
  }
#undef GATD
  CU(cudaGetLastError());
  return HT_OK;
}

int launch_gat_src(cudaStream_t s, const DevChunk& c, const float* GS, const float* AL,
                   const float* GT, const float* a_src, int d, float* GQ, float* GTS, float* part,
                   float* pgts, bool expanded = false, const float* sgt_add = nullptr,
                   const float* a_dst = nullptr) {
  // expanded: segments over every host row (gat_direct), outputs in row order
  const int64_t nseg = expanded ? c.bx_rows : c.nn;
  const int64_t np = expanded ? c.bx_np : c.bw_np, nf = expanded ? c.bx_nf : c.bw_nf;
  const DBuf &lo = expanded ? c.bx_lo : c.bw_lo, &hi = expanded ? c.bx_hi : c.bw_hi;
  if (nseg <= 0) return HT_OK;
  const int g = grid_for(nseg);
  const int64_t* off = expanded ? c.bx_off.as<int64_t>() : c.csr_off.as<int64_t>();
  const int32_t* dst = c.csr_dst.as<int32_t>();
  const int32_t* perm = c.csr_perm.as<int32_t>();
  count_launch(1 + (np ? 1 : 0) + (nf ? 1 : 0));
#define GATS(NV)                                                                                \
  ht::gat::k_gat_src<NV><<<g, kThreads, 0, s>>>(off, dst, perm, nseg, kSplit, GS, AL, GT, a_src, \
                                                d, GQ, GTS, sgt_add, a_dst);                     \
  if (np)                                                                                       \
    ht::gat::k_gat_src_pieces<NV><<<grid_for(np), kThreads, 0, s>>>(                            \
        lo.as<int64_t>(), hi.as<int64_t>(), np, dst, perm, GS, AL, GT, a_src, d, part, pgts)
  switch (nv_of(d)) {
    case 1: GATS(1); break;
    case 2: GATS(2); break;
    case 3: GATS(3); break;
    default: GATS(4); break;
  }
#undef GATS
  CU(cudaGetLastError());
  if (nf) {
    const DBuf &sg = expanded ? c.bx_seg : c.bw_seg, &fi = expanded ? c.bx_first : c.bw_first,
               &cn = expanded ? c.bx_cnt : c.bw_cnt;
    ht::gat::k_gat_src_fixup<<<grid_for(nf), kThreads, 0, s>>>(
        GQ, GTS, part, pgts, d, sg.as<int64_t>(), fi.as<int64_t>(), cn.as<int64_t>(), nf, sgt_add,
        a_dst);
    CU(cudaGetLastError());
  }
  return HT_OK;
}

// acc[c] += sum_r w[r] X[r][c], fixed-order two-stage reduction
int launch_wcolsum(cudaStream_t s, float* acc, const float* X, const float* w, int64_t rows, int d,
                   float* partial) {
  if (rows <= 0) return HT_OK;
  int64_t nb = std::min<int64_t>(kColBlocks, (rows + 63) / 64);
  const int64_t rpb = (rows + nb - 1) / nb;
  nb = (rows + rpb - 1) / rpb;
  count_launch(2);
  switch (nv_of(d)) {
    case 1: ht::gat::k_wcolsum<1><<<(int)nb, 256, 0, s>>>(partial, X, d, w, rows, d, rpb); break;
    case 2: ht::gat::k_wcolsum<2><<<(int)nb, 256, 0, s>>>(partial, X, d, w, rows, d, rpb); break;
    case 3: ht::gat::k_wcolsum<3><<<(int)nb, 256, 0, s>>>(partial, X, d, w, rows, d, rpb); break;
    default: ht::gat::k_wcolsum<4><<<(int)nb, 256, 0, s>>>(partial, X, d, w, rows, d, rpb); break;
  }
  ht::gat::k_colsum_reduce<<<(d + 127) / 128, 128, 0, s>>>(acc, partial, (int)nb, d);
  CU(cudaGetLastError());
  return HT_OK;
}

// C[M x d_out] = A[M x d_in] . W (3xTF32 on tcgen05, or SIMT FP32)
int gat_proj(Device& d, int precision, const float* A, int64_t M, int d_in, int d_out, float* C,
             LayerW& w) {
  if (M <= 0) return HT_OK;
  if (precision == HT_PREC_TF32)
    return ht::tc::rows<ht::tc::TC_STORE>(d.stream, true, A, d_in, M, d_in, w.Wt_hi.as<float>(),
                                          w.Wt_lo.as<float>(), d_in, d_out, C, d_out, nullptr, 0);
  return gemm<false, false, ht::EPI_STORE>(d.stream, A, d_in, w.W.as<float>(), d_out, C, d_out,
                                           nullptr, 0, M, d_out, d_in, 1, d_in);
}

// C[M x d_in] = G[M x d_out] . W^T
int gat_proj_t(Device& d, int precision, const float* G, int64_t M, int d_in, int d_out, float* C,
               LayerW& w) {
  if (M <= 0) return HT_OK;
  if (precision == HT_PREC_TF32)
    return ht::tc::rows<ht::tc::TC_STORE>(d.stream, false, G, d_out, M, d_out,
                                          w.Wp_hi.as<float>(), nullptr, d_out, d_in, C, d_in,
                                          nullptr, 0);
  return gemm<false, true, ht::EPI_STORE>(d.stream, G, d_out, w.W.as<float>(), d_out, C, d_in,
                                          nullptr, 0, M, d_in, d_out, 1, d_out);
}

// gW += A^T . G  (A: M x d_in, G: M x d_out), row slices reduced in order
int gat_wgrad(Device& d, int precision, const float* A, const float* G, int64_t M, int d_in,
              int d_out, float* gW) {
  if (M <= 0) return HT_OK;
  const int64_t nw = (int64_t)d_in * d_out;
  int used = 1;
  if (precision == HT_PREC_TF32) {
    HT_TRY(ht::tc::wgrad(d.stream, A, d_in, d_in, G, d_out, d_out, M, kSplitsMax,
                         d.gemm_ws.as<float>(), &used));
    count_launch();
  } else {
    int splits = (int)std::min<int64_t>(kSplitsMax, std::max<int64_t>(1, M / 2048));
    int64_t kps = ((M + splits - 1) / splits + 15) / 16 * 16;
    splits = (int)std::max<int64_t>(1, (M + kps - 1) / kps);
    HT_TRY((gemm<true, false, ht::EPI_STORE>(d.stream, A, d_in, G, d_out, d.gemm_ws.as<float>(),
                                             d_out, nullptr, 0, d_in, d_out, M, splits, kps)));
    used = splits;
  }
  count_launch();
  ht::k_reduce_splits<<<grid_for(nw / 32 + 1), 256, 0, d.stream>>>(gW, d.gemm_ws.as<float>(), nw,
                                                                    used);
  CU(cudaGetLastError());
  return HT_OK;
}

// attention vector of layer l ([a_dst | a_src]) into its device buffer
int upload_attn(Device& d, int l, const float* A, int d_out) {
  LayerW& w = d.lw[l];
  HT_TRY(w.A.ensure(2 * (int64_t)d_out * 4));
  float* pin = d.wpin + d.wpin_off[d.lw.size()] + d.gA_off[l];
  std::memcpy(pin, A, 2 * (int64_t)d_out * 4);
  CU(cudaMemcpyAsync(w.A.p, pin, 2 * (int64_t)d_out * 4, cudaMemcpyHostToDevice, d.stream));
  return HT_OK;
}

// step 1 of dedup_comm_fwd for batch j on device d (tin): host loads of
// the load (full) / owned (p2p) / neighbour (baseline) rows into slots
int gat_host_loads(ht_fleet* f, Device& d, DevChunk& c, const void* hin, int64_t rb) {
  if (c.h2d.dma) {
    for (int g = 0; g < kChunks; ++g)
      HT_TRY(xfer(d.tin, c.h2d, false, const_cast<void*>(hin), rb, d.value.p, rb, rb,
                  chunk_bound(f->nrows, g), chunk_bound(f->nrows, g + 1)));
    return HT_OK;
  }
  return launch_copy(d.tin, d.value.p, hin, c.h2d.dst.as<int64_t>(), c.h2d.src.as<int64_t>(), c.h2d.n,
                     rb, rb, rb, 0, kHostGrid);
}

// destination rows host -> device staging (tin)
int gat_dest_load(ht_fleet* f, Device& d, DevChunk& c, const void* host, float* dst, int64_t rb) {
  if (c.dest.dma) {
    for (int g = 0; g < kChunks; ++g)
      HT_TRY(xfer(d.tin, c.dest, false, const_cast<void*>(host), rb, dst, rb, rb,
                  chunk_bound(f->nrows, g), chunk_bound(f->nrows, g + 1)));
    return HT_OK;
  }
  return launch_copy(d.tin, dst, host, nullptr, c.dest_rows.as<int64_t>(), c.nv, rb, rb, rb, 0,
                     kHostGrid);
}

// Stage batch j's neighbour rows of layer input `hin` on every device and
// gather them into N_ij order (g_hn); destination rows of `hin` into
// g_hd[s] (and, when gsrc != null, destination rows of gsrc into g_gin[s]).
int gat_stage(ht_fleet* f, int layer, int j, const void* hin, int d_in, const void* gsrc,
              int d_out, bool first_of_layer, bool bwd) {
  const int64_t rbi = (int64_t)d_in * 4, rbo = (int64_t)d_out * 4;
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    DevChunk& c = d.chunks[j];
    int64_t& cnt = bwd ? d.bwd_count : d.fwd_count;
    const int s = (int)(cnt & 1);
    if (d.cache) {  // owned rows from the HBM mirror; destination rows are read in place
      if (!bwd && layer == 0 && j == 0) {
        HT_TRY(cache_upload(f, d, d.tin, hin, d.mh[0].as<float>(), rbi));
        HT_TRY(ev_rec(d.e_up, d.tin));
        HT_TRY(ev_wait(d.stream, d.e_up));
      }
      for (auto& o : f->dev) HT_TRY(ev_wait(d.stream, o.e_fetch));  // peers done with our slots
      if (!hbm_inputs(f, d, layer, hin))  // else the views are gathered from the mirror
        HT_TRY(launch_copy(d.stream, d.value.p, d.mh[layer].p, c.h2d.dst.as<int64_t>(),
                           c.h2d_m.as<int64_t>(), c.h2d.n, rbi, rbi, rbi));
      HT_TRY(ev_rec(d.e_in, d.stream));
      continue;
    }

    if (!first_of_layer) {  // slots of the previous batch gathered everywhere
      HT_TRY(ev_wait(d.tin, d.e_agg));
      for (auto& o : f->dev) HT_TRY(ev_wait(d.tin, o.e_fetch));
    }
    if (first_of_layer)  // inputs of this layer complete on every device
      for (auto& o : f->dev) {
        HT_TRY(ev_wait(d.tin, o.e_hst));  // forward stores (tout is in order)
        if (bwd) {
          HT_TRY(ev_wait(d.tin, o.e_loss));   // grad_h[L] rows
          HT_TRY(ev_wait(d.tin, o.e_flush));  // grad_h[l+1] rows of the layer above
        }
      }
    if (cnt >= 2) HT_TRY(ev_wait(d.tin, d.e_gcomp[s]));  // staging set s consumed
    if (!hbm_inputs(f, d, layer, hin)) {  // else the views are gathered from the HBM store
      TimerRec tr;
      timer_begin(f, d, tr, d.tin);
      HT_TRY(gat_host_loads(f, d, c, hin, rbi));
      timer_end(f, d, tr, 3, (double)c.h2d.n * rbi, d.tin);
    }
    HT_TRY(gat_dest_load(f, d, c, hin, d.g_hd[s].as<float>(), rbi));
    if (gsrc) HT_TRY(gat_dest_load(f, d, c, gsrc, d.g_gin[s].as<float>(), rbo));
    HT_TRY(ev_rec(d.e_in, d.tin));
  }
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    if (!d.local) continue;
    HT_TRY(set_dev(d));
    DevChunk& c = d.chunks[j];
    for (auto& o : f->dev) HT_TRY(ev_wait(d.stream, o.e_in));
    if (f->rank >= 0 && f->m > 1) HT_TRY(xbarrier(f));
    if (f->mode != HT_MODE_BASELINE)
      for (int st = 1; st < f->m; ++st) {
        const int k = (i + st) % f->m;
        const CopyList& cl = c.d2d[st];
        HT_TRY(launch_copy(d.stream, d.value.p, f->dev[k].value.p, cl.dst.as<int64_t>(),
                           cl.src.as<int64_t>(), cl.n, rbi, rbi, rbi));
      }
    if (f->rank >= 0 && f->m > 1) HT_TRY(xbarrier(f));
    HT_TRY(ev_rec(d.e_fetch, d.stream));
    // the reference's views: value[slot(N_ij)] in N_ij order (or h^l[N_ij]
    // straight from an HBM-resident input on a single device)
    const float* Xd = hbm_inputs(f, d, layer, hin);
    if (!gat_direct(f, d))  // (direct: the layer reads its input rows in place)
      HT_TRY(launch_copy(d.stream, d.g_hn.p, Xd ? (const void*)Xd : d.value.p, nullptr,
                         Xd ? c.nbr_gid.as<int64_t>() : c.nbr_slot.as<int64_t>(), c.nn, rbi, rbi,
                         rbi));
    HT_TRY(ev_rec(d.e_agg, d.stream));
  }
  return HT_OK;
}

}  // namespace

extern "C" int ht_gat_epoch_begin(ht_fleet* f, int L, const int* dims) {
  for (int l = 0; l <= L; ++l) HT_TRY(gat_width_ok(dims[l]));
  int64_t extra = 0;  // attention gradients live behind the weight gradients
  for (int l = 0; l < L; ++l) extra += 2 * (int64_t)dims[l + 1];
  HT_TRY(epoch_begin_impl(f, L, dims, extra, true));
  int dmax = 0;
  for (int l = 0; l <= L; ++l) dmax = std::max(dmax, dims[l]);
  for (int i = 0; i < f->m; ++i) {
    Device& d = f->dev[i];
    d.gA_off.assign(L + 1, 0);
    for (int l = 0; l < L; ++l) d.gA_off[l + 1] = d.gA_off[l] + 2 * (int64_t)dims[l + 1];
    if (!d.local) continue;
    HT_TRY(set_dev(d));
    int64_t mv = 1, mn = 1, me = 1;
    for (int j = 0; j < f->n; ++j) {
      DevChunk& c = d.chunks[j];
      HostSets& h = f->sets[i][j];
      mv = std::max(mv, c.nv);
      mn = std::max(mn, c.nn);
      me = std::max(me, c.ne);
      if (!c.gat_ready) {  // chunk-local CSC sources and CSR -> CSC edge ids
        std::vector<int32_t> loc(h.ne), perm(h.ne);
        for (int64_t e = 0; e < h.ne; ++e) {
          loc[e] = (int32_t)h.csc_src[e];
          perm[e] = (int32_t)h.csr_perm[e];
        }
        HT_TRY(upload(c.csc_loc, loc, d.stream));
        HT_TRY(upload(c.csr_perm, perm, d.stream));
        CU(cudaStreamSynchronize(d.stream));  // host vectors go out of scope
        c.gat_ready = true;
      }
    }
    if (f->m == 1 && f->n == 1) {  // gat_direct: row-order GQ / gts / views
      mn = std::max(mn, mv);
      HT_TRY(d.se.ensure(mn * dmax * 4));
    }
    HT_TRY(d.g_hn.ensure(mn * dmax * 4));
    HT_TRY(d.g_q.ensure(mn * dmax * 4));
    HT_TRY(d.g_p.ensure(mv * dmax * 4));
    if (f->m == 1 && f->n == 1) {  // per-layer projections for gat_direct (owner cache only)
      d.g_pl.resize(L);
      d.g_elsl.resize(L);
      for (int l = 0; l < L; ++l) {
        HT_TRY(d.g_pl[l].ensure(mv * dims[l + 1] * 4));
        HT_TRY(d.g_elsl[l].ensure(mv * 4));
      }
    }
    HT_TRY(d.g_els.ensure(mn * 4));
    HT_TRY(d.g_gs.ensure(mv * dmax * 4));
    HT_TRY(d.g_gp.ensure(mv * dmax * 4));
    HT_TRY(d.g_al.ensure(me * 4));
    HT_TRY(d.g_gt.ensure(me * 4));
    HT_TRY(d.g_sgt.ensure(mv * 4));
    HT_TRY(d.g_gq.ensure(mn * dmax * 4));
    HT_TRY(d.g_gts.ensure(mn * 4));
    HT_TRY(d.g_ghd.ensure(mv * dmax * 4));
    HT_TRY(d.g_cpart.ensure((int64_t)kColBlocks * dmax * 4));
    int64_t np = 1;
    for (int j = 0; j < f->n; ++j) np = std::max(np, d.chunks[j].bw_np);
    HT_TRY(d.g_pgts.ensure(np * 4));
    if (!d.cache)  // with the owner cache these rows are read in place
      for (int s = 0; s < 2; ++s) {
        HT_TRY(d.g_hd[s].ensure(mv * dmax * 4));
        HT_TRY(d.g_gin[s].ensure(mv * dmax * 4));
      }
    // pinned scratch: the weight slots of the epoch + the attention vectors
    const int64_t want = d.wpin_off[L] + d.gA_off[L];
    if (d.wpin_cap < want) {
      if (d.wpin) cudaFreeHost(d.wpin);
      CU(cudaHostAlloc(reinterpret_cast<void**>(&d.wpin), want * 4, cudaHostAllocPortable));
      d.wpin_cap = want;
    }
  }
  f->gat = true;
  return HT_OK;
}

extern "C" int ht_gat_forward_layer(ht_fleet* f, int layer, int d_in, int d_out, const float* W,
                                    const float* A, float slope, const void* h_in, void* h_out,
                                    int precision) {
  if (!f->gat) return fail(HT_ESTATE, "GAT layer before ht_gat_epoch_begin");
  if (layer < 0 || layer >= f->L || f->dims[layer] != d_in || f->dims[layer + 1] != d_out)
    return fail(HT_EINVAL, "layer %d shape does not match ht_gat_epoch_begin", layer);
  if (precision == HT_PREC_TF32 && (d_in > 256 || d_out > 256))
    return fail(HT_EINVAL, "tf32 GAT path supports widths <= 256");
  void *hin, *hout;
  HT_TRY(dev_ptr(h_in, &hin));
  HT_TRY(dev_ptr(h_out, &hout));
  f->dim = d_in;
  f->elem = 4;
  const bool last = layer == f->L - 1;
  const int64_t rbo = (int64_t)d_out * 4;
  f->hptr[layer + 1] = hout;
  f->hdev[layer + 1] = is_dev_mem(hout);
  for (auto& d : f->dev) {
    if (!d.local) continue;
    HT_TRY(set_dev(d));
    HT_TRY(upload_layer_weights(d, layer, W, d_in, d_out));
    HT_TRY(upload_attn(d, layer, A, d_out));
  }
  if (last) f->hL_dim = d_out;
  for (int j = 0; j < f->n; ++j) {
    HT_TRY(gat_stage(f, layer, j, hin, d_in, nullptr, d_out, j == 0, false));
    for (int i = 0; i < f->m; ++i) {
      Device& d = f->dev[i];
      if (!d.local) continue;
      HT_TRY(set_dev(d));
      DevChunk& c = d.chunks[j];
      const int s = (int)(d.fwd_count & 1);
      LayerW& w = d.lw[layer];
      if (d.fwd_count >= 2 && !d.cache) HT_TRY(ev_wait(d.stream, d.e_out[s]));  // output set s drained
      float* H = last     ? d.hL.as<float>() + d.hL_off[j] * d_out
                 : d.cache ? d.mh[layer + 1].as<float>() + c.dest_m0 * d_out
                           : d.fb[s].as<float>();
      const float* HD = d.cache ? d.mh[layer].as<float>() + c.dest_m0 * d_in : d.g_hd[s].as<float>();
      const bool dir = gat_direct(f, d);  // q = p row for row: one projection
      float* P = dir ? d.g_pl[layer].as<float>() : d.g_p.as<float>();  // (kept for the backward)
      float* els = dir ? d.g_elsl[layer].as<float>() : d.g_els.as<float>();
      const float* Q = dir ? P : d.g_q.as<float>();
      TimerRec tg;
      timer_begin(f, d, tg, d.stream);
      if (!dir)
        HT_TRY(gat_proj(d, precision, d.g_hn.as<float>(), c.nn, d_in, d_out, d.g_q.as<float>(), w));
      HT_TRY(gat_proj(d, precision, HD, c.nv, d_in, d_out, P, w));
      timer_end(f, d, tg, 2, 2.0 * (double)((dir ? 0 : c.nn) + c.nv) * d_in * d_out, d.stream);
      HT_TRY(ev_rec(d.e_gcomp[s], d.stream));  // destination inputs of set s consumed
      HT_TRY(launch_rowdot(d.stream, els, Q, w.A.as<float>() + d_out, d_out, dir ? c.nv : c.nn));
      TimerRec tr;
      timer_begin(f, d, tr, d.stream);
      HT_TRY(launch_gat_dst<false>(d.stream, c, Q, P, els, w.A.as<float>(), d_out, slope, H, nullptr,
                                   nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                   dir));
      timer_end(f, d, tr, 0,
                (double)c.ne * (12.0 + 4.0 * d_out) + (double)c.nv * (8.0 * d_out + 16.0), d.stream);
      HT_TRY(ev_rec(d.e_comp, d.stream));
      HT_TRY(ev_wait(d.tout, d.e_comp));
      if (!(last && f->lean && d.cache)) HT_TRY(put_dest(f, c, d.tout, hout, H, rbo, -1));
      HT_TRY(ev_rec(d.e_out[s], d.tout));
      if (j == f->n - 1) HT_TRY(ev_rec(d.e_hst, d.tout));  // layer output complete
      d.fwd_count++;
    }
  }
  return HT_OK;
}

extern "C" int ht_gat_backward_layer(ht_fleet* f, int layer, int d_in, int d_out, const float* W,
                                     const float* A, float slope, const void* h_in,
                                     const void* grad_out, void* grad_in, int precision) {
  if (!f->gat) return fail(HT_ESTATE, "GAT layer before ht_gat_epoch_begin");
  if (layer < 0 || layer >= f->L || f->dims[layer] != d_in || f->dims[layer + 1] != d_out)
    return fail(HT_EINVAL, "layer %d shape does not match ht_gat_epoch_begin", layer);
  if (precision == HT_PREC_TF32 && (d_in > 256 || d_out > 256))
    return fail(HT_EINVAL, "tf32 GAT path supports widths <= 256");
  void *hin, *gout, *gin;
  HT_TRY(dev_ptr(h_in, &hin));
  HT_TRY(dev_ptr(grad_out, &gout));
  HT_TRY(dev_ptr(grad_in, &gin));
  f->dim = d_in;
  f->elem = 4;
  for (auto& d : f->dev) {
    if (!d.local) continue;
    HT_TRY(set_dev(d));
    if (!d.lw[layer].valid) HT_TRY(upload_layer_weights(d, layer, W, d_in, d_out));
    HT_TRY(upload_attn(d, layer, A, d_out));
    if (f->mode != HT_MODE_BASELINE)  // begin_backward_layer: zeroed gradient slots
      CU(cudaMemsetAsync(d.grad.p, 0, d.cap * (int64_t)d_in * 4, d.stream));
    if (d.cache) CU(cudaMemsetAsync(d.mg[layer].p, 0, d.mcount * (int64_t)d_in * 4, d.stream));
  }
  Device& d0 = f->dev[f->rank >= 0 ? f->rank : 0];
  for (int j = 0; j < f->n; ++j) {
    // load_recomp_chkpt("gat"): inputs re-staged through the forward
    // machinery, destination inputs, then the destination gradients
    HT_TRY(gat_stage(f, layer, j, hin, d_in, gout, d_out, j == 0, true));
    for (int i = 0; i < f->m; ++i) {
      Device& d = f->dev[i];
      if (!d.local) continue;
      HT_TRY(set_dev(d));
      DevChunk& c = d.chunks[j];
      const int s = (int)(d.bwd_count & 1);
      LayerW& w = d.lw[layer];
      const float* a_dst = w.A.as<float>();
      const float* a_src = a_dst + d_out;
      const bool dir = gat_direct(f, d);
      float* HD = d.cache ? d.mh[layer].as<float>() + c.dest_m0 * d_in : d.g_hd[s].as<float>();
      float* HN = dir ? HD : d.g_hn.as<float>();
      const int64_t nq = dir ? c.nv : c.nn;  // rows of Q / GQ / gts
      const float* Gin = d.cache ? d.mg[layer + 1].as<float>() + c.dest_m0 * d_out
                                 : d.g_gin[s].as<float>();
      // direct: p and el_src as the forward left them (same weights: the
      // update comes after the whole backward)
      float *P = dir ? d.g_pl[layer].as<float>() : d.g_p.as<float>(), *Q = dir ? P : d.g_q.as<float>();
      float* els = dir ? d.g_elsl[layer].as<float>() : d.g_els.as<float>();
      float *GS = d.g_gs.as<float>(), *GP = d.g_gp.as<float>(), *GQ = d.g_gq.as<float>();
      float *AL = d.g_al.as<float>(), *GT = d.g_gt.as<float>();
      TimerRec tg;
      timer_begin(f, d, tg, d.stream);
      if (!dir) HT_TRY(gat_proj(d, precision, HN, c.nn, d_in, d_out, Q, w));
      if (!dir) HT_TRY(gat_proj(d, precision, HD, c.nv, d_in, d_out, P, w));
      timer_end(f, d, tg, 2, dir ? 0.0 : 2.0 * (double)(c.nn + c.nv) * d_in * d_out, d.stream);
      if (!dir) HT_TRY(launch_rowdot(d.stream, els, Q, a_src, d_out, nq));
      TimerRec tr;
      timer_begin(f, d, tr, d.stream);
      const int64_t* hrows = nullptr;
      const float* HO = hbm_outputs(f, d, j, layer, d_out, &hrows);
      // direct: gp_v = sgt_v a_dst (rank 1) is added into gq_v by the CSR pass
      // (rows are the same vertices), so dW and the input gradients take one
      // GEMM each over gq + gp instead of two plus an add
      HT_TRY(launch_gat_dst<true>(d.stream, c, Q, P, els, a_dst, d_out, slope,
                                  nullptr, Gin, GS, dir ? nullptr : GP, AL, GT, d.g_sgt.as<float>(),
                                  HO, hrows, dir));
      HT_TRY(launch_gat_src(d.stream, c, GS, AL, GT, a_src, d_out, GQ, d.g_gts.as<float>(),
                            d.partial.as<float>(), d.g_pgts.as<float>(), dir,
                            dir ? d.g_sgt.as<float>() : nullptr, a_dst));
      timer_end(f, d, tr, 1,
                (double)c.ne * (28.0 + 12.0 * d_out) + (double)c.nv * (16.0 * d_out + 16.0) +
                    (double)c.nn * (4.0 * d_out + 12.0),
                d.stream);
      // attention gradients: a_dst <- sum_v seg_gt_v p_v, a_src <- sum_u gts_u q_u
      float* gA = d.gWall.as<float>() + d.gW_off[f->L] + d.gA_off[layer];
      HT_TRY(launch_wcolsum(d.stream, gA, P, d.g_sgt.as<float>(), c.nv, d_out,
                            d.g_cpart.as<float>()));
      HT_TRY(launch_wcolsum(d.stream, gA + d_out, Q, d.g_gts.as<float>(), nq, d_out,
                            d.g_cpart.as<float>()));
      // dW += h_nbr^T gq + h_dst^T gp; input gradients gq W^T, gp W^T
      float* gW = d.gWall.as<float>() + d.gW_off[layer];
      TimerRec tw;
      timer_begin(f, d, tw, d.stream);
      HT_TRY(gat_wgrad(d, precision, HN, GQ, nq, d_in, d_out, gW));
      if (!dir) HT_TRY(gat_wgrad(d, precision, HD, GP, c.nv, d_in, d_out, gW));
      if (!(f->lean && layer == 0)) {  // lean: grad_h^0 is not produced
        // direct: (gq + gp) W^T is the only store into the zeroed grad mirror
        HT_TRY(gat_proj_t(d, precision, GQ, nq, d_in, d_out,
                          dir ? d.mg[layer].as<float>() : d.se.as<float>(), w));
        if (!dir)
          HT_TRY(gat_proj_t(d, precision, GP, c.nv, d_in, d_out, d.g_ghd.as<float>(), w));
      }
      timer_end(f, d, tw, 2, 4.0 * (double)(c.nn + c.nv) * d_in * d_out, d.stream);
      HT_TRY(ev_rec(d.e_gcomp[s], d.stream));  // staging set s consumed
      d.bwd_count++;
    }
    // add_dest_grads (src/devices.py:376-385), then the deduplicated
    // neighbour-gradient accumulation (baseline: after every device's adds)
    if (f->lean && layer == 0) continue;
    for (int i = 0; i < f->m; ++i) {
      Device& d = f->dev[i];
      if (!d.local) continue;
      HT_TRY(set_dev(d));
      DevChunk& c = d.chunks[j];
      if (gat_direct(f, d)) continue;  // written by the projection above
      if (d.cache)  // contiguous mirror rows of the destinations
        HT_TRY(launch_acc(d.stream, 4, d.mg[layer].as<float>() + c.dest_m0 * d_in, d.g_ghd.p,
                          nullptr, nullptr, nullptr, c.nv, d_in, 0));
      else
        HT_TRY(launch_acc(d.stream, 4, gin, d.g_ghd.p, c.dest_rows.as<int64_t>(), nullptr,
                          nullptr, c.nv, d_in, 0));
    }
    if (f->mode == HT_MODE_BASELINE) HT_TRY(barrier(f));
    if (gat_direct(f, d0)) {  // written in place by the projection above
    } else if (direct_bwd(f, d0)) {  // views added straight into the grad mirror rows
      HT_TRY(set_dev(d0));
      HT_TRY(launch_acc(d0.stream, 4, d0.mg[layer].p, d0.se.p, d0.chunks[j].nbr_gid.as<int64_t>(),
                        nullptr, nullptr, d0.chunks[j].nn, d_in, 0));
    } else {
      HT_TRY(push_flush(f, j, gin, false, layer));
    }
  }
  for (auto& d : f->dev) {
    if (!d.local) continue;
    HT_TRY(set_dev(d));
    if (d.cache && !(f->lean && layer == 0))
      HT_TRY(cache_writeback(f, d, gin, d.mg[layer].as<float>(), (int64_t)d_in * 4));
    HT_TRY(ev_rec(d.e_flush, d.stream));
  }
  return HT_OK;
}

namespace {
// param -= lr * sum_i grads_i (ascending device), on device d0; the summed
// gradient optionally copied out
}  // namespace

// ascending-device gradient sum + SGD for every parameter block of the
// epoch (W per layer, then the GAT attention vector of that layer) in one
// pass: the parameters and the pointer table go up in one pinned copy, one
// k_sgd per block, updated parameters and summed gradients come back in one
// pinned copy.  Persistent buffers: no allocation (and none of its implicit
// synchronization) per epoch.
extern "C" int ht_sgd2(ht_fleet* f, int L, const int* dims, float* const* W, float* const* A,
                       float lr, float* const* gW_out, float* const* gA_out) {
  // rank mode: every rank sums all ranks' accumulators (IPC views) in
  // ascending device order and applies the identical update
  Device& d0 = f->dev[f->rank >= 0 ? f->rank : 0];
  if (A && !f->gat) return fail(HT_ESTATE, "attention update without ht_gat_epoch_begin");
  if (f->rank >= 0 && f->m > 1) HT_TRY(xbarrier(f));  // every rank's dW complete
  HT_TRY(sync_all(f));
  HT_TRY(set_dev(d0));
  std::vector<float*> prm, grd;
  std::vector<int64_t> cnt, goff;  // block sizes, offsets into each device's gWall
  for (int l = 0; l < L; ++l) {
    prm.push_back(W[l]);
    grd.push_back(gW_out ? gW_out[l] : nullptr);
    cnt.push_back((int64_t)dims[l] * dims[l + 1]);
    goff.push_back(-1 - l);  // resolved per device below
    if (A) {
      prm.push_back(A[l]);
      grd.push_back(gA_out ? gA_out[l] : nullptr);
      cnt.push_back(2 * (int64_t)dims[l + 1]);
      goff.push_back(l);
    }
  }
  const int nb = (int)cnt.size();
  int64_t total = 0;
  std::vector<int64_t> off(nb);
  for (int k = 0; k < nb; ++k) off[k] = total, total += cnt[k];
  const int64_t ptr_bytes = (int64_t)nb * f->m * 8;
  const int64_t pin_bytes = ptr_bytes + 3 * total * 4;
  if (d0.sgd_pin_cap < pin_bytes) {
    if (d0.sgd_pin) cudaFreeHost(d0.sgd_pin);
    d0.sgd_pin = nullptr;
    d0.sgd_pin_cap = 0;
    CU(cudaHostAlloc(reinterpret_cast<void**>(&d0.sgd_pin), pin_bytes, cudaHostAllocPortable));
    d0.sgd_pin_cap = pin_bytes;
  }
  const float** ptab = reinterpret_cast<const float**>(d0.sgd_pin);
  float* pin_in = reinterpret_cast<float*>(d0.sgd_pin + ptr_bytes);
  float* pin_w = pin_in + total;
  float* pin_g = pin_w + total;
  for (int k = 0; k < nb; ++k) {
    std::memcpy(pin_in + off[k], prm[k], cnt[k] * 4);
    for (int i = 0; i < f->m; ++i) {
      const Device& di = f->dev[i];
      const int64_t o = goff[k] < 0 ? di.gW_off[-1 - goff[k]] : di.gW_off[L] + di.gA_off[goff[k]];
      ptab[(int64_t)k * f->m + i] = di.gWall.as<float>() + o;
    }
  }
  HT_TRY(d0.sgd_p.ensure(ptr_bytes));
  HT_TRY(d0.sgd_w.ensure(total * 4));
  HT_TRY(d0.sgd_t.ensure(total * 4));
  CU(cudaMemcpyAsync(d0.sgd_p.p, ptab, ptr_bytes, cudaMemcpyHostToDevice, d0.stream));
  CU(cudaMemcpyAsync(d0.sgd_w.p, pin_in, total * 4, cudaMemcpyHostToDevice, d0.stream));
  for (int k = 0; k < nb; ++k) {
    count_launch();
    ht::k_sgd<<<grid_for(cnt[k] / 32 + 1), 256, 0, d0.stream>>>(
        d0.sgd_w.as<float>() + off[k], d0.sgd_t.as<float>() + off[k],
        d0.sgd_p.as<const float*>() + (int64_t)k * f->m, f->m, cnt[k], lr);
    CU(cudaGetLastError());
  }
  CU(cudaMemcpyAsync(pin_w, d0.sgd_w.p, total * 4, cudaMemcpyDeviceToHost, d0.stream));
  CU(cudaMemcpyAsync(pin_g, d0.sgd_t.p, total * 4, cudaMemcpyDeviceToHost, d0.stream));
  CU(cudaStreamSynchronize(d0.stream));
  for (int k = 0; k < nb; ++k) {
    std::memcpy(prm[k], pin_w + off[k], cnt[k] * 4);
    if (grd[k]) std::memcpy(grd[k], pin_g + off[k], cnt[k] * 4);
  }
  if (f->rank >= 0 && f->m > 1) {  // nobody zeroes its dW while a peer still reads it
    HT_TRY(xbarrier(f));
    CU(cudaStreamSynchronize(d0.stream));
  }
  for (auto& d : f->dev)
    for (auto& w : d.lw) w.valid = false;
  return HT_OK;
}

extern "C" int ht_sgd(ht_fleet* f, int L, const int* dims, float* const* W, float lr,
                      float* const* grads_out) {
  return ht_sgd2(f, L, dims, W, nullptr, lr, grads_out, nullptr);
}

extern "C" int ht_set_timing(ht_fleet* f, int enabled) {
  f->timing = enabled != 0;
  for (int q = 0; q < 4; ++q) f->t_launch[q] = 0, f->t_ms[q] = 0, f->t_bytes[q] = 0;
  return HT_OK;
}

extern "C" int ht_kernel_stats(ht_fleet* f, int which, int64_t* launches, double* ms,
                               double* bytes) {
  if (which < 0 || which > 3) return fail(HT_EINVAL, "bad kernel class");
  timers_collect(f);
  *launches = f->t_launch[which];
  *ms = f->t_ms[which];
  *bytes = f->t_bytes[which];
  return HT_OK;
}

// ---------------------------------------------------------------------------
// device-timeline marks for the benchmark: events on every device stream
// ---------------------------------------------------------------------------
extern "C" int ht_fleet_mark(ht_fleet* f, int which) {
  if (which < 0 || which >= kMarks) return fail(HT_EINVAL, "mark index must be in [0, %d)", kMarks);
  for (auto& d : f->dev) {
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    if (!d.mark[which]) CU(cudaEventCreate(&d.mark[which]));
    CU(cudaEventRecord(d.mark[which], d.stream));
  }
  return HT_OK;
}

extern "C" int ht_fleet_elapsed_between(ht_fleet* f, int a, int b, double* ms) {
  if (a < 0 || b < 0 || a >= kMarks || b >= kMarks) return fail(HT_EINVAL, "mark index out of range");
  double mx = 0.0;
  for (auto& d : f->dev) {
    if (!d.local) continue;
    HT_TRY(set_dev(d));
    if (!d.mark[a] || !d.mark[b]) return fail(HT_ESTATE, "marks not recorded");
    CU(cudaEventSynchronize(d.mark[b]));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, d.mark[a], d.mark[b]));
    mx = std::max(mx, (double)t);
  }
  *ms = mx;
  return HT_OK;
}

extern "C" int ht_fleet_elapsed(ht_fleet* f, double* ms) {
  double mx = 0.0;
  for (auto& d : f->dev) {
    if (!d.local) continue;  // rank mode: a peer process drives it
    HT_TRY(set_dev(d));
    if (!d.mark[0] || !d.mark[1]) return fail(HT_ESTATE, "marks not recorded");
    CU(cudaEventSynchronize(d.mark[1]));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, d.mark[0], d.mark[1]));
    mx = std::max(mx, (double)t);
  }
  *ms = mx;
  return HT_OK;
}

extern "C" int64_t ht_launches(void) { return g_launches.load(); }

// ---------------------------------------------------------------------------
// PCIe peaks of this box (roofline denominators of the host-transfer
// kernels): copy-engine H2D, D2H, both directions at once, and the
// zero-copy row kernels reading / writing pinned memory (1 KB rows).
// ---------------------------------------------------------------------------
extern "C" int ht_pcie_probe(int device, int64_t bytes, double* out /* [5] GB/s */) {
  CU(cudaSetDevice(device));
  void *h0 = nullptr, *h1 = nullptr, *d0 = nullptr, *d1 = nullptr;
  CU(cudaHostAlloc(&h0, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  CU(cudaHostAlloc(&h1, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  CU(cudaMalloc(&d0, bytes));
  CU(cudaMalloc(&d1, bytes));
  memset(h0, 1, bytes);
  memset(h1, 2, bytes);
  cudaStream_t s0, s1;
  CU(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t a, b, c;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  CU(cudaEventCreate(&c));
  void *hd0 = nullptr, *hd1 = nullptr;
  CU(cudaHostGetDevicePointer(&hd0, h0, 0));
  CU(cudaHostGetDevicePointer(&hd1, h1, 0));
  const int64_t rb = 1024, rows = bytes / rb;
  for (int t = 0; t < 5; ++t) {
    double best = 0;
    for (int rep = 0; rep < 4; ++rep) {
      CU(cudaEventRecord(a, s0));
      if (t == 0) CU(cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, s0));
      if (t == 1) CU(cudaMemcpyAsync(h0, d0, bytes, cudaMemcpyDeviceToHost, s0));
      if (t == 2) {
        CU(cudaStreamWaitEvent(s1, a, 0));
        CU(cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, s0));
        CU(cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, s1));
        CU(cudaEventRecord(c, s1));
        CU(cudaStreamWaitEvent(s0, c, 0));
      }
      if (t == 3) HT_TRY(launch_copy(s0, d0, hd0, nullptr, nullptr, rows, rb, rb, rb));
      if (t == 4) HT_TRY(launch_copy(s0, hd1, d1, nullptr, nullptr, rows, rb, rb, rb));
      CU(cudaEventRecord(b, s0));
      CU(cudaEventSynchronize(b));
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, a, b));
      const double moved = (t == 2 ? 2.0 : 1.0) * (double)bytes;
      best = std::max(best, moved / (ms * 1e-3) / 1e9);
    }
    out[t] = best;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaEventDestroy(c);
  cudaStreamDestroy(s0);
  cudaStreamDestroy(s1);
  cudaFree(d0);
  cudaFree(d1);
  cudaFreeHost(h0);
  cudaFreeHost(h1);
  return HT_OK;
}

// ---------------------------------------------------------------------------
// GEMM unit entry (tests): the exact launchers the layer drivers use, on
// host arrays.  op 0: C = relu(A W); 1: C = [A W > 0] * G; 2: C = A W^T
// (A is M x N, W is K x N); 3: C = A^T G (A is M x K, G is M x N).
// precision: HT_PREC_FP32 (SIMT) or HT_PREC_TF32 (tcgen05; 3xTF32 for ops
// 0/1, 1xTF32 for ops 2/3).
// ---------------------------------------------------------------------------
extern "C" int ht_gemm_test(int op, int precision, const float* A, const float* W, const float* G,
                            float* C, int64_t M, int K, int N) {
  CU(cudaSetDevice(0));
  cudaStream_t s = nullptr;
  CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // row operands are staged with row strides padded to 4 floats (the TMA
  // alignment rule the layer drivers follow for their own staging)
  const int ka = op == 2 ? N : K, lda = pad4(ka), ldn = pad4(N);
  const int64_t c_rows = op == 3 ? K : M, c_cols = op == 2 ? K : N;
  Device d;
  d.stream = s;
  DBuf dA, dG, dC, ws;
  HT_TRY(dA.ensure(std::max<int64_t>(1, M * lda) * 4));
  HT_TRY(dG.ensure(std::max<int64_t>(1, M * ldn) * 4));
  HT_TRY(dC.ensure(std::max<int64_t>(1, c_rows * c_cols) * 4));
  HT_TRY(ws.ensure((int64_t)148 * K * N * 4 + 4));
  CU(cudaMemcpy2D(dA.p, lda * 4, A, ka * 4, ka * 4, M, cudaMemcpyHostToDevice));
  if (G) CU(cudaMemcpy2D(dG.p, ldn * 4, G, N * 4, N * 4, M, cudaMemcpyHostToDevice));
  if (W) HT_TRY(upload_weights(d, W, K, N));
  CU(cudaMemset(dC.p, 0, c_rows * c_cols * 4));
  const bool tc = precision == HT_PREC_TF32;
  int rc = HT_OK;
  if (op == 0) {
    rc = tc ? ht::tc::rows<ht::tc::TC_RELU>(s, true, dA.as<float>(), lda, M, K, d.Wt_hi.as<float>(),
                                            d.Wt_lo.as<float>(), K, N, dC.as<float>(), N, nullptr, 0)
            : gemm<false, false, ht::EPI_RELU>(s, dA.as<float>(), lda, d.W.as<float>(), N,
                                               dC.as<float>(), N, nullptr, 0, M, N, K, 1, K);
  } else if (op == 1) {
    rc = tc ? ht::tc::rows<ht::tc::TC_MASK>(s, true, dA.as<float>(), lda, M, K, d.Wt_hi.as<float>(),
                                            d.Wt_lo.as<float>(), K, N, dC.as<float>(), N,
                                            dG.as<float>(), ldn)
            : gemm<false, false, ht::EPI_MASK>(s, dA.as<float>(), lda, d.W.as<float>(), N,
                                               dC.as<float>(), N, dG.as<float>(), ldn, M, N, K, 1, K);
  } else if (op == 2) {
    rc = tc ? ht::tc::rows<ht::tc::TC_STORE>(s, false, dA.as<float>(), lda, M, N, d.Wp_hi.as<float>(),
                                             nullptr, pad4(N), K, dC.as<float>(), K, nullptr, 0)
            : gemm<false, true, ht::EPI_STORE>(s, dA.as<float>(), lda, d.W.as<float>(), N,
                                               dC.as<float>(), K, nullptr, 0, M, K, N, 1, N);
  } else if (op == 3) {
    int used = 1;
    if (tc) {
      rc = ht::tc::wgrad(s, dA.as<float>(), lda, K, dG.as<float>(), ldn, N, M, 148, ws.as<float>(),
                         &used);
    } else {
      int splits = (int)std::min<int64_t>(64, std::max<int64_t>(1, M / 2048));
      int64_t kps = ((M + splits - 1) / splits + 15) / 16 * 16;
      used = (int)std::max<int64_t>(1, (M + kps - 1) / kps);
      rc = gemm<true, false, ht::EPI_STORE>(s, dA.as<float>(), lda, dG.as<float>(), ldn,
                                            ws.as<float>(), N, nullptr, 0, K, N, M, used, kps);
    }
    if (rc == HT_OK) {
      ht::k_reduce_splits<<<64, 256, 0, s>>>(dC.as<float>(), ws.as<float>(), (int64_t)K * N, used);
      CU(cudaGetLastError());
    }
  } else {
    rc = fail(HT_EINVAL, "unknown gemm op %d", op);
  }
  if (rc == HT_OK) {
    CU(cudaStreamSynchronize(s));
    CU(cudaMemcpy(C, dC.p, c_rows * c_cols * 4, cudaMemcpyDeviceToHost));
  }
  for (DBuf* b : {&dA, &dG, &dC, &ws, &d.W, &d.Wt, &d.Wp, &d.Wt_hi, &d.Wt_lo, &d.Wp_hi, &d.Wp_lo})
    b->release();
  cudaStreamDestroy(s);
  return rc;
}
