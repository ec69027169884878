// Internal header of the fleet runtime (not part of the C ABI): the device /
// fleet state shared by the translation units
//   ht_runtime.cu     helpers: barriers, copies, segment launches, layer helpers
//   ht_fleet.cu       C ABI: memory, fleet construction, comm steps, epoch
//                     begin, SGD, timing
//   ht_gcn.cu         GCN forward / loss / backward layer drivers
//   ht_gat_layers.cu  GAT layer drivers
//   ht_probe.cu       PCIe probe, GEMM unit entry
// (devices.py / engine.py of the reference, re-designed for B200: slot
// buffers in HBM, zero-copy pinned host rows, peer-pointer fetches,
// per-device streams with event barriers at the Alg. 2/3 sync points).
#pragma once

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

namespace htf {

// long-segment piece length (edges); HT_SPLIT overrides it for tuning runs
const int64_t kSplit = [] {
  const char* e = getenv("HT_SPLIT");
  const long long v = e ? atoll(e) : 0;
  return (int64_t)(v >= 64 ? v : 1024);  // r1 sweep: 4096 -> 1024 saved 3 ms (GCN), 6 ms (GAT)
}();
constexpr int kThreads = 256;
constexpr int kMarks = 16;
extern std::atomic<int64_t> g_launches;  // kernels launched by this library
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
    const cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      return fail(e == cudaErrorMemoryAllocation ? HT_ENOMEM : HT_ECUDA,
                  "cudaMalloc of %lld bytes failed: %s (%lld of %lld bytes free)", (long long)want,
                  cudaGetErrorString(e), (long long)fr, (long long)tot);
    }
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
               const std::vector<uint8_t>* flag);

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

// Pieces of the long (> kSplit edges) segments of one offsets array: piece
// q covers edges [lo[q], hi[q]) of segment seg[pf[q]]; fixup f sums pieces
// first[f] .. first[f] + cnt[f] - 1 in piece order into segment seg[f].
struct Pieces {
  int64_t np = 0, nf = 0;
  DBuf lo, hi, seg, first, cnt;  // int64
  DBuf pf;                       // int32 [np]: fixup of each piece
  void release() {
    for (DBuf* b : {&lo, &hi, &seg, &first, &cnt, &pf}) b->release();
    np = nf = 0;
  }
};

struct DevChunk {
  int64_t nv = 0, nn = 0, ne = 0, nlive = 0;
  DBuf nbr_slot;   // int64 [nn]
  DBuf dest_rows;  // int64 [nv]
  bool dest_ident = false;  // dest_rows[r] == r for every r (one device, one batch)
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
  Pieces fw, bw;                     // long-segment pieces (forward CSC, backward CSR)
  // one device, one batch: the CSR offsets expanded to every host row
  // (empty segments for rows without out-edges) so the transposed
  // aggregation writes the dense grad mirror directly; pieces re-indexed
  DBuf bx_off;
  Pieces bx;
  int64_t bx_rows = -1;
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
  int gz_loss_ld = 0;  // > 0: the loss wrote the top layer's gz rows into sc (row stride)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev = nullptr;
  int64_t cap = 0;
  DBuf value, grad;                    // cap x dim slot buffers
  DBuf sa, sb, sc, sd, se, partial;    // staging
  DBuf work;                           // work-list counter + fixup tickets of launch_seg
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
  DBuf g_hn, g_hd[2], g_q, g_p, g_els, g_gs, g_gp, g_al, g_sgt, g_eld, g_gq, g_gts, g_ghd, g_gin[2];
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
  // recompute-cache hybrid: one scratch buffer serves every layer whose agg
  // mirror did not fit the HBM budget (ma[l] aliases it; the backward
  // re-aggregates agg^l from the h^l mirror)
  DBuf agg_scr;
  cudaEvent_t e_up = nullptr, e_mg = nullptr;
};

const float* hbm_outputs(ht_fleet* f, Device& d, int j, int layer, int d_out,
                         const int64_t** rows);

const float* hbm_inputs(ht_fleet* f, Device& d, int layer, const void* hin);

}  // namespace htf

using namespace htf;

// Validation switches: each turns one optimisation off
// to compare against the reference's association; read from the
// environment once per epoch (ht_epoch_begin), never inside the layer loops
struct Switches {
  bool no_project_first = false, no_narrow_bwd = false, no_gat_direct = false;
  bool no_direct_bwd = false, no_direct_read = false, no_recompute = false, no_gat_split = false;
  bool no_mask_fold = false;
  void read() {
    auto on = [](const char* k) { const char* e = getenv(k); return e && *e && atoi(e) != 0; };
    no_project_first = on("HT_NO_PROJECT_FIRST");
    no_narrow_bwd = on("HT_NO_NARROW_BWD");
    no_gat_direct = on("HT_NO_GAT_DIRECT");
    no_direct_bwd = on("HT_NO_DIRECT_BWD");
    no_direct_read = on("HT_NO_DIRECT_READ");
    no_recompute = on("HT_NO_RECOMPUTE");
    no_gat_split = on("HT_NO_GAT_SPLIT");
    no_mask_fold = on("HT_NO_MASK_FOLD");
  }
};

struct ht_fleet {
  int m = 0, n = 0, mode = HT_MODE_FULL, flush = HT_FLUSH_ON_EVICTION;
  Switches sw;
  std::vector<Device> dev;
  std::vector<std::vector<HostSets>> sets;  // [i][j]
  bool finalized = false;
  int dim = 0, elem = 4;
  int hL_dim = 0;
  // last forward layer was a GCN layer in this precision (-1: GAT / none):
  // the loss then also writes the top layer's gz = g * (h^L > 0) rows
  int top_gcn_prec = -1;
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
  // recompute-cache hybrid (the paper's policy): HBM budget
  // of the owner cache in bytes (0: free HBM less 4 GB of headroom) and the
  // layers whose agg^l is recomputed in the backward instead of kept
  int64_t hbm_budget = 0;
  std::vector<char> agg_recompute;
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

namespace htf {


inline int64_t chunk_bound(int64_t V, int g) { return V * g / kChunks; }

// grid of a persistent (work-list) kernel: its resident CTAs on every SM
template <class K>
inline int resident_grid(K kernel, int64_t warps_needed) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0) != cudaSuccess ||
      per_sm <= 0)
    per_sm = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (warps_needed * 32 + kThreads - 1) / kThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per_sm * sms));
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

int set_dev(const Device& d);

int xbarrier(ht_fleet* f);

int barrier(ht_fleet* f);

int sync_all(ht_fleet* f);

int ev_rec(cudaEvent_t& e, cudaStream_t s);

int ev_wait(cudaStream_t s, cudaEvent_t e);

int grid_for(int64_t warps_needed);

int dev_ptr(const void* p, void** out);

bool is_dev_mem(const void* p);

int launch_copy(cudaStream_t s, void* dst, const void* src, const int64_t* didx,
                const int64_t* sidx, int64_t rows, int64_t row_bytes, int64_t dstride,
                int64_t sstride, int64_t dbase = 0, int max_grid = 0);

int xfer(cudaStream_t s, const CopyList& cl, bool to_host, void* host_v, int64_t hld, void* dev_v,
         int64_t dld, int64_t rb, int64_t lo, int64_t hi);

int launch_acc(cudaStream_t s, int elem, void* dst, void* src, const int64_t* didx,
               const int64_t* sidx, const uint8_t* first, int64_t rows, int d, int zero_src,
               int64_t sbase = 0);

void timer_begin(ht_fleet* f, Device& d, TimerRec& r, cudaStream_t s = nullptr);

void timer_end(ht_fleet* f, Device& d, TimerRec& r, int which, double bytes,
               cudaStream_t s = nullptr);

void timers_collect(ht_fleet* f);

// Segment gather-sum over a chunk's CSC (forward) or CSR (backward) view:
// out[sg] = sum over edges e of segment sg of w[e] * X[idx[e]], sequential in
// e, long segments through their pieces (`pc`); d's partial / work buffers.
int launch_seg(cudaStream_t s, Device& dv, float* out, const float* X, int64_t ldx, int d,
               const int64_t* off, const int32_t* idx, const float* w, int64_t nseg,
               const Pieces& pc);

int upload_weights(Device& d, const float* W, int d_in, int d_out);

// pieces of the long segments of an offsets array, uploaded on stream s
int make_pieces(const std::vector<int64_t>& off, Pieces& pc, cudaStream_t s);

int lookup_slots(const HostSets& hs, const std::vector<int64_t>& rows, std::vector<int64_t>& out,
                 int i, int j);

std::vector<int64_t> vdiff(const std::vector<int64_t>& a, const std::vector<int64_t>& b);

std::vector<int64_t> visect(const std::vector<int64_t>& a, const std::vector<int64_t>& b);

int upload_list(CopyList& cl, const std::vector<int64_t>& src, const std::vector<int64_t>& dst,
                cudaStream_t s, const std::vector<uint8_t>* flag = nullptr);

int stage_batch(ht_fleet* f, int j, const void* host_rows_dev);

int push_flush(ht_fleet* f, int j, void* host_grad_dev, bool assume_zero, int layer = -1);

int upload_layer_weights(Device& d, int l, const float* W, int d_in, int d_out);

int check_chunks(ht_fleet* f);

bool direct_bwd(ht_fleet* f, Device& d);

bool gat_direct(ht_fleet* f, Device& d);

bool project_first(ht_fleet* f, Device& d, int d_in, int d_out, int precision);

int cache_upload(ht_fleet* f, Device& d, cudaStream_t s, const void* host, float* mirror,
                 int64_t rb);

int cache_writeback(ht_fleet* f, Device& d, void* host, const float* mirror, int64_t rb);

int put_dest(ht_fleet* f, DevChunk& c, cudaStream_t s, void* host, const float* dev, int64_t rb,
             int g);

int prefetch_checkpoints(ht_fleet* f, Device& d, int layer, void* aout, int64_t rbi);

int epoch_begin_impl(ht_fleet* f, int L, const int* dims, int64_t extra_grad, bool gat);

const float* hbm_outputs(ht_fleet* f, Device& d, int j, int layer, int d_out,
                         const int64_t** rows);

const float* hbm_inputs(ht_fleet* f, Device& d, int layer, const void* hin);

}  // namespace htf
