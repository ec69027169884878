// Fleet runtime helpers shared by the layer drivers (see ht_fleet_internal.h).

#include "ht_fleet_internal.h"

using ht::fail;

namespace htf {

std::atomic<int64_t> g_launches{0};

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
                int64_t sstride, int64_t dbase, int max_grid) {
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

int launch_acc(cudaStream_t s, int elem, void* dst, void* src, const int64_t* didx,
               const int64_t* sidx, const uint8_t* first, int64_t rows, int d, int zero_src,
               int64_t sbase) {
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

void timer_begin(ht_fleet* f, Device& d, TimerRec& r, cudaStream_t s) {
  if (!f->timing) return;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s ? s : d.stream);
}
void timer_end(ht_fleet* f, Device& d, TimerRec& r, int which, double bytes,
               cudaStream_t s) {
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

// Segment gather-sum over a chunk's CSC (forward) or CSR (backward) view.
// float4 rows (d % 4 == 0, the tf32 path's pad4 widths): ONE work-list
// launch - the pieces of the long segments first, then batches of short
// segments, taken from a device counter by whichever warp is free; the
// last piece of a long segment to finish sums its partials in piece order
// (k_seg_work_*).  Other widths (the fp32 validation path's odd widths):
// the per-segment kernel, the pieces kernel and the fixup in turn.

// work-list kernel shape: segment rows in flight (NV = 1 / 2 float4 words
// per lane), segments per unit, resident CTAs per SM - compile-time knobs
// for same-box A/B variant builds (build.py --variant), defaults measured
// (r2 sweep: US1 4, US2 4, B 8, MINB 3 - 42.6 vs 44.5 ms per cfg-2 epoch)
#ifndef HT_WL_US1
#define HT_WL_US1 4
#endif
#ifndef HT_WL_US2
#define HT_WL_US2 4
#endif
#ifndef HT_WL_B
#define HT_WL_B 8
#endif
#ifndef HT_WL_MINB
#define HT_WL_MINB 3
#endif
#ifndef HT_WL_UP
#define HT_WL_UP 8  // piece rows in flight
#endif
#ifndef HT_WL_SUB_U
#define HT_WL_SUB_U 8  // narrow rows: rows in flight per sub-group
#endif
#ifndef HT_WL_SUB_B
#define HT_WL_SUB_B 4
#endif
#ifndef HT_WL_SUB_MINB
#define HT_WL_SUB_MINB 4
#endif

int launch_seg(cudaStream_t s, Device& dv, float* out, const float* X, int64_t ldx, int d,
               const int64_t* off, const int32_t* idx, const float* w, int64_t nseg,
               const Pieces& pc) {
  if (nseg <= 0) return HT_OK;
  const int64_t np = pc.np, nf = pc.nf;
  static const bool sub_ok = [] {  // HT_NO_SUBWARP=1: narrow rows on the warp kernels
    const char* e = getenv("HT_NO_SUBWARP");
    return !(e && atoi(e));
  }();
  static const bool worklist = [] {  // HT_SEG_SPLIT_LAUNCH=1: r1's three-launch sequence
    const char* e = getenv("HT_SEG_SPLIT_LAUNCH");
    return !(e && atoi(e));
  }();
  float* partial = dv.partial.as<float>();
  if (d % 4 == 0 && d <= 512 && worklist) {
    ht::SegWork wk{off, idx, w, nseg, kSplit, pc.lo.as<int64_t>(), pc.hi.as<int64_t>(),
                   pc.pf.as<int32_t>(), np, pc.seg.as<int64_t>(), pc.first.as<int64_t>(),
                   pc.cnt.as<int64_t>(), dv.work.as<unsigned>(), dv.work.as<int>() + 1, partial};
    if (dv.work.bytes < (nf + 2) * 4) return fail(HT_ESTATE, "work-list buffer not sized");
    CU(cudaMemsetAsync(dv.work.p, 0, (nf + 2) * 4, s));  // counter + fixup tickets
    count_launch();
    if (d <= 64 && sub_ok) {  // narrow rows: 2 or 4 segments per warp
      if (d <= 32) {
        auto k = ht::k_seg_work_sub<8, HT_WL_SUB_U, HT_WL_SUB_B, HT_WL_SUB_MINB>;
        k<<<resident_grid(k, (nseg + 3) / 4), kThreads, 0, s>>>(out, X, ldx, d, wk);
      } else {
        auto k = ht::k_seg_work_sub<16, HT_WL_SUB_U, HT_WL_SUB_B, HT_WL_SUB_MINB>;
        k<<<resident_grid(k, (nseg + 1) / 2), kThreads, 0, s>>>(out, X, ldx, d, wk);
      }
    } else {
      switch ((d / 4 + 31) / 32) {
        case 1: { auto k = ht::k_seg_work_v4<1, HT_WL_US1, HT_WL_UP, HT_WL_B, HT_WL_MINB>; k<<<resident_grid(k, nseg), kThreads, 0, s>>>(out, X, ldx, d, wk); break; }
        case 2: { auto k = ht::k_seg_work_v4<2, HT_WL_US2, HT_WL_UP, HT_WL_B, HT_WL_MINB>; k<<<resident_grid(k, nseg), kThreads, 0, s>>>(out, X, ldx, d, wk); break; }
        case 3: { auto k = ht::k_seg_work_v4<3, 2, 4, 16, 2>; k<<<resident_grid(k, nseg), kThreads, 0, s>>>(out, X, ldx, d, wk); break; }
        default: { auto k = ht::k_seg_work_v4<4, 2, 4, 16, 2>; k<<<resident_grid(k, nseg), kThreads, 0, s>>>(out, X, ldx, d, wk); break; }
      }
    }
    CU(cudaGetLastError());
    return HT_OK;
  }
  const int g = grid_for(nseg);
  count_launch(1 + (np ? 1 : 0) + (nf ? 1 : 0));
  const DBuf &lo = pc.lo, &hi = pc.hi;
  if (d % 4 == 0 && d <= 64 && sub_ok) {
    if (d <= 32) {
      ht::k_seg_gather_sub<8><<<grid_for((nseg + 3) / 4), kThreads, 0, s>>>(out, X, ldx, d, off, idx,
                                                                           w, nseg, kSplit);
      if (np) ht::k_seg_pieces_sub<8><<<grid_for((np + 3) / 4), kThreads, 0, s>>>(
          partial, X, ldx, d, lo.as<int64_t>(), hi.as<int64_t>(), idx, w, np);
    } else {
      ht::k_seg_gather_sub<16, 8, 4><<<grid_for((nseg + 1) / 2), kThreads, 0, s>>>(
          out, X, ldx, d, off, idx, w, nseg, kSplit);
      if (np) ht::k_seg_pieces_sub<16><<<grid_for((np + 1) / 2), kThreads, 0, s>>>(
          partial, X, ldx, d, lo.as<int64_t>(), hi.as<int64_t>(), idx, w, np);
    }
  } else if (d % 4 == 0 && d <= 512) {
    const int nv = (d / 4 + 31) / 32;
#define SEGV(NV)                                                                               \
  ht::k_seg_gather_v4<NV, (NV == 1 ? 8 : 2), 4><<<g, kThreads, 0, s>>>(out, X, ldx, d, off, idx, \
                                                                       w, nseg, kSplit);       \
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
    ht::k_seg_fixup<<<grid_for(nf), kThreads, 0, s>>>(out, partial, d, pc.seg.as<int64_t>(),
                                                       pc.first.as<int64_t>(), pc.cnt.as<int64_t>(), nf);
    CU(cudaGetLastError());
  }
  return HT_OK;
}

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
int make_pieces(const std::vector<int64_t>& off, Pieces& pc, cudaStream_t s) {
  std::vector<int64_t> lo, hi, seg, first, cnt;
  std::vector<int32_t> pf;
  for (size_t sg = 0; sg + 1 < off.size(); ++sg) {
    const int64_t a = off[sg], b = off[sg + 1];
    if (b - a <= kSplit) continue;
    seg.push_back((int64_t)sg);
    first.push_back((int64_t)lo.size());
    int64_t c = 0;
    for (int64_t x = a; x < b; x += kSplit, ++c) {
      lo.push_back(x);
      hi.push_back(std::min(b, x + kSplit));
      pf.push_back((int32_t)(seg.size() - 1));
    }
    cnt.push_back(c);
  }
  pc.np = (int64_t)lo.size();
  pc.nf = (int64_t)seg.size();
  HT_TRY(upload(pc.lo, lo, s));
  HT_TRY(upload(pc.hi, hi, s));
  HT_TRY(upload(pc.seg, seg, s));
  HT_TRY(upload(pc.first, first, s));
  HT_TRY(upload(pc.cnt, cnt, s));
  HT_TRY(upload(pc.pf, pf, s));
  return HT_OK;
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
                cudaStream_t s, const std::vector<uint8_t>* flag) {
  cl.n = (int64_t)src.size();
  HT_TRY(upload(cl.src, src, s));
  HT_TRY(upload(cl.dst, dst, s));
  if (flag) HT_TRY(upload(cl.flag, *flag, s));
  return HT_OK;
}


// communication steps (Alg. 2 / Alg. 3)
// ===========================================================================

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
int push_flush(ht_fleet* f, int j, void* host_grad_dev, bool assume_zero, int layer) {
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
    *rows = c.dest_ident ? nullptr : c.dest_rows.as<int64_t>();  // (identity: row r is r)
    return static_cast<const float*>(f->hptr[layer + 1]);
  }
  return nullptr;
}

// m = 1: the layer input h^l as an HBM array indexed by global row (the
// owner-cache mirror when it is the identity map, or an HBM host store),
// or nullptr.  The gathers then read it in place: no slot loads.
const float* hbm_inputs(ht_fleet* f, Device& d, int layer, const void* hin) {
  if (f->m != 1 || !d.chunks[0].csc_gid.p || f->sw.no_direct_read) return nullptr;
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
         (d.mrows.empty() || d.mrows.back() == d.mcount - 1) && !f->sw.no_direct_bwd;
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
  return !f->sw.no_gat_direct && direct_bwd(f, d) && c.bx_rows == d.mcount && c.nv == d.mcount && c.dest_m0 == 0;
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
         !f->sw.no_project_first;
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
// Owner-cache decision of one device under the HBM budget (the recompute-
// cache hybrid).  The h^l and grad_h^l mirrors (and the
// one-device buffers of project-first layers / GAT kept projections) must
// fit; agg^l mirrors are kept greedily from the narrowest layer up, and a
// single scratch buffer of the widest remaining layer serves the others -
// their agg^l is re-aggregated in the backward from the h^l mirror (the
// forward's gather: bitwise the same rows).  Recompute needs the gathers to
// read the mirror in place (one device, identity mirror); elsewhere the
// cache is all or nothing.
int plan_cache(ht_fleet* f, Device& d, int L, const int* dims, bool gat, int64_t mv, int64_t mn,
               int dmax) {
  const int64_t R = std::max<int64_t>(1, d.mcount);
  int64_t base = 0;
  for (int l = 0; l < L; ++l) base += R * dims[l] * 4;   // h mirrors
  for (int l = 0; l <= L; ++l) base += R * dims[l] * 4;  // grad mirrors
  const bool one = f->m == 1 && d.mcount == f->nrows && d.chunks[0].csc_gid.p &&
                   (d.mrows.empty() || d.mrows.back() == d.mcount - 1) && !f->sw.no_direct_read;
  if (gat) {  // GAT staging allocated after this decision (ht_gat_epoch_begin)
    int64_t me = 1;
    for (int j = 0; j < f->n; ++j) me = std::max(me, d.chunks[j].ne);
    base += (3 * mn + 4 * mv) * (int64_t)dmax * 4 + 4 * me * 4;
    if (one && f->n == 1)  // gat_direct: each layer's projection and el_src kept
      for (int l = 0; l < L; ++l) base += R * (pad4(dims[l + 1]) + 1) * 4;
  } else if (one && f->n == 1) {  // project-first buffers (pf_p, pf_z)
    int pw = 0;
    for (int l = 0; l < L; ++l)
      if (dims[l + 1] < dims[l]) pw = std::max(pw, pad4(dims[l + 1]));
    base += 2 * R * pw * 4;
  }
  size_t fr = 0, tot = 0;
  CU(cudaMemGetInfo(&fr, &tot));
  // the previous epoch's mirrors / scratch / project-first buffers are
  // reused (grow-only): they count as available
  int64_t held = 0;
  for (auto* v : {&d.mh, &d.ma, &d.mg})
    for (auto& b : *v)
      if (!b.alias) held += b.bytes;
  for (DBuf* b : {&d.agg_scr, &d.pf_p, &d.pf_z}) held += b->bytes;
  int64_t avail = (int64_t)fr + held - ((int64_t)4 << 30);
  if (f->hbm_budget > 0) avail = std::min(avail, f->hbm_budget);
  int64_t agg_all = 0;
  if (!gat)
    for (int l = 0; l < L; ++l) agg_all += R * dims[l] * 4;
  if (getenv("HT_TRACE_CACHE"))
    fprintf(stderr, "[ht] owner cache plan: mirrors+buffers %.2f GB, agg %.2f GB, available %.2f GB "
                    "(free %.2f GB + held %.2f GB, budget %.2f GB)\n", base / 1e9, agg_all / 1e9,
            avail / 1e9, fr / 1e9, held / 1e9, f->hbm_budget / 1e9);
  if (base + agg_all <= avail) {
    d.cache = true;
    return HT_OK;
  }
  const bool recompute_ok = !gat && one && !f->sw.no_recompute;
  if (recompute_ok) {
    std::vector<int> order(L);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return dims[a] < dims[b]; });
    for (int keep = L - 1; keep >= 0; --keep) {  // keep the `keep` narrowest agg mirrors
      int64_t need = base;
      int scr = 0;
      for (int q = 0; q < L; ++q) {
        if (q < keep) need += R * dims[order[q]] * 4;
        else scr = std::max(scr, dims[order[q]]);
      }
      need += R * scr * 4;
      if (need <= avail) {
        for (int q = keep; q < L; ++q) f->agg_recompute[order[q]] = 1;
        d.cache = true;
        return HT_OK;
      }
    }
  }
  if (f->cache_req == 1)
    return fail(HT_ENOMEM, "HBM owner cache needs %lld bytes (%lld with recompute), %lld available",
                (long long)(base + agg_all), (long long)base, (long long)avail);
  d.cache = false;
  for (auto* v : {&d.mh, &d.ma, &d.mg})  // room for the host-path staging
    for (auto& b : *v) b.release();
  d.agg_scr.release();
  return HT_OK;
}

int epoch_begin_impl(ht_fleet* f, int L, const int* dims, int64_t extra_grad, bool gat) {
  if (!f->finalized) return fail(HT_ESTATE, "fleet not finalized");
  HT_TRY(check_chunks(f));
  HT_TRY(sync_all(f));
  f->sw.read();
  f->L = L;
  f->dims.assign(dims, dims + L + 1);
  f->hptr.assign(L + 1, nullptr);
  f->hdev.assign(L + 1, 0);
  f->agg_deferred.assign(L, 0);
  f->agg_recompute.assign(L, 0);
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
    int64_t mv = 1, mn = 1, np = 1, nf = 0;
    d.hL_off.assign(f->n + 1, 0);
    for (int j = 0; j < f->n; ++j) {
      mv = std::max(mv, d.chunks[j].nv);
      mn = std::max(mn, d.chunks[j].nn);
      np = std::max({np, d.chunks[j].fw.np, d.chunks[j].bw.np, d.chunks[j].bx.np});
      nf = std::max({nf, d.chunks[j].fw.nf, d.chunks[j].bw.nf, d.chunks[j].bx.nf});
      d.hL_off[j + 1] = d.hL_off[j] + d.chunks[j].nv;
    }
    // sized for 180 GB of HBM: the buffers every path needs first, then
    // either the owner-cache mirrors or the host-path staging sets
    HT_TRY(d.sc.ensure(mv * dmax * 4));
    HT_TRY(d.sd.ensure(mv * dmax * 4));
    int narrow_w = 0;  // widest d_out of the layers whose backward runs narrow-side
    for (int l = 0; l < L; ++l)
      if (dims[l + 1] < dims[l]) narrow_w = std::max(narrow_w, pad4(dims[l + 1]));
    if (narrow_w)  // (the expanded CSR of one device / one batch has a row per host row)
      HT_TRY(d.tT.ensure(std::max<int64_t>(mn, f->m == 1 && f->n == 1 ? f->nrows : 0) * narrow_w * 4));
    HT_TRY(d.partial.ensure(np * dmax * 4));
    HT_TRY(d.work.ensure((nf + 2) * 4));
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
        HT_TRY(plan_cache(f, d, L, dims, gat, mv, mn, dmax));
      }
    }
    // the slot value buffer: not needed when a single device's gathers read
    // the identity-mapped mirror in place (hbm_inputs)
    const bool direct = d.cache && f->m == 1 && d.chunks[0].csc_gid.p &&
                        d.mcount == f->nrows && !f->sw.no_direct_read;
    if (!direct) HT_TRY(d.value.ensure(std::max<int64_t>(1, d.cap) * dmax * 4));
    // slot gradients and neighbour-gradient views: not needed when one
    // device's backward writes the grad mirror in place (cfg 4's share: 22 GB)
    const bool dbwd = gat ? gat_direct(f, d) : direct_bwd(f, d);
    const bool dviews = gat ? gat_direct(f, d) : direct_bwd(f, d) && d.chunks[0].bx_rows == d.mcount;
    if (!dbwd) HT_TRY(d.grad.ensure(std::max<int64_t>(1, d.cap) * dmax * 4));
    if (!dviews) HT_TRY(d.se.ensure(mn * dmax * 4));
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
      int scr = 0;  // widest recomputed layer
      for (int l = 0; l < (gat ? 0 : L); ++l)
        if (f->agg_recompute[l]) scr = std::max(scr, dims[l]);
      if (scr) {
        HT_TRY(d.agg_scr.ensure(std::max<int64_t>(1, d.mcount) * scr * 4));
      } else {
        d.agg_scr.release();
      }
      for (int l = 0; l < (gat ? 0 : L); ++l) {
        if (f->agg_recompute[l])
          d.ma[l].set_alias(d.agg_scr.p);
        else
          HT_TRY(d.ma[l].ensure(std::max<int64_t>(1, d.mcount) * dims[l] * 4));
      }
      if (!gat && f->m == 1 && f->n == 1) {  // project-first buffers, sized once (no
        int pw = 0;                          // allocation inside a layer call)
        for (int l = 0; l < L; ++l)
          if (dims[l + 1] < dims[l]) pw = std::max(pw, pad4(dims[l + 1]));
        if (pw) {
          HT_TRY(d.pf_p.ensure(std::max<int64_t>(1, d.mcount) * pw * 4));
          HT_TRY(d.pf_z.ensure(std::max<int64_t>(1, d.mcount) * pw * 4));
        }
      }
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


}  // namespace htf
