// GAT epoch layer drivers (engine.py:196-289 of the reference).

#include "ht_fleet_internal.h"

using ht::fail;

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

#ifndef HT_GAT_S1B
#define HT_GAT_S1B 8  // sources per S1 work unit
#endif
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
int launch_gat_dst(cudaStream_t s, Device& dv, const DevChunk& c, const float* Q, const float* P,
                   const float* els, const float* a_dst, int d, float slope, float* H,
                   const float* G, float* GS, float* GP, float* AL, float* GT, float* SGT,
                   const float* HO = nullptr, const int64_t* ho_rows = nullptr,
                   bool global_src = false) {
  if (c.nv <= 0) return HT_OK;
  const int64_t* off = c.csc_off.as<int64_t>();
  // sources as chunk-local rows of Q, or (direct) as global rows of P
  const int32_t* idx = global_src ? c.csc_gid.as<int32_t>() : c.csc_loc.as<int32_t>();
  if (dv.work.bytes < 4) return fail(HT_ESTATE, "work buffer not sized");
  CU(cudaMemsetAsync(dv.work.p, 0, 4, s));  // the destination-batch counter
  count_launch();
#define GATD(NV)                                                                              \
  {                                                                                           \
    auto k = ht::gat::k_gat_dst<NV, BWD>;                                                     \
    k<<<resident_grid(k, c.nv), kThreads, 0, s>>>(off, idx, c.nv, Q, P, els, a_dst, d, slope, \
                                                  H, G, GS, GP, AL, GT, SGT, HO, ho_rows,    \
                                                  dv.work.as<unsigned>());                   \
  }
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

// Split backward (k_gat_bwd_a / s1 / b / s2, ht_gat.cuh) when the layer
// output is in HBM: one row gather per edge instead of two.  AL: per-edge
// {alpha, g_alpha -> g_t} records; GQ receives gq; ELD, SGT, GTS scalars.
int launch_gat_bwd_split(cudaStream_t s, Device& dv, const DevChunk& c, const float* Q,
                         const float* P, const float* els, const float* a_dst, const float* a_src,
                         int d, float slope, const float* G, const float* HO,
                         const int64_t* ho_rows, float* GS, float* GP, float* AL, float* ELD,
                         float* SGT, float* GQ, float* GTS, float* part, float* pgts,
                         bool expanded, const float* sgt_add) {
  const int64_t* coff = c.csc_off.as<int64_t>();
  const int32_t* cidx = expanded ? c.csc_gid.as<int32_t>() : c.csc_loc.as<int32_t>();
  const Pieces& pc = expanded ? c.bx : c.bw;
  const int64_t nseg = expanded ? c.bx_rows : c.nn;
  const int64_t* roff = expanded ? c.bx_off.as<int64_t>() : c.csr_off.as<int64_t>();
  const int32_t* dst = c.csr_dst.as<int32_t>();
  const int32_t* perm = c.csr_perm.as<int32_t>();
  if (dv.work.bytes < (pc.nf + 2) * 4) return fail(HT_ESTATE, "work buffer not sized");
  count_launch(4);
#define GATB(NV)                                                                                   \
  if (c.nv > 0) {                                                                                  \
    CU(cudaMemsetAsync(dv.work.p, 0, 4, s));                                                       \
    auto ka = ht::gat::k_gat_bwd_a<NV>;                                                            \
    ka<<<resident_grid(ka, c.nv), kThreads, 0, s>>>(coff, cidx, c.nv, P, els, a_dst, d, slope, G,   \
                                                    HO, ho_rows, GS, AL, ELD,                      \
                                                    dv.work.as<unsigned>());                       \
  }                                                                                                \
  if (nseg > 0) {                                                                                  \
    CU(cudaMemsetAsync(dv.work.p, 0, (pc.nf + 2) * 4, s)); /* S1 counter + tickets */               \
    auto k1 = ht::gat::k_gat_bwd_s1_work<NV, HT_GAT_S1B>;                                                    \
    k1<<<resident_grid(k1, nseg), kThreads, 0, s>>>(                                                \
        roff, dst, perm, nseg, kSplit, pc.lo.as<int64_t>(), pc.hi.as<int64_t>(),                    \
        pc.pf.as<int32_t>(), pc.seg.as<int64_t>(), pc.first.as<int64_t>(), pc.cnt.as<int64_t>(),     \
        pc.np, dv.work.as<unsigned>(), dv.work.as<int>() + 1, GS, Q, AL, d, part, GQ);             \
  }                                                                                                \
  if (c.nv > 0) {                                                                                  \
    CU(cudaMemsetAsync(dv.work.p, 0, 4, s));                                                       \
    auto kb = ht::gat::k_gat_bwd_b<NV>;                                                            \
    kb<<<resident_grid(kb, c.nv), kThreads, 0, s>>>(coff, cidx, c.nv, els, ELD, slope, AL, SGT,     \
                                                    GP, a_dst, d, dv.work.as<unsigned>());         \
  }                                                                                                \
  if (nseg > 0) {                                                                                  \
    CU(cudaMemsetAsync(dv.work.p, 0, (pc.nf + 2) * 4, s)); /* S2 counter + tickets */               \
    auto k2 = ht::gat::k_gat_bwd_s2<NV>;                                                           \
    k2<<<resident_grid(k2, nseg + pc.np), kThreads, 0, s>>>(                                       \
        roff, perm, nseg, kSplit, pc.lo.as<int64_t>(), pc.hi.as<int64_t>(), pc.pf.as<int32_t>(),   \
        pc.seg.as<int64_t>(), pc.first.as<int64_t>(), pc.cnt.as<int64_t>(), pc.np,                 \
        dv.work.as<unsigned>(), dv.work.as<int>() + 1, pgts, AL, a_src, sgt_add, a_dst, d, GQ,     \
        GTS);                                                                                      \
  }
  switch (nv_of(d)) {
    case 1: GATB(1); break;
    case 2: GATB(2); break;
    case 3: GATB(3); break;
    default: GATB(4); break;
  }
#undef GATB
  CU(cudaGetLastError());
  return HT_OK;
}

int launch_gat_src(cudaStream_t s, const DevChunk& c, const float* GS, const float* AL,
                   const float* GT, const float* a_src, int d, float* GQ, float* GTS, float* part,
                   float* pgts, bool expanded = false, const float* sgt_add = nullptr,
                   const float* a_dst = nullptr) {
  // expanded: segments over every host row (gat_direct), outputs in row order
  const int64_t nseg = expanded ? c.bx_rows : c.nn;
  const Pieces& pc = expanded ? c.bx : c.bw;
  const int64_t np = pc.np, nf = pc.nf;
  const DBuf &lo = pc.lo, &hi = pc.hi;
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
    const DBuf &sg = pc.seg, &fi = pc.first, &cn = pc.cnt;
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
    HT_TRY(d.g_al.ensure(me * 8));  // {alpha, g_t} records per edge
    HT_TRY(d.g_sgt.ensure(mv * 4));
    HT_TRY(d.g_eld.ensure(mv * 4));
    HT_TRY(d.g_gq.ensure(mn * dmax * 4));
    HT_TRY(d.g_gts.ensure(mn * 4));
    HT_TRY(d.g_ghd.ensure(mv * dmax * 4));
    HT_TRY(d.g_cpart.ensure((int64_t)kColBlocks * dmax * 4));
    int64_t np = 1;
    for (int j = 0; j < f->n; ++j) np = std::max({np, d.chunks[j].bw.np, d.chunks[j].bx.np});
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
  if (last) {
    f->hL_dim = d_out;
    f->top_gcn_prec = -1;  // (the loss writes no GCN gz rows)
  }
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
      HT_TRY(launch_gat_dst<false>(d.stream, d, c, Q, P, els, w.A.as<float>(), d_out, slope, H, nullptr,
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
    if (f->mode != HT_MODE_BASELINE && !gat_direct(f, d))  // zeroed gradient slots
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
      float *AL = d.g_al.as<float>(), *GT = AL + 1;  // interleaved {alpha, g_t}
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
      const bool split = HO && !f->sw.no_gat_split;
      if (split) {  // one row gather per edge (the h^{l+1} sign is in HBM)
        HT_TRY(launch_gat_bwd_split(d.stream, d, c, Q, P, els, a_dst, a_src, d_out, slope, Gin, HO,
                                    hrows, GS, dir ? nullptr : GP, AL, d.g_eld.as<float>(),
                                    d.g_sgt.as<float>(), GQ, d.g_gts.as<float>(),
                                    d.partial.as<float>(), d.g_pgts.as<float>(), dir,
                                    dir ? d.g_sgt.as<float>() : nullptr));
      } else {
        HT_TRY(launch_gat_dst<true>(d.stream, d, c, Q, P, els, a_dst, d_out, slope,
                                    nullptr, Gin, GS, dir ? nullptr : GP, AL, GT, d.g_sgt.as<float>(),
                                    HO, hrows, dir));
        HT_TRY(launch_gat_src(d.stream, c, GS, AL, GT, a_src, d_out, GQ, d.g_gts.as<float>(),
                              d.partial.as<float>(), d.g_pgts.as<float>(), dir,
                              dir ? d.g_sgt.as<float>() : nullptr, a_dst));
      }
      const int64_t nsrc = dir ? c.bx_rows : c.nn;
      // algorithmic bytes: split - per edge one gs row + 14 index / scalar
      // words; per destination p, h, g rows in, gs (+ gp) out; per source q
      // row in, gq out + read-modify-write.  Fused - per edge q and gs rows
      // (+ the recomputed sum without h in HBM)
      timer_end(f, d, tr, 1,
                split ? (double)c.ne * (56.0 + 4.0 * d_out) +
                            (double)c.nv * ((dir ? 16.0 : 20.0) * d_out + 12.0) +
                            (double)nsrc * (16.0 * d_out + 8.0)
                      : (double)c.ne * (28.0 + 12.0 * d_out) + (double)c.nv * (16.0 * d_out + 16.0) +
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

