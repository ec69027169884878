// C ABI of the fleet: memory, fleet construction, plan upload, the
// Alg. 2/3 comm steps, epoch begin, SGD and timing (include/hongtu_b200.h).

#include "ht_fleet_internal.h"

using ht::fail;

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
    for (auto* b : {&d.value, &d.grad, &d.sa, &d.sb, &d.sc, &d.sd, &d.se, &d.partial, &d.work,
                    &d.gemm_ws, &d.W, &d.Wt, &d.Wp, &d.Wt_hi, &d.Wt_lo, &d.Wp_hi, &d.Wp_lo, &d.hL,
                    &d.labels, &d.mask, &d.loss_part, &d.gWall, &d.flags})
      b->release();
    for (auto& c : d.chunks) {
      for (auto* b : {&c.nbr_slot, &c.dest_rows, &c.csc_off, &c.csc_slot, &c.csc_w, &c.csr_off,
                      &c.csr_dst, &c.csr_w, &c.bx_off, &c.csc_loc, &c.csr_perm, &c.h2d_m,
                      &c.flush_m, &c.csc_gid, &c.nbr_gid})
        b->release();
      for (Pieces* pc : {&c.fw, &c.bw, &c.bx}) pc->release();
      for (CopyList* cl : {&c.h2d, &c.flush, &c.base_bwd, &c.dest})
        cl->src.release(), cl->dst.release(), cl->flag.release();
      for (auto& cl : c.d2d) cl.src.release(), cl.dst.release(), cl.flag.release();
      for (auto& cl : c.push) cl.src.release(), cl.dst.release(), cl.flag.release();
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
                    &d.g_al, &d.g_sgt, &d.g_eld, &d.g_gq, &d.g_gts, &d.g_ghd, &d.g_gin[0],
                    &d.g_gin[1], &d.g_cpart, &d.g_pgts})
      b->release();
    for (auto* v : {&d.g_pl, &d.g_elsl})
      for (auto& b : *v) b.release();
    for (cudaEvent_t e : {d.e_gcomp[0], d.e_gcomp[1], d.e_up, d.e_mg})
      if (e) cudaEventDestroy(e);
    for (auto* v : {&d.mh, &d.ma, &d.mg})
      for (auto& b : *v) b.release();
    d.mrows_d.release();
    d.own.src.release(), d.own.dst.release(), d.own.flag.release();
    for (DBuf* b : {&d.sgd_p, &d.sgd_w, &d.sgd_t, &d.pf_p, &d.pf_z, &d.tT, &d.agg_scr}) b->release();
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
  f->flag_ptrs.release();
  delete f;
  return HT_OK;
}

static void release_lists(std::vector<CopyList>& v) {
  for (auto& cl : v) cl.src.release(), cl.dst.release(), cl.flag.release();
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
        release_lists(c.d2d);  // (a re-finalize: free the previous lists)
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
        c.dest_ident = true;
        for (int64_t r = 0; r < (int64_t)h.dest.size() && c.dest_ident; ++r)
          c.dest_ident = h.dest[r] == r;
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
        HT_TRY(make_pieces(h.csc_off, c.fw, s));
        HT_TRY(make_pieces(h.csr_off, c.bw, s));
        c.bx_rows = -1;
        if (m == 1 && n == 1 && f->nrows < ((int64_t)1 << 31)) {
          std::vector<int64_t> offx(f->nrows + 1);
          int64_t q = 0;
          for (int64_t g = 0; g <= f->nrows; ++g) {
            while (q < h.nn && h.nbr[q] < g) ++q;
            offx[g] = h.csr_off[q];
          }
          HT_TRY(make_pieces(offx, c.bx, s));
          HT_TRY(upload(c.bx_off, offx, s));
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
        release_lists(c.push);
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

extern "C" int ht_fleet_set_budget(ht_fleet* f, int64_t bytes) {
  if (bytes < 0) return fail(HT_EINVAL, "HBM budget must be >= 0 bytes");
  f->hbm_budget = bytes;
  return HT_OK;
}

extern "C" int ht_fleet_recompute_state(ht_fleet* f, int64_t* mask) {
  *mask = 0;
  for (size_t l = 0; l < f->agg_recompute.size() && l < 63; ++l)
    if (f->agg_recompute[l]) *mask |= (int64_t)1 << l;
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
  // recomputed layers share one scratch buffer: always re-aggregate on read
  const bool recomputed = layer < (int)f->agg_recompute.size() && f->agg_recompute[layer];
  for (auto& d : f->dev) {
    if (!d.local) continue;
    if (!d.cache || (int)d.ma.size() <= layer || !d.ma[layer].p)
      return fail(HT_ESTATE, "checkpoints are not held in HBM mirrors");
    HT_TRY(set_dev(d));
    if (deferred || recomputed) {  // agg^l = A.h^l now, the forward's gather
      const int din = f->dims[layer];
      for (auto& c : d.chunks)
        HT_TRY(launch_seg(d.stream, d, d.ma[layer].as<float>() + c.dest_m0 * din,
                          d.mh[layer].as<float>(), din, din, c.csc_off.as<int64_t>(),
                          c.csc_gid.as<int32_t>(), c.csc_w.as<float>(), c.nv, c.fw));
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

