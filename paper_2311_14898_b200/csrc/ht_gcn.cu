// GCN epoch layer drivers: forward, loss, backward (engine.py:128-171,
// 297-320, 387-480 of the reference).

#include "ht_fleet_internal.h"

using ht::fail;

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
  if (last) {
    f->hL_dim = d_out;
    f->top_gcn_prec = precision;
  }
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
        HT_TRY(launch_seg(d.stream, d, d.pf_z.as<float>(), d.pf_p.as<float>(), ldp, ldp,
                          c.csc_off.as<int64_t>(), c.csc_gid.as<int32_t>(), c.csc_w.as<float>(),
                          c.nv, c.fw));
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
      if (d.cache && f->agg_recompute[layer] && !f->ckpt_hbm) {
        // the recompute scratch is shared by layers: wait for the
        // write-through of the previous layer's checkpoint rows out of it
        HT_TRY(ev_wait(d.stream, d.e_out[0]));
        HT_TRY(ev_wait(d.stream, d.e_out[1]));
      }
      TimerRec tr;
      timer_begin(f, d, tr, d.stream);
      const float* Xd = hbm_inputs(f, d, layer, hin);
      HT_TRY(launch_seg(d.stream, d, agg, Xd ? Xd : d.value.as<float>(), d_in, d_in,
                        c.csc_off.as<int64_t>(),
                        Xd ? c.csc_gid.as<int32_t>() : c.csc_slot.as<int32_t>(), c.csc_w.as<float>(),
                        c.nv, c.fw));
      timer_end(f, d, tr, 0, (double)c.ne * (8.0 + 4.0 * d_in) + (double)c.nv * (4.0 * d_in + 4.0),
                d.stream);
      HT_TRY(ev_rec(d.e_agg, d.stream));
      float* hdst = last     ? d.hL.as<float>() + d.hL_off[j] * d_out
                    : d.cache ? d.mh[layer + 1].as<float>() + c.dest_m0 * d_out
                              : d.fb[s].as<float>();
      LayerW& w = d.lw[layer];
      const int64_t* rows = c.dest_rows.as<int64_t>();
      // K4 in host-row chunks when the destination rows are copy-engine
      // runs to host memory: chunk g's h rows go to the host (K5) while
      // chunk g+1 computes; one launch when h^{l+1} is HBM (nothing streams)
      const int nck = c.dest_pos.empty() || f->hdev[layer + 1] ? 1 : kChunks;
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
    // one batch, GCN top layer: the loss also writes gz = g * (h^L > 0)
    // (the top layer's ReLU' mask, with zero pad columns) into the GZ
    // scratch the top backward reads - its separate masking pass is skipped
    const int gz_ld = f->top_gcn_prec == HT_PREC_TF32 ? pad4(d_last) : d_last;
    d.gz_loss_ld = 0;
    const bool gz_fold = count > 0 && f->n == 1 && f->top_gcn_prec >= 0 &&
                         !f->sw.no_mask_fold && d.chunks[0].nv > 0 &&
                         d.sc.bytes >= d.chunks[0].nv * (int64_t)gz_ld * 4;
    if (count > 0)
      for (int j = 0; j < f->n; ++j) {
        DevChunk& c = d.chunks[j];
        count_launch();
        ht::k_loss<<<blocks, 256, 0, d.stream>>>(
            d.hL.as<float>() + d.hL_off[j] * d_last, c.nv, d_last, d.labels.as<int64_t>(),
            d.mask.as<uint8_t>(), c.dest_rows.as<int64_t>(),
            d.cache ? d.mg[f->L].as<float>() : (float*)gout, d.cache ? c.dest_m0 : -1,
            (float)count, d.loss_part.as<double>() + (int64_t)j * blocks,
            gz_fold ? d.sc.as<float>() : nullptr, gz_ld);
        CU(cudaGetLastError());
      }
    if (gz_fold) d.gz_loss_ld = gz_ld;
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
        const bool pf = layer < (int)f->agg_deferred.size() && f->agg_deferred[layer] &&
                        precision == HT_PREC_TF32;
        if (f->agg_recompute[layer] && !pf) {
          // recompute-cache hybrid: agg^l was not kept - re-aggregate it from
          // the h^l mirror (the forward's gather, bitwise the same rows)
          const float* Xd = hbm_inputs(f, d, layer, nullptr);
          if (!Xd) return fail(HT_ESTATE, "layer %d: agg recompute needs the in-place h mirror", layer);
          if (!f->ckpt_hbm) {  // the forward's write-through may still read the scratch
            HT_TRY(ev_wait(d.stream, d.e_out[0]));
            HT_TRY(ev_wait(d.stream, d.e_out[1]));
          }
          TimerRec tr;
          timer_begin(f, d, tr, d.stream);
          HT_TRY(launch_seg(d.stream, d, const_cast<float*>(A), Xd, d_in, d_in,
                            c.csc_off.as<int64_t>(), c.csc_gid.as<int32_t>(), c.csc_w.as<float>(),
                            c.nv, c.fw));
          timer_end(f, d, tr, 0, (double)c.ne * (8.0 + 4.0 * d_in) + (double)c.nv * (4.0 * d_in + 4.0),
                    d.stream);
        }
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
      const bool narrow = !no_in && HO && d_out < d_in && !f->sw.no_narrow_bwd;
      // project-first forward (agg^l never formed): the narrow-side rows
      // A^T gz give dW = h^T (A^T gz); needs them in row order (expanded CSR)
      const bool pfl = layer < (int)f->agg_deferred.size() && f->agg_deferred[layer] &&
                       precision == HT_PREC_TF32;
      // gz = g * (h > 0) formed inside the gz . W^T GEMM (TMA loads of the g
      // and h tiles, gz written back from the masked stage) when h's rows
      // are the chunk rows; otherwise a separate masking pass
      const bool fold = precision == HT_PREC_TF32 && HO && !hrows && !narrow && !no_in &&
                        M > 0 && !f->sw.no_mask_fold && (d_out & 3) == 0 &&
                        ((uintptr_t)G & 15) == 0 && ((uintptr_t)HO & 15) == 0;
      // (top layer: the loss kernel may already have written gz)
      const bool gz_loss = layer == f->L - 1 && d.gz_loss_ld == ldz && f->n == 1;
      d.gz_loss_ld = 0;
      if (HO && M > 0 && !fold && !gz_loss) {  // gz = g * (h > 0): z need not be recomputed
        count_launch();
        ht::k_relu_mask<<<grid_for(M), kThreads, 0, d.stream>>>(GZ, ldz, G, HO, hrows, M, d_out);
        CU(cudaGetLastError());
      }
      if (precision == HT_PREC_TF32) {
        if (!HO)
          HT_TRY(ht::tc::rows<ht::tc::TC_MASK>(d.stream, true, A, d_in, M, d_in, w.Wt_hi.as<float>(),
                                               w.Wt_lo.as<float>(), d_in, d_out, GZ, ldz, G, d_out));
        if (fold)
          HT_TRY(ht::tc::rows_masked(d.stream, G, d_out, HO, d_out, GZ, ldz, M, d_out,
                                     w.Wp_hi.as<float>(), ldz, d_in, GA, d_in));
        else if (!narrow && !no_in)
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
      HT_TRY(launch_seg(d.stream, d, (narrow || pfl) ? d.tT.as<float>() : views,
                        (narrow || pfl) ? GZ : GA, (narrow || pfl) ? ldz : kw,
                        (narrow || pfl) ? ldz : kw,
                        dx ? c.bx_off.as<int64_t>() : c.csr_off.as<int64_t>(),
                        c.csr_dst.as<int32_t>(), c.csr_w.as<float>(), nseg, dx ? c.bx : c.bw));
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

