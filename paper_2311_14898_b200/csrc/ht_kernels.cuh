// Device kernels of the HongTu GCN epoch path (sm_100a).
//
//   k_copy_rows     K1/K2/K5/K6: row gathers/scatters between pinned host
//                   memory (zero-copy over PCIe), peer HBM (NVLink/UVA) and
//                   local slot buffers; 16-byte vectors when rows allow.
//   k_acc_rows      K9/K10: owner-side gradient accumulation and the flush
//                   into host gradients (read-modify-write or first store).
//   k_seg_gather    K3/K8: warp-per-segment weighted gather-sum (CSC forward
//                   aggregation, CSR transposed aggregation) with strictly
//                   sequential multiply-then-add per segment (np.add.at order).
//   k_seg_pieces / k_seg_fixup: long power-law segments split into pieces,
//                   reduced deterministically in piece order.
//   k_gemm          K4/K7 FP32 SIMT GEMM with fused epilogues (validation
//                   precision; the tcgen05 TF32 path lives in ht_tc.cuh).
//   k_loss          K11 masked softmax cross-entropy, gradient rows written
//                   straight to the host gradient array.
//   k_sgd           K12 ascending-device gradient sum + SGD step.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ht {

constexpr int kWarp = 32;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int64_t global_warp() {
  return (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ int64_t num_warps() { return ((int64_t)gridDim.x * blockDim.x) >> 5; }

// ---------------------------------------------------------------------------
// row movement
// ---------------------------------------------------------------------------

// dst row didx[r] <- src row sidx[r]; a null index means identity.  `cpr` =
// vector words per row.  Each warp owns one row at a time and issues up to
// four 32-lane vector loads before its stores.
template <typename Vec>
__global__ void __launch_bounds__(256) k_copy_rows(char* __restrict__ dst, const char* __restrict__ src,
                                                   const int64_t* __restrict__ didx,
                                                   const int64_t* __restrict__ sidx, int64_t rows,
                                                   int cpr, int64_t dstride, int64_t sstride,
                                                   int64_t dbase) {
  const int lane = lane_id();
  for (int64_t r = global_warp(); r < rows; r += num_warps()) {
    const int64_t sr = sidx ? sidx[r] : r;
    const int64_t dr = (didx ? didx[r] : r) + dbase;
    const Vec* s = reinterpret_cast<const Vec*>(src + sr * sstride);
    Vec* d = reinterpret_cast<Vec*>(dst + dr * dstride);
    for (int w = lane; w < cpr; w += 4 * kWarp) {
      Vec t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (w + u * kWarp < cpr) t[u] = s[w + u * kWarp];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (w + u * kWarp < cpr) d[w + u * kWarp] = t[u];
    }
  }
}

// dst[didx[r]] += src[sidx[r]] (or = when store_first[r] != 0); optionally
// zero the source row afterwards (the flush of devices.py:336-339).
template <typename T>
__global__ void __launch_bounds__(256) k_acc_rows(T* __restrict__ dst, T* __restrict__ src,
                                                  const int64_t* __restrict__ didx,
                                                  const int64_t* __restrict__ sidx,
                                                  const uint8_t* __restrict__ store_first,
                                                  int64_t rows, int d, int zero_src,
                                                  int64_t sbase) {
  const int lane = lane_id();
  for (int64_t r = global_warp(); r < rows; r += num_warps()) {
    const int64_t sr = (sidx ? sidx[r] : r) + sbase;
    const int64_t dr = didx ? didx[r] : r;
    T* s = src + sr * d;
    T* o = dst + dr * d;
    const bool st = store_first && store_first[r];
    for (int c = lane; c < d; c += kWarp) {
      const T v = s[c];
      o[c] = st ? v : o[c] + v;
      if (zero_src) s[c] = T(0);
    }
  }
}

// float4 rows (d % 4 == 0, 16-byte aligned rows): two rows per warp in
// flight, so every lane has four independent 16-byte loads outstanding
static __global__ void __launch_bounds__(256) k_acc_rows4(float* __restrict__ dst, float* __restrict__ src,
                                                   const int64_t* __restrict__ didx,
                                                   const int64_t* __restrict__ sidx,
                                                   const uint8_t* __restrict__ store_first,
                                                   int64_t rows, int d, int zero_src,
                                                   int64_t sbase) {
  const int lane = lane_id();
  const int d4 = d >> 2;
  const int64_t nw = num_warps();
  for (int64_t r0 = global_warp() * 2; r0 < rows; r0 += nw * 2) {
    float4* s[2];
    float4* o[2];
    bool st[2], ok[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t r = r0 + q;
      ok[q] = r < rows;
      const int64_t rr = ok[q] ? r : r0;
      s[q] = reinterpret_cast<float4*>(src + ((sidx ? sidx[rr] : rr) + sbase) * d);
      o[q] = reinterpret_cast<float4*>(dst + (didx ? didx[rr] : rr) * d);
      st[q] = store_first && store_first[rr];
    }
    for (int c = lane; c < d4; c += 2 * kWarp) {
      float4 a[2][2], b[2][2];
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int cc = c + u * kWarp;
          if (ok[q] && cc < d4) {
            a[q][u] = s[q][cc];
            b[q][u] = st[q] ? make_float4(0.f, 0.f, 0.f, 0.f) : o[q][cc];
          }
        }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int cc = c + u * kWarp;
          if (ok[q] && cc < d4) {
            float4 v = a[q][u];
            if (!st[q]) v = make_float4(b[q][u].x + v.x, b[q][u].y + v.y, b[q][u].z + v.z,
                                        b[q][u].w + v.w);
            o[q][cc] = v;
            if (zero_src) s[q][cc] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
    }
  }
}

// ---------------------------------------------------------------------------
// segment gather-sum: out[seg] = sum_{e in [lo, hi)} w[e] * X[idx[e]]
// sequential in e, product rounded before the add (no FMA contraction)
// ---------------------------------------------------------------------------

// U edges' rows are requested before any is accumulated; the next 32
// edge indices/weights are prefetched while the current ones are summed.
template <int NV, int U = 8>
__device__ __forceinline__ void seg_sum_v4(float4 (&acc)[NV], const float* __restrict__ X,
                                           int64_t ldx, int d4, const int32_t* __restrict__ idx,
                                           const float* __restrict__ w, int64_t e0, int64_t e1,
                                           int lane) {
  int64_t base = e0;
  int cnt = (int)((e1 - base) < (int64_t)kWarp ? (e1 - base) : (int64_t)kWarp);
  int my_i = lane < cnt ? __ldg(idx + base + lane) : 0;
  float my_w = lane < cnt ? __ldg(w + base + lane) : 0.f;
  while (cnt > 0) {
    const int64_t nb = base + kWarp;
    const int ncnt = nb < e1 ? (int)((e1 - nb) < (int64_t)kWarp ? (e1 - nb) : (int64_t)kWarp) : 0;
    const int nx_i = lane < ncnt ? __ldg(idx + nb + lane) : 0;
    const float nx_w = lane < ncnt ? __ldg(w + nb + lane) : 0.f;
    int k = 0;
    for (; k + U <= cnt; k += U) {
      float4 x[U][NV];
      float ww[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = __shfl_sync(0xffffffffu, my_i, k + u);
        ww[u] = __shfl_sync(0xffffffffu, my_w, k + u);
        const float4* row = reinterpret_cast<const float4*>(X + (int64_t)s * ldx);
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          const int c = lane + t * kWarp;
          x[u][t] = c < d4 ? __ldg(row + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          acc[t].x = __fadd_rn(acc[t].x, __fmul_rn(ww[u], x[u][t].x));
          acc[t].y = __fadd_rn(acc[t].y, __fmul_rn(ww[u], x[u][t].y));
          acc[t].z = __fadd_rn(acc[t].z, __fmul_rn(ww[u], x[u][t].z));
          acc[t].w = __fadd_rn(acc[t].w, __fmul_rn(ww[u], x[u][t].w));
        }
    }
    for (; k < cnt; ++k) {
      const int s = __shfl_sync(0xffffffffu, my_i, k);
      const float wk = __shfl_sync(0xffffffffu, my_w, k);
      const float4* row = reinterpret_cast<const float4*>(X + (int64_t)s * ldx);
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const int c = lane + t * kWarp;
        if (c < d4) {
          const float4 x = __ldg(row + c);
          acc[t].x = __fadd_rn(acc[t].x, __fmul_rn(wk, x.x));
          acc[t].y = __fadd_rn(acc[t].y, __fmul_rn(wk, x.y));
          acc[t].z = __fadd_rn(acc[t].z, __fmul_rn(wk, x.z));
          acc[t].w = __fadd_rn(acc[t].w, __fmul_rn(wk, x.w));
        }
      }
    }
    base = nb;
    cnt = ncnt;
    my_i = nx_i;
    my_w = nx_w;
  }
}

template <int NS>
__device__ __forceinline__ void seg_sum_s(float (&acc)[NS], const float* __restrict__ X, int64_t ldx,
                                          int d, const int32_t* __restrict__ idx,
                                          const float* __restrict__ w, int64_t e0, int64_t e1,
                                          int lane) {
  for (int64_t base = e0; base < e1; base += kWarp) {
    const int cnt = (int)((e1 - base) < (int64_t)kWarp ? (e1 - base) : (int64_t)kWarp);
    const int my_i = lane < cnt ? idx[base + lane] : 0;
    const float my_w = lane < cnt ? w[base + lane] : 0.f;
    for (int k = 0; k < cnt; ++k) {
      const int s = __shfl_sync(0xffffffffu, my_i, k);
      const float wk = __shfl_sync(0xffffffffu, my_w, k);
      const float* row = X + (int64_t)s * ldx;
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        const int c = lane + t * kWarp;
        if (c < d) acc[t] = __fadd_rn(acc[t], __fmul_rn(wk, __ldg(row + c)));
      }
    }
  }
}

// One warp per segment; segments longer than `split` are skipped here and
// handled by k_seg_pieces.  out row stride = d (dense), optional row map
// `out_row` (null = identity).
template <int NV, int U = 4, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_seg_gather_v4(float* __restrict__ out,
                                                       const float* __restrict__ X, int64_t ldx,
                                                       int d, const int64_t* __restrict__ off,
                                                       const int32_t* __restrict__ idx,
                                                       const float* __restrict__ w, int64_t nseg,
                                                       int64_t split) {
  const int lane = lane_id();
  const int d4 = d >> 2;
  for (int64_t sg = global_warp(); sg < nseg; sg += num_warps()) {
    const int64_t e0 = off[sg], e1 = off[sg + 1];
    if (e1 - e0 > split) continue;
    float4 acc[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    seg_sum_v4<NV, U>(acc, X, ldx, d4, idx, w, e0, e1, lane);
    float4* o = reinterpret_cast<float4*>(out + sg * (int64_t)d);
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const int c = lane + t * kWarp;
      if (c < d4) o[c] = acc[t];
    }
  }
}

template <int NS>
__global__ void __launch_bounds__(256) k_seg_gather_s(float* __restrict__ out,
                                                      const float* __restrict__ X, int64_t ldx,
                                                      int d, const int64_t* __restrict__ off,
                                                      const int32_t* __restrict__ idx,
                                                      const float* __restrict__ w, int64_t nseg,
                                                      int64_t split) {
  const int lane = lane_id();
  for (int64_t sg = global_warp(); sg < nseg; sg += num_warps()) {
    const int64_t e0 = off[sg], e1 = off[sg + 1];
    if (e1 - e0 > split) continue;
    float acc[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) acc[t] = 0.f;
    seg_sum_s<NS>(acc, X, ldx, d, idx, w, e0, e1, lane);
    float* o = out + sg * (int64_t)d;
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const int c = lane + t * kWarp;
      if (c < d) o[c] = acc[t];
    }
  }
}

// Narrow rows (d4 = d/4 <= G float4 words): a warp is split into 32/G
// sub-groups of G lanes and each sub-group sums its own segment (or piece),
// sequentially in edge order as above - so one load instruction moves
// 32/G rows and a 48-float row no longer leaves 20 of 32 lanes idle.
template <int G, int U>
__device__ __forceinline__ void seg_sum_sub(float4& acc, const float* __restrict__ X, int64_t ldx,
                                            int d4, const int32_t* __restrict__ idx,
                                            const float* __restrict__ w, int64_t e0, int64_t e1,
                                            int sl) {
  // sub-groups of one warp run different segment lengths: every lane keeps
  // executing the loop until the longest segment of the warp is done
  int64_t len = e1 - e0;
  int64_t lmax = len;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t t = __shfl_xor_sync(0xffffffffu, lmax, o);
    lmax = t > lmax ? t : lmax;
  }
  for (int64_t b = 0; b < lmax; b += G) {
    const int cnt = (int)((len - b) < (int64_t)G ? ((len - b) > 0 ? (len - b) : 0) : (int64_t)G);
    const int my_i = sl < cnt ? __ldg(idx + e0 + b + sl) : 0;
    const float my_w = sl < cnt ? __ldg(w + e0 + b + sl) : 0.f;
    for (int k = 0; k < G; k += U) {
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = __shfl_sync(0xffffffffu, my_i, k + u, G);
        const float4* row = reinterpret_cast<const float4*>(X + (int64_t)s * ldx);
        x[u] = (k + u < cnt && sl < d4) ? __ldg(row + sl) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float wk = __shfl_sync(0xffffffffu, my_w, k + u, G);
        if (k + u < cnt) {
          acc.x = __fadd_rn(acc.x, __fmul_rn(wk, x[u].x));
          acc.y = __fadd_rn(acc.y, __fmul_rn(wk, x[u].y));
          acc.z = __fadd_rn(acc.z, __fmul_rn(wk, x[u].z));
          acc.w = __fadd_rn(acc.w, __fmul_rn(wk, x[u].w));
        }
      }
    }
  }
}

template <int G, int U = 8, int MINB = 4>
__global__ void __launch_bounds__(256, MINB) k_seg_gather_sub(float* __restrict__ out,
                                                              const float* __restrict__ X,
                                                              int64_t ldx, int d,
                                                              const int64_t* __restrict__ off,
                                                              const int32_t* __restrict__ idx,
                                                              const float* __restrict__ w,
                                                              int64_t nseg, int64_t split) {
  constexpr int S = 32 / G;  // segments per warp
  const int lane = lane_id(), sl = lane % G, sub = lane / G;
  const int d4 = d >> 2;
  const int64_t ngrp = (nseg + S - 1) / S;
  for (int64_t gi = global_warp(); gi < ngrp; gi += num_warps()) {
    const int64_t sg = gi * S + sub;
    int64_t e0 = 0, e1 = 0;
    const bool mine = sg < nseg;
    if (mine) {
      e0 = off[sg];
      e1 = off[sg + 1];
    }
    const bool skip = !mine || e1 - e0 > split;  // long: k_seg_pieces
    if (skip) e1 = e0;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    seg_sum_sub<G, U>(acc, X, ldx, d4, idx, w, e0, e1, sl);
    if (!skip && sl < d4) reinterpret_cast<float4*>(out + sg * (int64_t)d)[sl] = acc;
  }
}

template <int G, int U = 8>
__global__ void __launch_bounds__(256) k_seg_pieces_sub(float* __restrict__ partial,
                                                        const float* __restrict__ X, int64_t ldx,
                                                        int d, const int64_t* __restrict__ lo,
                                                        const int64_t* __restrict__ hi,
                                                        const int32_t* __restrict__ idx,
                                                        const float* __restrict__ w,
                                                        int64_t npieces) {
  constexpr int S = 32 / G;
  const int lane = lane_id(), sl = lane % G, sub = lane / G;
  const int d4 = d >> 2;
  const int64_t ngrp = (npieces + S - 1) / S;
  for (int64_t gi = global_warp(); gi < ngrp; gi += num_warps()) {
    const int64_t p = gi * S + sub;
    const bool mine = p < npieces;
    const int64_t e0 = mine ? lo[p] : 0, e1 = mine ? hi[p] : 0;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    seg_sum_sub<G, U>(acc, X, ldx, d4, idx, w, e0, e1, sl);
    if (mine && sl < d4) reinterpret_cast<float4*>(partial + p * (int64_t)d)[sl] = acc;
  }
}

// Pieces of long segments: piece p sums edges [lo[p], hi[p]) into
// partial row p.
template <int NV>
__global__ void __launch_bounds__(256) k_seg_pieces_v4(float* __restrict__ partial,
                                                       const float* __restrict__ X, int64_t ldx,
                                                       int d, const int64_t* __restrict__ lo,
                                                       const int64_t* __restrict__ hi,
                                                       const int32_t* __restrict__ idx,
                                                       const float* __restrict__ w,
                                                       int64_t npieces) {
  const int lane = lane_id();
  const int d4 = d >> 2;
  for (int64_t p = global_warp(); p < npieces; p += num_warps()) {
    float4 acc[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    seg_sum_v4<NV, (NV <= 2 ? 8 : 4)>(acc, X, ldx, d4, idx, w, lo[p], hi[p], lane);
    float4* o = reinterpret_cast<float4*>(partial + p * (int64_t)d);
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const int c = lane + t * kWarp;
      if (c < d4) o[c] = acc[t];
    }
  }
}

template <int NS>
__global__ void __launch_bounds__(256) k_seg_pieces_s(float* __restrict__ partial,
                                                      const float* __restrict__ X, int64_t ldx,
                                                      int d, const int64_t* __restrict__ lo,
                                                      const int64_t* __restrict__ hi,
                                                      const int32_t* __restrict__ idx,
                                                      const float* __restrict__ w,
                                                      int64_t npieces) {
  const int lane = lane_id();
  for (int64_t p = global_warp(); p < npieces; p += num_warps()) {
    float acc[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) acc[t] = 0.f;
    seg_sum_s<NS>(acc, X, ldx, d, idx, w, lo[p], hi[p], lane);
    float* o = partial + p * (int64_t)d;
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const int c = lane + t * kWarp;
      if (c < d) o[c] = acc[t];
    }
  }
}

// ---------------------------------------------------------------------------
// Work-list segment reduction: one launch per aggregation.  Work units
// [0, npu) are the pieces of the long segments (the heaviest items first),
// then batches of short segments; a warp takes the next unit from a device
// counter when it is free, so the pieces no longer form a serial tail
// launch.  A piece writes its partial row, and the piece of a long segment
// that finishes last (atomic ticket) sums the segment's partials in piece
// order - the fixed order of k_seg_fixup, so the results are bitwise those
// of the three-launch sequence.
// ---------------------------------------------------------------------------
struct SegWork {
  const int64_t* off;
  const int32_t* idx;
  const float* w;
  int64_t nseg, split;
  const int64_t *lo, *hi;  // pieces
  const int32_t* pf;       // fixup of each piece
  int64_t np;
  const int64_t *fseg, *ffirst, *fcnt;  // fixups
  unsigned* counter;                    // zeroed before the launch
  int* tickets;                         // [nf], zeroed before the launch
  float* partial;
};

// partials first .. first + cnt - 1 of one fixup, summed in piece order
// (L2 reads: they were written by other SMs), float4 column c
__device__ __forceinline__ float4 sum_partials(const float* __restrict__ partial, int64_t first,
                                               int64_t cnt, int d, int c) {
  const float4* p = reinterpret_cast<const float4*>(partial + first * (int64_t)d) + c;
  const int64_t d4 = d >> 2;
  float4 s = __ldcg(p);
  for (int64_t q = 1; q < cnt; ++q) {
    const float4 v = __ldcg(p + q * d4);
    s.x = __fadd_rn(s.x, v.x);
    s.y = __fadd_rn(s.y, v.y);
    s.z = __fadd_rn(s.z, v.z);
    s.w = __fadd_rn(s.w, v.w);
  }
  return s;
}

template <int NV, int US, int UP, int B, int MINB>
__global__ void __launch_bounds__(256, MINB) k_seg_work_v4(float* __restrict__ out,
                                                           const float* __restrict__ X,
                                                           int64_t ldx, int d, SegWork wk) {
  const int lane = lane_id();
  const int d4 = d >> 2;
  const int64_t nunits = wk.np + (wk.nseg + B - 1) / B;
  for (;;) {
    unsigned u = 0;
    if (lane == 0) u = atomicAdd(wk.counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if ((int64_t)u >= nunits) break;
    float4 acc[NV];
    if ((int64_t)u < wk.np) {  // a piece of a long segment
#pragma unroll
      for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      seg_sum_v4<NV, UP>(acc, X, ldx, d4, wk.idx, wk.w, wk.lo[u], wk.hi[u], lane);
      float4* prow = reinterpret_cast<float4*>(wk.partial + (int64_t)u * d);
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const int c = lane + t * kWarp;
        if (c < d4) prow[c] = acc[t];
      }
      __threadfence();  // this lane's partial stores, then the warp's ticket
      __syncwarp();
      const int f = wk.pf[u];
      int last = 0;
      if (lane == 0) last = atomicAdd(wk.tickets + f, 1) == (int)wk.fcnt[f] - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {  // every piece of the segment is written: fixed-order sum
        __threadfence();
        float4* o = reinterpret_cast<float4*>(out + wk.fseg[f] * (int64_t)d);
        for (int c = lane; c < d4; c += kWarp) o[c] = sum_partials(wk.partial, wk.ffirst[f], wk.fcnt[f], d, c);
      }
      continue;
    }
    const int64_t s0 = ((int64_t)u - wk.np) * B;
    const int64_t s1 = s0 + B < wk.nseg ? s0 + B : wk.nseg;
    for (int64_t sg = s0; sg < s1; ++sg) {
      const int64_t e0 = wk.off[sg], e1 = wk.off[sg + 1];
      if (e1 - e0 > wk.split) continue;  // a long segment: its pieces
#pragma unroll
      for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      seg_sum_v4<NV, US>(acc, X, ldx, d4, wk.idx, wk.w, e0, e1, lane);
      float4* o = reinterpret_cast<float4*>(out + sg * (int64_t)d);
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const int c = lane + t * kWarp;
        if (c < d4) o[c] = acc[t];
      }
    }
  }
}

// narrow rows (d4 <= G): 32/G sub-groups per warp, each its own piece or
// segment, summed sequentially in edge order (seg_sum_sub)
template <int G, int U, int B, int MINB>
__global__ void __launch_bounds__(256, MINB) k_seg_work_sub(float* __restrict__ out,
                                                            const float* __restrict__ X,
                                                            int64_t ldx, int d, SegWork wk) {
  constexpr int S = 32 / G;
  const int lane = lane_id(), sl = lane % G, sub = lane / G;
  const int d4 = d >> 2;
  const int64_t npu = (wk.np + S - 1) / S;
  const int64_t nunits = npu + (wk.nseg + S * B - 1) / (S * B);
  for (;;) {
    unsigned u = 0;
    if (lane == 0) u = atomicAdd(wk.counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if ((int64_t)u >= nunits) break;
    if ((int64_t)u < npu) {  // S pieces, one per sub-group
      const int64_t p = (int64_t)u * S + sub;
      const bool mine = p < wk.np;
      const int64_t e0 = mine ? wk.lo[p] : 0, e1 = mine ? wk.hi[p] : 0;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      seg_sum_sub<G, U>(acc, X, ldx, d4, wk.idx, wk.w, e0, e1, sl);
      if (mine && sl < d4) reinterpret_cast<float4*>(wk.partial + p * (int64_t)d)[sl] = acc;
      __threadfence();  // this lane's partial stores, then the warp's ticket
      __syncwarp();
      const int f = mine ? wk.pf[p] : 0;
      int last = 0;
      if (mine && sl == 0) last = atomicAdd(wk.tickets + f, 1) == (int)wk.fcnt[f] - 1;
      last = __shfl_sync(0xffffffffu, last, sub * G);
      if (mine && last) {
        __threadfence();
        if (sl < d4)
          reinterpret_cast<float4*>(out + wk.fseg[f] * (int64_t)d)[sl] =
              sum_partials(wk.partial, wk.ffirst[f], wk.fcnt[f], d, sl);
      }
      continue;
    }
    const int64_t s0 = ((int64_t)u - npu) * (S * B);
    for (int b = 0; b < B; ++b) {
      const int64_t sg = s0 + (int64_t)b * S + sub;
      if (s0 + (int64_t)b * S >= wk.nseg) break;  // warp-uniform
      int64_t e0 = 0, e1 = 0;
      const bool inr = sg < wk.nseg;
      if (inr) {
        e0 = wk.off[sg];
        e1 = wk.off[sg + 1];
      }
      const bool skip = !inr || e1 - e0 > wk.split;  // long: its pieces
      if (skip) e1 = e0;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      seg_sum_sub<G, U>(acc, X, ldx, d4, wk.idx, wk.w, e0, e1, sl);
      if (!skip && sl < d4) reinterpret_cast<float4*>(out + sg * (int64_t)d)[sl] = acc;
    }
  }
}

// out[seg[f]] = ((partial[first] + partial[first+1]) + ...) in piece order.
static __global__ void __launch_bounds__(256) k_seg_fixup(float* __restrict__ out,
                                                   const float* __restrict__ partial, int d,
                                                   const int64_t* __restrict__ seg,
                                                   const int64_t* __restrict__ first,
                                                   const int64_t* __restrict__ count, int64_t nfix) {
  const int lane = lane_id();
  for (int64_t f = global_warp(); f < nfix; f += num_warps()) {
    const float* p = partial + first[f] * (int64_t)d;
    float* o = out + seg[f] * (int64_t)d;
    for (int c = lane; c < d; c += kWarp) {
      float s = p[c];
      for (int64_t q = 1; q < count[f]; ++q) s = __fadd_rn(s, p[q * (int64_t)d + c]);
      o[c] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// FP32 SIMT GEMM  C = A(MxK) * B(KxN), A(m,k) = TA ? A[k*lda+m] : A[m*lda+k],
// B(k,n) = TB ? B[n*ldb+k] : B[k*ldb+n].  64x64x16 tiles, 4x4 per thread.
// EPI: 0 store, 1 relu, 2 mask: C = (acc > 0) ? G[m*ldg+n] : 0.
// Split-K over blockIdx.z writes slab z at C + z*M*ldc.
// ---------------------------------------------------------------------------
enum { EPI_STORE = 0, EPI_RELU = 1, EPI_MASK = 2 };

template <bool TA, bool TB, int EPI>
__global__ void __launch_bounds__(256) k_gemm(const float* __restrict__ A, int64_t lda,
                                              const float* __restrict__ B, int64_t ldb,
                                              float* __restrict__ C, int64_t ldc,
                                              const float* __restrict__ G, int64_t ldg, int64_t M,
                                              int64_t N, int64_t K, int64_t k_per_split) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = threadIdx.x + q * 256;  // 0..1023 over a BK x BM tile
      int kk, mm;
      if (TA) { mm = t % BM; kk = t / BM; } else { kk = t % BK; mm = t / BK; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < kend) v = TA ? A[gk * lda + gm] : A[gm * lda + gk];
      As[kk][mm] = v;
      int kb, nb;
      if (TB) { kb = t % BK; nb = t / BK; } else { nb = t % BN; kb = t / BN; }
      const int64_t gn = n0 + nb, gkb = k0 + kb;
      float u = 0.f;
      if (gn < N && gkb < kend) u = TB ? B[gn * ldb + gkb] : B[gkb * ldb + gn];
      Bs[kb][nb] = u;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* Cz = C + (int64_t)blockIdx.z * M * ldc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (EPI == EPI_RELU) v = v > 0.f ? v : 0.f;
      if (EPI == EPI_MASK) v = v > 0.f ? G[gm * ldg + gn] : 0.f;
      Cz[gm * ldc + gn] = v;
    }
  }
}

// acc[e] = acc[e] + ((slab0[e] + slab1[e]) + ...) over `splits` slabs.
static __global__ void k_reduce_splits(float* __restrict__ acc, const float* __restrict__ slabs,
                                int64_t n, int splits) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float s = slabs[e];
    for (int z = 1; z < splits; ++z) s = __fadd_rn(s, slabs[(int64_t)z * n + e]);
    acc[e] = __fadd_rn(acc[e], s);
  }
}

// ReLU' from the stored layer output: gz[r] = g[r] * (h[row(r)] > 0).  h =
// max(z, 0) was produced from the same z by the forward, so (h > 0) == (z >
// 0) bitwise: the backward needs no recompute of z when h is in HBM.
static __global__ void __launch_bounds__(256) k_relu_mask(float* __restrict__ gz, int64_t ldz,
                                                   const float* __restrict__ g,
                                                   const float* __restrict__ h,
                                                   const int64_t* __restrict__ hrows,
                                                   int64_t rows, int d) {
  const int lane = lane_id();
  for (int64_t r = global_warp(); r < rows; r += num_warps()) {
    const float* hr = h + (hrows ? hrows[r] : r) * (int64_t)d;
    const float* gr = g + r * (int64_t)d;
    float* o = gz + r * ldz;
    for (int c = lane; c < d; c += kWarp) o[c] = __ldg(hr + c) > 0.f ? __ldg(gr + c) : 0.f;
    for (int c = d + lane; c < ldz; c += kWarp) o[c] = 0.f;  // zero pad columns
  }
}

// ---------------------------------------------------------------------------
// out[r][c] = max(in[r][c], 0) for c < d (row strides ldo / ldi floats)
static __global__ void __launch_bounds__(256) k_relu_rows(float* __restrict__ out, int64_t ldo,
                                                   const float* __restrict__ in, int64_t ldi,
                                                   int64_t rows, int d) {
  const int64_t n = rows * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int c = (int)(e - r * d);
    out[r * ldo + c] = fmaxf(in[r * ldi + c], 0.f);
  }
}

// K11 loss: rows of H (ld = d); labels/mask aligned with rows; gradient rows
// written to out (host or device) at out_rows[r] (stride d), or at
// out_base + r when out_base >= 0.  One warp per
// row; per-block partial loss sums in double, fixed order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void loss_row(const float* __restrict__ z, float* __restrict__ g, int d,
                                         int64_t y, float count, int lane, double& my) {
  float mx = -INFINITY;
  for (int c = lane; c < d; c += kWarp) mx = fmaxf(mx, z[c]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = 0.f;
  for (int c = lane; c < d; c += kWarp) s += expf(z[c] - mx);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  for (int c = lane; c < d; c += kWarp) {
    const float p = __fdiv_rn(expf(z[c] - mx), s);
    if (c == y) my += -(double)logf(p);
    g[c] = __fdiv_rn(c == y ? __fsub_rn(p, 1.f) : p, count);
  }
}

// Rows are taken 32 at a time per warp: their vertex ids, mask bits and
// labels are loaded lane-parallel (one latency per 32 rows); rows of width
// <= 64 are held in registers and the next row's values are requested
// before the current one is reduced.
static __global__ void __launch_bounds__(256) k_loss(const float* __restrict__ H, int64_t rows, int d,
                                              const int64_t* __restrict__ labels,
                                              const uint8_t* __restrict__ mask,
                                              const int64_t* __restrict__ out_rows,
                                              float* __restrict__ out, int64_t out_base,
                                              float count, double* __restrict__ block_loss,
                                              float* __restrict__ gz = nullptr, int ldz = 0) {
  __shared__ double wsum[8];
  const int lane = lane_id(), wib = threadIdx.x >> 5;
  double my = 0.0;
  const int64_t nblk = (rows + kWarp - 1) / kWarp;
  for (int64_t blk = blockIdx.x * 8 + wib; blk < nblk; blk += (int64_t)gridDim.x * 8) {
    const int64_t r0 = blk * kWarp;
    const int nr = (int)((rows - r0) < (int64_t)kWarp ? (rows - r0) : (int64_t)kWarp);
    const int64_t my_v = lane < nr ? out_rows[r0 + lane] : 0;
    const int my_m = lane < nr ? (int)mask[my_v] : 0;
    const int my_y = lane < nr && my_m ? (int)labels[my_v] : 0;
    const bool reg = d <= 2 * kWarp;
    float z0 = 0.f, z1 = 0.f;
    if (reg && nr > 0) {
      z0 = lane < d ? H[r0 * d + lane] : -INFINITY;
      z1 = lane + kWarp < d ? H[r0 * d + lane + kWarp] : -INFINITY;
    }
    for (int j = 0; j < nr; ++j) {
      const int64_t r = r0 + j;
      const int64_t v = __shfl_sync(0xffffffffu, my_v, j);
      const int m = __shfl_sync(0xffffffffu, my_m, j);
      const int y = __shfl_sync(0xffffffffu, my_y, j);
      // gradient row: host row v, or mirror row out_base + r (HBM owner cache)
      float* g = out + (out_base >= 0 ? out_base + r : v) * d;
      if (!reg) {
        if (!m) {  // rows off the mask get a zero gradient (engine.py:305, 319)
          for (int c = lane; c < d; c += kWarp) g[c] = 0.f;
        } else {
          loss_row(H + r * d, g, d, y, count, lane, my);
        }
        if (gz)  // gz = g * (h > 0), pad columns zero (each lane rereads its own g)
          for (int c = lane; c < ldz; c += kWarp)
            gz[r * ldz + c] = (m && c < d && H[r * d + c] > 0.f) ? g[c] : 0.f;
        continue;
      }
      const float c0 = z0, c1 = z1;
      if (j + 1 < nr) {  // next row in flight while this one is reduced
        z0 = lane < d ? H[(r + 1) * d + lane] : -INFINITY;
        z1 = lane + kWarp < d ? H[(r + 1) * d + lane + kWarp] : -INFINITY;
      }
      if (!m) {
        if (lane < d) g[lane] = 0.f;
        if (lane + kWarp < d) g[lane + kWarp] = 0.f;
        if (gz) {
          if (lane < ldz) gz[r * ldz + lane] = 0.f;
          if (lane + kWarp < ldz) gz[r * ldz + lane + kWarp] = 0.f;
        }
        continue;
      }
      float mx = fmaxf(c0, c1);
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float e0 = lane < d ? expf(c0 - mx) : 0.f;
      const float e1 = lane + kWarp < d ? expf(c1 - mx) : 0.f;
      float sum = e0 + e1;
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      float g0 = 0.f, g1 = 0.f;
      if (lane < d) {
        const float p = __fdiv_rn(e0, sum);
        if (lane == y) my += -(double)logf(p);
        g0 = __fdiv_rn(lane == y ? __fsub_rn(p, 1.f) : p, count);
        g[lane] = g0;
      }
      if (lane + kWarp < d) {
        const float p = __fdiv_rn(e1, sum);
        if (lane + kWarp == y) my += -(double)logf(p);
        g1 = __fdiv_rn(lane + kWarp == y ? __fsub_rn(p, 1.f) : p, count);
        g[lane + kWarp] = g1;
      }
      if (gz) {  // gz = g * (h > 0) (c0 / c1 = -inf past d), pad columns zero
        if (lane < ldz) gz[r * ldz + lane] = c0 > 0.f ? g0 : 0.f;
        if (lane + kWarp < ldz) gz[r * ldz + lane + kWarp] = c1 > 0.f ? g1 : 0.f;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) my += __shfl_xor_sync(0xffffffffu, my, o);
  if (lane == 0) wsum[wib] = my;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t += wsum[q];
    block_loss[blockIdx.x] = t;
  }
}

// Cross-process barrier (rank mode): make this rank's prior writes visible
// system-wide, publish `seq`, then spin (acquire) until every rank's
// counter reached it.  Traps after 60 s so a dead peer fails loudly
// instead of hanging the GPU.
static __global__ void k_xbarrier(uint32_t* self, uint32_t* const* peers, int m, uint32_t seq) {
  __threadfence_system();
  __syncwarp();
  if (threadIdx.x == 0)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(self), "r"(seq) : "memory");
  if ((int)threadIdx.x < m) {
    const uint32_t* p = peers[threadIdx.x];
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      if ((int32_t)(v - seq) >= 0) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 60000000000ull) __trap();
      __nanosleep(256);
    }
  }
  __syncwarp();
  __threadfence_system();
}

// deterministic operand pattern in [-1, 1) for the measurement entries
static __global__ void k_fill_pattern(float* __restrict__ x, int64_t n, uint32_t seed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)e * 2654435761u ^ (seed * 0x9E3779B9u);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    x[e] = (float)(h & 0xFFFFFF) * (2.0f / 16777216.0f) - 1.0f;
  }
}

// K12: total = ((0 + g_0) + g_1) + ...; W = W - lr * total (separate roundings)
static __global__ void k_sgd(float* __restrict__ W, float* __restrict__ total_out,
                      const float* const* __restrict__ grads, int ndev, int64_t n, float lr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    float t = 0.f;
    for (int i = 0; i < ndev; ++i) t = __fadd_rn(t, grads[i][e]);
    if (total_out) total_out[e] = t;
    W[e] = __fsub_rn(W[e], __fmul_rn(lr, t));
  }
}

}  // namespace ht
