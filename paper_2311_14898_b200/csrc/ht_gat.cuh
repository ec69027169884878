// GAT layer kernels (src/engine.py:196-289) for sm_100a.
//
// Per chunk (i, j), with q = h_nbr.W (|N_ij| rows), p = h_dst.W (|V_ij|
// rows), both produced by the tcgen05 GEMM:
//
//   k_rowdot      el_src[u] = q_u . a_src (one warp per row)
//   k_gat_dst     one warp per destination v over its CSC in-edges:
//                 t_e = p_v.a_dst + el_src[u], LeakyReLU, max-subtracted
//                 softmax (lane-parallel over edges), s_v = sum_e alpha_e q_u
//                 (sequential multiply-then-add in CSC order, the np.add.at
//                 of src/engine.py:236), h_v = ReLU(s_v).
//                 BWD (recompute backward, src/engine.py:240-289): also
//                 gs = g_v * (s_v > 0), per-edge g_alpha = gs . q_u,
//                 g_t = alpha (g_alpha - sum alpha g_alpha) * LeakyReLU'(t),
//                 writes gs rows, alpha / g_t per edge (CSC order), the
//                 segment sum of g_t and the rank-1 gp_v = seg_gt_v * a_dst.
//                 alpha / g_t are stored interleaved per edge ({alpha, g_t}
//                 8-byte records in CSC order: AL = record base, GT = AL + 1).
//   k_gat_src     BWD, one warp per source u over its CSR out-edges:
//                 gq_u = sum_e (alpha_e gs_{dst e} + g_t_e a_src) in edge
//                 order (the np.add.at of src/engine.py:275/280), and
//                 gts_u = sum_e g_t_e.  Power-law hubs (> 1024 out-edges)
//                 are split into pieces (k_gat_src_pieces) summed in piece
//                 order (k_gat_src_fixup), as in the GCN transposed path.
//   k_wcolsum / k_colsum_reduce
//                 out[c] += sum_r w_r X[r][c] (attention-vector gradients),
//                 block partials reduced in a fixed order (deterministic).
//
// Feature widths are multiples of 4 (float4 rows) and at most 512.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "ht_kernels.cuh"  // sum_partials

namespace ht {
namespace gat {

constexpr int kW = 32;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int NV>
__device__ __forceinline__ void load4(float4 (&r)[NV], const float* __restrict__ row, int d4,
                                      int lane) {
  const float4* p = reinterpret_cast<const float4*>(row);
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = lane + t * kW;
    r[t] = c < d4 ? __ldg(p + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <int NV>
__device__ __forceinline__ void store4(float* __restrict__ row, const float4 (&r)[NV], int d4,
                                       int lane) {
  float4* p = reinterpret_cast<float4*>(row);
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    const int c = lane + t * kW;
    if (c < d4) p[c] = r[t];
  }
}

template <int NV>
__device__ __forceinline__ float dot4(const float4 (&a)[NV], const float4 (&b)[NV]) {
  float s = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    s = fmaf(a[t].x, b[t].x, s);
    s = fmaf(a[t].y, b[t].y, s);
    s = fmaf(a[t].z, b[t].z, s);
    s = fmaf(a[t].w, b[t].w, s);
  }
  return s;
}

// acc += a * x, product rounded before the add (np.add.at semantics)
__device__ __forceinline__ void axpy_rn(float4& acc, float a, const float4& x) {
  acc.x = __fadd_rn(acc.x, __fmul_rn(a, x.x));
  acc.y = __fadd_rn(acc.y, __fmul_rn(a, x.y));
  acc.z = __fadd_rn(acc.z, __fmul_rn(a, x.z));
  acc.w = __fadd_rn(acc.w, __fmul_rn(a, x.w));
}

__device__ __forceinline__ float leaky(float t, float slope) { return t > 0.f ? t : slope * t; }

// acc += (a x + g b), the per-edge value rounded before the add
__device__ __forceinline__ void edge_add(float4& acc, float a, const float4& x, float g,
                                         const float4& b) {
  acc.x = __fadd_rn(acc.x, __fadd_rn(__fmul_rn(a, x.x), __fmul_rn(g, b.x)));
  acc.y = __fadd_rn(acc.y, __fadd_rn(__fmul_rn(a, x.y), __fmul_rn(g, b.y)));
  acc.z = __fadd_rn(acc.z, __fadd_rn(__fmul_rn(a, x.z), __fmul_rn(g, b.z)));
  acc.w = __fadd_rn(acc.w, __fadd_rn(__fmul_rn(a, x.w), __fmul_rn(g, b.w)));
}

// out[r] = X[r] . a   (one warp per row)
template <int NV>
__global__ void __launch_bounds__(256) k_rowdot(float* __restrict__ out, const float* __restrict__ X,
                                                int64_t ldx, const float* __restrict__ a, int d,
                                                int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  float4 av[NV];
  load4<NV>(av, a, d4, lane);
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    float4 x[NV];
    load4<NV>(x, X + r * ldx, d4, lane);
    const float s = warp_sum(dot4<NV>(x, av));
    if (lane == 0) out[r] = s;
  }
}

// One warp per destination segment of a chunk's CSC view.  `idx` are
// chunk-local source ids (rows of Q / el_src), rows are d floats wide.
// DU source rows in flight per warp in the row passes.
#ifndef HT_GAT_DU
#define HT_GAT_DU 8
#endif
constexpr int DU = HT_GAT_DU;
#ifndef HT_GAT_DB
#define HT_GAT_DB 8
#endif
constexpr int kDstBatch = HT_GAT_DB;  // destinations per work unit
// Minimum resident 256-thread CTAs per SM asked of ptxas for the one-
// float4-per-lane (d <= 128) row passes; the grids follow the occupancy
// they get.  Both passes wait on random row fetches (long-scoreboard
// stalls 12-17 per issue at 40 / 64 registers): forward at 8 CTAs (32
// registers, 32 B of spill), S1 at 5 (48 registers) measured 59.2 -> 51.3
// ms per cfg-2 GAT value epoch on one box (forward edge pass 13.6 -> 8.4
// ms, backward 36.8 -> 30.9; profiles/r3_gat_occupancy_ab.txt).  Wider
// rows (NV > 1) and the fused backward keep the compiler's choice (they
// would spill hundreds of bytes).
#ifndef HT_GAT_DST_MINB
#define HT_GAT_DST_MINB 8
#endif
#ifndef HT_GAT_S1_MINB
#define HT_GAT_S1_MINB 5
#endif
#ifndef HT_GAT_AB_MINB  // split-backward destination passes A and B: 8 CTAs/SM (32 registers)
// took the GAT edge backward 32.1 -> 31.0 ms (profiles/r3_gat_ab8_ab.txt)
#define HT_GAT_AB_MINB 8
#endif
template <int NV, bool BWD>
__global__ void __launch_bounds__(256, (NV == 1 && !BWD) ? HT_GAT_DST_MINB : 1) k_gat_dst(
    const int64_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t nseg,
    const float* __restrict__ Q, const float* __restrict__ P, const float* __restrict__ el_src,
    const float* __restrict__ a_dst, int d, float slope, float* __restrict__ H,
    const float* __restrict__ G, float* __restrict__ GS, float* __restrict__ GP,
    float* __restrict__ AL, float* __restrict__ GT, float* __restrict__ SGT,
    const float* __restrict__ HO, const int64_t* __restrict__ ho_rows,
    unsigned* __restrict__ counter) {
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  float4 ad[NV];
  load4<NV>(ad, a_dst, d4, lane);
  // destinations in batches of kDstBatch from a device counter (zeroed
  // before the launch): whichever warp is free takes the next batch
  for (;;) {
    unsigned ub = 0;
    if (lane == 0) ub = atomicAdd(counter, 1u);
    ub = __shfl_sync(0xffffffffu, ub, 0);
    const int64_t vb = (int64_t)ub * kDstBatch;
    if (vb >= nseg) break;
    const int64_t ve = vb + kDstBatch < nseg ? vb + kDstBatch : nseg;
    for (int64_t v = vb; v < ve; ++v) {
      const int64_t e0 = off[v], e1 = off[v + 1];
      float4 pv[NV];
      load4<NV>(pv, P + v * (int64_t)d, d4, lane);
      const float el_d = warp_sum(dot4<NV>(pv, ad));
      // the first 32 in-edges (most destinations have fewer) stay in
      // registers across the passes: source id i0 and attention input t0
      const int c0 = (e1 - e0) < (int64_t)kW ? (int)(e1 - e0) : kW;
      const bool in0 = lane < c0;
      const int i0 = in0 ? __ldg(idx + e0 + lane) : 0;
      const float t0 = in0 ? el_d + __ldg(el_src + i0) : 0.f;
      // segment max and softmax denominator, lane-parallel over edges
      float mx = in0 ? leaky(t0, slope) : -CUDART_INF_F;
      for (int64_t e = e0 + kW + lane; e < e1; e += kW)
        mx = fmaxf(mx, leaky(el_d + __ldg(el_src + __ldg(idx + e)), slope));
      mx = warp_max(mx);
      const float x0 = in0 ? expf(leaky(t0, slope) - mx) : 0.f;
      float den = x0;
      for (int64_t e = e0 + kW + lane; e < e1; e += kW)
        den += expf(leaky(el_d + __ldg(el_src + __ldg(idx + e)), slope) - mx);
      den = warp_sum(den);
      const float a0 = in0 ? x0 / den : 0.f;  // alpha of the first chunk
      // s_v = sum alpha_e q_u, sequential in edge order.  Backward with the
      // layer output h = ReLU(s) in HBM (HO): (s > 0) == (h > 0) bitwise, so
      // only alpha is recomputed, not s (one row gather per edge saved)
      float4 acc[NV];
#pragma unroll
      for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (BWD && HO) {
        load4<NV>(acc, HO + (ho_rows ? ho_rows[v] : v) * (int64_t)d, d4, lane);
        if (in0) AL[2 * (e0 + lane)] = a0;
        for (int64_t e = e0 + kW + lane; e < e1; e += kW)
          AL[2 * (e)] = expf(leaky(el_d + __ldg(el_src + __ldg(idx + e)), slope) - mx) / den;
      }
      for (int64_t base = e0; base < ((BWD && HO) ? e0 : e1); base += kW) {
        const int cnt = (int)((e1 - base) < (int64_t)kW ? (e1 - base) : (int64_t)kW);
        int my_i = i0;
        float my_a = a0;
        if (base != e0 && lane < cnt) {
          my_i = __ldg(idx + base + lane);
          my_a = expf(leaky(el_d + __ldg(el_src + my_i), slope) - mx) / den;
        }
        if (BWD && lane < cnt) AL[2 * (base + lane)] = my_a;
        int k = 0;
        if (!BWD && NV == 1 && d4 <= 16) {
          // rows of <= 64 floats: each half-warp loads one row, so one
          // instruction brings two; the adds stay in edge order (lanes 0-15
          // hold the sums, lanes 16-31 hand over the odd rows)
          const int hl = lane >> 4, sl = lane & 15;
          for (; k + 8 <= cnt; k += 8) {
            float4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int s = __shfl_sync(0xffffffffu, my_i, k + 2 * u + hl);
              x[u] = sl < d4 ? __ldg(reinterpret_cast<const float4*>(Q + (int64_t)s * d) + sl)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float4 y;
              y.x = __shfl_down_sync(0xffffffffu, x[u].x, 16);
              y.y = __shfl_down_sync(0xffffffffu, x[u].y, 16);
              y.z = __shfl_down_sync(0xffffffffu, x[u].z, 16);
              y.w = __shfl_down_sync(0xffffffffu, x[u].w, 16);
              const float a0 = __shfl_sync(0xffffffffu, my_a, k + 2 * u);
              const float a1 = __shfl_sync(0xffffffffu, my_a, k + 2 * u + 1);
              axpy_rn(acc[0], a0, x[u]);
              axpy_rn(acc[0], a1, y);
            }
          }
        }
        for (; k + DU <= cnt; k += DU) {  // DU rows in flight
          float4 x[DU][NV];
          float a[DU];
#pragma unroll
          for (int u = 0; u < DU; ++u) {
            const int s = __shfl_sync(0xffffffffu, my_i, k + u);
            a[u] = __shfl_sync(0xffffffffu, my_a, k + u);
            load4<NV>(x[u], Q + (int64_t)s * d, d4, lane);
          }
#pragma unroll
          for (int u = 0; u < DU; ++u)
#pragma unroll
            for (int t = 0; t < NV; ++t) axpy_rn(acc[t], a[u], x[u][t]);
        }
        for (; k < cnt; ++k) {
          const int s = __shfl_sync(0xffffffffu, my_i, k);
          const float a = __shfl_sync(0xffffffffu, my_a, k);
          float4 x[NV];
          load4<NV>(x, Q + (int64_t)s * d, d4, lane);
#pragma unroll
          for (int t = 0; t < NV; ++t) axpy_rn(acc[t], a, x[t]);
        }
      }
      if (!BWD) {
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          acc[t].x = fmaxf(acc[t].x, 0.f);
          acc[t].y = fmaxf(acc[t].y, 0.f);
          acc[t].z = fmaxf(acc[t].z, 0.f);
          acc[t].w = fmaxf(acc[t].w, 0.f);
        }
        store4<NV>(H + v * (int64_t)d, acc, d4, lane);
        continue;
      }
      // ---- backward: gs = g * (s > 0) ----
      float4 gs[NV];
      load4<NV>(gs, G + v * (int64_t)d, d4, lane);
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        gs[t].x = acc[t].x > 0.f ? gs[t].x : 0.f;
        gs[t].y = acc[t].y > 0.f ? gs[t].y : 0.f;
        gs[t].z = acc[t].z > 0.f ? gs[t].z : 0.f;
        gs[t].w = acc[t].w > 0.f ? gs[t].w : 0.f;
      }
      store4<NV>(GS + v * (int64_t)d, gs, d4, lane);
      // g_alpha_e = gs . q_u, sum alpha_e g_alpha_e; the first chunk keeps
      // its g_alpha in a register (g0), later chunks park it in GT
      float sdot = 0.f, g0 = 0.f;
      for (int64_t base = e0; base < e1; base += kW) {
        const int cnt = (int)((e1 - base) < (int64_t)kW ? (e1 - base) : (int64_t)kW);
        const int my_i = base == e0 ? i0 : (lane < cnt ? __ldg(idx + base + lane) : 0);
        float my_g = 0.f;
        int k = 0;
        for (; k + DU <= cnt; k += DU) {  // DU rows in flight, DU interleaved reductions
          float4 x[DU][NV];
#pragma unroll
          for (int u = 0; u < DU; ++u) {
            const int s = __shfl_sync(0xffffffffu, my_i, k + u);
            load4<NV>(x[u], Q + (int64_t)s * d, d4, lane);
          }
          float g[DU];
#pragma unroll
          for (int u = 0; u < DU; ++u) g[u] = dot4<NV>(gs, x[u]);
#pragma unroll
          for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int u = 0; u < DU; ++u) g[u] += __shfl_xor_sync(0xffffffffu, g[u], o);
#pragma unroll
          for (int u = 0; u < DU; ++u)
            if (lane == k + u) my_g = g[u];
        }
        for (; k < cnt; ++k) {
          const int s = __shfl_sync(0xffffffffu, my_i, k);
          float4 x[NV];
          load4<NV>(x, Q + (int64_t)s * d, d4, lane);
          const float g = warp_sum(dot4<NV>(gs, x));
          if (lane == k) my_g = g;
        }
        if (lane < cnt) {
          if (base == e0) {
            g0 = my_g;
            sdot += a0 * my_g;
          } else {
            GT[2 * (base + lane)] = my_g;
            sdot += AL[2 * (base + lane)] * my_g;
          }
        }
      }
      sdot = warp_sum(sdot);
      float sgt = 0.f;
      if (in0) {
        const float gt = a0 * (g0 - sdot) * (t0 > 0.f ? 1.f : slope);
        GT[2 * (e0 + lane)] = gt;
        sgt = gt;
      }
      for (int64_t e = e0 + kW + lane; e < e1; e += kW) {
        const float t = el_d + __ldg(el_src + __ldg(idx + e));
        const float gt = AL[2 * (e)] * (GT[2 * (e)] - sdot) * (t > 0.f ? 1.f : slope);
        GT[2 * (e)] = gt;
        sgt += gt;
      }
      sgt = warp_sum(sgt);
      if (lane == 0) SGT[v] = sgt;
      if (GP) {  // (null: the rank-1 gp = sgt a_dst is folded into gq by k_gat_src)
        float4 gp[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t)
          gp[t] = make_float4(sgt * ad[t].x, sgt * ad[t].y, sgt * ad[t].z, sgt * ad[t].w);
        store4<NV>(GP + v * (int64_t)d, gp, d4, lane);
      }
    }
  }
}

// gq / gts contribution of CSR edges [e0, e1) of one source (one warp):
// per edge (alpha gs_dst + g_t a_src), added in edge order; four rows in
// flight.
#ifndef HT_GAT_SU
#define HT_GAT_SU 8
#endif
constexpr int SU = HT_GAT_SU;  // CSR rows in flight per warp
template <int NV>
__device__ __forceinline__ void src_sum(float4 (&acc)[NV], float& gts, int64_t e0, int64_t e1,
                                        const int32_t* __restrict__ dst,
                                        const int32_t* __restrict__ perm,
                                        const float* __restrict__ GS, const float* __restrict__ AL,
                                        const float* __restrict__ GT, const float4 (&as)[NV],
                                        int d, int d4, int lane) {
  for (int64_t base = e0; base < e1; base += kW) {
    const int cnt = (int)((e1 - base) < (int64_t)kW ? (e1 - base) : (int64_t)kW);
    int my_d = 0;
    float my_a = 0.f, my_t = 0.f;
    if (lane < cnt) {  // alpha and g_t of the edge: one 8-byte record (CSC order)
      my_d = __ldg(dst + base + lane);
      const int32_t pe = __ldg(perm + base + lane);
      const float2 at = __ldg(reinterpret_cast<const float2*>(AL) + pe);
      my_a = at.x;
      my_t = at.y;
      gts += my_t;
    }
    int k = 0;
    for (; k + SU <= cnt; k += SU) {
      float4 x[SU][NV];
      float a[SU], g[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int r = __shfl_sync(0xffffffffu, my_d, k + u);
        a[u] = __shfl_sync(0xffffffffu, my_a, k + u);
        g[u] = __shfl_sync(0xffffffffu, my_t, k + u);
        load4<NV>(x[u], GS + (int64_t)r * d, d4, lane);
      }
#pragma unroll
      for (int u = 0; u < SU; ++u)
#pragma unroll
        for (int t = 0; t < NV; ++t) edge_add(acc[t], a[u], x[u][t], g[u], as[t]);
    }
    for (; k < cnt; ++k) {
      const int r = __shfl_sync(0xffffffffu, my_d, k);
      const float a = __shfl_sync(0xffffffffu, my_a, k);
      const float g = __shfl_sync(0xffffffffu, my_t, k);
      float4 x[NV];
      load4<NV>(x, GS + (int64_t)r * d, d4, lane);
#pragma unroll
      for (int t = 0; t < NV; ++t) edge_add(acc[t], a, x[t], g, as[t]);
    }
  }
}

// One warp per source segment of a chunk's CSR view: dst = chunk-local
// destination rows of GS, perm = CSC edge id (index into AL / GT).
// Segments longer than `split` edges are left to k_gat_src_pieces.
template <int NV>
__global__ void __launch_bounds__(256) k_gat_src(
    const int64_t* __restrict__ off, const int32_t* __restrict__ dst,
    const int32_t* __restrict__ perm, int64_t nseg, int64_t split, const float* __restrict__ GS,
    const float* __restrict__ AL, const float* __restrict__ GT, const float* __restrict__ a_src,
    int d, float* __restrict__ GQ, float* __restrict__ GTS, const float* __restrict__ sgt_add,
    const float* __restrict__ a_dst) {
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  float4 as[NV];
  load4<NV>(as, a_src, d4, lane);
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nseg; u += nw) {
    const int64_t e0 = off[u], e1 = off[u + 1];
    if (e1 - e0 > split) continue;
    float4 acc[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    float gts = 0.f;
    const float g = sgt_add ? __ldg(sgt_add + u) : 0.f;  // requested before the edge loop
    src_sum<NV>(acc, gts, e0, e1, dst, perm, GS, AL, GT, as, d, d4, lane);
    if (sgt_add) {  // one device, one batch: row u's destination term gp_u = sgt_u a_dst
      const float4* ad4 = reinterpret_cast<const float4*>(a_dst);
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const int c = lane + t * kW;
        if (c < d4) {
          const float4 ad = __ldg(ad4 + c);
          acc[t].x += g * ad.x;
          acc[t].y += g * ad.y;
          acc[t].z += g * ad.z;
          acc[t].w += g * ad.w;
        }
      }
    }
    store4<NV>(GQ + u * (int64_t)d, acc, d4, lane);
    gts = warp_sum(gts);
    if (lane == 0) GTS[u] = gts;
  }
}

// pieces [lo, hi) of long source segments -> partial rows / gts partials
template <int NV>
__global__ void __launch_bounds__(256) k_gat_src_pieces(
    const int64_t* __restrict__ lo, const int64_t* __restrict__ hi, int64_t np,
    const int32_t* __restrict__ dst, const int32_t* __restrict__ perm,
    const float* __restrict__ GS, const float* __restrict__ AL, const float* __restrict__ GT,
    const float* __restrict__ a_src, int d, float* __restrict__ part, float* __restrict__ pgts) {
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  float4 as[NV];
  load4<NV>(as, a_src, d4, lane);
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < np; q += nw) {
    float4 acc[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    float gts = 0.f;
    src_sum<NV>(acc, gts, lo[q], hi[q], dst, perm, GS, AL, GT, as, d, d4, lane);
    store4<NV>(part + q * (int64_t)d, acc, d4, lane);
    gts = warp_sum(gts);
    if (lane == 0) pgts[q] = gts;
  }
}

// long segment s: GQ / GTS = sum of its pieces in piece order
static __global__ void __launch_bounds__(256) k_gat_src_fixup(
    float* __restrict__ GQ, float* __restrict__ GTS, const float* __restrict__ part,
    const float* __restrict__ pgts, int d, const int64_t* __restrict__ seg,
    const int64_t* __restrict__ first, const int64_t* __restrict__ cnt, int64_t nf,
    const float* __restrict__ sgt_add, const float* __restrict__ a_dst) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t f = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; f < nf; f += nw) {
    const int64_t q0 = first[f], qn = cnt[f];
    for (int c = lane; c < d; c += kW) {
      float s = 0.f;
      for (int64_t q = 0; q < qn; ++q) s = __fadd_rn(s, part[(q0 + q) * d + c]);
      if (sgt_add) s += sgt_add[seg[f]] * a_dst[c];
      GQ[seg[f] * (int64_t)d + c] = s;
    }
    if (lane == 0) {
      float s = 0.f;
      for (int64_t q = 0; q < qn; ++q) s += pgts[q0 + q];
      GTS[seg[f]] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Split backward (the layer output h = ReLU(s) in HBM, so s's sign is known
// without re-aggregating): ONE row gather per edge instead of two.
//   A  (per destination)  alpha_e, gs_v = g_v (s_v > 0), el_d[v]
//   S1 (per source, CSR)  gathers gs_v rows: g_alpha_e = gs_v . q_u (q_u in
//                         registers) and A_u = sum_e alpha_e gs_v in edge order;
//                         one work-list launch (hub pieces first)
//   B  (per destination)  sdot_v, g_t_e, seg sum of g_t (scalars only)
//   S2 (per source)       gts_u = sum_e g_t_e; gq_u = A_u + gts_u a_src
// alpha, g_alpha, g_t, sdot, gts are the fused kernels' values bitwise; gq
// is the same sum in a different association (A_u, then the a_src term).
// (A transposed reduction of eight edges' g_alpha sums in 9 shuffles
// instead of 40 measured 12 % slower in S1: the pass is memory-bound.)
// Per-edge records {alpha, g_alpha -> g_t} in CSC order.
// ---------------------------------------------------------------------------
template <int NV>
__global__ void __launch_bounds__(256, NV == 1 ? HT_GAT_AB_MINB : 1) k_gat_bwd_a(
    const int64_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t nseg,
    const float* __restrict__ P, const float* __restrict__ el_src, const float* __restrict__ a_dst,
    int d, float slope, const float* __restrict__ G, const float* __restrict__ HO,
    const int64_t* __restrict__ ho_rows, float* __restrict__ GS, float* __restrict__ AL,
    float* __restrict__ ELD,
    unsigned* __restrict__ counter) {
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  float4 ad[NV];
  load4<NV>(ad, a_dst, d4, lane);
  for (;;) {  // destinations in batches of kDstBatch from a device counter
    unsigned ub = 0;
    if (lane == 0) ub = atomicAdd(counter, 1u);
    ub = __shfl_sync(0xffffffffu, ub, 0);
    const int64_t vb = (int64_t)ub * kDstBatch;
    if (vb >= nseg) break;
    const int64_t ve = vb + kDstBatch < nseg ? vb + kDstBatch : nseg;
    for (int64_t v = vb; v < ve; ++v) {
      const int64_t e0 = off[v], e1 = off[v + 1];
      float4 pv[NV], ho[NV], gv[NV];
      load4<NV>(pv, P + v * (int64_t)d, d4, lane);
      load4<NV>(ho, HO + (ho_rows ? ho_rows[v] : v) * (int64_t)d, d4, lane);
      load4<NV>(gv, G + v * (int64_t)d, d4, lane);
      const float el_d = warp_sum(dot4<NV>(pv, ad));
      const int c0 = (e1 - e0) < (int64_t)kW ? (int)(e1 - e0) : kW;
      const bool in0 = lane < c0;
      const float t0 = in0 ? el_d + __ldg(el_src + __ldg(idx + e0 + lane)) : 0.f;
      float mx = in0 ? leaky(t0, slope) : -CUDART_INF_F;
      for (int64_t e = e0 + kW + lane; e < e1; e += kW)
        mx = fmaxf(mx, leaky(el_d + __ldg(el_src + __ldg(idx + e)), slope));
      mx = warp_max(mx);
      const float x0 = in0 ? expf(leaky(t0, slope) - mx) : 0.f;
      float den = x0;
      for (int64_t e = e0 + kW + lane; e < e1; e += kW)
        den += expf(leaky(el_d + __ldg(el_src + __ldg(idx + e)), slope) - mx);
      den = warp_sum(den);
      if (in0) AL[2 * (e0 + lane)] = x0 / den;
      for (int64_t e = e0 + kW + lane; e < e1; e += kW)
        AL[2 * e] = expf(leaky(el_d + __ldg(el_src + __ldg(idx + e)), slope) - mx) / den;
#pragma unroll
      for (int t = 0; t < NV; ++t) {  // gs = g (s > 0), (s > 0) == (h > 0)
        gv[t].x = ho[t].x > 0.f ? gv[t].x : 0.f;
        gv[t].y = ho[t].y > 0.f ? gv[t].y : 0.f;
        gv[t].z = ho[t].z > 0.f ? gv[t].z : 0.f;
        gv[t].w = ho[t].w > 0.f ? gv[t].w : 0.f;
      }
      store4<NV>(GS + v * (int64_t)d, gv, d4, lane);
      if (lane == 0) ELD[v] = el_d;
    }
  }
}

// S1 over CSR edges [e0, e1) of source u (one warp; q_u in registers):
// A_u += alpha_e gs_v in edge order; g_alpha_e -> record .y
template <int NV>
__device__ __forceinline__ void src_rows_a(float4 (&acc)[NV], const float4 (&qu)[NV], int64_t e0,
                                           int64_t e1, const int32_t* __restrict__ dst,
                                           const int32_t* __restrict__ perm,
                                           const float* __restrict__ GS, float* __restrict__ AL,
                                           int d, int d4, int lane) {
  for (int64_t base = e0; base < e1; base += kW) {
    const int cnt = (int)((e1 - base) < (int64_t)kW ? (e1 - base) : (int64_t)kW);
    int my_d = 0, my_p = 0;
    float my_a = 0.f;
    if (lane < cnt) {
      my_d = __ldg(dst + base + lane);
      my_p = __ldg(perm + base + lane);
      my_a = AL[2 * (int64_t)my_p];  // (plain load: the record's .y is written in this kernel)
    }
    float my_g = 0.f;
    int k = 0;
    for (; k + SU <= cnt; k += SU) {
      float4 x[SU][NV];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int r = __shfl_sync(0xffffffffu, my_d, k + u);
        load4<NV>(x[u], GS + (int64_t)r * d, d4, lane);
      }
      float g[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const float a = __shfl_sync(0xffffffffu, my_a, k + u);
#pragma unroll
        for (int t = 0; t < NV; ++t) axpy_rn(acc[t], a, x[u][t]);
        g[u] = dot4<NV>(x[u], qu);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int u = 0; u < SU; ++u) g[u] += __shfl_xor_sync(0xffffffffu, g[u], o);
#pragma unroll
      for (int u = 0; u < SU; ++u)
        if (lane == k + u) my_g = g[u];
    }
    for (; k < cnt; ++k) {
      const int r = __shfl_sync(0xffffffffu, my_d, k);
      const float a = __shfl_sync(0xffffffffu, my_a, k);
      float4 x[NV];
      load4<NV>(x, GS + (int64_t)r * d, d4, lane);
#pragma unroll
      for (int t = 0; t < NV; ++t) axpy_rn(acc[t], a, x[t]);
      const float g = warp_sum(dot4<NV>(x, qu));
      if (lane == k) my_g = g;
    }
    if (lane < cnt) AL[2 * (int64_t)my_p + 1] = my_g;
  }
}

// S1 as one work-list launch (like ht::k_seg_work_v4): units [0, np) are
// the hub pieces, then batches of B short source segments, taken from a
// device counter; the last piece of a hub (atomic ticket) sums the hub's
// partial rows in piece order into GQ (k_seg_fixup's order).  counter and
// tickets zeroed before the launch.
template <int NV, int B>
__global__ void __launch_bounds__(256, NV == 1 ? HT_GAT_S1_MINB : 1) k_gat_bwd_s1_work(
    const int64_t* __restrict__ off, const int32_t* __restrict__ dst,
    const int32_t* __restrict__ perm, int64_t nseg, int64_t split,
    const int64_t* __restrict__ lo, const int64_t* __restrict__ hi, const int32_t* __restrict__ pf,
    const int64_t* __restrict__ fseg, const int64_t* __restrict__ ffirst,
    const int64_t* __restrict__ fcnt, int64_t np, unsigned* __restrict__ counter,
    int* __restrict__ tickets, const float* __restrict__ GS, const float* __restrict__ Q,
    float* __restrict__ AL, int d, float* __restrict__ part, float* __restrict__ GQ) {
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  const int64_t nunits = np + (nseg + B - 1) / B;
  for (;;) {
    unsigned uu = 0;
    if (lane == 0) uu = atomicAdd(counter, 1u);
    uu = __shfl_sync(0xffffffffu, uu, 0);
    if ((int64_t)uu >= nunits) break;
    float4 acc[NV], qu[NV];
    if ((int64_t)uu < np) {  // a hub piece
      const int64_t q = uu;
      const int f = pf[q];
      const int64_t u = fseg[f];
#pragma unroll
      for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      load4<NV>(qu, Q + u * (int64_t)d, d4, lane);
      src_rows_a<NV>(acc, qu, lo[q], hi[q], dst, perm, GS, AL, d, d4, lane);
      store4<NV>(part + q * (int64_t)d, acc, d4, lane);
      __threadfence();
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(tickets + f, 1) == (int)fcnt[f] - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {  // every piece written: their sum in piece order
        __threadfence();
        float4* o = reinterpret_cast<float4*>(GQ + u * (int64_t)d);
        for (int c = lane; c < d4; c += kW) o[c] = ht::sum_partials(part, ffirst[f], fcnt[f], d, c);
      }
      continue;
    }
    const int64_t s0 = ((int64_t)uu - np) * B;
    const int64_t s1 = s0 + B < nseg ? s0 + B : nseg;
    for (int64_t u = s0; u < s1; ++u) {
      const int64_t e0 = off[u], e1 = off[u + 1];
      if (e1 - e0 > split) continue;  // a hub: its pieces
#pragma unroll
      for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e1 > e0) load4<NV>(qu, Q + u * (int64_t)d, d4, lane);
      src_rows_a<NV>(acc, qu, e0, e1, dst, perm, GS, AL, d, d4, lane);
      store4<NV>(GQ + u * (int64_t)d, acc, d4, lane);
    }
  }
}

// B: per destination, scalars only: sdot_v = sum alpha_e g_alpha_e (lane
// partial sums, then the warp sum: the fused kernel's association), g_t_e
// into record .y, sgt_v = seg sum of g_t, optionally gp_v = sgt_v a_dst
template <int NV>
__global__ void __launch_bounds__(256, NV == 1 ? HT_GAT_AB_MINB : 1) k_gat_bwd_b(
    const int64_t* __restrict__ off, const int32_t* __restrict__ idx, int64_t nseg,
    const float* __restrict__ el_src, const float* __restrict__ ELD, float slope,
    float* __restrict__ AL, float* __restrict__ SGT, float* __restrict__ GP,
    const float* __restrict__ a_dst, int d,
    unsigned* __restrict__ counter) {
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  for (;;) {  // destinations in batches of kDstBatch from a device counter
    unsigned ub = 0;
    if (lane == 0) ub = atomicAdd(counter, 1u);
    ub = __shfl_sync(0xffffffffu, ub, 0);
    const int64_t vb = (int64_t)ub * kDstBatch;
    if (vb >= nseg) break;
    const int64_t ve = vb + kDstBatch < nseg ? vb + kDstBatch : nseg;
    for (int64_t v = vb; v < ve; ++v) {
      const int64_t e0 = off[v], e1 = off[v + 1];
      const float el_d = ELD[v];
      float sdot = 0.f;
      for (int64_t e = e0 + lane; e < e1; e += kW) {
        const float2 r = *reinterpret_cast<const float2*>(AL + 2 * e);
        sdot += r.x * r.y;
      }
      sdot = warp_sum(sdot);
      float sgt = 0.f;
      for (int64_t e = e0 + lane; e < e1; e += kW) {
        float2 r = *reinterpret_cast<float2*>(AL + 2 * e);
        const float t = el_d + __ldg(el_src + __ldg(idx + e));
        const float gt = r.x * (r.y - sdot) * (t > 0.f ? 1.f : slope);
        AL[2 * e + 1] = gt;
        sgt += gt;
      }
      sgt = warp_sum(sgt);
      if (lane == 0) SGT[v] = sgt;
      if (GP) {
        float4 ad[NV], gp[NV];
        load4<NV>(ad, a_dst, d4, lane);
#pragma unroll
        for (int t = 0; t < NV; ++t)
          gp[t] = make_float4(sgt * ad[t].x, sgt * ad[t].y, sgt * ad[t].z, sgt * ad[t].w);
        store4<NV>(GP + v * (int64_t)d, gp, d4, lane);
      }
    }
  }
}

// S2: gts_u = sum of the g_t of u's out-edges (lane partial sums in edge
// order, then the warp sum - the fused kernel's association); hubs in
// pieces (partial gts, then summed in piece order by the last piece of
// the segment: atomic ticket).  gq_u = A_u + gts_u a_src (+ sgt_u a_dst
// when the destination term is folded in).
template <int NV>
__device__ __forceinline__ void s2_finish(float* __restrict__ GQ, float* __restrict__ GTS,
                                          int64_t u, float gts, const float* __restrict__ a_src,
                                          const float* __restrict__ sgt_add,
                                          const float* __restrict__ a_dst, int d, int d4, int lane) {
  float4 acc[NV], as[NV];
  load4<NV>(acc, GQ + u * (int64_t)d, d4, lane);
  load4<NV>(as, a_src, d4, lane);
  const float g = sgt_add ? __ldg(sgt_add + u) : 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    acc[t].x += gts * as[t].x;
    acc[t].y += gts * as[t].y;
    acc[t].z += gts * as[t].z;
    acc[t].w += gts * as[t].w;
  }
  if (sgt_add) {
    float4 ad[NV];
    load4<NV>(ad, a_dst, d4, lane);
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      acc[t].x += g * ad[t].x;
      acc[t].y += g * ad[t].y;
      acc[t].z += g * ad[t].z;
      acc[t].w += g * ad[t].w;
    }
  }
  store4<NV>(GQ + u * (int64_t)d, acc, d4, lane);
  if (lane == 0) GTS[u] = gts;
}

template <int NV>
__global__ void __launch_bounds__(256) k_gat_bwd_s2(
    const int64_t* __restrict__ off, const int32_t* __restrict__ perm, int64_t nseg,
    int64_t split, const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
    const int32_t* __restrict__ pf, const int64_t* __restrict__ fseg,
    const int64_t* __restrict__ ffirst, const int64_t* __restrict__ fcnt, int64_t np,
    unsigned* __restrict__ counter, int* __restrict__ tickets, float* __restrict__ pgts,
    const float* __restrict__ AL, const float* __restrict__ a_src,
    const float* __restrict__ sgt_add, const float* __restrict__ a_dst, int d,
    float* __restrict__ GQ, float* __restrict__ GTS) {
  const int lane = threadIdx.x & 31;
  const int d4 = d >> 2;
  const int64_t nunits = np + (nseg + kDstBatch - 1) / kDstBatch;
  for (;;) {  // hub pieces first, then batches of sources, from a device counter
    unsigned uu = 0;
    if (lane == 0) uu = atomicAdd(counter, 1u);
    uu = __shfl_sync(0xffffffffu, uu, 0);
    if ((int64_t)uu >= nunits) break;
    if ((int64_t)uu < np) {  // a piece of a hub source
      const int64_t w = uu;
      float gts = 0.f;
      for (int64_t e = lo[w] + lane; e < hi[w]; e += kW) gts += __ldg(AL + 2 * (int64_t)__ldg(perm + e) + 1);
      gts = warp_sum(gts);
      if (lane == 0) pgts[w] = gts;
      __threadfence();
      __syncwarp();
      const int f = pf[w];
      int last = 0;
      if (lane == 0) last = atomicAdd(tickets + f, 1) == (int)fcnt[f] - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence();
        float s = 0.f;
        for (int64_t q = 0; q < fcnt[f]; ++q) s += __ldcg(pgts + ffirst[f] + q);
        s2_finish<NV>(GQ, GTS, fseg[f], s, a_src, sgt_add, a_dst, d, d4, lane);
      }
      continue;
    }
    const int64_t u0 = ((int64_t)uu - np) * kDstBatch;
    const int64_t u1 = u0 + kDstBatch < nseg ? u0 + kDstBatch : nseg;
    for (int64_t u = u0; u < u1; ++u) {
      const int64_t e0 = off[u], e1 = off[u + 1];
      if (e1 - e0 > split) continue;
      float gts = 0.f;
      for (int64_t e = e0 + lane; e < e1; e += kW) gts += __ldg(AL + 2 * (int64_t)__ldg(perm + e) + 1);
      gts = warp_sum(gts);
      s2_finish<NV>(GQ, GTS, u, gts, a_src, sgt_add, a_dst, d, d4, lane);
    }
  }
}

// partial[b][c] = sum over block b's rows r of w[r] * X[r][c]: warps take
// rows, lanes float4 columns, the block's 8 warp sums combined in shared
// memory in warp order (deterministic)
template <int NV>
__global__ void __launch_bounds__(256) k_wcolsum(float* __restrict__ partial,
                                                 const float* __restrict__ X, int64_t ldx,
                                                 const float* __restrict__ w, int64_t rows, int d,
                                                 int64_t rows_per_block) {
  __shared__ float4 red[8][NV * kW];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int d4 = d >> 2;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float4 acc[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t r = r0 + wib; r < r1; r += 8) {
    const float wr = __ldg(w + r);
    float4 x[NV];
    load4<NV>(x, X + r * ldx, d4, lane);
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      acc[t].x = fmaf(wr, x[t].x, acc[t].x);
      acc[t].y = fmaf(wr, x[t].y, acc[t].y);
      acc[t].z = fmaf(wr, x[t].z, acc[t].z);
      acc[t].w = fmaf(wr, x[t].w, acc[t].w);
    }
  }
#pragma unroll
  for (int t = 0; t < NV; ++t) red[wib][lane + t * kW] = acc[t];
  __syncthreads();
  for (int c4 = threadIdx.x; c4 < d4; c4 += blockDim.x) {
    float4 s = red[0][c4];
    for (int q = 1; q < 8; ++q) {
      s.x += red[q][c4].x;
      s.y += red[q][c4].y;
      s.z += red[q][c4].z;
      s.w += red[q][c4].w;
    }
    reinterpret_cast<float4*>(partial + (int64_t)blockIdx.x * d)[c4] = s;
  }
}

// out[c] += sum_b partial[b][c], b ascending
static __global__ void k_colsum_reduce(float* __restrict__ out, const float* __restrict__ partial,
                                int nb, int d) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float s = 0.f;
  for (int b = 0; b < nb; ++b) s += partial[(int64_t)b * d + c];
  out[c] += s;
}

}  // namespace gat
}  // namespace ht
