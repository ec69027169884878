// Microbenchmark: random-row gather-sum on B200.  How many rows/s can a
// warp-per-row gather reach with (a) register-held rows, U in flight per
// warp, segment-local (the k_seg_gather_v4 scheme) vs (b) cp.async rows
// staged in shared memory, D in flight per warp across segment boundaries?
// Rows: X (nrows x d floats, 2.4 GB), idx: random (uniform) row ids,
// segments of 26 edges; out: one row per segment.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int NV, int U>
__global__ void __launch_bounds__(256) k_reg(float* out, const float* X, int d, const int* idx,
                                             int64_t nseg, int seglen) {
  const int lane = threadIdx.x & 31, d4 = d >> 2;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t s = blockIdx.x * 8 + (threadIdx.x >> 5); s < nseg; s += nw) {
    float4 acc[NV];
    for (int t = 0; t < NV; ++t) acc[t] = make_float4(0, 0, 0, 0);
    const int64_t e0 = s * seglen;
    const int my = lane < seglen ? idx[e0 + lane] : 0;
    for (int k = 0; k < seglen; k += U) {
      float4 x[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = __shfl_sync(0xffffffffu, my, (k + u) & 31);
        const float4* row = reinterpret_cast<const float4*>(X + (int64_t)r * d);
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          const int c = lane + 32 * t;
          x[u][t] = (k + u < seglen && c < d4) ? __ldg(row + c) : make_float4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          acc[t].x += x[u][t].x; acc[t].y += x[u][t].y; acc[t].z += x[u][t].z; acc[t].w += x[u][t].w;
        }
    }
    float4* o = reinterpret_cast<float4*>(out + s * (int64_t)d);
    for (int t = 0; t < NV; ++t) if (lane + 32 * t < d4) o[lane + 32 * t] = acc[t];
  }
}

__device__ __forceinline__ void cp16(void* smem, const void* g, bool p) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = p ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(g), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// D rows in flight per warp, streamed across segment boundaries; each lane
// consumes exactly the 16-byte words it copied (no cross-lane sync).
template <int NV, int D, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_cpa(float* out, const float* X, int d, const int* idx,
                                                  int64_t nseg, int seglen) {
  extern __shared__ float4 sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, d4 = d >> 2;
  float4* ring = sm + (int64_t)wib * D * NV * 32;
  const int64_t nw = (int64_t)gridDim.x * WPB;
  const int64_t w = blockIdx.x * WPB + wib;
  // warp w takes segments w, w+nw, ...: a flat stream of edges
  const int64_t nmine = w < nseg ? (nseg - 1 - w) / nw + 1 : 0;
  const int64_t ne = nmine * seglen;
  auto edge_row_lane = [&](int64_t q) -> int {  // lane-parallel: edge q of the stream
    if (q >= ne) return 0;
    const int64_t s = w + (q / seglen) * nw;
    return idx[s * seglen + q % seglen];
  };
  // edge-row windows of 32: w0 = [32k, 32k+32), w1 = the next (prefetched)
  int w0 = edge_row_lane(lane), w1 = edge_row_lane(32 + lane);
  auto row_of = [&](int64_t q, int64_t base) -> int {  // q in [base, base+64)
    const int o = (int)(q - base);
    const int a = __shfl_sync(0xffffffffu, w0, o & 31), b = __shfl_sync(0xffffffffu, w1, o & 31);
    return o < 32 ? a : b;
  };
  int64_t base = 0;
  // prologue
  for (int q = 0; q < D; ++q) {
    const bool p = q < ne;
    const int r = row_of(q, 0);
    const float4* row = reinterpret_cast<const float4*>(X + (int64_t)r * d);
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const int c = lane + 32 * t;
      cp16(&ring[(q % D) * NV * 32 + t * 32 + lane], row + (c < d4 ? c : 0), p && c < d4);
    }
    cp_commit();
  }
  float4 acc[NV];
  for (int t = 0; t < NV; ++t) acc[t] = make_float4(0, 0, 0, 0);
  for (int64_t q = 0; q < ne; ++q) {
    cp_wait<D - 1>();
    const int slot = (int)(q % D);
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const float4 v = ring[slot * NV * 32 + t * 32 + lane];
      acc[t].x += v.x; acc[t].y += v.y; acc[t].z += v.z; acc[t].w += v.w;
    }
    if ((q + 1) % seglen == 0) {
      const int64_t s = w + (q / seglen) * nw;
      float4* o = reinterpret_cast<float4*>(out + s * (int64_t)d);
      for (int t = 0; t < NV; ++t) {
        if (lane + 32 * t < d4) o[lane + 32 * t] = acc[t];
        acc[t] = make_float4(0, 0, 0, 0);
      }
    }
    const int64_t qn = q + D;
    const bool p = qn < ne;
    const int r = row_of(qn, base);
    const float4* row = reinterpret_cast<const float4*>(X + (int64_t)r * d);
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const int c = lane + 32 * t;
      cp16(&ring[slot * NV * 32 + t * 32 + lane], row + (c < d4 ? c : 0), p && c < d4);
    }
    cp_commit();
    if (qn + 1 == base + 32) {  // next issue is in w1: slide the windows, prefetch
      base += 32;
      w0 = w1;
      w1 = edge_row_lane(base + 32 + lane);
    }
  }
  cp_wait<0>();
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  CK(cudaGetLastError());
  return ms / 5;
}

int main() {
  const int64_t nrows = 2400000, seglen = 26, nseg = 2400000;
  const int64_t ne = nseg * seglen;
  float *X, *out; int* idx;
  CK(cudaMalloc(&X, nrows * 256 * 4)); CK(cudaMalloc(&out, nseg * 256 * 4)); CK(cudaMalloc(&idx, ne * 4));
  CK(cudaMemset(X, 0, nrows * 256 * 4));
  std::vector<int> h(ne);
  std::mt19937 g(1);
  for (auto& v : h) v = (int)(g() % nrows);
  CK(cudaMemcpy(idx, h.data(), ne * 4, cudaMemcpyHostToDevice));
  const int sms = 148;
  for (int d : {48, 100, 256}) {
    double rows = (double)ne, bytes = rows * d * 4;
    auto rep = [&](const char* name, float ms) {
      printf("d=%3d %-22s %7.3f ms  %6.2f Grows/s  %7.0f GB/s (row bytes)\n", d, name, ms, rows / ms / 1e6, bytes / ms / 1e6);
    };
    if (d <= 128) {
      rep("reg U=8", timeit([&] { k_reg<1, 8><<<sms * 16, 256>>>(out, X, d, idx, nseg, seglen); }));
      rep("reg U=16", timeit([&] { k_reg<1, 16><<<sms * 16, 256>>>(out, X, d, idx, nseg, seglen); }));
      for (int D : {8, 16}) {
        size_t smem = (size_t)8 * D * 1 * 32 * 16;
        if (D == 8) { auto k = k_cpa<1, 8, 8>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          rep("cp.async D=8", timeit([&] { k<<<sms * 8, 256, smem>>>(out, X, d, idx, nseg, seglen); })); }
        else { auto k = k_cpa<1, 16, 8>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          rep("cp.async D=16", timeit([&] { k<<<sms * 8, 256, smem>>>(out, X, d, idx, nseg, seglen); })); }
      }
    } else {
      rep("reg U=2", timeit([&] { k_reg<2, 2><<<sms * 16, 256>>>(out, X, d, idx, nseg, seglen); }));
      rep("reg U=4", timeit([&] { k_reg<2, 4><<<sms * 16, 256>>>(out, X, d, idx, nseg, seglen); }));
      { const int D = 4; size_t smem = (size_t)8 * D * 2 * 32 * 16; auto k = k_cpa<2, 4, 8>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rep("cp.async D=4", timeit([&] { k<<<sms * 8, 256, smem>>>(out, X, d, idx, nseg, seglen); })); }
      { const int D = 6; size_t smem = (size_t)8 * D * 2 * 32 * 16; auto k = k_cpa<2, 6, 8>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rep("cp.async D=6", timeit([&] { k<<<sms * 8, 256, smem>>>(out, X, d, idx, nseg, seglen); })); }
      { const int D = 12; size_t smem = (size_t)4 * D * 2 * 32 * 16; auto k = k_cpa<2, 12, 4>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rep("cp.async D=12 4w", timeit([&] { k<<<sms * 8, 128, smem>>>(out, X, d, idx, nseg, seglen); })); }
    }
  }
  return 0;
}
