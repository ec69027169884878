// tcgen05 (5th-generation tensor core) TF32 GEMMs of the dense transform.
//
// Shapes of the GCN layer (M = destination rows of a chunk, up to millions;
// d_in, d_out <= 256):
//   z    = agg . W          (forward K4 and backward recompute; 3xTF32)
//   gagg = gz . W^T         (backward K7; 1xTF32)
//   dW  += agg^T . gz       (backward K7; 1xTF32, split over rows)
//
// Kernel k_tc_rows (z and gagg): one 128-row tile of the row operand per
// MMA (M=128), a feature tile of BN columns (N=BN), K swept in 32-float
// chunks (one 128-byte swizzle atom).  The whole feature tile of the weight
// operand (BN x K, hi and lo halves) stays resident in shared memory for
// the CTA's lifetime; persistent CTAs walk row tiles, double-buffering the
// row operand through shared memory while the tensor core runs.  The
// accumulator lives in TMEM (BN columns) and is drained with tcgen05.ld
// into a fused epilogue (ReLU, or the ReLU'-mask times the incoming
// gradient).
//
// Kernel k_tc_wgrad (dW): both operands are MN-major (rows of agg and gz
// are read as-is), the reduction runs over chunk rows; each CTA owns a
// slice of rows and writes a partial 128 x BN tile, reduced afterwards in a
// fixed order.
//
// 3xTF32: x = hi + lo with hi = rna_tf32(x), lo = x - hi (exact), and
// a.b ~ hi.hi + hi.lo + lo.hi accumulated in FP32 in TMEM.
//
// Shared-memory layouts are the canonical SWIZZLE_128B UMMA layouts
// (cute/arch/mma_sm100_desc.hpp): 8-row x 128-byte atoms, 16-byte chunk
// index XOR (row & 7), 1024-byte aligned.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ht_common.h"

namespace ht {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor, SWIZZLE_128B, version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// instruction descriptor: A,B = TF32, D = F32, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

__host__ __device__ constexpr uint32_t tmem_cols(int n) {
  return n <= 32 ? 32u : n <= 64 ? 64u : n <= 128 ? 128u : 256u;
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// byte offset of 16-byte chunk c of row r inside a SWIZZLE_128B atom stack
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// four consecutive floats of a row, zero beyond `lim` (row-local count)
__device__ __forceinline__ float4 ld4(const float* __restrict__ p, int lim, bool vec_ok) {
  if (vec_ok && lim >= 4) return __ldg(reinterpret_cast<const float4*>(p));
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (lim > 0) v.x = __ldg(p);
  if (lim > 1) v.y = __ldg(p + 1);
  if (lim > 2) v.z = __ldg(p + 2);
  if (lim > 3) v.w = __ldg(p + 3);
  return v;
}

template <bool SPLIT>
__device__ __forceinline__ void put4(uint8_t* hi, uint8_t* lo, uint32_t off, float4 v) {
  float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
  *reinterpret_cast<float4*>(hi + off) = h;
  if (SPLIT) {
    float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
    *reinterpret_cast<float4*>(lo + off) = l;
  }
}

enum { TC_STORE = 0, TC_RELU = 1, TC_MASK = 2 };

// C[M x N] = A[M x K] . Bt[N x K]^T with epilogue; K <= 256.
// grid.x = feature tiles of BN, grid.y = persistent row-tile workers.
template <int BN, bool SPLIT, int EPI>
__global__ void __launch_bounds__(128, 1)
    k_tc_rows(const float* __restrict__ A, int64_t lda, int64_t M, int K,
              const float* __restrict__ Bt, int64_t ldb, int N, float* __restrict__ C,
              int64_t ldc, const float* __restrict__ G, int64_t ldg) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int KC = (K + 31) >> 5;
  constexpr int A_BYTES = 128 * 128;
  const uint32_t B_BYTES = (uint32_t)KC * BN * 128;
  uint8_t* bhi = smem;
  uint8_t* blo = bhi + B_BYTES;
  uint8_t* ast = SPLIT ? blo + B_BYTES : blo;
  constexpr int STAGE = (SPLIT ? 2 : 1) * A_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ast + 2 * STAGE);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int f0 = blockIdx.x * BN;
  constexpr uint32_t NCOL = tmem_cols(BN);
  if (warp == 0) tmem_alloc(slot, NCOL);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  // resident weight tile: rows f0..f0+BN-1 of Bt, all K
  const bool bvec = (ldb & 3) == 0;
  for (int idx = tid; idx < BN * KC * 8; idx += 128) {
    const int c = idx & 7, rest = idx >> 3, r = rest % BN, kc = rest / BN;
    const int f = f0 + r, k = kc * 32 + c * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (f < N) v = ld4(Bt + (int64_t)f * ldb + k, K - k, bvec);
    put4<SPLIT>(bhi, blo, (uint32_t)kc * BN * 128 + sw128(r, c), v);
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t idesc = idesc_tf32(BN, false, false);
  const bool avec = (lda & 3) == 0;
  const int64_t ntiles = (M + 127) >> 7;
  uint32_t phase0 = 0, phase1 = 0;
  bool pend0 = false, pend1 = false;
  int it = 0;
  for (int64_t t = blockIdx.y; t < ntiles; t += gridDim.y) {
    const int64_t m0 = t << 7;
    for (int kc = 0; kc < KC; ++kc, ++it) {
      const int s = it & 1;
      if (s == 0 && pend0) { mbar_wait(&bar[0], phase0); phase0 ^= 1; pend0 = false; }
      if (s == 1 && pend1) { mbar_wait(&bar[1], phase1); phase1 ^= 1; pend1 = false; }
      uint8_t* ahi = ast + s * STAGE;
      uint8_t* alo = ahi + A_BYTES;
#pragma unroll 4
      for (int idx = tid; idx < 128 * 8; idx += 128) {
        const int c = idx & 7, r = idx >> 3;
        const int64_t m = m0 + r;
        const int k = kc * 32 + c * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < M) v = ld4(A + m * lda + k, K - k, avec);
        put4<SPLIT>(ahi, alo, sw128(r, c), v);
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t a0 = smem_u32(ahi), b0 = smem_u32(bhi + (uint32_t)kc * BN * 128);
        const uint32_t al0 = smem_u32(alo), bl0 = smem_u32(blo + (uint32_t)kc * BN * 128);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t da = sdesc(a0 + ks * 32, 16, 1024);
          const uint64_t db = sdesc(b0 + ks * 32, 16, 1024);
          mma_tf32(tmem, da, db, idesc, (kc | ks) != 0);
          if (SPLIT) {
            mma_tf32(tmem, da, sdesc(bl0 + ks * 32, 16, 1024), idesc, 1);
            mma_tf32(tmem, sdesc(al0 + ks * 32, 16, 1024), db, idesc, 1);
          }
        }
        mma_commit(&bar[s]);
      }
      __syncwarp();
      if (s == 0) pend0 = true; else pend1 = true;
    }
    // drain: every MMA of this tile has completed once both stages are idle
    if (pend0) { mbar_wait(&bar[0], phase0); phase0 ^= 1; pend0 = false; }
    if (pend1) { mbar_wait(&bar[1], phase1); phase1 ^= 1; pend1 = false; }
    tc_fence_after();
    const int64_t m = m0 + warp * 32 + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
      if (m < M) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int f = f0 + c0 + q;
          if (f < N) {
            float x = v[q];
            if (EPI == TC_RELU) x = x > 0.f ? x : 0.f;
            if (EPI == TC_MASK) x = x > 0.f ? G[m * ldg + f] : 0.f;
            C[m * ldc + f] = x;
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, NCOL);
}

// Partial dW tiles: P[z][k][n] = sum over rows m of slice z of A[m][k] G[m][n].
// grid.x = k tiles of 128, grid.y = n tiles of BN, grid.z = row slices.
// Both operands MN-major: each staged row is 128 bytes of 32 features.
template <int BN>
__global__ void __launch_bounds__(128, 1)
    k_tc_wgrad(const float* __restrict__ A, int64_t lda, int K, const float* __restrict__ Gm,
               int64_t ldg, int N, int64_t M, int64_t rows_per_slice, float* __restrict__ P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int ROWS = 32;                       // reduction rows per stage
  constexpr int A_BYTES = 4 * ROWS * 128;        // 128 features = 4 atoms
  constexpr int B_BYTES = (BN / 32) * ROWS * 128;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int NST = 3;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + NST);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k0 = blockIdx.x * 128, n0 = blockIdx.y * BN;
  const int64_t r0 = (int64_t)blockIdx.z * rows_per_slice;
  const int64_t r1 = min(M, r0 + rows_per_slice);
  constexpr uint32_t NCOL = tmem_cols(BN);
  if (warp == 0) tmem_alloc(slot, NCOL);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  // K-major operands: MN-major TF32 operands read back as zeros on sm_100a
  // (measured), so tiles are transposed while staging instead
  const uint32_t idesc = idesc_tf32(BN, false, false);
  const bool avec = (lda & 3) == 0, gvec = (ldg & 3) == 0;
  uint32_t phase[NST] = {0, 0, 0};
  bool pend[NST] = {false, false, false};
  int it = 0;
  bool any = false;
  for (int64_t rb = r0; rb < r1; rb += ROWS, ++it) {
    const int s = it % NST;
    if (pend[s]) { mbar_wait(&bar[s], phase[s]); phase[s] ^= 1; pend[s] = false; }
    uint8_t* sa = smem + s * STAGE;
    uint8_t* sb = sa + A_BYTES;
    // Transposing loads into K-major tiles (feature rows, 32 reduction
    // values per 128-byte row): lane = reduction row, so each warp store
    // fills one swizzled 128-byte smem row without bank conflicts.
    for (int idx = tid; idx < ROWS * 32; idx += 128) {
      const int r = idx & 31, fc = idx >> 5;
      const int64_t m = rb + r;
      const int k = k0 + fc * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < r1 && k < K) v = ld4(A + m * lda + k, K - k, avec);
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float*>(sa + sw128(fc * 4 + q, r >> 2) + (r & 3) * 4) = tf32_rna(e[q]);
    }
    for (int idx = tid; idx < ROWS * (BN / 4); idx += 128) {
      const int r = idx & 31, fc = idx >> 5;
      const int64_t m = rb + r;
      const int n = n0 + fc * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < r1 && n < N) v = ld4(Gm + m * ldg + n, N - n, gvec);
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float*>(sb + sw128(fc * 4 + q, r >> 2) + (r & 3) * 4) = tf32_rna(e[q]);
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
#pragma unroll
      for (int ks = 0; ks < ROWS / 8; ++ks) {
        mma_tf32(tmem, sdesc(a0 + ks * 32, 16, 1024), sdesc(b0 + ks * 32, 16, 1024), idesc,
                 (any || ks) ? 1u : 0u);
      }
      mma_commit(&bar[s]);
    }
    __syncwarp();
    pend[s] = true;
    any = true;
  }
  for (int s = 0; s < NST; ++s)
    if (pend[s]) { mbar_wait(&bar[s], phase[s]); phase[s] ^= 1; pend[s] = false; }
  tc_fence_after();
  const int k = k0 + warp * 32 + lane;
  float* out = P + (int64_t)blockIdx.z * K * N;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    if (k < K) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int n = n0 + c0 + q;
        if (n < N) out[(int64_t)k * N + n] = any ? v[q] : 0.f;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, NCOL);
}

}  // namespace tc
}  // namespace ht

// ===========================================================================
// host-side launchers
// ===========================================================================
namespace ht {
namespace tc {

inline size_t rows_smem(int bn, bool split, int K) {
  const size_t kc = (size_t)(K + 31) / 32;
  return 1024 + kc * bn * 128 * (split ? 2 : 1) + 2 * 128 * 128 * (split ? 2 : 1) + 64;
}

template <int BN, bool SPLIT, int EPI>
int launch_rows_t(cudaStream_t s, const float* A, int64_t lda, int64_t M, int K, const float* Bt,
                  int64_t ldb, int N, float* C, int64_t ldc, const float* G, int64_t ldg) {
  const size_t smem = rows_smem(BN, SPLIT, K);
  auto kern = k_tc_rows<BN, SPLIT, EPI>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(HT_ECUDA, "tc smem attribute: %s", cudaGetErrorString(e));
  const int gx = (N + BN - 1) / BN;
  const int64_t ntiles = (M + 127) / 128;
  const int per_sm = smem <= 110 * 1024 ? 2 : 1;
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)148 * per_sm / gx));
  kern<<<dim3(gx, (unsigned)gy), 128, smem, s>>>(A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HT_ECUDA, "k_tc_rows launch: %s", cudaGetErrorString(e));
  return HT_OK;
}

// C = epi(A[M x K] . Bt[N x K]^T); split = 3xTF32
template <int EPI>
int rows(cudaStream_t s, bool split, const float* A, int64_t lda, int64_t M, int K,
         const float* Bt, int64_t ldb, int N, float* C, int64_t ldc, const float* G, int64_t ldg) {
  if (M <= 0 || N <= 0) return HT_OK;
  if (K > 256 || K < 1) return fail(HT_EINVAL, "tcgen05 GEMM supports 1 <= K <= 256 (got %d)", K);
  if (split) {
    if (N <= 16) return launch_rows_t<16, true, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
    if (N <= 32) return launch_rows_t<32, true, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
    if (N <= 48) return launch_rows_t<48, true, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
    return launch_rows_t<64, true, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
  }
  if (N <= 16) return launch_rows_t<16, false, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
  if (N <= 32) return launch_rows_t<32, false, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
  if (N <= 48) return launch_rows_t<48, false, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
  if (N <= 64) return launch_rows_t<64, false, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
  return launch_rows_t<128, false, EPI>(s, A, lda, M, K, Bt, ldb, N, C, ldc, G, ldg);
}

inline size_t wgrad_smem(int bn) { return 1024 + 3 * (size_t)(4 * 32 * 128 + (bn / 32) * 32 * 128) + 64; }

template <int BN>
int launch_wgrad_t(cudaStream_t s, const float* A, int64_t lda, int K, const float* G, int64_t ldg,
                   int N, int64_t M, int splits, int64_t rps, float* P) {
  const size_t smem = wgrad_smem(BN);
  auto kern = k_tc_wgrad<BN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(HT_ECUDA, "tc smem attribute: %s", cudaGetErrorString(e));
  dim3 grid((unsigned)((K + 127) / 128), (unsigned)((N + BN - 1) / BN), (unsigned)splits);
  kern<<<grid, 128, smem, s>>>(A, lda, K, G, ldg, N, M, rps, P);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HT_ECUDA, "k_tc_wgrad launch: %s", cudaGetErrorString(e));
  return HT_OK;
}

// P[z] = partial A^T G over row slice z; returns the number of slices used.
inline int wgrad(cudaStream_t s, const float* A, int64_t lda, int K, const float* G, int64_t ldg,
                 int N, int64_t M, int max_splits, float* P, int* splits_out) {
  if (K > 256 || N > 256) return fail(HT_EINVAL, "tcgen05 wgrad supports K, N <= 256");
  const int gx = (K + 127) / 128;
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>((M + 31) / 32, 148 / gx));
  splits = std::min(splits, max_splits);
  int64_t rps = ((M + splits - 1) / splits + 31) / 32 * 32;
  if (rps < 32) rps = 32;
  splits = (int)std::max<int64_t>(1, (M + rps - 1) / rps);
  *splits_out = splits;
  if (N <= 32) return launch_wgrad_t<32>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
  if (N <= 64) return launch_wgrad_t<64>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
  if (N <= 128) return launch_wgrad_t<128>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
  if (N <= 192) return launch_wgrad_t<192>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
  return launch_wgrad_t<256>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
}

}  // namespace tc
}  // namespace ht
