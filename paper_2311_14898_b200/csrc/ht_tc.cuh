// tcgen05 (5th-generation tensor core) TF32 GEMMs of the dense transform.
//
// Shapes of the GCN layer (M = destination rows of a chunk, up to millions;
// d_in, d_out <= 256):
//   z    = agg . W          (forward K4 and backward recompute; 3xTF32)
//   gagg = gz . W^T         (backward K7; 1xTF32)
//   dW  += agg^T . gz       (backward K7; 1xTF32, split over rows)
//
// k_tc_gemm (z, gz, gagg) - persistent, warp-specialized, one CTA per SM:
//   warp 0     TMA producer: 128-row x 32-float tiles of the row operand and
//              BN x 32 tiles of the (pre-split) weight operand per stage
//   warps 2-3  converters: round the row tile to TF32 in place (hi) and
//              write the residual (lo) for 3xTF32
//   warp 1     MMA issuer: tcgen05.mma kind::tf32, M=128, N=BN, K=8;
//              3xTF32 = hi.hi + hi.lo + lo.hi into one TMEM accumulator
//   warps 4-7  epilogue: tcgen05.ld, fused ReLU / ReLU'-mask, stores
//   Two TMEM accumulators (2 x BN columns) let the epilogue of tile t
//   overlap the MMAs of tile t+1.
//
// k_tc_wgrad (dW) - one CTA per row slice: both operands read MN-major
// straight from the row-major matrices (TMA SWIZZLE_128B_ATOM_32B boxes),
// rounded to TF32 in place, all of K x N accumulated in TMEM; the slices'
// partial tiles are reduced in a fixed order afterwards.
//
// Shared-memory operand layouts are the canonical SWIZZLE_128B K-major UMMA
// layouts (cute/arch/mma_sm100_desc.hpp): 8-row x 128-byte atoms, 16-byte
// chunk index XOR (row & 7), 1024-byte aligned; TMA writes exactly this
// layout with CU_TENSOR_MAP_SWIZZLE_128B.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ht_common.h"

namespace ht {
namespace tc {

// ---------------------------------------------------------------------------
// PTX primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B, version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;             // LBO 16 B (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO: 8-row groups 1024 B apart
  d |= (uint64_t)1 << 46;             // version
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

// instruction descriptor: A,B = TF32 (K-major), D = F32, M = m (128, or
// 256 for a CTA pair), N = n
__host__ __device__ constexpr uint32_t idesc_tf32(int n, int m = 128) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__host__ __device__ constexpr uint32_t tmem_cols(int n) {
  return n <= 32 ? 32u : n <= 64 ? 64u : n <= 128 ? 128u : n <= 256 ? 256u : 512u;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// CTA pair (cta_group::2, issued by the leader CTA): A rows split across the
// pair (each CTA's smem holds its 128 rows), B columns split (each holds
// N/2), D rows in each CTA's own TMEM lanes
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// the pair's MMAs done -> arrive on the barrier at this offset in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
// shared::cluster address of the same barrier in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_bar(uint64_t* bar, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(bar)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// wait with cluster-scope acquire (arrivals come from the peer CTA too)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
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

// wait until the phase with the given parity has completed
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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// shared -> global tensor store (TMA), bulk-group completion
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
      "r"(smem_u32(src)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
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

enum { TC_STORE = 0, TC_RELU = 1, TC_MASK = 2 };

// ---------------------------------------------------------------------------
// k_tc_gemm: C[M x N] = epi(A[M x K] . B^T), B given as hi/lo halves of a
// K-major N x K matrix (tensor maps tmBh / tmBl); A through tmA (row-major,
// lda*4 bytes per row).  BN >= N, multiple of 32.
// ---------------------------------------------------------------------------
// AM (masked-A, 1xTF32 only): the A operand is g * (h > 0) - TMA brings
// the g and h tiles (h in the A-lo slot), the converters mask and round in
// place, and one converter thread stores the masked tile to Z by TMA (the
// ReLU'-mask of the GCN backward folded into the gz . W^T GEMM: gz is
// written once here instead of by a separate read-g-read-h-write-gz pass).
// PAIR: a CTA pair (cluster of 2, cta_group::2) computes 256-row tiles with
// M = 256 MMAs; each CTA stages its 128 A rows and half of B's BN rows.
template <int BN, bool SPLIT, bool AM = false, bool PAIR = false>
struct GemmCfg {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * 128;
  static constexpr int STAGE = ((SPLIT || AM) ? 2 : 1) * A_BYTES + (SPLIT ? 2 : 1) * B_BYTES;
  static constexpr int STAGES = (200 * 1024 / STAGE) < 4 ? (200 * 1024 / STAGE) : 4;
  static constexpr int TX = (AM ? 2 : 1) * A_BYTES + (SPLIT ? 2 : 1) * B_BYTES;  // TMA bytes per stage
  // epilogue staging: per warp two 32 x 32 swizzled tiles for the TMA
  // stores (or one padded 32 x 33 transpose tile on the scalar-store path)
  static constexpr int EPI_BYTES = 4 * 2 * 32 * 32 * 4;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE + EPI_BYTES + 256;
};

template <int BN, bool SPLIT, int EPI, bool AM = false, bool PAIR = false>
__global__ void __launch_bounds__(256, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
              const __grid_constant__ CUtensorMap tmBl, const __grid_constant__ CUtensorMap tmC,
              const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmZ,
              int tma_store, int64_t M, int K, int N, float* __restrict__ C, int64_t ldc,
              const float* __restrict__ G, int64_t ldg) {
  static_assert(!(AM && SPLIT), "masked A is a 1xTF32 operand");
  static_assert(!(AM && PAIR), "masked A runs on single CTAs");
  using Cfg = GemmCfg<BN, SPLIT, AM, PAIR>;
  constexpr int ST = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // stage s: [A hi (raw)][A lo | h tile (AM)][B hi][B lo]
  auto sA = [&](int s) { return smem + (size_t)s * Cfg::STAGE; };
  auto sAlo = [&](int s) { return sA(s) + Cfg::A_BYTES; };
  auto sBh = [&](int s) { return sA(s) + ((SPLIT || AM) ? 2 : 1) * Cfg::A_BYTES; };
  auto sBl = [&](int s) { return sBh(s) + Cfg::B_BYTES; };
  uint8_t* epi = smem + (size_t)ST * Cfg::STAGE;  // 1024-aligned
  uint64_t* bar = reinterpret_cast<uint64_t*>(epi + Cfg::EPI_BYTES);
  uint64_t* full = bar;            // [ST] TMA landed
  uint64_t* conv = bar + ST;       // [ST] converters done
  uint64_t* empty = bar + 2 * ST;  // [ST] MMAs done reading
  uint64_t* tfull = bar + 3 * ST;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;    // [2] accumulator drained
  uint32_t* slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t NCOL = tmem_cols(2 * BN);
  // PAIR: rank 0 (the leader) issues the MMAs; its conv / tempty barriers
  // also count the peer's converters / epilogue warps (remote arrivals)
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  constexpr int TM = PAIR ? 256 : 128;  // rows per tile
  const int64_t first = PAIR ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
  const int64_t step = PAIR ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair(slot, NCOL);
    else tmem_alloc(slot, NCOL);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], PAIR ? 128 : 64);
      mbar_init(&empty[s], AM ? 2 : 1);  // (AM: + the Z store has read the stage)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 8 : 4);  // one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const int KC = (K + 31) >> 5;
  const int64_t ntiles = (M + TM - 1) / TM;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      int it = 0;
      const int brow = PAIR ? (int)rank * (BN / 2) : 0;  // this CTA's half of B
      for (int64_t t = first; t < ntiles; t += step)
        for (int kc = 0; kc < KC; ++kc, ++it) {
          const int s = it % ST;
          const int arow = (int)(t * TM) + (int)rank * 128;
          mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
          mbar_expect_tx(&full[s], Cfg::TX);
          tma_load_2d(sA(s), &tmA, &full[s], kc * 32, arow);
          if (AM) tma_load_2d(sAlo(s), &tmH, &full[s], kc * 32, arow);
          tma_load_2d(sBh(s), &tmBh, &full[s], kc * 32, brow);
          if (SPLIT) tma_load_2d(sBl(s), &tmBl, &full[s], kc * 32, brow);
        }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer ----------------
      const uint32_t idesc = idesc_tf32(BN, TM);
      int it = 0, acc = 0;
      for (int64_t t = first; t < ntiles; t += step, ++acc) {
        const int a = acc & 1;
        if (PAIR) mbar_wait_cluster(&tempty[a], ((acc >> 1) & 1) ^ 1);
        else mbar_wait(&tempty[a], ((acc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(a * BN);
        for (int kc = 0; kc < KC; ++kc, ++it) {
          const int s = it % ST;
          if (PAIR) mbar_wait_cluster(&conv[s], (it / ST) & 1);
          else mbar_wait(&conv[s], (it / ST) & 1);
          tc_fence_after();
          const uint32_t ah = smem_u32(sA(s)), al = smem_u32(sAlo(s));
          const uint32_t bh = smem_u32(sBh(s)), bl = smem_u32(sBl(s));
          // K-tail chunk: only the 8-wide k-steps that hold real columns
          // (K = 100: 13 of 16 steps; the zero-filled rest is skipped)
          const int nks = min(4, (K - kc * 32 + 7) >> 3);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            if (ks >= nks) break;
            const uint64_t dah = sdesc(ah + ks * 32), dbh = sdesc(bh + ks * 32);
            if (PAIR) {
              mma_tf32_pair(d, dah, dbh, idesc, (kc | ks) != 0);
              if (SPLIT) {
                mma_tf32_pair(d, dah, sdesc(bl + ks * 32), idesc, 1);
                mma_tf32_pair(d, sdesc(al + ks * 32), dbh, idesc, 1);
              }
            } else {
              mma_tf32(d, dah, dbh, idesc, (kc | ks) != 0);
              if (SPLIT) {
                mma_tf32(d, dah, sdesc(bl + ks * 32), idesc, 1);
                mma_tf32(d, sdesc(al + ks * 32), dbh, idesc, 1);
              }
            }
          }
          if (PAIR) mma_commit_pair(&empty[s]);
          else mma_commit(&empty[s]);
        }
        if (PAIR) mma_commit_pair(&tfull[a]);
        else mma_commit(&tfull[a]);
      }
    }
  } else if (warp < 4) {  // ---------------- converters (64 threads) ----------------
    const int ct = threadIdx.x - 64;
    const uint32_t conv0 = PAIR ? peer_bar(conv, 0) : 0;  // the leader's conv[0]
    int it = 0;
    for (int64_t t = first; t < ntiles; t += step)
      for (int kc = 0; kc < KC; ++kc, ++it) {
        const int s = it % ST;
        mbar_wait(&full[s], (it / ST) & 1);
        float4* hi = reinterpret_cast<float4*>(sA(s));
        float4* lo = reinterpret_cast<float4*>(sAlo(s));
#pragma unroll 4
        for (int q = ct; q < Cfg::A_BYTES / 16; q += 64) {
          float4 v = hi[q];
          if (AM) {  // gz = g * (h > 0) (same swizzled position in both tiles)
            const float4 m = lo[q];
            v = make_float4(m.x > 0.f ? v.x : 0.f, m.y > 0.f ? v.y : 0.f, m.z > 0.f ? v.z : 0.f,
                            m.w > 0.f ? v.w : 0.f);
          }
          const float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
          hi[q] = h;
          if (SPLIT) lo[q] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
        fence_proxy_async();
        if (PAIR) mbar_arrive_cluster(conv0 + (uint32_t)s * 8u);
        else mbar_arrive(&conv[s]);
        if (AM && ct == 0) {
          // every converter's writes are in (conv phase complete): the
          // rounded gz tile leaves by TMA (RNA rounding is idempotent, so
          // k_tc_wgrad's own rounding of it is unchanged); the stage is
          // released to the producer once the store has read it (lagging
          // one stage so the wait rarely blocks)
          mbar_wait(&conv[s], (it / ST) & 1);
          tma_store_2d(&tmZ, sA(s), kc * 32, (int)(t * 128));
          bulk_commit();
          if (it > 0) {
            bulk_wait_read<1>();
            mbar_arrive(&empty[(it - 1) % ST]);
          }
        }
      }
    if (AM && ct == 0) {
      if (it > 0) {
        bulk_wait_read<0>();
        mbar_arrive(&empty[(it - 1) % ST]);
      }
      bulk_wait_all();
    }
  } else if (tma_store) {  // ---------------- epilogue (warps 4-7), TMA stores ----------------
    // TMEM gives a thread one row; each 32-column block goes to a 32 x 32
    // SWIZZLE_128B smem tile (16-byte chunk j of row r at j ^ (r & 7):
    // conflict-free float4 writes) and leaves with one TMA tensor store per
    // warp; two tiles per warp so the next block is written while the
    // previous store drains.  Rows >= M and columns >= N are clipped by TMA.
    const int q4 = warp & 3;  // TMEM lane quarter this warp may access
    float* tiles = reinterpret_cast<float*>(epi) + q4 * 2 * 32 * 32;
    const bool g4 = (ldg & 3) == 0 && ((uintptr_t)G & 15) == 0;
    const uint32_t tempty0 = PAIR ? peer_bar(tempty, 0) : 0;
    int acc = 0, buf = 0;
    for (int64_t t = first; t < ntiles; t += step, ++acc) {
      const int a = acc & 1;
      mbar_wait(&tfull[a], (acc >> 1) & 1);
      tc_fence_after();
      const int64_t r0 = t * TM + rank * 128 + q4 * 32;
      const uint32_t base = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(a * BN);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        if (c0 >= N) break;
        float g[32];
        if (EPI == TC_MASK) {  // this thread's row of the incoming gradient
          const int64_t m = r0 + lane;
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (m < M) {
              if (c0 + q + 3 < N && g4) {
                v = __ldg(reinterpret_cast<const float4*>(G + m * ldg + c0 + q));
              } else {
                v.x = c0 + q < N ? __ldg(G + m * ldg + c0 + q) : 0.f;
                v.y = c0 + q + 1 < N ? __ldg(G + m * ldg + c0 + q + 1) : 0.f;
                v.z = c0 + q + 2 < N ? __ldg(G + m * ldg + c0 + q + 2) : 0.f;
                v.w = c0 + q + 3 < N ? __ldg(G + m * ldg + c0 + q + 3) : 0.f;
              }
            }
            g[q] = v.x; g[q + 1] = v.y; g[q + 2] = v.z; g[q + 3] = v.w;
          }
        }
        float v[32];
        tmem_ld32(base + (uint32_t)c0, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          if (EPI == TC_RELU) v[q] = v[q] > 0.f ? v[q] : 0.f;
          if (EPI == TC_MASK) v[q] = v[q] > 0.f ? g[q] : 0.f;
        }
        if (lane == 0) bulk_wait_read<1>();  // the store that used this tile has read it
        __syncwarp();
        float* tile = tiles + buf * 32 * 32;
        uint8_t* row = reinterpret_cast<uint8_t*>(tile) + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(row + ((j ^ (lane & 7)) << 4)) =
              make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmC, tile, c0, (int)r0);
          bulk_commit();
        }
        buf ^= 1;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_cluster(tempty0 + (uint32_t)a * 8u);
        else mbar_arrive(&tempty[a]);
      }
    }
    if (lane == 0) bulk_wait_all();
  } else {  // ---------------- epilogue (warps 4-7), scalar stores ----------------
    // (C rows not 16-byte aligned, e.g. a 47-wide last layer) a padded 32x32
    // smem transpose turns a thread's row into row-contiguous 128-byte
    // stores (and G loads) per warp instruction
    const int q4 = warp & 3;  // TMEM lane quarter this warp may access
    float* tile = reinterpret_cast<float*>(epi) + q4 * 32 * 33;
    const uint32_t tempty0 = PAIR ? peer_bar(tempty, 0) : 0;
    int acc = 0;
    for (int64_t t = first; t < ntiles; t += step, ++acc) {
      const int a = acc & 1;
      mbar_wait(&tfull[a], (acc >> 1) & 1);
      tc_fence_after();
      const int64_t r0 = t * TM + rank * 128 + q4 * 32;
      const uint32_t base = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(a * BN);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        // the mask epilogue's incoming-gradient block is fetched before the
        // accumulator so its 32 independent row loads overlap (one
        // 128-byte coalesced load per row per warp)
        float g[32];
        if (EPI == TC_MASK) {
          const int colg = c0 + lane;
#pragma unroll
          for (int r = 0; r < 32; ++r)
            g[r] = (r0 + r < M && colg < N) ? __ldg(G + (r0 + r) * ldg + colg) : 0.f;
        }
        float v[32];
        tmem_ld32(base + (uint32_t)c0, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) tile[lane * 33 + q] = v[q];
        __syncwarp();
        const int col = c0 + lane;
        if (c0 < N) {
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const int64_t m = r0 + r;
            float x = tile[r * 33 + lane];
            if (m < M && col < N) {
              if (EPI == TC_RELU) x = x > 0.f ? x : 0.f;
              if (EPI == TC_MASK) x = x > 0.f ? g[r] : 0.f;
              C[m * ldc + col] = x;
            }
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_cluster(tempty0 + (uint32_t)a * 8u);
        else mbar_arrive(&tempty[a]);
      }
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync();  // (the leader's MMAs read the peer's smem / TMEM)
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_pair(tmem, NCOL);
    else tmem_dealloc(tmem, NCOL);
  }
}

// ---------------------------------------------------------------------------
// k_tc_wgrad: P[z][k][n] = sum_{m in slice z} A[m][k] G[m][n] for all
// k < K <= 256, n < N <= 256 in one CTA per row slice (grid = slices).
//
// Both operands are consumed MN-major straight from their row-major HBM
// layout: A^T (features k x rows m) has k contiguous, so a TMA box of 32
// features x 32 rows lands as 32 rows of 128 B - the UMMA MN-major
// SWIZZLE_128B_BASE32B canonical layout (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
// the only MN-major smem layout for TF32, cutlass sm100_common.inl).  Each
// 32-feature block is one box; LBO = block stride (4 KB), SBO = 4-row group
// stride (512 B); one K=8 MMA step covers 8 rows (1 KB).  KT = ceil(K/128)
// accumulators of 128 x BN in TMEM (KT * BN <= 512 columns).
//   warp 0     TMA producer (KT*4 + BN/32 boxes per stage, in-bounds only)
//   warps 2-7  round the landed stage to TF32 in place (RNA; the tensor core
//              would truncate - a systematic 2^-11 bias per operand)
//   warp 1     MMA issuer
//   warps 4-7  epilogue: TMEM -> the slice's partial tile
// ---------------------------------------------------------------------------
template <int KT, int BN>
struct WgradCfg {
  static constexpr int R = 32;                       // reduction rows per stage
  static constexpr int BOX = 32 * R * 4;             // one 32-feature x R-row box
  static constexpr int ABYTES = KT * 4 * BOX;
  static constexpr int GBYTES = (BN / 32) * BOX;
  static constexpr int STAGE = ABYTES + GBYTES;
  static constexpr int S0 = (200 * 1024) / STAGE;
  static constexpr int STAGES = S0 > 6 ? 6 : S0;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE + 256;
};

// UMMA shared-memory descriptor, MN-major SWIZZLE_128B_BASE32B, version 1
__device__ __forceinline__ uint64_t sdesc_mn32(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;  // MN block stride
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;  // 4-row K group stride
  d |= (uint64_t)1 << 46;                       // version
  d |= (uint64_t)1 << 61;                       // SWIZZLE_128B_BASE32B
  return d;
}

// instruction descriptor: A,B = TF32 MN-major, D = F32, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_tf32_mn(int n) {
  return idesc_tf32(n) | (1u << 15) | (1u << 16);
}

template <int KT, int BN>
__global__ void __launch_bounds__(256, 1)
    k_tc_wgrad(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmG,
               int K, int N, int64_t M, int64_t rows_per_slice, float* __restrict__ P) {
  using Cfg = WgradCfg<KT, BN>;
  constexpr int ST = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + ST * Cfg::STAGE);
  uint64_t* full = bar;            // [ST] TMA landed
  uint64_t* conv = bar + ST;       // [ST] rounded in place
  uint64_t* empty = bar + 2 * ST;  // [ST] MMAs done
  uint64_t* accf = bar + 3 * ST;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 3 * ST + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_slice;
  const int64_t r1 = min(M, r0 + rows_per_slice);
  const int nst = r1 > r0 ? (int)((r1 - r0 + Cfg::R - 1) / Cfg::R) : 0;
  constexpr uint32_t NCOL = tmem_cols(KT * BN);
  if (warp == 1) tmem_alloc(slot, NCOL);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 192);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    if (lane == 0) {  // TMA producer: only boxes that start inside the matrix
      const int na = (K + 31) / 32, ng = (N + 31) / 32;
      const uint32_t tx = (uint32_t)(na + ng) * Cfg::BOX;
      for (int it = 0; it < nst; ++it) {
        const int s = it % ST;
        mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
        mbar_expect_tx(&full[s], tx);
        uint8_t* st = smem + s * Cfg::STAGE;
        const int row = (int)(r0 + (int64_t)it * Cfg::R);
        for (int b = 0; b < na; ++b) tma_load_2d(st + b * Cfg::BOX, &tmA, &full[s], b * 32, row);
        for (int b = 0; b < ng; ++b)
          tma_load_2d(st + Cfg::ABYTES + b * Cfg::BOX, &tmG, &full[s], b * 32, row);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = idesc_tf32_mn(BN);
      for (int it = 0; it < nst; ++it) {
        const int s = it % ST;
        mbar_wait(&conv[s], (it / ST) & 1);
        tc_fence_after();
        const uint32_t a = smem_u32(smem + s * Cfg::STAGE), g = a + Cfg::ABYTES;
#pragma unroll
        for (int t = 0; t < KT; ++t)
#pragma unroll
          for (int ks = 0; ks < Cfg::R / 8; ++ks)
            mma_tf32(tmem + (uint32_t)(t * BN),
                     sdesc_mn32(a + t * 4 * Cfg::BOX + ks * 1024, Cfg::BOX, 512),
                     sdesc_mn32(g + ks * 1024, Cfg::BOX, 512), idesc, (it | ks) != 0);
        mma_commit(&empty[s]);
      }
      mma_commit(accf);
    }
  } else {  // converters (warps 2-7, 192 threads); epilogue on warps 4-7
    const int tt = threadIdx.x - 64;
    for (int it = 0; it < nst; ++it) {
      const int s = it % ST;
      mbar_wait(&full[s], (it / ST) & 1);
      float4* st = reinterpret_cast<float4*>(smem + s * Cfg::STAGE);
#pragma unroll 4
      for (int w = tt; w < Cfg::STAGE / 16; w += 192) {
        float4 v = st[w];
        v.x = tf32_rna(v.x);
        v.y = tf32_rna(v.y);
        v.z = tf32_rna(v.z);
        v.w = tf32_rna(v.w);
        st[w] = v;
      }
      fence_proxy_async();
      mbar_arrive(&conv[s]);
    }
    if (warp >= 4) {  // epilogue: the KT accumulators -> the slice's partial tile
      const int q4 = warp & 3;
      float* out = P + (int64_t)blockIdx.x * K * N;
      if (nst > 0) {
        mbar_wait(accf, 0);
        tc_fence_after();
      }
#pragma unroll 1
      for (int t = 0; t < KT; ++t) {
        const int k = t * 128 + q4 * 32 + lane;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
          if (nst > 0)
            tmem_ld16(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(t * BN + c0), v);
          if (k < K) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = c0 + j;
              if (n < N) out[(int64_t)k * N + n] = nst > 0 ? v[j] : 0.f;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, NCOL);
  }
}

// W (rows x cols, ld) -> hi = rna_tf32(W), lo = W - hi (same layout)
static __global__ void k_split_tf32(const float* __restrict__ W, float* __restrict__ hi,
                             float* __restrict__ lo, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float h = tf32_rna(W[e]);
    hi[e] = h;
    lo[e] = W[e] - h;
  }
}

}  // namespace tc
}  // namespace ht

// ===========================================================================
// host-side launchers
// ===========================================================================
namespace ht {
namespace tc {

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D fp32 tensor map: inner dim `cols` (contiguous), outer `rows`, row
// stride `ld` floats; box = box_cols x box_rows.
inline int tmap(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld,
                int box_cols, int box_rows, bool swizzle,
                CUtensorMapSwizzle mode = CU_TENSOR_MAP_SWIZZLE_NONE) {
  auto fn = encode_fn();
  if (!fn) return fail(HT_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (((uintptr_t)base & 15) || (ld * 4) % 16)
    return fail(HT_EINVAL, "TMA operand needs 16-byte aligned base and row stride (ld=%lld)",
                (long long)ld);
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)std::max<int64_t>(rows, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : mode,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HT_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HT_OK;
}

inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool SPLIT, int EPI, bool AM = false, bool PAIR = false>
inline int launch_gemm_t(cudaStream_t s, const float* A, int64_t lda, int64_t M, int K, const float* Bh,
                  const float* Bl, int64_t ldb, int N, float* C, int64_t ldc, const float* G,
                  int64_t ldg, const float* Hm = nullptr, int64_t ldh = 0, float* Z = nullptr,
                  int64_t ldz = 0) {
  using Cfg = GemmCfg<BN, SPLIT, AM, PAIR>;
  constexpr int BR = PAIR ? BN / 2 : BN;  // B rows staged per CTA
  CUtensorMap ta, tbh, tbl, tc_, th, tz;
  HT_TRY(tmap(&ta, A, M, K, lda, 32, 128, true));
  if (AM) {  // h tiles like A's; Z is written ldz columns wide (zero pad columns)
    HT_TRY(tmap(&th, Hm, M, K, ldh, 32, 128, true));
    HT_TRY(tmap(&tz, Z, M, ldz, ldz, 32, 128, true));
  } else {
    th = ta;  // (unused)
    tz = ta;
  }
  HT_TRY(tmap(&tbh, Bh, N, K, ldb, 32, BR, true));
  HT_TRY(tmap(&tbl, SPLIT ? Bl : Bh, N, K, ldb, 32, BR, true));
  // TMA stores of the output when its rows are 16-byte aligned
  static const bool no_tma_store = [] {
    const char* e = getenv("HT_NO_TMA_STORE");
    return e && atoi(e);
  }();
  const int use_tma = !no_tma_store && ((uintptr_t)C & 15) == 0 && (ldc & 3) == 0;
  if (use_tma) HT_TRY(tmap(&tc_, C, M, N, ldc, 32, 32, true));
  else tc_ = ta;  // (unused)
  auto kern = k_tc_gemm<BN, SPLIT, EPI, AM, PAIR>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
  if (e != cudaSuccess) return fail(HT_ECUDA, "tc smem attribute: %s", cudaGetErrorString(e));
  if (PAIR) {  // persistent CTA pairs (clusters of 2: the two SMs of a TPC)
    const int64_t ntiles = (M + 255) / 256;
    const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, sm_count() / 2));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, ta, tbh, tbl, tc_, th, tz, use_tma, M, K, N, C, ldc, G, ldg);
    if (e != cudaSuccess) return fail(HT_ECUDA, "k_tc_gemm pair launch: %s", cudaGetErrorString(e));
    return HT_OK;
  }
  const int64_t ntiles = (M + 127) / 128;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, sm_count()));
  kern<<<grid, 256, Cfg::SMEM, s>>>(ta, tbh, tbl, tc_, th, tz, use_tma, M, K, N, C, ldc, G, ldg);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HT_ECUDA, "k_tc_gemm launch: %s", cudaGetErrorString(e));
  return HT_OK;
}

// C = epi(A[M x K] . B^T) with B = Bh (+ Bl) given K-major (N rows x K,
// row stride ldb); split = 3xTF32 (Bl required).
template <int EPI>
inline int rows(cudaStream_t s, bool split, const float* A, int64_t lda, int64_t M, int K,
         const float* Bh, const float* Bl, int64_t ldb, int N, float* C, int64_t ldc,
         const float* G, int64_t ldg) {
  if (M <= 0 || N <= 0) return HT_OK;
  if (K < 1 || N > 256) return fail(HT_EINVAL, "tcgen05 GEMM supports N <= 256 (got %d)", N);
  if (split) {
    // HT_PAIR=1: 3xTF32 with N > 128 on CTA pairs (M = 256 MMAs, half of B
    // per SM) - the 128 x 256 single-CTA tile is bound by shared-memory
    // bandwidth (three MMAs per k step each reading A and all of B).  The
    // pair kernel is faster alone (cfg 2, N = 256: 2.65 vs 2.89 ms for the
    // two launches, ncu) but the value epoch measured 0.3 ms slower with it
    // (42.5 vs 42.2 ms, three interleaved runs, sw_power_cap active), so
    // single CTAs are the default.  Narrower tiles are HBM-bound and the
    // pair handshake per stage costs more than it saves (N = 64: 1.38 vs
    // 0.81 ms), so pairs never apply to N <= 128.
    static const bool pair = [] {
      const char* e = getenv("HT_PAIR");
      return e && atoi(e);
    }();
    if (pair && N > 128)
      return launch_gemm_t<256, true, EPI, false, true>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
    if (N <= 32) return launch_gemm_t<32, true, EPI>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
    if (N <= 64) return launch_gemm_t<64, true, EPI>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
    if (N <= 128) return launch_gemm_t<128, true, EPI>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
    return launch_gemm_t<256, true, EPI>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
  }
  if (N <= 32) return launch_gemm_t<32, false, EPI>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
  if (N <= 64) return launch_gemm_t<64, false, EPI>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
  if (N <= 128) return launch_gemm_t<128, false, EPI>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
  return launch_gemm_t<256, false, EPI>(s, A, lda, M, K, Bh, Bl, ldb, N, C, ldc, G, ldg);
}

// C = (gz . B^T) with gz = G * (H > 0) formed in the GEMM and written to Z
// (ldz >= K columns, pad columns zero; TF32-rounded, RNA) - 1xTF32; G and H
// are M x K with row strides ldg / ldh.
inline int rows_masked(cudaStream_t s, const float* G, int64_t ldg, const float* Hm, int64_t ldh,
                       float* Z, int64_t ldz, int64_t M, int K, const float* Bh, int64_t ldb,
                       int N, float* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return HT_OK;
  if (K < 1 || N > 256 || ldz < K) return fail(HT_EINVAL, "masked tcgen05 GEMM: N <= 256, ldz >= K");
  if (N <= 32) return launch_gemm_t<32, false, TC_STORE, true>(s, G, ldg, M, K, Bh, nullptr, ldb, N, C, ldc, nullptr, 0, Hm, ldh, Z, ldz);
  if (N <= 64) return launch_gemm_t<64, false, TC_STORE, true>(s, G, ldg, M, K, Bh, nullptr, ldb, N, C, ldc, nullptr, 0, Hm, ldh, Z, ldz);
  if (N <= 128) return launch_gemm_t<128, false, TC_STORE, true>(s, G, ldg, M, K, Bh, nullptr, ldb, N, C, ldc, nullptr, 0, Hm, ldh, Z, ldz);
  return launch_gemm_t<256, false, TC_STORE, true>(s, G, ldg, M, K, Bh, nullptr, ldb, N, C, ldc, nullptr, 0, Hm, ldh, Z, ldz);
}

template <int KT, int BN>
inline int launch_wgrad_t(cudaStream_t s, const float* A, int64_t lda, int K, const float* G, int64_t ldg,
                   int N, int64_t M, int splits, int64_t rps, float* P) {
  using Cfg = WgradCfg<KT, BN>;
  CUtensorMap ta, tg;
  HT_TRY(tmap(&ta, A, M, K, lda, 32, Cfg::R, false, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B));
  HT_TRY(tmap(&tg, G, M, N, ldg, 32, Cfg::R, false, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B));
  auto kern = k_tc_wgrad<KT, BN>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
  if (e != cudaSuccess) return fail(HT_ECUDA, "tc smem attribute: %s", cudaGetErrorString(e));
  kern<<<(unsigned)splits, 256, Cfg::SMEM, s>>>(ta, tg, K, N, M, rps, P);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HT_ECUDA, "k_tc_wgrad launch: %s", cudaGetErrorString(e));
  return HT_OK;
}

template <int KT>
inline int wgrad_kt(cudaStream_t s, const float* A, int64_t lda, int K, const float* G, int64_t ldg,
             int N, int64_t M, int splits, int64_t rps, float* P) {
  if (N <= 32) return launch_wgrad_t<KT, 32>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
  if (N <= 64) return launch_wgrad_t<KT, 64>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
  if (N <= 128) return launch_wgrad_t<KT, 128>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
  return launch_wgrad_t<KT, 256>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
}

// P[z] = partial A^T G over row slice z (one CTA per slice, up to one per
// SM); *splits_out = number of slices.
inline int wgrad(cudaStream_t s, const float* A, int64_t lda, int K, const float* G, int64_t ldg,
                 int N, int64_t M, int max_splits, float* P, int* splits_out) {
  if (K > 256 || N > 256) return fail(HT_EINVAL, "tcgen05 wgrad supports K, N <= 256");
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>((M + 31) / 32, sm_count()));
  splits = std::max(1, std::min(splits, max_splits));
  int64_t rps = ((M + splits - 1) / splits + 31) / 32 * 32;
  if (rps < 32) rps = 32;
  splits = (int)std::max<int64_t>(1, (M + rps - 1) / rps);
  *splits_out = splits;
  if (K <= 128) return wgrad_kt<1>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
  return wgrad_kt<2>(s, A, lda, K, G, ldg, N, M, splits, rps, P);
}

inline int split_weights(cudaStream_t s, const float* W, float* hi, float* lo, int64_t n) {
  k_split_tf32<<<(int)std::min<int64_t>(1024, (n + 255) / 256), 256, 0, s>>>(W, hi, lo, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HT_ECUDA, "k_split_tf32: %s", cudaGetErrorString(e));
  return HT_OK;
}

}  // namespace tc
}  // namespace ht
