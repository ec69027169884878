// parametrized MN-major tcgen05 debug: one CTA, M=128 (features), N=128, 32 reduction rows
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2311_14898_b200/csrc/ht_common.h"
namespace ht { std::string& last_error() { static std::string s; return s; } }
#include "../paper_2311_14898_b200/csrc/ht_tc.cuh"
using namespace ht::tc;

__global__ void kdbg(const float* A, const float* G, float* P, int lbo, int sbo, int amn, int bmn, int kmajor_mode) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = smem; uint8_t* sb = smem + 16384;
  uint64_t* bar = (uint64_t*)(smem + 32768); uint32_t* slot = (uint32_t*)(bar + 1);
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc(slot, 128);
  if (tid == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  // A: 32 rows (m) x 128 features (k), row-major ld 128.  B: 32 rows x 128 (n)
  if (!kmajor_mode) {
    for (int idx = tid; idx < 32 * 32; idx += 128) {
      int c = idx & 7, atom = (idx >> 3) & 3, r = idx >> 5;
      float4 v = *(const float4*)(A + r * 128 + atom * 32 + c * 4);
      float4 w = *(const float4*)(G + r * 128 + atom * 32 + c * 4);
      *(float4*)(sa + atom * 4096 + sw128(r, c)) = v;
      *(float4*)(sb + atom * 4096 + sw128(r, c)) = w;
    }
  } else {
    // K-major transposed: row = feature (128 rows), 32 reduction values per row
    for (int idx = tid; idx < 128 * 32; idx += 128) {
      int f = idx & 127, m = idx >> 7;
      float v = A[m * 128 + f], w = G[m * 128 + f];
      uint32_t off = sw128(f, m >> 2) + (m & 3) * 4;
      *(float*)(sa + off) = v; *(float*)(sb + off) = w;
    }
  }
  fence_proxy_async(); tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = *slot;
  if (tid == 0) {
    uint32_t idesc = idesc_tf32(128, amn, bmn);
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t step = kmajor_mode ? 32 : 1024;
      mma_tf32(tmem, sdesc(smem_u32(sa) + ks * step, lbo, sbo), sdesc(smem_u32(sb) + ks * step, lbo, sbo), idesc, ks > 0);
    }
    mma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 128; c0 += 16) {
    float v[16]; tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int q = 0; q < 16; ++q) P[(warp * 32 + lane) * 128 + c0 + q] = v[q];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
}

int main() {
  const int M = 32, K = 128, N = 128;
  std::vector<float> A(M * K), G(M * N), P(K * N);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 37) % 11) - 5;
  for (int i = 0; i < M * N; ++i) G[i] = (float)((i * 13) % 7) - 3;
  std::vector<double> R(K * N);
  for (int k = 0; k < K; ++k) for (int n = 0; n < N; ++n) { double r = 0; for (int m = 0; m < M; ++m) r += (double)A[m*K+k]*G[m*N+n]; R[k*N+n] = r; }
  float *dA, *dG, *dP;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dG, G.size() * 4); cudaMalloc(&dP, P.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kdbg, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  struct V { int lbo, sbo, amn, bmn, km; const char* name; } vs[] = {
    {4096, 1024, 1, 1, 0, "MN lbo4096 sbo1024"},
    {1024, 4096, 1, 1, 0, "MN lbo1024 sbo4096"},
    {16, 1024, 0, 0, 1, "Kmajor-transposed (known layout)"},
    {4096, 1024, 0, 0, 0, "MN data, K flags"},
    {128, 1024, 1, 1, 0, "MN lbo128 sbo1024"},
  };
  for (auto& v : vs) {
    cudaMemset(dP, 0, P.size() * 4);
    kdbg<<<1, 128, 40000>>>(dA, dG, dP, v.lbo, v.sbo, v.amn, v.bmn, v.km);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(P.data(), dP, P.size() * 4, cudaMemcpyDeviceToHost);
    double me = 0, mr = 0; int nz = 0;
    for (int i = 0; i < K * N; ++i) { me = fmax(me, fabs(R[i] - P[i])); mr = fmax(mr, fabs(R[i])); nz += P[i] != 0; }
    printf("%-36s err=%s maxerr=%g maxref=%g nonzero=%d P00=%g R00=%g P10=%g R10=%g P01=%g R01=%g\n", v.name, cudaGetErrorString(e), me, mr, nz, P[0], R[0], P[N], R[N], P[1], R[1]);
  }
  return 0;
}
