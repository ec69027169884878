// debug harness for the MN-major tcgen05 wgrad kernel
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2311_14898_b200/csrc/ht_common.h"
namespace ht { std::string& last_error() { static std::string s; return s; } }
#include "../paper_2311_14898_b200/csrc/ht_tc.cuh"

int main() {
  const int M = 32, K = 128, N = 128;
  std::vector<float> A(M * K), G(M * N), P(K * N, -7.f);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 37) % 11) - 5;
  for (int i = 0; i < M * N; ++i) G[i] = (float)((i * 13) % 7) - 3;
  float *dA, *dG, *dP;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dG, G.size() * 4); cudaMalloc(&dP, P.size() * 4 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dG, G.data(), G.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dP, 0, P.size() * 4);
  int used = 0;
  int rc = ht::tc::wgrad(0, dA, K, K, dG, N, N, M, 148, dP, &used);
  cudaError_t e = cudaDeviceSynchronize();
  printf("rc %d used %d sync %s err=%s\n", rc, used, cudaGetErrorString(e), ht::last_error().c_str());
  cudaMemcpy(P.data(), dP, P.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0; int nz = 0;
  for (int k = 0; k < K; ++k) for (int n = 0; n < N; ++n) {
    double r = 0; for (int m = 0; m < M; ++m) r += (double)A[m * K + k] * G[m * N + n];
    maxerr = fmax(maxerr, fabs(r - P[k * N + n])); maxref = fmax(maxref, fabs(r)); nz += P[k*N+n] != 0;
  }
  printf("maxerr %g maxref %g nonzero %d\n", maxerr, maxref, nz);
  for (int q = 0; q < 4; ++q) { double r = 0; for (int m = 0; m < M; ++m) r += (double)A[m*K+q]*G[m*N]; printf("P[%d][0]=%g ref %g\n", q, P[q*N], r); }
  return 0;
}
