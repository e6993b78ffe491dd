// Microbenchmark of the cluster Gauss-Jordan coarse inverse (k_dense_invert_cl)
// on a random diagonally dominant block-stencil operator; checks A * Ainv = I.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1907_01252_b200/csrc \
//        tools/gj_bench.cu -o gj_bench && ./gj_bench 16 4 32
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <cstring>
#include "kernels_linalg.cuh"

using namespace pint;

int main(int argc, char** argv) {
  const int cx = argc > 1 ? atoi(argv[1]) : 16, cy = argc > 2 ? atoi(argv[2]) : 4, S = argc > 3 ? atoi(argv[3]) : 32;
  Grid g{};
  g.dim = 2; g.n[0] = cx + 1; g.n[1] = cy + 1; g.n[2] = 1;
  g.nn = g.n[0] * g.n[1]; g.np = (g.nn + 31) / 32 * 32; g.C = 5; g.noff = 9;
  const int C = 5, n = C * g.nn;
  std::vector<double> hA((size_t)S * 9 * C * C * g.np);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (auto& v : hA) v = U(rng);
  for (int s = 0; s < S; ++s)
    for (int c = 0; c < C; ++c)
      for (int nd = 0; nd < g.nn; ++nd)  // centre offset 4, diagonal entry: dominant, mixed scales
        hA[(size_t)s * 9 * C * C * g.np + ((size_t)(4 * C + c) * C + c) * g.np + nd] = (c == 4 ? 1e-3 : 1e3) * 60.0;
  double *dA, *dM;
  float* dM32;
  const int ld = (n + 3) / 4 * 4;
  cudaMalloc(&dA, hA.size() * 8);
  cudaMalloc(&dM, (size_t)S * 2 * n * n * 8);
  cudaMalloc(&dM32, (size_t)S * n * ld * 4);
  const int variant = argc > 4 ? atoi(argv[4]) : 0;  // 0: cluster, 1: single-CTA augmented fallback
  cudaMemcpy(dA, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
  const size_t smem = gj_smem_bytes(n);
  cudaFuncSetAttribute(k_dense_invert_cl<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    if (variant == 0) {
      k_dense_invert_cl<2><<<S * kGJCluster, kGJThreads, smem>>>(g, dA, dM32, n, ld, nullptr);
    } else {
      k_dense_build<2><<<dim3(1, S), 512>>>(g, dA, dM, nullptr);
      k_gauss_jordan<<<S, 512>>>(dM, n, nullptr);
      k_dense_to_f32<<<dim3((n * n + 255) / 256, S), 256>>>(dM, dM32, n, ld, nullptr);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("v%d n=%d S=%d smem=%zu: %.3f ms (%.2f us/pivot) err=%s\n", variant, n, S, smem, ms, 1e3 * ms / n,
           cudaGetErrorString(cudaGetLastError()));
  }
  // check slice 0: dense A * Minv = I
  std::vector<double> M((size_t)n * n), D((size_t)n * n, 0.0);
  {
    std::vector<float> M2((size_t)n * ld);
    cudaMemcpy(M2.data(), dM32, M2.size() * 4, cudaMemcpyDeviceToHost);
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < n; ++c) M[(size_t)r * n + c] = M2[(size_t)r * ld + c];
  }
  for (int row = 0; row < n; ++row) {
    const int ca = row / g.nn, node = row % g.nn;
    int i, j, k;
    node_coords(g, node, i, j, k);
    for (int off = 0; off < 9; ++off) {
      const int nb = neighbour(g, i, j, k, off);
      if (nb < 0) continue;
      for (int cb = 0; cb < C; ++cb) D[(size_t)row * n + cb * g.nn + nb] = hA[(((size_t)off * C + ca) * C + cb) * g.np + node];
    }
  }
  double worst = 0;
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) {
      double acc = 0;
      for (int q = 0; q < n; ++q) acc += D[(size_t)r * n + q] * M[(size_t)q * n + c];
      const double e = fabs(acc - (r == c ? 1.0 : 0.0));
      worst = e > worst ? e : worst;
    }
  unsigned long long h = 1469598103934665603ULL;
  for (double v : M) { unsigned long long b; memcpy(&b, &v, 8); h = (h ^ b) * 1099511628211ULL; }
  printf("max |A Ainv - I| = %.3e  hash %016llx\n", worst, h);
  return 0;
}
