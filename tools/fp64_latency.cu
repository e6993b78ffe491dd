// FP64 FMA throughput of one B200 SM partition as a function of the resident
// warps per SM and the independent FMA chains per thread (ILP): what occupancy /
// ILP the element kernels need to fill the FP64 pipe.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double* out, int iters) {
  double a[ILP];
#pragma unroll
  for (int u = 0; u < ILP; ++u) a[u] = threadIdx.x * 1e-9 + u;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int u = 0; u < ILP; ++u) a[u] = fma(a[u], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < ILP; ++u) s += a[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP>
void run(int sms, int warps_per_sm, double* out) {
  const int threads = 32 * warps_per_sm > 1024 ? 1024 : 32 * warps_per_sm;
  const int blocks_per_sm = (32 * warps_per_sm) / threads;
  const int blocks = sms * blocks_per_sm, iters = 2048;
  k<ILP><<<blocks, threads>>>(out, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<ILP><<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double flops = 2.0 * ILP * 16 * (double)iters * blocks * threads;
  printf("{\"warps_per_sm\": %d, \"ilp\": %d, \"tflops\": %.2f}\n", warps_per_sm, ILP, flops / best / 1e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 2048 * 2);
  for (int w : {4, 8, 12, 16, 24, 32, 64}) {
    run<1>(sms, w, out); run<2>(sms, w, out); run<3>(sms, w, out); run<4>(sms, w, out); run<8>(sms, w, out);
  }
  return 0;
}
