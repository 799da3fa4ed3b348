// Microbenchmark: FFMA lane-ops per cycle per SM vs independent chains per thread and warps per SM (one CTA per SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fpilp fp_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, int U>
__global__ void __launch_bounds__(1024, 1) k(float* out, int iters) {
  float a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float bb = 0.999f + threadIdx.x * 1e-9f, cc = 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < CH; ++i) a[i] = fmaf(a[i], bb, cc);
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 1234.5f) out[threadIdx.x] = r;
}
template <int CH, int U>
void run(const char* nm, int threads, float* out, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(k<CH, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  const int iters = 4000;
  k<CH, U><<<sms, threads, 120 * 1024>>>(out, 10);
  cudaEventRecord(e0);
  k<CH, U><<<sms, threads, 120 * 1024>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double lane = (double)threads * CH * U * iters / (ms * 1e-3 * 1.965e9);
  printf("%-28s threads %4d : %6.1f lane-op/cyc/SM\n", nm, threads, lane);
}
int main() {
  float* out; cudaMalloc(&out, 4096); int sms = 148;
  run<4, 16>("4 chains", 512, out, sms);
  run<8, 16>("8 chains", 512, out, sms);
  run<16, 8>("16 chains", 512, out, sms);
  run<32, 4>("32 chains", 512, out, sms);
  run<8, 16>("8 chains", 256, out, sms);
  run<16, 8>("16 chains", 256, out, sms);
  run<8, 16>("8 chains (1024 thr)", 1024, out, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
