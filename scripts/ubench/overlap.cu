// Microbenchmark (round-2 design input for the M = 16384 row kernel): can the SM overlap
// FP32 FMA-pipe work with shared-memory (LDS) traffic and with warp shuffles (SHFL)?
// One CTA of 512 threads per SM (128 KiB of dynamic shared memory forces it), like the
// c5 kernel.  Each warp runs `iters` iterations of: F x 8 independent FFMA, L x LDS.64
// (conflict-free), S x SHFL.  Modes compare the time of FP-only, LDS-only, SHFL-only runs
// with the same work mixed in every warp ("mixed") and split across warps ("split":
// warps 0-7 do 2x the FP work, warps 8-15 2x the LDS/SHFL work).  If mixed ~ max(FP, LDS)
// the pipes overlap; if ~ sum they serialise.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o overlap overlap.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k_mix(float* out, int iters, int F, int L, int S, int split) {
  extern __shared__ float2 sm[];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 16384; i += 512) sm[i] = make_float2(i * 1e-3f, 1.f);
  __syncthreads();
  int f = F, l = L, s = S;
  if (split) {
    if (warp < 8) { f = 2 * F; l = 0; s = 0; }
    else { f = 0; l = 2 * L; s = 2 * S; }
  }
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = tid * 1e-3f + i;
  const float bb = 0.999f + tid * 1e-9f, cc = 1e-3f;
  unsigned acc = 0;
  float sh = tid * 1.0f;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + tid * 8;
  for (int it = 0; it < iters; ++it) {
    for (int j = 0; j < f; ++j) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], bb, cc);
    }
    for (int j = 0; j < l; j += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        unsigned x, y;
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(base + ((j + u) & 31) * 4096));
        acc ^= x + y;
      }
    }
    for (int j = 0; j < s; j += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) sh = __shfl_sync(0xffffffffu, sh, (tid + u + 1) & 31);
    }
  }
  float r = sh + (float)acc;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1234.5f) out[tid] = r;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 512 * sizeof(float));
  const int smem = 128 * 1024;
  cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  struct Case { const char* name; int F, L, S, split; } cases[] = {
      {"FP only   F=8      ", 8, 0, 0, 0},  {"LDS only  L=16     ", 0, 16, 0, 0},
      {"mixed     F=8 L=16 ", 8, 16, 0, 0}, {"split     F=8 L=16 ", 8, 16, 0, 1},
      {"SHFL only S=16     ", 0, 0, 16, 0}, {"mixed     F=8 S=16 ", 8, 0, 16, 0},
      {"split     F=8 S=16 ", 8, 0, 16, 1}, {"LDS+SHFL  L=16 S=16", 0, 16, 16, 0},
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& c : cases) {
    k_mix<<<sms, 512, smem>>>(out, 10, c.F, c.L, c.S, c.split);
    cudaEventRecord(e0);
    k_mix<<<sms, 512, smem>>>(out, iters, c.F, c.L, c.S, c.split);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per SM per iteration, in cycles at the max clock
    const double cyc = ms * 1e-3 * clk * 1e3 / iters;
    const double fp_lane = 16.0 * 32 * 8 * c.F;           // FFMA lane-ops per SM per iteration
    const double lds_b = 16.0 * 32 * 8 * c.L;              // LDS bytes per SM per iteration
    const double shfl_w = 16.0 * c.S;                      // SHFL warp-instructions per SM per iteration
    printf("%s  %8.1f cyc/iter   FP %6.1f lane-op/cyc  LDS %6.1f B/cyc  SHFL %5.2f warp-inst/cyc\n", c.name, cyc,
           fp_lane / cyc, lds_b / cyc, shfl_w / cyc);
  }
  cudaError_t err = cudaGetLastError();
  printf("%s (SMs %d, clock %d kHz)\n", cudaGetErrorString(err), sms, clk);
  return 0;
}
