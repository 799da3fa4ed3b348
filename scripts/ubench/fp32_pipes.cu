// Microbenchmark of the sm_100a FP32 pipes the FFT kernels use (round-2 design input):
// lane-ops per cycle per SM for FFMA (register operands), FFMA (immediate), FADD, FMUL,
// and the paired f32x2 forms FFMA2 / FADD2 / FMUL2; plus shared-memory LDS.64/128 bytes
// per cycle per SM.  One CTA of 256 threads x 4 per SM, 8 independent chains per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_pipes fp32_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
template <int V>
__global__ void __launch_bounds__(256) k_fp(float* out, int iters, float b, float c) {
  float a[CH], d[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) { a[i] = threadIdx.x * 1e-3f + i; d[i] = a[i] * 0.5f; }
  float bb = b + threadIdx.x * 1e-9f, cc = c + threadIdx.x * 1e-9f;   // registers, not constants
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        if (V == 0) a[i] = fmaf(a[i], bb, cc);                      // FFMA R,R,R
        if (V == 1) a[i] = fmaf(a[i], 0.999f, 0.25f);               // FFMA imm
        if (V == 2) a[i] = a[i] + bb;                                // FADD R,R
        if (V == 3) a[i] = a[i] * bb;                                // FMUL R,R
        if (V == 4) a[i] = fmaf(a[i], d[i], cc);                     // FFMA 3 distinct regs
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i] + d[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r;
}
template <int V>
__global__ void __launch_bounds__(256) k_fp2(float* out, int iters, float b, float c) {
  unsigned long long a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = pk(threadIdx.x * 1e-3f + i, i * 0.5f);
  const unsigned long long bb = pk(b + threadIdx.x * 1e-9f, b), cc = pk(c, c + threadIdx.x * 1e-9f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        if (V == 0) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(bb), "l"(cc));
        if (V == 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(bb));
        if (V == 2) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(bb));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); s += x + y; }
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int W>   // W = 8 (LDS.64) or 16 (LDS.128) bytes per thread per load
__global__ void __launch_bounds__(256) k_lds(float* out, int iters) {
  __shared__ float4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += 256) buf[i] = make_float4(i, i, i, i);
  __syncthreads();
  float acc = 0.f;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (W == 16) { float4 v = buf[(idx + u * 256) & 2047]; acc += v.x + v.w; }
      else { float2 v = reinterpret_cast<float2*>(buf)[(idx + u * 256) & 4095]; acc += v.x + v.y; }
    }
    idx = (idx + 37) & 255;
  }
  if (acc == 1234.5f) out[threadIdx.x] = acc;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);   // kHz (max)
  float* out; cudaMalloc(&out, 4096 * sizeof(float));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = nsm * 4, iters = 8192;
  auto run = [&](const char* name, void (*k)(float*, int, float, float), double ops_per_thread_iter) {
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); k<<<blocks, 256>>>(out, iters, 0.999f, 0.25f); cudaEventRecord(b);
      cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
      double lane_ops = ops_per_thread_iter * iters * 256.0 * blocks;
      if (r) best = best > lane_ops / (ms * 1e-3) ? best : lane_ops / (ms * 1e-3);
    }
    printf("%-22s %8.2f Tlane-op/s  %6.1f lane-op/cyc/SM (at max clock %d MHz)\n", name, best / 1e12,
           best / nsm / (clk * 1e3), clk / 1000);
  };
  run("FFMA R,R,R (shared)", k_fp<0>, 16.0 * CH);
  run("FFMA R,imm,imm", k_fp<1>, 16.0 * CH);
  run("FADD R,R", k_fp<2>, 16.0 * CH);
  run("FMUL R,R", k_fp<3>, 16.0 * CH);
  run("FFMA 3 distinct R", k_fp<4>, 16.0 * CH);
  run("FFMA2 (x2 lanes)", k_fp2<0>, 32.0 * CH);
  run("FADD2 (x2 lanes)", k_fp2<1>, 32.0 * CH);
  run("FMUL2 (x2 lanes)", k_fp2<2>, 32.0 * CH);
  auto runl = [&](const char* name, void (*k)(float*, int), double bytes_per_thread_iter) {
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); k<<<blocks, 256>>>(out, iters); cudaEventRecord(b);
      cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
      double by = bytes_per_thread_iter * iters * 256.0 * blocks;
      if (r) best = best > by / (ms * 1e-3) ? best : by / (ms * 1e-3);
    }
    printf("%-22s %8.2f TB/s        %6.1f B/cyc/SM\n", name, best / 1e12, best / nsm / (clk * 1e3));
  };
  runl("LDS.64", k_lds<8>, 16.0 * 8);
  runl("LDS.128", k_lds<16>, 16.0 * 16);
  printf("SMs %d\n", nsm);
  return 0;
}
