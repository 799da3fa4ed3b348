// Microbenchmark (round-2 design input): tcgen05.ld / tcgen05.st (32x32b.x16) throughput
// per SM, alone and concurrent with shared-memory LDS.64, one 512-thread CTA per SM owning
// 256 TMEM columns (the c5 kernel's allocation).  Mode 0: TMEM ld only; 1: TMEM st only;
// 2: LDS only; 3: TMEM ld + LDS in every warp; 4: TMEM ld + st (read-modify-write).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld16(uint32_t a, float (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]),
                 "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11]), "=f"(r[12]), "=f"(r[13]), "=f"(r[14]), "=f"(r[15])
               : "r"(a) : "memory");
}
__device__ __forceinline__ void st16(uint32_t a, const float (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(a), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]),
               "f"(r[8]), "f"(r[9]), "f"(r[10]), "f"(r[11]), "f"(r[12]), "f"(r[13]), "f"(r[14]), "f"(r[15]) : "memory");
}
__device__ __forceinline__ void wait_ld(float (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+f"(r[0]), "+f"(r[1]), "+f"(r[2]), "+f"(r[3]), "+f"(r[4]),
               "+f"(r[5]), "+f"(r[6]), "+f"(r[7]), "+f"(r[8]), "+f"(r[9]), "+f"(r[10]), "+f"(r[11]), "+f"(r[12]),
               "+f"(r[13]), "+f"(r[14]), "+f"(r[15]) :: "memory");
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float* out, int iters) {
  extern __shared__ float2 sm[];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 16384; i += 512) sm[i] = make_float2(i * 1e-6f, 1e-6f);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ta = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = tid * 1e-3f + i;
  float s = 0.f;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm + tid);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (MODE == 0 || MODE == 3 || MODE == 4) {
        float r[16];
        ld16(ta + 16 * c, r);
        wait_ld(r);
        if (MODE == 4) {
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] += 1e-7f;
          st16(ta + 16 * c, r);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) s += r[i];
        }
      }
      if (MODE == 1) st16(ta + 16 * c, acc);
      if (MODE == 2 || MODE == 3) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float x, y;
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(sbase + (j + 8 * c) * 4096));
          s += x;
        }
      }
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot) : "memory");
  if (s == 1234.5f) out[tid] = s;
}

template <int MODE>
void run(const char* nm, float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int iters = 2000;
  k<MODE><<<148, 512, 128 * 1024>>>(out, 10);
  cudaEventRecord(e0);
  k<MODE><<<148, 512, 128 * 1024>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * 1.965e9 / iters;
  // per iteration per SM: TMEM 4 x (512 threads x 16 words x 4 B) = 128 KiB; LDS 32 x 512 x 8 B = 128 KiB
  const double tb = (MODE == 0 || MODE == 1 || MODE == 3 || MODE == 4) ? 131072.0 : 0.0;
  const double lb = (MODE == 2 || MODE == 3) ? 131072.0 : 0.0;
  printf("%-26s %7.1f cyc/iter/SM  TMEM %6.1f B/cyc  LDS %6.1f B/cyc\n", nm, cyc, tb / cyc, lb / cyc);
}
int main() {
  float* out;
  cudaMalloc(&out, 4096);
  run<0>("TMEM ld only", out);
  run<1>("TMEM st only", out);
  run<2>("LDS only", out);
  run<3>("TMEM ld + LDS", out);
  run<4>("TMEM ld + st (RMW)", out);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
