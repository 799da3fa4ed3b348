// Standalone check of the TMEM accumulator pattern used by af_rows_kernel at M = 16384:
// 512-thread CTAs, warp 0 allocates 256 columns, every thread zeroes / read-modify-writes
// its 64 columns (lane 32 (w % 4) + lane, columns 64 (w / 4) ..), then writes them out.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_test tmem_test.cu
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

__global__ void __launch_bounds__(512, 1) k(float* out, int rows) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"((unsigned)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ta = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
  float z[16];
  for (int i = 0; i < 16; ++i) z[i] = 0.f;
  for (int c = 0; c < 4; ++c) st16(ta + 16 * c, z);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  for (int r = 0; r < rows; ++r) {
    for (int c = 0; c < 4; ++c) {
      float a[16];
      ld16(ta + 16 * c, a);
      wait_ld(a);
      for (int i = 0; i < 16; ++i) a[i] += (float)(threadIdx.x * 64 + 16 * c + i) + r;
      st16(ta + 16 * c, a);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  for (int c = 0; c < 4; ++c) {
    float a[16];
    ld16(ta + 16 * c, a);
    wait_ld(a);
    for (int i = 0; i < 16; ++i) out[(size_t)blockIdx.x * 512 * 64 + threadIdx.x * 64 + 16 * c + i] = a[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(slot) : "memory");
  }
}

int main() {
  const int blocks = 148 * 3, rows = 10;
  float* d; cudaMalloc(&d, sizeof(float) * blocks * 512 * 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<blocks, 512, 140 * 1024>>>(d, rows);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  float* h = new float[(size_t)blocks * 512 * 64];
  cudaMemcpy(h, d, sizeof(float) * blocks * 512 * 64, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (long b = 0; b < blocks; ++b)
    for (long i = 0; i < 512 * 64; ++i) {
      const double want = rows * (double)i + rows * (rows - 1) / 2.0;
      if (h[b * 512 * 64 + i] != (float)want) ++bad;
    }
  printf("bad %ld of %ld\n", bad, (long)blocks * 512 * 64);
  return 0;
}
