// Microbenchmark (round-2 design input for the M = 16384 row kernel): does a second,
// independent CTA per SM hide the exchange phases of a barrier-synchronised Stockham FFT?
// Each iteration models one FFT pass of the c5 row: an FP phase (NF FFMA on 8 chains per
// thread), then the exchange: 32 STS.64 to a transposed slot, a CTA barrier, 32 LDS.64, a CTA
// barrier.  Same per-thread work and 512 threads per SM in every layout:
//   A: one 512-thread CTA per SM (one 16384-point row: the current c5 kernel)
//   B: two 256-thread CTAs per SM, each with its own barriers (two 8192-point half rows)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o two_cta_overlap two_cta_overlap.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ int g_ticket[256];
template <int THREADS, int NF, int MODE>   // MODE 0: FP only, 1: exchange only, 2: both, 3: FP + STS phase, 4: FP + LDS phase
__global__ void __launch_bounds__(THREADS, 512 / THREADS) k(float* out, int iters, int zmask, int delay) {
  extern __shared__ float2 sm[];
  const int tid = threadIdx.x;
  // the second CTA to arrive on an SM starts `delay` cycles late (per-SM ticket)
  __shared__ int ticket;
  int role = 0;   // delay < 0: the first CTA of an SM runs only the exchange, the second only FP
  if (delay) {
    if (tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      ticket = atomicAdd(&g_ticket[smid], 1) & 1;
    }
    __syncthreads();
    if (delay < 0) {
      role = ticket ? 1 : 2;
    } else if (ticket) {
      const long long t0 = clock64();
      while (clock64() - t0 < delay) {}
    }
  }
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = tid * 1e-3f + i;
  const float bb = 0.999f + tid * 1e-9f;
  // transposed exchange: thread t writes slot t + e*THREADS, reads (t*32 + e) padded
  const int rbase = (tid * 32) + ((tid * 32) >> 5);
  for (int it = 0; it < iters; ++it) {
    float2 x[32];
    if (MODE != 0 && role != 1) {
      const int off = (__float_as_int(a[0]) ^ __float_as_int(a[7])) & zmask;
      if (MODE != 4) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int y = tid + e * THREADS;
          sm[y + (y >> 5) + off] = make_float2(a[e & 7], a[(e + 1) & 7]);
        }
      }
      __syncthreads();
      if (MODE != 3) {
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = sm[rbase + e + off];
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = make_float2(1e-6f * e + a[0], 1e-6f);
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = make_float2(1e-6f * e, 1e-6f);
    }
    if (MODE != 1 && role != 2) {
#pragma unroll
      for (int u = 0; u < NF; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], bb, u < 4 ? x[i + 8 * u].x + x[i + 8 * u].y : 1e-7f);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] += x[i].x + x[i + 8].y + x[i + 16].x + x[i + 24].y;
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1234.5f) out[tid] = r;
}
template <int THREADS, int NF, int MODE>
double run(float* out, int delay = 0) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = THREADS * 32 * 8 + THREADS * 8 + 64;
  cudaFuncSetAttribute(k<THREADS, NF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<THREADS, NF, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  static bool said[2] = {false, false};
  if (!said[THREADS == 256]) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k<THREADS, NF, MODE>, THREADS, smem);
    if (0) printf("   %d threads: %d resident CTAs per SM (smem %d B)\n", THREADS, nb, smem);
    said[THREADS == 256] = true;
  }
  const int grid = 148 * (512 / THREADS);
  const int iters = 2000;
  k<THREADS, NF, MODE><<<grid, THREADS, smem>>>(out, 10, 0, delay);
  cudaEventRecord(e0);
  k<THREADS, NF, MODE><<<grid, THREADS, smem>>>(out, iters, 0, delay);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e-3 * 1.965e9 / iters;   // cycles per iteration per SM (all 512 threads)
}
template <int NF>
void row(float* out) {
  const double fa = run<512, NF, 0>(out), xa = run<512, NF, 1>(out), ba = run<512, NF, 2>(out);
  const double fb = run<256, NF, 0>(out), xb = run<256, NF, 1>(out), bb = run<256, NF, 2>(out);
  const double bd = run<256, NF, 2>(out, (int)((fb + xb) * 0.5)), bq = run<256, NF, 2>(out, (int)((fb + xb) * 0.25));
  const double s1 = run<512, NF, 3>(out), s2 = run<256, NF, 3>(out, (int)((fb + xb) * 0.5));
  const double l1 = run<512, NF, 4>(out), l2 = run<256, NF, 4>(out, (int)((fb + xb) * 0.5));
  const double sp = run<256, NF, 2>(out, -1);
  printf("   split roles (CTA 0 exchange only, CTA 1 FP only, same SM): %6.0f  vs FP-only 2x256 %6.0f\n", sp, fb);
  printf("   FP+STS only: 1x512 %6.0f  2x256(delayed) %6.0f | FP+LDS only: 1x512 %6.0f  2x256(delayed) %6.0f\n", s1, s2, l1, l2);
  printf("NF=%3d | 1x512: FP %6.0f  exch %6.0f  both %6.0f (sum %6.0f) | 2x256: FP %6.0f  exch %6.0f  both %6.0f"
         "  -> %.2fx | 2x256, 2nd CTA delayed 1/2 iter: %6.0f (%.2fx), 1/4 iter: %6.0f (%.2fx)\n",
         NF, fa, xa, ba, fa + xa, fb, xb, bb, ba / bb, bd, ba / bd, bq, ba / bq);
}
int main() {
  float* out;
  cudaMalloc(&out, 1 << 20);
  row<16>(out);
  row<32>(out);
  row<48>(out);
  row<64>(out);
  row<96>(out);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
