// Microbenchmark (round-2 design input for the M = 16384 row kernel): can a WARP-LOCAL
// exchange (32 STS.64, __syncwarp, 32 LDS.64 inside a warp-private shared region) overlap
// with the FP work of the other warps, where a CTA-wide exchange (same bytes, two CTA
// barriers) cannot?  One 512-thread CTA per SM, 32 values per thread, as in the c5 row.
// Each iteration = FP phase (NF FFMA on 8 chains) + one exchange:
//   mode 0: FP only            mode 1: CTA exchange only      mode 2: FP + CTA exchange
//   mode 3: warp exchange only mode 4: FP + warp exchange     mode 5: FP + alternating
//   (CTA exchange on even iterations, warp-local exchange on odd: the four-step layout)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o warp_local_xchg warp_local_xchg.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int TH = 512;
template <int NF, int MODE>
__global__ void __launch_bounds__(TH, 1) k(float* out, int iters, int zmask) {
  extern __shared__ float2 sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = tid * 1e-3f + i;
  const float bb = 0.999f + tid * 1e-9f;
  float2* wreg = sm + warp * (32 * 33);   // warp-private 32 x 32 (+1 pad) region
  for (int it = 0; it < iters; ++it) {
    float2 x[32];
    const int off = (__float_as_int(a[0]) ^ __float_as_int(a[7])) & zmask;
    const bool cta = (MODE == 1 || MODE == 2) || (MODE == 5 && (it & 1) == 0);
    const bool wl = (MODE == 3 || MODE == 4) || (MODE == 5 && (it & 1) == 1);
    if (cta) {
      // CTA-wide transpose: thread t writes slot t + e*512, reads 32 consecutive of (t*32)
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int y = tid + e * TH;
        sm[y + (y >> 5) + off] = make_float2(a[e & 7], a[(e + 1) & 7]);
      }
      __syncthreads();
      const int rb = tid * 32 + tid;
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = sm[rb + e + off];
      __syncthreads();
    } else if (wl) {
      // warp-local 32 x 32 transpose: lane l writes row l, reads column l
#pragma unroll
      for (int e = 0; e < 32; ++e) wreg[lane * 33 + e + off] = make_float2(a[e & 7], a[(e + 1) & 7]);
      __syncwarp();
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = wreg[e * 33 + lane + off];
      __syncwarp();
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) x[e] = make_float2(1e-6f * e, 1e-6f);
    }
    if (MODE != 1 && MODE != 3) {
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
template <int NF, int MODE>
double run(float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = 16384 * 8 + 512 * 8 + 64;
  cudaFuncSetAttribute(k<NF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k<NF, MODE><<<148, TH, smem>>>(out, 10, 0);
  cudaEventRecord(e0);
  k<NF, MODE><<<148, TH, smem>>>(out, iters, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e-3 * 1.965e9 / iters;   // cycles per iteration per SM
}
template <int NF>
void row(float* out) {
  const double f = run<NF, 0>(out), xc = run<NF, 1>(out), fc = run<NF, 2>(out);
  const double xw = run<NF, 3>(out), fw = run<NF, 4>(out), fa = run<NF, 5>(out);
  printf("NF=%3d  FP %5.0f | CTA exch %5.0f, FP+CTA %5.0f (sum %5.0f) | warp exch %5.0f, FP+warp %5.0f (sum %5.0f)"
         " | FP + alternating %5.0f\n",
         NF, f, xc, fc, f + xc, xw, fw, f + xw, fa);
}
int main() {
  float* out;
  cudaMalloc(&out, 1 << 20);
  row<16>(out);
  row<32>(out);
  row<48>(out);
  row<64>(out);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
