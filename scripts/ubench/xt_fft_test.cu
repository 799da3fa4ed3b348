// Standalone check + timing of the tensor-memory-exchange M = 16384 FFT (graf_fft_xt.cuh)
// against a float64 DFT on the host (forward) and against the input (inverse of forward),
// and timing of 16384-point row FFTs: the graf_fft.cuh Stockham plan vs the XT plan.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o xt_fft_test xt_fft_test.cu
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "graf_fft_xt.cuh"
using namespace graf;

struct CtaSync {
  __device__ void operator()() const { __syncthreads(); }
  __device__ void before_writing() const {}
  __device__ void done_reading() const { __syncthreads(); }
};

__device__ __forceinline__ void tm_alloc512(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(slot)) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

// MODE 0: X = FFT(x) (out in natural order), 1: y = IFFT(X) for X given in natural order,
// 2: timing loop of forward + inverse (XT), 3: the same with the Stockham plan
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(const float2* in, float2* out, int iters) {
  extern __shared__ float4 smraw[];
  float2* sh = reinterpret_cast<float2*>(smraw);
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) tm_alloc512(&slot);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t lanef = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  const uint32_t tw1 = lanef + kXtTw1Col, xq = lanef + (GRAF_XT_ONE_ROUND ? kXtXchCol1 : kXtXchCol);
  if ((warp >> 2) == 0 && !GRAF_XT_ONE_ROUND) xt_fill_tw1(tw1, t);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  CtaSync sync;
  float2* xtab = sh + 16384 + 512 + 1024;
  xt_fill_tab(xtab, t, 512);
  __syncthreads();
  const float2* x = in + (size_t)blockIdx.x * 16384;
  float2* y = out + (size_t)blockIdx.x * 16384;
  float2 v[32];
  if (MODE == 0) {
    for (int e = 0; e < 32; ++e) v[e] = x[t + 512 * e];
    fft16384_xt_fwd(v, sh, tw1, xq, t, sync, xtab);
    for (int e = 0; e < 32; ++e) y[xt_freq(t, e)] = v[e];
  } else if (MODE == 1) {
    for (int e = 0; e < 32; ++e) v[e] = x[xt_freq(t, e)];
    fft16384_xt_inv(v, sh, tw1, xq, t, sync, xtab);
    for (int e = 0; e < 32; ++e) y[t + 512 * e] = v[e];
  } else {
    for (int e = 0; e < 32; ++e) v[e] = x[t + 512 * e];
    Twiddles<16384, 32> tw;
    tw.init(t);
    float2* tab = reinterpret_cast<float2*>(sh + 16384 + 512);
    Twiddles<16384, 32>::fill_tab1(tab, t, 512);
    tw.tab1 = tab;
    if (MODE == 9) {
      // production c5 layout: every thread's 31 pass-1 twiddles W_1024^((t mod 32) r) in its own
      // TMEM columns 256 + 64 (w / 4) .. (tmem_tw_ld16 reads them; the table is not used)
      const uint32_t ttw = slot + ((uint32_t)(32 * (warp & 3)) << 16) + 256 + 64 * (warp >> 2);
      const int jm = t & 31;
      for (int c = 0; c < 4; ++c) {
        float w16[16];
        for (int i = 0; i < 8; ++i) {
          const int r = 8 * c + i + 1;
          const float2 w = r < 32 ? g_tw[(jm * r * 16) & 16383] : make_float2(0.f, 0.f);
          w16[2 * i] = w.x;
          w16[2 * i + 1] = w.y;
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16};" ::"r"(ttw + 16 * c),
            "f"(w16[0]), "f"(w16[1]), "f"(w16[2]), "f"(w16[3]), "f"(w16[4]), "f"(w16[5]), "f"(w16[6]), "f"(w16[7]),
            "f"(w16[8]), "f"(w16[9]), "f"(w16[10]), "f"(w16[11]), "f"(w16[12]), "f"(w16[13]), "f"(w16[14]),
            "f"(w16[15]) : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tw.ttw = ttw;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int it = 0; it < iters; ++it) {
      if (MODE >= 4 && MODE <= 8) {
        const int w = t >> 5;
        // ablations of one forward + inverse: 4 = no B<->C exchange, 5 = no A<->B exchange,
        // 6 = no twiddle 1, 7 = only the two B<->C exchanges, 8 = only the two A<->B exchanges
        if (MODE != 7 && MODE != 8) dft<32, false>(v);
        if (MODE != 5 && MODE != 7) xt_exchange_ab<true>(v, sh, t, sync);
        if (MODE != 6 && MODE != 7 && MODE != 8) xt_twiddle1<false>(v, tw1, xtab, t);
        if (MODE != 7 && MODE != 8) dft<32, false>(v);
        if (MODE != 4 && MODE != 8) xt_exchange_bc(v, xq, w & 3, w >> 2);
        if (MODE != 7 && MODE != 8) xt_pass2<false>(v, t);
        for (int e = 0; e < 32; ++e) v[e] = make_float2(v[e].x * 1e-4f, v[e].y * 1e-4f);
        if (MODE != 7 && MODE != 8) xt_pass2<true>(v, t);
        if (MODE != 4 && MODE != 8) xt_exchange_cb(v, xq, w & 3, w >> 2);
        if (MODE != 7 && MODE != 8) dft<32, true>(v);
        if (MODE != 6 && MODE != 7 && MODE != 8) xt_twiddle1<true>(v, tw1, xtab, t);
        if (MODE != 5 && MODE != 7) xt_exchange_ab<false>(v, sh, t, sync);
        if (MODE != 7 && MODE != 8) dft<32, true>(v);
      } else if (MODE == 2) {
        fft16384_xt_fwd(v, sh, tw1, xq, t, sync, xtab);
        for (int e = 0; e < 32; ++e) v[e] = make_float2(v[e].x * 1e-4f, v[e].y * 1e-4f);
        fft16384_xt_inv(v, sh, tw1, xq, t, sync, xtab);
      } else {
        fft_rows<16384, 32, 0, false>(v, sh, t, tw, sync);
        for (int e = 0; e < 32; ++e) v[e] = make_float2(v[e].x * 1e-4f, v[e].y * 1e-4f);
        fft_rows<16384, 32, 0, true>(v, sh, t, tw, sync);
      }
      for (int e = 0; e < 32; ++e) v[e] = make_float2(v[e].x * 6.1035e-5f, v[e].y * 6.1035e-5f);
    }
    for (int e = 0; e < 32; ++e) y[t + 512 * e] = v[e];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}

int main() {
  const int M = 16384;
  launch_tw_init(0);
  std::vector<float2> hx(M);
  srand(1);
  for (int i = 0; i < M; ++i) hx[i] = make_float2(rand() / (float)RAND_MAX - 0.5f, rand() / (float)RAND_MAX - 0.5f);
  float2 *dx, *dy, *dz;
  cudaMalloc(&dx, 148 * M * 8);
  cudaMalloc(&dy, 148 * M * 8);
  cudaMalloc(&dz, 148 * M * 8);
  cudaMemcpy(dx, hx.data(), M * 8, cudaMemcpyHostToDevice);
  const int smem = (16384 + 512 + 2048) * 8;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<0><<<1, 512, smem>>>(dx, dy, 0);
  k<1><<<1, 512, smem>>>(dy, dz, 0);
  cudaError_t err = cudaDeviceSynchronize();
  printf("kernels: %s\n", cudaGetErrorString(err));
  std::vector<float2> hy(M), hz(M);
  cudaMemcpy(hy.data(), dy, M * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hz.data(), dz, M * 8, cudaMemcpyDeviceToHost);
  // float64 DFT (direct; twiddles by exact index arithmetic)
  std::vector<std::complex<double>> W(M);
  for (int i = 0; i < M; ++i) W[i] = std::polar(1.0, -2.0 * M_PI * i / M);
  double emax = 0, xmax = 0, imax = 0;
  for (int m = 0; m < M; ++m) {
    std::complex<double> acc = 0;
    for (int n = 0; n < M; ++n) acc += std::complex<double>(hx[n].x, hx[n].y) * W[(long long)n * m % M];
    emax = std::max(emax, std::abs(acc - std::complex<double>(hy[m].x, hy[m].y)));
    xmax = std::max(xmax, std::abs(acc));
  }
  for (int n = 0; n < M; ++n)
    imax = std::max(imax, std::abs(std::complex<double>(hz[n].x, hz[n].y) / (double)M -
                                   std::complex<double>(hx[n].x, hx[n].y)));
  printf("forward: max |err| %.3e of max |X| %.3e (rel %.2e); inverse(forward)/M - x: max %.3e\n", emax, xmax,
         emax / xmax, imax);
  // timing: 148 CTAs, forward + inverse per iteration
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 200;
    float ms2, ms3;
    k<2><<<148, 512, smem>>>(dx, dy, 10);
    cudaEventRecord(e0);
    k<2><<<148, 512, smem>>>(dx, dy, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms2, e0, e1);
    k<3><<<148, 512, smem>>>(dx, dy, 10);
    cudaEventRecord(e0);
    k<3><<<148, 512, smem>>>(dx, dy, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms3, e0, e1);
    printf("fwd+inv per row-pair per SM: XT %.0f cycles, Stockham %.0f cycles (%.2fx)\n",
           ms2 * 1e-3 * 1.965e9 / iters, ms3 * 1e-3 * 1.965e9 / iters, ms3 / ms2);
  }
  {
    cudaFuncSetAttribute(k<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
      k<9><<<148, 512, smem>>>(dx, dy, 10);
      cudaEventRecord(e0);
      k<9><<<148, 512, smem>>>(dx, dy, 200);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("Stockham with TMEM pass-1 twiddles (production c5 plan): %.0f cycles\n", ms * 1e-3 * 1.965e9 / 200);
    }
  }
  const char* nm[] = {"", "", "", "", "no B<->C (TMEM) exchanges", "no A<->B (smem) exchanges", "no twiddle 1",
                      "only the 2 TMEM exchanges", "only the 2 smem exchanges"};
  for (int m = 4; m <= 8; ++m) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    auto go = [&](int it) {
      switch (m) {
        case 4: k<4><<<148, 512, smem>>>(dx, dy, it); break;
        case 5: k<5><<<148, 512, smem>>>(dx, dy, it); break;
        case 6: k<6><<<148, 512, smem>>>(dx, dy, it); break;
        case 7: k<7><<<148, 512, smem>>>(dx, dy, it); break;
        case 8: k<8><<<148, 512, smem>>>(dx, dy, it); break;
      }
    };
    go(10);
    cudaEventRecord(e0);
    go(200);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("XT fwd+inv, %-28s %.0f cycles\n", nm[m], ms * 1e-3 * 1.965e9 / 200);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
