// Microbenchmark (round-2 design input for the M = 16384 row kernel): an FFT exchange of
// 32 complex values per thread (512 threads, one CTA per SM) through TENSOR MEMORY instead
// of shared memory.  A warp may only touch the 32 TMEM lanes of its quarter (w % 4), so
// the TMEM exchange reaches the 4 warps of a quarter group: each thread writes its 64
// floats with one tcgen05.st.32x32b.x64 into its warp's 64-column region, the quarter
// group meets at a named barrier, and each thread reads 8 x tcgen05.ld.16x128b.x4 (two
// 16-lane halves x four regions): reader (lane l) gets lanes (l>>2) and (l>>2)+8 of each
// half, column l&3 (+4 per repetition).  Checks that mapping, then times:
//   FP phase only, shared-memory exchange, TMEM exchange, and each exchange with FP.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_xchg tmem_xchg.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st64(uint32_t a, const float (&r)[64]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,"
      "%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(a),
      "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]), "f"(r[8]), "f"(r[9]),
      "f"(r[10]), "f"(r[11]), "f"(r[12]), "f"(r[13]), "f"(r[14]), "f"(r[15]), "f"(r[16]), "f"(r[17]), "f"(r[18]),
      "f"(r[19]), "f"(r[20]), "f"(r[21]), "f"(r[22]), "f"(r[23]), "f"(r[24]), "f"(r[25]), "f"(r[26]), "f"(r[27]),
      "f"(r[28]), "f"(r[29]), "f"(r[30]), "f"(r[31]), "f"(r[32]), "f"(r[33]), "f"(r[34]), "f"(r[35]), "f"(r[36]),
      "f"(r[37]), "f"(r[38]), "f"(r[39]), "f"(r[40]), "f"(r[41]), "f"(r[42]), "f"(r[43]), "f"(r[44]), "f"(r[45]),
      "f"(r[46]), "f"(r[47]), "f"(r[48]), "f"(r[49]), "f"(r[50]), "f"(r[51]), "f"(r[52]), "f"(r[53]), "f"(r[54]),
      "f"(r[55]), "f"(r[56]), "f"(r[57]), "f"(r[58]), "f"(r[59]), "f"(r[60]), "f"(r[61]), "f"(r[62]), "f"(r[63])
      : "memory");
}
__device__ __forceinline__ void ld16x128x4(uint32_t a, float* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "r"(a)
               : "memory");
}
__device__ __forceinline__ void wait_ld64(float (&r)[64]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) asm volatile("" : "+f"(r[i]));
}
__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// TMEM exchange: write own 64 floats, quarter-group barrier, gather 64 floats
__device__ __forceinline__ void tmem_exchange(uint32_t tbase, int warp, float (&v)[64], bool cta_bar) {
  const int q = warp & 3, h = warp >> 2;
  st64(tbase + ((uint32_t)(32 * q) << 16) + 64 * h, v);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (cta_bar) __syncthreads(); else bar_named(1 + q, 128);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
  for (int hh = 0; hh < 4; ++hh)
#pragma unroll
    for (int half = 0; half < 2; ++half)
      ld16x128x4(tbase + ((uint32_t)(32 * q + 16 * half) << 16) + 64 * hh + 16 * h, &v[16 * hh + 8 * half]);
  wait_ld64(v);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (cta_bar) __syncthreads(); else bar_named(1 + q, 128);   // WAR before the next write
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__global__ void __launch_bounds__(512, 1) check(int* bad, float* dump) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = (float)(tid * 64 + i);   // writer thread, column
  tmem_exchange(slot, warp, v, false);
  // predicted: reg 16 hh + 8 half + 2 rep + v1 <- writer warp (q, hh), lane 16 half + (l>>2) + 8 v1,
  // its column 16 h + 4 rep + (l & 3)
  const int q = warp & 3, h = warp >> 2;
  int nb = 0;
  for (int hh = 0; hh < 4; ++hh)
    for (int half = 0; half < 2; ++half)
      for (int rep = 0; rep < 4; ++rep)
        for (int v1 = 0; v1 < 2; ++v1) {
          const int wl = 16 * half + (lane >> 2) + 8 * v1;
          const int wt = 32 * (q + 4 * hh) + wl;
          const int col = 16 * h + 4 * rep + (lane & 3);
          const float want = (float)(wt * 64 + col);
          const int r = 16 * hh + 8 * half + 2 * rep + v1;
          if (v[r] != want) ++nb;
        }
  if (tid < 64 && blockIdx.x == 0)
    for (int i = 0; i < 64; ++i) dump[tid * 64 + i] = v[i];
  atomicAdd(bad, nb);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}

template <int NF, int MODE>   // 0 FP, 1 smem exch, 2 TMEM exch (quarter bar), 3 FP+smem, 4 FP+TMEM, 5 FP+TMEM (CTA bar)
__global__ void __launch_bounds__(512, 1) k(float* out, int iters, int zmask) {
  extern __shared__ float2 sm[];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = tid * 1e-3f + i;
  const float bb = 0.999f + tid * 1e-9f;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1 || MODE == 3) {
      const int off = (__float_as_int(v[0]) ^ __float_as_int(v[63])) & zmask;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int y = tid + e * 512;
        sm[y + (y >> 5) + off] = make_float2(v[2 * e], v[2 * e + 1]);
      }
      __syncthreads();
      const int rb = tid * 32 + tid;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float2 x = sm[rb + e + off];
        v[2 * e] = x.x;
        v[2 * e + 1] = x.y;
      }
      __syncthreads();
    }
    if (MODE == 2 || MODE == 4) tmem_exchange(slot, warp, v, false);
    if (MODE == 5) tmem_exchange(slot, warp, v, true);
    if (MODE == 0 || MODE >= 3) {
#pragma unroll
      for (int u = 0; u < NF / 8; ++u)
#pragma unroll
        for (int i = 0; i < 64; ++i) v[i] = fmaf(v[i], bb, 1e-7f);
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) r += v[i];
  if (r == 1234.5f) out[tid] = r;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}
template <int NF, int MODE>
double run(float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem = 16384 * 8 + 512 * 8 + 64;
  cudaFuncSetAttribute(k<NF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k<NF, MODE><<<148, 512, smem>>>(out, 10, 0);
  cudaEventRecord(e0);
  k<NF, MODE><<<148, 512, smem>>>(out, iters, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e-3 * 1.965e9 / iters;
}
template <int NF>
void row(float* out) {
  const double f = run<NF, 0>(out), xs = run<NF, 1>(out), xt = run<NF, 2>(out);
  const double fs = run<NF, 3>(out), ft = run<NF, 4>(out), ftc = run<NF, 5>(out);
  printf("FFMA/thread %4d: FP %5.0f | smem exch %5.0f, FP+smem %5.0f | TMEM exch %5.0f, FP+TMEM %5.0f "
         "(CTA barriers: %5.0f)  cycles/iter/SM\n",
         NF * 8, f, xs, fs, xt, ft, ftc);
}
int main() {
  int* bad;
  float *out, *dump;
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&dump, 64 * 64 * 4);
  check<<<148, 512>>>(bad, dump);
  int hb = -1;
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  float hd[64 * 64];
  cudaMemcpy(hd, dump, sizeof hd, cudaMemcpyDeviceToHost);
  printf("mapping check: %d mismatches (%s)\n", hb, cudaGetErrorString(cudaGetLastError()));
  for (int t = 0; t < 6; ++t) {
    printf("  thread %d regs:", t);
    for (int i = 0; i < 10; ++i) printf(" (%d,%d)", (int)hd[t * 64 + i] / 64, (int)hd[t * 64 + i] % 64);
    printf("\n");
  }
  row<32>(out);
  row<48>(out);
  row<64>(out);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
