// graf_kernels.cuh — the delay-row kernel and the reductions of the GRAF hot path.
//
// One kernel template, `af_rows_kernel<M, KIND, WGT>`, covers SURVEY.md §8(a) rows a0-a7:
//   a0  stage s[b] in shared memory, energy E_b (double, fixed order)
//   a1  lag product r_k[n] = s[n] conj(s[n-k]) straight into the FFT registers
//       (Eqs. 8-10; the shift matrix S of Eq. 9 is never built)
//   a2  Stockham FFT over Doppler (Eq. 11)
//   a3F surface epilogue: A, |A| or chi (Eq. 12; Alg. 1 steps 4-5, L251-252),
//       rows +k and -k from one FFT (A[-k,m] = e^{2 pi i m k/M} conj(A[k,-m]))
//   a3L loss epilogue: ISL numerator, online max / sum-exp (Eqs. 19-20)
//   a5  cotangent G = f' A / E^2 (Eq. 14)
//   a6  inverse Doppler FFT H = M*IFFT(G) (L230)
//   a7  delay correlation g[p] += H[k,p] s[p-k] + conj(H[k,p+k]) s[p+k] (Eq. 15)
// KIND selects the pass at compile time:
//   K_FWD   a0-a3F/a3L            (graf_af_forward; pass 1 of soft-PSL)
//   K_ISL   a0-a7 in ONE pass      (ISL-only losses: f' = lambda_isl*w is known up front)
//   K_PASS2 a0-a7 with f' from the combined pass-1 partials (soft-PSL)
//   K_ADJ   dA row -> a6-a7        (graf_af_backward, unfolded rows)
//   K_FWDA  K_FWD that also tracks the hard-PSL argmax cell (its own instantiation,
//           so the plain forward pass carries none of that code)
// Rows are folded to k >= 0 (symmetric masks/weights): row k > 0 stands for
// rows +k and -k (loss sums and gradient terms counted twice; SURVEY §8(c)
// "symmetric-loss identities").
#pragma once
#include <cooperative_groups.h>
#include <type_traits>
#include "../../include/graf.h"
#include "graf_fft.cuh"

namespace graf {

enum : int { K_FWD = 0, K_ISL = 1, K_PASS2 = 2, K_ADJ = 3, K_FWDA = 4, K_MATCH = 5 };
// K_FWDA: K_FWD + hard-PSL argmax;  K_MATCH: one pass with f' = lambda_isl w + match term
constexpr int kPart = 8;  // doubles per CTA partial record: S, max, Z, C, fchi, -, -, -

struct RowParams {
  const float2* s;   // [B][N]
  int N, B, b0;      // b0: first waveform of this launch (grid.y chunking)
  int U;             // rows enumerated per waveform
  int row_lo, row_step;
  // surface window / dA rows
  int kb, ke;
  void* surface;
  int out_kind, layout, norm_out;
  const float2* dA;
  // loss
  int loss_on, kloss;  // kloss = min(k_max, N-1)
  int d_max, ml_k, ml_d;
  const float* w_k;
  const float* w_d;
  float lam_isl, lam_psl, invT, T;
  int normalize;
  int shard_index, shard_count;
  int centred;
  int const_sum;       // the region is constant-sum (full plane, normalised, unweighted, M >= N):
                       // the ISL term's gradient is identically zero (volume identity), so pass 2
                       // leaves it out instead of cancelling O(1) terms in fp32 (reading R13 (iii))
  // the region spans the whole plane except a mainlobe block (normalised, unweighted, M >= N):
  // the ISL over the whole plane is constant (volume identity), so the ISL gradient equals
  // MINUS that of the excluded cells; the kernels give f' = -lambda_isl to the excluded cells
  // and nothing to the region, instead of summing O(1) terms that cancel (round 2)
  int complement;
  float xbar;
  double omega;        // |Omega| (full region, for the centred mean)
  const graf_partials* stats;  // combined partials [B] for K_PASS2
  // outputs
  double* part;        // [B][P][kPart]
  float2* gpart;       // [B][P][N]
  const float2* s_pad; // [B][NL+M] zero-padded s (global-memory path, M > 8192)
  const float2* s_pad1; // the same rows shifted by one sample (odd delays read aligned pairs)
  int bulk;            // surface rows staged in shared memory + bulk async copies: 1 dedicated
                       // buffer (stg_floats per slot), 2 aliased to the slot's exchange buffer
  int stg_floats;      // staging floats per row slot (2*M*{1,2}: rows +k and -k)
  int gpad;            // 1: left-padded gradient accumulators (M == N, folded rows)
  int periodic;        // 1: circular lag products (the paper's Eq. 2 / Alg. 1), M == N
  // hard PSL (K_FWD): track the argmax cell of x over the region as a row-major key
  // (delay index from key_lo) * M + raw Doppler bin, ties -> lowest key (reading R23)
  int want_argmax;
  int key_lo;
  // band cache of two-pass losses: pass 1 (K_FWD/K_FWDA, cache = 1) stores the FFT
  // outputs of the loss band |d| <= d_max of every loss row, pass 2 (K_PASS2,
  // cache = 2) reads them instead of recomputing the lag product and forward FFT
  float2* acache;      // [B][U][nband]
  int cache, nband;
  // optimistic single pass of the full-plane centred soft-PSL (K_PASS2, onepass = 1):
  // f' = lambda expm1((x - xbar)/T) needs no global statistic (constant shifts of f'
  // are gradient-neutral on a constant-sum region, reading R13) and 1/Z_c scales the
  // result in the finalize.  The guarded fallback launches skip the waveforms whose
  // single pass is valid (guard[b].reserved == 1).
  int onepass;
  const graf_partials* guard;
  // caller's per-waveform skip mask (graf_af_desc.skip, ABI v6): skip[b] != 0 -> no work,
  // no output for waveform b
  const int32_t* skip;
  // cross-ambiguity (CROSS kernels): X = sum s[n] conj(s2[n-k]) W^{mn}; rows unfolded
  const float2* s2;    // [B][N]
  float2* gpart2;      // [B][P][N] partial dL/ds2*
  // match loss (K_MATCH): target laid out like the surface window, per waveform stride
  float lam_match;
  const float* target;
  long long target_stride;
  // fused finalize (K_ISL, P <= 8 CTAs per waveform launched as one thread-block
  // cluster): cluster rank 0 combines the CTAs' partials over distributed shared
  // memory and writes loss and grad directly (no partial records, no finalize kernel)
  int fuse;
  double* loss_out;    // [B] (nullable)
  float2* grad_out;    // [B][N]
  int smem_bytes;      // dynamic shared memory of the launch (the pass-1 twiddle table ends it)
};

template <int M>
struct Cfg;
#ifndef GRAF_SPLIT_16384
#define GRAF_SPLIT_16384 0   // 1 = round-1 A/B build: the radix-2 split with the smem accumulator
#endif
#ifndef GRAF_TMEM_8192
#define GRAF_TMEM_8192 1     // 0 = round-1 A/B build for M = 8192 (padded s, smem accumulator)
#endif
#define GRAF_TMEM_8192_OK(M_) ((M_) != 8192 || GRAF_TMEM_8192)
#ifndef GRAF_TMEM_1024
#define GRAF_TMEM_1024 0     // 1: M = 1024 with TMEM accumulators + unpadded s (measured slower for c3: profiles/r02/tune_c3_ab.txt)
#endif
#ifndef GRAF_MINB_1024G
#define GRAF_MINB_1024G 4    // resident CTAs per SM of the M = 1024 gradient kernels with GRAF_TMEM_1024
#endif
#ifndef GRAF_MINB_8192
#define GRAF_MINB_8192 2     // M = 8192 with the trimmed s: two resident CTAs per SM (64 registers)
#endif
// E = values per thread, T = threads per row slot, S = row slots per CTA.
// M = 16384: one 16384-point Stockham FFT per row (E = 32, passes 32 x 32 x 16, a 132 KiB
// exchange buffer) with the gradient accumulator in TENSOR MEMORY (G_TMEM: 128 KiB of the
// SM's 256 KiB TMEM, thread-private columns), s read from a zero-padded global copy.
// (SPLIT, the round-1 layout kept for A/B builds: a radix-2 split into two M/2-point
// sub-FFTs sharing one M/2 exchange buffer, the accumulator in shared memory.)
#define GRAF_CFG(M_, E_, S_)                                         \
  template <>                                                        \
  struct Cfg<M_> {                                                   \
    static constexpr int M = M_, E = E_, T = M_ / E_, S = S_;        \
    static constexpr int THREADS = T * S;                            \
    static constexpr bool SPLIT = (M_ >= 16384) && GRAF_SPLIT_16384;  \
    static constexpr int MX = SPLIT ? M_ / 2 : M_;  /* exchanged FFT length */ \
    static constexpr int XS = MX + MX / Pad<SPLIT ? E_ / 2 : E_>::P;  /* padded exchange */ \
    static constexpr bool S_SMEM = (M_ <= 8192);                     \
    static constexpr bool G_TMEM = ((M_ >= 8192) && !SPLIT && GRAF_TMEM_8192_OK(M_)) || \
                                   ((M_ == 1024) && GRAF_TMEM_1024);                  \
    /* M = 8192: s staged WITHOUT zero padding (aperiodic: [N samples]; every read of it is \
       predicated to the row's support), so two CTAs fit an SM beside the exchange buffer */ \
    static constexpr bool S_TRIM = (M_ == 8192 || M_ == 1024) && G_TMEM; \
    static constexpr bool G_SMEM = !G_TMEM;                          \
  };
// Defaults; a tuning build may override one size with -DGRAF_E_<M>=.. -DGRAF_S_<M>=..
#ifndef GRAF_E_64
#define GRAF_E_64 8
#endif
#ifndef GRAF_S_64
#define GRAF_S_64 16
#endif
#ifndef GRAF_E_128
#define GRAF_E_128 16
#endif
#ifndef GRAF_S_128
#define GRAF_S_128 16
#endif
#ifndef GRAF_E_256
#define GRAF_E_256 16
#endif
#ifndef GRAF_S_256
#define GRAF_S_256 8
#endif
#ifndef GRAF_E_512
#define GRAF_E_512 8
#endif
#ifndef GRAF_S_512
#define GRAF_S_512 2
#endif
#ifndef GRAF_E_1024
#define GRAF_E_1024 32
#endif
#ifndef GRAF_S_1024
#define GRAF_S_1024 4
#endif
#ifndef GRAF_E_2048
#define GRAF_E_2048 16
#endif
#ifndef GRAF_S_2048
#define GRAF_S_2048 1
#endif
#ifndef GRAF_E_4096
#define GRAF_E_4096 16
#endif
#ifndef GRAF_S_4096
#define GRAF_S_4096 1
#endif
#ifndef GRAF_E_8192
#define GRAF_E_8192 16
#endif
#ifndef GRAF_S_8192
#define GRAF_S_8192 1
#endif
#ifndef GRAF_E_16384
#define GRAF_E_16384 32
#endif
GRAF_CFG(2, 2, 64)
GRAF_CFG(4, 4, 64)
GRAF_CFG(8, 8, 64)
GRAF_CFG(16, 16, 64)
GRAF_CFG(32, 16, 32)
GRAF_CFG(64, GRAF_E_64, GRAF_S_64)
GRAF_CFG(128, GRAF_E_128, GRAF_S_128)
GRAF_CFG(256, GRAF_E_256, GRAF_S_256)
GRAF_CFG(512, GRAF_E_512, GRAF_S_512)
GRAF_CFG(1024, GRAF_E_1024, GRAF_S_1024)
GRAF_CFG(2048, GRAF_E_2048, GRAF_S_2048)
GRAF_CFG(4096, GRAF_E_4096, GRAF_S_4096)
GRAF_CFG(8192, GRAF_E_8192, GRAF_S_8192)
GRAF_CFG(16384, GRAF_E_16384, 1)
#undef GRAF_CFG

// mbarrier helpers (split write-after-read barriers of the exchange buffer)
__device__ __forceinline__ void mbar_init(uint32_t mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mb) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(mb) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(mb),
      "r"(parity)
      : "memory");
}
#ifndef GRAF_TW1_TMEM_16384
#define GRAF_TW1_TMEM_16384 1   // M = 16384 gradient kernels: pass-1 twiddles in tensor memory
#endif
#ifndef GRAF_SPLIT_WAR
// one-slot CTAs: 1 = split write-after-read barriers, 0 = a full barrier after every read
// phase (default: the split form measured SLOWER, c5 13.48 -> 15.01 ms, c4 2.064 -> 2.106 ms,
// profiles/r02/tune_c5_war.txt: the read-after-write barrier of every exchange stays, so warps
// gain little skew, and 512 threads polling the mbarrier compete with the exchange's LDS)
#define GRAF_SPLIT_WAR 0
#endif

// Synchronisation of one row slot's exchange buffer.  operator() orders writes before
// reads (read-after-write: a full barrier of the slot).  done_reading() / before_writing()
// bracket the write-after-read hazard: by default done_reading() is a full barrier and
// before_writing() nothing.  In a one-slot CTA (S == 1) with `mb` set, done_reading() is an
// mbarrier arrival per warp and before_writing() waits for every warp's arrival, so a warp
// that has read its data runs the next pass's arithmetic while slower warps are still
// reading (the shared-memory and FP32 phases of different warps overlap; a full barrier
// after every read phase serialises them: scripts/ubench/phase_overlap.cu).  Every write
// phase of the buffer is preceded by before_writing() and every read phase followed by
// done_reading(), in the same order in every warp (one arrival is made at the start).
template <int T, int S>
struct SlotSync {
  int id;
  uint32_t mb = 0;            // S == 1: shared address of the WAR mbarrier (0: full barriers)
  mutable uint32_t ph = 0;    // parity of the next phase before_writing() waits for
  __device__ __forceinline__ void operator()() const {
    if constexpr (T <= 32) {
      __syncwarp();
    } else if constexpr (S == 1) {
      __syncthreads();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(T) : "memory");
    }
  }
  __device__ __forceinline__ void done_reading() const {
    if constexpr (S == 1 && T >= 64) {
      if (mb) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(mb);
        return;
      }
    }
    (*this)();
  }
  __device__ __forceinline__ void before_writing() const {
    if constexpr (S == 1 && T >= 64) {
      if (mb) {
        mbar_wait(mb, ph);
        ph ^= 1u;
      }
    }
  }
};

// E_b = sum |s|^2 in double, fixed order: lane l sums n = l (mod 32), then a
// shuffle-down tree; lane 0's value is THE energy (identical in every kernel).
__device__ __forceinline__ double warp_energy(const float2* sb, int N, int lane) {
  double acc = 0.0;
  for (int n = lane; n < N; n += 32) {
    const float2 v = sb[n];
    acc += (double)v.x * v.x + (double)v.y * v.y;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  return acc;  // valid in lane 0
}

// Deterministic CTA reductions (fixed shuffle tree, fixed warp order); result in thread 0.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  constexpr int NW = (THREADS + 31) / 32;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if constexpr (NW == 1) {
    return v;
  } else {
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
      for (int w = 0; w < NW; ++w) r += scratch[w];
    __syncthreads();
    return r;
  }
}

template <int THREADS>
__device__ __forceinline__ float block_max_all(float v, double* scratch) {
  constexpr int NW = (THREADS + 31) / 32;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
  if constexpr (NW == 1) {
    return v;
  } else {
    float* sc = reinterpret_cast<float*>(scratch);
    if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = v;
    __syncthreads();
    float r = -INFINITY;
    for (int w = 0; w < NW; ++w) r = fmaxf(r, sc[w]);
    __syncthreads();
    return r;  // in every thread
  }
}

// CTA argmax of (value, key) pairs: largest value, ties -> smallest key; the key of
// the winner in thread 0 (fixed shuffle tree and warp order: deterministic)
template <int THREADS>
__device__ __forceinline__ int block_argmax_key(float x, int key, double* scratch) {
  constexpr int NW = (THREADS + 31) / 32;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ox = __shfl_xor_sync(0xffffffffu, x, off);
    const int ok = __shfl_xor_sync(0xffffffffu, key, off);
    if (ox > x || (ox == x && ok < key)) {
      x = ox;
      key = ok;
    }
  }
  if constexpr (NW == 1) {
    return key;
  } else {
    float* sx = reinterpret_cast<float*>(scratch);
    int* sk = reinterpret_cast<int*>(scratch) + 32;
    if ((threadIdx.x & 31) == 0) {
      sx[threadIdx.x >> 5] = x;
      sk[threadIdx.x >> 5] = key;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < NW; ++w)
        if (sx[w] > x || (sx[w] == x && sk[w] < key)) {
          x = sx[w];
          key = sk[w];
        }
    }
    __syncthreads();
    return key;
  }
}

// argmax-key merge that goes with lse_merge: called BEFORE lse_merge updates m
__device__ __forceinline__ void key_merge(double m, double& key, double m2, double key2) {
  if (m2 > m || (m2 == m && key2 < key)) key = key2;
}

// exact merge of (max, sum exp((x - max)/T)) pairs, in double (maxima are exact floats)
__device__ __forceinline__ void lse_merge(double& m, double& Z, double m2, double Z2, float T) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2;
    Z = Z2;
    return;
  }
  if (m2 > m) {
    Z = Z * exp((m - m2) / (double)T) + Z2;
    m = m2;
  } else {
    Z = Z + Z2 * exp((m2 - m) / (double)T);
  }
}

// sqrt through the MUFU unit (sqrt.approx: ~1 ulp-scale relative error, sqrt(0) = 0)
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// float exp(x) for x <= 0 through the MUFU ex2 unit (rel. error ~2 ulp)
__device__ __forceinline__ float exp_fast(float x) { return exp2f(x * 1.4426950408889634f); }

// expm1(u) to ~1 ulp-scale relative error: degree-7 Taylor on |u| < 0.5 (remainder
// < u^8/40320 ~ 1e-7 |u|), exp(u) - 1 beyond (no cancellation there)
__device__ __forceinline__ float expm1_fast(float u) {
  const float p = fmaf(u, fmaf(u, fmaf(u, fmaf(u, fmaf(u, fmaf(u, 1.f / 5040.f, 1.f / 720.f), 1.f / 120.f),
                                                       1.f / 24.f), 1.f / 6.f), 0.5f), 1.f);
  return fabsf(u) < 0.5f ? u * p : exp_fast(u) - 1.f;
}

// minimum resident CTAs per SM requested from ptxas (caps registers per thread);
// a tuning build may force one value for every size with -DGRAF_MINB=..
// (measured on B200, scripts/tune.py: M = 1024 runs E = 32 radix-32 passes, one
// exchange per FFT; 3 CTAs/SM for the forward pass, 2 for the gradient kernels)
template <int M, int KIND>
struct MinBlocks {
#ifdef GRAF_MINB
  static constexpr int value = GRAF_MINB;
#else
  static constexpr int value = M <= 16 ? 2 : M == 1024 ? ((KIND == 0 || KIND == 4) ? 3 : GRAF_TMEM_1024 ? GRAF_MINB_1024G : 2)
                              : M <= 1024 ? 4 : M <= 4096 ? 2
                              : (M == 8192 && GRAF_TMEM_8192) ? GRAF_MINB_8192 : 1;
#endif
};
// radix-2 split stage between the two M/2-point halves (twiddle W_M^{t + e T} =
// W_M^t * W_{2*E2}^e, the second factor a compile-time constant)
template <int E2, int K, bool INV>
__device__ __forceinline__ void split_combine(float2* v, const float2* a, const float2* c, float2 wt) {
  if constexpr (K < E2) {
    const float2 wb = twc<K, 2 * E2, false>(cmul(c[K], wt));
    v[K] = cadd(a[K], wb);
    v[K + E2] = csub(a[K], wb);
    split_combine<E2, K + 1, INV>(v, a, c, wt);
  }
}
template <int E2, int K>
__device__ __forceinline__ void split_dif(const float2* v, float2* a, float2* c, float2 wt) {
  if constexpr (K < E2) {
    a[K] = cadd(v[K], v[K + E2]);
    c[K] = twc<K, 2 * E2, true>(cmulc(csub(v[K], v[K + E2]), wt));
    split_dif<E2, K + 1>(v, a, c, wt);
  }
}

// Length-M FFT of one row slot: direct Stockham, or (SPLIT) two M/2-point
// sub-FFTs of the even/odd time samples joined by one radix-2 stage in registers.
// Slot layout in frequency is e <-> m = t + e*T either way; in time it is
// n = t + e*T (direct) or n = 2(t + e'T) + parity (SPLIT, e = e' + parity*E/2).
template <int M, int E, bool SPLIT, bool INV, class TW, class Sync>
__device__ __forceinline__ void row_fft(float2 (&v)[E], float2* sh, int t, const TW& tw, const Sync& sync,
                                        float2 wt) {
  if constexpr (!SPLIT) {
    fft_rows<M, E, 0, INV>(v, sh, t, tw, sync);
  } else {
    constexpr int E2 = E / 2, M2 = M / 2;
    float2 a[E2], c[E2];
    if constexpr (!INV) {
#pragma unroll
      for (int e = 0; e < E2; ++e) {
        a[e] = v[e];
        c[e] = v[e + E2];
      }
      fft_rows<M2, E2, 0, false>(a, sh, t, tw, sync);
      fft_rows<M2, E2, 0, false>(c, sh, t, tw, sync);
      split_combine<E2, 0, false>(v, a, c, wt);
    } else {
      split_dif<E2, 0>(v, a, c, wt);
      fft_rows<M2, E2, 0, true>(a, sh, t, tw, sync);
      fft_rows<M2, E2, 0, true>(c, sh, t, tw, sync);
#pragma unroll
      for (int e = 0; e < E2; ++e) {
        v[e] = a[e];
        v[e + E2] = c[e];
      }
    }
  }
}

// ---- bulk asynchronous shared -> global row stores (the TMA engine's 1-D bulk
// copy; no tensor map).  The surface epilogue stages each finished row in shared
// memory at its final column order and one thread per row slot hands it to the
// copy engine, so the HBM stream runs beside the next row's FFT instead of
// through the LSU pipe as 4-byte stores.
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ---- tensor memory (TMEM) as a thread-private accumulator (G_TMEM, M = 16384).  A CTA
// allocates 256 of the SM's 512 TMEM columns; warp w may touch lanes 32 (w % 4) .. +31,
// so thread (w, lane) owns TMEM lane 32 (w % 4) + lane and the 64 columns 64 (w / 4) ..:
// with 512 threads that is 16384 complex accumulators, one per time index n = t + e T.
// (M = 8192, E = 16: 128 columns per CTA, so two CTAs share an SM's TMEM)
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {   // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(slot)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {   // one full warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// wait::ld that also ties the loaded registers to the wait, so no use of them can be
// scheduled above it
__device__ __forceinline__ void tmem_wait_ld16(float (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(r[0]), "+f"(r[1]), "+f"(r[2]), "+f"(r[3]), "+f"(r[4]), "+f"(r[5]), "+f"(r[6]), "+f"(r[7]),
                 "+f"(r[8]), "+f"(r[9]), "+f"(r[10]), "+f"(r[11]), "+f"(r[12]), "+f"(r[13]), "+f"(r[14]), "+f"(r[15])
               :
               : "memory");
}
// 8 columns (4 complex accumulators)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld8(float (&r)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(r[0]), "+f"(r[1]), "+f"(r[2]), "+f"(r[3]), "+f"(r[4]), "+f"(r[5]), "+f"(r[6]), "+f"(r[7])
               :
               : "memory");
}
// 16 consecutive 32-bit columns of this thread's lane (8 complex accumulators)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]),
        "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11]), "=f"(r[12]), "=f"(r[13]), "=f"(r[14]), "=f"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]), "f"(r[8]), "f"(r[9]),
      "f"(r[10]), "f"(r[11]), "f"(r[12]), "f"(r[13]), "f"(r[14]), "f"(r[15])
      : "memory");
}

// generic chunk of C columns (C = 8 or 16)
template <int C>
__device__ __forceinline__ void tmem_ldc(uint32_t a, float (&r)[C]) {
  if constexpr (C == 16) tmem_ld16(a, r); else tmem_ld8(a, r);
}
template <int C>
__device__ __forceinline__ void tmem_stc(uint32_t a, const float (&r)[C]) {
  if constexpr (C == 16) tmem_st16(a, r); else tmem_st8(a, r);
}
template <int C>
__device__ __forceinline__ void tmem_wait_ldc(float (&r)[C]);
template <>
__device__ __forceinline__ void tmem_wait_ldc<16>(float (&r)[16]) { tmem_wait_ld16(r); }
template <>
__device__ __forceinline__ void tmem_wait_ldc<8>(float (&r)[8]) { tmem_wait_ld8(r); }
#ifndef GRAF_SOWN_TMEM_16384
#define GRAF_SOWN_TMEM_16384 1   // M = 16384 gradient kernels: own samples in TMEM (see kSown)
#endif
#ifndef GRAF_LAZY_MASKS
#define GRAF_LAZY_MASKS 1
#endif
#ifndef GRAF_ACC_TMEM_8192
#define GRAF_ACC_TMEM_8192 1
#endif
#ifndef GRAF_TMEM_SLOTS
#define GRAF_TMEM_SLOTS 8    // slots per TMEM read-modify-write chunk in the correlation (8 or 4)
#endif

// slots per batch of predicated accumulator loads in the correlation (loads of a
// batch are issued back to back, then the stores)
#ifndef GRAF_CORR_CHUNK
#define GRAF_CORR_CHUNK 8   // must divide E
#endif
constexpr int kCorrChunk = GRAF_CORR_CHUNK;

// predicated shared-memory accesses: a false predicate skips the access (the load
// returns 0) without a branch
template <int OFF>
__device__ __forceinline__ float2 ld_shared_if(unsigned a, bool q) {
  float2 r;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n mov.b32 %0, 0;\n mov.b32 %1, 0;\n"
      " @q ld.shared.v2.f32 {%0, %1}, [%2+%4];\n}"
      : "=f"(r.x), "=f"(r.y)
      : "r"(a), "r"((int)q), "n"(OFF)
      : "memory");
  return r;
}
template <int OFF>
__device__ __forceinline__ void st_shared_if(unsigned a, float2 v, bool q) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.shared.v2.f32 [%0+%4], {%1, %2};\n}" ::"r"(a),
               "f"(v.x), "f"(v.y), "r"((int)q), "n"(OFF)
               : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// compile-time loop helper: f(integral_constant<int, I>) for I in [B, E)
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Inverse FFT of a band-limited row whose only nonzero slots are e = 0 and e = E - 1
// (the loss band |d| < T = M/E; c4): the first pass's radix-E DFT of two nonzero inputs
// is X[r] = x_0 + x_{E-1} W_E^{(E-1) r} (compile-time twiddles), the rest is fft_rows.
template <int M, int E, class TW, class Sync>
__device__ __forceinline__ void ifft_band_edges(float2 (&v)[E], float2* sh, int t, const TW& tw, const Sync& sync) {
  constexpr int T = M / E;
  static_assert(pass_radix(M, E, 0) == E && E <= Pad<E>::P, "first pass must be one radix-E butterfly");
  const float2 x0 = v[0], xl = v[E - 1];
  float2* b = sh + padded<E>(t * E);
  sync.before_writing();
  static_for<0, E>([&](auto r) {
    constexpr int K = ((E - 1) * decltype(r)::value) % E;
    b[decltype(r)::value] = cadd(x0, twc<K, E, true>(xl));
  });
  sync();
  if constexpr (PadStride<E, T>::AFFINE) {
    const float2* c = sh + padded<E>(t);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = c[e * PadStride<E, T>::value];
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = sh[padded<E>(t + e * T)];
  }
  sync.done_reading();
  fft_rows<M, E, 1, true>(v, sh, t, tw, sync);
}

// bits e of [e_lo, e_hi) as a mask over the E register slots
__device__ __forceinline__ unsigned long long slot_range_mask(int e_lo, int e_hi) {
  const unsigned long long hi = e_hi >= 64 ? ~0ull : ((1ull << e_hi) - 1ull);
  const unsigned long long lo = e_lo >= 64 ? ~0ull : ((1ull << e_lo) - 1ull);
  return hi & ~lo;
}

// CROSS: cross-ambiguity of two waveforms: rows unfolded (no
// mirror symmetry), lag product s[n] conj(s2[n-k]), normalisation by E1 E2 (reading
// R25), and the correlation split into dL/ds* (term 1, with s2) and dL/ds2* (term 2,
// with s) accumulated separately.
// FLV (flavour, M >= 8192 where the register budget is tight; the host picks it per call):
//   0 the general kernel;  1 loss-only, the surface epilogue compiled out (c4 -6 %, c5 -2.5 %,
//   profiles/r02/tune_nosurf.txt);  2 loss-only on a band narrower than T bins (c4).  (A third flavour with only the full-plane single pass
//   compiled in spilled 352 B and measured 14.68 ms against 12.65: not kept.)
template <int M, int KIND, bool WGT, bool CROSS = false, int FLV = 0>
__global__ void __launch_bounds__(Cfg<M>::THREADS, MinBlocks<M, KIND>::value) af_rows_kernel(RowParams p) {
  using C = Cfg<M>;
  // cross-ambiguity kernels keep the padded s and the shared-memory accumulators
  // (two accumulator sets and unfolded rows): the TMEM / unpadded layouts are auto only
  constexpr bool kGtmem = C::G_TMEM && !CROSS, kGsmem = !kGtmem, kStrim = C::S_TRIM && !CROSS;
  constexpr int E = C::E, T = C::T, S = C::S, THREADS = C::THREADS, XS = C::XS;
  constexpr int LT = ilog2(T);
  constexpr bool FWD = (KIND == K_FWD || KIND == K_FWDA);
  constexpr bool GRAD = !FWD;
  constexpr bool SPLIT = C::SPLIT;
  constexpr int E2 = SPLIT ? E / 2 : E;
  extern __shared__ float4 smem_raw[];
  float2* smem = reinterpret_cast<float2*>(smem_raw);

  const int N = p.N;
  const int b = p.b0 + blockIdx.y;
  const int P = gridDim.x, pb = blockIdx.x;
  const int slot = threadIdx.x / T, t0 = threadIdx.x % T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float2* sg = p.s + (size_t)b * N;
  if (p.guard && p.guard[b].reserved == 1.0) return;   // fallback launch: this waveform is done
  if (p.skip && p.skip[b]) return;                       // the caller skips this waveform

  // ---- shared-memory carve-up: [scratch 64 doubles][s_pad N+M][exchange x S][g x S]
  // s_pad holds s[n] for n in [-N, M): N zeros, the N samples, M-N zeros, so the
  // lag product and the correlation read s[n-k] with no bounds arithmetic.
  double* red = reinterpret_cast<double*>(smem);
  float2* s_pad = smem + 64;
  const int NP2 = kStrim ? (((p.periodic ? 2 * N : N) + 1) & ~1) : ((N + M + 1) & ~1);
  // CROSS: the second waveform, zero-padded over [-N, M + N): unfolded rows k < 0 read
  // s2[n - k] for every slot n < M (s[n] = 0 beyond N, but 0 * garbage may be NaN)
  float2* s2_pad = s_pad + (C::S_SMEM ? NP2 : 0);
  const int NP2X = (2 * N + M + 1) & ~1;
  float2* xch = s2_pad + (CROSS ? NP2X : 0);
  float2* gacc_sh = xch + S * XS;
  // global copy (M = 16384): rows of NL + M + 2 with NL = N rounded up to even, so every
  // row and the sample origin are 16-byte aligned (the SPLIT path loads sample pairs); the
  // 2 extra keep s[N-1] inside the row of the shifted copy when N == M
  const int NL = N + (N & 1);
  const size_t RP = (size_t)(NL + M + 2);
  // (S_TRIM: aperiodic [N samples], periodic [N-sample copy][N samples])
  const float2* sv = C::S_SMEM ? s_pad + ((kStrim && !p.periodic) ? 0 : N) : p.s_pad + (size_t)b * RP + NL;
  // zero-padded Doppler axis (2N <= M, aperiodic): time slots e >= E/2 hold n >= M/2 >= N
  // (compiled for M >= 2048 only: the extra code path measured 3 % slower at M = 1024)
  constexpr bool kHalfSizes = (M >= 2048) && !SPLIT;
  const bool half = kHalfSizes && !p.periodic && 2 * N <= M;
  // loss band |d| <= d_max < T: a loss pass's cotangent G lives in slots e = 0 and E - 1
  // only (M >= 2048, first pass one radix-E butterfly)
  constexpr bool kEdgeBand = kHalfSizes && (KIND == K_ISL || KIND == K_PASS2 || KIND == K_MATCH) &&
                             pass_radix(M, E, 0) == E && E <= GRAF_MAX_RADIX && num_passes(M, E) > 1;
  // (FLV 2: the loss band is known to be narrower than T bins, |d| <= d_max < T; the host
  // launches it only then, so the band-edge forms are compile-time and the other slots'
  // epilogue code is not compiled)
  const bool edge_band = kEdgeBand && (FLV == 2 || p.d_max < T);
  // ... and the loss epilogues, the band cache and (pass 1) the loss statistics then touch
  // slots 0 and E - 1 only (the others are outside the band: their terms are 0)
  const bool eb = FWD ? (kHalfSizes && (FLV == 2 || p.d_max < T)) : edge_band;
  constexpr bool kEdgeFwd = kHalfSizes && FWD && num_passes(M, E) >= 3 && !Twiddles<C::MX, E2>::CACHE;
  // s[n] at sv_o + n with sv_o + n 16-byte aligned for ODD n (the shifted copy)
  const float2* sv_o = C::S_SMEM ? sv : p.s_pad1 + (size_t)b * RP + NL + 1;
  const float2* sv2 = CROSS ? s2_pad + N : sv;               // the conjugated (shifted) factor
  // per-slot accumulator stride: N, or 2N with N zero-padding on the left (p.gpad: folded
  // rows with M == N need no support predicates, out-of-support terms land in the pad)
  // (compiled for the small sizes only: at M >= 1024 the padded accumulators never fit
  // beside the resident CTAs the gradient kernels need)
  constexpr bool kGpadSizes = (M <= 512);
  const int GS = p.gpad ? 2 * N : N;
  float2* gacc = kGsmem ? gacc_sh + (size_t)slot * GS + (p.gpad ? N : 0) : p.gpart + ((size_t)b * P + pb) * N;
  constexpr int NG = CROSS ? 2 : 1;                           // accumulator sets (CROSS: g1, g2)
  float2* gacc2 = gacc + (size_t)S * GS;                      // CROSS: dL/ds2* accumulators
  // surface staging (bulk path): after the gradient accumulators, 16-byte aligned
  float* stg = reinterpret_cast<float*>(
                   xch + (((size_t)S * XS + (GRAD && kGsmem ? (size_t)NG * S * GS : 0) + 1) & ~(size_t)1)) +
               (size_t)slot * p.stg_floats;

  // ---- a0: stage s, zero the gradient accumulators, energy
  if constexpr (kStrim) {
    const int n_st = p.periodic ? 2 * N : N;
    for (int i = threadIdx.x; i < n_st; i += THREADS) s_pad[i] = sg[i >= N ? i - N : i];
  } else if constexpr (C::S_SMEM) {
    for (int i = threadIdx.x; i < N + M; i += THREADS)
      // aperiodic: N zeros on the left; periodic: a copy of s, so s_pad[n - k] = s[(n - k) mod N]
      s_pad[i] = (i < 2 * N && (i >= N || p.periodic)) ? sg[i >= N ? i - N : i] : make_float2(0.f, 0.f);
    if constexpr (CROSS) {
      const float2* sg2 = p.s2 + (size_t)b * N;
      for (int i = threadIdx.x; i < NP2X; i += THREADS)
        s2_pad[i] = (i >= N && i < 2 * N) ? sg2[i - N] : make_float2(0.f, 0.f);
    }
  }
  if constexpr (GRAD) {
    if constexpr (kGsmem) {
      for (int i = threadIdx.x; i < NG * S * GS; i += THREADS) gacc_sh[i] = make_float2(0.f, 0.f);
    } else {
      for (int i = threadIdx.x; i < N; i += THREADS) gacc[i] = make_float2(0.f, 0.f);
    }
  }
  if (warp == 0) {
    const double e = warp_energy(sg, N, lane);
    if (lane == 0) red[0] = e;
  }
  if constexpr (CROSS) {
    if (warp == (THREADS > 32 ? 1 : 0)) {
      if (THREADS <= 32) __syncwarp();
      const double e2 = warp_energy(p.s2 + (size_t)b * N, N, lane);
      if (lane == 0) red[1] = e2;
    }
  }
  Twiddles<C::MX, E2> tw;
  tw.init(t0);
  // pass-1 twiddle table: the last TAB1 float2 of the dynamic allocation (host adds it)
  if constexpr (Twiddles<C::MX, E2>::SMEM1) {
    float2* tab = reinterpret_cast<float2*>(reinterpret_cast<char*>(smem_raw) + p.smem_bytes) -
                  Twiddles<C::MX, E2>::TAB1;
    Twiddles<C::MX, E2>::fill_tab1(tab, threadIdx.x, THREADS);
    tw.tab1 = tab;
  }
  const float2 wt = SPLIT ? g_tw[t0 * (kMaxM / M)] : make_float2(1.f, 0.f);  // W_M^t (split stage)
  // TMEM gradient accumulator (G_TMEM): warp 0 allocates, the address is read after the
  // prologue barrier; thread (w, lane) owns lane 32 (w % 4) + lane, columns 64 (w / 4) ..
  constexpr bool kTmem = GRAD && kGtmem;
  // columns: THREADS / 128 warps per lane quarter, 2E columns (E complex) per thread
  // (M = 16384: a second block of 256 columns holds every thread's 31 pass-1 twiddles)
  // (GRAF_SOWN_TMEM_16384: the second block holds every thread's own samples s[t + eT] instead,
  // written once per kernel; the lag product and the correlation's second term then read
  // one sample per slot from L2 instead of two, and the pass-1 twiddles come from tab1)
  constexpr bool kSown = kTmem && (M == 16384) && !SPLIT && !CROSS && GRAF_SOWN_TMEM_16384 && (E == 32);
  constexpr bool kTwTmem = kTmem && !kSown && (M == 16384) && !SPLIT && GRAF_TW1_TMEM_16384 && (E == 32) &&
                           (num_passes(M, E) >= 2) && (pass_radix(M, E, 1) == 32);
  constexpr int kTmemNC = 2 * E * (THREADS / 128) * ((kTwTmem || kSown) ? 2 : 1);
  // (M = 8192, GRAF_ACC_TMEM_8192: the per-thread running sums of the loss partials live in 16
  // tensor-memory columns per thread instead of registers, loaded at each loss row's epilogue and
  // stored back, so they are not live, and not spilled to local memory, across the FFTs: with
  // two 105 KiB CTAs per SM the small L1 sends spill reloads to L2)
  constexpr bool kAccTm = (M == 8192) && !CROSS && (KIND != K_ADJ) && (S == 1) && GRAF_ACC_TMEM_8192;
  constexpr int kAccCol = kTmem ? kTmemNC : 0;                    // the running sums' column block
  constexpr int kAllocNC = kTmem ? (kAccTm ? 2 * kTmemNC : kTmemNC) : (kAccTm ? 16 * (THREADS / 128) : 0);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(red + 60);
  if constexpr (kTmem || kAccTm) {
    static_assert(THREADS % 128 == 0 && (E % 8) == 0, "TMEM accumulator layout: whole lane quarters");
    static_assert(kAllocNC == 32 || kAllocNC == 64 || kAllocNC == 128 || kAllocNC == 256 || kAllocNC == 512,
                  "TMEM allocation: a power of two >= 32 columns");
    if (warp == 0) tmem_alloc<kAllocNC>(tslot);
    tmem_fence_before();
  }
  // per-thread Doppler masks (depend on the slot's frequency m = t + e*T only)
  using Mask = typename std::conditional<(E > 32), unsigned long long, unsigned>::type;
  using VMask = Mask;
  // (M >= 8192, GRAF_LAZY_MASKS: not kept in registers across the FFTs; each use tests the
  // slot's |d| against the limit from the per-row copy of the thread index instead)
  constexpr bool kLazyMask = (M >= 8192) && GRAF_LAZY_MASKS;
  Mask band = 0, mlb = 0;
  if constexpr (!kLazyMask) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = t0 + e * T;
      const int d = m < M / 2 ? m : m - M;
      const int ad = d < 0 ? -d : d;
      band |= (Mask)(ad <= p.d_max ? 1 : 0) << e;
      mlb |= (Mask)(ad <= p.ml_d ? 1 : 0) << e;
    }
  }
  // |d| of slot e of thread tt (centred Doppler distance of frequency m = tt + e T)
  auto adop = [&](int tt, int e) {
    const int m = tt + e * T;
    const int d = m < M / 2 ? m : m - M;
    return d < 0 ? -d : d;
  };
  // split write-after-read barrier of the exchange buffer (one-slot CTAs; not when the
  // surface staging is aliased onto the exchange buffer, p.bulk == 2)
  const uint32_t war_mb = smem_u32(red + 62);
  const bool split_war = (S == 1) && (T >= 64) && GRAF_SPLIT_WAR && p.bulk != 2;
  if (split_war && threadIdx.x == 0) mbar_init(war_mb, THREADS / 32);
  __syncthreads();
  uint32_t tacc = 0;   // this thread's TMEM accumulator address (lane field | column)
  if constexpr (kTmem) {
    tmem_fence_after();
    tacc = *tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(2 * E * (warp >> 2));
    float z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0.f;
#pragma unroll
    for (int c = 0; c < E / 8; ++c) tmem_st16(tacc + 16 * c, z);
    if constexpr (kTwTmem) {
      // pass-1 twiddles W_M^(jm r (M / (NS1 R1))) with jm = t mod NS1 (the tab1 entries)
      constexpr int NS1 = pass_ns(M, E, 1), R1 = pass_radix(M, E, 1);
      const int jm = t0 & (NS1 - 1);
      const uint32_t ttw = tacc + kTmemNC / 2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float w16[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 8 * c + i + 1;
          const float2 w = r < R1 ? g_tw[(jm * r * (M / (NS1 * R1))) * (kMaxM / M)] : make_float2(0.f, 0.f);
          w16[2 * i] = w.x;
          w16[2 * i + 1] = w.y;
        }
        tmem_st16(ttw + 16 * c, w16);
      }
      tw.ttw = ttw;
    }
    if constexpr (kSown) {
      const float2* so = p.s_pad + (size_t)b * RP + NL + t0;   // zero beyond N
#pragma unroll
      for (int c = 0; c < E / 8; ++c) {
        float f16[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 x = so[(8 * c + i) * T];
          f16[2 * i] = x.x;
          f16[2 * i + 1] = x.y;
        }
        tmem_st16(tacc + kTmemNC / 2 + 16 * c, f16);
      }
    }
    tmem_wait_st();
  }
  uint32_t tacs = 0;   // kAccTm: this thread's 16 running-sum columns
  if constexpr (kAccTm) {
    if constexpr (!kTmem) tmem_fence_after();
    tacs = *tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(kAccCol + 16 * (warp >> 2));
  }
  const double Ed = red[0];
  // CROSS: normalisation by E1 E2 (reading R25); invE = 1/sqrt(E1 E2) for the surface
  const double Ed2 = CROSS ? red[1] : Ed;
  const float invE = CROSS ? (float)(1.0 / sqrt(Ed * Ed2)) : (float)(1.0 / Ed);
  const float invE2 = (float)(1.0 / Ed / Ed2);
  const float scaleG = p.normalize ? invE2 : 1.0f;

  // pass-2 statistics from the combined partials (reading R13)
  float lse = 0.f, ebar = 0.f, invZc = 0.f;
  bool use_centred = false;
  if (KIND == K_PASS2 && p.onepass) {
    use_centred = true;   // f' = lambda expm1((x - xbar)/T); 1/Z_c applied by the finalize
    invZc = 1.f;
  } else if constexpr (KIND == K_PASS2) {
    const graf_partials g = p.stats[b];
    // without a soft-PSL term the exp factor must vanish, not become 0 * inf
    lse = p.lam_psl != 0.f ? (float)(g.lse_max + (double)p.T * log(g.lse_sum)) : INFINITY;
    if (p.centred) {
      const double zc = p.omega + g.cen_sum;
      use_centred = isfinite(zc) && (g.lse_max - p.xbar) * p.invT <= 40.0;
      ebar = (float)(g.cen_sum / p.omega);
      invZc = (float)(1.0 / zc);
    }
  }
  const bool want_lse = FWD && p.loss_on && p.lam_psl != 0.f;

  SlotSync<T, S> sync{1 + slot};
  if (split_war) {
    sync.mb = war_mb;
    __syncwarp();
    if (lane == 0) mbar_arrive(war_mb);   // the buffer starts free: the first wait passes
  }
  float2* sh = xch + (size_t)slot * XS;
  // aliased staging (p.bulk == 2): the row lives in the slot's exchange buffer, which
  // is free between the last pass of one FFT and the first exchange of the next
  if (p.bulk == 2) stg = reinterpret_cast<float*>(sh);
  auto stg_release = [&]() {   // before an FFT reuses an aliased staging buffer
    if (p.bulk == 2) {
      if (t0 == 0) bulk_wait_read_all();
      sync();
    }
  };

  // per-thread accumulators (double across rows, float within a row)
  double accS = 0.0, accZ = 0.0, accC = 0.0, accF = 0.0, accMt = 0.0;
  float accM = -INFINITY;
  float argX = -INFINITY;   // hard-PSL argmax (value, key) of this thread
  int argK = 0x7fffffff;
  // kAccTm: [S, F, Z, C, Mt as (lo, hi) pairs, M, argX, argK] in the thread's 16 TMEM columns
  auto acc_store = [&]() {
    if constexpr (kAccTm) {
      float r[16];
      const double dv[5] = {accS, accF, accZ, accC, accMt};
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        r[2 * i] = __int_as_float(__double2loint(dv[i]));
        r[2 * i + 1] = __int_as_float(__double2hiint(dv[i]));
      }
      r[10] = accM;
      r[11] = argX;
      r[12] = __int_as_float(argK);
      r[13] = r[14] = r[15] = 0.f;
      tmem_st16(tacs, r);
    }
  };
  auto acc_load = [&]() {
    if constexpr (kAccTm) {
      tmem_wait_st();
      float r[16];
      tmem_ld16(tacs, r);
      tmem_wait_ld16(r);
      accS = __hiloint2double(__float_as_int(r[1]), __float_as_int(r[0]));
      accF = __hiloint2double(__float_as_int(r[3]), __float_as_int(r[2]));
      accZ = __hiloint2double(__float_as_int(r[5]), __float_as_int(r[4]));
      accC = __hiloint2double(__float_as_int(r[7]), __float_as_int(r[6]));
      accMt = __hiloint2double(__float_as_int(r[9]), __float_as_int(r[8]));
      accM = r[10];
      argX = r[11];
      argK = __float_as_int(r[12]);
    }
  };
  acc_store();

  const int rows_per_iter = P * S;
  const int iters = (p.U + rows_per_iter - 1) / rows_per_iter;
  const size_t surf_rows = (size_t)(p.ke - p.kb);
  const int lay = p.layout ? M / 2 : 0;

  for (int it = 0; it < iters; ++it) {
    const int t = launder(t0);   // per-row opaque copy of the thread index (see launder())
    const int u = it * rows_per_iter + pb * S + slot;
    const bool valid = u < p.U;
    const int k = p.row_lo + (valid ? u : 0) * p.row_step;
    // time support of the row (periodic rows use every n < N = M)
    const int lo = (k > 0 && !p.periodic) ? k : 0;
    const int hi = (k < 0 && !p.periodic) ? N + k : N;
    // slots e whose time index n lies in the row's support [lo, hi)
    VMask vmask;
    if constexpr (!SPLIT) {
      vmask = slot_range_mask(lo > t ? (lo - t + T - 1) >> LT : 0, hi > t ? (hi - t + T - 1) >> LT : 0);
    } else {
      // n = 2(t + j T) + par: j in [ceil((lo - par - 2t) / 2T), ceil((hi - par - 2t) / 2T))
      const int t2 = 2 * t;
      auto rng = [&](int par) {
        const int a = lo - par - t2, z = hi - par - t2;
        return slot_range_mask(a > 0 ? (a + 2 * T - 1) >> (LT + 1) : 0, z > 0 ? (z + 2 * T - 1) >> (LT + 1) : 0);
      };
      vmask = rng(0) | (rng(1) << E2);
    }
    float2 v[E];
    bool lrow;

    if constexpr (KIND != K_ADJ) {
      // ---- a1: lag product into the first-pass registers (time index n = t + e*T);
      //      s_pad makes out-of-support terms exactly zero
      // window rows of delays +k and -k (periodic: the window row holding that residue mod N)
      const int nrow = p.ke - p.kb;
      auto wrow = [&](int kk) {
        int q = kk - p.kb;
        if (p.periodic && (q < 0 || q >= nrow)) q += (q < 0 ? N : -N);
        return (q >= 0 && q < nrow) ? q : -1;
      };
      // (CROSS rows are unfolded: every row stands for itself)
      const bool self = CROSS || (k == 0) || (p.periodic && 2 * k == N);   // row -k is row +k
      const int rowp = wrow(k), rown = self ? -1 : wrow(-k);
      const bool wpos = valid && p.surface && rowp >= 0;
      const bool wneg = valid && p.surface && rown >= 0;
      lrow = valid && p.loss_on &&
             (CROSS ? (k <= p.kloss && -k <= p.kloss) : (k <= p.kloss && (k % p.shard_count) == p.shard_index));
      const float mult = self ? 1.f : 2.f;
      // pass 2 with the band cache: the row's in-band FFT outputs come from pass 1
      const bool cread = (KIND == K_PASS2) && p.cache == 2;
      float2* crow = p.acache + ((size_t)b * p.U + (valid ? u : 0)) * p.nband + p.d_max;
      if (cread) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (eb && e != 0 && e != E - 1) {
            v[e] = make_float2(0.f, 0.f);
            continue;
          }
          const int m = t + e * T;
          const int d = m < M / 2 ? m : m - M;
          v[e] = (valid && (kLazyMask ? adop(t, e) <= p.d_max : ((band >> e) & 1))) ? crow[d] : make_float2(0.f, 0.f);
        }
      } else {
      if constexpr (!SPLIT) {
        const float2* a = sv + t;
        const float2* c = sv2 + t - k;
        if (kHalfSizes && half) {
          // zero-padded row (2N <= M): the samples n = t + eT >= M/2 >= N are zero
#pragma unroll
          for (int e = 0; e < E / 2; ++e) {
            if constexpr (kStrim) {   // unpadded s: loads only inside the row's support
              float2 x = make_float2(0.f, 0.f), y = x;
              if ((vmask >> e) & 1) {
                x = a[e * T];
                y = c[e * T];
              }
              v[e] = cmulc(x, y);
            } else {
              v[e] = cmulc(a[e * T], c[e * T]);
            }
          }
#pragma unroll
          for (int e = E / 2; e < E; ++e) v[e] = make_float2(0.f, 0.f);
        } else if constexpr (!C::S_SMEM || kStrim) {
          // global s copy (M = 16384) or the unpadded smem copy (M = 8192): slots outside the
          // row's support load nothing; their lag products are exactly zero
          if constexpr (kSown) {
            // s[n] from this thread's tensor-memory copy, s[n - k] from L2: every load of the
            // row is issued before the first tcgen05.ld (whose memory clobber orders them)
            // (predicated to the row's support: unconditional loads from the zero padding
            // measured slower, 13.52 vs 12.96 ms, profiles/r02/tune_c5_sown_affine.txt)
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = ((vmask >> e) & 1) ? c[e * T] : make_float2(0.f, 0.f);
#pragma unroll
            for (int cc = 0; cc < E / 8; ++cc) {
              float xs[16];
              tmem_ld16(tacc + kTmemNC / 2 + 16 * cc, xs);
              tmem_wait_ld16(xs);
#pragma unroll
              for (int i = 0; i < 8; ++i) v[8 * cc + i] = cmulc(make_float2(xs[2 * i], xs[2 * i + 1]), v[8 * cc + i]);
            }
          } else
#pragma unroll
          for (int e = 0; e < E; ++e) {
#ifdef GRAF_ABL_NO_LAG   // timing ablation only (scripts/tune.py): no loads, synthetic row
            v[e] = make_float2(1e-3f * (float)(t + e), 1e-3f * (float)k);
            continue;
#endif
            float2 x = make_float2(0.f, 0.f), y = x;
            if ((vmask >> e) & 1) {
              x = a[e * T];
              y = c[e * T];
            }
            v[e] = cmulc(x, y);
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) v[e] = cmulc(a[e * T], c[e * T]);
        }
      } else {
        // slots e and e + E2 hold the adjacent samples 2(t + eT) and 2(t + eT) + 1: one
        // 16-byte load of the pair (s_pad rows are 16-byte aligned; the shifted factor
        // only when k is even)
        const float2* a = sv + 2 * t;
        const float2* c = sv2 + 2 * t - k;
        const float4* a4 = reinterpret_cast<const float4*>(a);
        // (odd k: the shifted copy holds s[2t - k + 2eT] at an even, aligned, position)
        const float4* c4 = reinterpret_cast<const float4*>((k & 1) == 0 ? c : sv_o + 2 * t - k);
#pragma unroll
        for (int e = 0; e < E2; ++e) {
#ifdef GRAF_ABL_NO_LAG   // timing ablation only (scripts/tune.py): no loads, synthetic row
          v[e] = make_float2(1e-3f * (float)(t + e), 1e-3f);
          v[e + E2] = make_float2(1e-3f, 1e-3f * (float)e);
          continue;
#endif
          // pairs outside the row's support [lo, hi) are zero: no loads (about half of
          // the pairs of a full-plane row)
          if ((((vmask >> e) | (vmask >> (e + E2))) & 1) == 0) {
            v[e] = make_float2(0.f, 0.f);
            v[e + E2] = make_float2(0.f, 0.f);
            continue;
          }
          const float4 x = a4[e * T], y = c4[e * T];
          v[e] = cmulc(make_float2(x.x, x.y), make_float2(y.x, y.y));
          v[e + E2] = cmulc(make_float2(x.z, x.w), make_float2(y.z, y.w));
        }
      }
      // ---- a2: forward Doppler FFT (a loss pass over a band narrower than T bins with
      //      no surface output needs slots 0 and E - 1 only: the last pass is pruned)
      stg_release();
      if constexpr (kEdgeFwd) {
        if (eb && p.surface == nullptr) {
          if (half) fft_rows_edges<M, E, 0, true>(v, sh, t, tw, sync);
          else fft_rows_edges<M, E, 0, false>(v, sh, t, tw, sync);
        }
        else row_fft<M, E, SPLIT, false>(v, sh, t, tw, sync, wt);
      } else {
#ifndef GRAF_ABL_NO_FWD   // timing ablation only
        row_fft<M, E, SPLIT, false>(v, sh, t, tw, sync, wt);
#endif
      }
      asm volatile("" ::: "memory");
      if (FWD && p.cache == 1 && lrow) {
        // pass 1: keep the loss band of this row for pass 2
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (eb && e != 0 && e != E - 1) continue;
          const int m = t + e * T;
          const int d = m < M / 2 ? m : m - M;
          if (kLazyMask ? adop(t, e) <= p.d_max : ((band >> e) & 1)) crow[d] = v[e];
        }
      }
      }

      // ---- a3F: surface epilogue (rows +k and, folded, -k)
      if (FLV >= 1) {
      } else if (p.bulk) {
        // dedicated staging: the slot's previous bulk copies must have finished reading it
        if (p.bulk == 1) {
          if (t0 == 0) bulk_wait_read_all();
          sync();
        }
        // Rows are staged in natural frequency order: row +k at q = m, row -k at
        // q = (-m) mod M (A[-k, -m] from A[k, m]); the Doppler layout is applied by
        // the copies (centred: the two halves swap).  Only slot e = 0 can hold m = 0,
        // so every other slot's staging address is affine in t.
        bool wr = wpos || wneg;
        if constexpr (T < 32) wr = __any_sync(0xffffffffu, wr);   // slot syncs below are warp-wide
        if (wr) {
          const float nrm = p.norm_out ? invE : 1.f;
          if (p.out_kind == GRAF_OUT_C64) {
            float2* sp = reinterpret_cast<float2*>(stg);
            float2* sn = sp + M;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const int m = t + e * T;
              if (wpos) sp[m] = cscale(v[e], nrm);
              if (wneg) {
                const float2 w = g_tw[(int)(((long long)m * k) & (M - 1)) * (kMaxM / M)];
                sn[e == 0 ? (M - t) & (M - 1) : M - t - e * T] = cscale(cconj(cmulc(v[e], w)), nrm);
              }
            }
          } else {
            const bool absk = p.out_kind == GRAF_OUT_ABS_F32;
            const float sc = absk ? nrm : nrm * nrm;
            float* sp = stg;
            float* sn = stg + M;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const float chi = v[e].x * v[e].x + v[e].y * v[e].y;
              const float val = (absk ? sqrt_approx(chi) : chi) * sc;
              if (wpos) sp[t + e * T] = val;
              if (wneg) sn[e == 0 ? (M - t) & (M - 1) : M - t - e * T] = val;
            }
          }
          fence_async_shared();
          sync();
          if (t0 == 0 && (wpos || wneg)) {
            const unsigned rb = (unsigned)(p.stg_floats / 2) * 4u;   // bytes per staged row
            const char* sp = reinterpret_cast<const char*>(stg);
            char* out = reinterpret_cast<char*>(p.surface);
            auto put = [&](char* dst, const char* src) {
              if (lay) {   // centred: column c <- q = (c - M/2) mod M
                bulk_store(dst, src + rb / 2, rb / 2);
                bulk_store(dst + rb / 2, src, rb / 2);
              } else {
                bulk_store(dst, src, rb);
              }
            };
            if (wpos) put(out + ((size_t)b * surf_rows + (rowp < 0 ? 0 : rowp)) * rb, sp);
            if (wneg) put(out + ((size_t)b * surf_rows + (rown < 0 ? 0 : rown)) * rb, sp + rb);
            bulk_commit();
          }
        }
      } else if (wpos || wneg) {
        const float nrm = p.norm_out ? invE : 1.f;
        // column of frequency m in row +k: (m + lay) mod M; in row -k: (lay - m) mod M
        if (p.out_kind == GRAF_OUT_C64) {
          float2* out = reinterpret_cast<float2*>(p.surface);
          float2* rp = out + ((size_t)b * surf_rows + (rowp < 0 ? 0 : rowp)) * M;
          float2* rn = out + ((size_t)b * surf_rows + (rown < 0 ? 0 : rown)) * M;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int m = t + e * T;
            if (wpos) __stcs(rp + t + (e < E / 2 ? e * T + lay : e * T - lay), cscale(v[e], nrm));
            if (wneg) {
              // A[-k, -m] = e^{-2 pi i m k / M} conj(A[k, m]) = conj(W^{-mk} A) with W^{-mk} = conj(g_tw)
              const float2 w = g_tw[(int)(((long long)m * k) & (M - 1)) * (kMaxM / M)];
              __stcs(rn + ((lay - m) & (M - 1)), cscale(cconj(cmulc(v[e], w)), nrm));
            }
          }
        } else {
          float* out = reinterpret_cast<float*>(p.surface);
          float* rp = out + ((size_t)b * surf_rows + (rowp < 0 ? 0 : rowp)) * M;
          float* rn = out + ((size_t)b * surf_rows + (rown < 0 ? 0 : rown)) * M;
          const bool absk = p.out_kind == GRAF_OUT_ABS_F32;
          const float sc = absk ? nrm : nrm * nrm;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int m = t + e * T;
            const float chi = v[e].x * v[e].x + v[e].y * v[e].y;
            const float val = (absk ? sqrt_approx(chi) : chi) * sc;
            if (wpos) __stcs(rp + t + (e < E / 2 ? e * T + lay : e * T - lay), val);
            if (wneg) __stcs(rn + ((lay - m) & (M - 1)), val);
          }
        }
      }

      // ---- a3L (+ a5): loss partials and the cotangent.  Branch-free over the
      //      slots: out-of-region slots select 0 (never multiply: exp of an
      //      out-of-region value may overflow).
      if (lrow) {
        acc_load();
        const Mask inm = band & ~((k < 0 ? -k : k) <= p.ml_k ? mlb : (Mask)0);   // (CROSS rows may be k < 0)
        const bool kml = (k < 0 ? -k : k) <= p.ml_k;                            // (kLazyMask)
        auto in_region = [&](int e) -> bool {
          if constexpr (kLazyMask) {
            const int ad = adop(t, e);
            return ad <= p.d_max && !(kml && ad <= p.ml_d);
          } else {
            return (inm >> e) & 1;
          }
        };
        const float wk = WGT && p.w_k ? p.w_k[k + N - 1] : 1.f;
        float rowS = 0.f, rowM = -INFINITY, rowF = 0.f, rowMt = 0.f, rowC1 = 0.f, rowM1 = -INFINITY, rowX = 0.f;
        const float gsc = scaleG * mult;
        // ISL cotangent factors inside / outside the region (complement form: f' = -lambda_isl
        // on the excluded mainlobe block only, nothing inside)
        const float isl_in = p.complement ? 0.f : p.lam_isl * gsc;
        const float lam_isl_in = (p.const_sum || p.complement) ? 0.f : p.lam_isl;   // pass 2
        const float lam_isl_out = p.complement ? -p.lam_isl : 0.f;
        const float isl_out = p.complement ? -p.lam_isl * gsc : 0.f;
        if constexpr (KIND == K_ISL) {
          // complement form: sum f' chi over the excluded cells = -lambda_isl sum chi over the
          // mainlobe block, present in rows |k| <= ml_k only (before G overwrites v)
          if (p.complement && (k < 0 ? -k : k) <= p.ml_k) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const float chi = v[e].x * v[e].x + v[e].y * v[e].y;
              rowX += (kLazyMask ? adop(t, e) <= p.ml_d : ((mlb >> e) & 1)) ? chi : 0.f;
            }
          }
        }
        // match targets of rows +k and -k (K_MATCH; the host checked the window holds them)
        const float* tgp = nullptr;
        const float* tgn = nullptr;
        if constexpr (KIND == K_MATCH) {
          const float* tb0 = p.target + (size_t)b * p.target_stride;
          tgp = tb0 + (size_t)(rowp < 0 ? 0 : rowp) * M;
          tgn = tb0 + (size_t)(rown < 0 ? 0 : rown) * M;
        }
        // Full-plane centred single pass (R13; c5's loss), fast form.  The region is the whole
        // plane minus the origin, so only slot 0 of thread 0 in row 0 is outside it.  When
        // every u = (x - xbar)/T of this warp's row lies in (-1/8, 1/8) (c5: |u| < 0.11),
        // expm1(u) = u (1 + u/2 + u^2/6 + u^3/24 + u^4/120) to < 5e-8 relative, with no MUFU
        // and no selects; otherwise the general loop below runs.
        // (T >= 32: a warp works on one row, so the vote below is warp-uniform; with T < 32
        // the lanes of a warp hold different rows and some may skip this block)
        bool fast_done = false;
        if constexpr (KIND == K_PASS2 && !WGT && !CROSS && T >= 32) {
          if (p.onepass) {
            const bool in0 = !(k == 0 && t0 == 0);          // the origin cell (k, m) = (0, 0)
            float mchi = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const float chi = fmaf(v[e].y, v[e].y, v[e].x * v[e].x);
              mchi = fmaxf(mchi, (e == 0 && !in0) ? 0.f : chi);
            }
            const float cu = invE2 * p.invT, cb = -p.xbar * p.invT;
            const bool ok = (-cb < 0.125f) && (fmaf(mchi, cu, cb) < 0.125f);
            if (__all_sync(0xffffffffu, ok)) {
#ifdef GRAF_MUTATE_NO_PSL   // mutation check only: drop the soft-PSL term of f'
              const float gl = 0.f;
#else
              const float gl = p.lam_psl * gsc;
#endif
              float sS = 0.f, sC = 0.f, sF = 0.f;
#pragma unroll
              for (int e = 0; e < E; ++e) {
                const float chi = fmaf(v[e].y, v[e].y, v[e].x * v[e].x);
                const float u = fmaf(chi, cu, cb);
                const float q = fmaf(u, fmaf(u, fmaf(u, fmaf(u, 1.f / 120.f, 1.f / 24.f), 1.f / 6.f), 0.5f), 1.f);
                float ec = u * q;
                float ch = chi;
                if (e == 0) {   // (compile-time slot: the origin test costs two selects per row)
                  ec = in0 ? ec : 0.f;
                  ch = in0 ? chi : 0.f;
                }
                sS += ch;
                sC += ec;
                sF = fmaf(ec, chi, sF);
                const float sc = ec * gl;
                v[e] = make_float2(v[e].x * sc, v[e].y * sc);
              }
              rowS = sS;
              rowC1 = sC;
              rowF = p.lam_psl * sF;
              rowM1 = mchi * invE2;
              fast_done = true;
            }
          }
        }
        if (!fast_done) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (eb && e != 0 && e != E - 1) continue;   // outside the band: no term, G unused
          const bool in = in_region(e);
          float w = 1.f;
          if constexpr (WGT) {
            const int m = t + e * T;
            const int d = m < M / 2 ? m : m - M;
            w = wk * (p.w_d ? p.w_d[d + M / 2] : 1.f);
          }
          const float chi = v[e].x * v[e].x + v[e].y * v[e].y;
          rowS = fmaf(in ? w : 0.f, chi, rowS);
          if constexpr (FWD) {
            const float x = p.normalize ? chi * invE2 : chi;
            rowM = fmaxf(rowM, in ? x : -INFINITY);
            if constexpr (KIND == K_FWDA) {
              // canonical (row-major first) cell of the mirrored pair holding this value
              const int m = t + e * T;
              const int mm = (M - m) & (M - 1);
              const bool self = (k == 0) || (p.periodic && 2 * k == N);
              const int key = self ? (k - p.key_lo) * M + min(m, mm) : (-k - p.key_lo) * M + mm;
              const bool better = in && (x > argX || (x == argX && key < argK));
              argX = better ? x : argX;
              argK = better ? key : argK;
            }
          } else if constexpr (KIND == K_ISL) {
            v[e] = cscale(v[e], in ? isl_in * w : isl_out);   // G (x2 for a folded row pair)
          } else if constexpr (KIND == K_MATCH) {
            // f' of the folded pair (k, m), (-k, -m) / mult: lambda (2x - t1 - t2); a row that is
            // its own mirror uses t2 = t1
            const float x = p.normalize ? chi * invE2 : chi;
            const int m = t + e * T;
            const float t1 = tgp[(m + lay) & (M - 1)];
            const float t2 = self ? t1 : tgn[(lay - m) & (M - 1)];
            float fp = p.lam_isl * w + p.lam_match * (2.f * x - t1 - t2);
            fp = in ? fp : 0.f;
            rowF = fmaf(fp, chi, rowF);
            v[e] = cscale(v[e], fp * gsc);
            const float d1 = x - t1, d2 = self ? 0.f : x - t2;
            rowMt += in ? d1 * d1 + d2 * d2 : 0.f;
          } else {
            const float x = p.normalize ? chi * invE2 : chi;
            float fp;
            if (use_centred) {
              const float ec = expm1_fast((x - p.xbar) * p.invT);
              fp = p.lam_psl * (ec - ebar) * invZc;
#ifdef GRAF_MUTATE_NO_PSL
              fp = 0.f;
#endif
              rowC1 += in ? ec : 0.f;                      // (single pass: Z_c and the validity max)
              rowM1 = fmaxf(rowM1, in ? x : -INFINITY);
            } else {
              fp = lam_isl_in * w + p.lam_psl * exp_fast((x - lse) * p.invT);   // lse = +inf without soft-PSL
#ifdef GRAF_MUTATE_NO_PSL
              fp = p.lam_isl * w;
#endif
            }
            fp = in ? fp : lam_isl_out;
            rowF = fmaf(fp, chi, rowF);
            v[e] = cscale(v[e], fp * gsc);
          }
        }
        }
        if constexpr (KIND == K_ISL) rowF = p.complement ? -p.lam_isl * rowX : p.lam_isl * rowS;
        accS += (double)(mult * rowS);
        accF += (double)(mult * rowF);
        if constexpr (KIND == K_MATCH) accMt += (double)rowMt;
        if constexpr (KIND == K_PASS2) {
          if (p.onepass) {
            accC += (double)(mult * rowC1);
            accM = fmaxf(accM, rowM1);
          }
        }
        if constexpr (FWD) {
          if (want_lse && rowM > -INFINITY) {
            if (rowM > accM) {
              accZ = (accM == -INFINITY) ? 0.0 : accZ * (double)exp_fast((accM - rowM) * p.invT);
              accM = rowM;
            }
            float rowZ = 0.f, rowC = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              if (eb && e != 0 && e != E - 1) continue;
              const bool in = in_region(e);
              const float chi = v[e].x * v[e].x + v[e].y * v[e].y;
              const float x = p.normalize ? chi * invE2 : chi;
              const float z = exp_fast((x - accM) * p.invT);
              rowZ += in ? z : 0.f;
              if (p.centred) {
                const float c = expm1_fast((x - p.xbar) * p.invT);
                rowC += in ? c : 0.f;
              }
            }
            accZ += (double)(mult * rowZ);
            accC += (double)(mult * rowC);
          } else {
            accM = fmaxf(accM, rowM);
          }
        }
        acc_store();
      } else if constexpr (GRAD) {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = make_float2(0.f, 0.f);
      }
    } else {
      // ---- K_ADJ: G = dA row (unfolded k = kb + u)
      lrow = valid;
      const float2* drow = p.dA + ((size_t)b * surf_rows + (k - p.kb)) * M + t;
#pragma unroll
      for (int e = 0; e < E; ++e)
        v[e] = valid ? __ldcs(drow + (e < E / 2 ? e * T + lay : e * T - lay)) : make_float2(0.f, 0.f);
    }

    // ---- a6 + a7: inverse Doppler FFT and the delay correlation
    if constexpr (GRAD) {
      bool do_adj = lrow;
      if constexpr (T < 32) do_adj = __any_sync(0xffffffffu, do_adj);
      if (do_adj) {
        stg_release();
        if constexpr (kEdgeBand) {
          if (edge_band) ifft_band_edges<M, E>(v, sh, t, tw, sync);
#ifndef GRAF_ABL_NO_INV   // timing ablation only
          else row_fft<M, E, SPLIT, true>(v, sh, t, tw, sync, wt);
#endif
        } else {
#ifndef GRAF_ABL_NO_INV   // timing ablation only
          row_fft<M, E, SPLIT, true>(v, sh, t, tw, sync, wt);
#endif
        }
        // keep the correlation's loads below the last inverse pass
        asm volatile("" ::: "memory");
        // term 1 at p = n: g[n] += H[n] s[n-k];  term 2 at p = n-k: g[n-k] += conj(H[n]) s[n],
        // for n in the row's support (vmask); each address is touched once per phase.
        const VMask m1 = lrow ? vmask : (VMask)0;
        // time offset of slot e relative to the thread's base index
        constexpr auto toff = [](int e) constexpr { return SPLIT ? (e < E2 ? 2 * e * T : 2 * (e - E2) * T + 1) : e * T; };
        const int tb = SPLIT ? 2 * t : t;
        // predicated shared-memory read-modify-writes (no branches; an out-of-support
        // slot neither loads nor stores its accumulator)
#ifdef GRAF_ABL_NO_CORR   // timing ablation only: keep v live, skip the correlation
        if constexpr (kTmem) {
          if (v[0].x == 1234.5f) p.gpart[t] = v[1];
        } else
#endif
        if constexpr (kTmem) {
          // Both terms accumulate at the thread's OWN positions p = t + eT, so the
          // accumulator is thread-private (TMEM):
          //   g[p] += H[k,p] s[p-k]             (p in the row's support [lo, hi))
          //         + conj(H[k,p+k]) s[p+k]      (p+k in [lo, hi): the shifted H from smem)
          // (periodic: every index mod N).  H goes through the exchange buffer once.
          // (a zero-padded row, 2N <= M: positions n >= M/2 >= N carry no support, so only
          // the lower half of the slots writes H or touches its accumulators)
          float2* hb = sh;
          const int nch = (kHalfSizes && half) ? E / 16 : E / 8;
          sync.before_writing();
          if constexpr (kSown) {
            // term 2 needs conj(H[q]) s[q] at q = p + k: form it at the owner of q (s[q] from
            // tensor memory) and pass the product through the exchange buffer
#pragma unroll
            for (int cc = 0; cc < E / 8; ++cc) {
              if (8 * cc >= 8 * nch) break;
              float xs[16];
              tmem_ld16(tacc + kTmemNC / 2 + 16 * cc, xs);
              tmem_wait_ld16(xs);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                hb[t + (8 * cc + i) * T] = cmulc(make_float2(xs[2 * i], xs[2 * i + 1]), v[8 * cc + i]);
            }
          } else {
#pragma unroll
            for (int e = 0; e < E; ++e)
              if (8 * nch > e) hb[t + e * T] = v[e];
          }
          sync();
          const bool per = p.periodic != 0;
          constexpr int CS = GRAF_TMEM_SLOTS;      // slots per chunk (2 CS columns)
          if (!per) {
            // aperiodic rows: term 1 of slot e reads s at (t - k) + eT, term 2 the exchange
            // buffer at (t + k) + eT: one base address each and immediate offsets; the
            // supports are two slot masks (p in [lo, hi) and p + k in [lo, hi)), no per-slot
            // index arithmetic
            const int lo2 = lo - k, hi2 = hi - k;
            const VMask m2 = lrow ? (VMask)slot_range_mask(lo2 > t ? (lo2 - t + T - 1) >> LT : 0,
                                                           hi2 > t ? (hi2 - t + T - 1) >> LT : 0)
                                  : (VMask)0;
            const float2* s1p = sv + t - k;
            const float2* s2p = sv + t + k;
            const float2* h2p = hb + t + k;
#pragma unroll
            for (int c = 0; c < E / CS; ++c) {
              if (c * CS >= 8 * nch) break;
              float acc[2 * CS], d[2 * CS];
              tmem_ldc<2 * CS>(tacc + 2 * CS * c, acc);
#pragma unroll
              for (int i = 0; i < CS; ++i) {
                const int e = CS * c + i;
                float2 s1 = make_float2(0.f, 0.f), s2 = s1, h2 = s1;
                if ((m1 >> e) & 1) s1 = s1p[e * T];
                if ((m2 >> e) & 1) {
                  if constexpr (!kSown) s2 = s2p[e * T];
                  h2 = h2p[e * T];
                }
                const float2 a1 = cmul(v[e], s1);
                const float2 a2 = kSown ? h2 : cmulc(s2, h2);
                d[2 * i] = a1.x + a2.x;
                d[2 * i + 1] = a1.y + a2.y;
              }
              tmem_wait_ldc<2 * CS>(acc);
#pragma unroll
              for (int i = 0; i < 2 * CS; ++i) acc[i] += d[i];
              tmem_stc<2 * CS>(tacc + 2 * CS * c, acc);
            }
          } else
#pragma unroll
          for (int c = 0; c < E / CS; ++c) {
            if (c * CS >= 8 * nch) break;
            float acc[2 * CS], d[2 * CS];
            tmem_ldc<2 * CS>(tacc + 2 * CS * c, acc);   // in flight while this chunk's terms are formed
#pragma unroll
            for (int i = 0; i < CS; ++i) {
              const int e = CS * c + i;
              const int pp = t + e * T;
              const int q1 = per ? ((pp - k) & (N - 1)) : pp - k;            // s index, term 1
              const int q2 = per ? ((pp + k) & (N - 1)) : pp + k;            // H and s index, term 2
              const bool in1 = lrow && (per || (pp >= lo && pp < hi));
              const bool in2 = lrow && (per || (q2 >= lo && q2 < hi));
              float2 s1 = make_float2(0.f, 0.f), s2 = s1, h2 = s1;
              if (in1) s1 = sv[q1];
              if (in2) {
                if constexpr (!kSown) s2 = sv[q2];
                h2 = hb[q2];
              }
              const float2 a1 = cmul(v[e], s1);
              const float2 a2 = kSown ? h2 : cmulc(s2, h2);      // conj(H) s
              d[2 * i] = a1.x + a2.x;
              d[2 * i + 1] = a1.y + a2.y;
            }
            tmem_wait_ldc<2 * CS>(acc);
#pragma unroll
            for (int i = 0; i < 2 * CS; ++i) acc[i] += d[i];
            tmem_stc<2 * CS>(tacc + 2 * CS * c, acc);
          }
          sync.done_reading();   // H has been read: the next row's first pass may overwrite it
          tmem_wait_st();
        } else if (p.periodic) {
          // circular lag products (M == N): every slot is in the support; term 1 reads
          // s[(n - k) mod N] from the periodic copy in s_pad, term 2 wraps its position.
          const int kc = k < 0 ? k + N : k;   // K_ADJ rows may be negative delays
          {
            float2* g1 = gacc + tb;
            const float2* s1 = sv + tb - kc;
#pragma unroll
            for (int e = 0; e < E; ++e) g1[toff(e)] = cadd(g1[toff(e)], cmul(v[e], s1[toff(e)]));
          }
          sync();
          {
            const float2* s2 = sv + tb;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              float2* gq = gacc + ((tb + toff(e) - kc) & (N - 1));
              *gq = cadd(*gq, cmulc(s2[toff(e)], v[e]));
            }
          }
        } else if (KIND != K_ADJ && kGpadSizes && p.gpad) {
          // M == N, k >= 0: every term-1 position n < N is in the slot's range and
          // s[n - k] = 0 below the support; term-2 positions n - k >= -k land in the
          // left pad when n < k.  No predicates.
          {
            float2* g1 = gacc + tb;
            const float2* s1 = sv + tb - k;
#pragma unroll
            for (int e = 0; e < E; ++e) g1[toff(e)] = cadd(g1[toff(e)], cmul(v[e], s1[toff(e)]));
          }
          sync();
          {
            float2* g2 = gacc + tb - k;
            const float2* s2 = sv + tb;
#pragma unroll
            for (int e = 0; e < E; ++e) g2[toff(e)] = cadd(g2[toff(e)], cmulc(s2[toff(e)], v[e]));
          }
#ifdef GRAF_ABL_NO_CORR
        } else if constexpr (SPLIT) {   // timing ablation only: keep v live, skip the correlation
          if (v[0].x == 1234.5f) gacc[t] = v[1];
#endif
        } else if constexpr (SPLIT && !CROSS) {
          // SPLIT rows: process the slot pairs (j, j + E2) = samples (2(t + jT), 2(t + jT) + 1)
          // together so the global s reads are 16-byte pair loads (term 2 always, term 1
          // when k is even)
          constexpr int CP = (E < kCorrChunk ? E : kCorrChunk) / 2;
          const bool even = (k & 1) == 0;
          {
            const unsigned g1 = smem_u32(gacc + tb);
            const float2* s1 = sv2 + tb - k;
            static_for<0, E2 / CP>([&](auto c) {
              constexpr int j0 = decltype(c)::value * CP;
              constexpr VMask cbits = (((VMask)1 << CP) - 1) << j0;
              if ((m1 & (cbits | (cbits << E2))) == 0) return;   // no slot of this chunk in the support
              float2 a[2 * CP], sl[2 * CP];
              static_for<0, CP>([&](auto i) {
                constexpr int j = j0 + decltype(i)::value;
                a[2 * decltype(i)::value] = ld_shared_if<8 * toff(j)>(g1, (m1 >> j) & 1);
                a[2 * decltype(i)::value + 1] = ld_shared_if<8 * toff(j + E2)>(g1, (m1 >> (j + E2)) & 1);
              });
              // (odd k: from the shifted copy, where the pair is aligned too)
              const float4* s14 = reinterpret_cast<const float4*>(even ? s1 : sv_o + tb - k);
              static_for<0, CP>([&](auto i) {
                constexpr int j = j0 + decltype(i)::value;
                const float4 q = s14[j * T];
                sl[2 * decltype(i)::value] = make_float2(q.x, q.y);
                sl[2 * decltype(i)::value + 1] = make_float2(q.z, q.w);
              });
              static_for<0, CP>([&](auto i) {
                constexpr int j = j0 + decltype(i)::value;
                constexpr int ii = 2 * decltype(i)::value;
                st_shared_if<8 * toff(j)>(g1, cadd(a[ii], cmul(v[j], sl[ii])), (m1 >> j) & 1);
                st_shared_if<8 * toff(j + E2)>(g1, cadd(a[ii + 1], cmul(v[j + E2], sl[ii + 1])), (m1 >> (j + E2)) & 1);
              });
            });
          }
          sync();
          {
            const unsigned g2 = smem_u32(gacc + tb - k);
            const float4* s2 = reinterpret_cast<const float4*>(sv + tb);
            static_for<0, E2 / CP>([&](auto c) {
              constexpr int j0 = decltype(c)::value * CP;
              constexpr VMask cbits = (((VMask)1 << CP) - 1) << j0;
              if ((m1 & (cbits | (cbits << E2))) == 0) return;
              float2 a[2 * CP];
              float4 q[CP];
              static_for<0, CP>([&](auto i) {
                constexpr int j = j0 + decltype(i)::value;
                a[2 * decltype(i)::value] = ld_shared_if<8 * toff(j)>(g2, (m1 >> j) & 1);
                a[2 * decltype(i)::value + 1] = ld_shared_if<8 * toff(j + E2)>(g2, (m1 >> (j + E2)) & 1);
                q[decltype(i)::value] = s2[j * T];
              });
              static_for<0, CP>([&](auto i) {
                constexpr int j = j0 + decltype(i)::value;
                constexpr int ii = 2 * decltype(i)::value;
                const float4 x = q[decltype(i)::value];
                st_shared_if<8 * toff(j)>(g2, cadd(a[ii], cmulc(make_float2(x.x, x.y), v[j])), (m1 >> j) & 1);
                st_shared_if<8 * toff(j + E2)>(g2, cadd(a[ii + 1], cmulc(make_float2(x.z, x.w), v[j + E2])),
                                               (m1 >> (j + E2)) & 1);
              });
            });
          }
        } else {
          constexpr int CC = E < kCorrChunk ? E : kCorrChunk;
          // NCH chunks of CC slots; a zero-padded row (2N <= M) has no support in the upper
          // half of the slots (n >= M/2 >= N), so it runs the lower half only
          auto corr = [&](auto nch) {
            constexpr int NCH = decltype(nch)::value;
            {
              // CROSS: term 1 is dL/ds* with the conjugated factor s2[n-k]
              const unsigned g1 = smem_u32(gacc + tb);
              const float2* s1 = sv2 + tb - k;
              static_for<0, NCH>([&](auto c) {
                constexpr int e0 = decltype(c)::value * CC;
                if ((m1 & ((((VMask)1 << CC) - 1) << e0)) == 0) return;   // chunk outside the support
                float2 a[CC];
                static_for<0, CC>([&](auto i) {
                  constexpr int e = e0 + decltype(i)::value;
                  a[decltype(i)::value] = ld_shared_if<8 * toff(e)>(g1, (m1 >> e) & 1);
                });
                static_for<0, CC>([&](auto i) {
                  constexpr int e = e0 + decltype(i)::value;
                  st_shared_if<8 * toff(e)>(g1, cadd(a[decltype(i)::value], cmul(v[e], s1[toff(e)])), (m1 >> e) & 1);
                });
              });
            }
            sync();
            {
              // CROSS: term 2 is dL/ds2* (its own accumulator) with s[n]
              const unsigned g2 = smem_u32((CROSS ? gacc2 : gacc) + tb - k);
              const float2* s2 = sv + tb;
              static_for<0, NCH>([&](auto c) {
                constexpr int e0 = decltype(c)::value * CC;
                if ((m1 & ((((VMask)1 << CC) - 1) << e0)) == 0) return;   // chunk outside the support
                float2 a[CC];
                static_for<0, CC>([&](auto i) {
                  constexpr int e = e0 + decltype(i)::value;
                  a[decltype(i)::value] = ld_shared_if<8 * toff(e)>(g2, (m1 >> e) & 1);
                });
                static_for<0, CC>([&](auto i) {
                  constexpr int e = e0 + decltype(i)::value;
                  st_shared_if<8 * toff(e)>(g2, cadd(a[decltype(i)::value], cmulc(s2[toff(e)], v[e])), (m1 >> e) & 1);
                });
              });
            }
          };
          if constexpr (kHalfSizes && (E / CC) % 2 == 0) {
            if (half) corr(std::integral_constant<int, E / CC / 2>{});
            else corr(std::integral_constant<int, E / CC>{});
          } else {
            corr(std::integral_constant<int, E / CC>{});
          }
        }
        // (the TMEM branch released the buffer with done_reading(); shared-memory
        // accumulators need the full barrier before the next row's read-modify-writes)
        if (!kTmem) sync();
      }
    }
  }

  // ---- CTA reduction of the scalar partials -> part[b][pb] (or, fused, shared memory)
  if (p.bulk && t0 == 0) bulk_wait_all();
  __syncthreads();
  double* scratch = reinterpret_cast<double*>(xch);  // exchange space is free now
  double* rec = p.fuse ? red + 8 : p.part + ((size_t)b * P + pb) * kPart;
  if constexpr (KIND != K_ADJ) {
    acc_load();
    const double S0 = block_sum<THREADS>(accS, scratch);
    const double F0 = block_sum<THREADS>(accF, scratch);
    double Z0 = 0.0, C0 = 0.0;
    float M0 = -INFINITY;
    if constexpr (KIND == K_PASS2) {
      if (p.onepass) {
        M0 = block_max_all<THREADS>(accM, scratch);
        C0 = block_sum<THREADS>(accC, scratch);
      }
    }
    if constexpr (FWD) {
      M0 = block_max_all<THREADS>(accM, scratch);
      if (want_lse) {
        const double zs = (accM == -INFINITY) ? 0.0 : accZ * (double)exp_fast((accM - M0) * p.invT);
        Z0 = block_sum<THREADS>(zs, scratch);
        C0 = block_sum<THREADS>(accC, scratch);
      }
    }
    int K0 = 0x7fffffff;
    if constexpr (KIND == K_FWDA) K0 = block_argmax_key<THREADS>(argX, argK, scratch);
    double Mt0 = 0.0;
    if constexpr (KIND == K_MATCH) Mt0 = block_sum<THREADS>(accMt, scratch);
    if (threadIdx.x == 0) {
      rec[0] = S0;
      rec[1] = (double)M0;
      rec[2] = Z0;
      rec[3] = C0;
      rec[4] = F0;
      rec[5] = (double)K0;
      rec[6] = Mt0;
    }
  } else {
    if (threadIdx.x == 0) {
      rec[0] = 0.0;
      rec[1] = -INFINITY;
      rec[2] = 0.0;
      rec[3] = 0.0;
      rec[4] = 0.0;
      rec[5] = (double)0x7fffffff;
      rec[6] = 0.0;
    }
  }

  // ---- TMEM accumulator -> this CTA's partial g (thread-private: no ordering question),
  //      then the TMEM columns go back
  if constexpr (kTmem) {
    float2* gout = p.gpart + ((size_t)b * P + pb) * N;
    // one row slot: the thread's columns ARE the CTA's partial gradient; several slots (M =
    // 1024: four rows per CTA, a warp each): every slot's columns go to the free exchange
    // space as [slot][N], then a fixed-order sum over the slots (deterministic)
    float2* gb = S == 1 ? gout : xch + (size_t)slot * N;
#pragma unroll
    for (int c = 0; c < E / 8; ++c) {
      float acc[16];
      tmem_ld16(tacc + 16 * c, acc);
      tmem_wait_ld16(acc);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int n = t0 + (8 * c + i) * T;
        if (n < N) gb[n] = make_float2(acc[2 * i], acc[2 * i + 1]);
      }
    }
    if constexpr (S > 1) {
      static_assert(S == 1 || XS >= 1, "");
      __syncthreads();
      for (int n = threadIdx.x; n < N; n += THREADS) {
        float2 a = xch[n];
#pragma unroll 1
        for (int sl = 1; sl < S; ++sl) a = cadd(a, xch[(size_t)sl * N + n]);
        gout[n] = a;
      }
    }
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
      tmem_fence_after();
      tmem_dealloc<kAllocNC>(*tslot);
    }
  } else if constexpr (kAccTm) {
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
      tmem_fence_after();
      tmem_dealloc<kAllocNC>(*tslot);
    }
  }

  // ---- gradient accumulators of all slots -> this CTA's partial g (fixed slot order)
  if constexpr (GRAD && kGsmem) {
    float2* gout = p.fuse ? gacc_sh + (p.gpad ? N : 0) : p.gpart + ((size_t)b * P + pb) * N;
    for (int n = threadIdx.x; n < N; n += THREADS) {
      const float2* g0 = gacc_sh + (p.gpad ? N : 0) + n;
      float2 a = g0[0];
#pragma unroll 1
      for (int sl = 1; sl < S; ++sl) a = cadd(a, g0[(size_t)sl * GS]);
      gout[n] = a;   // fused: in place over slot 0 (each n is owned by one thread)
    }
    if constexpr (CROSS) {
      float2* gout2 = p.gpart2 + ((size_t)b * P + pb) * N;
      for (int n = threadIdx.x; n < N; n += THREADS) {
        const float2* g0 = gacc_sh + (size_t)S * GS + n;
        float2 a = g0[0];
#pragma unroll 1
        for (int sl = 1; sl < S; ++sl) a = cadd(a, g0[(size_t)sl * GS]);
        gout2[n] = a;
      }
    }
  }

  // ---- fused finalize over the cluster (SURVEY §8(a) a4 + a7 final, K5)
  if constexpr (KIND == K_ISL && kGsmem) {
    if (p.fuse) {
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      cl.sync();   // every CTA's record and combined gradient are visible cluster-wide
      if (cl.block_rank() == 0) {
        const float2* gl = gacc_sh + (p.gpad ? N : 0);
        if (threadIdx.x == 0) {
          double St = 0.0, Ft = 0.0;
          for (int r = 0; r < P; ++r) {
            const double* rr = cl.map_shared_rank(red + 8, r);
            St += rr[0];
            Ft += rr[4];
          }
          const double Ed = red[0];
          if (p.loss_out) p.loss_out[b] = (double)p.lam_isl * (p.normalize ? St / (Ed * Ed) : St);
          red[16] = Ft;
        }
        __syncthreads();
        const double Ed = red[0];
        const float coef = p.normalize ? (float)(2.0 * red[16] / (Ed * Ed * Ed)) : 0.f;
        const float2* sg = p.s + (size_t)b * N;
        for (int n = threadIdx.x; n < N; n += THREADS) {
          double gx = 0.0, gy = 0.0;
          for (int r = 0; r < P; ++r) {
            const float2 a = *cl.map_shared_rank(gl + n, r);
            gx += a.x;
            gy += a.y;
          }
          const float2 sn = sg[n];
          p.grad_out[(size_t)b * N + n] = make_float2((float)gx - coef * sn.x, (float)gy - coef * sn.y);
        }
      }
      cl.sync();   // keep every CTA's shared memory alive until rank 0 has read it
    }
  }
}

#ifdef GRAF_API_UNIT   // the reductions and small kernels live in the ABI unit only
// zero-padded copy of s for the global-memory path: s_pad[b][i] = s[b][i - N] for
// i in [N, 2N), 0 elsewhere in [0, N + M)
// rows of NL + M + 2 samples, NL = N rounded up to even: s[n] at NL + n, zeros elsewhere
// (periodic: s[n + N] at NL + n for -N <= n < 0), so row starts and the origin are 16-byte
// aligned.  s_pad1 holds the same rows shifted by one sample (s[n] at NL + 1 + n), so a
// pair starting at an odd sample index is aligned there.
__global__ void pad_s_kernel(const float2* s, float2* s_pad, float2* s_pad1, int N, int M, long long B,
                             int periodic) {
  const int NL = N + (N & 1);
  const long long R = NL + M + 2;
  const long long total = B * R;
  auto val = [&](long long b, int n) {
    if (n >= 0 && n < N) return s[b * N + n];
    if (periodic && n < 0 && n >= -N) return s[b * N + n + N];
    return make_float2(0.f, 0.f);
  };
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / R;
    const int j = (int)(i - b * R);
    s_pad[i] = val(b, j - NL);
    s_pad1[i] = val(b, j - NL - 1);
  }
}

// ---------------------------------------------------------------------------
// K3: combine the P CTA partial records of each waveform -> graf_partials[B].
// One thread per waveform, fixed order.
// ---------------------------------------------------------------------------
struct ReduceParams {
  const double* part;
  int P, B;
  float invT, T;
  graf_partials* out;
  int onepass;   // records of the single pass: reserved = 1 where it is valid (R13 rule)
  float xbar;
  const int32_t* skip;   // skipped waveforms get identity partials (no stale records)
};

// one warp per waveform: lane l merges records l, l+32, ... in order, then a fixed
// shuffle-down tree merges the lanes (deterministic)
__device__ __forceinline__ void merge_rec(double& S, double& m, double& Z, double& Cs, double& key, double S2,
                                          double m2, double Z2, double C2, double key2, float T) {
  S += S2;
  Cs += C2;
  key_merge(m, key, m2, key2);
  lse_merge(m, Z, m2, Z2, T);
}

__global__ void partials_reduce_kernel(ReduceParams r) {
  const int b = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= r.B) return;   // warp-uniform
  double S = 0, Z = 0, Cs = 0, key = (double)0x7fffffff;
  double m = -INFINITY;
  const int P = (r.skip && r.skip[b]) ? 0 : r.P;
  for (int q = lane; q < P; q += 32) {
    const double* rec = r.part + ((size_t)b * r.P + q) * kPart;
    merge_rec(S, m, Z, Cs, key, rec[0], rec[1], rec[2], rec[3], rec[5], r.T);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double S2 = __shfl_down_sync(0xffffffffu, S, off), m2 = __shfl_down_sync(0xffffffffu, m, off);
    const double Z2 = __shfl_down_sync(0xffffffffu, Z, off), C2 = __shfl_down_sync(0xffffffffu, Cs, off);
    const double k2 = __shfl_down_sync(0xffffffffu, key, off);
    if (lane + off < 32) merge_rec(S, m, Z, Cs, key, S2, m2, Z2, C2, k2, r.T);
  }
  if (lane == 0) {
    graf_partials g;
    g.isl_sum = S;
    g.lse_max = m;
    g.lse_sum = Z;
    g.cen_sum = Cs;
    g.psl_key = key;
    g.reserved = (r.onepass && isfinite(Cs) && isfinite(m) && (m - (double)r.xbar) * (double)r.invT <= 40.0) ? 1.0 : 0.0;
    r.out[b] = g;
  }
}

// ---------------------------------------------------------------------------
// K5: finalize — g[b] = sum_q gpart[b][q] (fixed order) - (2/E^3)(sum f' chi) s
// and loss[b] (from `global` partials, else from this call's own partials).
// ---------------------------------------------------------------------------
struct FinalizeParams {
  const float2* s;
  const double* part;
  const float2* gpart;
  const graf_partials* global;   // may be NULL
  int P, N, B;
  int normalize, grad_norm_term;
  float lam_isl, lam_psl, invT, T;
  float lam_match;
  double* loss;                  // may be NULL
  float2* grad;                  // may be NULL
  // cross-ambiguity: the second waveform, its partial gradients and output (else NULL)
  const float2* s2;
  const float2* gpart2;
  float2* grad2;
  // single-pass soft-PSL results (valid where one[b].reserved == 1), else NULL
  const graf_partials* one;
  double omega;
  float xbar;
  // delay-sharded single pass (graf_af_loss_grad_sp_end): the ISL sum comes from `global`,
  // and a waveform whose global single pass is invalid gets loss NaN and grad 0
  int sp;
  const int32_t* skip;   // skipped waveforms: outputs left untouched
};

constexpr int kFinChunk = 1024;   // gradient positions per finalize CTA (grid.y)

__global__ void __launch_bounds__(256) finalize_kernel(FinalizeParams f) {
  const int b = blockIdx.x;
  if (f.skip && f.skip[b]) return;
  const int N = f.N;
  const float2* sg = f.s + (size_t)b * N;
  const float2* sg2 = f.s2 ? f.s2 + (size_t)b * N : nullptr;
  __shared__ double sh[4];
  const bool one = f.one && f.one[b].reserved == 1.0;   // single-pass soft-PSL result is valid
  // grid.y splits the gradient's N positions over CTAs (c5: 8 waveforms would otherwise be
  // 8 CTAs summing 16384 x P partials each); every CTA recomputes the O(N) scalars, and
  // only chunk 0 writes the loss
  const int n0 = blockIdx.y * kFinChunk, n1 = min(N, n0 + kFinChunk);
  double* const loss_out = blockIdx.y == 0 ? f.loss : nullptr;
  if (threadIdx.x < 32) {
    const double e = warp_energy(sg, N, threadIdx.x);
    // cross-ambiguity: E1 E2 replaces E^2 (reading R25)
    const double e2 = sg2 ? warp_energy(sg2, N, threadIdx.x) : e;
    if (threadIdx.x == 0) {
      sh[0] = e;
      sh[2] = e2;
      double S = 0, Z = 0, F = 0, Mt = 0;
      double m = -INFINITY;
      for (int q = 0; q < f.P; ++q) {
        const double* rec = f.part + ((size_t)b * f.P + q) * kPart;
        S += rec[0];
        F += rec[4];
        Mt += rec[6];
        lse_merge(m, Z, rec[1], rec[2], f.T);
      }
      sh[1] = F;
      sh[3] = 1.0;
      if (one) {
        // single pass: p - pbar = (e - ebar) / Z_c; the gradient accumulated with f' = lambda e
        // is scaled by 1/Z_c; LSE = xbar + T log Z_c (reading R13)
        const double zc = f.omega + f.one[b].cen_sum;
        sh[3] = 1.0 / zc;
#ifdef GRAF_MUTATE_NO_ZC   // mutation check only: drop the 1/Z_c scale of the single pass
        sh[3] = 1.0;
#endif
        const double Sg = f.sp ? f.global[b].isl_sum : S;
        if (loss_out)
          loss_out[b] = f.lam_isl * (f.normalize ? Sg / (e * e2) : Sg) + f.lam_psl * ((double)f.xbar + (double)f.T * log(zc));
      } else if (f.sp) {
        sh[3] = 0.0;   // invalid global single pass: the caller recomputes with two passes
        if (loss_out) loss_out[b] = __longlong_as_double(0x7ff8000000000000ll);
      } else if (loss_out) {
        double Sg = S, mg = m, Zg = Z;
        if (f.global) {
          Sg = f.global[b].isl_sum;
          mg = f.global[b].lse_max;
          Zg = f.global[b].lse_sum;
        }
        double L = f.lam_isl * (f.normalize ? Sg / (e * e2) : Sg);
        if (f.lam_psl != 0.f) L += f.lam_psl * (mg + (double)f.T * log(Zg));
        if (f.lam_match != 0.f) L += f.lam_match * Mt;
        loss_out[b] = L;
      }
    }
  }
  __syncthreads();
  if (!f.grad) return;
  const double E = sh[0], E2 = sh[2];
  const bool nt = f.grad_norm_term && f.normalize;
  const double gs = sh[3];   // 1/Z_c for the single pass (0 for an invalid sharded one), else 1
  // auto: -(2/E^3) F s;  cross: -F/(E1^2 E2) s1 and -F/(E1 E2^2) s2
  const float coef = nt ? (float)((sg2 ? 1.0 : 2.0) * sh[1] * gs / (E * E * E2)) : 0.f;
  const float coef2 = nt ? (float)(sh[1] / (E * E2 * E2)) : 0.f;
  if (f.sp && !one) {   // invalid sharded single pass: the unscaled sums may hold inf (expm1 overflow)
    for (int n = n0 + threadIdx.x; n < n1; n += blockDim.x) f.grad[(size_t)b * N + n] = make_float2(0.f, 0.f);
    return;
  }
  for (int n = n0 + threadIdx.x; n < n1; n += blockDim.x) {
    double gx = 0, gy = 0;
    for (int q = 0; q < f.P; ++q) {
      const float2 a = f.gpart[((size_t)b * f.P + q) * N + n];
      gx += a.x;
      gy += a.y;
    }
    const float2 sv = sg[n];
    f.grad[(size_t)b * N + n] = make_float2((float)(gx * gs) - coef * sv.x, (float)(gy * gs) - coef * sv.y);
    if (sg2) {
      double hx = 0, hy = 0;
      for (int q = 0; q < f.P; ++q) {
        const float2 a = f.gpart2[((size_t)b * f.P + q) * N + n];
        hx += a.x;
        hy += a.y;
      }
      const float2 s2v = sg2[n];
      f.grad2[(size_t)b * N + n] = make_float2((float)hx - coef2 * s2v.x, (float)hy - coef2 * s2v.y);
    }
  }
}

// A shard that owns no loss rows: grad = 0 (and loss = 0 for losses that are sums over
// rows), skipped waveforms untouched.
__global__ void zero_outputs_kernel(float2* grad, double* loss, long long B, int N, const int32_t* skip) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < B * N;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / N;
    if (skip && skip[b]) continue;
    grad[i] = make_float2(0.f, 0.f);
    if (loss && i - b * N == 0) loss[b] = 0.0;
  }
}

// Delay-sharded single pass, phase 1 tail: fold this shard's P CTA records and partial
// gradients into one record and one unscaled gradient per waveform (fixed order), so
// phase 2 needs neither the CTA count nor the per-CTA buffers.
struct SpFoldParams {
  const double* part;   // [B][P][kPart]
  const float2* gpart;  // [B][P][N]
  double* rec1;         // [B][kPart]
  float2* gsum;         // [B][N]
  int P, N;
  float T;
};

// grid (B, ceil(N / 256)): one CTA per waveform and 256-sample chunk, so the fold of c5's
// 8 x 37 x 16384 partial-gradient entries runs on every SM (round 2's first version ran one
// CTA per waveform: 0.40 ms of a 2.05 ms G = 8 shard step; profiles/r02/shard/)
__global__ void __launch_bounds__(256) sp_fold_kernel(SpFoldParams f) {
  const int b = blockIdx.x;
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    double S = 0, Z = 0, C = 0, F = 0, Mt = 0, m = -INFINITY;
    for (int q = 0; q < f.P; ++q) {
      const double* rec = f.part + ((size_t)b * f.P + q) * kPart;
      S += rec[0];
      lse_merge(m, Z, rec[1], rec[2], f.T);
      C += rec[3];
      F += rec[4];
      Mt += rec[6];
    }
    double* o = f.rec1 + (size_t)b * kPart;
    o[0] = S;
    o[1] = m;
    o[2] = Z;
    o[3] = C;
    o[4] = F;
    o[5] = (double)0x7fffffff;
    o[6] = Mt;
    o[7] = 0.0;
  }
  const int n = blockIdx.y * blockDim.x + threadIdx.x;
  if (n >= f.N) return;
  const float2* gp = f.gpart + (size_t)b * f.P * f.N + n;
  double gx = 0, gy = 0;
  int q = 0;
  for (; q + 8 <= f.P; q += 8) {   // 8 loads in flight, summed in the fixed order q = 0, 1, ...
    float2 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = gp[(size_t)(q + i) * f.N];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      gx += a[i].x;
      gy += a[i].y;
    }
  }
  for (; q < f.P; ++q) {
    const float2 a = gp[(size_t)q * f.N];
    gx += a.x;
    gy += a.y;
  }
  f.gsum[(size_t)b * f.N + n] = make_float2((float)gx, (float)gy);
}

// Phase 2 head: the R13 validity rule on the GLOBAL (rank-order combined) partials.
struct SpValidateParams {
  const graf_partials* global;
  graf_partials* out;   // global with reserved = validity
  int32_t* valid;       // may be NULL
  int B;
  float xbar, invT;
};

__global__ void sp_validate_kernel(SpValidateParams v) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= v.B) return;
  graf_partials g = v.global[b];
  const bool ok = isfinite(g.cen_sum) && isfinite(g.lse_max) && (g.lse_max - (double)v.xbar) * (double)v.invT <= 40.0;
  g.reserved = ok ? 1.0 : 0.0;
  v.out[b] = g;
  if (v.valid) v.valid[b] = ok ? 1 : 0;
}

struct CombineParams {
  const graf_partials* shards;
  int G, B;
  float T;
  graf_partials* out;
};

__global__ void combine_partials_kernel(CombineParams c) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= c.B) return;
  double S = 0, Z = 0, Cs = 0, key = (double)0x7fffffff;
  double m = -INFINITY;
  for (int q = 0; q < c.G; ++q) {
    const graf_partials g = c.shards[(size_t)q * c.B + b];
    S += g.isl_sum;
    Cs += g.cen_sum;
    key_merge(m, key, g.lse_max, g.psl_key);
    lse_merge(m, Z, g.lse_max, g.lse_sum, c.T);
  }
  graf_partials o;
  o.isl_sum = S;
  o.lse_max = m;
  o.lse_sum = Z;
  o.cen_sum = Cs;
  o.psl_key = key;
  o.reserved = 0.0;
  c.out[b] = o;
}

// ---------------------------------------------------------------------------
// Hard PSL (Eq. 19; the section-7 loss L416): loss += lambda * x*
// and its argmax subgradient, from the combined partials (lse_max = x*, psl_key =
// the argmax cell).  One CTA per waveform, O(N):
//   A* = sum_n s[n] conj(s[n-k*]) W^{m* n}        (the one cell, double accumulation)
//   G  = lambda A*/E^2 (normalized) | lambda A*   (d x*/dA*)
//   g[p] += H[p] s[p-k*] + conj(H[p+k*]) s[p+k*],  H[n] = G W^{-m* n}
//   normalized: g -= (2 lambda / E^3) chi* s.
// Only shard 0 adds the gradient term (the sum over shards is the full gradient);
// every shard adds the loss (x* is global).
// ---------------------------------------------------------------------------
struct PslParams {
  const float2* s;
  const graf_partials* stats;
  int N, M, key_lo, periodic, normalize;
  float lam;
  int add_grad;       // 0: this shard does not hold the term
  int accumulate;     // 1: add into loss/grad (a finalize wrote them), 0: overwrite
  double* loss;       // nullable
  float2* grad;
  const int32_t* skip;
};

__global__ void __launch_bounds__(256) psl_grad_kernel(PslParams q) {
  const int b = blockIdx.x;
  if (q.skip && q.skip[b]) return;
  const int N = q.N, M = q.M;
  const float2* sg = q.s + (size_t)b * N;
  const graf_partials st = q.stats[b];
  const long long key = (long long)st.psl_key;
  const int k = (int)(key / M) + q.key_lo, m = (int)(key % M);
  const int stride = kMaxM / M;
  __shared__ double red[2 * 32 + 2];
  // A* = sum_n s[n] conj(s[n-k]) W^{m n}
  double ax = 0.0, ay = 0.0;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    int j = n - k;
    bool ok = true;
    if (q.periodic) j = ((j % N) + N) % N;
    else ok = (j >= 0 && j < N);
    if (ok) {
      const float2 r = cmulc(sg[n], sg[j]);
      const float2 w = g_tw[(int)(((long long)m * n) & (M - 1)) * stride];
      ax += (double)r.x * w.x - (double)r.y * w.y;
      ay += (double)r.x * w.y + (double)r.y * w.x;
    }
  }
  ax = block_sum<256>(ax, red);
  ay = block_sum<256>(ay, red);
  double E = 0.0;
  if (threadIdx.x < 32) {
    const double e = warp_energy(sg, N, threadIdx.x);
    if (threadIdx.x == 0) E = e;
  }
  if (threadIdx.x == 0) {
    red[64] = ax;
    red[65] = ay;
    red[0] = E;
    if (q.loss) q.loss[b] = (q.accumulate ? q.loss[b] : 0.0) + (double)q.lam * st.lse_max;
  }
  __syncthreads();
  const double Ax = red[64], Ay = red[65], Ed = red[0];
  const double sc = q.normalize ? (double)q.lam / (Ed * Ed) : (double)q.lam;
  const float2 G = make_float2((float)(sc * Ax), (float)(sc * Ay));
  const float coef = q.normalize ? (float)(2.0 * q.lam * (Ax * Ax + Ay * Ay) / (Ed * Ed * Ed)) : 0.f;
  for (int p = threadIdx.x; p < N; p += blockDim.x) {
    float2 acc = make_float2(0.f, 0.f);
    if (q.add_grad) {
      // term 1 (n = p): H[p] s[p-k]
      int j = p - k;
      bool ok = true;
      if (q.periodic) j = ((j % N) + N) % N;
      else ok = (j >= 0 && j < N);
      if (ok) {
        const float2 w = cconj(g_tw[(int)(((long long)m * p) & (M - 1)) * stride]);   // W^{-m p}
        acc = cadd(acc, cmul(cmul(G, w), sg[j]));
      }
      // term 2 (n = p + k): conj(H[p+k]) s[p+k]
      int n = p + k;
      ok = true;
      if (q.periodic) n = ((n % N) + N) % N;
      else ok = (n >= 0 && n < N);
      if (ok) {
        const float2 w = cconj(g_tw[(int)(((long long)m * n) & (M - 1)) * stride]);
        acc = cadd(acc, cmul(cconj(cmul(G, w)), sg[n]));
      }
      const float2 sp = sg[p];
      acc = make_float2(acc.x - coef * sp.x, acc.y - coef * sp.y);
    }
    float2* gp = q.grad + (size_t)b * N + p;
    *gp = q.accumulate ? cadd(*gp, acc) : acc;
  }
}

// ---------------------------------------------------------------------------
// Spectral variance (the section-7 LPI term; reading R22):
//   S = DFT_N(s), p = |S|^2 / P, SV = sum (p - mean p)^2 / (N - ddof)
//   dSV/dS* = (c - sum c p) S / P, c = 2 (p - mean p) / (N - ddof);  g = DFT^H (dSV/dS*)
// N <= 1024: the DFT as its sum (one CTA per waveform, a thread per bin; the
// section-7 N = 256 costs microseconds); N >= 2048: the Stockham row FFT.
// Reductions: fixed-order shared-memory trees (deterministic).
// ---------------------------------------------------------------------------
struct SvParams {
  const float2* s;
  int N;
  float weight;
  const float* weights;   // [B] or NULL (= weight)
  int accumulate;
  double* loss;
  float2* grad;
  int ddof;               // variance denominator N - ddof (0: population; 1: unbiased)
};

// sum over the CTA (blockDim.x a power of two <= 1024), result in every thread
__device__ __forceinline__ double cta_tree_sum(double v, double* buf) {
  const int t = threadIdx.x;
  buf[t] = v;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (t < h) buf[t] += buf[t + h];
    __syncthreads();
  }
  const double r = buf[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) sv_direct_kernel(SvParams q) {
  extern __shared__ float4 smem_raw[];
  const int N = q.N, b = blockIdx.x, t = threadIdx.x;
  float2* ss = reinterpret_cast<float2*>(smem_raw);        // s [N], then dS [N]
  float2* ds = ss + N;
  double* buf = reinterpret_cast<double*>(ds + N);          // [blockDim]
  const float2* sg = q.s + (size_t)b * N;
  for (int i = t; i < N; i += blockDim.x) ss[i] = sg[i];
  __syncthreads();
  const int stride = kMaxM / N;
  // bins j = t (blockDim >= N): S_j = sum_n s_n W^{jn} (fp32 FMA chains, 4 partial
  // sums for ILP; N <= 1024 terms keep the relative error ~1e-6)
  double Sx = 0.0, Sy = 0.0;
  if (t < N) {
    float ax[4] = {0.f, 0.f, 0.f, 0.f}, ay[4] = {0.f, 0.f, 0.f, 0.f};
    for (int n = 0; n < N; n += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (n + u < N) {
          const float2 w = g_tw[((t * (n + u)) & (N - 1)) * stride];
          const float2 x = ss[n + u];
          ax[u] = fmaf(x.x, w.x, fmaf(-x.y, w.y, ax[u]));
          ay[u] = fmaf(x.x, w.y, fmaf(x.y, w.x, ay[u]));
        }
      }
    }
    Sx = (double)((ax[0] + ax[1]) + (ax[2] + ax[3]));
    Sy = (double)((ay[0] + ay[1]) + (ay[2] + ay[3]));
  }
  const double pw = Sx * Sx + Sy * Sy;
  const double P = cta_tree_sum(t < N ? pw : 0.0, buf);
  const double pe = pw / P;
  const double mean = cta_tree_sum(t < N ? pe : 0.0, buf) / N;
  const double d = pe - mean;
  const double var = cta_tree_sum(t < N ? d * d : 0.0, buf);
  const double ce = 2.0 * d / (N - q.ddof);
  const double cp = cta_tree_sum(t < N ? ce * pe : 0.0, buf);
  const float wb = q.weights ? q.weights[b] : q.weight;
  if (t == 0 && q.loss) q.loss[b] = (q.accumulate ? q.loss[b] : 0.0) + (double)wb * (var / (N - q.ddof));
  if (t < N) {
    const double f = (double)wb * (ce - cp) / P;
    ds[t] = make_float2((float)(f * Sx), (float)(f * Sy));
  }
  __syncthreads();
  // g_n = sum_j dS_j W^{-jn}
  if (t < N) {
    float gx[4] = {0.f, 0.f, 0.f, 0.f}, gy[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < N; j += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j + u < N) {
          const float2 w = g_tw[((t * (j + u)) & (N - 1)) * stride];   // conj below
          const float2 x = ds[j + u];
          gx[u] = fmaf(x.x, w.x, fmaf(x.y, w.y, gx[u]));
          gy[u] = fmaf(x.y, w.x, fmaf(-x.x, w.y, gy[u]));
        }
      }
    }
    float2* gp = q.grad + (size_t)b * N + t;
    const float2 g = make_float2((gx[0] + gx[1]) + (gx[2] + gx[3]), (gy[0] + gy[1]) + (gy[2] + gy[3]));
    *gp = q.accumulate ? cadd(*gp, g) : g;
  }
}

// the spectral-variance FFT: one row slot of T = M/E >= 32 threads per waveform
template <int M, int E>
struct SvCfg {
  static constexpr int T = M / E;
  static constexpr int XS = M + M / Pad<E>::P;
  static_assert(T >= 32, "one full warp at least");
};

template <int M, int E>
__global__ void __launch_bounds__(M / E) sv_fft_kernel(SvParams q) {
  constexpr int T = SvCfg<M, E>::T;
  constexpr bool SPLIT = false;
  constexpr int E2 = E;
  extern __shared__ float4 smem_raw[];
  float2* sh = reinterpret_cast<float2*>(smem_raw);
  double* buf = reinterpret_cast<double*>(sh + ((SvCfg<M, E>::XS + 1) & ~1));
  const int b = blockIdx.x, t = threadIdx.x;
  const float2* sg = q.s + (size_t)b * M;
  Twiddles<M, E2> tw;
  tw.init(t);
  const float2 wt = make_float2(1.f, 0.f);
  SlotSync<T, 1> sync{1};
  auto toff = [](int e) { return SPLIT ? (e < E2 ? 2 * e * T : 2 * (e - E2) * T + 1) : e * T; };
  const int tb = SPLIT ? 2 * t : t;
  float2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = sg[tb + toff(e)];
  row_fft<M, E, SPLIT, false>(v, sh, t, tw, sync, wt);      // S[m], m = t + e T
  double pw = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) pw += (double)v[e].x * v[e].x + (double)v[e].y * v[e].y;
  const double P = cta_tree_sum(pw, buf);
  double sp = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) sp += ((double)v[e].x * v[e].x + (double)v[e].y * v[e].y) / P;
  const double mean = cta_tree_sum(sp, buf) / M;
  double var = 0.0, cp = 0.0;
  float c[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const double pe = ((double)v[e].x * v[e].x + (double)v[e].y * v[e].y) / P;
    const double d = pe - mean;
    var += d * d;
    const double ce = 2.0 * d / (M - q.ddof);
    c[e] = (float)ce;
    cp += ce * pe;
  }
  var = cta_tree_sum(var, buf);
  cp = cta_tree_sum(cp, buf);
  const float wb = q.weights ? q.weights[b] : q.weight;
  if (t == 0 && q.loss) q.loss[b] = (q.accumulate ? q.loss[b] : 0.0) + (double)wb * (var / (M - q.ddof));
  const float sc = (float)((double)wb / P);
  const float cpf = (float)cp;
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = cscale(v[e], (c[e] - cpf) * sc);
  row_fft<M, E, SPLIT, true>(v, sh, t, tw, sync, wt);       // g[n] = sum_m dS_m W^{-mn}
  float2* gg = q.grad + (size_t)b * M;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    float2* gp = gg + tb + toff(e);
    *gp = q.accumulate ? cadd(*gp, v[e]) : v[e];
  }
}

// ---------------------------------------------------------------------------
// Adam on the phases of s = exp(j theta), one CTA per waveform (the
// waveform's step counter is read and advanced by its own CTA: graph-replayable)
// ---------------------------------------------------------------------------
struct AdamParams {
  float* theta;
  float* m;
  float* v;
  int* step;
  const float2* grad;
  float2* s_out;
  int N;
  float lr, beta1, beta2, eps;
};

__global__ void __launch_bounds__(256) phase_adam_kernel(AdamParams a) {
  const int b = blockIdx.x;
  const int t = a.step[b] + 1;
  const float bc1 = 1.f - powf(a.beta1, (float)t), bc2 = 1.f - powf(a.beta2, (float)t);
  for (int i = threadIdx.x; i < a.N; i += blockDim.x) {
    const size_t j = (size_t)b * a.N + i;
    const float th = a.theta[j];
    float sn, cs;
    sincosf(th, &sn, &cs);
    const float2 g = a.grad[j];
    // dL/dtheta = -2 Im(s conj(g)), s = (cs, sn)
    const float d = -2.f * (sn * g.x - cs * g.y);
    const float mm = a.beta1 * a.m[j] + (1.f - a.beta1) * d;
    const float vv = a.beta2 * a.v[j] + (1.f - a.beta2) * d * d;
    a.m[j] = mm;
    a.v[j] = vv;
    const float thn = th - a.lr * (mm / bc1) / (sqrtf(vv / bc2) + a.eps);
    a.theta[j] = thn;
    float s2, c2;
    sincosf(thn, &s2, &c2);
    a.s_out[j] = make_float2(c2, s2);
  }
  __syncthreads();
  if (threadIdx.x == 0) a.step[b] = t;
}

// ---------------------------------------------------------------------------
// Mainlobe width (reading R26):
//   W = sum_tau |tau| sigma(gamma (chi(tau,0) - E^2/2)),  chi(tau,0) = |A_tau|^2,
//   A_tau = sum_n s[n] conj(s[n - tau]) (the zero-Doppler cut; A_{-tau} = conj A_tau),
//   dW/ds*[p] = sum_tau c_tau (A_tau s[p-tau] + conj(A_tau) s[p+tau]) - (sum_tau c_tau) E s[p],
//   c_tau = |tau| gamma sigma'(u_tau).
// One CTA per waveform, O(N^2) direct sums (the cut is one Doppler bin of every
// delay row); A_tau for tau >= 0 kept in shared memory.
// ---------------------------------------------------------------------------
struct MlwParams {
  const float2* s;
  int N, periodic, accumulate;
  float gamma, weight;
  double* loss;
  float2* grad;
};

__global__ void __launch_bounds__(1024) mainlobe_kernel(MlwParams q) {
  extern __shared__ float4 smem_raw[];
  const int N = q.N, b = blockIdx.x, t = threadIdx.x;
  const int K = q.periodic ? N / 2 : N - 1;            // taus 0..K (mirrors implied)
  float2* At = reinterpret_cast<float2*>(smem_raw);     // [K + 1]
  float* ct = reinterpret_cast<float*>(At + K + 1);     // [K + 1] c_tau * mult
  double* buf = reinterpret_cast<double*>(ct + ((K + 2) & ~1));   // [blockDim]
  const float2* sg = q.s + (size_t)b * N;
  double E = 0.0;
  for (int n = t; n < N; n += blockDim.x) E += (double)sg[n].x * sg[n].x + (double)sg[n].y * sg[n].y;
  E = cta_tree_sum(E, buf);
  const double halfE2 = 0.5 * E * E;
  double Wsum = 0.0, Csum = 0.0;
  for (int tau = t; tau <= K; tau += blockDim.x) {
    float ax = 0.f, ay = 0.f;
    for (int n = 0; n < N; ++n) {
      int j = n - tau;
      if (q.periodic) j = j < 0 ? j + N : j;
      else if (j < 0) continue;
      const float2 r = cmulc(sg[n], sg[j]);
      ax += r.x;
      ay += r.y;
    }
    At[tau] = make_float2(ax, ay);
    const bool self = (tau == 0) || (q.periodic && 2 * tau == N);
    const float mult = self ? 1.f : 2.f;
    const double chi = (double)ax * ax + (double)ay * ay;
    const double u = (double)q.gamma * (chi - halfE2);
    const double sig = 0.5 * (1.0 + tanh(0.5 * u));
    Wsum += mult * tau * sig;
    const double c = (double)tau * q.gamma * sig * (1.0 - sig);
    ct[tau] = (float)(mult * c);
    Csum += mult * c;
  }
  Wsum = cta_tree_sum(Wsum, buf);
  Csum = cta_tree_sum(Csum, buf);
  if (t == 0 && q.loss) q.loss[b] = (q.accumulate ? q.loss[b] : 0.0) + (double)q.weight * Wsum;
  const float cE = (float)(Csum * E);
  for (int p = t; p < N; p += blockDim.x) {
    float gx = 0.f, gy = 0.f;
    for (int tau = 1; tau <= K; ++tau) {
      const float c = ct[tau];
      if (c == 0.f) continue;
      const float2 A = At[tau];
      int j1 = p - tau, j2 = p + tau;
      bool o1 = true, o2 = true;
      if (q.periodic) {
        j1 = j1 < 0 ? j1 + N : j1;
        j2 = j2 >= N ? j2 - N : j2;
      } else {
        o1 = j1 >= 0;
        o2 = j2 < N;
      }
      // (mult already in c: the -tau mirror contributes the same pair of terms)
      if (o1) {
        const float2 v = cmul(A, sg[j1]);
        gx = fmaf(c, v.x, gx);
        gy = fmaf(c, v.y, gy);
      }
      if (o2) {
        const float2 v = cmul(cconj(A), sg[j2]);
        gx = fmaf(c, v.x, gx);
        gy = fmaf(c, v.y, gy);
      }
    }
    const float2 sp = sg[p];
    const float2 g = make_float2(q.weight * (gx - cE * sp.x), q.weight * (gy - cE * sp.y));
    float2* gp = q.grad + (size_t)b * N + p;
    *gp = q.accumulate ? cadd(*gp, g) : g;
  }
}

#endif  // GRAF_API_UNIT

}  // namespace graf
