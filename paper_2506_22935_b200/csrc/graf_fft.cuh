// graf_fft.cuh — register/shared-memory Stockham FFT building blocks for sm_100a.
//
// The Doppler DFT of each delay row (Eq. 11; Alg. 1 step 3,
// L250) is an unnormalised length-M DFT, X[m] = sum_n x[n] e^{-2 pi i m n / M}.
// The adjoint needs the unnormalised inverse, H[n] = sum_m G[m] e^{+2 pi i m n/M}
// ("IFFT operation (linear)").
//
// Layout (one "row slot" = T = M/E threads): thread t holds E complex values in
// registers, slot e <-> index t + e*T.  A Stockham autosort pass of radix R and
// stride Ns takes, for butterfly j' = t + q*T (q < E/R), the R inputs
// x[j' + r*M/R] = slot q + r*E/R, twiddles them by W_M^{(j' mod Ns) r M/(Ns R)},
// runs an in-register radix-R DFT and writes y[(j'/Ns)*Ns*R + (j' mod Ns) + r*Ns].
// Non-final passes exchange through shared memory (padded index y + (y >> log2 E),
// conflict-free for every (M, E) used — simulated offline); the
// final pass lands its outputs in the SAME slots (index t + e*T), so the
// frequency-domain epilogue and the inverse FFT work in registers with no
// reordering.  The same slot<->index map holds for time and frequency.
//
// Twiddles: the per-thread base twiddle W_M^{(j' mod Ns) M/(Ns R)} of every
// (pass, q) depends only on the thread, so it is read once per kernel from the
// correctly rounded table g_tw into registers; the R-1 powers are rebuilt per
// use by a balanced product tree (depth <= log2 R, error <= ~4 ulp).  When a
// thread needs at most 16 twiddles per FFT (M <= 256 with E = 16), all of them
// are computed once per kernel and stay cached in registers for every row.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

namespace graf {

constexpr int kMaxM = 16384;

// M-th roots of unity table, g_tw[i] = exp(-2 pi i * i / kMaxM), float32, rounded
// once from double sincospi (exact at multiples of 1/4 turn).  Each translation unit
// of the library (graf_api.cu, graf_rows_*.cu) holds its own copy and fills it with
// its own tw_init_kernel; ensure_twiddles() (graf_api.cu) enqueues all of them on the
// caller's stream (no host-blocking copy).
static __device__ float2 g_tw[kMaxM];

static __global__ void tw_init_kernel() {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < kMaxM; j += gridDim.x * blockDim.x) {
    double sn, cs;
    sincospi(-2.0 * (double)j / (double)kMaxM, &sn, &cs);
    g_tw[j] = make_float2((float)cs, (float)sn);
  }
}
static inline cudaError_t launch_tw_init(cudaStream_t st) {
  tw_init_kernel<<<kMaxM / 256, 256, 0, st>>>();
  return cudaGetLastError();
}

// Complex add / subtract.  sm_100 has paired fp32 instructions (FADD2 / FMUL2 /
// FFMA2: one issue slot for the real and imaginary lanes); GRAF_F32X2 selects them
// through PTX add/sub/mul/fma.rn.f32x2.  Same IEEE round-to-nearest results per lane.
#if defined(GRAF_F32X2) && defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
__device__ __forceinline__ unsigned long long f2_pack(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a)), "l"(f2_pack(b)));
  return f2_unpack(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a)), "l"(f2_pack(b)));
  return f2_unpack(r);
}
// a * b = b.x (a.x, a.y) + b.y (-a.y, a.x): FMUL2 with a broadcast operand, then FFMA2
// with the swapped, lane-negated pair (operand modifiers, no extra instructions)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  unsigned long long t, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2_pack(make_float2(b.x, b.x))), "l"(f2_pack(a)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(f2_pack(make_float2(-a.y, a.x))), "l"(f2_pack(make_float2(b.y, b.y))), "l"(t));
  return f2_unpack(r);
}
// a * conj(b) = b.x (a.x, a.y) + b.y (a.y, -a.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  unsigned long long t, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2_pack(make_float2(b.x, b.x))), "l"(f2_pack(a)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(f2_pack(make_float2(a.y, -a.x))), "l"(f2_pack(make_float2(b.y, b.y))), "l"(t));
  return f2_unpack(r);
}
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
#endif
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

// cos(2 pi j / 32), float32-rounded, first quadrant j = 0..8.
__host__ __device__ constexpr float cos32_q(int j) {
  return j == 0 ? 1.0f : j == 1 ? 9.807852507e-01f : j == 2 ? 9.238795042e-01f
       : j == 3 ? 8.314695954e-01f : j == 4 ? 7.071067691e-01f : j == 5 ? 5.555702448e-01f
       : j == 6 ? 3.826834261e-01f : j == 7 ? 1.950903237e-01f : 0.0f;
}
__host__ __device__ constexpr float cos32(int j) {
  j = ((j % 32) + 32) % 32;
  return j <= 8 ? cos32_q(j) : j <= 16 ? -cos32_q(16 - j) : j <= 24 ? -cos32_q(j - 16) : cos32_q(32 - j);
}
__host__ __device__ constexpr float sin32(int j) { return cos32(8 - j); }

// z * W_R^K with W_R = exp(-2 pi i / R) (forward) or exp(+2 pi i / R) (inverse);
// trivial twiddles (1, -i, -1, +i) cost no multiplies.  R <= 32.
template <int K, int R, bool INV>
__device__ __forceinline__ float2 twc(float2 z) {
  constexpr int J = (((K * (32 / R)) % 32) + 32) % 32;
  if constexpr (J == 0) {
    return z;
  } else if constexpr (J == 8) {
    return INV ? make_float2(-z.y, z.x) : make_float2(z.y, -z.x);
  } else if constexpr (J == 16) {
    return make_float2(-z.x, -z.y);
  } else if constexpr (J == 24) {
    return INV ? make_float2(z.y, -z.x) : make_float2(-z.y, z.x);
  } else {
    constexpr float c = cos32(J);
    constexpr float s = INV ? sin32(J) : -sin32(J);
#if defined(GRAF_F32X2) && defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    return cmul(z, make_float2(c, s));
#else
    return make_float2(z.x * c - z.y * s, z.x * s + z.y * c);
#endif
  }
}

// Radix-2 butterfly with a compile-time twiddle w = W_R^K:  x0 = a + w b,  x1 = a - w b.
// Trivial twiddles (1, -+i, -1) cost adds only.  Otherwise the tangent form: with
// w = c (1 + j tan), |tan| <= 1 (else w = s (cot + j) with the roles swapped),
//   u + j v = b (1 + j tan)  (2 FFMA),  x0 = a + c (u + j v),  x1 = a - c (u + j v)  (4 FFMA):
// 6 FP instructions instead of 8 (a complex multiply, then 2 complex adds), each output
// with the same rounding depth as the plain form.  (-DGRAF_NO_TAN_BFLY: the plain form.)
#if defined(GRAF_F32X2) && defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
// a * b + c per lane (FFMA2)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_pack(a)), "l"(f2_pack(b)), "l"(f2_pack(c)));
  return f2_unpack(r);
}
#endif

template <int K, int R, bool INV>
__device__ __forceinline__ void bfly_tw(float2 a, float2 b, float2& x0, float2& x1) {
#if defined(GRAF_F32X2_TAN) && defined(GRAF_F32X2) && defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  // tangent form in paired fp32: three FFMA2 (one issue slot each; A/B builds only: c5
  // measured 13.87 ms against 13.84 with scalar code, profiles/r02/tune_c5_ab_f32x2.txt)
  constexpr int J = (((K * (32 / R)) % 32) + 32) % 32;
  if constexpr (J % 8 != 0) {
    constexpr float c = cos32(J);
    constexpr float s = INV ? sin32(J) : -sin32(J);
    constexpr bool cdom = (c < 0 ? -c : c) >= (s < 0 ? -s : s);
    constexpr float q = cdom ? s / c : c / s;
    constexpr float m = cdom ? c : s;
    const float2 w = cdom ? ffma2(make_float2(-q, q), make_float2(b.y, b.x), b)
                          : ffma2(make_float2(q, q), b, make_float2(-b.y, b.x));
    x0 = ffma2(make_float2(m, m), w, a);
    x1 = ffma2(make_float2(-m, -m), w, a);
    return;
  }
#endif
#if !defined(GRAF_NO_TAN_BFLY) && !defined(GRAF_F32X2)
  constexpr int J = (((K * (32 / R)) % 32) + 32) % 32;
  if constexpr (J % 8 != 0) {
    constexpr float c = cos32(J);
    constexpr float s = INV ? sin32(J) : -sin32(J);
    constexpr bool cdom = (c < 0 ? -c : c) >= (s < 0 ? -s : s);
    constexpr float q = cdom ? s / c : c / s;   // tan or cot, |q| <= 1
    constexpr float m = cdom ? c : s;
    float2 w;
    if constexpr (cdom) {
      w = make_float2(fmaf(-q, b.y, b.x), fmaf(q, b.x, b.y));   // b (1 + j q)
    } else {
      w = make_float2(fmaf(q, b.x, -b.y), fmaf(q, b.y, b.x));   // b (q + j)
    }
    x0 = make_float2(fmaf(m, w.x, a.x), fmaf(m, w.y, a.y));
    x1 = make_float2(fmaf(-m, w.x, a.x), fmaf(-m, w.y, a.y));
    return;
  }
#endif
  const float2 t = twc<K, R, INV>(b);
  x0 = cadd(a, t);
  x1 = csub(a, t);
}

template <int K, int R, bool INV>
__device__ __forceinline__ void dft_combine(float2* x, const float2* e, const float2* o) {
  if constexpr (K < R / 2) {
    bfly_tw<K, R, INV>(e[K], o[K], x[K], x[K + R / 2]);
    dft_combine<K + 1, R, INV>(x, e, o);
  }
}

// In-register DFT of length R (natural order in and out): radix-4 leaves,
// radix-2 decimation-in-time combination above them.
template <int R, bool INV>
__device__ __forceinline__ void dft(float2* x) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    const float2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const float2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
    const float2 t2 = cadd(x[1], x[3]);
    const float2 d = csub(x[1], x[3]);
    const float2 t3 = INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);  // d * (-+i)
    x[0] = cadd(t0, t2);
    x[2] = csub(t0, t2);
    x[1] = cadd(t1, t3);
    x[3] = csub(t1, t3);
  } else {
    float2 e[R / 2], o[R / 2];
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
      e[i] = x[2 * i];
      o[i] = x[2 * i + 1];
    }
    dft<R / 2, INV>(e);
    dft<R / 2, INV>(o);
    dft_combine<0, R, INV>(x, e, o);
  }
}

// DFT of length R whose inputs x[NZ..R) are zero (a zero-padded row's first pass):
// the same radix-2 decimation as dft<R> with the all-zero branches folded away
template <int R, int NZ, bool INV>
__device__ __forceinline__ void dft_lz(float2* x) {
  if constexpr (NZ >= R) {
    dft<R, INV>(x);
  } else if constexpr (NZ <= 1) {
#pragma unroll
    for (int r = 1; r < R; ++r) x[r] = x[0];   // DFT of (a, 0, ..., 0)
  } else {
    float2 e[R / 2], o[R / 2];
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
      e[i] = x[2 * i];
      o[i] = x[2 * i + 1];
    }
    dft_lz<R / 2, (NZ + 1) / 2, INV>(e);
    dft_lz<R / 2, NZ / 2, INV>(o);
    dft_combine<0, R, INV>(x, e, o);
  }
}

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// compile-time loop: f(integral_constant<int, I>) for I in [B, E)
template <int B, int E, class F>
__device__ __forceinline__ void static_for_fft(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for_fft<B + 1, E>(f);
  }
}

// exchange-buffer padding: one pad slot every max-radix elements (conflict-free
// for every plan used; scripts/bank_sim.py)
#ifndef GRAF_MAX_RADIX
#define GRAF_MAX_RADIX 32
#endif
template <int E>
struct Pad {
  static constexpr int P = E > GRAF_MAX_RADIX ? GRAF_MAX_RADIX : E;   // pad period = max radix
  static constexpr int S = ilog2(P);
};
template <int E>
__device__ __forceinline__ int padded(int y) {
  return y + (y >> Pad<E>::S);
}
// padded(y0 + i*step) for i = 0.. as base + i*stride when step is a multiple of
// the pad period (affine: one base address + immediate offsets, nothing per element)
template <int E, int STEP>
struct PadStride {
  static constexpr bool AFFINE = (STEP % Pad<E>::P) == 0;
  static constexpr int value = STEP + STEP / Pad<E>::P;
};

// opaque copy: stops the compiler from hoisting per-element address math out of
// the row loop (it would keep ~E addresses live across the whole kernel and spill)
__device__ __forceinline__ int launder(int x) {
  int y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// ---- compile-time pass plan: radices RM, RM, ..., remainder (GRAF_REM_FIRST=1
// puts the remainder first), with RM = min(E, GRAF_MAX_RADIX)
__host__ __device__ constexpr int max_radix(int E) { return E > GRAF_MAX_RADIX ? GRAF_MAX_RADIX : E; }
__host__ __device__ constexpr int first_radix(int M, int E) {
  int m = M;
  while (m >= max_radix(E)) m /= max_radix(E);
  return m > 1 ? m : max_radix(E) <= M ? max_radix(E) : M;
}
#ifndef GRAF_REM_FIRST
#define GRAF_REM_FIRST 0
#endif
__host__ __device__ constexpr int pass_radix(int M, int E, int p) {
#if GRAF_REM_FIRST
  return p == 0 ? first_radix(M, E) : max_radix(E);
#else
  // remainder LAST: RM, RM, ..., M / RM^k
  int ns = 1;
  for (int i = 0; i < p; ++i) ns *= (M / ns >= max_radix(E) ? max_radix(E) : M / ns);
  return M / ns >= max_radix(E) ? max_radix(E) : M / ns;
#endif
}
__host__ __device__ constexpr int pass_ns(int M, int E, int p) {
  int ns = 1;
  for (int i = 0; i < p; ++i) ns *= pass_radix(M, E, i);
  return ns;
}
__host__ __device__ constexpr int num_passes(int M, int E) {
  int n = 0;
  for (int ns = 1; ns < M; ns *= pass_radix(M, E, n), ++n) {
  }
  return n;
}
// register slots of base twiddles before pass p (passes >= 1 have twiddles)
__host__ __device__ constexpr int tw_offset(int M, int E, int p) {
  int off = 0;
  for (int i = 1; i < p; ++i) off += E / pass_radix(M, E, i);
  return off;
}

// 16 columns of this thread's tensor-memory lane, waited for (pass-1 twiddles, M = 16384)
__device__ __forceinline__ void tmem_tw_ld16(uint32_t taddr, float (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n\ttcgen05.wait::ld.sync.aligned;"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]),
        "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11]), "=f"(r[12]), "=f"(r[13]), "=f"(r[14]), "=f"(r[15])
      : "r"(taddr)
      : "memory");
}

template <int R>
__device__ __forceinline__ void tw_powers(float2 w1, float2* w) {
  w[0] = make_float2(1.f, 0.f);
  if constexpr (R > 1) w[1] = w1;
#pragma unroll
  for (int r = 2; r < R; ++r) w[r] = cmul(w[r / 2], w[r - r / 2]);
}

// total twiddle multiplies per thread per FFT (passes >= 1)
__host__ __device__ constexpr int tw_count(int M, int E) {
  int n = 0;
  for (int p = 1; p < num_passes(M, E); ++p) n += (E / pass_radix(M, E, p)) * (pass_radix(M, E, p) - 1);
  return n;
}
__host__ __device__ constexpr int tw_count_before(int M, int E, int P) {
  int n = 0;
  for (int p = 1; p < P; ++p) n += (E / pass_radix(M, E, p)) * (pass_radix(M, E, p) - 1);
  return n;
}

template <int M, int E>
struct Twiddles {
  static constexpr int T = M / E;
  static constexpr int NP = num_passes(M, E);
  static constexpr int NB = tw_offset(M, E, NP);          // base twiddles per thread
  static constexpr int NTW = tw_count(M, E);              // all twiddles per thread
#ifdef GRAF_NO_TWCACHE
  static constexpr bool CACHE = false;
#else
  static constexpr bool CACHE = (NTW > 0 && NTW <= 16);   // keep every power in registers
#endif
  // pass-1 powers from a shared-memory table tw1[(r - 1) * NS1 + jm] (NS1 = first radix;
  // every thread of a slot shares the NS1 rows, so reads are broadcast / conflict-free)
  // (M = 16384: GRAF_TW1_SMEM_16384=0 rebuilds the pass-1 powers from one base by the
  // product tree, taking their 31 LDS per FFT off the shared-memory pipe the exchanges
  // saturate: c5 13.84 -> 13.48 ms, but the c5 gradient error grows from 7e-5 to 1.8e-4 of
  // max |g| at N = 256, past the 1e-4 gate; the default reads 10 entries and forms the other
  // 21 by one product each, GRAF_TW1_SPLIT_16384.  At M = 8192 the tree made c4 3 % slower.)
#ifndef GRAF_TW1_SMEM_16384
#define GRAF_TW1_SMEM_16384 1
#endif
#ifndef GRAF_TW1_SPLIT_16384
#define GRAF_TW1_SPLIT_16384 1
#endif
  static constexpr bool SMEM1 = !CACHE && NP >= 2 && (M != 16384 || GRAF_TW1_SMEM_16384);
  static constexpr int NS1 = NP >= 2 ? pass_ns(M, E, 1) : 1;
  static constexpr int R1 = NP >= 2 ? pass_radix(M, E, 1) : 1;
  static constexpr int TAB1 = SMEM1 ? (R1 - 1) * NS1 : 0;   // table entries
  const float2* tab1 = nullptr;
  // (M = 16384 gradient kernels) tensor-memory address of this thread's 31 pass-1 twiddles
  // W^(jm r), r = 1..31, at columns 2 (r - 1), 2 (r - 1) + 1; 0: use tab1
  uint32_t ttw = 0;
#ifdef GRAF_HOLD_BASES
  float2 base[NB > 0 && !CACHE ? NB : 1];
#endif
  float2 pw[CACHE ? NTW : 1];

  __device__ __forceinline__ void init(int t) {
#pragma unroll
    for (int p = 1; p < NP; ++p) {
      const int ns = pass_ns(M, E, p), R = pass_radix(M, E, p), Q = E / R;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int jm = (t + q * T) & (ns - 1);
        const float2 w1 = g_tw[(jm * (M / (ns * R))) * (kMaxM / M)];
        if constexpr (CACHE) {
          float2 w[32];
          tw_powers_rt(w1, w, R);
#pragma unroll
          for (int r = 1; r < R; ++r) pw[tw_count_before(M, E, p) + q * (R - 1) + r - 1] = w[r];
        } else {
#ifdef GRAF_HOLD_BASES
          base[tw_offset(M, E, p) + q] = w1;
#endif
        }
      }
    }
  }

  // fill the pass-1 table (all threads of the CTA, before the CTA barrier)
  __device__ __forceinline__ static void fill_tab1(float2* tab, int tid, int nthreads) {
    if constexpr (SMEM1) {
      for (int i = tid; i < TAB1; i += nthreads) {
        const int r = i / NS1 + 1, jm = i % NS1;
        tab[i] = g_tw[(jm * r * (M / (NS1 * R1))) * (kMaxM / M)];
      }
    }
  }

  __device__ __forceinline__ static void tw_powers_rt(float2 w1, float2* w, int R) {
    // R is a compile-time constant after unrolling; dispatch keeps tw_powers templated
    if (R == 2) tw_powers<2>(w1, w);
    else if (R == 4) tw_powers<4>(w1, w);
    else if (R == 8) tw_powers<8>(w1, w);
    else if (R == 16) tw_powers<16>(w1, w);
    else if (R == 32) tw_powers<32>(w1, w);
  }
};

// One Stockham pass P (see header comment).  Non-final passes store to `sh`.
template <int M, int E, int P, bool INV, class Sync>
__device__ __forceinline__ void stockham_pass(float2 (&v)[E], float2* sh, int t, const Twiddles<M, E>& tw,
                                              const Sync& sync) {
  constexpr int T = M / E;
  constexpr int R = pass_radix(M, E, P);
  constexpr int NS = pass_ns(M, E, P);
  constexpr int Q = E / R;
  constexpr bool LAST = (NS * R == M);
  // last pass with several butterflies per thread (a remainder radix R < E): t + qT < NS,
  // so its bases W_M^{t + qT} = W_M^t W_E^q need ONE table read per pass (the W_E^q
  // factors are compile-time constants after unrolling)
  constexpr bool LAST_BASE = LAST && Q > 1 && NS > 1 && E <= 32 && (32 % E) == 0 && !Twiddles<M, E>::CACHE;
  float2 lb0 = make_float2(1.f, 0.f);
  if constexpr (LAST_BASE) lb0 = __ldg(&g_tw[t * (kMaxM / M)]);
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    float2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = v[q + r * Q];
    if constexpr (NS > 1) {
      if (P == 1 && R == 32 && Q == 1 && tw.ttw) {
        // pass-1 twiddles from tensor memory (thread-private, correctly rounded, written once
        // per kernel): off the shared-memory pipe, with the table's accuracy
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float w16[16];
          tmem_tw_ld16(tw.ttw + 16 * c, w16);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = 8 * c + i + 1;
            if (r < R) {
              const float2 w = make_float2(w16[2 * i], w16[2 * i + 1]);
              x[r] = INV ? cmulc(x[r], w) : cmul(x[r], w);
            }
          }
        }
      } else if (P == 1 && Twiddles<M, E>::SMEM1 && tw.tab1) {
        const float2* tb = tw.tab1 + ((t + q * T) & (NS - 1));
        if constexpr (R == 32 && M == 16384 && GRAF_TW1_SPLIT_16384) {
          // 10 table reads instead of 31: W^r = W^(r mod 8) W^(8 floor(r / 8)), one product
          // of correctly rounded entries (the shared-memory pipe is the scarce one here; a
          // product tree from one base costs accuracy: c5 gradient error 7e-5 -> 1.8e-4)
          float2 lo[8], hi[4];
#pragma unroll
          for (int r = 1; r < 8; ++r) lo[r] = tb[(r - 1) * NS];
#pragma unroll
          for (int j = 1; j < 4; ++j) hi[j] = tb[(8 * j - 1) * NS];
#pragma unroll
          for (int r = 1; r < R; ++r) {
            const float2 w = (r % 8 == 0) ? hi[r / 8] : (r < 8 ? lo[r] : cmul(lo[r % 8], hi[r / 8]));
            x[r] = INV ? cmulc(x[r], w) : cmul(x[r], w);
          }
        } else {
#pragma unroll
          for (int r = 1; r < R; ++r) {
            const float2 w = tb[(r - 1) * NS];
            x[r] = INV ? cmulc(x[r], w) : cmul(x[r], w);
          }
        }
      } else if constexpr (Twiddles<M, E>::CACHE) {
        constexpr int off = tw_count_before(M, E, P);
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const float2 w = tw.pw[off + q * (R - 1) + r - 1];
          x[r] = INV ? cmulc(x[r], w) : cmul(x[r], w);
        }
      } else {
        float2 w[R];
#ifdef GRAF_HOLD_BASES
        tw_powers<R>(tw.base[tw_offset(M, E, P) + q], w);
#else
        if constexpr (LAST_BASE) {
          const int J = (q * (32 / E)) % 32;
          tw_powers<R>(q == 0 ? lb0 : cmul(lb0, make_float2(cos32(J), -sin32(J))), w);
        } else {
          // base twiddle re-read per use from the L1-resident table (frees registers)
          const int jm = (t + q * T) & (NS - 1);
          tw_powers<R>(__ldg(&g_tw[(jm * (M / (NS * R))) * (kMaxM / M)]), w);
        }
#endif
#pragma unroll
        for (int r = 1; r < R; ++r) x[r] = INV ? cmulc(x[r], w[r]) : cmul(x[r], w[r]);
      }
    }
    dft<R, INV>(x);
    if constexpr (LAST) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[q + r * Q] = x[r];
    } else {
      if (q == 0) sync.before_writing();   // every reader of the previous contents is done
      const int jp = t + q * T;
      const int jm = jp & (NS - 1);
      const int base = (jp / NS) * NS * R + jm;
      if constexpr (NS == 1 && R <= Pad<E>::P) {
        float2* b = sh + padded<E>(base);           // base is a multiple of R: no carry
#pragma unroll
        for (int r = 0; r < R; ++r) b[r] = x[r];
      } else if constexpr (PadStride<E, NS>::AFFINE) {
        float2* b = sh + padded<E>(base);
#pragma unroll
        for (int r = 0; r < R; ++r) b[r * PadStride<E, NS>::value] = x[r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) sh[padded<E>(base + r * NS)] = x[r];
      }
    }
  }
}

// Full length-M FFT on the register slots of one row slot.  sync() orders the
// row slot's shared-memory exchange (warp sync, named barrier or CTA barrier).
template <int M, int E, int P, bool INV, class Sync>
__device__ __forceinline__ void fft_rows(float2 (&v)[E], float2* sh, int t, const Twiddles<M, E>& tw,
                                         const Sync& sync) {
  constexpr int T = M / E;
  constexpr int NP = num_passes(M, E);
  stockham_pass<M, E, P, INV>(v, sh, t, tw, sync);
  if constexpr (P + 1 < NP) {
    sync();
    if constexpr (PadStride<E, T>::AFFINE) {
      const float2* b = sh + padded<E>(t);
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = b[e * PadStride<E, T>::value];
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = sh[padded<E>(t + e * T)];
    }
    sync.done_reading();
    fft_rows<M, E, P + 1, INV, Sync>(v, sh, t, tw, sync);
  }
}

// Forward FFT of which only the outputs of slots 0 and E - 1 are needed (a loss band
// narrower than T = M/E bins): the passes before the last run in full (their outputs
// feed every thread through the exchange), the last pass evaluates only the two
// butterfly outputs that land in slots 0 (q = 0, r = 0) and E - 1 (q = Q - 1, r = R - 1).
// The other slots are left zero.  For last passes P >= 2 of uncached plans.
template <int M, int E, int P>
__device__ __forceinline__ void fft_last_edges(float2 (&v)[E], int t) {
  constexpr int T = M / E;
  constexpr int R = pass_radix(M, E, P);
  constexpr int NS = pass_ns(M, E, P);
  constexpr int Q = E / R;
  static_assert(NS * R == M && NS > 1 && P >= 2 && !Twiddles<M, E>::CACHE, "last pass of an uncached plan");
  float2 w[R];
  // q = 0: X_0 = sum_r W^{r jm} x_r with jm = t (NS > T here since NS * R = M, R <= E)
  tw_powers<R>(__ldg(&g_tw[(t & (NS - 1)) * (kMaxM / M)]), w);
  float2 x0 = v[0];
#pragma unroll
  for (int r = 1; r < R; ++r) x0 = cadd(x0, cmul(v[r * Q], w[r]));
  // q = Q - 1: X_{R-1} = sum_r W_R^{r (R-1)} W^{r jm} x_r with jm = t + (Q-1) T
  if constexpr (Q > 1) tw_powers<R>(__ldg(&g_tw[((t + (Q - 1) * T) & (NS - 1)) * (kMaxM / M)]), w);
  float2 xl = v[Q - 1];
  static_for_fft<1, R>([&](auto rc) {
    constexpr int r = decltype(rc)::value;
    xl = cadd(xl, twc<(r * (R - 1)) % R, R, false>(cmul(v[(Q - 1) + r * Q], w[r])));
  });
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = make_float2(0.f, 0.f);
  v[0] = x0;
  v[E - 1] = xl;
}

template <int M, int E, int P, bool HZ, class Sync>
__device__ __forceinline__ void fft_rows_edges(float2 (&v)[E], float2* sh, int t, const Twiddles<M, E>& tw,
                                               const Sync& sync) {
  constexpr int T = M / E;
  constexpr int NP = num_passes(M, E);
  if constexpr (P + 1 < NP) {
    if constexpr (P == 0 && HZ && pass_radix(M, E, 0) == E && E <= Pad<E>::P) {
      // zero-padded row (2N <= M): the first butterfly's inputs v[E/2..E) are zero
      dft_lz<E, E / 2, false>(v);
      sync.before_writing();
      float2* b = sh + padded<E>(t * E);
#pragma unroll
      for (int r = 0; r < E; ++r) b[r] = v[r];
    } else {
      stockham_pass<M, E, P, false>(v, sh, t, tw, sync);
    }
    sync();
    if constexpr (PadStride<E, T>::AFFINE) {
      const float2* b = sh + padded<E>(t);
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = b[e * PadStride<E, T>::value];
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = sh[padded<E>(t + e * T)];
    }
    sync.done_reading();
    fft_rows_edges<M, E, P + 1, HZ, Sync>(v, sh, t, tw, sync);
  } else {
    fft_last_edges<M, E, P>(v, t);
  }
}

}  // namespace graf
