// graf_kernels.cuh — the delay-row kernel and the reductions of the GRAF hot path.
//
// One kernel template, `af_rows_kernel<M>`, covers SURVEY.md §8(a) rows a0-a7:
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
// Rows are folded to k >= 0 (symmetric masks/weights): row k > 0 stands for
// rows +k and -k (loss sums and gradient terms counted twice; SURVEY §8(c)
// "symmetric-loss identities").  The generic adjoint (graf_af_backward) runs
// the same kernel in MODE_ADJ on unfolded rows read from dA.
#pragma once
#include "graf_fft.cuh"
#include "../../include/graf.h"

namespace graf {

enum : int { MODE_FWD = 0, MODE_ADJ = 1 };
enum : int { GRAD_NONE = 0, GRAD_ISL = 1, GRAD_PASS2 = 2, GRAD_ADJ = 3 };
constexpr int kPart = 8;  // doubles per CTA partial record: S, max, Z, C, fchi, -, -, -

struct RowParams {
  const float2* s;   // [B][N]
  int N, B, b0;      // b0: first waveform of this launch (grid.y chunking)
  int U;             // rows enumerated per waveform
  int row_lo, row_step;
  int mode;          // MODE_FWD (lag products, folded rows) | MODE_ADJ (rows from dA, unfolded)
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
  float xbar;
  double omega;        // |Omega| (full region, for the centred mean)
  int grad;            // GRAD_*
  const graf_partials* stats;  // combined partials [B] for GRAD_PASS2
  // outputs
  double* part;        // [B][P][kPart]
  float2* gpart;       // [B][P][N]
};

template <int M>
struct Cfg;
// E = values per thread, T = threads per row slot, S = row slots per CTA.
#define GRAF_CFG(M_, E_, S_)                                         \
  template <>                                                        \
  struct Cfg<M_> {                                                   \
    static constexpr int M = M_, E = E_, T = M_ / E_, S = S_;        \
    static constexpr int THREADS = T * S;                            \
    static constexpr int XS = M_ + M_ / E_; /* padded exchange */    \
    static constexpr bool S_SMEM = (M_ <= 8192);                     \
    static constexpr bool G_SMEM = (M_ <= 8192);                     \
  };
GRAF_CFG(2, 2, 64)
GRAF_CFG(4, 4, 64)
GRAF_CFG(8, 8, 64)
GRAF_CFG(16, 16, 64)
GRAF_CFG(32, 16, 32)
GRAF_CFG(64, 8, 16)
GRAF_CFG(128, 16, 16)
GRAF_CFG(256, 16, 8)
GRAF_CFG(512, 8, 2)
GRAF_CFG(1024, 16, 2)
GRAF_CFG(2048, 16, 1)
GRAF_CFG(4096, 16, 1)
GRAF_CFG(8192, 16, 1)
GRAF_CFG(16384, 16, 1)
#undef GRAF_CFG

template <int T, int S>
struct SlotSync {
  int id;
  __device__ __forceinline__ void operator()() const {
    if constexpr (T <= 32) {
      __syncwarp();
    } else if constexpr (S == 1) {
      __syncthreads();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(T) : "memory");
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

struct LsePart {
  double S, Z, C, F;
  float mx;
};

__device__ __forceinline__ void lse_merge(float& m, double& Z, float m2, double Z2, float invT) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) { m = m2; Z = Z2; return; }
  if (m2 > m) {
    Z = Z * exp((double)(m - m2) * invT) + Z2;
    m = m2;
  } else {
    Z = Z + Z2 * exp((double)(m2 - m) * invT);
  }
}

template <int M>
__global__ void __launch_bounds__(Cfg<M>::THREADS) af_rows_kernel(RowParams p) {
  using C = Cfg<M>;
  constexpr int E = C::E, T = C::T, S = C::S, THREADS = C::THREADS, XS = C::XS;
  extern __shared__ float4 smem_raw[];
  float2* smem = reinterpret_cast<float2*>(smem_raw);

  const int N = p.N;
  const int b = p.b0 + blockIdx.y;
  const int P = gridDim.x, pb = blockIdx.x;
  const int slot = threadIdx.x / T, t = threadIdx.x % T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float2* sg = p.s + (size_t)b * N;

  // ---- shared-memory carve-up: [energy scratch][s][exchange x S][g x S]
  double* red = reinterpret_cast<double*>(smem);  // 64 doubles of scratch
  float2* s_sh = smem + 64;
  float2* xch = s_sh + (C::S_SMEM ? ((N + 1) & ~1) : 0);
  float2* gacc_sh = xch + S * XS;
  const float2* sv = C::S_SMEM ? s_sh : sg;
  const bool want_g = (p.grad != GRAD_NONE);
  float2* gacc = C::G_SMEM ? gacc_sh + (size_t)slot * N
                           : p.gpart + ((size_t)b * P + pb) * N;  // S == 1 when !G_SMEM

  // ---- a0: stage s, zero the gradient accumulators, energy
  if constexpr (C::S_SMEM) {
    for (int i = threadIdx.x; i < N; i += THREADS) s_sh[i] = sg[i];
  }
  if (want_g) {
    if constexpr (C::G_SMEM) {
      for (int i = threadIdx.x; i < S * N; i += THREADS) gacc_sh[i] = make_float2(0.f, 0.f);
    } else {
      for (int i = threadIdx.x; i < N; i += THREADS) gacc[i] = make_float2(0.f, 0.f);
    }
  }
  if (warp == 0) {
    const double e = warp_energy(sg, N, lane);
    if (lane == 0) red[0] = e;
  }
  __syncthreads();
  const double Ed = red[0];
  const float invE = (float)(1.0 / Ed);
  const float invE2 = (float)(1.0 / Ed / Ed);
  const float scaleG = p.normalize ? invE2 : 1.0f;

  // pass-2 statistics from the combined partials (reading R13)
  float lse = 0.f, ebar = 0.f, invZc = 0.f;
  bool use_centred = false;
  if (p.grad == GRAD_PASS2) {
    const graf_partials g = p.stats[b];
    const double lse_d = g.lse_max + (double)p.T * log(g.lse_sum);
    lse = (float)lse_d;
    if (p.centred) {
      const double zc = p.omega + g.cen_sum;
      use_centred = isfinite(zc) && (g.lse_max - p.xbar) * p.invT <= 40.0;
      ebar = (float)(g.cen_sum / p.omega);
      invZc = (float)(1.0 / zc);
    }
  }

  SlotSync<T, S> sync{1 + slot};
  float2* sh = xch + (size_t)slot * XS;

  // per-thread accumulators (double across rows, float within a row)
  double accS = 0.0, accZ = 0.0, accC = 0.0, accF = 0.0;
  float accM = -INFINITY;

  const int rows_per_iter = P * S;
  const int iters = (p.U + rows_per_iter - 1) / rows_per_iter;
  const size_t surf_rows = (size_t)(p.ke - p.kb);

  for (int it = 0; it < iters; ++it) {
    const int u = it * rows_per_iter + pb * S + slot;
    const bool valid = u < p.U;
    const int k = p.row_lo + (valid ? u : 0) * p.row_step;
    float2 v[E];

    bool lrow = false, wpos = false, wneg = false;
    float mult = 1.f;
    const int lo = k > 0 ? k : 0;
    const int hi = k < 0 ? N + k : N;

    if (p.mode == MODE_FWD) {
      // ---- a1: lag product into the first-pass registers (time index n = t + e*T)
      wpos = valid && p.surface && k >= p.kb && k < p.ke;
      wneg = valid && p.surface && k > 0 && -k >= p.kb && -k < p.ke;
      lrow = valid && p.loss_on && k <= p.kloss && (k % p.shard_count) == p.shard_index;
      mult = (k == 0) ? 1.f : 2.f;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int n = t + e * T;
        float2 r = make_float2(0.f, 0.f);
        if (valid && n >= lo && n < hi) r = cmulc(sv[n], sv[n - k]);
        v[e] = r;
      }
      // ---- a2: forward Doppler FFT
      fft_rows<M, E, 1, false>(v, sh, t, sync);

      // ---- a3F: surface epilogue (rows +k and, folded, -k)
      if (wpos || wneg) {
        const float nrm = p.norm_out ? invE : 1.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int m = t + e * T;
          const float2 A = v[e];
          if (p.out_kind == GRAF_OUT_C64) {
            float2* out = reinterpret_cast<float2*>(p.surface);
            if (wpos) {
              const int col = p.layout ? ((m + M / 2) & (M - 1)) : m;
              __stcs(out + ((size_t)b * surf_rows + (k - p.kb)) * M + col, cscale(A, nrm));
            }
            if (wneg) {
              const int mn = (M - m) & (M - 1);
              const int col = p.layout ? ((mn + M / 2) & (M - 1)) : mn;
              const float2 w = g_tw[(int)(((long long)mn * k) & (M - 1)) * (kMaxM / M)];
              // A[-k, mn] = e^{+2 pi i mn k / M} conj(A[k, m]) = conj(w) * conj(A)
              const float2 val = cconj(cmul(w, A));
              __stcs(out + ((size_t)b * surf_rows + (-k - p.kb)) * M + col, cscale(val, nrm));
            }
          } else {
            float* out = reinterpret_cast<float*>(p.surface);
            const float chi = A.x * A.x + A.y * A.y;
            const float val = (p.out_kind == GRAF_OUT_ABS_F32) ? sqrtf(chi) * nrm : chi * nrm * nrm;
            if (wpos) {
              const int col = p.layout ? ((m + M / 2) & (M - 1)) : m;
              __stcs(out + ((size_t)b * surf_rows + (k - p.kb)) * M + col, val);
            }
            if (wneg) {
              const int mn = (M - m) & (M - 1);
              const int col = p.layout ? ((mn + M / 2) & (M - 1)) : mn;
              __stcs(out + ((size_t)b * surf_rows + (-k - p.kb)) * M + col, val);
            }
          }
        }
      }

      // ---- a3L (+ a5): loss partials and the cotangent
      if (lrow) {
        const float wk = p.w_k ? p.w_k[k + N - 1] : 1.f;
        float rowS = 0.f, rowM = -INFINITY;
        unsigned inmask = 0u;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int m = t + e * T;
          const int d = m < M / 2 ? m : m - M;
          const int ad = d < 0 ? -d : d;
          const bool in = ad <= p.d_max && !(k <= p.ml_k && ad <= p.ml_d);
          if (in) {
            inmask |= 1u << e;
            const float w = wk * (p.w_d ? p.w_d[d + M / 2] : 1.f);
            const float chi = v[e].x * v[e].x + v[e].y * v[e].y;
            rowS = fmaf(w, chi, rowS);
            const float x = p.normalize ? chi * invE2 : chi;
            rowM = fmaxf(rowM, x);
          }
        }
        accS += (double)mult * rowS;
        if (p.lam_psl != 0.f && p.grad != GRAD_PASS2 && inmask) {
          if (rowM > accM) {
            accZ = (accM == -INFINITY) ? 0.0 : accZ * exp((double)(accM - rowM) * p.invT);
            accM = rowM;
          }
          float rowZ = 0.f, rowC = 0.f;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            if (inmask & (1u << e)) {
              const float chi = v[e].x * v[e].x + v[e].y * v[e].y;
              const float x = p.normalize ? chi * invE2 : chi;
              rowZ += __expf((x - accM) * p.invT);
              if (p.centred) rowC += expm1f((x - p.xbar) * p.invT);
            }
          }
          accZ += (double)mult * rowZ;
          accC += (double)mult * rowC;
        } else if (p.lam_psl == 0.f && inmask) {
          accM = fmaxf(accM, rowM);
        }
        if (p.grad == GRAD_ISL || p.grad == GRAD_PASS2) {
          float rowF = 0.f;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            float2 G = make_float2(0.f, 0.f);
            if (inmask & (1u << e)) {
              const int m = t + e * T;
              const int d = m < M / 2 ? m : m - M;
              const float w = wk * (p.w_d ? p.w_d[d + M / 2] : 1.f);
              const float chi = v[e].x * v[e].x + v[e].y * v[e].y;
              float fp;
              if (p.grad == GRAD_ISL) {
                fp = p.lam_isl * w;
              } else {
                const float x = p.normalize ? chi * invE2 : chi;
                if (use_centred) {
                  fp = p.lam_psl * (expm1f((x - p.xbar) * p.invT) - ebar) * invZc;
                } else {
                  fp = p.lam_isl * w + p.lam_psl * __expf((x - lse) * p.invT);
                }
              }
              rowF = fmaf(fp, chi, rowF);
              G = cscale(v[e], fp * scaleG);
            }
            v[e] = G;
          }
          accF += (double)mult * rowF;
        }
      }
    } else {
      // ---- MODE_ADJ: G = dA row (unfolded k = kb + u)
      lrow = valid;
      mult = 1.f;
      const float2* drow = p.dA + ((size_t)b * surf_rows + (k - p.kb)) * M;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = t + e * T;
        const int col = p.layout ? ((m + M / 2) & (M - 1)) : m;
        v[e] = valid ? __ldcs(drow + col) : make_float2(0.f, 0.f);
      }
    }

    // ---- a6 + a7: inverse Doppler FFT and the delay correlation
    bool do_adj = want_g && p.grad != GRAD_NONE && lrow;
    if constexpr (T < 32) do_adj = __any_sync(0xffffffffu, do_adj);
    if (do_adj) {
      if (!lrow) {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = make_float2(0.f, 0.f);
      }
      fft_rows<M, E, 1, true>(v, sh, t, sync);
      if (lrow) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int n = t + e * T;
          if (n >= lo && n < hi) {
            const float2 add = cscale(cmul(v[e], sv[n - k]), mult);  // term 1 at p = n
            gacc[n] = cadd(gacc[n], add);
          }
        }
      }
      sync();
      if (lrow) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int n = t + e * T;
          if (n >= lo && n < hi) {
            const float2 add = cscale(cmul(cconj(v[e]), sv[n]), mult);  // term 2 at p = n - k
            gacc[n - k] = cadd(gacc[n - k], add);
          }
        }
      }
      sync();
    }
  }

  // ---- CTA reduction of the scalar partials (fixed shuffle tree + fixed warp order)
  __syncthreads();
  {
    double vS = accS, vZ = accZ, vC = accC, vF = accF;
    float vM = accM;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double oS = __shfl_down_sync(0xffffffffu, vS, off);
      const double oZ = __shfl_down_sync(0xffffffffu, vZ, off);
      const double oC = __shfl_down_sync(0xffffffffu, vC, off);
      const double oF = __shfl_down_sync(0xffffffffu, vF, off);
      const float oM = __shfl_down_sync(0xffffffffu, vM, off);
      if (lane + off < 32) {
        vS += oS; vC += oC; vF += oF;
        lse_merge(vM, vZ, oM, oZ, p.invT);
      }
    }
    double* wred = reinterpret_cast<double*>(xch);  // reuse exchange space
    constexpr int NW = (THREADS + 31) / 32;
    if (lane == 0) {
      wred[warp * 5 + 0] = vS;
      wred[warp * 5 + 1] = vZ;
      wred[warp * 5 + 2] = vC;
      wred[warp * 5 + 3] = vF;
      wred[warp * 5 + 4] = (double)vM;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double S0 = 0, Z0 = 0, C0 = 0, F0 = 0;
      float M0 = -INFINITY;
      for (int w = 0; w < NW; ++w) {
        S0 += wred[w * 5 + 0];
        C0 += wred[w * 5 + 2];
        F0 += wred[w * 5 + 3];
        lse_merge(M0, Z0, (float)wred[w * 5 + 4], wred[w * 5 + 1], p.invT);
      }
      double* rec = p.part + ((size_t)b * P + pb) * kPart;
      rec[0] = S0;
      rec[1] = (double)M0;
      rec[2] = Z0;
      rec[3] = C0;
      rec[4] = F0;
    }
  }

  // ---- gradient accumulators of all slots -> this CTA's partial g (fixed slot order)
  if (want_g && C::G_SMEM) {
    float2* gout = p.gpart + ((size_t)b * P + pb) * N;
    for (int n = threadIdx.x; n < N; n += THREADS) {
      float2 a = gacc_sh[n];
#pragma unroll 1
      for (int sl = 1; sl < S; ++sl) a = cadd(a, gacc_sh[(size_t)sl * N + n]);
      gout[n] = a;
    }
  }
}

// ---------------------------------------------------------------------------
// K3: combine the P CTA partial records of each waveform -> graf_partials[B]
// (+ the loss when `loss_out` != NULL).  One thread per waveform, fixed order.
// ---------------------------------------------------------------------------
struct ReduceParams {
  const double* part;
  int P, B;
  float invT, T;
  graf_partials* out;   // may be NULL
};

__global__ void partials_reduce_kernel(ReduceParams r) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= r.B) return;
  double S = 0, Z = 0, Cs = 0;
  float m = -INFINITY;
  for (int q = 0; q < r.P; ++q) {
    const double* rec = r.part + ((size_t)b * r.P + q) * kPart;
    S += rec[0];
    Cs += rec[3];
    lse_merge(m, Z, (float)rec[1], rec[2], r.invT);
  }
  graf_partials g;
  g.isl_sum = S;
  g.lse_max = (double)m;
  g.lse_sum = Z;
  g.cen_sum = Cs;
  r.out[b] = g;
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
  double* loss;                  // may be NULL
  float2* grad;                  // may be NULL
};

__global__ void __launch_bounds__(256) finalize_kernel(FinalizeParams f) {
  const int b = blockIdx.x;
  const int N = f.N;
  const float2* sg = f.s + (size_t)b * N;
  __shared__ double sh[2];
  if (threadIdx.x < 32) {
    const double e = warp_energy(sg, N, threadIdx.x);
    if (threadIdx.x == 0) {
      sh[0] = e;
      double S = 0, Z = 0, F = 0;
      float m = -INFINITY;
      for (int q = 0; q < f.P; ++q) {
        const double* rec = f.part + ((size_t)b * f.P + q) * kPart;
        S += rec[0];
        F += rec[4];
        lse_merge(m, Z, (float)rec[1], rec[2], f.invT);
      }
      sh[1] = F;
      if (f.loss) {
        double Sg = S, mg = m, Zg = Z;
        if (f.global) {
          Sg = f.global[b].isl_sum;
          mg = f.global[b].lse_max;
          Zg = f.global[b].lse_sum;
        }
        double L = f.lam_isl * (f.normalize ? Sg / (e * e) : Sg);
        if (f.lam_psl != 0.f) L += f.lam_psl * (mg + (double)f.T * log(Zg));
        f.loss[b] = L;
      }
    }
  }
  __syncthreads();
  if (!f.grad) return;
  const double E = sh[0];
  const float coef = (f.grad_norm_term && f.normalize) ? (float)(2.0 * sh[1] / (E * E * E)) : 0.f;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    double gx = 0, gy = 0;
    for (int q = 0; q < f.P; ++q) {
      const float2 a = f.gpart[((size_t)b * f.P + q) * N + n];
      gx += a.x;
      gy += a.y;
    }
    const float2 sv = sg[n];
    f.grad[(size_t)b * N + n] = make_float2((float)gx - coef * sv.x, (float)gy - coef * sv.y);
  }
}

struct CombineParams {
  const graf_partials* shards;
  int G, B;
  float invT;
  graf_partials* out;
};

__global__ void combine_partials_kernel(CombineParams c) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= c.B) return;
  double S = 0, Z = 0, Cs = 0;
  float m = -INFINITY;
  for (int q = 0; q < c.G; ++q) {
    const graf_partials g = c.shards[(size_t)q * c.B + b];
    S += g.isl_sum;
    Cs += g.cen_sum;
    lse_merge(m, Z, (float)g.lse_max, g.lse_sum, c.invT);
  }
  graf_partials o;
  o.isl_sum = S;
  o.lse_max = m;
  o.lse_sum = Z;
  o.cen_sum = Cs;
  c.out[b] = o;
}

}  // namespace graf
