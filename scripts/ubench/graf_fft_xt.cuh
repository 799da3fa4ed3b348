// graf_fft_xt.cuh — EXPERIMENT (round 2, not in the library): the M = 16384 row FFT with one
// of its two exchanges through TENSOR MEMORY.  Correct (scripts/ubench/xt_fft_test.cu: forward
// 6.4e-7 relative to a float64 DFT, inverse exact to 1.2e-6), and it halves the shared-memory
// wavefronts of the FFTs, but a forward + inverse pair takes the same 19.1-19.5 K cycles per SM
// as the production Stockham plan (profiles/r02/ubench/ncu_xt_vs_stockham.txt): the FP work is
// identical and the quarter barriers / tcgen05 waits replace the shared-memory stalls.  Kept as
// the measured evidence behind DESIGN.md §7 ("what bounds c5").
//
// Same transform as the Stockham plan of graf_fft.cuh (Eq. 11;
// the adjoint's inverse DFT, L230): 16384 = 32 x 32 x 16, the time index
// n = n_lo + 16 n_mid + 512 n_hi and the frequency m = m_a + 32 m_b + 1024 m_c,
//   pass 0: DFT-32 over n_hi -> m_a
//   twiddle 1: W_1024^(m_a n_mid);        pass 1: DFT-32 over n_mid -> m_b
//   twiddle 2: W_16384^(n_lo (m_a + 32 m_b));  pass 2: DFT-16 over n_lo -> m_c
// (exponents add up to n m mod 16384).  What differs is WHERE the data lives between
// passes.  512 threads hold 32 values each; thread t = lane l + 32 w, w = q + 4 h with
// q = w mod 4 the warp's TMEM lane quarter and h = w / 4.
//   layout A (time; lag product, correlation): thread t holds n = t + 512 e in slot e.
//   layout B (pass 1): m_a = (l & 7) + 8 q, n_lo = (l >> 3) + 4 h; slot e = n_mid.
//   layout C (pass 2, frequency): m_a = (l >> 2) + 8 q, m_b = (l & 3) + 4 h + 16 (e >> 4);
//     slot e = 16 m_b4 + n_lo before pass 2, 16 m_b4 + m_c after it (xt_freq).
// A -> B moves the quarter bits q, which tensor memory cannot (a warp reaches only the 32
// lanes of its quarter), so it goes through shared memory: one write, one CTA barrier,
// one read, with an XOR swizzle that makes both sides conflict-free (2 wavefronts per
// 64-bit warp access; checked offline).  B -> C only moves bits within the four warps of a
// quarter (h) and within a warp's lanes, which is exactly what tcgen05 can do: every thread
// stores its values into its own lane with the 32x32b shape, the quarter's 128 threads meet
// at a named barrier, and each thread gathers with the 16x128b shape, whose thread <-> lane
// map (thread l reads lanes (l >> 2) and (l >> 2) + 8, column l & 3) performs the lane-bit
// part of the permutation.  Measured on B200 (scripts/ubench/tmem_xchg.cu): a full
// 128 KiB exchange takes 549 cycles through tensor memory against 2061 through shared
// memory, and it overlaps the FP32 work of the other quarters.  The exchange runs in two
// rounds of 16 values (m_b4 = 0, 1) so its region is 128 columns: the CTA's 512 columns
// hold the gradient accumulator [0, 256), the pass-1 twiddles [256, 320) and the exchange
// region [384, 512).  The inverse runs the adjoint steps in reverse order (layouts C -> B
// -> A), so the epilogue and the correlation see the same layouts as before.
#pragma once
#include "../../paper_2506_22935_b200/csrc/graf_fft.cuh"

namespace graf {

constexpr int kXtTw1Col = 256;   // pass-1 twiddles: 62 columns per lane
constexpr int kXtXchCol = 384;   // B <-> C exchange region: 4 warps x 32 columns

// conflict-free swizzle of the A <-> B shared-memory exchange (a permutation of each
// 16-entry group: low 4 bits ^= (y6, y7, y8, y5))
__device__ __forceinline__ int xt_swz(int y) { return y ^ (((y >> 6) & 7) | (((y >> 5) & 1) << 3)); }

// frequency index m held in slot e of thread t (layout C, after the forward FFT)
__host__ __device__ constexpr int xt_freq(int t, int e) {
  return ((t & 31) >> 2) + 8 * ((t >> 5) & 3) +
         32 * ((t & 3) + 4 * (t >> 7) + 16 * (e >> 4)) + 1024 * (e & 15);
}

__device__ __forceinline__ void xt_st32x32b_x32(uint32_t a, const float (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
      "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]), "f"(r[8]), "f"(r[9]),
      "f"(r[10]), "f"(r[11]), "f"(r[12]), "f"(r[13]), "f"(r[14]), "f"(r[15]), "f"(r[16]), "f"(r[17]), "f"(r[18]),
      "f"(r[19]), "f"(r[20]), "f"(r[21]), "f"(r[22]), "f"(r[23]), "f"(r[24]), "f"(r[25]), "f"(r[26]), "f"(r[27]),
      "f"(r[28]), "f"(r[29]), "f"(r[30]), "f"(r[31])
      : "memory");
}
__device__ __forceinline__ void xt_ld16x128b_x2(uint32_t a, float* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
               : "r"(a)
               : "memory");
}
__device__ __forceinline__ void xt_st16x128b_x2(uint32_t a, const float* r) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(r[0]), "f"(r[1]),
               "f"(r[2]), "f"(r[3])
               : "memory");
}
__device__ __forceinline__ void xt_ld32x32b_x8(uint32_t a, float* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "r"(a)
               : "memory");
}
// wait::ld tied to the 32 loaded registers (no use of them is scheduled above it)
__device__ __forceinline__ void xt_wait_ld32(float (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(r[0]), "+f"(r[1]), "+f"(r[2]), "+f"(r[3]), "+f"(r[4]), "+f"(r[5]), "+f"(r[6]), "+f"(r[7]),
                 "+f"(r[8]), "+f"(r[9]), "+f"(r[10]), "+f"(r[11]), "+f"(r[12]), "+f"(r[13]), "+f"(r[14]),
                 "+f"(r[15]), "+f"(r[16]), "+f"(r[17]), "+f"(r[18]), "+f"(r[19]), "+f"(r[20]), "+f"(r[21]),
                 "+f"(r[22]), "+f"(r[23]), "+f"(r[24]), "+f"(r[25]), "+f"(r[26]), "+f"(r[27]), "+f"(r[28]),
                 "+f"(r[29]), "+f"(r[30]), "+f"(r[31])
               :
               : "memory");
}
// the 128 threads of TMEM lane quarter q (warps q, q + 4, q + 8, q + 12): named barrier 8 + q
__device__ __forceinline__ void xt_quarter_sync(int q) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("bar.sync %0, 128;" ::"r"(8 + q) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Pass-1 twiddles of this thread's lane (layout B: m_a = (l & 7) + 8 q), written once per
// kernel by the warps with h = 0; tw1 = tmem base + lane field of the warp's quarter.
__device__ __forceinline__ void xt_fill_tw1(uint32_t tw1, int t) {
  const int ma = (t & 7) + 8 * ((t >> 5) & 3);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float w16[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 8 * c + i + 1;
      const float2 w = r < 32 ? g_tw[16 * ((ma * r) & 1023)] : make_float2(0.f, 0.f);
      w16[2 * i] = w.x;
      w16[2 * i + 1] = w.y;
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};" ::"r"(tw1 + 16 * c),
        "f"(w16[0]), "f"(w16[1]), "f"(w16[2]), "f"(w16[3]), "f"(w16[4]), "f"(w16[5]), "f"(w16[6]), "f"(w16[7]),
        "f"(w16[8]), "f"(w16[9]), "f"(w16[10]), "f"(w16[11]), "f"(w16[12]), "f"(w16[13]), "f"(w16[14]),
        "f"(w16[15])
        : "memory");
  }
}

// slot <-> column of the B-side values in the exchange region (per round, u = m_b & 15):
// column bits (m_b0, m_b1, re/im, m_b2, m_b3)
__host__ __device__ constexpr int xt_bcol(int u, int im) { return (u & 3) + 4 * im + 8 * ((u >> 2) & 3); }

// layout B -> C (forward) through the exchange region; xq = tmem base + quarter lane field
// + kXtXchCol.  Round rho moves the slots 16 rho .. 16 rho + 15 (m_b4 = rho) and the
// gathered values land in the same slots (slot 16 m_b4 + n_lo), so no value is overwritten
// before it is stored.
__device__ __forceinline__ void xt_exchange_bc(float2 (&v)[32], uint32_t xq, int q, int h) {
#pragma unroll
  for (int rho = 0; rho < 2; ++rho) {
    float f[32];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      f[xt_bcol(u, 0)] = v[16 * rho + u].x;
      f[xt_bcol(u, 1)] = v[16 * rho + u].y;
    }
    xt_st32x32b_x32(xq + 32 * h, f);   // own lane, own warp's 32 columns
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    xt_quarter_sync(q);
    // reader: n_lo = v1 + 2 half + 4 hh from writer lane (l >> 2) + 8 v1 + 16 half of warp
    // (q, hh); columns 8 h + 4 (re/im) + (l & 3) = (m_b0, m_b1) of the reader's m_b
    float g[32];
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll
      for (int hh = 0; hh < 4; ++hh)
        xt_ld16x128b_x2(xq + ((uint32_t)(16 * half) << 16) + 32 * hh + 8 * h, &g[4 * (4 * half + hh)]);
    xt_wait_ld32(g);
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll
      for (int hh = 0; hh < 4; ++hh)
#pragma unroll
        for (int v1 = 0; v1 < 2; ++v1) {
          const int i = 4 * (4 * half + hh);
          v[16 * rho + v1 + 2 * half + 4 * hh] = make_float2(g[i + v1], g[i + 2 + v1]);
        }
    xt_quarter_sync(q);   // the region is free again
  }
}

// layout C -> B (the inverse's adjoint of xt_exchange_bc): the C side stores with the
// 16x128b shape, the B side gathers its own lane with 32x32b
__device__ __forceinline__ void xt_exchange_cb(float2 (&v)[32], uint32_t xq, int q, int h) {
#pragma unroll
  for (int rho = 0; rho < 2; ++rho) {
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        const float2 a = v[16 * rho + 2 * half + 4 * cb], c = v[16 * rho + 1 + 2 * half + 4 * cb];
        const float f[4] = {a.x, c.x, a.y, c.y};
        xt_st16x128b_x2(xq + ((uint32_t)(16 * half) << 16) + 32 * h + 8 * cb, f);
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    xt_quarter_sync(q);
    float g[32];
#pragma unroll
    for (int hw = 0; hw < 4; ++hw) xt_ld32x32b_x8(xq + 32 * hw + 8 * h, &g[8 * hw]);
    xt_wait_ld32(g);
    // columns (m_b0, m_b1, re/im) of region hw = (m_b2, m_b3)
#pragma unroll
    for (int hw = 0; hw < 4; ++hw)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[16 * rho + c + 4 * hw] = make_float2(g[8 * hw + c], g[8 * hw + 4 + c]);
    xt_quarter_sync(q);
  }
}

// One-round forms (GRAF_XT_ONE_ROUND = 1): the whole exchange at once in a 256-column region
// (columns [256, 512); the pass-1 twiddles must then come from shared memory, GRAF_XT_TW1 = 2)
#ifndef GRAF_XT_ONE_ROUND
#define GRAF_XT_ONE_ROUND 0
#endif
constexpr int kXtXchCol1 = 256;
__device__ __forceinline__ void xt_st32x32b_x64(uint32_t a, const float (&r)[64]) {
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
__device__ __forceinline__ void xt_exchange_bc1(float2 (&v)[32], uint32_t xq, int q, int h) {
  {
    float f[64];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      f[xt_bcol(e, 0) + 32 * (e >> 4)] = v[e].x;
      f[xt_bcol(e, 1) + 32 * (e >> 4)] = v[e].y;
    }
    xt_st32x32b_x64(xq + 64 * h, f);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  xt_quarter_sync(q);
#pragma unroll
  for (int rho = 0; rho < 2; ++rho) {
    float g[32];
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll
      for (int hh = 0; hh < 4; ++hh)
        xt_ld16x128b_x2(xq + ((uint32_t)(16 * half) << 16) + 64 * hh + 32 * rho + 8 * h, &g[4 * (4 * half + hh)]);
    xt_wait_ld32(g);
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll
      for (int hh = 0; hh < 4; ++hh)
#pragma unroll
        for (int v1 = 0; v1 < 2; ++v1) {
          const int i = 4 * (4 * half + hh);
          v[16 * rho + v1 + 2 * half + 4 * hh] = make_float2(g[i + v1], g[i + 2 + v1]);
        }
  }
  xt_quarter_sync(q);
}
__device__ __forceinline__ void xt_exchange_cb1(float2 (&v)[32], uint32_t xq, int q, int h) {
#pragma unroll
  for (int rho = 0; rho < 2; ++rho)
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        const float2 a = v[16 * rho + 2 * half + 4 * cb], c = v[16 * rho + 1 + 2 * half + 4 * cb];
        const float f[4] = {a.x, c.x, a.y, c.y};
        xt_st16x128b_x2(xq + ((uint32_t)(16 * half) << 16) + 64 * h + 32 * rho + 8 * cb, f);
      }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  xt_quarter_sync(q);
#pragma unroll
  for (int rho = 0; rho < 2; ++rho) {
    float g[32];
#pragma unroll
    for (int hw = 0; hw < 4; ++hw) xt_ld32x32b_x8(xq + 64 * hw + 32 * rho + 8 * h, &g[8 * hw]);
    xt_wait_ld32(g);
#pragma unroll
    for (int hw = 0; hw < 4; ++hw)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[16 * rho + c + 4 * hw] = make_float2(g[8 * hw + c], g[8 * hw + 4 + c]);
  }
  xt_quarter_sync(q);
}

// pass-1 twiddles (layout B slot e = n_mid): x_e *= W_1024^(m_a e) (conjugate for INV).
// GRAF_XT_TW1: 0 = tensor memory, one wait per 8 twiddles; 1 = tensor memory, two loads in
// flight per wait; 2 = shared-memory table tab[(e - 1) 32 + m_a] (8 distinct m_a per warp:
// broadcast reads, one wavefront each)
#ifndef GRAF_XT_TW1
#define GRAF_XT_TW1 1
#endif
template <bool INV>
__device__ __forceinline__ void xt_twiddle1(float2 (&v)[32], uint32_t tw1, const float2* tab, int t) {
  if constexpr (GRAF_XT_TW1 == 2) {
    const float2* tb = tab + (t & 7) + 8 * ((t >> 5) & 3) - 32;
#pragma unroll
    for (int r = 1; r < 32; ++r) {
      const float2 w = tb[32 * r];
      v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
    }
  } else if constexpr (GRAF_XT_TW1 == 1) {
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
      float w32[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
          "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=f"(w32[0]), "=f"(w32[1]), "=f"(w32[2]), "=f"(w32[3]), "=f"(w32[4]), "=f"(w32[5]), "=f"(w32[6]),
            "=f"(w32[7]), "=f"(w32[8]), "=f"(w32[9]), "=f"(w32[10]), "=f"(w32[11]), "=f"(w32[12]), "=f"(w32[13]),
            "=f"(w32[14]), "=f"(w32[15]), "=f"(w32[16]), "=f"(w32[17]), "=f"(w32[18]), "=f"(w32[19]),
            "=f"(w32[20]), "=f"(w32[21]), "=f"(w32[22]), "=f"(w32[23]), "=f"(w32[24]), "=f"(w32[25]),
            "=f"(w32[26]), "=f"(w32[27]), "=f"(w32[28]), "=f"(w32[29]), "=f"(w32[30]), "=f"(w32[31])
          : "r"(tw1 + 32 * c2)
          : "memory");
      xt_wait_ld32(w32);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = 16 * c2 + i + 1;
        if (r < 32) {
          const float2 w = make_float2(w32[2 * i], w32[2 * i + 1]);
          v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
        }
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float w16[16];
      tmem_tw_ld16(tw1 + 16 * c, w16);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 8 * c + i + 1;
        if (r < 32) {
          const float2 w = make_float2(w16[2 * i], w16[2 * i + 1]);
          v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
        }
      }
    }
  }
}
// fill the shared pass-1 table (GRAF_XT_TW1 == 2): 31 x 32 entries, all threads of the CTA
__device__ __forceinline__ void xt_fill_tab(float2* tab, int tid, int nthreads) {
  for (int i = tid; i < 31 * 32; i += nthreads) {
    const int r = i / 32 + 1, ma = i % 32;
    tab[i] = g_tw[16 * ((ma * r) & 1023)];
  }
}

// pass 2 (layout C): for m_b4 = 0, 1 a radix-16 DFT over n_lo (slots 16 m_b4 + 0..15) with
// the twiddles W^(n_lo j), j = m_a + 32 m_b: powers of ONE table read per thread (m_b4 = 1
// adds 512 to j: the compile-time factor W_32^r)
template <bool INV>
__device__ __forceinline__ void xt_pass2(float2 (&v)[32], int t) {
  const int l = t & 31, w = t >> 5;
  const int j0 = (l >> 2) + 8 * (w & 3) + 32 * ((l & 3) + 4 * (w >> 2));
  const float2 b0 = __ldg(&g_tw[j0]);
#pragma unroll
  for (int qq = 0; qq < 2; ++qq) {
    float2 wp[16];
    tw_powers<16>(qq == 0 ? b0 : cmul(b0, make_float2(cos32(1), -sin32(1))), wp);
    float2 x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = v[16 * qq + r];
    if constexpr (!INV) {
#pragma unroll
      for (int r = 1; r < 16; ++r) x[r] = cmul(x[r], wp[r]);
      dft<16, false>(x);
    } else {
      dft<16, true>(x);
#pragma unroll
      for (int r = 1; r < 16; ++r) x[r] = cmulc(x[r], wp[r]);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) v[16 * qq + r] = x[r];
  }
}

// A <-> B through the (unpadded, swizzled) shared-memory exchange buffer sh[16384]
template <bool A_TO_B, class Sync>
__device__ __forceinline__ void xt_exchange_ab(float2 (&v)[32], float2* sh, int t, const Sync& sync) {
  const int l = t & 31, w = t >> 5;
  const int abase = 32 * (t & 15) + 512 * (t >> 4);                 // A: y = m_a + abase
  const int bbase = (l & 7) + 8 * (w & 3) + 32 * ((l >> 3) + 4 * (w >> 2));   // B: y = bbase + 512 n_mid
  sync.before_writing();
#pragma unroll
  for (int e = 0; e < 32; ++e) sh[xt_swz(A_TO_B ? abase + e : bbase + 512 * e)] = v[e];
  sync();
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = sh[xt_swz(A_TO_B ? bbase + 512 * e : abase + e)];
  sync.done_reading();
}

// Forward FFT: v in layout A (time) -> layout C (frequency, xt_freq).
// tw1 / xq: this thread's lane field + kXtTw1Col / + kXtXchCol in the CTA's TMEM.
template <class Sync>
__device__ __forceinline__ void fft16384_xt_fwd(float2 (&v)[32], float2* sh, uint32_t tw1, uint32_t xq, int t,
                                                const Sync& sync, const float2* tab = nullptr) {
  const int w = t >> 5;
  dft<32, false>(v);                      // pass 0 over n_hi
  xt_exchange_ab<true>(v, sh, t, sync);
  xt_twiddle1<false>(v, tw1, tab, t);
  dft<32, false>(v);                      // pass 1 over n_mid
  if constexpr (GRAF_XT_ONE_ROUND) xt_exchange_bc1(v, xq, w & 3, w >> 2);
  else xt_exchange_bc(v, xq, w & 3, w >> 2);
  xt_pass2<false>(v, t);                  // twiddle 2 + pass 2 over n_lo
}

// Inverse (unnormalised, e^{+}) FFT: v in layout C -> layout A; the adjoint of every
// forward step in reverse order
template <class Sync>
__device__ __forceinline__ void fft16384_xt_inv(float2 (&v)[32], float2* sh, uint32_t tw1, uint32_t xq, int t,
                                                const Sync& sync, const float2* tab = nullptr) {
  const int w = t >> 5;
  xt_pass2<true>(v, t);
  if constexpr (GRAF_XT_ONE_ROUND) xt_exchange_cb1(v, xq, w & 3, w >> 2);
  else xt_exchange_cb(v, xq, w & 3, w >> 2);
  dft<32, true>(v);
  xt_twiddle1<true>(v, tw1, tab, t);
  xt_exchange_ab<false>(v, sh, t, sync);
  dft<32, true>(v);
}

}  // namespace graf
