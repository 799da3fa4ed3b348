// graf_api.cu — the C ABI (include/graf.h): argument checks, launch planning,
// workspace layout and the kernel sequences of each entry point.
#include <cuda_runtime.h>

#define GRAF_API_UNIT 1   // this unit defines the non-template kernels of graf_kernels.cuh

#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/graf.h"
#include "graf_launch.cuh"

namespace graf {
thread_local int t_launches = 0;   // kernels / memsets enqueued by this thread's last entry-point call
std::vector<TwFill>& tw_fillers() {
  static std::vector<TwFill> v;   // filled by the row-kernel translation units at load time
  return v;
}
namespace {

thread_local std::string t_last_error;
// cross-ambiguity operands of a graf_xaf_* call (both NULL for the auto entry points)
struct CallCtx {
  const void* s2 = nullptr;
  void* grad2 = nullptr;
  bool cross() const { return s2 != nullptr; }
};
thread_local cudaEvent_t t_prof_start = nullptr, t_prof_stop = nullptr;

cudaError_t prof_mark(bool start, cudaStream_t st) {
  cudaEvent_t ev = start ? t_prof_start : t_prof_stop;
  if (!t_prof_start || !t_prof_stop) return cudaSuccess;
  // inside stream capture the record must be an external event node to be timeable
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    return cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  return cudaEventRecord(ev, st);
}

graf_status fail(graf_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
graf_status fail(graf_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = buf;
  return st;
}

graf_status cuda_fail(cudaError_t e, const char* what) {
  return fail(GRAF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// per-device twiddle table (immutable once filled).  The fill is a kernel per
// translation unit, enqueued on the stream of the first call (never a host-blocking
// copy).  State per device: 0 not filled, 1 fill enqueued on `st` (event `ev`
// recorded after it), 2 known complete.  A call on another stream while the fill is
// in flight waits on `ev` (device-side); a call inside CUDA-graph capture that cannot
// prove the fill complete records its own (idempotent) fill into the graph.
// ---------------------------------------------------------------------------
struct TwState {
  std::mutex mu;
  int state = 0;
  cudaStream_t st = nullptr;
  cudaEvent_t ev = nullptr;
};
TwState g_tws[kMaxDev];

cudaError_t fill_all_twiddles(cudaStream_t st) {
  cudaError_t e = launch_tw_init(st);   // this unit's copy (graf_fft.cuh)
  for (auto f : tw_fillers())
    if (e == cudaSuccess) e = f(st);
  if (e == cudaSuccess) t_launches += 1 + (int)tw_fillers().size();
  return e;
}

cudaError_t ensure_twiddles(cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  TwState& s = g_tws[dev];
  std::lock_guard<std::mutex> lk(s.mu);
  if (s.state == 2) return cudaSuccess;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if ((e = cudaStreamIsCapturing(st, &cs)) != cudaSuccess) return e;
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  if (s.state == 1) {
    if (st == s.st) return cudaSuccess;               // stream-ordered after the fill
    if (capturing) return fill_all_twiddles(st);      // the graph carries its own fill
    const cudaError_t q = cudaEventQuery(s.ev);
    if (q == cudaSuccess) {
      s.state = 2;
      return cudaSuccess;
    }
    if (q != cudaErrorNotReady) return q;
    (void)cudaGetLastError();                         // NotReady is a status, not an error
    return cudaStreamWaitEvent(st, s.ev, 0);
  }
  if ((e = fill_all_twiddles(st)) != cudaSuccess) return e;
  if (capturing) return cudaSuccess;                  // not marked: the fill runs at replay
  if (!s.ev && (e = cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(s.ev, st)) != cudaSuccess) return e;
  s.st = st;
  s.state = 1;
  return cudaSuccess;
}

struct CfgInfo {
  int M, E, T, S, threads, XS, tab1;
  bool s_smem, g_smem, s_trim;
};

template <int M>
CfgInfo cfg_info() {
  using C = Cfg<M>;
  constexpr int E2 = C::SPLIT ? C::E / 2 : C::E;
  return CfgInfo{M, C::E, C::T, C::S, C::THREADS, C::XS, Twiddles<C::MX, E2>::TAB1, C::S_SMEM, C::G_SMEM, C::S_TRIM};
}

bool cfg_for(int M, CfgInfo* ci) {
  switch (M) {
    case 2: *ci = cfg_info<2>(); return true;
    case 4: *ci = cfg_info<4>(); return true;
    case 8: *ci = cfg_info<8>(); return true;
    case 16: *ci = cfg_info<16>(); return true;
    case 32: *ci = cfg_info<32>(); return true;
    case 64: *ci = cfg_info<64>(); return true;
    case 128: *ci = cfg_info<128>(); return true;
    case 256: *ci = cfg_info<256>(); return true;
    case 512: *ci = cfg_info<512>(); return true;
    case 1024: *ci = cfg_info<1024>(); return true;
    case 2048: *ci = cfg_info<2048>(); return true;
    case 4096: *ci = cfg_info<4096>(); return true;
    case 8192: *ci = cfg_info<8192>(); return true;
    case 16384: *ci = cfg_info<16384>(); return true;
    default: return false;
  }
}


bool is_pow2(long long x) { return x > 0 && (x & (x - 1)) == 0; }
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

graf_status check_af(const graf_af_desc* af) {
  if (!af) return fail(GRAF_EINVAL, "af descriptor is NULL");
  if (af->abi_version != GRAF_ABI_VERSION)
    return fail(GRAF_EINVAL, "abi_version %d != %d", af->abi_version, GRAF_ABI_VERSION);
  if (af->n < 1) return fail(GRAF_EINVAL, "N = %d < 1", af->n);
  if (af->batch < 1) return fail(GRAF_EINVAL, "batch = %lld < 1", (long long)af->batch);
  if (!is_pow2(af->m) || af->m < 2) return fail(GRAF_EINVAL, "M = %d is not a power of two >= 2", af->m);
  if (af->m > GRAF_MAX_M) return fail(GRAF_EUNSUPPORTED, "M = %d > %d", af->m, GRAF_MAX_M);
  if (af->m < af->n) return fail(GRAF_EUNSUPPORTED, "M = %d < N = %d (v1 device path needs M >= N)", af->m, af->n);
  if (af->out_kind < GRAF_OUT_NONE || af->out_kind > GRAF_OUT_POW_F32)
    return fail(GRAF_EINVAL, "out_kind %d", af->out_kind);
  if (af->doppler_layout != GRAF_DOPPLER_RAW && af->doppler_layout != GRAF_DOPPLER_CENTERED)
    return fail(GRAF_EINVAL, "doppler_layout %d", af->doppler_layout);
  const int sc = af->shard_count <= 0 ? 1 : af->shard_count;
  if (af->shard_index < 0 || af->shard_index >= sc)
    return fail(GRAF_EINVAL, "shard_index %d not in [0, %d)", af->shard_index, sc);
  if (af->periodic != 0 && af->periodic != 1) return fail(GRAF_EINVAL, "periodic must be 0 or 1");
  if (af->periodic && af->m != af->n)
    return fail(GRAF_EUNSUPPORTED, "periodic surface needs M == N (M = %d, N = %d)", af->m, af->n);
  return GRAF_OK;
}

graf_status check_window(const graf_af_desc* af) {
  if (af->k_begin < -(af->n - 1) || af->k_end > af->n || af->k_begin >= af->k_end)
    return fail(GRAF_EINVAL, "row window [%d, %d) not inside [-(N-1), N) = [%d, %d)", af->k_begin, af->k_end,
                -(af->n - 1), af->n);
  if (af->periodic && af->k_end - af->k_begin > af->n)
    return fail(GRAF_EINVAL, "periodic row window [%d, %d) holds more than N = %d delays", af->k_begin,
                af->k_end, af->n);
  return GRAF_OK;
}

graf_status check_loss(const graf_af_desc* af, const graf_loss_desc* L) {
  if (L->k_max < 0 || L->d_max < 0 || L->ml_k < 0 || L->ml_d < 0)
    return fail(GRAF_EINVAL, "negative region bound");
  if (L->normalize != 0 && L->normalize != 1) return fail(GRAF_EINVAL, "normalize must be 0 or 1");
  if (L->lambda_psl != 0.f && !(L->temperature > 0.f)) return fail(GRAF_EINVAL, "temperature must be > 0");
  if (!std::isfinite(L->lambda_isl) || !std::isfinite(L->lambda_psl) || !std::isfinite(L->lambda_hpsl) ||
      !std::isfinite(L->lambda_match))
    return fail(GRAF_EINVAL, "non-finite lambda");
  if (L->lambda_match != 0.f) {
    if (!L->target || (reinterpret_cast<uintptr_t>(L->target) & 3u)) return fail(GRAF_EINVAL, "match target NULL or misaligned");
    if (L->lambda_psl != 0.f) return fail(GRAF_EUNSUPPORTED, "match loss with soft-PSL (v1: ISL and hard PSL only)");
    if (L->target_stride < 0) return fail(GRAF_EINVAL, "negative target_stride");
    // the target window must hold every delay of the region (R24)
    const int klm = std::min(L->k_max, af->periodic ? af->n / 2 : af->n - 1);
    if (af->periodic ? (af->k_end - af->k_begin != af->n) : (af->k_begin > -klm || af->k_end <= klm))
      return fail(GRAF_EINVAL, "match target window [%d, %d) does not cover the region's delays", af->k_begin,
                  af->k_end);
    if (af->k_begin < -(af->n - 1) || af->k_end > af->n || af->k_begin >= af->k_end)
      return fail(GRAF_EINVAL, "match target window [%d, %d) invalid", af->k_begin, af->k_end);
  }
  const int kl = std::min(L->k_max, af->periodic ? af->n / 2 : af->n - 1);
  const int dl = std::min(L->d_max, af->m / 2);
  const bool nonempty = kl > L->ml_k || dl > L->ml_d;
  if (!nonempty) return fail(GRAF_EINVAL, "empty sidelobe region (mainlobe covers the mask)");
  return GRAF_OK;
}

bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }

// fold the unfolded window [kb, ke) to |k|: a contiguous range [lo, hi]
void folded_window(int kb, int ke, int* lo, int* hi) {
  const int a = kb, z = ke - 1;
  if (a <= 0 && z >= 0) {
    *lo = 0;
    *hi = std::max(-a, z);
  } else if (a > 0) {
    *lo = a;
    *hi = z;
  } else {
    *lo = -z;
    *hi = -a;
  }
}

enum class Kind { Forward, LossGrad, Backward };

// elements of one global s copy (pad_s_kernel): B rows of NL + M + 2, NL = N rounded up to
// even (the +2 holds s[N-1] of the shifted copy when N == M), plus N + 2 of tail slack
// (kept even so the second copy starts 16-byte aligned)
size_t spad_elems(long long B, int N, int M) {
  return (size_t)B * (size_t)(N + (N & 1) + M + 2) + (size_t)(N + (N & 1) + 2);
}

Plan make_plan(const graf_af_desc* af, const graf_loss_desc* L, Kind kind, bool cross = false) {
  Plan pl;
  pl.cross = cross;
  CfgInfo ci;
  cfg_for(af->m, &ci);
  pl.M = af->m;
  pl.threads = ci.threads;
  pl.S = ci.S;
  pl.T = ci.T;
  pl.s_smem = ci.s_smem;
  pl.g_smem = ci.g_smem;
  const int N = af->n;
  const int sc = af->shard_count <= 0 ? 1 : af->shard_count;
  const bool grad = (kind != Kind::Forward);
  if (kind == Kind::Backward) {
    pl.row_lo = af->k_begin;
    pl.row_step = 1;
    pl.U = af->k_end - af->k_begin;
  } else {
    const bool surf = af->out_kind != GRAF_OUT_NONE;
    const int kfold = af->periodic ? N / 2 : N - 1;   // largest folded delay
    const int kloss = L ? std::min(L->k_max, kfold) : -1;
    if (cross) {
      // unfolded rows: the loss rows [-kloss, kloss] and the surface window
      int lo = L ? -kloss : INT32_MAX, hi = L ? kloss : INT32_MIN;
      if (surf) {
        lo = std::min(lo, af->k_begin);
        hi = std::max(hi, af->k_end - 1);
      }
      pl.row_lo = lo;
      pl.row_step = 1;
      pl.U = (L || surf) ? hi - lo + 1 : 0;
    } else if (surf) {
      int lo, hi;
      if (af->periodic) {   // every folded residue pair may meet the window
        lo = 0;
        hi = kfold;
      } else {
        folded_window(af->k_begin, af->k_end, &lo, &hi);
      }
      if (L) {
        lo = 0;
        hi = std::max(hi, kloss);
      }
      pl.row_lo = lo;
      pl.row_step = 1;
      pl.U = hi - lo + 1;
    } else if (L) {
      pl.row_lo = af->shard_index;
      pl.row_step = sc;
      pl.U = af->shard_index <= kloss ? (kloss - af->shard_index) / sc + 1 : 0;
    } else {
      pl.U = 0;
    }
  }
  const size_t nsig = cross ? 2 : 1;   // staged waveforms and gradient accumulator sets
  // staged s: [N zeros][N samples][M - N zeros], or unpadded (s_trim: [N] / periodic [2N])
  // (cross-ambiguity kernels keep the padded s and shared-memory accumulators, graf_kernels.cuh)
  const bool s_trim = ci.s_trim && !cross, g_smem = ci.g_smem || cross;
  const size_t s_elems = !ci.s_smem ? 0 : s_trim ? (size_t)(((af->periodic ? 2 * N : N) + 1) & ~1)
                                                 : (size_t)((N + af->m + 1) & ~1);
  pl.smem = sizeof(float2) * (64 + s_elems +
                              (cross ? (size_t)((2 * N + af->m + 1) & ~1) : 0) + (size_t)ci.S * ci.XS +
                              (grad && g_smem ? nsig * ci.S * N : 0) + (size_t)ci.tab1);
  if (kind == Kind::LossGrad && af->n == af->m && ci.g_smem && af->m <= 512 && !af->periodic && !cross) {
    pl.gpad_ok = true;
    pl.smem_gpad = sizeof(float2) * (size_t)ci.S * N;
  }
  if (kind != Kind::Backward && af->out_kind != GRAF_OUT_NONE) {
    const size_t row_bytes = (size_t)af->m * (af->out_kind == GRAF_OUT_C64 ? 8 : 4);
    // the copies move whole rows (raw) or half rows (centred) in 16-byte units
#ifndef GRAF_NO_BULK
    if ((af->doppler_layout == GRAF_DOPPLER_CENTERED ? row_bytes / 2 : row_bytes) % 16 == 0) {
#else
    if (false) {
#endif
      pl.bulk_ok = true;
      pl.stg_floats = (int)(2 * row_bytes / 4);
      pl.smem_stg = (size_t)ci.S * 2 * row_bytes + 16;
      pl.alias_ok = 2 * row_bytes <= sizeof(float2) * (size_t)ci.XS && ci.XS % 2 == 0;
    }
  }
  // Upper bound on CTAs per waveform (sizes the workspace); the launch picks the
  // actual P <= bound from the kernel's measured occupancy (choose_P).
  const long long B = af->batch;
  const long long maxP = std::max(1, (pl.U + ci.S - 1) / ci.S);
#ifndef GRAF_CAP_MULT
#define GRAF_CAP_MULT 8   // CTAs per SM (summed over the batch) that bound P; tuning builds override it
#endif
  const long long capP = std::max(1LL, (long long)(device_sm_count() * GRAF_CAP_MULT + B - 1) / B);
  pl.P = (int)std::max(1LL, std::min(maxP, capP));
  pl.Pbound = pl.P;
  size_t off = 0;
  pl.off_part = off;
  off = align256(off + sizeof(double) * kPart * (size_t)B * pl.Pbound);
  pl.off_gpart = off;
  if (grad) off = align256(off + (cross ? 2 : 1) * sizeof(float2) * (size_t)B * pl.Pbound * N);
  pl.off_comb = off;
  off = align256(off + 2 * sizeof(graf_partials) * (size_t)B);   // combined partials (+ fallback set)
  pl.off_spad = off;
  // pad_s_kernel rows (NL + M + 2 each, NL = N rounded up to even), twice (the second copy
  // shifted by one sample), each + tail slack: the adjoint's negative-delay rows read (and
  // mask) up to N samples past a row's end
  if (!ci.s_smem) off = align256(off + 2 * sizeof(float2) * spad_elems(B, N, af->m));
  if (kind == Kind::LossGrad && sc > 1 && !cross) {
    pl.off_sp_rec = off;
    off = align256(off + sizeof(double) * kPart * (size_t)B);
    pl.off_sp_g = off;
    off = align256(off + sizeof(float2) * (size_t)B * N);
  }
  // band cache: a two-pass loss (soft or hard PSL) on a narrow Doppler band keeps pass 1's
  // in-band FFT outputs (nband complex per loss row) so pass 2 skips the lag product and
  // the forward FFT; only when the band is at most M/4 bins and the cache at most 1 GiB
  if (kind == Kind::LossGrad && L && (L->lambda_psl != 0.f || L->lambda_hpsl != 0.f) &&
      af->out_kind == GRAF_OUT_NONE && !cross && pl.U > 0) {
    const int dm = std::min(L->d_max, af->m / 2);
    const int nband = 2 * dm + 1;
    const size_t bytes = sizeof(float2) * (size_t)B * pl.U * nband;
    if (nband <= af->m / 4 && bytes <= (size_t(1) << 30)) {
      pl.cache_ok = true;
      pl.nband = nband;
      pl.off_cache = off;
      off = align256(off + bytes);
    }
  }
  pl.total = off;
  return pl;
}


cudaError_t launch_rows(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
#ifdef GRAF_ONLY_M  // tuning builds (scripts/tune.py) link a single size
  if (pl.M == GRAF_ONLY_M) return launch_rows_size<GRAF_ONLY_M>(pl, rp, B, st, kind);
  return cudaErrorNotSupported;
#else
  switch (pl.M) {
    case 2: return launch_rows_size<2>(pl, rp, B, st, kind);
    case 4: return launch_rows_size<4>(pl, rp, B, st, kind);
    case 8: return launch_rows_size<8>(pl, rp, B, st, kind);
    case 16: return launch_rows_size<16>(pl, rp, B, st, kind);
    case 32: return launch_rows_size<32>(pl, rp, B, st, kind);
    case 64: return launch_rows_size<64>(pl, rp, B, st, kind);
    case 128: return launch_rows_size<128>(pl, rp, B, st, kind);
    case 256: return launch_rows_size<256>(pl, rp, B, st, kind);
    case 512: return launch_rows_size<512>(pl, rp, B, st, kind);
    case 1024: return launch_rows_size<1024>(pl, rp, B, st, kind);
    case 2048: return launch_rows_size<2048>(pl, rp, B, st, kind);
    case 4096: return launch_rows_size<4096>(pl, rp, B, st, kind);
    case 8192: return launch_rows_size<8192>(pl, rp, B, st, kind);
    case 16384: return launch_rows_size<16384>(pl, rp, B, st, kind);
    default: return cudaErrorInvalidValue;
  }
#endif
}

void fill_loss(RowParams& rp, const graf_af_desc* af, const graf_loss_desc* L) {
  const int N = af->n, M = af->m;
  rp.loss_on = 1;
  rp.kloss = std::min(L->k_max, af->periodic ? N / 2 : N - 1);
  rp.d_max = L->d_max;
  rp.ml_k = L->ml_k;
  rp.ml_d = L->ml_d;
  rp.w_k = L->w_k;
  rp.w_d = L->w_d;
  rp.lam_isl = L->lambda_isl;
  rp.lam_psl = L->lambda_psl;
  rp.T = L->lambda_psl != 0.f ? L->temperature : 1.f;
  rp.invT = 1.f / rp.T;
  rp.normalize = L->normalize;
  // reading R13: constant-sum region -> centred soft-PSL weights
  const bool full = rp.kloss == (af->periodic ? N / 2 : N - 1) && L->d_max >= M / 2 && L->ml_k == 0 && L->ml_d == 0;
  rp.centred = (L->normalize && !L->w_k && !L->w_d && full && L->lambda_psl != 0.f) ? 1 : 0;
  rp.const_sum = (L->normalize && !L->w_k && !L->w_d && full && af->m >= af->n) ? 1 : 0;
  // whole delay / Doppler extent with a mainlobe block cut out: the complement form of the
  // ISL gradient (kernels: f' = -lambda_isl on the block only)
  const bool full_extent = rp.kloss == (af->periodic ? N / 2 : N - 1) && L->d_max >= M / 2;
  rp.complement = (L->normalize && !L->w_k && !L->w_d && full_extent && af->m >= af->n && !rp.const_sum &&
                   L->lambda_match == 0.f) ? 1 : 0;
  rp.omega = (double)(af->periodic ? N : 2 * N - 1) * M - 1.0;   // |Omega| of the full plane
  rp.want_argmax = L->lambda_hpsl != 0.f ? 1 : 0;
  rp.lam_match = L->lambda_match;
  rp.target = L->target;
  rp.target_stride = L->target_stride;
  rp.key_lo = (af->periodic && 2 * rp.kloss == N) ? -rp.kloss + 1 : -rp.kloss;
  rp.xbar = (float)((M - 1) / rp.omega);
}

RowParams base_params(const graf_af_desc* af, const void* s, const Plan& pl, void* ws, const CallCtx& cx) {
  RowParams rp;
  std::memset(&rp, 0, sizeof(rp));
  rp.s = static_cast<const float2*>(s);
  rp.N = af->n;
  rp.B = (int)af->batch;
  rp.U = pl.U;
  rp.row_lo = pl.row_lo;
  rp.row_step = pl.row_step;
  rp.kb = af->k_begin;
  rp.ke = af->k_end;
  rp.out_kind = af->out_kind;
  rp.layout = af->doppler_layout;
  rp.norm_out = af->normalize_output;
  rp.shard_index = af->shard_index;
  rp.shard_count = af->shard_count <= 0 ? 1 : af->shard_count;
  rp.periodic = af->periodic;
  rp.T = 1.f;
  rp.invT = 1.f;
  char* w = static_cast<char*>(ws);
  rp.part = reinterpret_cast<double*>(w + pl.off_part);
  rp.gpart = reinterpret_cast<float2*>(w + pl.off_gpart);
  if (pl.cross) {
    rp.s2 = static_cast<const float2*>(cx.s2);
    rp.gpart2 = rp.gpart + (size_t)af->batch * pl.Pbound * af->n;
  }
  rp.skip = af->skip;
  rp.s_pad = pl.s_smem ? nullptr : reinterpret_cast<const float2*>(w + pl.off_spad);
  rp.s_pad1 = pl.s_smem ? nullptr : rp.s_pad + spad_elems(af->batch, af->n, af->m);
  return rp;
}

// global zero-padded s for the sizes whose s does not fit in shared memory
cudaError_t prepare_spad(const Plan& pl, const graf_af_desc* af, const void* s, void* ws, cudaStream_t st) {
  if (pl.s_smem) return cudaSuccess;
  float2* sp = reinterpret_cast<float2*>(static_cast<char*>(ws) + pl.off_spad);
  float2* sp1 = sp + spad_elems(af->batch, af->n, af->m);
  const long long total = af->batch * (long long)(af->n + af->m);
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  pad_s_kernel<<<blocks, 256, 0, st>>>(static_cast<const float2*>(s), sp, sp1, af->n, af->m, af->batch,
                                       af->periodic);
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++t_launches;
  return e;
}

graf_status common_checks(const graf_af_desc* af, const graf_loss_desc* L, const void* s, void* surface,
                          bool need_surface_window) {
  graf_status st = check_af(af);
  if (st) return st;
  if (af->batch > (1LL << 31) - 1) return fail(GRAF_EUNSUPPORTED, "batch too large");
  if (!s) return fail(GRAF_EINVAL, "s is NULL");
  if (!aligned8(s)) return fail(GRAF_EINVAL, "s is not 8-byte aligned");
  if (af->out_kind != GRAF_OUT_NONE || need_surface_window) {
    st = check_window(af);
    if (st) return st;
  }
  if (af->out_kind != GRAF_OUT_NONE) {
    if (!surface) return fail(GRAF_EINVAL, "out_kind set but surface is NULL");
    if (!aligned8(surface)) return fail(GRAF_EINVAL, "surface is not 8-byte aligned");
  }
  if (L) {
    st = check_loss(af, L);
    if (st) return st;
  }
  return GRAF_OK;
}

graf_status check_ws(const Plan& pl, void* ws, size_t ws_bytes) {
  if (ws_bytes < pl.total) return fail(GRAF_EWORKSPACE, "workspace %zu < %zu bytes", ws_bytes, pl.total);
  if (pl.total && !ws) return fail(GRAF_EINVAL, "workspace is NULL");
  if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return fail(GRAF_EINVAL, "workspace not 256-byte aligned");
  return GRAF_OK;
}

graf_status run_finalize(const graf_af_desc* af, const graf_loss_desc* L, const Plan& pl, const void* s,
                         void* ws, const graf_partials* global, double* loss, void* grad, bool norm_term,
                         cudaStream_t st, const graf_partials* one = nullptr, const RowParams* rpo = nullptr,
                         const CallCtx& cx = CallCtx{}, int sp = 0) {
  FinalizeParams f;
  std::memset(&f, 0, sizeof(f));
  char* w = static_cast<char*>(ws);
  f.s = static_cast<const float2*>(s);
  f.part = reinterpret_cast<const double*>(w + pl.off_part);
  f.gpart = reinterpret_cast<const float2*>(w + pl.off_gpart);
  f.global = global;
  f.P = pl.P;
  f.N = af->n;
  f.B = (int)af->batch;
  f.normalize = L ? L->normalize : 0;
  f.grad_norm_term = norm_term ? 1 : 0;
  f.lam_isl = L ? L->lambda_isl : 0.f;
  f.lam_psl = L ? L->lambda_psl : 0.f;
  f.T = (L && L->lambda_psl != 0.f) ? L->temperature : 1.f;
  f.invT = 1.f / f.T;
  f.lam_match = L ? L->lambda_match : 0.f;
  f.one = one;
  f.sp = sp;
  if (rpo) {
    f.omega = rpo->omega;
    f.xbar = rpo->xbar;
  }
  f.loss = loss;
  f.grad = static_cast<float2*>(grad);
  f.skip = af->skip;
  if (pl.cross) {
    f.s2 = static_cast<const float2*>(cx.s2);
    f.gpart2 = f.gpart + (size_t)af->batch * pl.Pbound * af->n;
    f.grad2 = static_cast<float2*>(cx.grad2);
  }
  const long long B = af->batch;
  for (long long b0 = 0; b0 < B; b0 += 65535) {
    FinalizeParams fc = f;
    const long long nb = std::min<long long>(65535, B - b0);
    fc.s = f.s + b0 * af->n;
    fc.part = f.part + b0 * pl.P * kPart;
    fc.gpart = f.gpart + b0 * pl.P * (long long)af->n;
    fc.global = global ? global + b0 : nullptr;
    fc.one = one ? one + b0 : nullptr;
    fc.loss = loss ? loss + b0 : nullptr;
    fc.grad = grad ? f.grad + b0 * af->n : nullptr;
    fc.skip = f.skip ? f.skip + b0 : nullptr;
    if (f.s2) {
      fc.s2 = f.s2 + b0 * af->n;
      fc.gpart2 = f.gpart2 + b0 * pl.P * (long long)af->n;
      fc.grad2 = f.grad2 ? f.grad2 + b0 * af->n : nullptr;
    }
    fc.B = (int)nb;
    finalize_kernel<<<dim3((unsigned)nb, (unsigned)((af->n + kFinChunk - 1) / kFinChunk)), 256, 0, st>>>(fc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "finalize_kernel launch");
    ++t_launches;
  }
  return GRAF_OK;
}

graf_status run_partials_reduce(const graf_af_desc* af, const graf_loss_desc* L, const Plan& pl, void* ws,
                                graf_partials* out, cudaStream_t st, int onepass = 0, float xbar = 0.f) {
  ReduceParams r;
  r.part = reinterpret_cast<const double*>(static_cast<char*>(ws) + pl.off_part);
  r.P = pl.P;
  r.B = (int)af->batch;
  r.T = L->lambda_psl != 0.f ? L->temperature : 1.f;
  r.invT = 1.f / r.T;
  r.out = out;
  r.onepass = onepass;
  r.xbar = xbar;
  r.skip = af->skip;
  partials_reduce_kernel<<<(r.B + 3) / 4, 128, 0, st>>>(r);   // a warp per waveform
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++t_launches;
  return e == cudaSuccess ? GRAF_OK : cuda_fail(e, "partials_reduce_kernel launch");
}

graf_status check_cross(const graf_af_desc* af, const graf_loss_desc* L, const void* s2) {
  if (!s2 || !aligned8(s2)) return fail(GRAF_EINVAL, "s2 is NULL or not 8-byte aligned");
  if (af->periodic) return fail(GRAF_EUNSUPPORTED, "cross-ambiguity is aperiodic in v1");
  if (af->shard_count > 1) return fail(GRAF_EUNSUPPORTED, "cross-ambiguity is unsharded in v1");
  if (af->skip) return fail(GRAF_EUNSUPPORTED, "cross-ambiguity: af->skip is not supported");
  if (af->m > 4096) return fail(GRAF_EUNSUPPORTED, "cross-ambiguity needs M <= 4096 in v1");
  if (L && (L->lambda_hpsl != 0.f || L->lambda_match != 0.f || L->w_k || L->w_d))
    return fail(GRAF_EUNSUPPORTED, "cross-ambiguity losses: unweighted ISL and soft-PSL in v1");
  return GRAF_OK;
}

// hard PSL term (loss and argmax subgradient) from the combined partials
graf_status run_psl(const graf_af_desc* af, const graf_loss_desc* L, const Plan& pl, const void* s,
                    const graf_partials* stats, double* loss_out, void* grad, int accumulate, cudaStream_t st) {
  (void)pl;
  PslParams q;
  std::memset(&q, 0, sizeof(q));
  const int N = af->n;
  const int kl = std::min(L->k_max, af->periodic ? N / 2 : N - 1);
  q.s = static_cast<const float2*>(s);
  q.stats = stats;
  q.N = N;
  q.M = af->m;
  q.key_lo = (af->periodic && 2 * kl == N) ? -kl + 1 : -kl;
  q.periodic = af->periodic;
  q.normalize = L->normalize;
  q.lam = L->lambda_hpsl;
  q.add_grad = (af->shard_index == 0) ? 1 : 0;
  q.accumulate = accumulate;
  q.loss = loss_out;
  q.grad = static_cast<float2*>(grad);
  q.skip = af->skip;
  psl_grad_kernel<<<(unsigned)af->batch, 256, 0, st>>>(q);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "psl_grad_kernel launch");
  ++t_launches;
  return GRAF_OK;
}

}  // namespace
}  // namespace graf

using namespace graf;

extern "C" {

int32_t graf_abi_version(void) { return GRAF_ABI_VERSION; }

graf_status graf_init(void* stream) {
  t_launches = 0;
  const cudaError_t e = ensure_twiddles(static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GRAF_OK : cuda_fail(e, "twiddle table init");
}

const char* graf_status_string(graf_status s) {
  switch (s) {
    case GRAF_OK: return "GRAF_OK";
    case GRAF_EINVAL: return "GRAF_EINVAL: invalid argument";
    case GRAF_EUNSUPPORTED: return "GRAF_EUNSUPPORTED: outside v1 device limits";
    case GRAF_ECUDA: return "GRAF_ECUDA: CUDA error";
    case GRAF_EWORKSPACE: return "GRAF_EWORKSPACE: workspace too small";
    default: return "GRAF_UNKNOWN";
  }
}

const char* graf_last_error(void) { return t_last_error.c_str(); }

int32_t graf_last_launch_count(void) { return t_launches; }

int32_t graf_plan_ctas_per_waveform(int32_t rows, int32_t slots, int64_t batch, int32_t occ, int32_t nsm,
                                    int32_t p_bound) {
  if (rows <= 0 || slots <= 0 || batch <= 0 || occ <= 0 || nsm <= 0 || p_bound <= 0) return 0;
  Plan pl;
  pl.U = rows;
  pl.S = slots;
  pl.Pbound = p_bound;
  return choose_P(pl, batch, occ, nsm);
}

static size_t impl_workspace_bytes(const graf_af_desc* af, const graf_loss_desc* loss, bool cross) {
  if (check_af(af) != GRAF_OK) return 0;
  if (loss && check_loss(af, loss) != GRAF_OK) return 0;
  size_t need = make_plan(af, loss, Kind::LossGrad, cross).total;
  if (af->k_begin >= -(af->n - 1) && af->k_end <= af->n && af->k_begin < af->k_end)
    need = std::max(need, make_plan(af, nullptr, Kind::Backward, cross).total);
  return need;
}

static graf_status impl_forward(const CallCtx& cx, const graf_af_desc* af, const graf_loss_desc* loss, const void* s, void* surface,
                            graf_partials* partials, void* ws, size_t ws_bytes, void* stream) {
  t_launches = 0;
  graf_status st = common_checks(af, loss, s, surface, false);
  if (st) return st;
  if (loss && !partials) return fail(GRAF_EINVAL, "loss given but partials is NULL");
  Plan pl = make_plan(af, loss, Kind::Forward, cx.cross());
  if ((st = check_ws(pl, ws, ws_bytes))) return st;
  if (reinterpret_cast<uintptr_t>(surface) & 15u) pl.bulk_ok = false;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaError_t e = ensure_twiddles(cs);
  if (e != cudaSuccess) return cuda_fail(e, "twiddle table init");
  if (pl.U > 0 && (e = prepare_spad(pl, af, s, ws, cs)) != cudaSuccess) return cuda_fail(e, "pad_s_kernel");
  RowParams rp = base_params(af, s, pl, ws, cx);
  rp.surface = af->out_kind != GRAF_OUT_NONE ? surface : nullptr;
  if (loss) fill_loss(rp, af, loss);
  if (pl.U > 0) {
    prof_mark(true, cs);
    e = launch_rows(pl, rp, (int)af->batch, cs, K_FWD);
    if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (forward) launch");
    prof_mark(false, cs);
  }
  if (loss) {
    if (pl.U == 0) {
      Plan p0 = pl;  // this shard owns no rows: identity partials (P = 0 records)
      p0.P = 0;
      return run_partials_reduce(af, loss, p0, ws, partials, cs);
    }
    return run_partials_reduce(af, loss, pl, ws, partials, cs);
  }
  return GRAF_OK;
}

static graf_status impl_loss_grad(const CallCtx& cx, const graf_af_desc* af, const graf_loss_desc* loss, const void* s,
                              const graf_partials* global, double* loss_out, void* grad, void* surface, void* ws,
                              size_t ws_bytes, void* stream) {
  t_launches = 0;
  graf_status st = common_checks(af, loss, s, surface, false);
  if (st) return st;
  if (!loss) return fail(GRAF_EINVAL, "loss descriptor is NULL");
  if (!grad) return fail(GRAF_EINVAL, "grad is NULL");
  if (!aligned8(grad)) return fail(GRAF_EINVAL, "grad is not 8-byte aligned");
  Plan pl = make_plan(af, loss, Kind::LossGrad, cx.cross());
  if ((st = check_ws(pl, ws, ws_bytes))) return st;
  if (reinterpret_cast<uintptr_t>(surface) & 15u) pl.bulk_ok = false;
  const bool needs_global = loss->lambda_psl != 0.f || loss->lambda_hpsl != 0.f;
  if (pl.U == 0 && !global && needs_global)
    return fail(GRAF_EINVAL, "a shard with no loss rows needs `global` for soft-PSL / hard-PSL losses");
  if (loss->lambda_match != 0.f && global)
    return fail(GRAF_EUNSUPPORTED, "match loss with global partials (v1: unsharded)");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaError_t e = ensure_twiddles(cs);
  if (e != cudaSuccess) return cuda_fail(e, "twiddle table init");
  if (pl.U == 0) {
    // no rows here: grad 0; a loss that is a sum over rows (ISL, match) is 0 too, else it
    // comes from the global partials below (finalize with no partial records)
    const bool zero_loss = loss_out && !global;
    const long long tot = af->batch * (long long)af->n;
    zero_outputs_kernel<<<(unsigned)std::min<long long>((tot + 255) / 256, 148 * 8), 256, 0, cs>>>(
        static_cast<float2*>(grad), zero_loss ? loss_out : nullptr, af->batch, af->n, af->skip);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "zero_outputs_kernel launch");
    ++t_launches;
  }
  if (pl.U > 0 && (e = prepare_spad(pl, af, s, ws, cs)) != cudaSuccess) return cuda_fail(e, "pad_s_kernel");
  RowParams rp = base_params(af, s, pl, ws, cx);
  fill_loss(rp, af, loss);
  rp.surface = af->out_kind != GRAF_OUT_NONE ? surface : nullptr;
  graf_partials* comb = reinterpret_cast<graf_partials*>(static_cast<char*>(ws) + pl.off_comb);
  const graf_partials* stats = global;
  const bool hpsl = loss->lambda_hpsl != 0.f;       // hard PSL (section-7 loss), reading R23
  const bool soft = loss->lambda_psl != 0.f;
  const bool match = loss->lambda_match != 0.f;    // match loss, reading R24
  const bool dense = loss->lambda_isl != 0.f || soft || match;   // terms with a per-cell f'
  if (match && !hpsl) {
    // one pass: f' = lambda_isl w + lambda_match (2x - t1 - t2) is known per cell
    if (pl.U > 0) {
      prof_mark(true, cs);
      e = launch_rows(pl, rp, (int)af->batch, cs, K_MATCH);
      if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (match) launch");
      prof_mark(false, cs);
    }
  } else if (!soft && !hpsl) {
    // single fused pass (f' = lambda_isl * w known up front); unsharded calls also
    // fuse the finalize into the row kernel when a waveform's CTAs fit one cluster
    pl.fuse_req = (global == nullptr);
    rp.loss_out = loss_out;
    rp.grad_out = static_cast<float2*>(grad);
    if (pl.U > 0) {
      prof_mark(true, cs);
      e = launch_rows(pl, rp, (int)af->batch, cs, K_ISL);
      if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (isl) launch");
      prof_mark(false, cs);
    }
  } else {
    if (pl.U > 0) prof_mark(true, cs);
    const bool use_cache = pl.cache_ok && !stats && dense && !match;
    if (use_cache) {
      rp.acache = reinterpret_cast<float2*>(static_cast<char*>(ws) + pl.off_cache);
      rp.nband = pl.nband;
    }
    // full-plane centred soft-PSL (reading R13): one optimistic pass with f' = lambda
    // expm1((x - xbar)/T), then guarded fallback passes that only run the waveforms whose
    // single pass is outside the R13 validity rule (max x - xbar > 40 T)
#ifdef GRAF_NO_ONEPASS   // A/B builds only
    constexpr bool kOnePass = false;
#else
    constexpr bool kOnePass = true;
#endif
    const bool onepass = kOnePass && !stats && rp.centred && !hpsl && !match && !use_cache &&
                         rp.surface == nullptr && rp.shard_count <= 1 && pl.U > 0;
    if (onepass) {
      graf_partials* comb2 = comb + af->batch;
      RowParams r0 = rp;
      r0.onepass = 1;
      e = launch_rows(pl, r0, (int)af->batch, cs, K_PASS2);
      if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (single pass) launch");
      if ((st = run_partials_reduce(af, loss, pl, ws, comb, cs, 1, rp.xbar))) return st;
      RowParams r1 = rp;
      r1.guard = comb;
      e = launch_rows(pl, r1, (int)af->batch, cs, K_FWD);
      if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (fallback pass 1) launch");
      if ((st = run_partials_reduce(af, loss, pl, ws, comb2, cs))) return st;
      RowParams r2 = rp;
      r2.guard = comb;
      r2.stats = comb2;
      e = launch_rows(pl, r2, (int)af->batch, cs, K_PASS2);
      if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (fallback pass 2) launch");
      prof_mark(false, cs);
      return run_finalize(af, loss, pl, s, ws, comb2, loss_out, grad, true, cs, comb, &rp, cx);
    }
    if (!stats) {
      RowParams r1 = rp;
      r1.surface = nullptr;
      r1.cache = use_cache ? 1 : 0;
      e = launch_rows(pl, r1, (int)af->batch, cs, K_FWD);
      if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (pass 1) launch");
      if ((st = run_partials_reduce(af, loss, pl, ws, comb, cs))) return st;
      stats = comb;
    }
    rp.stats = stats;
    rp.cache = use_cache ? 2 : 0;
    if (pl.U > 0 && dense) {
      e = launch_rows(pl, rp, (int)af->batch, cs, match ? K_MATCH : K_PASS2);
      if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (pass 2) launch");
    }
    if (pl.U > 0) prof_mark(false, cs);
  }
  if (pl.U == 0) {
    if (loss_out && dense) {
      // no rows here: loss purely from the global partials
      Plan p0 = pl;
      p0.P = 0;
      if ((st = run_finalize(af, loss, p0, s, ws, global, loss_out, nullptr, false, cs))) return st;
    }
    if (hpsl) return run_psl(af, loss, pl, s, stats, loss_out, grad, dense ? 1 : 0, cs);
    return GRAF_OK;
  }
  if (!pl.fused && dense) {
    if ((st = run_finalize(af, loss, pl, s, ws, stats, loss_out, grad, true, cs, nullptr, nullptr, cx))) return st;
  }
  if (hpsl) return run_psl(af, loss, pl, s, stats, loss_out, grad, dense ? 1 : 0, cs);
  return GRAF_OK;
}

// ---------------------------------------------------------------------------
// Delay-sharded single pass of the full-plane centred soft-PSL (reading R13, R27).
// Phase 1 runs this shard's rows once (f' = lambda expm1((x - xbar)/T)) and returns its
// partials; the caller combines the shards' partials in rank order; phase 2 applies the
// GLOBAL R13 rule and scales this shard's gradient by the global 1/Z_c.
// ---------------------------------------------------------------------------
static bool sp_eligible(const graf_af_desc* af, const graf_loss_desc* L) {
  if (!af || !L || check_af(af) != GRAF_OK || check_loss(af, L) != GRAF_OK) return false;
  if (af->out_kind != GRAF_OUT_NONE || L->lambda_hpsl != 0.f || L->lambda_match != 0.f) return false;
  RowParams rp;
  std::memset(&rp, 0, sizeof(rp));
  fill_loss(rp, af, L);
  return rp.centred != 0;
}

static graf_status sp_common(const graf_af_desc* af, const graf_loss_desc* L, const void* s, void* ws,
                             size_t ws_bytes, Plan* pl) {
  graf_status st = common_checks(af, L, s, nullptr, false);
  if (st) return st;
  if (!L) return fail(GRAF_EINVAL, "loss descriptor is NULL");
  if ((af->shard_count <= 0 ? 1 : af->shard_count) < 2)
    return fail(GRAF_EINVAL, "the sharded single pass needs shard_count >= 2 (unsharded calls use graf_af_loss_grad)");
  if (!sp_eligible(af, L))
    return fail(GRAF_EUNSUPPORTED, "sharded single pass: only the full-plane, normalised, unweighted soft-PSL "
                                   "(graf_af_single_pass_eligible)");
  if (af->skip) return fail(GRAF_EUNSUPPORTED, "sharded single pass: af->skip is not supported");
  *pl = make_plan(af, L, Kind::LossGrad, false);
  return check_ws(*pl, ws, ws_bytes);
}

static graf_status impl_sp_begin(const graf_af_desc* af, const graf_loss_desc* L, const void* s,
                                 graf_partials* partials, void* ws, size_t ws_bytes, void* stream) {
  t_launches = 0;
  Plan pl;
  graf_status st = sp_common(af, L, s, ws, ws_bytes, &pl);
  if (st) return st;
  if (!partials || (reinterpret_cast<uintptr_t>(partials) & 7u)) return fail(GRAF_EINVAL, "partials is NULL or misaligned");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaError_t e = ensure_twiddles(cs);
  if (e != cudaSuccess) return cuda_fail(e, "twiddle table init");
  RowParams rp = base_params(af, s, pl, ws, CallCtx{});
  fill_loss(rp, af, L);
  Plan p0 = pl;
  if (pl.U > 0) {
    if ((e = prepare_spad(pl, af, s, ws, cs)) != cudaSuccess) return cuda_fail(e, "pad_s_kernel");
    RowParams r0 = rp;
    r0.onepass = 1;
    prof_mark(true, cs);
    e = launch_rows(pl, r0, (int)af->batch, cs, K_PASS2);
    if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (sharded single pass) launch");
    prof_mark(false, cs);
    p0 = pl;
  } else {
    p0.P = 0;   // this shard owns no rows: identity partials, zero gradient
  }
  if ((st = run_partials_reduce(af, L, p0, ws, partials, cs, 1, rp.xbar))) return st;
  char* w = static_cast<char*>(ws);
  SpFoldParams f;
  f.part = reinterpret_cast<const double*>(w + pl.off_part);
  f.gpart = reinterpret_cast<const float2*>(w + pl.off_gpart);
  f.rec1 = reinterpret_cast<double*>(w + pl.off_sp_rec);
  f.gsum = reinterpret_cast<float2*>(w + pl.off_sp_g);
  f.P = p0.P;
  f.N = af->n;
  f.T = rp.T;
  for (long long b0 = 0; b0 < af->batch; b0 += 65535) {
    SpFoldParams fc = f;
    const long long nb = std::min<long long>(65535, af->batch - b0);
    fc.part = f.part + b0 * f.P * kPart;
    fc.gpart = f.gpart + b0 * f.P * (long long)af->n;
    fc.rec1 = f.rec1 + b0 * kPart;
    fc.gsum = f.gsum + b0 * af->n;
    sp_fold_kernel<<<dim3((unsigned)nb, (unsigned)((af->n + 255) / 256)), 256, 0, cs>>>(fc);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "sp_fold_kernel launch");
    ++t_launches;
  }
  return GRAF_OK;
}

static graf_status impl_sp_end(const graf_af_desc* af, const graf_loss_desc* L, const void* s,
                               const graf_partials* global, double* loss_out, void* grad, int32_t* valid, void* ws,
                               size_t ws_bytes, void* stream) {
  t_launches = 0;
  Plan pl;
  graf_status st = sp_common(af, L, s, ws, ws_bytes, &pl);
  if (st) return st;
  if (!global) return fail(GRAF_EINVAL, "global partials are NULL");
  if (!grad || !aligned8(grad)) return fail(GRAF_EINVAL, "grad is NULL or not 8-byte aligned");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  RowParams rp;
  std::memset(&rp, 0, sizeof(rp));
  fill_loss(rp, af, L);
  char* w = static_cast<char*>(ws);
  graf_partials* comb = reinterpret_cast<graf_partials*>(w + pl.off_comb);
  SpValidateParams v;
  v.global = global;
  v.out = comb;
  v.valid = valid;
  v.B = (int)af->batch;
  v.xbar = rp.xbar;
  v.invT = rp.invT;
  sp_validate_kernel<<<(unsigned)((af->batch + 127) / 128), 128, 0, cs>>>(v);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sp_validate_kernel launch");
  ++t_launches;
  // the folded records / gradients of phase 1 play the role of P = 1 CTA partials
  Plan p1 = pl;
  p1.P = 1;
  p1.Pbound = 1;
  p1.off_part = pl.off_sp_rec;
  p1.off_gpart = pl.off_sp_g;
  return run_finalize(af, L, p1, s, ws, global, loss_out, grad, true, cs, comb, &rp, CallCtx{}, 1);
}

static graf_status impl_backward(const CallCtx& cx, const graf_af_desc* af, const void* s, const void* dA, void* grad, void* ws,
                             size_t ws_bytes, void* stream) {
  t_launches = 0;
  graf_status st = common_checks(af, nullptr, s, nullptr, true);
  if (st) return st;
  if (!dA || !aligned8(dA)) return fail(GRAF_EINVAL, "dA is NULL or not 8-byte aligned");
  if (!grad || !aligned8(grad)) return fail(GRAF_EINVAL, "grad is NULL or not 8-byte aligned");
  Plan pl = make_plan(af, nullptr, Kind::Backward, cx.cross());
  if ((st = check_ws(pl, ws, ws_bytes))) return st;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaError_t e = ensure_twiddles(cs);
  if (e != cudaSuccess) return cuda_fail(e, "twiddle table init");
  if ((e = prepare_spad(pl, af, s, ws, cs)) != cudaSuccess) return cuda_fail(e, "pad_s_kernel");
  RowParams rp = base_params(af, s, pl, ws, cx);
  rp.dA = static_cast<const float2*>(dA);
  prof_mark(true, cs);
  e = launch_rows(pl, rp, (int)af->batch, cs, K_ADJ);
  if (e != cudaSuccess) return cuda_fail(e, "af_rows_kernel (adjoint) launch");
  prof_mark(false, cs);
  return run_finalize(af, nullptr, pl, s, ws, nullptr, nullptr, grad, false, cs, nullptr, nullptr, cx);
}

size_t graf_workspace_bytes(const graf_af_desc* af, const graf_loss_desc* loss) {
  return impl_workspace_bytes(af, loss, false);
}

graf_status graf_af_forward(const graf_af_desc* af, const graf_loss_desc* loss, const void* s, void* surface,
                            graf_partials* partials, void* ws, size_t ws_bytes, void* stream) {
  return impl_forward(CallCtx{}, af, loss, s, surface, partials, ws, ws_bytes, stream);
}

graf_status graf_af_loss_grad(const graf_af_desc* af, const graf_loss_desc* loss, const void* s,
                              const graf_partials* global, double* loss_out, void* grad, void* surface, void* ws,
                              size_t ws_bytes, void* stream) {
  return impl_loss_grad(CallCtx{}, af, loss, s, global, loss_out, grad, surface, ws, ws_bytes, stream);
}

int32_t graf_af_single_pass_eligible(const graf_af_desc* af, const graf_loss_desc* loss) {
  return sp_eligible(af, loss) ? 1 : 0;
}

graf_status graf_af_loss_grad_sp_begin(const graf_af_desc* af, const graf_loss_desc* loss, const void* s,
                                       graf_partials* partials, void* ws, size_t ws_bytes, void* stream) {
  return impl_sp_begin(af, loss, s, partials, ws, ws_bytes, stream);
}

graf_status graf_af_loss_grad_sp_end(const graf_af_desc* af, const graf_loss_desc* loss, const void* s,
                                     const graf_partials* global, double* loss_out, void* grad, int32_t* valid,
                                     void* ws, size_t ws_bytes, void* stream) {
  return impl_sp_end(af, loss, s, global, loss_out, grad, valid, ws, ws_bytes, stream);
}

graf_status graf_af_backward(const graf_af_desc* af, const void* s, const void* dA, void* grad, void* ws,
                             size_t ws_bytes, void* stream) {
  return impl_backward(CallCtx{}, af, s, dA, grad, ws, ws_bytes, stream);
}

size_t graf_xaf_workspace_bytes(const graf_af_desc* af, const graf_loss_desc* loss) {
  return impl_workspace_bytes(af, loss, true);
}

graf_status graf_xaf_forward(const graf_af_desc* af, const graf_loss_desc* loss, const void* s1, const void* s2,
                             void* surface, graf_partials* partials, void* ws, size_t ws_bytes, void* stream) {
  t_launches = 0;
  if (!af) return fail(GRAF_EINVAL, "af descriptor is NULL");
  graf_status st = check_cross(af, loss, s2);
  if (st) return st;
  CallCtx cx;
  cx.s2 = s2;
  return impl_forward(cx, af, loss, s1, surface, partials, ws, ws_bytes, stream);
}

graf_status graf_xaf_loss_grad(const graf_af_desc* af, const graf_loss_desc* loss, const void* s1, const void* s2,
                               const graf_partials* global, double* loss_out, void* grad1, void* grad2,
                               void* surface, void* ws, size_t ws_bytes, void* stream) {
  t_launches = 0;
  if (!af) return fail(GRAF_EINVAL, "af descriptor is NULL");
  graf_status st = check_cross(af, loss, s2);
  if (st) return st;
  if (!grad2 || !aligned8(grad2)) return fail(GRAF_EINVAL, "grad2 is NULL or not 8-byte aligned");
  CallCtx cx;
  cx.s2 = s2;
  cx.grad2 = grad2;
  return impl_loss_grad(cx, af, loss, s1, global, loss_out, grad1, surface, ws, ws_bytes, stream);
}

graf_status graf_xaf_backward(const graf_af_desc* af, const void* s1, const void* s2, const void* dA, void* grad1,
                              void* grad2, void* ws, size_t ws_bytes, void* stream) {
  t_launches = 0;
  if (!af) return fail(GRAF_EINVAL, "af descriptor is NULL");
  graf_status st = check_cross(af, nullptr, s2);
  if (st) return st;
  if (!grad2 || !aligned8(grad2)) return fail(GRAF_EINVAL, "grad2 is NULL or not 8-byte aligned");
  CallCtx cx;
  cx.s2 = s2;
  cx.grad2 = grad2;
  return impl_backward(cx, af, s1, dA, grad1, ws, ws_bytes, stream);
}

// FP32 peak probe (bench.py's measured ALU denominator): every thread runs 8 independent
// FFMA chains for `iters` iterations, 2 flops per FFMA; the chains' sum is written so
// nothing is optimised away.  Grid: 4 CTAs of 256 threads per SM.
__global__ void __launch_bounds__(256) fp32_probe_kernel(float* out, int iters, float b) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (float)(threadIdx.x + i) * 1e-3f;
  const float c = 0.5f * b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;   // (practically never)
}

graf_status graf_probe_fp32(float* scratch, int32_t iters, double* flops, void* stream) {
  t_launches = 0;
  if (!scratch || iters < 1 || !flops) return fail(GRAF_EINVAL, "scratch / flops NULL or iters < 1");
  const int blocks = device_sm_count() * 4;
  fp32_probe_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(scratch, iters, 0.999f);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "fp32_probe_kernel launch");
  ++t_launches;
  *flops = 2.0 * 8.0 * 16.0 * (double)iters * 256.0 * (double)blocks;
  return GRAF_OK;
}

graf_status graf_set_profile_events(void* start, void* stop) {
  if ((start == nullptr) != (stop == nullptr)) return fail(GRAF_EINVAL, "set both events or neither");
  t_prof_start = static_cast<cudaEvent_t>(start);
  t_prof_stop = static_cast<cudaEvent_t>(stop);
  return GRAF_OK;
}

graf_status graf_combine_partials(const graf_loss_desc* loss, const graf_partials* shards, int32_t G, int64_t B,
                                  graf_partials* out, int32_t on_device, void* stream) {
  t_launches = 0;
  if (!loss || !shards || !out) return fail(GRAF_EINVAL, "NULL argument");
  if (G < 1 || B < 1) return fail(GRAF_EINVAL, "G = %d, B = %lld", G, (long long)B);
  const float T = loss->lambda_psl != 0.f ? loss->temperature : 1.f;
  if (!(T > 0.f)) return fail(GRAF_EINVAL, "temperature must be > 0");
  if (on_device) {
    CombineParams c{shards, G, (int)B, T, out};
    combine_partials_kernel<<<(unsigned)((B + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(c);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) ++t_launches;
    return e == cudaSuccess ? GRAF_OK : cuda_fail(e, "combine_partials_kernel launch");
  }
  for (int64_t b = 0; b < B; ++b) {
    double S = 0, Z = 0, Cs = 0, key = (double)0x7fffffff;
    double m = -INFINITY;
    for (int q = 0; q < G; ++q) {
      const graf_partials& g = shards[(size_t)q * B + b];
      S += g.isl_sum;
      Cs += g.cen_sum;
      const double m2 = g.lse_max;
      const double Z2 = g.lse_sum;
      if (m2 > m || (m2 == m && g.psl_key < key)) key = g.psl_key;
      if (m2 == -INFINITY) continue;
      if (m == -INFINITY) {
        m = m2;
        Z = Z2;
      } else if (m2 > m) {
        Z = Z * std::exp((m - m2) / (double)T) + Z2;
        m = m2;
      } else {
        Z = Z + Z2 * std::exp((m2 - m) / (double)T);
      }
    }
    out[b] = graf_partials{S, m, Z, Cs, key, 0.0};
  }
  return GRAF_OK;
}

graf_status graf_spectral_variance(int64_t batch, int32_t n, const void* s, float weight,
                                   const float* weights, double* loss, void* grad, int32_t accumulate,
                                   int32_t ddof, void* stream) {
  t_launches = 0;
  if (batch < 1 || batch > (1LL << 31) - 1) return fail(GRAF_EINVAL, "batch = %lld", (long long)batch);
  if (!is_pow2(n) || n < 2) return fail(GRAF_EINVAL, "N = %d is not a power of two >= 2", n);
  if (n > GRAF_MAX_M) return fail(GRAF_EUNSUPPORTED, "N = %d > %d", n, GRAF_MAX_M);
  if (!s || !grad || !aligned8(s) || !aligned8(grad)) return fail(GRAF_EINVAL, "s / grad NULL or misaligned");
  if (!std::isfinite(weight)) return fail(GRAF_EINVAL, "non-finite weight");
  if (ddof != 0 && ddof != 1) return fail(GRAF_EINVAL, "ddof must be 0 or 1");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaError_t e = ensure_twiddles(cs);
  if (e != cudaSuccess) return cuda_fail(e, "twiddle table init");
  SvParams q{static_cast<const float2*>(s), n, weight, weights, accumulate ? 1 : 0, loss,
             static_cast<float2*>(grad), (int)ddof};
  if (n <= 32) {
    const int threads = 32;
    const size_t smem = sizeof(float2) * 2 * (size_t)n + sizeof(double) * threads;
    sv_direct_kernel<<<(unsigned)batch, threads, smem, cs>>>(q);
  } else {
    // Stockham FFT with T = N/E >= 32 threads (E = N/32 up to 16)
    auto go = [&](auto kern, int T, int XS) -> cudaError_t {
      const size_t smem = sizeof(float2) * (size_t)((XS + 1) & ~1) + sizeof(double) * T;
      cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (ea != cudaSuccess) return ea;
      kern<<<(unsigned)batch, T, smem, cs>>>(q);
      return cudaSuccess;
    };
#define GRAF_SV(M_, E_) go(sv_fft_kernel<M_, E_>, SvCfg<M_, E_>::T, SvCfg<M_, E_>::XS)
    switch (n) {
      case 64: e = GRAF_SV(64, 2); break;
      case 128: e = GRAF_SV(128, 4); break;
      case 256: e = GRAF_SV(256, 8); break;
      case 512: e = GRAF_SV(512, 16); break;
      case 1024: e = GRAF_SV(1024, 16); break;
      case 2048: e = GRAF_SV(2048, 16); break;
      case 4096: e = GRAF_SV(4096, 16); break;
      case 8192: e = GRAF_SV(8192, 16); break;
      default: e = GRAF_SV(16384, 16); break;
    }
#undef GRAF_SV
    if (e != cudaSuccess) return cuda_fail(e, "sv_fft_kernel attribute");
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "spectral variance kernel launch");
  ++t_launches;
  return GRAF_OK;
}

graf_status graf_mainlobe_width(int64_t batch, int32_t n, const void* s, float gamma, float weight,
                                int32_t periodic, double* loss, void* grad, int32_t accumulate, void* stream) {
  t_launches = 0;
  if (batch < 1 || batch > (1LL << 31) - 1 || n < 1) return fail(GRAF_EINVAL, "batch / N out of range");
  if (n > 8192) return fail(GRAF_EUNSUPPORTED, "mainlobe width: N = %d > 8192 (v1)", n);
  if (periodic && !is_pow2(n)) return fail(GRAF_EINVAL, "periodic mainlobe width needs N a power of two");
  if (!s || !grad || !aligned8(s) || !aligned8(grad)) return fail(GRAF_EINVAL, "s / grad NULL or misaligned");
  if (!std::isfinite(gamma) || !std::isfinite(weight)) return fail(GRAF_EINVAL, "non-finite gamma / weight");
  MlwParams q{static_cast<const float2*>(s), n, periodic ? 1 : 0, accumulate ? 1 : 0, gamma, weight, loss,
              static_cast<float2*>(grad)};
  const int K = periodic ? n / 2 : n - 1;
  int threads = 32;
  while (threads < 1024 && threads < n) threads *= 2;
  const size_t smem = sizeof(float2) * (size_t)(K + 1) + sizeof(float) * (size_t)((K + 2) & ~1) +
                      sizeof(double) * threads;
  cudaError_t e = cudaFuncSetAttribute(mainlobe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "mainlobe_kernel attribute");
  mainlobe_kernel<<<(unsigned)batch, threads, smem, static_cast<cudaStream_t>(stream)>>>(q);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "mainlobe_kernel launch");
  ++t_launches;
  return GRAF_OK;
}

graf_status graf_phase_adam_step(int64_t batch, int32_t n, float* theta, float* m, float* v, int32_t* step,
                                 const void* grad, void* s_out, float lr, float beta1, float beta2, float eps,
                                 void* stream) {
  t_launches = 0;
  if (batch < 1 || batch > (1LL << 31) - 1 || n < 1) return fail(GRAF_EINVAL, "batch / N out of range");
  if (!theta || !m || !v || !step || !grad || !s_out) return fail(GRAF_EINVAL, "NULL argument");
  if (!(lr > 0.f) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) || !(eps >= 0.f))
    return fail(GRAF_EINVAL, "Adam hyper-parameters out of range");
  AdamParams a{theta, m, v, step, static_cast<const float2*>(grad), static_cast<float2*>(s_out), n,
               lr, beta1, beta2, eps};
  phase_adam_kernel<<<(unsigned)batch, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "phase_adam_kernel launch");
  ++t_launches;
  return GRAF_OK;
}

}  // extern "C"
