// graf_launch.cuh — launch planning shared by the ABI translation unit
// (graf_api.cu) and the per-size row-kernel translation units (graf_rows_*.cu,
// compiled in parallel; each instantiates af_rows_kernel for its sizes).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cmath>
#include <mutex>
#include <vector>

#include "../../include/graf.h"
#include "graf_kernels.cuh"

namespace graf {

extern thread_local int t_launches;   // kernels / memsets enqueued by the current entry-point call
constexpr int kMaxDev = 64;

// SM count of the current device (cached per device; the workspace bound and the
// launch plan use the same value for the same device)
inline int device_sm_count() {
  static int cache[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

// ---------------------------------------------------------------------------
// launch plan
// ---------------------------------------------------------------------------
struct Plan {
  int M = 0, threads = 0, S = 0, T = 0, P = 1, Pbound = 1;
  int U = 0, row_lo = 0, row_step = 1;
  bool fixedP = false;
  bool s_smem = true, g_smem = true;
  size_t smem = 0;
  // surface staging for bulk async row stores: per-slot floats,
  // whether the rows qualify, and whether they fit the slot's exchange buffer (alias)
  int stg_floats = 0;
  bool bulk_ok = false, alias_ok = false;
  size_t smem_stg = 0;
  int bulk_mode = -1;   // decided at the first launch of a call: 0 direct, 1 dedicated, 2 alias
  // left-padded gradient accumulators (M == N loss calls), if they cost no resident CTA
  bool gpad_ok = false;
  size_t smem_gpad = 0;
  int gpad_mode = -1;
  // fused finalize (K_ISL only): requested by the caller, granted when P <= 8
  bool fuse_req = false, fused = false;
  bool cross = false;   // cross-ambiguity (two waveforms, unfolded rows)
  size_t off_part = 0, off_gpart = 0, off_comb = 0, off_spad = 0, total = 0;
  // band cache of two-pass losses (pass 1 stores the loss band, pass 2 reads it)
  size_t off_cache = 0;
  int nband = 0;
  bool cache_ok = false;
  // delay-sharded single pass (graf_af_loss_grad_sp_begin / _end): one folded record and
  // one unscaled gradient per waveform, kept in the workspace between the two phases
  size_t off_sp_rec = 0, off_sp_g = 0;
};


// Cost model: waves x (row iterations + CTA setup), setup ~ one row iteration.
// Candidates within 2 % of the best are then ranked by a second model in which the last,
// partial wave is cheaper than a full one: its CTAs share their SM with fewer neighbours
// (j of occ resident), and a throughput-bound CTA then runs in about (j / occ)^0.75 of the
// time.  Measured on c3's half batch (B = 512, scripts/p_variants.sh): the plain model
// ties P = 1 (514) with P = 2 (516) and took P = 1 at 3.13 ms; P = 2 runs in 2.89 ms.  The
// discount is only a tie-break because latency-bound kernels (c2) do not speed up alone.
inline int choose_P(const Plan& pl, long long B, int occ, int nsm) {
  const int oc = std::max(occ, 1);
  const long long cap = (long long)nsm * oc;
  int best = 1;
  double best_t = 1e300;
  auto plain = [&](int P) {
    const long long ctas = (long long)P * B;
    const double waves = (double)((ctas + cap - 1) / cap);
    const double iters = (double)((pl.U + (long long)P * pl.S - 1) / ((long long)P * pl.S));
    return waves * (iters + 1.0);
  };
  for (int P = 1; P <= pl.Pbound; ++P) {
    const double t = plain(P);
    if (t < best_t - 1e-9) {
      best_t = t;
      best = P;
    }
  }
  int pick = best;
  double pick_t = 1e300;
  for (int P = 1; P <= pl.Pbound; ++P) {
    if (plain(P) > 1.02 * best_t) continue;
    const long long ctas = (long long)P * B;
    const long long full = ctas / cap, rest = ctas - full * cap;
    const double j = (double)((rest + nsm - 1) / nsm);   // CTAs per SM in the partial wave
    const double waves = (double)full + (rest ? pow(j / (double)oc, 0.75) : 0.0);
    const double iters = (double)((pl.U + (long long)P * pl.S - 1) / ((long long)P * pl.S));
    const double t = waves * (iters + 1.0);
    if (t < pick_t - 1e-9) {
      pick_t = t;
      pick = P;
    }
  }
  return pick;
}

template <int M, int KIND, bool WGT, bool CROSS = false, int FLV = 0>
cudaError_t kernel_occupancy(size_t smem, int* occ, int* nsm) {
  static std::once_flag once[kMaxDev];
  static cudaError_t attr_err[kMaxDev];
  static int sm_count[kMaxDev];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::call_once(once[dev], [dev] {
    attr_err[dev] = cudaFuncSetAttribute(af_rows_kernel<M, KIND, WGT, CROSS, FLV>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (attr_err[dev] == cudaSuccess)
      attr_err[dev] = cudaDeviceGetAttribute(&sm_count[dev], cudaDevAttrMultiProcessorCount, dev);
  });
  if (attr_err[dev] != cudaSuccess) return attr_err[dev];
  *nsm = sm_count[dev];
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, af_rows_kernel<M, KIND, WGT, CROSS, FLV>, Cfg<M>::THREADS, smem);
  if (e != cudaSuccess) return e;
  // The occupancy API reported 1 for the M = 8192 kernels (2 x 104 832 B of dynamic shared
  // memory) although two CTAs are resident per SM (ncu: launch__occupancy_limit_shared_mem and
  // _registers = 2; scripts/block_one.py), so the launch model planned c4's blocks for 148
  // slots instead of 296.  __launch_bounds__ guarantees registers and threads for MinBlocks
  // CTAs; with the SM's 228 KiB of shared memory (1 KiB reserved per CTA) that is a lower
  // bound on the resident CTAs.
  const int by_smem = (int)((228 * 1024) / (smem + 1024));
  *occ = std::max(*occ, std::min(MinBlocks<M, KIND>::value, by_smem));
  return cudaSuccess;
}

template <int M, int KIND, bool WGT, bool CROSS = false, int FLV = 0>
cudaError_t launch_kernel(Plan& pl, RowParams rp, int B, cudaStream_t st) {
  int occ = 1, nsm = device_sm_count();
  // (also sets the instantiation's large-shared-memory attribute, once per device)
  cudaError_t e0 = kernel_occupancy<M, KIND, WGT, CROSS, FLV>(pl.smem, &occ, &nsm);
  if (e0 != cudaSuccess) return e0;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  size_t smem = pl.smem;
  rp.gpad = 0;
  if (pl.gpad_ok && KIND != K_ADJ && KIND != K_FWD && KIND != K_FWDA) {
    if (pl.gpad_mode < 0) {
      int occ_g = 0;
      const bool fits = pl.smem + pl.smem_gpad <= 227 * 1024;
      if (fits) {
        e0 = kernel_occupancy<M, KIND, WGT, CROSS, FLV>(pl.smem + pl.smem_gpad, &occ_g, &nsm);
        if (e0 != cudaSuccess) return e0;
      }
      pl.gpad_mode = (fits && occ_g >= occ) ? 1 : 0;
    }
    if (pl.gpad_mode == 1) {
      rp.gpad = 1;
      smem += pl.smem_gpad;
    }
  }
  if (rp.surface && pl.bulk_ok) {
    if (pl.bulk_mode < 0) {
      // dedicated staging unless it costs resident CTAs and the exchange buffer can hold the rows
      int occ_d = 0;
      const bool fits = smem + pl.smem_stg <= 227 * 1024;
      if (fits) {
        e0 = kernel_occupancy<M, KIND, WGT, CROSS, FLV>(smem + pl.smem_stg, &occ_d, &nsm);
        if (e0 != cudaSuccess) return e0;
      }
      pl.bulk_mode = (fits && (occ_d >= occ || !pl.alias_ok) && occ_d >= 1) ? 1 : pl.alias_ok ? 2 : 0;
    }
    rp.bulk = pl.bulk_mode;
    rp.stg_floats = pl.stg_floats;
    if (rp.bulk == 1) {
      smem += pl.smem_stg;
      e0 = kernel_occupancy<M, KIND, WGT, CROSS, FLV>(smem, &occ, &nsm);
      if (e0 != cudaSuccess) return e0;
    }
  } else {
    rp.bulk = 0;
  }
  if (!pl.fixedP) {
    pl.P = choose_P(pl, B, occ, nsm);
#ifdef GRAF_FORCE_P   // tuning builds only (scripts/c2_rows.py): -DGRAF_FORCE_P=<P> overrides the model
    pl.P = std::min(GRAF_FORCE_P, std::max(pl.Pbound, 1));
#endif
    pl.fixedP = true;   // later passes of the same call reuse it
#ifdef GRAF_DEBUG_PLAN   // tuning builds only: what the launch model saw and chose
    fprintf(stderr, "[graf plan] M=%d kind=%d flv=%d B=%d U=%d S=%d occ=%d nsm=%d Pbound=%d P=%d smem=%zu\n", M, KIND, FLV, B,
            pl.U, pl.S, occ, nsm, pl.Pbound, pl.P, smem);
#endif
  }
  rp.fuse = 0;
  if (KIND == K_ISL && !CROSS && Cfg<M>::G_SMEM && pl.fuse_req && pl.P >= 2 && pl.P <= 8) {   // (P = 1: measured slower as a cluster launch)
    rp.fuse = 1;
    pl.fused = true;
  }
  for (int b0 = 0; b0 < B; b0 += 65535) {
    rp.b0 = b0;
    dim3 grid(pl.P, std::min(65535, B - b0));
    rp.smem_bytes = (int)smem;
    if (rp.fuse) {
      // the P CTAs of a waveform form one thread-block cluster (rank 0 finalizes)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(pl.threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = (unsigned)pl.P;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, af_rows_kernel<M, KIND, WGT, CROSS, FLV>, rp);
      if (e != cudaSuccess) return e;
    } else {
      af_rows_kernel<M, KIND, WGT, CROSS, FLV><<<grid, pl.threads, smem, st>>>(rp);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++t_launches;
  }
  return cudaSuccess;
}

template <int M>
cudaError_t launch_rows_t(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind, bool wgt) {
  if (pl.cross) {
    // cross-ambiguity kernels: unweighted, M <= 4096 (the second waveform is staged too)
    if constexpr (M <= 4096) {
      switch (kind) {
        case K_FWD: return launch_kernel<M, K_FWD, false, true>(pl, rp, B, st);
        case K_ISL: return launch_kernel<M, K_ISL, false, true>(pl, rp, B, st);
        case K_PASS2: return launch_kernel<M, K_PASS2, false, true>(pl, rp, B, st);
        case K_ADJ: return launch_kernel<M, K_ADJ, false, true>(pl, rp, B, st);
        default: return cudaErrorNotSupported;
      }
    } else {
      return cudaErrorNotSupported;
    }
  }
#ifndef GRAF_NOSURF_SPEC
#define GRAF_NOSURF_SPEC 1
#endif
#ifndef GRAF_EDGE_FLAVOUR
#define GRAF_EDGE_FLAVOUR 1
#endif
#ifndef GRAF_NOSURF_MIN_M
#define GRAF_NOSURF_MIN_M 8192
#endif
  if constexpr (M >= GRAF_NOSURF_MIN_M && GRAF_NOSURF_SPEC) {
    if (rp.surface == nullptr && GRAF_EDGE_FLAVOUR && rp.loss_on && rp.d_max < Cfg<M>::T && !wgt) {
      // loss-only on a band narrower than T bins (c4): the band-edge flavour
      switch (kind) {
        case K_FWD:
          if (!rp.want_argmax) return launch_kernel<M, K_FWD, false, false, 2>(pl, rp, B, st);
          break;
        case K_PASS2: return launch_kernel<M, K_PASS2, false, false, 2>(pl, rp, B, st);
        case K_ISL: return launch_kernel<M, K_ISL, false, false, 2>(pl, rp, B, st);
        default: break;
      }
    }
    if (rp.surface == nullptr) {   // loss-only calls: the instantiations without the surface epilogue
      switch (kind) {
        case K_FWD:
          if (rp.want_argmax)
            return wgt ? launch_kernel<M, K_FWDA, true, false, 1>(pl, rp, B, st)
                       : launch_kernel<M, K_FWDA, false, false, 1>(pl, rp, B, st);
          return wgt ? launch_kernel<M, K_FWD, true, false, 1>(pl, rp, B, st)
                     : launch_kernel<M, K_FWD, false, false, 1>(pl, rp, B, st);
        case K_ISL:
          return wgt ? launch_kernel<M, K_ISL, true, false, 1>(pl, rp, B, st)
                     : launch_kernel<M, K_ISL, false, false, 1>(pl, rp, B, st);
        case K_PASS2:
          return wgt ? launch_kernel<M, K_PASS2, true, false, 1>(pl, rp, B, st)
                     : launch_kernel<M, K_PASS2, false, false, 1>(pl, rp, B, st);
        case K_MATCH:
          return wgt ? launch_kernel<M, K_MATCH, true, false, 1>(pl, rp, B, st)
                     : launch_kernel<M, K_MATCH, false, false, 1>(pl, rp, B, st);
        default: break;
      }
    }
  }
  switch (kind) {
    case K_FWD:
      if (rp.want_argmax)
        return wgt ? launch_kernel<M, K_FWDA, true>(pl, rp, B, st) : launch_kernel<M, K_FWDA, false>(pl, rp, B, st);
      return wgt ? launch_kernel<M, K_FWD, true>(pl, rp, B, st) : launch_kernel<M, K_FWD, false>(pl, rp, B, st);
    case K_ISL: return wgt ? launch_kernel<M, K_ISL, true>(pl, rp, B, st) : launch_kernel<M, K_ISL, false>(pl, rp, B, st);
    case K_PASS2:
      return wgt ? launch_kernel<M, K_PASS2, true>(pl, rp, B, st) : launch_kernel<M, K_PASS2, false>(pl, rp, B, st);
    case K_ADJ: return launch_kernel<M, K_ADJ, false>(pl, rp, B, st);
    case K_MATCH:
      return wgt ? launch_kernel<M, K_MATCH, true>(pl, rp, B, st) : launch_kernel<M, K_MATCH, false>(pl, rp, B, st);
    default: return cudaErrorInvalidValue;
  }
}


// one instantiation per size, defined in graf_rows_*.cu
template <int M>
cudaError_t launch_rows_size(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind);
// fill of one translation unit's copy of the twiddle table, enqueued on a stream
using TwFill = cudaError_t (*)(cudaStream_t);
std::vector<TwFill>& tw_fillers();

}  // namespace graf
