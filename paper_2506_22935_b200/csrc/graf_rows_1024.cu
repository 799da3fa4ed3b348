// graf_rows_1024.cu — af_rows_kernel instantiations for M in {1024} (see graf_launch.cuh)
//
// Paired fp32 arithmetic (FADD2 / FMUL2 / FFMA2, graf_fft.cuh) in this unit only: at
// M = 1024 the row kernels are issue-bound (72 % issue-slot use in full-surface mode)
// and the paired forms cut the FP instruction count by ~45 %: c3 -15 %, c3 forward -4 %
// (profiles/r01_f32x2_ab.txt).  The other sizes are bound by latency and the FMA pipe
// (a paired instruction holds it for two cycles) and measured neutral or slower.
#ifndef GRAF_NO_F32X2
#define GRAF_F32X2 1
#endif
#include "graf_launch.cuh"

namespace graf {
namespace {
// this unit's copy of the twiddle table, filled on the caller's stream
cudaError_t tw_fill(cudaStream_t st) { return launch_tw_init(st); }
struct Register {
  Register() { tw_fillers().push_back(&tw_fill); }
} register_tw;
}  // namespace

template <>
cudaError_t launch_rows_size<1024>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<1024>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

}  // namespace graf
