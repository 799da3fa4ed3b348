// graf_rows_2048.cu — af_rows_kernel instantiations for M in {2048} (see graf_launch.cuh)
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
cudaError_t launch_rows_size<2048>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<2048>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

}  // namespace graf
