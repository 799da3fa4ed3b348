// graf_rows_small.cu — af_rows_kernel instantiations for M in {2, 4, 8, 16, 32, 64, 128} (see graf_launch.cuh)
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
cudaError_t launch_rows_size<2>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<2>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

template <>
cudaError_t launch_rows_size<4>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<4>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

template <>
cudaError_t launch_rows_size<8>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<8>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

template <>
cudaError_t launch_rows_size<16>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<16>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

template <>
cudaError_t launch_rows_size<32>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<32>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

template <>
cudaError_t launch_rows_size<64>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<64>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

template <>
cudaError_t launch_rows_size<128>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<128>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

}  // namespace graf
