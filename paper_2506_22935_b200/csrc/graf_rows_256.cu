// graf_rows_256.cu — af_rows_kernel instantiations for M in {256} (see graf_launch.cuh)
#include "graf_launch.cuh"

namespace graf {
namespace {
cudaError_t upload(const float2* h) { return cudaMemcpyToSymbol(g_tw, h, sizeof(float2) * kMaxM); }
struct Register {
  Register() { tw_uploaders().push_back(&upload); }
} register_tw;
}  // namespace

template <>
cudaError_t launch_rows_size<256>(Plan& pl, const RowParams& rp, int B, cudaStream_t st, int kind) {
  return launch_rows_t<256>(pl, rp, B, st, kind, (rp.w_k != nullptr) || (rp.w_d != nullptr));
}

}  // namespace graf
