// Explicit instantiation unit: dtype float, 3-D grids (all features, parametrisations, KP).
#include "launch.cuh"
namespace sr {
SR_DEFINE_INST(f32, float, 3)
cudaError_t pass2_stream_d3(const Launch& L, const Args& a, const float* V, const float* G, long long vstride) {
  return run_pass2_stream<3>(L, a, V, G, vstride);
}
cudaError_t ngf_pass1_d3(const Launch& L, const Args& a, const NgfBufs& B, double* part, size_t cap, int* nblk) {
  return run_ngf_pass1<3>(L, a, B, part, cap, nblk);
}
cudaError_t ngf_pass2_d3(const Launch& L, const Args& a, const NgfBufs& B) { return run_ngf_pass2<3>(L, a, B); }
}  // namespace sr
