// Throughput mode: T = float (fp32 u, SFU rsqrt); see octf_arith.cuh.
#include "solver_impl.cuh"

namespace octf {
void iterate_pass_f32(Ctx& c, IterArgs& a, cudaStream_t st) {
  iterate_pass_impl<float>(c, a, st);
}
void propagate_ctx_f32(Ctx& c, float* value, const int32_t* child,
                       cudaStream_t st) {
  propagate_impl<float>(c, value, child, st);
}
double energy_f32(Ctx& c, const float* u, const int32_t* child,
                  const PassParams& p, double* terms, cudaStream_t st) {
  return energy_impl<float>(c, u, child, p, terms, st);
}
}  // namespace octf

namespace octf {
void frozen_passes_f32(Ctx& c, FrozenArgs& a, cudaStream_t st) {
  frozen_passes_impl<float>(c, a, st);
}
}  // namespace octf

namespace octf {
void propagate_levels_f32(Ctx& c, float* v, const int32_t* child, int lo, int hi,
                         cudaStream_t st) {
  propagate_levels_impl<float>(c, v, child, lo, hi, st);
}
}  // namespace octf

namespace octf {
void pass_tiles_f32(Ctx& c, TileArgs& a, cudaStream_t st) {
  pass_tiles_impl<float>(c, a, st);
}
void pass_finish_f32(Ctx& c, void* uval, const int32_t* child,
                     double* dev_energy, cudaStream_t st) {
  pass_finish_impl<float>(c, (float*)uval, child, dev_energy, st);
}
void pd_restructure_f32(Ctx& c, PdRsArgs& a, cudaStream_t st) {
  pd_restructure_impl<float>(c, a, st);
}
void pd_passes_f32(Ctx& c, PdHostArgs& a, cudaStream_t st) {
  pd_passes_impl<float>(c, a, st);
}
}  // namespace octf
