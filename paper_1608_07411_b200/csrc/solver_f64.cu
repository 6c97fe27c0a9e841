// Parity mode: T = double, compiled with -fmad=false (see octf_arith.cuh).
#include "solver_impl.cuh"

namespace octf {
void iterate_pass_f64(Ctx& c, IterArgs& a, cudaStream_t st) {
  iterate_pass_impl<double>(c, a, st);
}
void propagate_ctx_f64(Ctx& c, double* value, const int32_t* child,
                       cudaStream_t st) {
  propagate_impl<double>(c, value, child, st);
}
double energy_f64(Ctx& c, const double* u, const int32_t* child,
                  const PassParams& p, double* terms, cudaStream_t st) {
  return energy_impl<double>(c, u, child, p, terms, st);
}
}  // namespace octf

namespace octf {
void frozen_passes_f64(Ctx& c, FrozenArgs& a, cudaStream_t st) {
  frozen_passes_impl<double>(c, a, st);
}
}  // namespace octf

namespace octf {
void propagate_levels_f64(Ctx& c, double* v, const int32_t* child, int lo, int hi,
                         cudaStream_t st) {
  propagate_levels_impl<double>(c, v, child, lo, hi, st);
}
}  // namespace octf

namespace octf {
void pass_tiles_f64(Ctx& c, TileArgs& a, cudaStream_t st) {
  pass_tiles_impl<double>(c, a, st);
}
void pass_finish_f64(Ctx& c, void* uval, const int32_t* child,
                     double* dev_energy, cudaStream_t st) {
  pass_finish_impl<double>(c, (double*)uval, child, dev_energy, st);
}
void pd_restructure_f64(Ctx& c, PdRsArgs& a, cudaStream_t st) {
  pd_restructure_impl<double>(c, a, st);
}
void pd_passes_f64(Ctx& c, PdHostArgs& a, cudaStream_t st) {
  pd_passes_impl<double>(c, a, st);
}
}  // namespace octf
