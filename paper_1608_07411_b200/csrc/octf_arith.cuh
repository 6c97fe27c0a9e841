// Arithmetic of the descent update in the two precision modes.
//
// double: the parity ("exact") mode.  Every expression keeps the reference's
//   operand order (_kernels.pyx:205-253, 517-533) and the translation unit is
//   compiled with -fmad=false, so no FMA contraction changes a rounding;
//   sqrt and division are the IEEE correctly-rounded defaults.  Division by
//   the cell spacing h = 2^(d_max-L) is done as multiplication by 2^-(...),
//   which rounds the same real number and is therefore bit-identical.
// float: the throughput mode (fp32 u and arithmetic, SFU rsqrt; the
//   north_star's "u within 1e-4" tolerance).
#pragma once
#include <cuda_runtime.h>

namespace octf {
namespace {

template <typename T>
struct Arith;

template <>
struct Arith<double> {
  // p = g / sqrt(|g|^2 + eps^2)  (flux3, _kernels.pyx:217-220)
  __device__ __forceinline__ static void flux(double gx, double gy, double gz,
                                              double eps2, double& px,
                                              double& py, double& pz) {
    double gn = sqrt(gx * gx + gy * gy + gz * gz + eps2);
    px = gx / gn;
    py = gy / gn;
    pz = gz / gn;
  }
  // one component only (backward fluxes use a single component)
  __device__ __forceinline__ static double flux1(double g, double gx, double gy,
                                                 double gz, double eps2) {
    double gn = sqrt(gx * gx + gy * gy + gz * gz + eps2);
    return g / gn;
  }
  // w * d / sqrt(d^2 + eps^2)  (_kernels.pyx:251)
  __device__ __forceinline__ static double data_grad(double w, double d,
                                                     double eps2) {
    return w * d / sqrt(d * d + eps2);
  }
  // w * sqrt(d^2 + eps^2)  (_kernels.pyx:531)
  __device__ __forceinline__ static double data_val(double w, double d,
                                                    double eps2) {
    return w * sqrt(d * d + eps2);
  }
  __device__ __forceinline__ static double smooth_val(double gx, double gy,
                                                      double gz, double eps2) {
    return sqrt(gx * gx + gy * gy + gz * gz + eps2);
  }
  // both data terms from one root: gradient w*d/s (_kernels.pyx:251) and
  // value w*s (_kernels.pyx:531), s = sqrt(d^2 + eps^2)
  __device__ __forceinline__ static void data_both(double w, double d,
                                                   double eps2, double& g,
                                                   double& e) {
    const double s = sqrt(d * d + eps2);
    g = w * d / s;
    e = w * s;
  }
  __device__ __forceinline__ static double div(double a, double b) {
    return a / b;
  }
};

template <>
struct Arith<float> {
  __device__ __forceinline__ static void flux(float gx, float gy, float gz,
                                              float eps2, float& px, float& py,
                                              float& pz) {
    float r = rsqrtf(gx * gx + gy * gy + gz * gz + eps2);
    px = gx * r;
    py = gy * r;
    pz = gz * r;
  }
  __device__ __forceinline__ static float flux1(float g, float gx, float gy,
                                                float gz, float eps2) {
    return g * rsqrtf(gx * gx + gy * gy + gz * gz + eps2);
  }
  __device__ __forceinline__ static float data_grad(float w, float d,
                                                    float eps2) {
    return w * d * rsqrtf(d * d + eps2);
  }
  __device__ __forceinline__ static float data_val(float w, float d,
                                                   float eps2) {
    return w * sqrtf(d * d + eps2);
  }
  __device__ __forceinline__ static float smooth_val(float gx, float gy,
                                                     float gz, float eps2) {
    return sqrtf(gx * gx + gy * gy + gz * gz + eps2);
  }
  __device__ __forceinline__ static void data_both(float w, float d, float eps2,
                                                   float& g, float& e) {
    const float q = d * d + eps2;
    const float r = rsqrtf(q);
    g = w * d * r;
    e = w * q * r;
  }
  __device__ __forceinline__ static float div(float a, float b) {
    return __fdividef(a, b);
  }
};

}  // namespace
}  // namespace octf
