// Scene-generator entry points implemented in scenes.cu.
#pragma once
#include <cuda_runtime.h>

namespace octf {

constexpr int kMaxOctaves = 4;

// cam = {fx, fy, cx, cy, R (3x3 camera-to-world, row-major), centre} (host);
// z = H x W camera-frame depths (f64, device), 0 = no hit
void trace_blob(const double* cam, int width, int height, const double* centre,
                double radius, double amp, double base_freq,
                const double* const* lattices, const int* lat_n, int noct,
                double lipschitz, double t_max, int steps, double eps,
                double* z, cudaStream_t st);
// objects (device) = nb boxes {centre, half extents} then ns spheres
// {centre, radius}
void trace_room(const double* cam, int width, int height, const double* objects,
                int nb, int ns, double size, double lipschitz, double t_max,
                int steps, double eps, double* z, cudaStream_t st);

}  // namespace octf
