// Mesh comparison entry point implemented in mesh_diff.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace octf {

// dist[i] = distance from a[i] to its nearest point of b (na x 3 and nb x 3
// f64 device arrays); synchronises the stream before returning
void nearest_vertex(const double* a, int64_t na, const double* b, int64_t nb,
                    double* dist, cudaStream_t st);

}  // namespace octf
