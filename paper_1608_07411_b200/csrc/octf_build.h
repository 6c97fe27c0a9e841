// Construction / readout entry points implemented in build.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace octf {

// inputs of the spread-rule build (reference _kernels.pyx:21-25)
struct BuildIn {
  const double* meanf;
  const double* minf;
  const double* maxf;
  const int64_t* offs;   // host level offsets (null: dense 8^l layout)
  int has_w;
  const uint8_t* wminf;
  const uint8_t* wmaxf;
  const double* wmeanf;
  double tau;
  int d_max;
  int64_t cap;
  // a box subtree of an enclosing tree (octf_build_octree_box): the global
  // level of the box root, the global depth, the root's depth-first rank and
  // slot; whole tree: 0, d_max, 0, 0
  int level0 = 0;
  int d_glob = -1;
  int64_t root_rank = 0;
  int32_t root_slot = 0;
  int64_t* nsplit_out = nullptr;  // splitting nodes of the (box) tree
};

void view_tsdf(const float* depth, int width, int height, const double* cam,
               const double* origin, double voxel, int n, const int* box,
               double delta, double eta, float* f, uint8_t* w, double* wf_sum,
               double* w_sum, cudaStream_t st);
void initial_field(const double* wf, const double* ws, double gamma, int64_t n,
                   double* u, cudaStream_t st);
void pyramids(const void* f, int f_dtype, const uint8_t* w, int d_max,
              double* minf, double* maxf, double* meanf, uint8_t* wminf,
              uint8_t* wmaxf, double* wmeanf, double* wf_tmp, double* pl_tmp,
              cudaStream_t st);
void build_tree(const BuildIn& in, void* value, int dtype, float* weight,
                int32_t* child, int64_t* state, bool do_propagate,
                cudaStream_t st);
void densify(int dtype, const void* value, const int32_t* child, int d_max,
             double* out, cudaStream_t st);

void locate(const int32_t* child, int level, const int32_t* cells, int64_t n,
            int32_t* node, int32_t* lvl, cudaStream_t st);

}  // namespace octf
