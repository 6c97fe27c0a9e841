// Zero-isosurface readout on the GPU: the
// reference's marching cubes over a dense cell-centred grid
// (octfuse/mesh.py:63-125, extract_zero_surface + marching_cubes), same
// vertex and face order, same f64 vertex arithmetic.  Compiled -fmad=false.
//
//   1. per cube (x, y, z) of the m = n-1 cubes per axis: its 8-corner
//      inside pattern (bit c = corner (c>>2&1, c>>1&1, c&1) has value < 0)
//      and 3 x the case's triangle count if every corner is observed;
//   2. exclusive scan -> each active cube's slot in the edge list, which
//      holds, in cube order then table order, the key
//      ((axis*n + ex)*n + ey)*n + ez of every triangle corner's grid edge;
//   3. sorted unique keys = the vertices (ascending key, numpy.unique);
//      faces = each edge's rank among them (numpy's inverse);
//   4. a vertex interpolates the zero crossing along its edge,
//      t = v0 / (v0 - v1), then origin + (p + 1/2) * voxel in world mode.
#include <cub/cub.cuh>

#include "octf_ctx.h"
#include "../../include/octfuse_b200.h"

namespace octf {
namespace {

constexpr int kMT = 256;

inline unsigned grid_of(int64_t n) {
  int64_t g = (n + kMT - 1) / kMT;
  return (unsigned)(g < 1 ? 1 : g);
}

__constant__ int8_t c_tri[256 * 32];
__constant__ int8_t c_cnt[256];
// edge e: axis, and the cube-local offset of its low corner
__constant__ int8_t c_eax[12];
__constant__ int8_t c_eoff[12 * 3];

__global__ void k_mc_count(const double* __restrict__ v,
                           const uint8_t* __restrict__ mask, int n,
                           int32_t* cnt, uint8_t* cases) {
  const int64_t m = n - 1;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m * m * m) return;
  const int64_t x = q / (m * m), y = (q / m) % m, z = q % m;
  unsigned cs = 0;
  bool usable = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int64_t g = ((x + ((c >> 2) & 1)) * n + (y + ((c >> 1) & 1))) * n +
                      (z + (c & 1));
    cs |= (v[g] < 0.0 ? 1u : 0u) << c;
    if (mask) usable = usable && mask[g] != 0;
  }
  cases[q] = (uint8_t)cs;
  cnt[q] = usable ? 3 * (int32_t)c_cnt[cs] : 0;
}

__global__ void k_mc_emit(const int32_t* __restrict__ cnt,
                          const int32_t* __restrict__ off,
                          const uint8_t* __restrict__ cases, int n,
                          int64_t* keys) {
  const int64_t m = n - 1;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m * m * m) return;
  const int k = cnt[q];
  if (!k) return;
  const int64_t x = q / (m * m), y = (q / m) % m, z = q % m;
  const int cs = cases[q];
  int64_t* out = keys + off[q];
  for (int j = 0; j < k; ++j) {
    const int e = c_tri[cs * 32 + j];
    out[j] = (((int64_t)c_eax[e] * n + x + c_eoff[3 * e]) * n + y +
              c_eoff[3 * e + 1]) * n + z + c_eoff[3 * e + 2];
  }
}

__global__ void k_mc_faces(const int64_t* __restrict__ keys, int64_t ne,
                           const int64_t* __restrict__ ukeys, int64_t nu,
                           int32_t* faces) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= ne) return;
  const int64_t k = keys[p];
  int64_t lo = 0, hi = nu;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ukeys[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  faces[p] = (int32_t)lo;
}

__global__ void k_mc_verts(const int64_t* __restrict__ ukeys, int64_t nu,
                           const double* __restrict__ v, int n, int world,
                           double ox, double oy, double oz, double voxel,
                           double* verts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nu) return;
  const int64_t k = ukeys[i];
  const int64_t uz = k % n, uy = (k / n) % n, ux = (k / ((int64_t)n * n)) % n;
  const int ax = (int)(k / ((int64_t)n * n * n));
  const double v0 = v[(ux * n + uy) * n + uz];
  const double v1 = v[((ux + (ax == 0)) * n + uy + (ax == 1)) * n + uz +
                      (ax == 2)];
  const double t = v0 / (v0 - v1);
  // numpy: u + t * (axis == a), the boolean as 1.0 / 0.0
  double p0 = (double)ux + t * (ax == 0 ? 1.0 : 0.0);
  double p1 = (double)uy + t * (ax == 1 ? 1.0 : 0.0);
  double p2 = (double)uz + t * (ax == 2 ? 1.0 : 0.0);
  if (world) {  // origin + (p + 0.5) * voxel_size (mesh.py:122-123)
    p0 = ox + (p0 + 0.5) * voxel;
    p1 = oy + (p1 + 0.5) * voxel;
    p2 = oz + (p2 + 0.5) * voxel;
  }
  verts[3 * i] = p0;
  verts[3 * i + 1] = p1;
  verts[3 * i + 2] = p2;
}

template <typename T>
T* dalloc(size_t n) {
  T* p = nullptr;
  if (cudaMalloc((void**)&p, (n ? n : 1) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    throw Error(kENoMem, "device allocation failed");
  }
  return p;
}

struct Scratch {  // freed on every exit path
  std::vector<void*> ptrs;
  template <typename T>
  T* get(size_t n) {
    T* p = dalloc<T>(n);
    ptrs.push_back(p);
    return p;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFree(p);
  }
};

}  // namespace

void marching_cubes(const double* values, const uint8_t* mask, int n,
                    const int8_t* tri_table, const int8_t* tri_count,
                    const int8_t* edge_axis, const int8_t* edge_off,
                    const double* origin, double voxel, int world,
                    octf_mesh* out, cudaStream_t st) {
  if (n < 2) throw Error(kEArg, "values must be a cubic grid with edge >= 2");
  OCTF_CUDA(cudaMemcpyToSymbolAsync(c_tri, tri_table, 256 * 32, 0,
                                    cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyToSymbolAsync(c_cnt, tri_count, 256, 0,
                                    cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyToSymbolAsync(c_eax, edge_axis, 12, 0,
                                    cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyToSymbolAsync(c_eoff, edge_off, 36, 0,
                                    cudaMemcpyHostToDevice, st));
  const int64_t m = n - 1, M = m * m * m;
  Scratch sc;
  int32_t* cnt = sc.get<int32_t>(M);
  int32_t* off = sc.get<int32_t>(M);
  uint8_t* cases = sc.get<uint8_t>(M);
  k_mc_count<<<grid_of(M), kMT, 0, st>>>(values, mask, n, cnt, cases);
  OCTF_CUDA(cudaGetLastError());
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, off, (int)M, st);
  void* tmp = sc.get<uint8_t>(bytes);
  OCTF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, off, (int)M, st));
  int32_t last_off = 0, last_cnt = 0;
  OCTF_CUDA(cudaMemcpyAsync(&last_off, off + M - 1, 4, cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaMemcpyAsync(&last_cnt, cnt + M - 1, 4, cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  const int64_t ne = (int64_t)last_off + last_cnt;
  out->nf = ne / 3;
  if (ne == 0) {
    out->nv = 0;
    return;
  }
  int64_t* keys = sc.get<int64_t>(ne);
  k_mc_emit<<<grid_of(M), kMT, 0, st>>>(cnt, off, cases, n, keys);
  OCTF_CUDA(cudaGetLastError());
  // sorted unique keys
  int64_t* sorted = sc.get<int64_t>(ne);
  int64_t* ukeys = sc.get<int64_t>(ne);
  int64_t* nu_d = sc.get<int64_t>(1);
  bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys, sorted, (int)ne, 0, 64,
                                 st);
  size_t b2 = 0;
  cub::DeviceSelect::Unique(nullptr, b2, sorted, ukeys, nu_d, (int)ne, st);
  void* tmp2 = sc.get<uint8_t>(bytes > b2 ? bytes : b2);
  OCTF_CUDA(cub::DeviceRadixSort::SortKeys(tmp2, bytes, keys, sorted, (int)ne,
                                           0, 64, st));
  OCTF_CUDA(cub::DeviceSelect::Unique(tmp2, b2, sorted, ukeys, nu_d, (int)ne,
                                      st));
  int64_t nu = 0;
  OCTF_CUDA(cudaMemcpyAsync(&nu, nu_d, 8, cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  out->nv = nu;
  out->faces = dalloc<int32_t>(ne);
  out->verts = dalloc<double>(3 * nu);
  k_mc_faces<<<grid_of(ne), kMT, 0, st>>>(keys, ne, ukeys, nu, out->faces);
  k_mc_verts<<<grid_of(nu), kMT, 0, st>>>(ukeys, nu, values, n, world,
                                          origin[0], origin[1], origin[2],
                                          voxel, out->verts);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace octf
