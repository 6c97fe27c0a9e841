// Zero-isosurface readout straight from the leaf store (SURVEY.md §8(f)
// row 1): the reference reads a mesh as densify (octree.py:327-342) + marching
// cubes over the (2^d)^3 grid (mesh.py:63-125) -- 69 GB at BASELINE config 3's
// depth 11, 550 GB at config 4's depth 12.  Here no dense grid exists:
//
//   1. bricks of 8^3 cubes; a cube's 8 corners are finest cells, so a cube can
//      only cross zero where its corners lie in leaves of both signs.  Every
//      leaf ORs its sign into the bricks whose corner region (the brick's 9^3
//      cells) it meets -- the shell of a coarse leaf only, its interior bricks
//      see that leaf alone;
//   2. bricks that saw both signs are compacted;
//   3. one CTA per such brick reads its 9^3 corner values by root descents
//      (the value of the leaf covering the cell: densify's value) and the
//      optional observed mask from a second tree, and does the reference's
//      per-cube work: case, usable (all corners observed), table triangles;
//      every triangle corner is emitted with a global order key (cube index
//      << 4 | table position) and its grid-edge key and crossing t;
//   4. a radix sort on the order key restores the reference's face order
//      (cube order, then table order), a sort + unique-by-key on the edge
//      keys its vertex order (numpy.unique), faces are each corner's rank.
// Vertex arithmetic is the dense path's (t = v0/(v0 - v1), p = i + t*[axis],
// origin + (p + 1/2) * voxel), compiled -fmad=false: the mesh equals
// marching_cubes(densify(u), seen) bit for bit (tests/test_mesh.py).
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

#include "octf_ctx.h"
#include "../../include/octfuse_b200.h"

namespace octf {
namespace {

constexpr int kB = 8;           // cubes per brick edge
constexpr int kC = kB + 1;      // corner cells per brick edge
constexpr int kMT = 256;

__constant__ int8_t c_tri[256 * 32];
__constant__ int8_t c_cnt[256];
__constant__ int8_t c_eax[12];
__constant__ int8_t c_eoff[12 * 3];

inline unsigned grid_of(int64_t n) {
  const int64_t g = (n + kMT - 1) / kMT;
  return (unsigned)(g < 1 ? 1 : (g > 2147483647 ? 2147483647 : g));
}

// leaf covering finest cell (x, y, z): its value as f64
template <typename T>
__device__ __forceinline__ double cell_value(const T* __restrict__ value,
                                             const int32_t* __restrict__ child,
                                             int d, int x, int y, int z) {
  return (double)value[descend(child, d, x, y, z)];
}

// 1. sign marks: one warp per leaf block of the context's list, its leaves
// one after the other, lanes over the bricks of the leaf's shell
template <typename T>
__global__ void k_brick_marks(const int4* __restrict__ lmeta, int64_t nlb,
                              const T* __restrict__ value, int d, int nb,
                              uint32_t* marks) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nlb) return;
  const int4 m = lmeta[w];
  int L, pz;
  unsigned mask;
  unpack_meta_w(m.w, pz, mask, L);
  if (m.x == 0) mask &= 1u;
  const int n = 1 << d;
  for (int c = 0; c < 8; ++c) {
    if (!((mask >> c) & 1u)) continue;
    const int S = 1 << (d - L);
    const int cx = m.x == 0 ? 0 : 2 * meta_px(m.y) + ((c >> 2) & 1);
    const int cy = m.x == 0 ? 0 : 2 * m.z + ((c >> 1) & 1);
    const int cz = m.x == 0 ? 0 : 2 * pz + (c & 1);
    const int x0 = cx * S, y0 = cy * S, z0 = cz * S;
    const unsigned bit = value[m.x + c] < (T)0 ? 1u : 2u;
    // bricks whose corner cells [8b, 8b+8] meet [x0, x0+S)
    auto lo = [](int a0) { return a0 == 0 ? 0 : (a0 - 1) / kB; };
    auto hi = [&](int a0) {
      const int h = (a0 + S - 1) / kB;
      return h < nb ? h : nb - 1;
    };
    // interior along an axis: the corner cells lie inside the leaf
    auto in = [&](int b, int a0) { return kB * b >= a0 && kB * b + kB <= a0 + S - 1; };
    const int xl = lo(x0), xh = hi(x0), yl = lo(y0), yh = hi(y0);
    const int zl = lo(z0), zh = hi(z0);
    const int ny = yh - yl + 1, nz = zh - zl + 1;
    const int64_t nxy = (int64_t)(xh - xl + 1) * ny;
    for (int64_t q = lane; q < nxy; q += 32) {
      const int bx = xl + (int)(q / ny), by = yl + (int)(q % ny);
      const bool ixy = in(bx, x0) && in(by, y0);
      for (int k = 0; k < nz; ++k) {
        const int bz = zl + k;
        if (ixy && in(bz, z0)) {  // skip to the far shell plane
          k = nz - 2 > k ? nz - 2 : k;
          continue;
        }
        const int64_t bi = ((int64_t)bx * nb + by) * nb + bz;
        atomicOr(marks + (bi >> 4), bit << (2 * (bi & 15)));
      }
    }
  }
  (void)n;
}

// 2. bricks that saw both signs
// (bricks with x index in [bx0, bx1) only: a slab of the readout)
__global__ void k_brick_list(const uint32_t* __restrict__ marks, int64_t nbr,
                             int64_t nb2, int64_t bx0, int64_t bx1,
                             int64_t* list, int32_t* count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool on = false;
  if (i < nbr && i / nb2 >= bx0 && i / nb2 < bx1)
    on = ((marks[i >> 4] >> (2 * (i & 15))) & 3u) == 3u;
  const unsigned q = __ballot_sync(0xffffffffu, on);
  int base = 0;
  if ((threadIdx.x & 31) == 0 && q) base = atomicAdd(count, __popc(q));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (on) list[base + __popc(q & ((1u << (threadIdx.x & 31)) - 1u))] = i;
}

// 3. per brick: corner values, cases, triangles.  EMIT = false counts the
// brick's triangle corners; EMIT = true writes them from off[brick]
template <typename T, typename S, bool EMIT>
__global__ void __launch_bounds__(kMT) k_brick_mc(
    const int64_t* __restrict__ bricks, const T* __restrict__ value,
    const int32_t* __restrict__ child, const S* __restrict__ seen_v,
    const int32_t* __restrict__ seen_c, int d, int nb, int32_t* cnt,
    const int64_t* __restrict__ off, uint64_t* okey, int64_t* ekey,
    double* tval) {
  __shared__ double sv[kC * kC * kC];
  __shared__ uint8_t ss[kC * kC * kC];
  const int64_t bi = bricks[blockIdx.x];
  const int bx = (int)(bi / ((int64_t)nb * nb)), by = (int)((bi / nb) % nb),
            bz = (int)(bi % nb);
  const int n = 1 << d;
  for (int q = threadIdx.x; q < kC * kC * kC; q += kMT) {
    const int x = kB * bx + q / (kC * kC), y = kB * by + (q / kC) % kC,
              z = kB * bz + q % kC;
    double v = 0.0;
    uint8_t o = 0;
    if (x < n && y < n && z < n) {
      v = cell_value(value, child, d, x, y, z);
      o = seen_c ? (seen_v[descend(seen_c, d, x, y, z)] != (S)0) : 1;
    }
    sv[q] = v;
    ss[q] = o;
  }
  __syncthreads();
  // two cubes per thread (8^3 = 512 per brick)
  int k[2] = {0, 0};
  unsigned cs[2] = {0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = threadIdx.x + h * kMT;
    const int lx = q >> 6, ly = (q >> 3) & 7, lz = q & 7;
    const int x = kB * bx + lx, y = kB * by + ly, z = kB * bz + lz;
    if (x >= n - 1 || y >= n - 1 || z >= n - 1) continue;
    bool usable = true;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int g = ((lx + ((c >> 2) & 1)) * kC + ly + ((c >> 1) & 1)) * kC +
                    lz + (c & 1);
      cs[h] |= (sv[g] < 0.0 ? 1u : 0u) << c;
      usable = usable && ss[g] != 0;
    }
    k[h] = usable ? 3 * (int)c_cnt[cs[h]] : 0;
  }
  typedef cub::BlockScan<int, kMT> BS;
  __shared__ typename BS::TempStorage tmp;
  int mine = k[0] + k[1], pre = 0, tot = 0;
  BS(tmp).ExclusiveSum(mine, pre, tot);
  if (!EMIT) {
    if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
    return;
  }
  int64_t o = off[blockIdx.x] + pre;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!k[h]) continue;
    const int q = threadIdx.x + h * kMT;
    const int lx = q >> 6, ly = (q >> 3) & 7, lz = q & 7;
    const int64_t x = kB * bx + lx, y = kB * by + ly, z = kB * bz + lz;
    const uint64_t cube = ((uint64_t)x * n + y) * n + z;
    for (int j = 0; j < k[h]; ++j, ++o) {
      const int e = c_tri[cs[h] * 32 + j];
      const int ax = c_eax[e];
      const int ex = lx + c_eoff[3 * e], ey = ly + c_eoff[3 * e + 1],
                ez = lz + c_eoff[3 * e + 2];
      const double v0 = sv[(ex * kC + ey) * kC + ez];
      const double v1 = sv[((ex + (ax == 0)) * kC + ey + (ax == 1)) * kC + ez +
                           (ax == 2)];
      okey[o] = (cube << 4) | (uint64_t)j;
      ekey[o] = (((int64_t)ax * n + kB * bx + ex) * n + kB * by + ey) * n +
                kB * bz + ez;
      tval[o] = v0 / (v0 - v1);
    }
  }
}

__global__ void k_gather_face(const int32_t* __restrict__ perm, int64_t ne,
                              const int64_t* __restrict__ ekey,
                              const double* __restrict__ tval, int64_t* fkey,
                              double* ft) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ne) return;
  const int64_t p = perm[i];
  fkey[i] = ekey[p];
  ft[i] = tval[p];
}

__global__ void k_tree_faces(const int64_t* __restrict__ keys, int64_t ne,
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

__global__ void k_tree_verts(const int64_t* __restrict__ ukeys,
                             const double* __restrict__ ut, int64_t nu, int n,
                             int world, double ox, double oy, double oz,
                             double voxel, double* verts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nu) return;
  const int64_t k = ukeys[i];
  const int64_t uz = k % n, uy = (k / n) % n, ux = (k / ((int64_t)n * n)) % n;
  const int ax = (int)(k / ((int64_t)n * n * n));
  const double t = ut[i];
  double p0 = (double)ux + t * (ax == 0 ? 1.0 : 0.0);
  double p1 = (double)uy + t * (ax == 1 ? 1.0 : 0.0);
  double p2 = (double)uz + t * (ax == 2 ? 1.0 : 0.0);
  if (world) {
    p0 = ox + (p0 + 0.5) * voxel;
    p1 = oy + (p1 + 0.5) * voxel;
    p2 = oz + (p2 + 0.5) * voxel;
  }
  verts[3 * i] = p0;
  verts[3 * i + 1] = p1;
  verts[3 * i + 2] = p2;
}

__global__ void k_widen(const int32_t* __restrict__ a, int64_t n, int64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) out[i] = i < n ? (int64_t)a[i] : 0;
}

__global__ void k_iota(int32_t* a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}

template <typename U>
U* tree_alloc(size_t n) {
  U* p = nullptr;
  if (cudaMalloc((void**)&p, (n ? n : 1) * sizeof(U)) != cudaSuccess) {
    cudaGetLastError();
    throw Error(kENoMem, "device allocation failed");
  }
  return p;
}

struct TreeScratch {
  std::vector<void*> ptrs;
  template <typename U>
  U* get(size_t n) {
    U* p = tree_alloc<U>(n);
    ptrs.push_back(p);
    return p;
  }
  void drop(void* p) {  // free early (the large per-corner temporaries)
    for (auto& q : ptrs)
      if (q == p) {
        cudaFree(q);
        q = nullptr;
      }
  }
  ~TreeScratch() {
    for (void* p : ptrs) cudaFree(p);
  }
};

template <typename T, typename S>
void mc_tree_impl(Ctx& c, const T* value, const int32_t* child, int d,
                  const S* seen_v, const int32_t* seen_c, const double* origin,
                  double voxel, int world, int64_t bx0, int64_t bx1,
                  octf_mesh* out, cudaStream_t st) {
  const int n = 1 << d;
  const int nb = (n - 1 + kB - 1) / kB;  // bricks per axis (n - 1 cubes)
  const int64_t nbr = (int64_t)nb * nb * nb;
  TreeScratch sc;
  uint32_t* marks = sc.get<uint32_t>((nbr + 15) / 16);
  OCTF_CUDA(cudaMemsetAsync(marks, 0, ((nbr + 15) / 16) * 4, st));
  if (c.nlb)
    k_brick_marks<T><<<grid_of(c.nlb * 32), kMT, 0, st>>>(c.lmeta.p, c.nlb,
                                                          value, d, nb, marks);
  OCTF_CUDA(cudaGetLastError());
  int64_t* list = sc.get<int64_t>(nbr);
  int32_t* dcount = sc.get<int32_t>(1);
  OCTF_CUDA(cudaMemsetAsync(dcount, 0, 4, st));
  k_brick_list<<<grid_of(nbr), kMT, 0, st>>>(
      marks, nbr, (int64_t)nb * nb, bx0 < 0 ? 0 : bx0,
      bx1 < 0 ? nb : bx1, list, dcount);
  OCTF_CUDA(cudaGetLastError());
  int32_t nlist = 0;
  OCTF_CUDA(cudaMemcpyAsync(&nlist, dcount, 4, cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  out->nv = out->nf = 0;
  if (!nlist) return;
  // per-brick corner counts -> offsets
  int32_t* cnt = sc.get<int32_t>(nlist);
  int64_t* off = sc.get<int64_t>(nlist + 1);
  k_brick_mc<T, S, false><<<nlist, kMT, 0, st>>>(
      list, value, child, seen_v, seen_c, d, nb, cnt, nullptr, nullptr,
      nullptr, nullptr);
  OCTF_CUDA(cudaGetLastError());
  int64_t* cnt64 = sc.get<int64_t>(nlist + 1);
  k_widen<<<grid_of(nlist + 1), kMT, 0, st>>>(cnt, nlist, cnt64);
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt64, off, (int)(nlist + 1),
                                st);
  void* tmp = sc.get<uint8_t>(bytes);
  OCTF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt64, off,
                                          (int)(nlist + 1), st));
  int64_t ne = 0;
  OCTF_CUDA(cudaMemcpyAsync(&ne, off + nlist, 8, cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  if (const char* md = std::getenv("OCTF_MESH_DEBUG"); md && md[0] == '1')
    fprintf(stderr, "mesh_tree: %d of %lld bricks mixed, %lld corners\n",
            nlist, (long long)nbr, (long long)ne);
  if (ne == 0) return;
  if (ne > (int64_t)2147483647)
    throw Error(kENoMem, "mesh too large for one call: read it in slabs");
  uint64_t* okey = sc.get<uint64_t>(2 * ne);
  int64_t* ekey = sc.get<int64_t>(ne);
  double* tval = sc.get<double>(ne);
  k_brick_mc<T, S, true><<<nlist, kMT, 0, st>>>(
      list, value, child, seen_v, seen_c, d, nb, nullptr, off, okey, ekey,
      tval);
  OCTF_CUDA(cudaGetLastError());
  // 4. face order: sort corner indices by (cube, table position); the
  // large per-corner temporaries are reused / freed as soon as they are
  // consumed (peak ~56 B per triangle corner)
  int32_t* idx = sc.get<int32_t>(2 * ne);
  k_iota<<<grid_of(ne), kMT, 0, st>>>(idx, ne);
  bytes = 0;
  const int obits = 3 * d + 4;
  cub::DoubleBuffer<uint64_t> ok(okey, okey + ne);
  cub::DoubleBuffer<int32_t> ov(idx, idx + ne);
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, ok, ov, (int)ne, 0, obits,
                                  st);
  void* tmp2 = sc.get<uint8_t>(bytes);
  OCTF_CUDA(cub::DeviceRadixSort::SortPairs(tmp2, bytes, ok, ov, (int)ne, 0,
                                            obits, st));
  int64_t* fkey = sc.get<int64_t>(ne);
  double* ft = sc.get<double>(ne);
  k_gather_face<<<grid_of(ne), kMT, 0, st>>>(ov.Current(), ne, ekey, tval,
                                             fkey, ft);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaStreamSynchronize(st));
  sc.drop(idx);
  sc.drop(tmp2);
  // vertices: the sorted unique edge keys, each with its crossing (the
  // sort writes into the consumed ekey / tval, the unique into okey)
  int64_t* skey = ekey;
  double* st_ = tval;
  int64_t* ukey = reinterpret_cast<int64_t*>(okey);
  double* ut = reinterpret_cast<double*>(okey + ne);
  int64_t* nu_d = sc.get<int64_t>(1);
  const int kbits = 3 * d + 2;
  bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, fkey, skey, ft, st_, (int)ne,
                                  0, kbits, st);
  size_t b2 = 0;
  cub::DeviceSelect::UniqueByKey(nullptr, b2, skey, st_, ukey, ut, nu_d,
                                 (int)ne, st);
  void* tmp3 = sc.get<uint8_t>(bytes > b2 ? bytes : b2);
  OCTF_CUDA(cub::DeviceRadixSort::SortPairs(tmp3, bytes, fkey, skey, ft, st_,
                                            (int)ne, 0, kbits, st));
  OCTF_CUDA(cub::DeviceSelect::UniqueByKey(tmp3, b2, skey, st_, ukey, ut, nu_d,
                                           (int)ne, st));
  int64_t nu = 0;
  OCTF_CUDA(cudaMemcpyAsync(&nu, nu_d, 8, cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  out->nf = ne / 3;
  out->nv = nu;
  out->faces = tree_alloc<int32_t>(ne);
  out->verts = tree_alloc<double>(3 * nu);
  k_tree_faces<<<grid_of(ne), kMT, 0, st>>>(fkey, ne, ukey, nu, out->faces);
  k_tree_verts<<<grid_of(nu), kMT, 0, st>>>(ukey, ut, nu, n, world, origin[0],
                                            origin[1], origin[2], voxel,
                                            out->verts);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

void marching_cubes_tree(Ctx& c, int dtype, const void* value,
                         const int32_t* child, int d_max, int seen_dtype,
                         const void* seen_v, const int32_t* seen_c,
                         const int8_t* tri_table, const int8_t* tri_count,
                         const int8_t* edge_axis, const int8_t* edge_off,
                         const double* origin, double voxel, int world,
                         int64_t bx0, int64_t bx1, octf_mesh* out,
                         cudaStream_t st) {
  if (d_max < 1) throw Error(kEArg, "values must be a cubic grid with edge >= 2");
  OCTF_CUDA(cudaMemcpyToSymbolAsync(c_tri, tri_table, 256 * 32, 0,
                                    cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyToSymbolAsync(c_cnt, tri_count, 256, 0,
                                    cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyToSymbolAsync(c_eax, edge_axis, 12, 0,
                                    cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyToSymbolAsync(c_eoff, edge_off, 36, 0,
                                    cudaMemcpyHostToDevice, st));
  const bool s64 = seen_dtype == OCTF_F64;
#define OCTF_MCT(T, S)                                                        \
  mc_tree_impl<T, S>(c, (const T*)value, child, d_max, (const S*)seen_v,      \
                     seen_c, origin, voxel, world, bx0, bx1, out, st)
  if (dtype == OCTF_F64) {
    if (s64) OCTF_MCT(double, double); else OCTF_MCT(double, float);
  } else {
    if (s64) OCTF_MCT(float, double); else OCTF_MCT(float, float);
  }
#undef OCTF_MCT
}

}  // namespace octf
