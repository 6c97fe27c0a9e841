// Shared device helpers for the octree fusion kernels (sm_100a).
//
// Node pools keep the reference layout (reference octree.py:49-71,
// _kernels.pyx:21-77): node 0 is the root, the children of a node are eight
// contiguous slots starting at child[n] (or child[n] == -1 for a leaf), and
// every allocated block of eight starts at a slot b with b % 8 == 1.  Block
// ids are k = (b + 7) >> 3, so the root's pseudo-block (b = 0) is k = 0 and
// the first real block (b = 1) is k = 1.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace octf {

constexpr int kMaxDepth = 19;   // 3*19 coordinate bits + 5 level bits fit u64
constexpr int32_t kNone = -1;   // neighbour table: outside the domain

__host__ __device__ __forceinline__ int octant(int x, int y, int z) {
  return ((x & 1) << 2) | ((y & 1) << 1) | (z & 1);
}

__host__ __device__ __forceinline__ int block_id(int64_t b) {
  return (int)((b + 7) >> 3);
}

// level (5 bits) | x | y | z (19 bits each): one u64 per block or cell
__host__ __device__ __forceinline__ uint64_t pack_cell(int L, uint32_t x,
                                                       uint32_t y, uint32_t z) {
  return ((uint64_t)L << 57) | ((uint64_t)x << 38) | ((uint64_t)y << 19) |
         (uint64_t)z;
}
__host__ __device__ __forceinline__ void unpack_cell(uint64_t p, int& L, int& x,
                                                     int& y, int& z) {
  L = (int)(p >> 57);
  x = (int)((p >> 38) & 0x7ffff);
  y = (int)((p >> 19) & 0x7ffff);
  z = (int)(p & 0x7ffff);
}

// leaf-block metadata word: pz (19 bits) | leaf mask (8) << 19 | level << 27
__host__ __device__ __forceinline__ int pack_meta_w(int pz, unsigned mask,
                                                    int L) {
  return (int)((unsigned)pz | (mask << 19) | ((unsigned)L << 27));
}
__host__ __device__ __forceinline__ void unpack_meta_w(int w, int& pz,
                                                       unsigned& mask, int& L) {
  pz = w & 0x7ffff;
  mask = ((unsigned)w >> 19) & 0xffu;
  L = (int)((unsigned)w >> 27);
}

// Per-leaf samples are stored in tiles of 256 leaves (one leaf-kernel CTA),
// view-major inside a tile: [tile][view][256].  A warp reading one view
// touches 128 contiguous bytes, and a whole tile is one contiguous
// nvp*1 KiB block that a single TMA bulk copy stages into shared memory.
constexpr int kTileLeaves = 256;
constexpr int kLeafParts = kTileLeaves / 32;  // energy partials per tile (warps)
// Sparse per-tile sample layout (ELL, many views): tile t = leaves
// [256t, 256t+256) holds K_t rows of 256 entries from off[t]; row j of a leaf
// is its j-th observed view in view order, rows past its count are zero.
__host__ __device__ __forceinline__ int64_t ell_idx(const int64_t* off,
                                                    int64_t leaf, int row) {
  return off[leaf >> 8] + ((int64_t)row << 8) + (leaf & 255);
}

__host__ __device__ __forceinline__ int64_t samp_idx(int64_t leaf, int v,
                                                     int64_t nvp) {
  return (leaf >> 8) * (nvp << 8) + ((int64_t)v << 8) + (leaf & 255);
}

// The dense sample store (Ctx::sd): tiles of 256 slots = the 32 leaf blocks
// a leaf-kernel CTA covers (leaf-block list entries 32t .. 32t+31), nvp rows
// (views padded to 4) each.
//  * slot layout: [tile][view][256], entry = the slot (samp_idx) -- inner
//    and free siblings of a leaf block own an (empty) entry too;
//  * packed layout (OCTF_CTX_PACKED, frozen trees): a leaf's entry is its
//    rank r among the tile's LEAVES, stored in chunks of kChunk = 16
//    leaves, [tile][r / 16][view][16].  The list keeps its spatial order
//    (neighbour values stay in L2 / L1); a tile's n_t leaves fill its
//    first ceil(n_t / 16) chunks, so the kernels stream only those -- no
//    entries for the inner siblings a leaf block spans (12 % of the slots
//    on BASELINE config 4).  Any prefix of chunks is valid whatever n_t
//    is, so the chunks of the first 192 leaves are staged at once and the
//    rest once n_t is known (leaf_kernel.cuh stage_packed).  A block's
//    first rank lives in the top byte of lmeta.y (px < 2^19).  Chunks of
//    16 halve the partly used last chunk of 32 (cfg5: 225 of a tile's 256
//    slots are leaves; descent kernel 0.787 -> 0.818 of HBM,
//    profiles/r02/ab_chunk16.txt) at the price of a 2-way bank conflict on
//    the staged reads (a warp's 32 ranks span two chunks a multiple of 32
//    banks apart); chunks of 8 lose.
#ifndef OCTF_CHUNK
#define OCTF_CHUNK 16
#endif
constexpr int kChunk = OCTF_CHUNK;  // leaves per chunk (a power of two <= 32)
// chunks staged before n_t is known: 192 leaves
constexpr int kEarlyChunks = 192 / kChunk;
struct SDesc {
  int packed = 0;
  int64_t nvp = 0;  // rows per tile (views padded to 4)
};
__host__ __device__ __forceinline__ int meta_px(int y) { return y & 0xffffff; }
__host__ __device__ __forceinline__ int meta_rbase(int y) {
  return (int)((unsigned)y >> 24);
}
__host__ __device__ __forceinline__ int popc8(unsigned m) {
#ifdef __CUDA_ARCH__
  return __popc(m);
#else
  return __builtin_popcount(m);
#endif
}
struct SIdx {
  int64_t f;  // F / W index of view 0 (view v at f + v * pitch)
  int64_t m;  // M index
  int pitch;  // distance between views
};
// store position of slot c of list block i (its lmeta y word and leaf mask)
__host__ __device__ __forceinline__ SIdx sidx(const SDesc& d, int64_t i, int c,
                                              int y, unsigned mask) {
  const int64_t t = i >> 5;
  const int64_t base = t * d.nvp * 256;
  if (!d.packed) {
    const int r = (int)((i & 31) << 3) + c;
    return {base + r, t * 256 + r, 256};
  }
  const int r = meta_rbase(y) + popc8(mask & ((1u << c) - 1u));
  return {base + (int64_t)(r / kChunk) * d.nvp * kChunk + (r % kChunk),
          t * 256 + r,
          kChunk};
}

// spread the low 21 bits of v to every third bit
__host__ __device__ __forceinline__ uint64_t spread3(uint64_t v) {
  v &= 0x1fffff;
  v = (v | (v << 32)) & 0x1f00000000ffffULL;
  v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
  v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
  v = (v | (v << 2)) & 0x1249249249249249ULL;
  return v;
}
// x-major Morton key: the child index c = x<<2|y<<1|z at every level, so
// ascending keys are the reference's canonical leaf order (octree.py:168-181)
__host__ __device__ __forceinline__ uint64_t morton3(uint32_t x, uint32_t y,
                                                     uint32_t z) {
  return (spread3(x) << 2) | (spread3(y) << 1) | spread3(z);
}

// depth-first pre-order position (parents before children, children in
// visit order) of a cell: (first finest key << 5) | level
__host__ __device__ __forceinline__ uint64_t preorder_key(int L, int x, int y,
                                                          int z, int d_max,
                                                          bool reverse) {
  if (reverse) {
    int m = (1 << L) - 1;
    x = m - x;
    y = m - y;
    z = m - z;
  }
  uint64_t first = morton3(x, y, z) << (3 * (d_max - L));
  return (first << 5) | (uint64_t)L;
}
// post-order position (children before parents): (last finest key << 5) |
// (31 - level)
__host__ __device__ __forceinline__ uint64_t postorder_key(int L, int x, int y,
                                                           int z, int d_max,
                                                           bool reverse) {
  if (reverse) {
    int m = (1 << L) - 1;
    x = m - x;
    y = m - y;
    z = m - z;
  }
  uint64_t last = ((morton3(x, y, z) + 1) << (3 * (d_max - L))) - 1;
  return (last << 5) | (uint64_t)(31 - L);
}

// deepest node at level <= L on the root path of cell (x,y,z)@L
// (reference octree.py:148-166, _kernels.pyx:193-202)
__device__ __forceinline__ int32_t descend(const int32_t* __restrict__ child,
                                           int L, int x, int y, int z,
                                           int* lvl_out = nullptr) {
  int32_t n = 0;
  int l = 0;
  for (; l < L; ++l) {
    int32_t b = __ldg(child + n);
    if (b < 0) break;
    int s = L - l - 1;
    n = b + octant(x >> s, y >> s, z >> s);
  }
  if (lvl_out) *lvl_out = l;
  return n;
}

// the view-tree nodes of cell (x,y,z)@L for views v = q*32 + lane, q < NCH
// (descend() per view), the NCH root descents advanced in lock-step so their
// dependent loads overlap (one load latency per level instead of NCH); -1
// for views past n
template <int NCH>
__device__ __forceinline__ void descend_views(const int32_t* const* vchild,
                                              int n, int L, int x, int y,
                                              int z, int lane,
                                              int32_t (&nd)[NCH]) {
  const int32_t* ch[NCH];
  unsigned live = 0;
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    const int v = q * 32 + lane;
    nd[q] = v < n ? 0 : -1;
    ch[q] = v < n ? vchild[v] : nullptr;
    if (v < n) live |= 1u << q;
  }
  for (int l = 0; l < L && live; ++l) {
    const int sh = L - l - 1;
    const int oc = octant(x >> sh, y >> sh, z >> sh);
    int32_t b[NCH];
#pragma unroll
    for (int q = 0; q < NCH; ++q) b[q] = (live >> q) & 1u ? __ldg(ch[q] + nd[q]) : -1;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      if (!((live >> q) & 1u)) continue;
      if (b[q] < 0)
        live &= ~(1u << q);
      else
        nd[q] = b[q] + oc;
    }
  }
}

// neighbour-table direction of a parent-level block offset (ox,oy,oz):
// faces -x +x -y +y -z +z, then the six edge offsets the 13-point stencil
// reaches: (-x+y) (-x+z) (+x-y) (-y+z) (+x-z) (+y-z); -1 = never used
__host__ __device__ __forceinline__ int nbr_dir(int ox, int oy, int oz) {
  const int nz = (ox != 0) + (oy != 0) + (oz != 0);
  if (nz == 1) return ox ? (ox < 0 ? 0 : 1) : oy ? (oy < 0 ? 2 : 3)
                                                 : (oz < 0 ? 4 : 5);
  if (nz != 2) return -1;
  if (oz == 0) return ox == -oy ? (ox < 0 ? 6 : 8) : -1;   // (-x+y) (+x-y)
  if (oy == 0) return ox == -oz ? (ox < 0 ? 7 : 10) : -1;  // (-x+z) (+x-z)
  return oy == -oz ? (oy < 0 ? 9 : 11) : -1;               // (-y+z) (+y-z)
}

// (ox,oy,oz) of each of the 12 table directions
__host__ __device__ __forceinline__ void dir_offset(int d, int& ox, int& oy,
                                                    int& oz) {
  constexpr int kOff[12][3] = {{-1, 0, 0}, {1, 0, 0},  {0, -1, 0}, {0, 1, 0},
                               {0, 0, -1}, {0, 0, 1},  {-1, 1, 0}, {-1, 0, 1},
                               {1, -1, 0}, {0, -1, 1}, {1, 0, -1}, {0, 1, -1}};
  ox = kOff[d][0];
  oy = kOff[d][1];
  oz = kOff[d][2];
}

struct PassParams {
  int d_max;
  double lam, eps2, gamma, xi, tau_s, tau_j;
  int clamp;
  int reverse;
};

// per-view tree pools as device arrays of device pointers
struct ViewSet {
  const float* const* val;
  const float* const* w;
  const int32_t* const* child;
  int n;
};

}  // namespace octf
