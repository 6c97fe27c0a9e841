#include <cstdio>
// Solver-context structure rebuild: level lists, leaf-block list, neighbour
// tables, per-leaf sample gather and the free-list mirror.
//
// The reference recomputes neighbours by descending from the root on every
// access (_kernels.pyx:193-202, 16 descents per node per pass).  Here the
// descents happen once per structure: each leaf block (8 sibling leaves, the
// reference's contiguous child block) gets a 12-entry table of the blocks or
// coarser leaves that hold its 13-point stencil, and each leaf gets its N
// per-view samples (the reference's per-view cursors, _kernels.pyx:265-273)
// gathered into a coalesced [view][leaf] store.
#include <chrono>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "octf_ctx.h"
#include "sample_sort.cuh"

namespace octf {

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(kECuda, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// keep freed stream-ordered allocations cached in the default pool (once)
// the device's default stream-ordered pool keeps freed memory (no release
// threshold), so DevBuf scratch is not remapped on every call: the input
// stage's per-view GB-sized pyramids cost ~0.2 s per view without it
void pool_keep() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if (done[dev & 63]) return;
  done[dev & 63] = true;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
}

Ctx::Ctx() {
  pool_keep();
  const char* fg = std::getenv("OCTF_FULL_GATHER");
  no_regather = fg && fg[0] == '1';
  const char* fe = std::getenv("OCTF_FORCE_ELL");  // tests: ELL from 33 views
  force_ell = fe && fe[0] == '1';
  const char* lj = std::getenv("OCTF_LEVEL_JOINS");  // A/B switch
  coop_off = lj && lj[0] == '1';
  const char* lw = std::getenv("OCTF_COOP_WALK");  // A/B switch
  walk_coop = lw && lw[0] == '1';
  const char* pm = std::getenv("OCTF_PHASES");  // rebuild phase marks
  phase_marks = pm && pm[0] == '1';
  const char* fp = std::getenv("OCTF_NO_FUSED_PARENT");  // A/B switch
  fuse_off = fp && fp[0] == '1';
  const char* nm = std::getenv("OCTF_NO_MORTON");  // A/B switch
  no_morton = nm && nm[0] == '1';
  OCTF_CUDA(cudaMallocHost((void**)&h_counters, 64 * sizeof(int32_t)));
  OCTF_CUDA(cudaMallocHost((void**)&h_scalar, 8 * sizeof(double)));
}
Ctx::~Ctx() {
  if (h_counters) cudaFreeHost(h_counters);
  if (h_scalar) cudaFreeHost(h_scalar);
  for (auto& e : tev)
    if (e) cudaEventDestroy(e);
  for (auto& e : pev) cudaEventDestroy(e);
  for (auto& e : tile_ev) cudaEventDestroy(e);
}

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(int64_t n, int per_thread = 1) {
  int64_t t = (n + per_thread - 1) / per_thread;
  int64_t g = (t + kThreads - 1) / kThreads;
  return (unsigned)(g < 1 ? 1 : g);
}

__device__ __forceinline__ void slot_cell(int32_t b, int c, uint64_t pc,
                                          int& x, int& y, int& z) {
  if (b == 0) {
    x = y = z = 0;
    return;
  }
  int L, px, py, pz;
  unpack_cell(pc, L, px, py, pz);
  x = 2 * px + ((c >> 2) & 1);
  y = 2 * py + ((c >> 1) & 1);
  z = 2 * pz + (c & 1);
}

// one level of the top-down walk: every inner slot of a level-L block emits
// its child block into the level-(L+1) list
__global__ void k_expand(const int32_t* __restrict__ child,
                         const int32_t* __restrict__ blocks, int64_t nblk,
                         int L, int64_t used, int8_t* blevel, uint64_t* bcoord,
                         int32_t* bparent, int32_t* next, int32_t* counter,
                         int32_t* bad) {
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = gid >> 3;
  int c = (int)(gid & 7);
  if (i >= nblk) return;
  int32_t b = blocks[i];
  if (b == 0 && c != 0) return;
  int32_t s = b + c;
  int32_t nb = child[s];
  if (nb < 0) return;
  if (nb + 8 > used || (nb & 7) != 1) {
    atomicExch(bad, 1);
    return;
  }
  int x, y, z;
  slot_cell(b, c, bcoord[block_id(b)], x, y, z);
  int k = block_id(nb);
  blevel[k] = (int8_t)(L + 1);
  bcoord[k] = pack_cell(L, x, y, z);
  bparent[k] = s;
  int pos = atomicAdd(counter, 1);
  next[pos] = nb;
}

// positions claimed by the threads of a CTA with one atomic per CTA on the
// shared counter (per-thread or per-warp atomics on one address serialise
// in L2: the level walk of a 60M-node tree spent ~0.3 ms on them): the
// first of `cnt` consecutive positions (any value when cnt == 0).  Every
// thread of the CTA must call it.
__device__ __forceinline__ int64_t cta_alloc_n(int cnt, int32_t* global) {
  __shared__ int s_warp[kThreads / 32];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = cnt;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      const int t = s_warp[k];
      s_warp[k] = acc;
      acc += t;
    }
    s_base = acc ? atomicAdd(global, acc) : 0;
  }
  __syncthreads();
  const int64_t r = (int64_t)s_base + s_warp[w] + (incl - cnt);
  __syncthreads();
  return r;
}

// one level of the walk without a host round trip: the level's range comes
// from device counters (dcnt, doff), the next level's start is written by
// thread 0; a fixed grid strides over the level (its size is only known on
// the device), CTA-uniform so the slots of a CTA are claimed together.
// Lists, counters and cells written by the level above are read past L1
// (volatile / __ldcg): in the all-level kernel another CTA wrote them.
__device__ __forceinline__ void expand_level(
    const int32_t* __restrict__ child, int32_t* lvl_blocks, int L, int64_t used,
    int64_t cap_blocks, int8_t* blevel, uint64_t* bcoord, int32_t* bparent,
    int32_t* dcnt, int32_t* doff, int32_t* bad) {
  const int64_t n = *(volatile int32_t*)(dcnt + L);
  const int64_t off = *(volatile int32_t*)(doff + L);
  const int64_t next = off + n;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) doff[L + 1] = (int32_t)next;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // a thread per block of the level: its inner children claim consecutive
  // positions of the next level together (one atomic per CTA and step)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
       base += stride) {
    const int64_t i = base + threadIdx.x;
    int32_t b = 0;
    int32_t nbs[8];
    unsigned inner = 0;
    if (i < n) {
      b = __ldcg(lvl_blocks + off + i);
      const int nc = b == 0 ? 1 : 8;
      for (int c = 0; c < 8; ++c) {
        nbs[c] = c < nc ? child[b + c] : -1;
        if (nbs[c] >= 0) {
          if (nbs[c] + 8 > used || (nbs[c] & 7) != 1)
            atomicExch(bad, 1);
          else
            inner |= 1u << c;
        }
      }
    }
    int64_t pos = next + cta_alloc_n(__popc(inner), dcnt + L + 1);
    if (!inner) continue;
    const uint64_t pc = __ldcg(bcoord + block_id(b));
    for (int c = 0; c < 8; ++c) {
      if (!((inner >> c) & 1u)) continue;
      const int32_t nb = nbs[c];
      int x, y, z;
      slot_cell(b, c, pc, x, y, z);
      const int k = block_id(nb);
      blevel[k] = (int8_t)(L + 1);
      bcoord[k] = pack_cell(L, x, y, z);
      bparent[k] = b + c;
      if (pos >= cap_blocks) {
        atomicExch(bad, 1);
      } else {
        lvl_blocks[pos] = nb;
      }
      ++pos;
    }
  }
}

__global__ void k_expand_dev(const int32_t* __restrict__ child,
                             int32_t* lvl_blocks, int L, int64_t used,
                             int64_t cap_blocks, int8_t* blevel,
                             uint64_t* bcoord, int32_t* bparent, int32_t* dcnt,
                             int32_t* doff, int32_t* bad) {
  expand_level(child, lvl_blocks, L, used, cap_blocks, blevel, bcoord, bparent,
               dcnt, doff, bad);
}

// every level in one cooperative launch (grid barrier between levels): the
// nine to twelve tiny launches of the per-level walk cost more in launch
// gaps than in work on a restructuring pass
__global__ void __launch_bounds__(kThreads)
k_expand_all(const int32_t* __restrict__ child, int32_t* lvl_blocks, int d_max,
             int64_t used, int64_t cap_blocks, int8_t* blevel,
             uint64_t* bcoord, int32_t* bparent, int32_t* dcnt, int32_t* doff,
             int32_t* bad) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  for (int L = 0; L < d_max; ++L) {
    expand_level(child, lvl_blocks, L, used, cap_blocks, blevel, bcoord,
                 bparent, dcnt, doff, bad);
    grid.sync();
    if (*(volatile int32_t*)(dcnt + L + 1) == 0) {
      // no deeper blocks: the remaining offsets all equal this level's end
      if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int q = L + 2; q <= d_max; ++q)
          doff[q] = *(volatile int32_t*)(doff + L + 1);
      break;
    }
  }
}

// levels [0, l1) in one single-CTA launch (a level L < 5 has at most 8^(L-1)
// blocks: the CTA strides over them), barrier between levels
__global__ void __launch_bounds__(kThreads)
k_expand_top(const int32_t* __restrict__ child, int32_t* lvl_blocks, int l1,
             int64_t used, int64_t cap_blocks, int8_t* blevel,
             uint64_t* bcoord, int32_t* bparent, int32_t* dcnt, int32_t* doff,
             int32_t* bad) {
  // the root entry of the walk (block id 0 = the root slot alone, level 0,
  // cell 0; one block at level 0): written here instead of by four small
  // host-to-device copies per rebuild
  if (threadIdx.x == 0) {
    blevel[0] = 0;
    bcoord[0] = 0;
    lvl_blocks[0] = 0;
    dcnt[0] = 1;
  }
  __threadfence();
  __syncthreads();
  for (int L = 0; L < l1; ++L) {
    expand_level(child, lvl_blocks, L, used, cap_blocks, blevel, bcoord,
                 bparent, dcnt, doff, bad);
    __threadfence();
    __syncthreads();
  }
}

// add a per-thread count to a global counter with one atomic per CTA
// (per-warp atomics on one address serialised in L2: ~0.2 ms for the 250k
// warps of a 7M-leaf list).  Every thread of the CTA must call it.
__device__ __forceinline__ void cta_count_add(int cnt, int32_t* global) {
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd_block(&s_cnt, cnt);
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt) atomicAdd(global, s_cnt);
}

// grid of at most one wave of kThreads CTAs (grid-stride kernels)
static unsigned wave_grid(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return (unsigned)(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
}

__global__ void k_leaf_flags(const int32_t* __restrict__ child,
                             const int32_t* __restrict__ blocks, int64_t nblk,
                             uint8_t* flags, int32_t* nleaves) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int n = 0;
  if (i < nblk) {
    const int32_t b = blocks[i];
    if (b == 0) {
      n = child[0] < 0;
    } else {
      for (int c = 0; c < 8; ++c) n += child[b + c] < 0;
    }
    flags[i] = n > 0;
  }
  cta_count_add(n, nleaves);
}

// per leaf block: packed (level, parent cell) and the 12 neighbour refs.
// ref >= 0: base slot of the same-level block holding that neighbour octet;
// ref <= -2: node -(ref+2), a coarser leaf covering it; kNone: outside.
__device__ __forceinline__ void leaf_table_entry(
    const int32_t* __restrict__ child, const int32_t* __restrict__ lblocks,
    const int8_t* __restrict__ blevel, const uint64_t* __restrict__ bcoord,
    const int32_t* __restrict__ bparent, uint64_t* lkey, int4* lmeta,
    int32_t* lpar, int32_t* nbr, int64_t i, int d) {
  int32_t b = lblocks[i];
  if (b < 0) {  // hole of a patched list: no active slot
    if (d == 0) {
      lkey[i] = 0;
      lmeta[i] = make_int4(0, 0, 0, pack_meta_w(0, 0u, 0));
      lpar[i] = -1;
    }
    nbr[i * 12 + d] = kNone;
    return;
  }
  int k = block_id(b);
  int L = b == 0 ? 0 : blevel[k];
  int pL, px, py, pz;
  unpack_cell(bcoord[k], pL, px, py, pz);
  if (b == 0) px = py = pz = 0;
  if (d == 0) {
    lkey[i] = pack_cell(L, px, py, pz);
    unsigned mask = 0;
    if (b == 0)
      mask = child[0] < 0 ? 1u : 0u;
    else
      for (int c = 0; c < 8; ++c) mask |= (child[b + c] < 0 ? 1u : 0u) << c;
    lmeta[i] = make_int4(b, px, py, pack_meta_w(pz, mask, L));
    lpar[i] = b == 0 ? -1 : bparent[k];
  }
  int32_t ref = kNone;
  if (b != 0) {
    int ox, oy, oz;
    dir_offset(d, ox, oy, oz);
    int qx = px + ox, qy = py + oy, qz = pz + oz;
    int m = 1 << (L - 1);
    if (qx >= 0 && qy >= 0 && qz >= 0 && qx < m && qy < m && qz < m) {
      int lq;
      int32_t q = descend(child, L - 1, qx, qy, qz, &lq);
      int32_t qb = child[q];
      ref = (lq == L - 1 && qb >= 0) ? qb : -q - 2;
    }
  }
  nbr[i * 12 + d] = ref;
}

__global__ void k_leaf_tables(const int32_t* __restrict__ child,
                              const int32_t* __restrict__ lblocks, int64_t nlb,
                              const int8_t* __restrict__ blevel,
                              const uint64_t* __restrict__ bcoord,
                              const int32_t* __restrict__ bparent,
                              uint64_t* lkey, int4* lmeta, int32_t* lpar,
                              int32_t* nbr, const int32_t* __restrict__ sel,
                              const int32_t* __restrict__ nsel) {
  // incremental update: only the `*nsel` entries listed in `sel` (the count
  // stays on the device: the grid strides over it, no host round trip)
  if (nsel) nlb = *nsel;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       gid < nlb * 12; gid += (int64_t)gridDim.x * blockDim.x)
    leaf_table_entry(child, lblocks, blevel, bcoord, bparent, lkey, lmeta,
                     lpar, nbr, sel ? sel[gid / 12] : gid / 12,
                     (int)(gid % 12));
}


// ---- view lookups by level (replaces a root descent per leaf and view):
// vm[y][s] = the node of view v0+y answering at slot s's cell and level,
// filled top-down: a slot's node is its parent's node's child c if that
// node has children, else the parent's node (descend() semantics,
// _kernels.pyx:265-273 cursors).  One load per (node, view) instead of one
// per level.
__global__ void k_vmap_level(const int32_t* __restrict__ blocks, int64_t nblk,
                             const int32_t* __restrict__ bparent, ViewSet vs,
                             int v0, int64_t cap, int32_t* vm) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  if (i >= nblk) return;
  const int y = blockIdx.y;
  const int32_t b = blocks[i];
  const int32_t p = bparent[block_id(b)];
  int32_t* m = vm + (int64_t)y * cap;
  const int32_t vp = m[p];
  const int32_t vc = __ldg(vs.child[v0 + y] + vp);
  m[b + c] = vc >= 0 ? vc + c : vp;
}

// ELL through the view map: pass 1 counts observed views per slot, pass 2
// appends them in view order at the slot's running row (one thread per slot
// per chunk: no atomics, order = view order)
__global__ void k_vcount(const int32_t* __restrict__ ucs,
                         const int32_t* __restrict__ lblocks, int64_t nlb,
                         ViewSet vs, int v0, int nc, int64_t cap,
                         const int32_t* __restrict__ vm, int32_t* cnt) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  if (i >= nlb) return;
  const int32_t b = lblocks[i];
  if (!(b >= 0 && !(b == 0 && c != 0) && ucs[b + c] < 0)) return;
  int k = 0;
  for (int y = 0; y < nc; ++y)
    k += __ldg(vs.w[v0 + y] + vm[(int64_t)y * cap + b + c]) != 0.f;
  cnt[gid] += k;
}

__global__ void k_vput(const int32_t* __restrict__ ucs,
                       const int32_t* __restrict__ lblocks, int64_t nlb,
                       ViewSet vs, int v0, int nc, int64_t cap,
                       const int32_t* __restrict__ vm,
                       const int64_t* __restrict__ tileOff, int32_t* cur,
                       float* F, float* W) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  if (i >= nlb) return;
  const int32_t b = lblocks[i];
  if (!(b >= 0 && !(b == 0 && c != 0) && ucs[b + c] < 0)) return;
  int r = cur[gid];
  for (int y = 0; y < nc; ++y) {
    const int32_t n = vm[(int64_t)y * cap + b + c];
    const float w = __ldg(vs.w[v0 + y] + n);
    if (w != 0.f) {
      F[ell_idx(tileOff, gid, r)] = __ldg(vs.val[v0 + y] + n);
      W[ell_idx(tileOff, gid, r)] = w;
      ++r;
    }
  }
  cur[gid] = r;
}

// rows [cur, K) of every slot (all rows of non-leaf slots) to zero
__global__ void k_ell_pad(const int32_t* __restrict__ cur, int64_t nslot,
                          const int32_t* __restrict__ tileK,
                          const int64_t* __restrict__ tileOff, float* F,
                          float* W) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslot) return;
  const int K = tileK[s >> 8];
  for (int r = cur[s]; r < K; ++r) {
    F[ell_idx(tileOff, s, r)] = 0.f;
    W[ell_idx(tileOff, s, r)] = 0.f;
  }
}

// samples of the list's leaf slots from the view map (dense layout)
__global__ void k_vgather(const int32_t* __restrict__ ucs,
                          const int32_t* __restrict__ lblocks, int64_t nlb,
                          ViewSet vs, int v0, int64_t cap,
                          const int32_t* __restrict__ vm, float* F, float* W,
                          int32_t* nonbin, const int4* __restrict__ lmeta,
                          SDesc sd) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  if (i >= nlb) return;
  const int y = blockIdx.y;
  const int32_t b = lblocks[i];
  // the list's (possibly rank-restricted) leaf mask
  const int4 mt = lmeta[i];
  const unsigned mask = ((unsigned)mt.w >> 19) & 0xffu;
  const bool active = b >= 0 && !(b == 0 && c != 0) && ucs[b + c] < 0 &&
                      ((mask >> c) & 1u);
  if (!active) return;
  const int32_t n = vm[(int64_t)y * cap + b + c];
  const float f = __ldg(vs.val[v0 + y] + n);
  const float w = __ldg(vs.w[v0 + y] + n);
  const SIdx q = sidx(sd, i, c, mt.y, mask);
  F[q.f + (int64_t)(v0 + y) * q.pitch] = f;
  W[q.f + (int64_t)(v0 + y) * q.pitch] = w;
  // flags: bit 0 a weight other than 0/1, bit 1 a zero weight on a leaf
  if (w != 0.f && w != 1.f) atomicOr(nonbin, 1);
  if (w == 0.f) atomicOr(nonbin, 2);
}

// per (leaf, view) from caller-supplied per-slot arrays [view][cap]
// (W null: every sample has weight 1)
__global__ void k_gather_slots(const int32_t* __restrict__ ucs,
                               const int32_t* __restrict__ lblocks, int64_t nlb,
                               const float* __restrict__ Fs,
                               const float* __restrict__ Ws, int64_t cap,
                               int nv, float* F, float* W, int32_t* nonbin,
                               const int4* __restrict__ lmeta, SDesc sd) {
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = gid >> 3;
  int c = (int)(gid & 7);
  if (i >= nlb) return;
  int32_t b = lblocks[i];
  // only the list's (possibly rank-restricted) leaves hold samples
  const int4 mt = lmeta[i];
  const unsigned mask = ((unsigned)mt.w >> 19) & 0xffu;
  const bool active = b >= 0 && !(b == 0 && c != 0) && ucs[b + c] < 0 &&
                      ((mask >> c) & 1u);
  if (!active) return;
  const SIdx q = sidx(sd, i, c, mt.y, mask);
  int flag = 0;
  for (int v = 0; v < nv; ++v) {
    const float f = Fs[(int64_t)v * cap + b + c];
    const float w = Ws ? Ws[(int64_t)v * cap + b + c] : 1.f;
    flag |= (w != 0.f && w != 1.f) ? 1 : 0;
    flag |= w == 0.f ? 2 : 0;
    F[q.f + (int64_t)v * q.pitch] = f;
    W[q.f + (int64_t)v * q.pitch] = w;
  }
  if (flag) atomicOr(nonbin, flag);
}

// ---- stable leaf-block list (ctx_list_update) ----
__device__ __forceinline__ unsigned leaf_mask_of(const int32_t* child,
                                                 int32_t b) {
  if (b == 0) return child[0] < 0 ? 1u : 0u;
  unsigned m = 0;
  for (int c = 0; c < 8; ++c) m |= (child[b + c] < 0 ? 1u : 0u) << c;
  return m;
}

// listed blocks that were freed or hold no leaf any more become holes; the
// previous leaf masks are kept for the sample update.  A listed block that
// is still live is the same block at the same cell: live blocks never move,
// and a block freed by a pass is reused only by a later pass.
__global__ void k_list_mark(int32_t* lblocks, const int4* __restrict__ lmeta,
                            int64_t n, const int32_t* __restrict__ child,
                            const int8_t* __restrict__ blevel, int32_t* lpos,
                            uint8_t* oldmask, int32_t* nholes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t b = lblocks[i];
  if (b < 0) {
    oldmask[i] = 0;
    return;
  }
  int pz, L;
  unsigned om;
  unpack_meta_w(lmeta[i].w, pz, om, L);
  oldmask[i] = (uint8_t)om;
  const int k = block_id(b);
  const unsigned nm = blevel[k] >= 0 ? leaf_mask_of(child, b) : 0u;
  if (!nm) {
    lblocks[i] = -1;
    lpos[k] = -1;
    atomicAdd(nholes, 1);
  }
}

// list entries whose tables must be recomputed after a patch: appended
// ones, new holes, changed leaf masks, and entries whose neighbour refs went
// stale -- a same-level block that was freed, or a coarser leaf that was
// split or whose block was freed (a live block never moves, so every other
// ref still answers the same root descent)
__global__ void k_table_dirty(const int32_t* __restrict__ lblocks, int64_t n,
                              int64_t nold, const uint8_t* __restrict__ oldmask,
                              const int32_t* __restrict__ child,
                              const int8_t* __restrict__ blevel,
                              const int32_t* __restrict__ nbr, int32_t* out,
                              int32_t* cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t b = lblocks[i];
  bool d = i >= nold;
  if (!d) {
    if (b < 0) {
      d = oldmask[i] != 0;  // a hole since this patch
    } else {
      d = leaf_mask_of(child, b) != oldmask[i];
      if (!d) {
        // the 12 refs as three 16 B loads and their checks' loads issued
        // together (independent), not one dependent round trip per ref
        const int4* n4 = reinterpret_cast<const int4*>(nbr + i * 12);
        const int4 a0 = n4[0], a1 = n4[1], a2 = n4[2];
        const int32_t r[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y,
                               a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
        int8_t lv[12];
        int32_t ch[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          const int32_t q = r[k] >= 0 ? r[k] : (r[k] <= -2 ? -r[k] - 2 : -1);
          lv[k] = q >= 0 ? blevel[block_id(q)] : 0;
          ch[k] = r[k] <= -2 ? child[q] : -1;
        }
#pragma unroll
        for (int k = 0; k < 12; ++k)
          d |= (r[k] >= 0 || r[k] <= -2) && (lv[k] < 0 || ch[k] >= 0);
      }
    }
  }
  if (d) out[atomicAdd(cnt, 1)] = (int32_t)i;
}

// live leaf blocks not in the list yet
__global__ void k_list_new(const int32_t* __restrict__ blocks, int64_t total,
                           const int32_t* __restrict__ child,
                           const int32_t* __restrict__ lpos, int32_t* out,
                           int32_t* cnt) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= total) return;
  const int32_t b = blocks[j];
  if (lpos[block_id(b)] < 0 && leaf_mask_of(child, b))
    out[atomicAdd(cnt, 1)] = b;
}

__global__ void k_list_put(const int32_t* __restrict__ in, int64_t a,
                           int64_t base, int32_t* lblocks, int32_t* lpos) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a) return;
  const int32_t b = in[r];
  lblocks[base + r] = b;
  lpos[block_id(b)] = (int32_t)(base + r);
}

__global__ void k_set_lpos(const int32_t* __restrict__ lblocks, int64_t n,
                           int32_t* lpos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t b = lblocks[i];
  if (b >= 0) lpos[block_id(b)] = (int32_t)i;
}

// per slot of the patched list: a leaf that was a leaf at the same position
// keeps its samples; a new leaf is queued for k_gather_fresh
template <bool BINW>
__global__ void k_sample_update(const int32_t* __restrict__ lblocks,
                                const int4* __restrict__ lmeta, int64_t n,
                                int64_t nold,
                                const uint8_t* __restrict__ oldmask,
                                int64_t stride, float* F, float* W,
                                uint32_t* M, int32_t* fresh, int32_t* nfresh,
                                int32_t* nleaves) {
  // CTA-uniform grid-stride, a thread per list entry: one count atomic per
  // CTA at the end and one queue claim per CTA and step (cta_alloc_n)
  int cnt = 0;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
       base += step) {
    const int64_t i = base + threadIdx.x;
    unsigned add = 0;
    if (i < n) {
      const int32_t b = lblocks[i];
      if (b >= 0) {
        int pz, L;
        unsigned nm;
        unpack_meta_w(lmeta[i].w, pz, nm, L);
        cnt += __popc(nm);
        if (b == 0) nm &= 1u;  // the root's pseudo-block has one slot
        const unsigned was = i < nold ? oldmask[i] : 0u;
        add = nm & ~was;
      }
    }
    int64_t r = cta_alloc_n(__popc(add), nfresh);
    for (int c = 0; c < 8; ++c)
      if ((add >> c) & 1u) fresh[r++] = (int32_t)(i * 8 + c);
  }
  cta_count_add(cnt, nleaves);
  // (slots that stopped being leaves keep stale samples: kernels read the
  // samples of active leaves only)
}

// zero the store slots [from, to) (tile padding after the last entry)
template <bool BINW>
__global__ void k_zero_slots(int64_t from, int64_t to, int64_t stride,
                             float* F, float* W, uint32_t* M) {
  const int64_t s = from + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= to) return;
  for (int v = 0; v < stride; ++v) {
    F[samp_idx(s, v, stride)] = 0.f;
    if (!BINW) W[samp_idx(s, v, stride)] = 0.f;
  }
  if (BINW) M[s] = 0u;
}

// samples of the leaves k_sample_update queued: one warp per leaf, lanes over
// views, so each lane walks one root descent instead of one per view
template <bool BINW>
__global__ void k_gather_fresh(const int32_t* __restrict__ fresh,
                               const int32_t* __restrict__ nfresh,
                               const int4* __restrict__ lmeta, ViewSet vs,
                               int64_t stride, float* F, float* W, uint32_t* M,
                               int32_t* nonbin) {
  const int lane = threadIdx.x & 31;
  const int nw = (int)(gridDim.x * (blockDim.x >> 5));
  const int n = *nfresh;
  for (int k = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
       k < n; k += nw) {
    const int64_t s = fresh[k];
    const int4 m = lmeta[s >> 3];
    const int c = (int)(s & 7);
    const int32_t b = m.x;
    int L, pz;
    unsigned mask;
    unpack_meta_w(m.w, pz, mask, L);
    const int x = b == 0 ? 0 : 2 * meta_px(m.y) + ((c >> 2) & 1);
    const int y = b == 0 ? 0 : 2 * m.z + ((c >> 1) & 1);
    const int z = b == 0 ? 0 : 2 * pz + (c & 1);
    uint32_t bits = 0;
    int flag = 0;
    // the dense store holds <= 64 views: both chunks' descents in lock-step
    int32_t nd2[2];
    descend_views<2>(vs.child, vs.n, L, x, y, z, lane, nd2);
    for (int v0 = 0; v0 < stride; v0 += 32) {
      const int v = v0 + lane;
      float f = 0.f, w = 0.f;
      if (v < vs.n) {
        const int32_t nd = v0 == 0 ? nd2[0] : v0 == 32 ? nd2[1]
                                             : descend(vs.child[v], L, x, y, z);
        f = vs.val[v][nd];
        w = vs.w[v][nd];
        flag |= (w != 0.f && w != 1.f) ? 1 : 0;
        flag |= w == 0.f ? 2 : 0;
      }
      if (v < stride) {
        F[samp_idx(s, v, stride)] = f;
        if (!BINW) W[samp_idx(s, v, stride)] = w;
      }
      if (BINW) bits |= __ballot_sync(0xffffffffu, w != 0.f);
    }
    if (BINW && lane == 0) M[s] = bits;
    flag = __reduce_or_sync(0xffffffffu, flag);
    if (flag && lane == 0) atomicOr(nonbin, flag);
  }
}

// ---- ELL incremental update (stable list): k_ell_update classifies the
// slots like k_sample_update; fresh leaves gather with one warp each
__global__ void k_ell_update(const int32_t* __restrict__ lblocks,
                             const int4* __restrict__ lmeta, int64_t n,
                             int64_t nold, const uint8_t* __restrict__ oldmask,
                             const int32_t* __restrict__ tileK,
                             const int64_t* __restrict__ tileOff, float* F,
                             float* W, int32_t* fresh, int32_t* nfresh,
                             int32_t* nleaves) {
  // CTA-uniform grid-stride, a thread per list entry: one count atomic per
  // CTA at the end and one queue claim per CTA and step (cta_alloc_n)
  int cnt = 0;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
       base += step) {
    const int64_t i = base + threadIdx.x;
    unsigned add = 0;
    if (i < n) {
      const int32_t b = lblocks[i];
      if (b >= 0) {
        int pz, L;
        unsigned nm;
        unpack_meta_w(lmeta[i].w, pz, nm, L);
        cnt += __popc(nm);
        if (b == 0) nm &= 1u;  // the root's pseudo-block has one slot
        const unsigned was = i < nold ? oldmask[i] : 0u;
        add = nm & ~was;
      }
    }
    int64_t r = cta_alloc_n(__popc(add), nfresh);
    for (int c = 0; c < 8; ++c)
      if ((add >> c) & 1u) fresh[r++] = (int32_t)(i * 8 + c);
  }
  cta_count_add(cnt, nleaves);
  // (no zeroing: only active leaves' rows are ever read)
}

// one warp per queued leaf: views over lanes, observed ones compacted in
// view order by ballot; more than the tile's rows flags an overflow and
// queues the leaf in `redo` (the second attempt after the tile moves gathers
// only those).  The view-tree node of each view is found once (root
// descent) and kept in registers for the first 512 views.
constexpr int kFreshChunks = 16;
__global__ void k_ell_fresh(const int32_t* __restrict__ fresh,
                            const int32_t* __restrict__ nfresh,
                            const int4* __restrict__ lmeta, ViewSet vs,
                            const int32_t* __restrict__ tileK,
                            const int64_t* __restrict__ tileOff, float* F,
                            float* W, int32_t* overflow, int32_t* need,
                            int32_t* redo, int32_t* nredo) {
  const int lane = threadIdx.x & 31;
  const int nw = (int)(gridDim.x * (blockDim.x >> 5));
  const int n = *nfresh;
  for (int k = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
       k < n; k += nw) {
    const int64_t s = fresh[k];
    const int4 m = lmeta[s >> 3];
    const int c = (int)(s & 7);
    const int32_t b = m.x;
    int L, pz;
    unsigned mask;
    unpack_meta_w(m.w, pz, mask, L);
    const int x = b == 0 ? 0 : 2 * meta_px(m.y) + ((c >> 2) & 1);
    const int y = b == 0 ? 0 : 2 * m.z + ((c >> 1) & 1);
    const int z = b == 0 ? 0 : 2 * pz + (c & 1);
    const int K = tileK[s >> 8];
    int32_t nd[kFreshChunks];
    int j = 0;
    // count first: a leaf that does not fit leaves its tile untouched
    descend_views<kFreshChunks>(vs.child, vs.n, L, x, y, z, lane, nd);
#pragma unroll
    for (int q = 0; q < kFreshChunks; ++q) {
      if (q * 32 < vs.n) {
        const bool on = nd[q] >= 0 && vs.w[q * 32 + lane][nd[q]] != 0.f;
        j += __popc(__ballot_sync(0xffffffffu, on));
      }
    }
    for (int v0 = kFreshChunks * 32; v0 < vs.n; v0 += 32) {
      const int v = v0 + lane;
      bool on = false;
      if (v < vs.n) on = vs.w[v][descend(vs.child[v], L, x, y, z)] != 0.f;
      j += __popc(__ballot_sync(0xffffffffu, on));
    }
    if (j > K) {
      if (lane == 0) {
        atomicExch(overflow, 1);
        atomicMax(need + (s >> 8), j);
        if (redo) redo[atomicAdd(nredo, 1)] = (int32_t)s;
      }
      continue;
    }
    j = 0;
    auto put = [&](int v, int32_t node) {
      float f = 0.f, w = 0.f;
      if (v < vs.n) {
        f = vs.val[v][node];
        w = vs.w[v][node];
      }
      const unsigned on = __ballot_sync(0xffffffffu, w != 0.f);
      const int r = j + __popc(on & ((1u << lane) - 1u));
      if (w != 0.f && r < K) {
        F[ell_idx(tileOff, s, r)] = f;
        W[ell_idx(tileOff, s, r)] = w;
      }
      j += __popc(on);
    };
#pragma unroll
    for (int q = 0; q < kFreshChunks; ++q)
      if (q * 32 < vs.n) put(q * 32 + lane, nd[q]);
    for (int v0 = kFreshChunks * 32; v0 < vs.n; v0 += 32) {
      const int v = v0 + lane;
      put(v, v < vs.n ? descend(vs.child[v], L, x, y, z) : 0);
    }
    for (int r = j + lane; r < K; r += 32) {
      F[ell_idx(tileOff, s, r)] = 0.f;
      W[ell_idx(tileOff, s, r)] = 0.f;
    }
  }
}

__global__ void k_ell_offsets(const int64_t* __restrict__ scan, int64_t n,
                              int64_t total, int64_t* off) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) off[i] = total + scan[i];
}

// device-side move plan: rows of the bigger range of each overflowing tile
// (need + need/4 + 4 rows, as before), 0 for the others; rows[nt] = 0 for
// the scan; rows[nt + 1] accumulates the abandoned rows (ell_waste)
__global__ void k_ell_plan(const int32_t* __restrict__ need,
                           const int32_t* __restrict__ tileK, int64_t nt,
                           int64_t* rows, int32_t* mlist) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nt) return;
  if (t == nt) {
    rows[nt] = 0;
    return;
  }
  const int nd = need[t], k0 = tileK[t];
  const bool mv = nd > k0;
  rows[t] = mv ? (int64_t)(nd + nd / 4 + 4) * 256 : 0;
  if (mv) {
    atomicAdd(reinterpret_cast<unsigned long long*>(rows + nt + 1),
              (unsigned long long)k0 * 256);
    mlist[1 + atomicAdd(mlist, 1)] = (int32_t)t;  // the tiles to move
  }
}

// a CTA per overflowing tile (mlist[0] of them, listed from mlist[1]; the
// grid strides over the list): its rows move to [total + scan[t], ...) with
// the new rows zeroed, then its K and offset are switched
__global__ void k_ell_move_dev(const int32_t* __restrict__ mlist,
                               const int32_t* __restrict__ need,
                               int32_t* tileK, int64_t* tileOff,
                               const int64_t* __restrict__ scan, int64_t total,
                               float* F, float* W) {
  const int nm = mlist[0];
  for (int q = blockIdx.x; q < nm; q += gridDim.x) {
    const int64_t t = mlist[1 + q];
    const int nd = need[t], k0 = tileK[t];
    const int k1 = nd + nd / 4 + 4;
    const int64_t o0 = tileOff[t], o1 = total + scan[t];
    for (int64_t e = threadIdx.x; e < (int64_t)k1 * 256; e += blockDim.x) {
      const bool keep = e < (int64_t)k0 * 256;
      F[o1 + e] = keep ? F[o0 + e] : 0.f;
      W[o1 + e] = keep ? W[o0 + e] : 0.f;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tileK[t] = k1;
      tileOff[t] = o1;
    }
  }
}

// ---- ELL sample store (views > 32) ----

// k_ell_count for a few slots (tiles appended by a list patch): one warp
// per slot, views over lanes
__global__ void k_ell_count_warp(const int32_t* __restrict__ ucs,
                                 const int32_t* __restrict__ lblocks,
                                 int64_t nlb, const uint64_t* __restrict__ lkey,
                                 ViewSet vs, int32_t* cnt, int64_t slot0,
                                 int64_t slot1) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t s = slot0 + (int64_t)blockIdx.x * (blockDim.x >> 5) +
                   (threadIdx.x >> 5);
       s < slot1; s += nw) {
    const int64_t i = s >> 3;
    const int c = (int)(s & 7);
    const int32_t b = i < nlb ? lblocks[i] : -1;
    const bool active = b >= 0 && !(b == 0 && c != 0) && ucs[b + c] < 0;
    int k = 0;
    if (active) {
      int L, px, py, pz;
      unpack_cell(lkey[i], L, px, py, pz);
      const int x = b == 0 ? 0 : 2 * px + ((c >> 2) & 1);
      const int y = b == 0 ? 0 : 2 * py + ((c >> 1) & 1);
      const int z = b == 0 ? 0 : 2 * pz + (c & 1);
      for (int v0 = 0; v0 < vs.n; v0 += 32) {
        const int v = v0 + lane;
        bool on = false;
        if (v < vs.n) on = vs.w[v][descend(vs.child[v], L, x, y, z)] != 0.f;
        k += __popc(__ballot_sync(0xffffffffu, on));
      }
    }
    if (lane == 0) cnt[s] = k;
  }
}

// per tile: rows = max count of its 256 slots (one CTA of 256 per tile)
__global__ void k_ell_tilemax(const int32_t* __restrict__ cnt, int64_t n,
                              int64_t tile0, int32_t* tileK, int64_t* rowsz) {
  const int64_t t = tile0 + blockIdx.x;
  const int64_t s = t * 256 + threadIdx.x;
  int k = s < n ? cnt[s] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, o));
  __shared__ int wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = k;
  __syncthreads();
  if (threadIdx.x == 0) {
    int mx = 0;
    for (int q = 0; q < 8; ++q) mx = max(mx, wm[q]);
    tileK[t] = mx;
    rowsz[blockIdx.x] = (int64_t)mx * 256;
  }
}


// binary weights -> the bit-mask format, per leaf of the list
__global__ void k_masks(const float* __restrict__ W, const int4* __restrict__ lmeta,
                        int64_t nlb, int nv, SDesc sd, uint32_t* M) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  if (i >= nlb) return;
  const int4 mt = lmeta[i];
  const unsigned mask = ((unsigned)mt.w >> 19) & 0xffu;
  if (!((mask >> c) & 1u) || (mt.x == 0 && c != 0)) return;
  const SIdx q = sidx(sd, i, c, mt.y, mask);
  uint32_t m = 0;
  for (int v = 0; v < nv; ++v)
    m |= (W[q.f + (int64_t)v * q.pitch] != 0.f ? 1u : 0u) << v;
  M[q.m] = m;
}

// packed store (octf_common.cuh SDesc): one warp per tile of 32 leaf
// blocks; each block's first rank (exclusive scan of the leaf counts) into
// the top byte of lmeta.y; nonfull counts the tiles holding a block that is
// not 8 leaves (without one, ranks are slots and the plain layout is kept)
__global__ void k_pack_ranks(int4* lmeta, int64_t nlb, int64_t ntiles,
                             int32_t* nonfull) {
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  const int64_t i = t * 32 + lane;
  int4 m = make_int4(0, 0, 0, 0);
  unsigned mask = 0;
  if (i < nlb) {
    m = lmeta[i];
    mask = ((unsigned)m.w >> 19) & 0xffu;
    if (m.x == 0) mask &= 1u;  // the root's pseudo-block has one slot
  }
  const int cnt = __popc(mask);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (i < nlb) {
    m.y = meta_px(m.y) | ((incl - cnt) << 24);
    lmeta[i] = m;
  }
  const bool odd = i < nlb && mask != 0xffu;
  if (__any_sync(0xffffffffu, odd) && lane == 0) atomicAdd(nonfull, 1);
}

// Morton (depth-first pre-order) key of a leaf block: its parent cell's
__global__ void k_block_keys(const int32_t* __restrict__ lblocks, int64_t n,
                             const int8_t* __restrict__ blevel,
                             const uint64_t* __restrict__ bcoord, int d_max,
                             uint64_t* keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t b = lblocks[i];
  if (b == 0) {  // the root's pseudo-block
    keys[i] = 0;
    return;
  }
  const int k = block_id(b);
  int pL, px, py, pz;
  unpack_cell(bcoord[k], pL, px, py, pz);
  keys[i] = preorder_key(blevel[k] - 1, px, py, pz, d_max, false);
}

// the reference's canonical order (octree.py:168-181 leaves, :413-431
// serialize: depth-first pre-order, children in index order) as sort keys:
// every live node's preorder key (first finest Morton key << 5 | level) and
// slot, appended in any order (octf_node_order sorts them)
__global__ void k_node_keys(const int32_t* __restrict__ blocks, int64_t nblk,
                            const int8_t* __restrict__ blevel,
                            const uint64_t* __restrict__ bcoord,
                            const int32_t* __restrict__ child, int d_max,
                            int leaves_only, uint64_t* keys, int32_t* slots,
                            int32_t* count) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool on = false;
  uint64_t key = 0;
  int32_t s = 0;
  if (gid < nblk * 8) {
    const int32_t b = blocks[gid >> 3];
    const int c = (int)(gid & 7);
    if (b == 0) {  // the root's pseudo-block: slot 0 only
      on = c == 0 && (!leaves_only || child[0] < 0);
    } else {
      const int k = block_id(b);
      int pL, px, py, pz;
      unpack_cell(bcoord[k], pL, px, py, pz);
      s = b + c;
      on = !leaves_only || child[s] < 0;
      key = preorder_key(blevel[k], 2 * px + ((c >> 2) & 1),
                         2 * py + ((c >> 1) & 1), 2 * pz + (c & 1), d_max,
                         false);
    }
  }
  const unsigned q = __ballot_sync(0xffffffffu, on);
  int base = 0;
  if ((threadIdx.x & 31) == 0 && q) base = atomicAdd(count, __popc(q));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (on) {
    const int r = base + __popc(q & ((1u << (threadIdx.x & 31)) - 1u));
    keys[r] = key;
    slots[r] = s;
  }
}

// OCTF_ELL_STATS: per thread one 8-slot block of the per-slot counts
__global__ void k_ell_stats(const int32_t* __restrict__ cnt, int64_t nt,
                            unsigned long long* acc) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long obs = 0, blk = 0, tile = 0;
  if (b < nt * 32) {
    int mx = 0;
    for (int c = 0; c < 8; ++c) {
      obs += cnt[b * 8 + c];
      mx = max(mx, cnt[b * 8 + c]);
    }
    blk = 8ull * mx;
  }
  // per-tile max over the tile's 32 blocks (one warp = one tile)
  int tmx = (int)(blk / 8);
  for (int o = 16; o > 0; o >>= 1)
    tmx = max(tmx, __shfl_xor_sync(0xffffffffu, tmx, o));
  if ((threadIdx.x & 31) == 0) tile = 256ull * tmx;
  for (int o = 16; o > 0; o >>= 1) {
    obs += __shfl_xor_sync(0xffffffffu, obs, o);
    blk += __shfl_xor_sync(0xffffffffu, blk, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc, obs);
    atomicAdd(acc + 1, tile);
    atomicAdd(acc + 2, blk);
  }
}

__global__ void k_walk_free(const int32_t* __restrict__ child, int64_t head,
                            int64_t nmax, int32_t* chain, int32_t* count) {
  // single thread: follow the free list links (child[b] of a free block)
  int64_t n = 0;
  int64_t b = head;
  while (b >= 0 && n < nmax) {
    chain[n++] = (int32_t)b;
    b = child[b];
  }
  *count = (int32_t)n;
}

__global__ void k_reverse(const int32_t* in, int64_t n, int32_t* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[n - 1 - i] = in[i];
}

}  // namespace

// stream-ordered sorts with the context's persistent scratch (no
// allocation, no host sync: cudaMalloc/cudaFree per call used to dominate
// small restructuring passes)
void sort_u64_i32(Ctx& c, uint64_t* keys, int32_t* vals, int64_t n,
                  cudaStream_t st) {
  if (n <= 1) return;
  uint64_t* k2 = c.sort_k64.ensure(n);
  int32_t* v2 = c.sort_v32.ensure(n);
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, k2, vals, v2, (int)n,
                                  0, 64, st);
  c.cub_tmp.ensure(bytes);
  OCTF_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, bytes, keys, k2, vals,
                                            v2, (int)n, 0, 64, st));
  OCTF_CUDA(cudaMemcpyAsync(keys, k2, n * sizeof(uint64_t),
                            cudaMemcpyDeviceToDevice, st));
  OCTF_CUDA(cudaMemcpyAsync(vals, v2, n * sizeof(int32_t),
                            cudaMemcpyDeviceToDevice, st));
}

void sort_i32(Ctx& c, int32_t* keys, int64_t n, cudaStream_t st) {
  if (n <= 1) return;
  int32_t* k2 = c.sort_k32.ensure(n);
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys, k2, (int)n, 0, 32, st);
  c.cub_tmp.ensure(bytes);
  OCTF_CUDA(cub::DeviceRadixSort::SortKeys(c.cub_tmp.p, bytes, keys, k2,
                                           (int)n, 0, 32, st));
  OCTF_CUDA(cudaMemcpyAsync(keys, k2, n * sizeof(int32_t),
                            cudaMemcpyDeviceToDevice, st));
}

void ctx_free_stack(Ctx& c, const int32_t* child, const int64_t* state,
                    cudaStream_t st) {
  int64_t used = state[0];
  int64_t nmax = (used + 7) / 8 + 1;
  c.free_stack.ensure(nmax);
  c.nfree = 0;
  c.nfree_head = state[1];
  if (state[1] < 0) return;
  int32_t* chain = c.sort_k32.ensure(nmax);
  c.counters.ensure(64);
  k_walk_free<<<1, 1, 0, st>>>(child, state[1], nmax, chain, c.counters.p);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p, sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  int64_t n = c.h_counters[0];
  // stack order: bottom = last link, top = head
  if (n) k_reverse<<<grid_for(n), kThreads, 0, st>>>(chain, n, c.free_stack.p);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaStreamSynchronize(st));
  c.nfree = n;
}

void ph_start(Ctx& c, cudaStream_t st) {
  if (!c.timing || !c.phase_marks) return;
  OCTF_CUDA(cudaStreamSynchronize(st));
  c.ph_t0 = std::chrono::steady_clock::now();
}
void ph_mark(Ctx& c, int phase, cudaStream_t st) {
  if (!c.timing || !c.phase_marks) return;
  OCTF_CUDA(cudaStreamSynchronize(st));
  const auto now = std::chrono::steady_clock::now();
  c.t_ph[phase] +=
      std::chrono::duration<double, std::milli>(now - c.ph_t0).count();
  c.ph_t0 = now;
}

void ctx_prepare(Ctx& c, const int32_t* child, int64_t cap,
                 const int64_t* state, int d_max, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  ph_start(c, st);
  if (d_max < 0 || d_max > kMaxDepth)
    throw Error(kEDepth, "tree depth out of range");
  int64_t used = state[0];
  if (used < 1 || used > cap)
    throw Error(kEArg, "pool state is inconsistent with its capacity");
  int64_t nbid = block_id(used) + 1;
  // patch the leaf-block list in place when this rebuild follows our own
  // restructuring of the same pool (ctx_list_update)
  const bool incremental = !c.no_regather && !c.pack_opt && c.own_change &&
                           c.store_ok &&
                           c.list_full && c.nviews > 0 && !c.ext_F &&
                           c.child_key == child && c.cap == cap &&
                           c.d_max == d_max;
  c.own_change = false;
  c.store_ok = false;
  c.blevel.ensure(nbid);
  c.bcoord.ensure(nbid);
  c.bparent.ensure(nbid);
  c.lvl_blocks.ensure(nbid + 1);
  c.counters.ensure(64);
  OCTF_CUDA(cudaMemsetAsync(c.blevel.p, 0xff, nbid, st));
  c.lvl_off.assign(d_max + 2, 0);
  c.lvl_cnt.assign(d_max + 2, 0);
  // top-down walk, one launch per level, counts kept on the device and read
  // once at the end (counters: [0] bad link, [8..] counts, [8+d_max+2..]
  // offsets)
  c.counters.ensure(8 + 2 * (kMaxDepth + 2));
  int32_t* dcnt = c.counters.p + 8;
  int32_t* doff = dcnt + (d_max + 2);
  OCTF_CUDA(cudaMemsetAsync(c.counters.p, 0,
                            (8 + 2 * (d_max + 2)) * sizeof(int32_t), st));
  // the levels near the root in one single-CTA launch, a launch per level
  // below them
  const int l_top = c.walk_coop ? 0 : std::min(d_max, 5);
  {
    k_expand_top<<<1, kThreads, 0, st>>>(
        child, c.lvl_blocks.p, l_top, used, nbid + 1, c.blevel.p, c.bcoord.p,
        c.bparent.p, dcnt, doff, c.counters.p);
    OCTF_CUDA(cudaGetLastError());
  }
  if (c.walk_coop && d_max > 0) {
    // all levels in one cooperative launch (measured slower than the
    // launches below: cfg3 walk 0.10 -> 0.13 ms; kept for A/B)
    static int coop_per_dev[64] = {};
    int dev = 0;
    OCTF_CUDA(cudaGetDevice(&dev));
    int& coop_blocks = coop_per_dev[dev & 63];
    if (!coop_blocks) {
      int per_sm = 0, nsm = 0;
      OCTF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, k_expand_all, kThreads, 0));
      OCTF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount,
                                       dev));
      if (per_sm * nsm < 1) throw Error(kECuda, "walk: no resident CTA");
      coop_blocks = std::min(per_sm, 4) * nsm;
    }
    int32_t* lvl_blocks = c.lvl_blocks.p;
    int64_t cap_blocks = nbid + 1;
    int8_t* blevel = c.blevel.p;
    uint64_t* bcoord = c.bcoord.p;
    int32_t* bparent = c.bparent.p;
    int32_t* bad = c.counters.p;
    int dm = d_max;
    // a small tree does not need the whole wave (grid barriers cost by CTA)
    const int grid_blocks = (int)std::min<int64_t>(
        coop_blocks, std::max<int64_t>(1, (nbid + kThreads - 1) / kThreads));
    void* kargs[] = {(void*)&child, &lvl_blocks, &dm,     &used,
                     &cap_blocks,   &blevel,     &bcoord, &bparent,
                     &dcnt,         &doff,       &bad};
    OCTF_CUDA(cudaLaunchCooperativeKernel((const void*)k_expand_all,
                                          grid_blocks, kThreads, kargs, 0, st));
  }
  for (int L = l_top; L < d_max && !c.walk_coop; ++L) {
    // level L holds at most min(8^L, live blocks) blocks: a grid of at
    // most one wave strides over them
    const int64_t bound = L < 7 ? std::min<int64_t>(int64_t(1) << (3 * L), nbid)
                                : nbid;
    const int64_t wave = (int64_t)148 * 8 * kThreads;
    k_expand_dev<<<grid_for(std::min<int64_t>(bound, wave)), kThreads, 0,
                   st>>>(
        child, c.lvl_blocks.p, L, used, nbid + 1, c.blevel.p, c.bcoord.p,
        c.bparent.p, dcnt, doff, c.counters.p);
    OCTF_CUDA(cudaGetLastError());
  }
  OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p,
                            (8 + 2 * (d_max + 2)) * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  if (c.h_counters[0]) throw Error(kEArg, "corrupt child links in pool");
  int64_t total = 0;
  for (int L = 0; L <= d_max; ++L) {
    c.lvl_cnt[L] = c.h_counters[8 + L];
    c.lvl_off[L] = c.h_counters[8 + (d_max + 2) + L];
    total += c.lvl_cnt[L];
  }
  if (total > nbid) throw Error(kEArg, "corrupt child links in pool");
  c.nblocks = total;
  // a finest-level node must be a leaf
  // (checked implicitly: blocks at level d_max are never expanded)

  ph_mark(c, kPhWalk, st);
  const bool patched =
      incremental && ctx_list_update(c, child, total, nbid, st);
  if (!patched) {
    ctx_list_full(c, child, total, nbid, d_max, st);
    ph_mark(c, kPhFull, st);
  }

  c.smark.ensure(cap);
  OCTF_CUDA(cudaMemsetAsync(c.smark.p, 0, cap, st));
  // the free-list mirror survives our own restructuring (passes pop and
  // push it); walk the pool's linked free list only for a foreign pool
  if (!c.free_ok || c.child_key != child || c.nfree_head != state[1]) {
    ctx_free_stack(c, child, state, st);
    c.free_ok = true;
  }
  c.child_key = child;
  c.cap = cap;
  c.d_max = d_max;
  c.hstate[0] = state[0];
  c.hstate[1] = state[1];
  c.hstate[2] = state[2];
  c.valid = true;
  ph_mark(c, kPhTail, st);
  if (c.nviews > 0 && !patched && !c.defer_gather) {
    ctx_gather(c, st);
    ph_mark(c, kPhGather, st);
  }
  if (c.timing) {
    OCTF_CUDA(cudaStreamSynchronize(st));  // only for the timer
    c.t_prep_ms += std::chrono::duration<double, std::milli>(
                       std::chrono::steady_clock::now() - t0).count();
    ++c.n_prep;
  }
}

// the sorted leaf-block list of every live block holding a leaf, its tables
// and the block -> position map
void ctx_list_full(Ctx& c, const int32_t* child, int64_t total, int64_t nbid,
                   int d_max, cudaStream_t st) {
  // leaf blocks, ascending base slot
  uint8_t* flags = c.flags.ensure(total);
  c.lblocks.ensure(total);
  OCTF_CUDA(cudaMemsetAsync(c.counters.p, 0, 2 * sizeof(int32_t), st));
  k_leaf_flags<<<grid_for(total), kThreads, 0, st>>>(
      child, c.lvl_blocks.p, total, flags, c.counters.p + 1);
  OCTF_CUDA(cudaGetLastError());
  size_t bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, bytes, c.lvl_blocks.p, flags,
                             c.lblocks.p, c.counters.p, (int)total, st);
  c.cub_tmp.ensure(bytes);
  OCTF_CUDA(cub::DeviceSelect::Flagged(c.cub_tmp.p, bytes, c.lvl_blocks.p,
                                       flags, c.lblocks.p, c.counters.p,
                                       (int)total, st));
  OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p, 2 * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  c.nlb = c.h_counters[0];
  c.nleaves = c.h_counters[1];
  if (c.pack_opt && !c.defer_gather && !c.no_morton && c.nlb > 1) {
    // a frozen tree's list in Morton order of the blocks' parent cells
    // (depth-first pre-order): spatial neighbours of every level are
    // processed together, so their values are re-read from L2, not HBM
    uint64_t* keys = c.sort_k64.ensure(2 * c.nlb);
    int32_t* v2 = c.sort_k32.ensure(c.nlb);
    k_block_keys<<<grid_for(c.nlb), kThreads, 0, st>>>(
        c.lblocks.p, c.nlb, c.blevel.p, c.bcoord.p, d_max, keys);
    OCTF_CUDA(cudaGetLastError());
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys + c.nlb,
                                    c.lblocks.p, v2, (int)c.nlb, 0, 64, st);
    c.cub_tmp.ensure(bytes);
    OCTF_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, bytes, keys,
                                              keys + c.nlb, c.lblocks.p, v2,
                                              (int)c.nlb, 0, 64, st));
    OCTF_CUDA(cudaMemcpyAsync(c.lblocks.p, v2, c.nlb * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, st));
    c.list_morton = true;
  } else {
    sort_i32(c, c.lblocks.p, c.nlb, st);
    c.list_morton = false;
  }
  c.lkey.ensure(c.nlb);
  c.lmeta.ensure(c.nlb);
  c.lpar.ensure(c.nlb);
  c.nbr.ensure(c.nlb * 12);
  k_leaf_tables<<<grid_for(c.nlb * 12), kThreads, 0, st>>>(
      child, c.lblocks.p, c.nlb, c.blevel.p, c.bcoord.p, c.bparent.p,
      c.lkey.p, c.lmeta.p, c.lpar.p, c.nbr.p, nullptr, nullptr);
  OCTF_CUDA(cudaGetLastError());
  c.lpos.ensure(nbid);
  OCTF_CUDA(cudaMemsetAsync(c.lpos.p, 0xff, nbid * sizeof(int32_t), st));
  if (c.nlb)
    k_set_lpos<<<grid_for(c.nlb), kThreads, 0, st>>>(c.lblocks.p, c.nlb,
                                                     c.lpos.p);
  OCTF_CUDA(cudaGetLastError());
  c.lpos_n = nbid;
  c.nholes = 0;
  c.list_full = true;
}

// ELL store after a list patch: tiles appended by the patch get counts,
// rows and offsets after the existing store; kept leaves keep their rows,
// new leaves gather (a warp each); a leaf with more observed views than
// its tile's rows -> false (full rebuild).
static bool ell_list_samples(Ctx& c, int64_t nold, int64_t nnew,
                             const uint8_t* oldmask,
                             std::chrono::steady_clock::time_point t0,
                             cudaStream_t st) {
  const int64_t nt_old = c.ell_tiles;
  const int64_t nt_new = (nnew * 8 + kTileLeaves - 1) / kTileLeaves;
  int64_t total = c.ell_size;
  // compact (full rebuild) once abandoned rows pass half the store: with
  // many views a rebuild regathers every leaf's samples (cfg4 depth 9,
  // 300 views: 38 ms, ~100 passes' worth of the holes' cost)
  if (2 * c.ell_waste > total) return false;
  if (nt_new > nt_old) {
    int32_t* cnt = c.sort_k32.ensure(nt_new * 256 + 1);
    OCTF_CUDA(cudaMemsetAsync(cnt, 0, nt_new * 256 * sizeof(int32_t), st));
    // counts for the new tiles' slots (the list tables are current)
    const int64_t s0 = nt_old * 256, s1 = nnew * 8;
    if (s1 > s0)
      k_ell_count_warp<<<148 * 8, kThreads, 0, st>>>(
          c.child_key, c.lblocks.p, nnew, c.lkey.p, ctx_views(c), cnt, s0, s1);
    int64_t* rowsz =
        reinterpret_cast<int64_t*>(c.sort_k64.ensure(nt_new - nt_old + 1));
    c.tileK.grow_keep(nt_new + 1, nt_old, st);
    c.tileOff.grow_keep(nt_new + 1, nt_old + 1, st);
    k_ell_tilemax<<<(unsigned)(nt_new - nt_old), 256, 0, st>>>(
        cnt, nnew * 8, nt_old, c.tileK.p, rowsz);
    OCTF_CUDA(cudaMemsetAsync(rowsz + (nt_new - nt_old), 0, sizeof(int64_t),
                              st));
    int64_t* scan = reinterpret_cast<int64_t*>(c.app_buf.ensure(
        2 * (nt_new - nt_old + 1)));
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, rowsz, scan,
                                  (int)(nt_new - nt_old + 1), st);
    c.cub_tmp.ensure(bytes);
    OCTF_CUDA(cub::DeviceScan::ExclusiveSum(c.cub_tmp.p, bytes, rowsz, scan,
                                            (int)(nt_new - nt_old + 1), st));
    // offsets of the new tiles continue after the existing store (written
    // on the device; the host reads back only the added size)
    k_ell_offsets<<<grid_for(nt_new - nt_old + 1), kThreads, 0, st>>>(
        scan, nt_new - nt_old + 1, total, c.tileOff.p + nt_old);
    OCTF_CUDA(cudaGetLastError());
    int64_t add = 0;
    OCTF_CUDA(cudaMemcpyAsync(&add, scan + (nt_new - nt_old), sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
    OCTF_CUDA(cudaStreamSynchronize(st));
    c.F.grow_keep((size_t)(total + add) + 1, (size_t)total, st);
    c.W.grow_keep((size_t)(total + add) + 1, (size_t)total, st);
    total += add;
  }
  ph_mark(c, kPhEllGrow, st);
  int32_t* fresh = c.sort_v32.ensure(nnew * 8 + 1);
  k_ell_update<<<wave_grid(nnew), kThreads, 0, st>>>(
      c.lblocks.p, c.lmeta.p, nnew, nold, oldmask, c.tileK.p, c.tileOff.p,
      c.F.p, c.W.p, fresh, c.counters.p + 2, c.counters.p + 4);
  // (slots past the list's end are never leaves: their rows are not read)
  int32_t* need = c.app_buf.ensure(nt_new + 1);
  OCTF_CUDA(cudaMemsetAsync(need, 0, (nt_new + 1) * sizeof(int32_t), st));
  ph_mark(c, kPhEllUpdate, st);
  // second attempt: only the leaves that overflowed (queued in redo)
  int32_t* redo = c.split_list.ensure(nnew * 8 + 1);
  OCTF_CUDA(cudaMemsetAsync(c.counters.p + 7, 0, sizeof(int32_t), st));
  for (int attempt = 0; attempt < 2; ++attempt) {
    k_ell_fresh<<<148 * 8, kThreads, 0, st>>>(
        attempt == 0 ? fresh : redo,
        attempt == 0 ? c.counters.p + 2 : c.counters.p + 7, c.lmeta.p,
        ctx_views(c), c.tileK.p, c.tileOff.p, c.F.p, c.W.p, c.counters.p + 3,
        need, attempt == 0 ? redo : nullptr, c.counters.p + 7);
    OCTF_CUDA(cudaGetLastError());
    OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p, 8 * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, st));
    OCTF_CUDA(cudaStreamSynchronize(st));
    ph_mark(c, kPhFresh, st);
    if (!c.h_counters[3]) break;
    if (attempt == 1) return false;
    // some new leaves see more views than their tile has rows: give those
    // tiles bigger row ranges at the end of the store (with headroom) and
    // gather again (writes are idempotent).  Planned on the device; the
    // host reads back only the added size (to grow the store).
    int64_t* rows = reinterpret_cast<int64_t*>(c.sort_k64.ensure(2 * nt_new + 3));
    int64_t* scan = rows + nt_new + 2;
    OCTF_CUDA(cudaMemsetAsync(rows + nt_new + 1, 0, sizeof(int64_t), st));
    int32_t* mlist = c.sort_k32.ensure(nt_new + 2);
    OCTF_CUDA(cudaMemsetAsync(mlist, 0, sizeof(int32_t), st));
    k_ell_plan<<<grid_for(nt_new + 1), kThreads, 0, st>>>(need, c.tileK.p,
                                                          nt_new, rows, mlist);
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, rows, scan,
                                  (int)(nt_new + 1), st);
    c.cub_tmp.ensure(bytes);
    OCTF_CUDA(cub::DeviceScan::ExclusiveSum(c.cub_tmp.p, bytes, rows, scan,
                                            (int)(nt_new + 1), st));
    int64_t hv[2] = {0, 0};
    OCTF_CUDA(cudaMemcpyAsync(&hv[0], scan + nt_new, sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
    OCTF_CUDA(cudaMemcpyAsync(&hv[1], rows + nt_new + 1, sizeof(int64_t),
                              cudaMemcpyDeviceToHost, st));
    OCTF_CUDA(cudaStreamSynchronize(st));
    const int64_t keep = total;
    c.ell_waste += hv[1];
    total += hv[0];
    // (the old ranges stay unused until the next full rebuild compacts)
    c.F.grow_keep((size_t)total + 1, (size_t)keep, st);
    c.W.grow_keep((size_t)total + 1, (size_t)keep, st);
    k_ell_move_dev<<<(unsigned)std::min<int64_t>(nt_new, 148 * 8), 256, 0,
                     st>>>(mlist, need, c.tileK.p, c.tileOff.p, scan, keep,
                           c.F.p, c.W.p);
    OCTF_CUDA(cudaGetLastError());
    OCTF_CUDA(cudaMemsetAsync(c.counters.p + 3, 0, sizeof(int32_t), st));
    OCTF_CUDA(cudaStreamSynchronize(st));
    ph_mark(c, kPhMove, st);
  }
  if (c.sorted) {  // solver='pd': the new leaves' rows in (f, view) order
    k_sort_ell<<<148 * 8, kThreads, 0, st>>>(fresh, c.counters.p + 2, 0,
                                             c.tileK.p, c.tileOff.p, c.F.p,
                                             c.W.p);
    OCTF_CUDA(cudaGetLastError());
  }
  c.nlb = nnew;
  c.nleaves = c.h_counters[4];
  c.ell_tiles = nt_new;
  c.ell_size = total;
  c.store_ok = true;
  if (c.timing) {
    c.t_gather_ms += std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now() - t0).count();
    ++c.n_gather;
    ++c.n_regather;
  }
  return true;
}

// patch the list after our own restructure (see Ctx::lpos): holes for
// blocks without leaves, appended new leaf blocks, all tables recomputed,
// samples kept where a leaf stayed at its position and gathered for new
// leaves.  false: compaction due (or a fractional weight met the mask
// format): the caller rebuilds everything.
bool ctx_list_update(Ctx& c, const int32_t* child, int64_t total, int64_t nbid,
                     cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t nold = c.nlb;
  if (c.lpos_n < nbid) {  // block ids the pool grew by start unlisted
    c.lpos.grow_keep(nbid, c.lpos_n, st);
    OCTF_CUDA(cudaMemsetAsync(c.lpos.p + c.lpos_n, 0xff,
                              (nbid - c.lpos_n) * sizeof(int32_t), st));
    c.lpos_n = nbid;
  }
  uint8_t* oldmask = c.flags.ensure(nold > total ? nold : total);
  int32_t* app = c.app_buf.ensure(total + 1);
  OCTF_CUDA(cudaMemsetAsync(c.counters.p, 0, 8 * sizeof(int32_t), st));
  if (nold)
    k_list_mark<<<grid_for(nold), kThreads, 0, st>>>(
        c.lblocks.p, c.lmeta.p, nold, child, c.blevel.p, c.lpos.p, oldmask,
        c.counters.p);
  k_list_new<<<grid_for(total), kThreads, 0, st>>>(
      c.lvl_blocks.p, total, child, c.lpos.p, app, c.counters.p + 1);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p, 2 * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  c.nholes += c.h_counters[0];
  const int64_t na = c.h_counters[1];
  const int64_t nnew = nold + na;
  ph_mark(c, kPhListDiff, st);
  // compact past 25 % holes or appended entries (half with the ELL store,
  // whose rebuild is the expensive many-view gather)
  const int64_t lim = c.ell ? 2 : 4;
  if (lim * c.nholes > nnew || lim * na > nnew) return false;
  if (na) {
    sort_i32(c, app, na, st);  // appended in base order: deterministic
    c.lblocks.grow_keep(nnew, nold, st);
    k_list_put<<<grid_for(na), kThreads, 0, st>>>(app, na, nold, c.lblocks.p,
                                                   c.lpos.p);
    OCTF_CUDA(cudaGetLastError());
  }
  c.lkey.grow_keep(nnew, nold, st);
  c.lmeta.grow_keep(nnew, nold, st);
  c.lpar.grow_keep(nnew, nold, st);
  c.nbr.grow_keep(nnew * 12, nold * 12, st);
  // tables only for the entries the patch touched (k_table_dirty)
  int32_t* dirty = c.split_list.ensure(nnew + 1);
  OCTF_CUDA(cudaMemsetAsync(c.counters.p + 6, 0, sizeof(int32_t), st));
  k_table_dirty<<<grid_for(nnew), kThreads, 0, st>>>(
      c.lblocks.p, nnew, nold, oldmask, child, c.blevel.p, c.nbr.p, dirty,
      c.counters.p + 6);
  // the dirty count stays on the device: one wave strides over it
  k_leaf_tables<<<(unsigned)std::min<int64_t>(grid_for(nnew * 12), 148 * 8),
                  kThreads, 0, st>>>(
      child, c.lblocks.p, 0, c.blevel.p, c.bcoord.p, c.bparent.p, c.lkey.p,
      c.lmeta.p, c.lpar.p, c.nbr.p, dirty, c.counters.p + 6);
  OCTF_CUDA(cudaGetLastError());
  ph_mark(c, kPhTables, st);
  if (c.ell) return ell_list_samples(c, nold, nnew, oldmask, t0, st);
  // samples, in place (the store only grows; its tail is zeroed)
  const int64_t nvp = c.sstride;
  auto pad = [](int64_t n) {
    return (n * 8 + kTileLeaves - 1) / kTileLeaves * kTileLeaves;
  };
  const int64_t npo = pad(nold), npn = pad(nnew);
  c.F.grow_keep((size_t)nvp * npn, (size_t)nvp * npo, st);
  if (c.binw) c.M.grow_keep(npn, npo, st);
  else c.W.grow_keep((size_t)nvp * npn, (size_t)nvp * npo, st);
  int32_t* fresh = c.sort_v32.ensure(nnew * 8 + 1);
  if (c.binw)
    k_sample_update<true><<<wave_grid(nnew), kThreads, 0, st>>>(
        c.lblocks.p, c.lmeta.p, nnew, nold, oldmask, nvp, c.F.p, nullptr,
        c.M.p, fresh, c.counters.p + 2, c.counters.p + 4);
  else
    k_sample_update<false><<<wave_grid(nnew), kThreads, 0, st>>>(
        c.lblocks.p, c.lmeta.p, nnew, nold, oldmask, nvp, c.F.p, c.W.p,
        nullptr, fresh, c.counters.p + 2, c.counters.p + 4);
  if (npn > nnew * 8) {
    const int64_t from = nnew * 8, to = npn;
    if (c.binw)
      k_zero_slots<true><<<grid_for(to - from), kThreads, 0, st>>>(
          from, to, nvp, c.F.p, nullptr, c.M.p);
    else
      k_zero_slots<false><<<grid_for(to - from), kThreads, 0, st>>>(
          from, to, nvp, c.F.p, c.W.p, nullptr);
  }
  const unsigned gw = 148 * 8;  // warps stride over the queued leaves
  if (c.binw)
    k_gather_fresh<true><<<gw, kThreads, 0, st>>>(
        fresh, c.counters.p + 2, c.lmeta.p, ctx_views(c), nvp, c.F.p, nullptr,
        c.M.p, c.counters.p + 3);
  else
    k_gather_fresh<false><<<gw, kThreads, 0, st>>>(
        fresh, c.counters.p + 2, c.lmeta.p, ctx_views(c), nvp, c.F.p, c.W.p,
        nullptr, c.counters.p + 3);
  OCTF_CUDA(cudaGetLastError());
  ctx_sort_samples(c, fresh, c.counters.p + 2, st);  // pd: new leaves only
  OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p, 8 * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  if (c.binw && (c.h_counters[3] & 1)) return false;  // needs the weight format
  if (c.h_counters[3] & 2) c.allv = false;  // a new leaf misses a sample
  c.nlb = nnew;
  c.nleaves = c.h_counters[4];
  c.store_ok = true;
  if (c.timing) {
    c.t_gather_ms += std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now() - t0).count();
    ++c.n_gather;
    ++c.n_regather;
  }
  return true;
}

void ctx_set_views(Ctx& c, int nviews, const float* const* vval,
                   const float* const* vw, const int32_t* const* vchild,
                   cudaStream_t st) {
  if (nviews == 0 && c.ext_F) return;  // samples supplied per slot
  c.ext_F = nullptr;
  c.ext_W = nullptr;
  std::vector<const void*> key;
  for (int v = 0; v < nviews; ++v) {
    key.push_back(vval[v]);
    key.push_back(vw[v]);
    key.push_back(vchild[v]);
  }
  if (key == c.vkey && nviews == c.nviews) return;
  c.vkey = key;
  c.nviews = nviews;
  c.dv_val.ensure(nviews);
  c.dv_w.ensure(nviews);
  c.dv_child.ensure(nviews);
  OCTF_CUDA(cudaMemcpyAsync(c.dv_val.p, vval, nviews * sizeof(void*),
                            cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyAsync(c.dv_w.p, vw, nviews * sizeof(void*),
                            cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyAsync(c.dv_child.p, vchild, nviews * sizeof(void*),
                            cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  if (c.valid && !c.defer_gather) ctx_gather(c, st);
}

void ctx_set_samples(Ctx& c, const float* F, const float* W, int nviews,
                     int64_t cap, cudaStream_t st) {
  if (!F || nviews < 1) throw Error(kEArg, "samples and a view count needed");
  c.ext_F = F;
  c.ext_W = W;
  c.ext_cap = cap;
  c.nviews = nviews;
  c.vkey.clear();
  if (c.valid && !c.defer_gather) ctx_gather(c, st);
  OCTF_CUDA(cudaStreamSynchronize(st));
}

ViewSet ctx_views(const Ctx& c) {
  ViewSet v;
  v.val = c.dv_val.p;
  v.w = c.dv_w.p;
  v.child = c.dv_child.p;
  v.n = c.nviews;
  return v;
}

// the per-level view maps of every live slot, views in chunks of 32;
// fn(v0, nc, vm) consumes each chunk's maps (vm[y * cap + slot])
template <typename Fn>
static void view_maps(Ctx& c, cudaStream_t st, Fn fn) {
  const int nv = c.nviews;
  // views per chunk: 32, fewer when the maps would pass ~16 GB (a pool of
  // 7e8 slots at BASELINE config 3's depth 11)
  int chunk = nv < 32 ? nv : 32;
  while (chunk > 1 && (double)chunk * c.cap * 4.0 > 16e9) chunk /= 2;
  int32_t* vm = c.vmap.ensure((size_t)chunk * c.cap);
  for (int v0 = 0; v0 < nv; v0 += chunk) {
    const int nc = nv - v0 < chunk ? nv - v0 : chunk;
    for (int y = 0; y < nc; ++y)  // root slot -> root node
      OCTF_CUDA(cudaMemsetAsync(vm + (int64_t)y * c.cap, 0, sizeof(int32_t), st));
    for (int L = 1; L <= c.d_max && L < (int)c.lvl_cnt.size(); ++L) {
      const int64_t nb = c.lvl_cnt[L];
      if (!nb) continue;
      k_vmap_level<<<dim3(grid_for(nb * 8), nc), kThreads, 0, st>>>(
          c.lvl_blocks.p + c.lvl_off[L], nb, c.bparent.p, ctx_views(c), v0,
          c.cap, vm);
    }
    fn(v0, nc, vm);
  }
  OCTF_CUDA(cudaGetLastError());
}

// dense gather through the view maps
static void gather_by_levels(Ctx& c, int64_t nvp, cudaStream_t st) {
  const int64_t n = c.nlb * 8;
  view_maps(c, st, [&](int v0, int nc, const int32_t* vm) {
    k_vgather<<<dim3(grid_for(n), nc), kThreads, 0, st>>>(
        c.child_key, c.lblocks.p, c.nlb, ctx_views(c), v0, c.cap, vm, c.F.p,
        c.W.p, c.counters.p, c.lmeta.p, c.sd);
  });
}

void ctx_gather_ell(Ctx& c, cudaStream_t st) {
  const int64_t n = c.nlb * 8;
  const int64_t nt = (n + kTileLeaves - 1) / kTileLeaves;
  // one pass over the tiles: counts -> rows -> offsets (from 0)
  int32_t* cnt = c.sort_k32.ensure(nt * 256 + 1);
  OCTF_CUDA(cudaMemsetAsync(cnt, 0, nt * 256 * sizeof(int32_t), st));
  view_maps(c, st, [&](int v0, int nc, const int32_t* vm) {
    k_vcount<<<grid_for(n), kThreads, 0, st>>>(c.child_key, c.lblocks.p,
                                                c.nlb, ctx_views(c), v0, nc,
                                                c.cap, vm, cnt);
  });
  if (const char* es = std::getenv("OCTF_ELL_STATS"); es && es[0] == '1') {
    // diagnosis: observed samples, and the store sizes per-tile (this
    // layout) / per-block row counts would need
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(
        c.dscalar.ensure(4));
    OCTF_CUDA(cudaMemsetAsync(acc, 0, 4 * sizeof(double), st));
    k_ell_stats<<<grid_for(nt * 32), kThreads, 0, st>>>(cnt, nt, acc);
    unsigned long long h[3] = {0, 0, 0};
    OCTF_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, st));
    OCTF_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr,
            "ell_stats: leaves %lld, observed samples %llu, per-tile rows "
            "%llu entries, per-block rows %llu entries\n",
            (long long)c.nleaves, h[0], h[1], h[2]);
  }
  int64_t* rowsz = reinterpret_cast<int64_t*>(c.sort_k64.ensure(nt + 1));
  c.tileK.ensure(nt + 1);
  c.tileOff.ensure(nt + 1);
  if (nt)
    k_ell_tilemax<<<(unsigned)nt, 256, 0, st>>>(cnt, n, 0, c.tileK.p, rowsz);
  OCTF_CUDA(cudaMemsetAsync(rowsz + nt, 0, sizeof(int64_t), st));
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, rowsz, c.tileOff.p,
                                (int)(nt + 1), st);
  c.cub_tmp.ensure(bytes);
  OCTF_CUDA(cub::DeviceScan::ExclusiveSum(c.cub_tmp.p, bytes, rowsz,
                                          c.tileOff.p, (int)(nt + 1), st));
  OCTF_CUDA(cudaGetLastError());
  int64_t total = 0;
  OCTF_CUDA(cudaMemcpyAsync(&total, c.tileOff.p + nt, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  c.F.ensure((size_t)total + 1);
  c.W.ensure((size_t)total + 1);
  int32_t* cur = cnt;  // reuse: running row per slot
  OCTF_CUDA(cudaMemsetAsync(cur, 0, nt * 256 * sizeof(int32_t), st));
  view_maps(c, st, [&](int v0, int nc, const int32_t* vm) {
    k_vput<<<grid_for(n), kThreads, 0, st>>>(c.child_key, c.lblocks.p, c.nlb,
                                              ctx_views(c), v0, nc, c.cap, vm,
                                              c.tileOff.p, cur, c.F.p, c.W.p);
  });
  if (nt)
    k_ell_pad<<<grid_for(nt * 256), kThreads, 0, st>>>(cur, nt * 256,
                                                        c.tileK.p, c.tileOff.p,
                                                        c.F.p, c.W.p);
  OCTF_CUDA(cudaGetLastError());
  if (c.sorted && nt) {  // solver='pd': every leaf's rows in (f, view) order
    k_sort_ell<<<148 * 8, kThreads, 0, st>>>(nullptr, nullptr, nt * 256,
                                             c.tileK.p, c.tileOff.p, c.F.p,
                                             c.W.p);
    OCTF_CUDA(cudaGetLastError());
  }
  c.M.release();
  c.binw = false;
  c.allv = false;
  c.ell = true;
  c.packed = false;
  c.sd = SDesc();
  c.ell_tiles = nt;
  c.ell_size = total;
  c.ell_waste = 0;
  c.sstride = 0;
}

void ctx_sort_samples(Ctx& c, const int32_t* list, const int32_t* nlist,
                      cudaStream_t st) {
  if (!c.sorted || c.ell) return;
  const int64_t n = c.nlb * 8;
  const uint32_t* M = c.binw ? c.M.p : nullptr;
  float* W = c.binw ? nullptr : c.W.p;
  const unsigned g = 148 * 8;  // grid-stride (the list count is on the device)
#define OCTF_SORT(N)                                                          \
  k_sort_samples<N><<<g, kThreads, 0, st>>>(list, nlist, n, c.nviews, c.F.p, \
                                             W, M, c.lmeta.p, c.sd)
  switch (c.sstride) {
    case 4: OCTF_SORT(4); break;
    case 8: OCTF_SORT(8); break;
    case 16: OCTF_SORT(16); break;
    case 32: OCTF_SORT(32); break;
    case 64: OCTF_SORT(64); break;
    default: return;  // the pd kernel rejects other view counts
  }
#undef OCTF_SORT
  OCTF_CUDA(cudaGetLastError());
}

void ctx_gather(Ctx& c, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  // per-tile (ELL) store: above 64 views, from 33 with OCTF_CTX_ELL, and at
  // any view count for OCTF_CTX_ELL | OCTF_CTX_SORTED (solver='pd' with a
  // view count the dense sorted store has no instantiation for)
  if (!c.ext_F && !c.dense_only &&
      (c.nviews > 64 || (c.force_ell && (c.nviews > 32 || c.sorted)))) {
    ctx_gather_ell(c, st);
    OCTF_CUDA(cudaStreamSynchronize(st));
    c.store_ok = true;
    if (c.timing) {
      c.t_gather_ms += std::chrono::duration<double, std::milli>(
                           std::chrono::steady_clock::now() - t0).count();
      ++c.n_gather;
    }
    return;
  }
  c.ell = false;
  // tiles of 256 slots, view-major inside a tile (octf_common.cuh SDesc);
  // views padded to 4; packed: a group-k tile holds its 32 k leaves only
  int64_t n = c.nlb * 8;
  const int64_t ntiles = (n + kTileLeaves - 1) / kTileLeaves;
  int nv = c.nviews;
  const int64_t nvp = (nv + 3) & ~3;
  c.sstride = nvp;
  // packed positions (a frozen tree's full list; a shard's subset keeps
  // slot positions): block ranks first, kept only if some block is not full
  SDesc d;
  d.nvp = nvp;
  if (c.pack_opt && c.list_full && ntiles) {
    OCTF_CUDA(cudaMemsetAsync(c.counters.p + 1, 0, sizeof(int32_t), st));
    k_pack_ranks<<<grid_for(ntiles * 32), kThreads, 0, st>>>(
        c.lmeta.p, c.nlb, ntiles, c.counters.p + 1);
    OCTF_CUDA(cudaGetLastError());
    OCTF_CUDA(cudaMemcpyAsync(c.h_counters + 1, c.counters.p + 1,
                              sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    OCTF_CUDA(cudaStreamSynchronize(st));
    d.packed = c.h_counters[1] > 0 ? 1 : 0;
  }
  const int64_t nf = ntiles * nvp * kTileLeaves, nm = ntiles * kTileLeaves;
  c.sd = d;
  c.packed = d.packed != 0;
  c.F.ensure((size_t)nf);
  c.W.ensure((size_t)nf);
  OCTF_CUDA(cudaMemsetAsync(c.F.p, 0, (size_t)nf * sizeof(float), st));
  OCTF_CUDA(cudaMemsetAsync(c.W.p, 0, (size_t)nf * sizeof(float), st));
  OCTF_CUDA(cudaMemsetAsync(c.counters.p, 0, sizeof(int32_t), st));
  if (c.ext_F)  // per-slot sample arrays supplied by the caller
    k_gather_slots<<<grid_for(n), kThreads, 0, st>>>(
        c.child_key, c.lblocks.p, c.nlb, c.ext_F, c.ext_W, c.ext_cap, nv, c.F.p,
        c.W.p, c.counters.p, c.lmeta.p, c.sd);
  else
    gather_by_levels(c, nvp, st);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p, sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  c.binw = !(c.h_counters[0] & 1) && nv <= 32;
  // every leaf has every sample (weight 1): kernels skip the mask
  c.allv = c.binw && !(c.h_counters[0] & 2) && nv == nvp &&
           (nv == 8 || nv == 16 || nv == 32);
  if (c.binw) {
    c.M.ensure(nm);
    OCTF_CUDA(cudaMemsetAsync(c.M.p, 0, (size_t)nm * sizeof(uint32_t), st));
    k_masks<<<grid_for(n), kThreads, 0, st>>>(c.W.p, c.lmeta.p, c.nlb, nv,
                                              c.sd, c.M.p);
    OCTF_CUDA(cudaGetLastError());
    OCTF_CUDA(cudaStreamSynchronize(st));
    c.W.release();  // the mask format replaces the weight vectors
  } else {
    c.M.release();
  }
  ctx_sort_samples(c, nullptr, nullptr, st);
  c.store_ok = true;
  if (c.timing) {
    c.t_gather_ms += std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now() - t0).count();
    ++c.n_gather;
  }
}

// every live node (or leaf) of the prepared pool in the reference's
// canonical order: slots and preorder keys (radix sort of the keys)
int64_t ctx_node_order(Ctx& c, const int32_t* child, int d_max,
                       bool leaves_only, int32_t* out_slots,
                       uint64_t* out_keys, cudaStream_t st) {
  if (!c.valid || c.child_key != child)
    throw Error(kEArg, "context not prepared for this pool");
  // the level lists hold every live block, the root's pseudo-block 0 first
  const int64_t nblk = c.nblocks;
  const int32_t* blocks = c.lvl_blocks.p;
  const int64_t n8 = nblk * 8;
  uint64_t* keys = c.sort_k64.ensure(2 * n8);
  int32_t* slots = c.sort_k32.ensure(2 * n8);
  OCTF_CUDA(cudaMemsetAsync(c.counters.p, 0, sizeof(int32_t), st));
  k_node_keys<<<grid_for(n8), kThreads, 0, st>>>(
      blocks, nblk, c.blevel.p, c.bcoord.p, child, d_max, leaves_only ? 1 : 0,
      keys, slots, c.counters.p);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p, sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  const int64_t n = c.h_counters[0];
  if (n > c.hstate[2] + 0 && !leaves_only)
    throw Error(kEArg, "corrupt pool: more nodes than state[2]");
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys + n8, slots,
                                  slots + n8, (int)n, 0, 64, st);
  c.cub_tmp.ensure(bytes);
  OCTF_CUDA(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, bytes, keys,
                                            keys + n8, slots, slots + n8,
                                            (int)n, 0, 64, st));
  if (out_slots)
    OCTF_CUDA(cudaMemcpyAsync(out_slots, slots + n8, n * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, st));
  if (out_keys)
    OCTF_CUDA(cudaMemcpyAsync(out_keys, keys + n8, n * sizeof(uint64_t),
                              cudaMemcpyDeviceToDevice, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  return n;
}

}  // namespace octf

namespace octf {
namespace {

__global__ void k_select(const int32_t* __restrict__ sel,
                         const uint8_t* __restrict__ masks, int64_t nsel,
                         const int32_t* lblocks, const uint64_t* lkey,
                         const int4* lmeta, const int32_t* lpar,
                         const int32_t* nbr, int32_t* o_lblocks,
                         uint64_t* o_lkey, int4* o_lmeta, int32_t* o_lpar,
                         int32_t* o_nbr) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nsel) return;
  const int32_t i = sel[j];
  if (i < 0) {  // padding hole (aligns the boundary range to a tile)
    o_lblocks[j] = -1;
    o_lkey[j] = 0;
    o_lmeta[j] = make_int4(0, 0, 0, pack_meta_w(0, 0u, 0));
    o_lpar[j] = -1;
    for (int d = 0; d < 12; ++d) o_nbr[j * 12 + d] = kNone;
    return;
  }
  o_lblocks[j] = lblocks[i];
  o_lkey[j] = lkey[i];
  int4 m = lmeta[i];
  // keep only the rank's leaves active (bits 19..26 of .w)
  m.w = (int)(((unsigned)m.w & ~(0xffu << 19)) | ((unsigned)masks[j] << 19));
  o_lmeta[j] = m;
  o_lpar[j] = lpar[i];
  for (int d = 0; d < 12; ++d) o_nbr[j * 12 + d] = nbr[(int64_t)i * 12 + d];
}

}  // namespace

void ctx_select(Ctx& c, const int32_t* sel, const uint8_t* masks, int64_t nsel,
                cudaStream_t st) {
  if (!c.valid) throw Error(kEArg, "context not prepared");
  DevBuf<int32_t> dsel, olb, onbr, opar;
  DevBuf<uint8_t> dmask;
  DevBuf<uint64_t> okey;
  DevBuf<int4> ometa;
  dsel.ensure(nsel);
  dmask.ensure(nsel);
  olb.ensure(nsel);
  okey.ensure(nsel);
  ometa.ensure(nsel);
  opar.ensure(nsel);
  onbr.ensure(nsel * 12);
  if (nsel) {
    OCTF_CUDA(cudaMemcpyAsync(dsel.p, sel, nsel * sizeof(int32_t),
                              cudaMemcpyHostToDevice, st));
    OCTF_CUDA(cudaMemcpyAsync(dmask.p, masks, nsel, cudaMemcpyHostToDevice, st));
    k_select<<<grid_for(nsel), kThreads, 0, st>>>(
        dsel.p, dmask.p, nsel, c.lblocks.p, c.lkey.p, c.lmeta.p, c.lpar.p,
        c.nbr.p, olb.p, okey.p, ometa.p, opar.p, onbr.p);
    OCTF_CUDA(cudaGetLastError());
  }
  OCTF_CUDA(cudaStreamSynchronize(st));
  c.lblocks.swap(olb);
  c.lkey.swap(okey);
  c.lmeta.swap(ometa);
  c.lpar.swap(opar);
  c.nbr.swap(onbr);
  c.nlb = nsel;
  c.list_full = false;  // a shard's subset: never patched in place
  c.defer_gather = false;  // the subset's samples are gathered now
  if (c.nviews > 0) ctx_gather(c, st);
  OCTF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace octf

// ---- halo exchange staging (shard.HaloExchange): the values of up to five
// fields at a slot list, packed field-major into one contiguous buffer per
// peer, and the received buffer scattered back
namespace octf {
namespace {

template <typename T>
struct HaloFields {
  T* v[kMaxHaloFields];
};

template <typename T>
__global__ void k_halo_pack(HaloFields<T> f, int nf, const int32_t* __restrict__ idx,
                            int64_t n, T* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int32_t s = __ldg(idx + j);
#pragma unroll
  for (int k = 0; k < kMaxHaloFields; ++k)
    if (k < nf) out[k * n + j] = f.v[k][s];
}

template <typename T>
__global__ void k_halo_unpack(HaloFields<T> f, int nf,
                              const int32_t* __restrict__ idx, int64_t n,
                              const T* __restrict__ in) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int32_t s = __ldg(idx + j);
#pragma unroll
  for (int k = 0; k < kMaxHaloFields; ++k)
    if (k < nf) f.v[k][s] = in[k * n + j];
}

}  // namespace

template <typename T>
void halo_pack(T* const* fields, int nf, const int32_t* idx, int64_t n,
               T* buf, bool unpack, cudaStream_t st) {
  if (nf < 1 || nf > kMaxHaloFields)
    throw Error(kEArg, "halo: 1 to 5 fields");
  if (n <= 0) return;
  HaloFields<T> f{};
  for (int k = 0; k < nf; ++k) f.v[k] = fields[k];
  if (unpack)
    k_halo_unpack<T><<<grid_for(n), kThreads, 0, st>>>(f, nf, idx, n, buf);
  else
    k_halo_pack<T><<<grid_for(n), kThreads, 0, st>>>(f, nf, idx, n, buf);
  OCTF_CUDA(cudaGetLastError());
}

template void halo_pack<float>(float* const*, int, const int32_t*, int64_t,
                               float*, bool, cudaStream_t);
template void halo_pack<double>(double* const*, int, const int32_t*, int64_t,
                                double*, bool, cudaStream_t);

}  // namespace octf
