// The leaf-update kernel: the hot path of every solver pass.
//
// Included by solver_impl.cuh inside namespace octf::{anonymous}.
//
// Mapping: one CTA = 256 threads = 32 leaf blocks; the 8 lanes of a group are
// the 8 sibling slots of one block (the reference's contiguous child block,
// octree.py:49-71), so
//  * the block's own values reach every lane with one __shfl_xor per stencil
//    point: a +-1 step along an axis flips exactly that axis's bit of the
//    child index, for the own block and the neighbour block alike;
//  * only lanes whose step leaves the block read memory, through the
//    block's 12-entry neighbour table (compile-time direction per stencil
//    point and lane parity);
//  * the CTA's 256 leaves are one sample tile ([view][256], contiguous in
//    HBM, octf_common.cuh samp_idx): with N known at compile time one thread
//    issues a single TMA bulk copy (cp.async.bulk + mbarrier) of the whole
//    tile into shared memory at kernel entry, so the dominant 4N B/leaf
//    stream is in flight while the stencil runs and costs no registers;
//    lanes read their samples back conflict-free after the barrier.
// ENERGY also evaluates the reference's per-leaf energy term
// (_kernels.pyx:517-533) of the incoming (snapshot) state, which is the
// previous pass's post-propagate state, from the same values and roots.
#pragma once

// Measured and dropped (profiles/r01/pd_kernel_notes.md): per-warp
// staging (17 bulk copies of 128 B per warp: slower than one CTA copy) and
// per-warp energy partials (faster at N = 16, slower at N = 32).
#ifndef OCTF_LEAF_MINB
#define OCTF_LEAF_MINB 1
#endif
// resident CTAs per SM the register budget is cut for, by sample count:
// measured best 6 (<= 40 registers) for N <= 16 (cfg2: 0.341 -> 0.327 ms)
// but 4 for N = 32 (cfg5: 6 costs 6 %); OCTF_LEAF_MINB sets the latter
#ifndef OCTF_LEAF_MINB_SMALL
#define OCTF_LEAF_MINB_SMALL 6
#endif
// the runtime-N instantiation (restructuring configurations: dense general
// weights, or the per-tile ELL store whose row batches want registers)
#ifndef OCTF_LEAF_MINB_GENERIC
#define OCTF_LEAF_MINB_GENERIC OCTF_LEAF_MINB
#endif
#ifndef OCTF_ELL_PRE
#define OCTF_ELL_PRE 4
#endif
#ifndef OCTF_ELL_BATCH
#define OCTF_ELL_BATCH 8
#endif
constexpr int leaf_minb(int nv, int tbytes) {
  // (the f64 parity mode needs the registers: 40 or 48 would spill)
  return tbytes == 8 ? 2
         : nv == 0 ? OCTF_LEAF_MINB_GENERIC
         : nv <= 16 ? OCTF_LEAF_MINB_SMALL
                    : OCTF_LEAF_MINB;
}

template <typename T>
struct LeafArgs {
  const int32_t* __restrict__ lblocks;
  int64_t nlb;
  const uint64_t* __restrict__ lkey;
  const int4* __restrict__ lmeta;
  const int32_t* __restrict__ lpar;  // parent slot of each leaf block
  int32_t* join_bot;  // restructuring passes: parents of bottom candidates
  const int32_t* __restrict__ nbr;
  const int32_t* __restrict__ child;
  const T* __restrict__ snap;
  T* __restrict__ uval;
  const float* __restrict__ F;
  const float* __restrict__ W;
  const uint32_t* __restrict__ M;
  int64_t stride;  // floats per leaf sample vector (views padded to 4)
  int nv;
  LeafParams<T> p;
  uint8_t* smark;
  int32_t* split_list;
  int32_t* counters;
  double* epart;  // per-CTA energy partial sums
  int tile0 = 0;  // first tile of this launch (sharded overlap: sub-ranges)
  int ntiles = 0;  // tiles of this launch ([tile0, tile0 + ntiles))
  const int32_t* __restrict__ tileK = nullptr;    // ELL store (views > 32)
  const int64_t* __restrict__ tileOff = nullptr;
  SDesc sd;  // the dense sample store's layout (octf_common.cuh)
};

// slot read for the cell (x+DX, y+DY, z+DZ) at the leaf's level, from the
// block's 12 neighbour-table entries (in registers): -1 when the cell is the
// sibling c^mask of the own block (value by shuffle) or is not read; else a
// slot of the same-level neighbour block or the coarser leaf covering it
template <int DX, int DY, int DZ>
__device__ __forceinline__ int step_idx_r(int c, int cx, int cy, int cz,
                                          bool inside, const int32_t (&N)[12]) {
  const bool ex = DX > 0 ? cx : (DX < 0 ? !cx : false);
  const bool ey = DY > 0 ? cy : (DY < 0 ? !cy : false);
  const bool ez = DZ > 0 ? cz : (DZ < 0 ? !cz : false);
  constexpr int mask = (DX ? 4 : 0) | (DY ? 2 : 0) | (DZ ? 1 : 0);
  constexpr int fx = DX < 0 ? 0 : 1, fy = DY < 0 ? 2 : 3, fz = DZ < 0 ? 4 : 5;
  constexpr int exy = DX < 0 ? 6 : 8, exz = DX < 0 ? 7 : 10, eyz = DY < 0 ? 9 : 11;
  int32_t r;
  if (DX != 0 && DY != 0) r = ex ? (ey ? N[exy] : N[fx]) : N[fy];
  else if (DX != 0 && DZ != 0) r = ex ? (ez ? N[exz] : N[fx]) : N[fz];
  else if (DY != 0 && DZ != 0) r = ey ? (ez ? N[eyz] : N[fy]) : N[fz];
  else r = DX != 0 ? N[fx] : (DY != 0 ? N[fy] : N[fz]);
  const int idx = r >= 0 ? r + (c ^ mask) : -r - 2;
  return ((ex || ey || ez) && inside) ? idx : -1;
}

template <typename T>
__device__ __forceinline__ T pick(T own, int idx, const T* __restrict__ arr) {
  return idx >= 0 ? arr[idx] : own;
}

// ---- TMA bulk copy global -> shared with an mbarrier (sm_90+ / sm_100a)
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  uint64_t state;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
               : "=l"(state)
               : "r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  (void)state;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src,
                                         unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

// the staged kernels are persistent: a CTA walks tiles tile0 + blockIdx.x,
// + gridDim.x, ... with OCTF_STAGES sample-tile buffers in shared memory, the
// bulk copy of a later tile in flight while the current one is computed
// (one stage = the sample tile, then the mask or the weight tile)
// Measured on cfg5 (profiles/r02/ab_stages.txt): 2 and 3 stages force 3
// and 2 resident CTAs per SM (shared memory) and lose more to the stencil's
// load latency than they gain (leaf 3.52 / 4.10 / 4.78 ms for 1 / 2 / 3
// stages); one CTA per tile (OCTF_PERSIST=0, the hardware scheduler
// balancing tiles of uneven cost) with one stage is the default.
#ifndef OCTF_STAGES
#define OCTF_STAGES 1
#endif
#ifndef OCTF_PERSIST
#define OCTF_PERSIST 0
#endif
constexpr int kStages = OCTF_STAGES;
// sample formats (the BW template parameter): general weights, binary
// weights as a bit mask, or every sample present with weight 1 (no mask)
constexpr int kWeights = 0, kMask = 1, kAllValid = 2;
constexpr size_t leaf_stage_floats(int nv, int bw) {
  return nv <= 0 ? 0
                 : (size_t)((nv + 3) & ~3) * kTileLeaves +
                       (bw == kAllValid ? 0
                        : bw == kMask   ? (size_t)kTileLeaves
                                        : (size_t)((nv + 3) & ~3) * kTileLeaves);
}
constexpr size_t leaf_smem_bytes(int nv, int bw) {
  return leaf_stage_floats(nv, bw) * 4 * kStages;
}

// issue the bulk copy of tile `tile` into stage buffer `buf` (thread 0):
// the whole [view][256] slot tile, then its mask or weight tile
template <int NVP, int BW>
__device__ __forceinline__ void stage_tile(float* buf, uint64_t* bar,
                                           const float* F, const void* A,
                                           size_t tile) {
  const unsigned fbytes = NVP * kTileLeaves * 4;
  const unsigned abytes = BW == kAllValid ? 0u
                          : BW == kMask   ? kTileLeaves * 4u
                                          : fbytes;
  mbar_expect_tx(bar, fbytes + abytes);
  bulk_g2s(buf, F + tile * NVP * kTileLeaves, fbytes, bar);
  if (abytes)
    bulk_g2s(buf + NVP * kTileLeaves,
             BW == kMask ? (const void*)((const uint32_t*)A + tile * kTileLeaves)
                         : (const void*)((const float*)A + tile * NVP * kTileLeaves),
             abytes, bar);
}

// packed store (octf_common.cuh SDesc): a tile's n_t leaves fill its first
// ceil(n_t / 32) chunks of NV x 32 samples.  Thread 0 stages the first
// kEarlyChunks chunks (and the mask tile) at once, before anything is
// known about the tile; thread kT-1 stages the remaining chunks as soon as
// its own block's lmeta (first rank + leaf count = n_t) has arrived.  The
// barrier expects both arrivals.  nchunks < 0: the early part.
template <int NVP, int BW>
__device__ __forceinline__ void stage_packed(float* buf, uint64_t* bar,
                                             const float* F, const void* A,
                                             size_t tile, int nchunks) {
  constexpr unsigned cb = NVP * kChunk * 4;  // bytes per chunk
  const size_t fo = tile * NVP * kTileLeaves;
  if (nchunks < 0) {
    const unsigned fbytes = kEarlyChunks * cb;
    const unsigned abytes = BW == kAllValid ? 0u
                            : BW == kMask   ? kTileLeaves * 4u
                                            : fbytes;
    mbar_expect_tx(bar, fbytes + abytes);
    bulk_g2s(buf, F + fo, fbytes, bar);
    if (abytes)
      bulk_g2s(buf + NVP * kTileLeaves,
               BW == kMask ? (const void*)((const uint32_t*)A + tile * kTileLeaves)
                           : (const void*)((const float*)A + fo),
               abytes, bar);
    return;
  }
  const int rest = nchunks > kEarlyChunks ? nchunks - kEarlyChunks : 0;
  const unsigned bytes = rest * cb;
  mbar_expect_tx(bar, BW == kWeights ? 2 * bytes : bytes);
  if (!rest) return;
  const size_t off = (size_t)kEarlyChunks * NVP * kChunk;
  bulk_g2s(buf + off, F + fo + off, bytes, bar);
  if (BW == kWeights)
    bulk_g2s(buf + NVP * kTileLeaves + off, (const float*)A + fo + off, bytes,
             bar);
}

// packed fp32 pairs (sm_100a FADD2 / FFMA2)
__device__ __forceinline__ unsigned long long f2u(float2 v) {
  return *reinterpret_cast<unsigned long long*>(&v);
}
__device__ __forceinline__ float2 u2f(unsigned long long v) {
  return *reinterpret_cast<float2*>(&v);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)),
      "l"(f2u(c)));
  return u2f(r);
}

// PK: the packed sample store (octf_common.cuh SDesc; frozen trees, staged N)
template <typename T, bool FROZEN, int BW, bool ENERGY, int NV, bool PK = false>
__global__ void __launch_bounds__(kT, leaf_minb(NV, sizeof(T))) k_leaf_pass(LeafArgs<T> a) {
  using A = Arith<T>;
  const LeafParams<T> p = a.p;
  const T* __restrict__ snap = a.snap;
  // samples: tile by tile through kStages shared-memory buffers; the CTA's
  // first kStages tiles are requested up front, and each buffer is refilled
  // with the tile kStages steps ahead as soon as the CTA is done with it, so
  // the dominant 4N B/leaf stream stays in flight during the compute.
  // Padding leaves and non-leaf slots hold zeros, so copies are in bounds.
  constexpr int NVP = (NV + 3) & ~3;
  constexpr bool BINW = BW != kWeights;  // unit weights (mask or all valid)
  static_assert(BW != kAllValid || NV > 0, "all-valid needs a staged N");
  constexpr size_t STAGE = leaf_stage_floats(NV, BW);
  extern __shared__ __align__(128) float s_smem[];
  __shared__ __align__(8) uint64_t s_bar[kStages];
  const int tend = a.tile0 + a.ntiles;
  const void* aux = BINW ? (const void*)a.M : (const void*)a.W;
  // packed store: each tile is staged at the top of its own iteration by
  // threads 0 and kT-1 (stage_packed; no prefetch across tiles)
  constexpr bool packed = PK && NV > 0;
  // PK with the runtime-N instantiation (NV == 0): the per-tile ELL store --
  // its own instantiation, so its row batches do not cost the dense
  // runtime-N loop registers
  constexpr bool ELLV = PK && NV == 0;
  if (NV > 0) {
    if (threadIdx.x == 0) {
      for (int k = 0; k < kStages; ++k) mbar_init(&s_bar[k], packed ? 2 : 1);
      for (int k = 0; k < kStages && !packed; ++k) {
        const int t = a.tile0 + (int)blockIdx.x + k * (int)gridDim.x;
        if (t < tend)
          stage_tile<NVP, BW>(s_smem + k * STAGE, &s_bar[k], a.F, aux, t);
      }
    }
    __syncthreads();  // barriers initialised before anyone waits on them
  }
  int it = 0;
  for (int tile_id = a.tile0 + (int)blockIdx.x; tile_id < tend;
       tile_id += (int)gridDim.x, ++it) {
  const int stage = NV > 0 ? it % kStages : 0;
  float* const s_tile = s_smem + stage * STAGE;
  // the pool is int32-indexed, so every leaf index fits 32 bits
  const int gid = tile_id * kT + (int)threadIdx.x;
  const int i = gid >> 3;
  const int c = gid & 7;
  const bool inrange = i < (int)a.nlb;
  if (NV > 0 && packed && threadIdx.x == 0)
    stage_packed<NVP, BW>(s_tile, &s_bar[stage], a.F, aux, tile_id, -1);

  // ELL store (NV == 0 instantiations): the tile's row count and offset, and
  // the leaf's first rows, are requested here so that their latency runs
  // under the stencil's table lookups
  constexpr int kEllPre = OCTF_ELL_PRE;      // rows requested before the stencil
  constexpr int kEllBatch = OCTF_ELL_BATCH;  // rows per batch after it
  const int ellK = ELLV ? __ldg(a.tileK + tile_id) : 0;
  const int64_t ell0 =
      ELLV ? __ldg(a.tileOff + tile_id) + (int64_t)threadIdx.x : 0;
  float ew0[kEllPre], ef0[kEllPre];
#pragma unroll
  for (int q = 0; q < kEllPre; ++q) {
    const bool on = q < ellK;
    ew0[q] = on ? __ldg(a.W + ell0 + ((int64_t)q << 8)) : 0.f;
    ef0[q] = on ? __ldg(a.F + ell0 + ((int64_t)q << 8)) : 0.f;
  }

  // one 16 B load: base slot, parent cell, leaf mask and level
  const int4 meta = inrange ? __ldg(a.lmeta + i) : make_int4(0, 0, 0, 0);
  const int32_t b = meta.x;
  const int32_t s = b + c;
  int L, pz;
  unsigned lmask;
  unpack_meta_w(meta.w, pz, lmask, L);
  const int px = meta_px(meta.y), py = meta.z;
  const bool slot_ok = inrange && !(b == 0 && c != 0);
  const bool active = slot_ok && ((lmask >> c) & 1u);
  // the leaf's entry in the staged tile: its slot, or (packed) its rank r
  // among the tile's leaves at chunk r / kChunk, entry r % kChunk, views
  // kChunk apart
  int sbase = threadIdx.x;
  constexpr int sstr = PK ? kChunk : kTileLeaves;
  if (packed) {
    const int r = (meta_rbase(meta.y) + __popc(lmask & ((1u << c) - 1u))) & 255;
    sbase = (r / kChunk) * NVP * kChunk + (r % kChunk);
    if (NV > 0 && threadIdx.x == kT - 1)  // n_t from the tile's last block
      stage_packed<NVP, BW>(
          s_tile, &s_bar[stage], a.F, aux, tile_id,
          inrange ? (meta_rbase(meta.y) + __popc(lmask) + kChunk - 1) / kChunk
                  : kTileLeaves / kChunk);
  }
  const int cx = (c >> 2) & 1, cy = (c >> 1) & 1, cz = c & 1;
  const int x = 2 * px + cx, y = 2 * py + cy, z = 2 * pz + cz;
  const int m = 1 << L;
  const T ih = inv_spacing<T>(p.d_max, L);
  const int32_t* nb = a.nbr + i * 12;
  const T S0 = slot_ok ? snap[s] : (T)0;
  const unsigned FULL = 0xffffffffu;
  const bool xp = x + 1 < m, yp = y + 1 < m, zp = z + 1 < m;
  const bool xm = x > 0, ym = y > 0, zm = z > 0;
  // own-block values of the 12 neighbours (all lanes take part)
  const T o_x = __shfl_xor_sync(FULL, S0, 4);
  const T o_y = __shfl_xor_sync(FULL, S0, 2);
  const T o_z = __shfl_xor_sync(FULL, S0, 1);
  const T o_xy = __shfl_xor_sync(FULL, S0, 6);
  const T o_xz = __shfl_xor_sync(FULL, S0, 5);
  const T o_yz = __shfl_xor_sync(FULL, S0, 3);
  // the block's 12 table entries as three 16 B loads, indices by selects
  // (the primal-dual kernel's form)
  int32_t NB[12];
  {
    const int4* nb4 = reinterpret_cast<const int4*>(nb);
    const int4 n0 = active ? __ldg(nb4) : make_int4(-1, -1, -1, -1);
    const int4 n1 = active ? __ldg(nb4 + 1) : make_int4(-1, -1, -1, -1);
    const int4 n2 = active ? __ldg(nb4 + 2) : make_int4(-1, -1, -1, -1);
    NB[0] = n0.x; NB[1] = n0.y; NB[2] = n0.z; NB[3] = n0.w;
    NB[4] = n1.x; NB[5] = n1.y; NB[6] = n1.z; NB[7] = n1.w;
    NB[8] = n2.x; NB[9] = n2.y; NB[10] = n2.z; NB[11] = n2.w;
  }
#define SV(DX, DY, DZ, OWN, PRED) \
  pick(OWN, step_idx_r<DX, DY, DZ>(c, cx, cy, cz, active && (PRED), NB), snap)
  const T Sx = SV(1, 0, 0, o_x, xp);
  const T Sy = SV(0, 1, 0, o_y, yp);
  const T Sz = SV(0, 0, 1, o_z, zp);
  const T Smx = SV(-1, 0, 0, o_x, xm);
  const T Smxy = SV(-1, 1, 0, o_xy, xm && yp);
  const T Smxz = SV(-1, 0, 1, o_xz, xm && zp);
  const T Smy = SV(0, -1, 0, o_y, ym);
  const T Smyx = SV(1, -1, 0, o_xy, ym && xp);
  const T Smyz = SV(0, -1, 1, o_yz, ym && zp);
  const T Smz = SV(0, 0, -1, o_z, zm);
  const T Smzx = SV(1, 0, -1, o_xz, zm && xp);
  const T Smzy = SV(0, 1, -1, o_yz, zm && yp);
#undef SV

  // flux at the cell (_kernels.pyx:205-220)
  const T gx = xp ? (Sx - S0) * ih : (T)0;
  const T gy = yp ? (Sy - S0) * ih : (T)0;
  const T gz = zp ? (Sz - S0) * ih : (T)0;
  T p0, p1, p2;
  A::flux(gx, gy, gz, p.eps2, p0, p1, p2);
  // backward fluxes, one component each (_kernels.pyx:234-242); the
  // backward cell's own forward step lands on this cell
  T bx = 0, by = 0, bz = 0;
  if (xm) {
    const T hx = (S0 - Smx) * ih;
    const T hy = yp ? (Smxy - Smx) * ih : (T)0;
    const T hz = zp ? (Smxz - Smx) * ih : (T)0;
    bx = A::flux1(hx, hx, hy, hz, p.eps2);
  }
  if (ym) {
    const T hx = xp ? (Smyx - Smy) * ih : (T)0;
    const T hy = (S0 - Smy) * ih;
    const T hz = zp ? (Smyz - Smy) * ih : (T)0;
    by = A::flux1(hy, hx, hy, hz, p.eps2);
  }
  if (zm) {
    const T hx = xp ? (Smzx - Smz) * ih : (T)0;
    const T hy = yp ? (Smzy - Smz) * ih : (T)0;
    const T hz = (S0 - Smz) * ih;
    bz = A::flux1(hz, hx, hy, hz, p.eps2);
  }
  const T div = ((p0 - bx) + (p1 - by) + (p2 - bz)) * ih;

  // data term in view order, zero weights skipped (_kernels.pyx:244-252)
  T num = 0, den = p.gamma, enm = 0;
  auto sample = [&](T wv, float fv) {
    const T d = S0 - (T)fv;
    if (ENERGY) {
      T g, e;
      A::data_both(wv, d, p.eps2, g, e);
      num += g;
      enm += e;
    } else {
      num += A::data_grad(wv, d, p.eps2);
    }
    den += wv;
  };
  if (NV > 0) {
    mbar_wait(&s_bar[stage], (unsigned)(it / kStages) & 1u);
    // view v of the leaf at sf[v * R]; its mask word at the mask tile's
    // entry for the slot / rank
    constexpr int R = sstr;
    const float* sf = s_tile + sbase;
    const int t = packed ? (meta_rbase(meta.y) +
                            __popc(lmask & ((1u << c) - 1u))) & 255
                         : (int)threadIdx.x;
    if (BW == kAllValid && sizeof(T) == 4) {
      // fp32 throughput mode, every sample present: no mask, den = gamma + N,
      // and the samples in pairs through the packed fp32 pipes (FADD2/FFMA2;
      // the two partial sums are added at the end)
      const float2 S2 = make_float2((float)S0, (float)S0);
      const float2 E2 = make_float2((float)p.eps2, (float)p.eps2);
      float2 n2 = make_float2(0.f, 0.f), m2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int v = 0; v < NV; v += 2) {
        const float2 d = sub2(S2, make_float2(sf[v * R],
                                              sf[(v + 1) * R]));
        const float2 q = fma2(d, d, E2);
        const float2 r = make_float2(rsqrtf(q.x), rsqrtf(q.y));
        n2 = fma2(d, r, n2);
        if (ENERGY) m2 = fma2(q, r, m2);
      }
      num = (T)(n2.x + n2.y);
      if (ENERGY) enm = (T)(m2.x + m2.y);
      den += (T)NV;
    } else if (BW == kAllValid) {
      // parity mode: the reference's sequential order, unit weights
#pragma unroll
      for (int v = 0; v < NV; ++v) sample((T)1, sf[v * R]);
    } else if (BINW && sizeof(T) == 4 && NV <= 16) {
      // fp32 throughput mode: unit weights, so den = gamma + count (one
      // rounding instead of one per view; the fp64 parity mode keeps the
      // reference's sequential sum).  cfg2 leaf kernel 0.306 -> 0.298 ms;
      // measured slower at N = 32 (cfg5 3.47 -> 3.53 ms), not used there
      const uint32_t mk = reinterpret_cast<const uint32_t*>(s_tile + NVP * kTileLeaves)[t];
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (mk & (1u << v)) {
          const T d = S0 - (T)sf[v * R];
          if (ENERGY) {
            T g, e;
            A::data_both((T)1, d, p.eps2, g, e);
            num += g;
            enm += e;
          } else {
            num += A::data_grad((T)1, d, p.eps2);
          }
        }
      den += (T)__popc(mk);
    } else if (BINW) {
      const uint32_t mk = reinterpret_cast<const uint32_t*>(s_tile + NVP * kTileLeaves)[t];
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (mk & (1u << v)) sample((T)1, sf[v * R]);
    } else {
      const float* sw = s_tile + NVP * kTileLeaves + sbase;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const float wv = sw[v * R];
        if (wv != 0.f) sample((T)wv, sf[v * R]);
      }
    }
  } else if (ELLV) {  // ELL: the leaf's observed views, in order
    if (active) {
    // rows in batches (kEllPre, then kEllBatch): the (w, f) loads of a batch are issued
    // together (f also for zero-weight padding rows) and consumed in row
    // order -- one load latency per batch instead of two per row; the
    // first batch was requested at the top of the tile
#pragma unroll
    for (int q = 0; q < kEllPre; ++q)
      if (ew0[q] != 0.f) sample((T)ew0[q], ef0[q]);
    for (int r = kEllPre; r < ellK; r += kEllBatch) {
      float wv[kEllBatch], fv[kEllBatch];
#pragma unroll
      for (int q = 0; q < kEllBatch; ++q) {
        const bool on = r + q < ellK;
        wv[q] = on ? __ldg(a.W + ell0 + ((int64_t)(r + q) << 8)) : 0.f;
        fv[q] = on ? __ldg(a.F + ell0 + ((int64_t)(r + q) << 8)) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kEllBatch; ++q)
        if (wv[q] != 0.f) sample((T)wv[q], fv[q]);
    }
    }
  } else if (active) {
    const SIdx q = sidx(a.sd, i, c, meta.y, lmask);
    uint32_t mk = BINW ? __ldg(a.M + q.m) : 0u;
#pragma unroll 4
    for (int v = 0; v < a.nv; ++v) {
      const float fv = __ldg(a.F + q.f + (int64_t)v * q.pitch);
      if (BINW) {
        if ((mk >> v) & 1u) sample((T)1, fv);
      } else {
        const float wv = __ldg(a.W + q.f + (int64_t)v * q.pitch);
        if (wv != 0.f) sample((T)wv, fv);
      }
    }
  }
  const T du = p.lam * div - A::div(num, den);
  T dn = S0 + p.xi * du;
  bool ok_join = false, positive = false;
  double eterm = 0.0;
  if (active) {
    if (ENERGY) {
      const T h = pow2<T>(p.d_max - L);
      const T smooth = p.lam * A::smooth_val(gx, gy, gz, p.eps2);
      eterm = (double)((A::div(enm, den) + smooth) * (h * h * h));
    }
    if (!FROZEN && L < p.d_max && fabs((double)dn) < p.tau_s) {
      a.smark[s] = 1;
      a.split_list[atomicAdd(a.counters, 1)] = s;
    } else {
      if (p.clamp) dn = clamp1(dn);
      a.uval[s] = dn;
      ok_join = (double)dn > p.tau_j || (double)dn < -p.tau_j;
      positive = dn > (T)0;
    }
  }
  if (!FROZEN) {
    // bottom join candidates: blocks of 8 unsplit leaves past tau_j with one
    // sign; without one no join can happen anywhere this pass
    unsigned all = ok_join, pos = ok_join && positive,
             neg = ok_join && !positive;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      all &= __shfl_xor_sync(FULL, all, o);
      pos |= __shfl_xor_sync(FULL, pos, o);
      neg |= __shfl_xor_sync(FULL, neg, o);
    }
    if (c == 0 && inrange && b != 0 && all && !(pos && neg))
      a.join_bot[atomicAdd(a.counters + 1, 1)] = __ldg(a.lpar + i);
  }
  if (ENERGY) {
    // one energy partial per warp (kLeafParts per tile, fixed order: the
    // sum stays deterministic) -- no CTA barrier, so each warp retires as
    // soon as it is done.  fp32 throughput mode at N >= 32: the terms are
    // fp32 values summed in fp32 across the warp; otherwise in double.
    double e;
    if (sizeof(T) == 4 && NV >= 32) {
      float ef = (float)eterm;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ef += __shfl_xor_sync(FULL, ef, o);
      e = (double)ef;
    } else {
      e = eterm;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(FULL, e, o);
    }
    if ((threadIdx.x & 31) == 0)
      a.epart[(int64_t)tile_id * kLeafParts + (threadIdx.x >> 5)] = e;
  }
  // one CTA per tile (the default launch: grid = tiles): no refill, no
  // trailing barrier (measured: the persistent loop's tail cost cfg2 11 %)
  if (!OCTF_PERSIST) break;
  if (NV > 0) {
    // every thread is done with this stage (and the energy scratch): refill
    // it with the tile kStages steps ahead
    __syncthreads();
    const int nt = tile_id + kStages * (int)gridDim.x;
    if (threadIdx.x == 0 && nt < tend && !packed)
      stage_tile<NVP, BW>(s_tile, &s_bar[stage], a.F, aux, nt);
  } else if (ENERGY) {
    __syncthreads();  // the energy scratch is reused by the next tile
  }
  }  // tiles
}
