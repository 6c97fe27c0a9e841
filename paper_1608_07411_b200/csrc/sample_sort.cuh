// One-time per-leaf sort of the sample store for solver="pd".
//
// The primal-dual prox is a generalised weighted median of a leaf's samples
// (oracle/pd_oracle.c wmedian_prox).  The samples never change while a leaf
// exists, so instead of sorting them in every pass the context sorts each
// leaf's vector once, when it is gathered (ctx_gather; new leaves after a pd
// restructure through ctx_list_update), and k_pd_pass only selects on the
// sorted tile.  Order: ascending (f, view index), a -0 sample taken as +0,
// absent samples (weight 0, or a clear mask bit) last as f = +inf with
// weight 0 -- exactly the order the oracle sorts into.
//
// Layout stays [tile][rank][256] (octf_common.cuh samp_idx): rank k of a leaf
// holds its k-th smallest sample; the weight store (general weights) is
// permuted alongside; the mask store is left as gathered (the pd kernel
// counts the finite entries instead).
#pragma once

#include <cstdint>

#include "octf_common.cuh"

namespace octf {
namespace {

// total order of floats as unsigned keys (no NaNs in the store)
__device__ __forceinline__ uint32_t f_ord(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float f_unord(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ void cx_u64(uint64_t& a, uint64_t& b) {
  const uint64_t lo = a < b ? a : b;
  b = a < b ? b : a;
  a = lo;
}

// Batcher odd-even merge sort of N (power of two) keys in registers, by
// template recursion so every index is a compile-time constant
template <int LO, int N, int R>
struct KeyMerge {
  static __device__ __forceinline__ void run(uint64_t* k) {
    if constexpr (2 * R < N) {
      KeyMerge<LO, N, 2 * R>::run(k);
      KeyMerge<LO + R, N, 2 * R>::run(k);
#pragma unroll
      for (int i = LO + R; i + R < LO + N; i += 2 * R) cx_u64(k[i], k[i + R]);
    } else {
      cx_u64(k[LO], k[LO + R]);
    }
  }
};
template <int LO, int N>
struct KeySort {
  static __device__ __forceinline__ void run(uint64_t* k) {
    if constexpr (N > 1) {
      KeySort<LO, N / 2>::run(k);
      KeySort<LO + N / 2, N / 2>::run(k);
      KeyMerge<LO, N, 1>::run(k);
    }
  }
};

// sorts the sample vectors of the leaves list[0 .. *nlist) (slot ids i*8+c
// of the leaf-block list; list null: every leaf of the n slots); NV = the
// store stride (views padded), nv = real views.  M non-null: binary weights
// (bit v of M); else weights in W.  Positions from the store layout sd.
template <int NV>
__global__ void k_sort_samples(const int32_t* __restrict__ list,
                               const int32_t* __restrict__ nlist, int64_t n,
                               int nv, float* F, float* W,
                               const uint32_t* __restrict__ M,
                               const int4* __restrict__ lmeta, SDesc sd) {
  const int64_t cnt = list ? (int64_t)*nlist : n;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
       k += step) {
    const int64_t s = list ? (int64_t)list[k] : k;
    const int4 mt = lmeta[s >> 3];
    const unsigned mask = ((unsigned)mt.w >> 19) & 0xffu;
    const int c = (int)(s & 7);
    if (!list && (!((mask >> c) & 1u) || (mt.x == 0 && c != 0))) continue;
    const SIdx q = sidx(sd, s >> 3, c, mt.y, mask);
    const uint32_t mk = M ? M[q.m] : 0u;
    uint64_t key[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float f = F[q.f + (int64_t)v * q.pitch];
      const bool on = v < nv && (M ? ((mk >> v) & 1u) != 0u
                                   : W[q.f + (int64_t)v * q.pitch] != 0.f);
      const float fz = on ? __fadd_rn(f, 0.f) : __int_as_float(0x7f800000);
      key[v] = ((uint64_t)f_ord(fz) << 32) | (uint32_t)v;
    }
    KeySort<0, NV>::run(key);
    if (!M) {
      // permute the weights (all read before the in-place writes; w is
      // indexed at run time, so it lives in local memory -- a one-time pass)
      float w[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) w[v] = W[q.f + (int64_t)v * q.pitch];
      const uint32_t inf_key = f_ord(__int_as_float(0x7f800000));
#pragma unroll
      for (int r = 0; r < NV; ++r) {
        const int v = (int)(key[r] & 0xffu);
        W[q.f + (int64_t)r * q.pitch] =
            (uint32_t)(key[r] >> 32) == inf_key ? 0.f : w[v];
      }
    }
#pragma unroll
    for (int r = 0; r < NV; ++r)
      F[q.f + (int64_t)r * q.pitch] = f_unord((uint32_t)(key[r] >> 32));
  }
}

// The same order for the per-tile (ELL) store of many-view configurations:
// row r of slot s is at off[s >> 8] + r * 256 + (s & 255), K_t rows per tile.
// A leaf's rows hold its observed views in view order when gathered; a
// stable insertion sort by f (zero-weight padding rows last, as +inf) gives
// the oracle's (f, view) order.  One thread per leaf, in place in global
// memory (a row is coalesced across the tile's threads); O(K^2) moves, once
// per leaf.
__global__ void k_sort_ell(const int32_t* __restrict__ list,
                           const int32_t* __restrict__ nlist, int64_t n,
                           const int32_t* __restrict__ tileK,
                           const int64_t* __restrict__ tileOff, float* F,
                           float* W) {
  const int64_t cnt = list ? (int64_t)*nlist : n;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  constexpr int64_t P = kTileLeaves;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
       k += step) {
    const int64_t s = list ? (int64_t)list[k] : k;
    const int K = tileK[s >> 8];
    float* f = F + tileOff[s >> 8] + (s & 255);
    float* w = W + tileOff[s >> 8] + (s & 255);
    for (int r = 0; r < K; ++r)
      f[r * P] = w[r * P] != 0.f ? __fadd_rn(f[r * P], 0.f)
                                 : __int_as_float(0x7f800000);
    for (int a = 1; a < K; ++a) {
      const float fa = f[a * P], wa = w[a * P];
      int b = a - 1;
      while (b >= 0 && f[b * P] > fa) {
        f[(b + 1) * P] = f[b * P];
        w[(b + 1) * P] = w[b * P];
        --b;
      }
      f[(b + 1) * P] = fa;
      w[(b + 1) * P] = wa;
    }
  }
}

}  // namespace
}  // namespace octf
