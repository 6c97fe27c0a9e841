// TV-L1 primal-dual leaf kernel (solver="pd").
//
// Included by solver_impl.cuh inside namespace octf::{anonymous}.
// The reference has no primal-dual solver; the definition
// this kernel implements is written down in oracle/pd_oracle.c, which is the
// (unpinned) oracle it is tested against.  Per leaf, Jacobi on a frozen
// tree, from the pass-start snapshots of u, ubar and p = (px, py, pz):
//   dual    p'(q) = P(p(q) + sigma*lam*grad ubar(q)) at the cell and at its
//           three backward neighbours (each evaluated at the leaf's level),
//   primal  u' = prox_{tau D}(u + tau*lam*div p'): generalised weighted
//           median of the samples, pre-sorted once per leaf when gathered
//           (sample_sort.cuh): a binary search (unit weights) or one scan,
//   ubar' = 2u' - u, and the energy of the incoming u (exact TV + L1 data).
// Same mapping as k_leaf_pass: 8 lanes per block, own-block values by
// shuffle, neighbour blocks through the 12-entry table.
#pragma once

#ifndef OCTF_PD_F32_ESUM_MIN
// fp32 warp energy sums from this N (cfg2 pd pass 0.589 -> 0.577 ms, cfg5
// kernel 5.41 -> 5.34 ms; the fp64 parity mode keeps the double reduction)
#define OCTF_PD_F32_ESUM_MIN 16
#endif
#ifndef OCTF_PD_MINB
#define OCTF_PD_MINB 5  // 5 CTAs of 256 per SM: <= 48 registers (profiles/r02)
#endif
#ifndef OCTF_PD_MINB_SMALL
#define OCTF_PD_MINB_SMALL 5  // binary weights, N <= 16 (48 regs: cfg2 pd 54.8 -> 58.3 %)
#endif
constexpr int pd_minb(bool binw, int nv, int tbytes) {
  // (the f64 parity mode: 48 registers would spill)
  return tbytes == 8 || !binw ? 1
                              : (nv <= 16 ? OCTF_PD_MINB_SMALL : OCTF_PD_MINB);
}

template <typename T>
struct PdArgs {
  const int32_t* __restrict__ lblocks;
  int64_t nlb;
  const int4* __restrict__ lmeta;
  const int32_t* __restrict__ nbr;
  const T* __restrict__ u;
  const T* __restrict__ ub;
  const T* __restrict__ px;
  const T* __restrict__ py;
  const T* __restrict__ pz;
  T* __restrict__ u_o;
  T* __restrict__ ub_o;
  T* __restrict__ px_o;
  T* __restrict__ py_o;
  T* __restrict__ pz_o;
  const float* __restrict__ F;
  const float* __restrict__ W;
  const uint32_t* __restrict__ M;
  int64_t stride;
  int nv;
  int d_max;
  T lam, tl, sl, tau, gamma;  // tl = tau*lam, sl = sigma*lam
  int clamp;
  double* epart;
  const int32_t* __restrict__ lpar;  // parent slot of each leaf block
  const int32_t* __restrict__ tileK = nullptr;   // ELL store (views > 64):
  const int64_t* __restrict__ tileOff = nullptr; // rows per tile, offsets
  SDesc sd;  // the dense sample store's layout (octf_common.cuh)
};

template <typename T>
__device__ __forceinline__ T maxT(T a, T b) {
  return a > b ? a : b;
}

// dual update of one cell: P(p + sl*g); returns the requested component
template <typename T>
__device__ __forceinline__ void dual3(T p0, T p1, T p2, T gx, T gy, T gz, T sl,
                                      T& o0, T& o1, T& o2) {
  const T ax = p0 + sl * gx;
  const T ay = p1 + sl * gy;
  const T az = p2 + sl * gz;
  const T nrm = sqrt(ax * ax + ay * ay + az * az);
  const T s = maxT(nrm, (T)1);
  o0 = ax / s;
  o1 = ay / s;
  o2 = az / s;
}

// shared memory of k_pd_pass: the sorted f tile, then (general weights,
// NV <= 32) the weight tile permuted alongside; at NV = 64 the weights are
// read from global memory (coalesced, once per scan)
constexpr size_t pd_smem_bytes(int nv, bool binw) {  // one stage
  return (size_t)nv * kTileLeaves * 4 +
         (binw || nv > 32 ? 0 : (size_t)nv * kTileLeaves * 4);
}

// WP: also write the bottom propagate level of the five fields (frozen
// passes over a full leaf-block list)
// EL: the per-tile (ELL) store of many-view configurations -- a leaf's rows
// are its observed views' (f, w), sorted by (f, view) once at gather
// (k_sort_ell), K_t rows per tile read from global memory (coalesced: a
// row holds the tile's 256 slots); zero-weight rows are padding and are
// skipped, as in the descent kernel.  NV is unused (1).
template <typename T, int BW, int NV, bool WP = false, bool PK = false,
          bool EL = false>
__global__ void __launch_bounds__(kT, pd_minb(BW != kWeights, NV, sizeof(T))) k_pd_pass(PdArgs<T> a) {
  static_assert(NV > 0 && (NV & (NV - 1)) == 0, "NV: power of two");
  static_assert(!EL || (BW == kWeights && !WP && !PK), "ELL: weights only");
  constexpr bool BINW = BW != kWeights;  // unit weights (+inf = absent)
  // NV = 64, general weights: only the f tile is staged (weights from global)
  constexpr bool WGLOB = NV > 32;
  static_assert(!(WGLOB && BINW), "the mask format holds 32 views");
  // persistent, as k_leaf_pass: kStages buffers of the sorted sample tile
  // (and the weight tile), the copy of a later tile in flight while the
  // current one is computed
  constexpr size_t STAGE = pd_smem_bytes(NV, BINW) / 4;
  extern __shared__ __align__(128) float s_smem[];
  __shared__ __align__(8) uint64_t s_bar[kStages];
  const int ntiles = (int)((a.nlb * 8 + kTileLeaves - 1) / kTileLeaves);
  // the sorted sample tile (and the weight tile): whole (nchunks = -2),
  // or packed (octf_common.cuh SDesc) in two parts like k_leaf_pass's
  // stage_packed -- the first kEarlyChunks chunks (nchunks = -1), then the
  // rest of the tile's ceil(n_t / 32) chunks
  constexpr bool packed = PK;  // the packed sample store (SDesc)
  auto stage_pd = [&](float* buf, uint64_t* bar, int tile, int nchunks) {
    constexpr bool WST = !(BINW || WGLOB);  // weights staged too
    const size_t fo = (size_t)tile * NV * kTileLeaves;
    size_t off = 0;
    unsigned bytes = NV * kTileLeaves * 4;
    if (nchunks == -1) {
      bytes = kEarlyChunks * NV * kChunk * 4;
    } else if (nchunks >= 0) {
      const int rest = nchunks > kEarlyChunks ? nchunks - kEarlyChunks : 0;
      off = (size_t)kEarlyChunks * NV * kChunk;
      bytes = rest * NV * kChunk * 4;
    }
    mbar_expect_tx(bar, WST ? 2 * bytes : bytes);
    if (!bytes) return;
    bulk_g2s(buf + off, a.F + fo + off, bytes, bar);
    if (WST) bulk_g2s(buf + NV * kTileLeaves + off, a.W + fo + off, bytes, bar);
  };
  if (threadIdx.x == 0 && !EL) {
    for (int k = 0; k < kStages; ++k) mbar_init(&s_bar[k], packed ? 2 : 1);
    for (int k = 0; k < kStages && !packed; ++k) {
      const int t = (int)blockIdx.x + k * (int)gridDim.x;
      if (t < ntiles) stage_pd(s_smem + k * STAGE, &s_bar[k], t, -2);
    }
  }
  __syncthreads();
  int it = 0;
  for (int tile_id = (int)blockIdx.x; tile_id < ntiles;
       tile_id += (int)gridDim.x, ++it) {
  const int stage = it % kStages;
  float* const s_tile = s_smem + stage * STAGE;
  const int gid = tile_id * kT + (int)threadIdx.x;
  const int i = gid >> 3;
  const int c = gid & 7;
  const bool inrange = i < (int)a.nlb;
  if (packed && threadIdx.x == 0)
    stage_pd(s_tile, &s_bar[stage], tile_id, -1);
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
  // among the tile's leaves at chunk r / kChunk, entry r % kChunk, sorted ranks kChunk
  // apart
  int sp = threadIdx.x;
  constexpr int R = PK ? kChunk : kTileLeaves;
  if (packed) {
    const int r = (meta_rbase(meta.y) + __popc(lmask & ((1u << c) - 1u))) & 255;
    sp = (r / kChunk) * NV * kChunk + (r % kChunk);
    if (threadIdx.x == kT - 1)  // n_t from the tile's last block
      stage_pd(s_tile, &s_bar[stage], tile_id,
               inrange ? (meta_rbase(meta.y) + __popc(lmask) + kChunk - 1) / kChunk
                       : kTileLeaves / kChunk);
  }
  const int cx = (c >> 2) & 1, cy = (c >> 1) & 1, cz = c & 1;
  const int x = 2 * px + cx, y = 2 * py + cy, z = 2 * pz + cz;
  const int m = 1 << L;
  const T ih = inv_spacing<T>(a.d_max, L);
  const int32_t* nb = a.nbr + i * 12;
  const unsigned FULL = 0xffffffffu;
  const bool xp = x + 1 < m, yp = y + 1 < m, zp = z + 1 < m;
  const bool xm = x > 0, ym = y > 0, zm = z > 0;

  const int32_t par_blk =
      (WP && c == 0 && inrange && lmask == 0xffu && L == a.d_max)
          ? __ldg(a.lpar + i) : -1;
  const T U0 = slot_ok ? a.u[s] : (T)0;
  const T B0 = slot_ok ? a.ub[s] : (T)0;
  const T P0 = slot_ok ? a.px[s] : (T)0;
  const T P1 = slot_ok ? a.py[s] : (T)0;
  const T P2 = slot_ok ? a.pz[s] : (T)0;
  // one neighbour-table lookup per stencil direction, shared by the fields
  int32_t N[12];
  {
    const int4* nb4 = reinterpret_cast<const int4*>(nb);
    const int4 n0 = active ? __ldg(nb4) : make_int4(-1, -1, -1, -1);
    const int4 n1 = active ? __ldg(nb4 + 1) : make_int4(-1, -1, -1, -1);
    const int4 n2 = active ? __ldg(nb4 + 2) : make_int4(-1, -1, -1, -1);
    N[0] = n0.x; N[1] = n0.y; N[2] = n0.z; N[3] = n0.w;
    N[4] = n1.x; N[5] = n1.y; N[6] = n1.z; N[7] = n1.w;
    N[8] = n2.x; N[9] = n2.y; N[10] = n2.z; N[11] = n2.w;
  }
#define IX(DX, DY, DZ, PRED) step_idx_r<DX, DY, DZ>(c, cx, cy, cz, active && (PRED), N)
  const int ixp = IX(1, 0, 0, xp), iyp = IX(0, 1, 0, yp), izp = IX(0, 0, 1, zp);
  const int ixm = IX(-1, 0, 0, xm), iym = IX(0, -1, 0, ym), izm = IX(0, 0, -1, zm);
  const int ixmyp = IX(-1, 1, 0, xm && yp), ixmzp = IX(-1, 0, 1, xm && zp);
  const int iymxp = IX(1, -1, 0, ym && xp), iymzp = IX(0, -1, 1, ym && zp);
  const int izmxp = IX(1, 0, -1, zm && xp), izmyp = IX(0, 1, -1, zm && yp);
#undef IX
#define SH(V, MASK) __shfl_xor_sync(FULL, V, MASK)
  // ubar at the 13-point stencil
  const T Bx = pick(SH(B0, 4), ixp, a.ub);
  const T By = pick(SH(B0, 2), iyp, a.ub);
  const T Bz = pick(SH(B0, 1), izp, a.ub);
  const T Bmx = pick(SH(B0, 4), ixm, a.ub);
  const T Bmxy = pick(SH(B0, 6), ixmyp, a.ub);
  const T Bmxz = pick(SH(B0, 5), ixmzp, a.ub);
  const T Bmy = pick(SH(B0, 2), iym, a.ub);
  const T Bmyx = pick(SH(B0, 6), iymxp, a.ub);
  const T Bmyz = pick(SH(B0, 3), iymzp, a.ub);
  const T Bmz = pick(SH(B0, 1), izm, a.ub);
  const T Bmzx = pick(SH(B0, 5), izmxp, a.ub);
  const T Bmzy = pick(SH(B0, 3), izmyp, a.ub);
  // p at the three backward neighbours (all components, for the norms)
  const T Qx0 = pick(SH(P0, 4), ixm, a.px), Qx1 = pick(SH(P1, 4), ixm, a.py),
          Qx2 = pick(SH(P2, 4), ixm, a.pz);
  const T Qy0 = pick(SH(P0, 2), iym, a.px), Qy1 = pick(SH(P1, 2), iym, a.py),
          Qy2 = pick(SH(P2, 2), iym, a.pz);
  const T Qz0 = pick(SH(P0, 1), izm, a.px), Qz1 = pick(SH(P1, 1), izm, a.py),
          Qz2 = pick(SH(P2, 1), izm, a.pz);
  // u at the forward neighbours (energy of the incoming state)
  const T Ux = pick(SH(U0, 4), ixp, a.u);
  const T Uy = pick(SH(U0, 2), iyp, a.u);
  const T Uz = pick(SH(U0, 1), izp, a.u);
#undef SH

  // dual at the cell
  const T gx = xp ? (Bx - B0) * ih : (T)0;
  const T gy = yp ? (By - B0) * ih : (T)0;
  const T gz = zp ? (Bz - B0) * ih : (T)0;
  T D0, D1, D2, t0, t1, t2;
  dual3<T>(P0, P1, P2, gx, gy, gz, a.sl, D0, D1, D2);
  T bx = 0, by = 0, bz = 0;
  if (xm) {
    dual3<T>(Qx0, Qx1, Qx2, (B0 - Bmx) * ih, yp ? (Bmxy - Bmx) * ih : (T)0,
             zp ? (Bmxz - Bmx) * ih : (T)0, a.sl, t0, t1, t2);
    bx = t0;
  }
  if (ym) {
    dual3<T>(Qy0, Qy1, Qy2, xp ? (Bmyx - Bmy) * ih : (T)0, (B0 - Bmy) * ih,
             zp ? (Bmyz - Bmy) * ih : (T)0, a.sl, t0, t1, t2);
    by = t1;
  }
  if (zm) {
    dual3<T>(Qz0, Qz1, Qz2, xp ? (Bmzx - Bmz) * ih : (T)0,
             yp ? (Bmzy - Bmz) * ih : (T)0, (B0 - Bmz) * ih, a.sl, t0, t1, t2);
    bz = t2;
  }
  const T div = ((D0 - bx) + (D1 - by) + (D2 - bz)) * ih;
  const T v0 = U0 + a.tl * div;

  // samples: the leaf's vector is sorted ascending by (f, view), absent
  // entries last as +inf with weight 0 (sample_sort.cuh, once per leaf)
  if (!EL) mbar_wait(&s_bar[stage], (unsigned)(it / kStages) & 1u);
  const int t = threadIdx.x;
  const float* ft = s_tile + sp;  // rank k at ft[k * R]
  const float* wsm = s_tile + NV * kTileLeaves + sp;
  const float* wgl = a.W + (size_t)tile_id * NV * kTileLeaves + sp;
  auto wt = [&](int k) -> float {
    return WGLOB ? __ldg(wgl + k * R) : wsm[k * R];
  };
  // weight sum and the energy numerator, sorted order (pd_oracle.c)
  T W = 0, num = 0;
  const int ellK = EL ? __ldg(a.tileK + tile_id) : 0;
  const float* const ef = EL ? a.F + __ldg(a.tileOff + tile_id) + t : nullptr;
  const float* const ew = EL ? a.W + __ldg(a.tileOff + tile_id) + t : nullptr;
  // (ELL rows in batches of four: the (w, f) loads of a batch are issued
  // together and consumed in row order, as in the descent kernel)
  constexpr int kEB = 4;
  if (EL) {
    for (int k0 = 0; k0 < ellK; k0 += kEB) {
      float wv[kEB], fv[kEB];
#pragma unroll
      for (int q = 0; q < kEB; ++q) {
        const bool on = k0 + q < ellK;
        wv[q] = on ? __ldg(ew + (size_t)(k0 + q) * kTileLeaves) : 0.f;
        fv[q] = on ? __ldg(ef + (size_t)(k0 + q) * kTileLeaves) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kEB; ++q)
        if (wv[q] != 0.f) {
          W += (T)wv[q];
          num += (T)wv[q] * fabs(U0 - (T)fv[q]);
        }
    }
  } else if (BW == kAllValid) {  // every sample present: W = N
#pragma unroll
    for (int k = 0; k < NV; ++k) num += (T)fabs(U0 - (T)ft[k * R]);
    W = (T)NV;
  } else if (BW == kMask) {
    // unit weights: the present samples are the finite prefix; its length by
    // bisection on the +inf tail, then the sum over it
    int nval = 0;
#pragma unroll
    for (int step = NV / 2; step >= 1; step >>= 1)
      nval = ft[(nval + step - 1) * R] == __int_as_float(0x7f800000)
                 ? nval : nval + step;
    nval += ft[nval * R] == __int_as_float(0x7f800000) ? 0 : 1;
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (k < nval) num += (T)fabs(U0 - (T)ft[k * R]);
    W = (T)nval;
  } else {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const float wv = wt(k);
      if (wv != 0.f) {
        W += (T)wv;
        num += (T)wv * fabs(U0 - (T)ft[k * R]);
      }
    }
  }
  const T den = W + a.gamma;
  const T cc = a.tau / den;
  // generalised weighted median (oracle/pd_oracle.c wmedian_prox): with S_k
  // the weight of the first k sorted samples and c_k = v0 - cc*(2 S_k - W)
  // (non-increasing in k) against the non-decreasing f_k (+inf past the
  // present samples), the oracle's scan stops at the first k* with
  // c_k* <= f_k* and returns max(f_(k*-1), c_k*)
  T res0;
  if (EL) {
    // the general-weight scan below over the leaf's observed rows
    res0 = -(T)INFINITY;
    T S = 0;
    for (int k0 = 0; k0 < ellK; k0 += kEB) {
      float wv[kEB], fv[kEB];
#pragma unroll
      for (int q = 0; q < kEB; ++q) {
        const bool on = k0 + q < ellK;
        wv[q] = on ? __ldg(ew + (size_t)(k0 + q) * kTileLeaves) : 0.f;
        fv[q] = on ? __ldg(ef + (size_t)(k0 + q) * kTileLeaves) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kEB; ++q) {
        if (wv[q] == 0.f) continue;
        const T cand = v0 - cc * ((T)2 * S - W);
        res0 = fmax(res0, fmin(cand, (T)fv[q]));
        S += (T)wv[q];
      }
    }
    res0 = fmax(res0, v0 - cc * ((T)2 * S - W));
  } else if (BW != kWeights) {
    // unit weights, S_k = k: k* by branch-free bisection on the tile (the
    // predicate is monotone over all NV ranks; k* = NV only if none holds)
    auto below = [&](int k) {  // c_k > f_k: k* lies beyond k
      return v0 - cc * ((T)2 * (T)k - W) > (T)ft[k * R];
    };
    int pos = 0;
#pragma unroll
    for (int step = NV / 2; step >= 1; step >>= 1)
      pos = below(pos + step - 1) ? pos + step : pos;
    pos += below(pos) ? 1 : 0;
    const T ck = v0 - cc * ((T)2 * (T)pos - W);
    res0 = pos > 0 ? fmax((T)ft[(pos - 1) * R], ck) : ck;
  } else {
    // general weights: the prefix sums are needed, so one branch-free scan
    // (min(f_k, c_k) is f_k below k* and c_k from k*: the max is the value)
    res0 = -(T)INFINITY;
    T S = 0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const T cand = v0 - cc * ((T)2 * S - W);
      res0 = fmax(res0, fmin(cand, (T)ft[k * R]));
      S += (T)wt(k);
    }
    res0 = fmax(res0, v0 - cc * ((T)2 * S - W));
  }
  T res = res0;
  if (a.clamp) res = clamp1(res);
  double eterm = 0.0;
  const T ubv = (T)2 * res - U0;
  if (active) {
    a.u_o[s] = res;
    a.ub_o[s] = ubv;
    a.px_o[s] = D0;
    a.py_o[s] = D1;
    a.pz_o[s] = D2;
    const T ugx = xp ? (Ux - U0) * ih : (T)0;
    const T ugy = yp ? (Uy - U0) * ih : (T)0;
    const T ugz = zp ? (Uz - U0) * ih : (T)0;
    const T tv = a.lam * sqrt(ugx * ugx + ugy * ugy + ugz * ugz);
    const T h = pow2<T>(a.d_max - L);
    eterm = (double)((num / den + tv) * (h * h * h));
  }
  // the bottom propagate level of the five fields for the CTA's finest-level
  // blocks (as k_leaf_pass): staged in shared memory, summed after the
  // energy reduction's barrier by one thread per block
  __shared__ T s_v[WP ? 5 : 1][WP ? kT : 1];
  __shared__ int32_t s_par[WP ? kT / 8 : 1];
  if (WP) {
    s_v[0][t] = res;
    s_v[1][t] = ubv;
    s_v[2][t] = D0;
    s_v[3][t] = D1;
    s_v[4][t] = D2;
    if (c == 0) s_par[t >> 3] = par_blk;
  }
  if (sizeof(T) == 4 && NV >= OCTF_PD_F32_ESUM_MIN) {
    // fp32 throughput mode: warps sum the (fp32) terms in fp32, thread 0
    // adds the eight warp sums in double (fixed order)
    __shared__ double s_w[kT / 32];
    float e = (float)eterm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(FULL, e, o);
    if ((t & 31) == 0) s_w[t >> 5] = (double)e;
    __syncthreads();
    if (t == 0) {
      double tot = 0.0;
#pragma unroll
      for (int k = 0; k < kT / 32; ++k) tot += s_w[k];
      a.epart[tile_id] = tot;
    }
  } else {
    typedef cub::BlockReduce<double, kT> BR;
    __shared__ typename BR::TempStorage tmp;
    const double tot = BR(tmp).Sum(eterm);
    if (threadIdx.x == 0) a.epart[tile_id] = tot;
  }
  if (WP && t < 5 * (kT / 8)) {
    // warp q writes field q of the 32 blocks (a short tail: the CTA's slot
    // is held until its last warp exits)
    const int q = t >> 5, j = t & 31;
    const int32_t par = s_par[j];
    if (par >= 0) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += (double)s_v[q][j * 8 + k];
      T* const o = q == 0 ? a.u_o : q == 1 ? a.ub_o : q == 2 ? a.px_o
                 : q == 3 ? a.py_o : a.pz_o;
      o[par] = (T)(acc / 8.0);
    }
  }
  if (!OCTF_PERSIST) break;  // one CTA per tile (the default launch)
  // every thread is done with this stage and the shared scratch: refill the
  // stage with the tile kStages steps ahead
  __syncthreads();
  const int nt = tile_id + kStages * (int)gridDim.x;
  if (threadIdx.x == 0 && nt < ntiles && !packed)
    stage_pd(s_tile, &s_bar[stage], nt, -2);
  }  // tiles
}
