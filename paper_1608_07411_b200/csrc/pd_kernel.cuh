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
//           median of the samples, sorted in registers by a bitonic network,
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
#define OCTF_PD_MINB 4  // 4 CTAs of 256 per SM: <= 64 registers
#endif
#ifndef OCTF_PD_MINB_SMALL
#define OCTF_PD_MINB_SMALL 5  // binary weights, N <= 16 (48 regs: cfg2 pd 54.8 -> 58.3 %)
#endif
constexpr int pd_minb(bool binw, int nv) {
  return !binw ? 1 : (nv <= 16 ? OCTF_PD_MINB_SMALL : OCTF_PD_MINB);
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

// ascending compare-exchange: keys only (binary weights: equal keys are
// interchangeable, so min/max suffices) or (key, weight, view index) with the
// index tie-break of oracle/pd_oracle.c
template <bool WEIGHTED>
__device__ __forceinline__ void cx(float& fa, float& wa, int& ia, float& fb,
                                   float& wb, int& ib) {
  if (WEIGHTED) {
    const bool gt = fa > fb || (fa == fb && ia > ib);
    if (gt) {
      float t = fa; fa = fb; fb = t;
      t = wa; wa = wb; wb = t;
      int u = ia; ia = ib; ib = u;
    }
  } else {
    const float lo = fminf(fa, fb);
    fb = fmaxf(fa, fb);
    fa = lo;
  }
}

// Batcher odd-even merge sort of N (power of two) entries in registers,
// ascending: 191 comparators at N = 32 (bitonic: 240).  Written as template
// recursion so every register index is a compile-time constant.
template <int LO, int N, int R, bool WEIGHTED>
struct OeMerge {
  static __device__ __forceinline__ void run(float* f, float* w, int* ix) {
    if constexpr (2 * R < N) {
      OeMerge<LO, N, 2 * R, WEIGHTED>::run(f, w, ix);
      OeMerge<LO + R, N, 2 * R, WEIGHTED>::run(f, w, ix);
#pragma unroll
      for (int i = LO + R; i + R < LO + N; i += 2 * R)
        cx<WEIGHTED>(f[i], w[i], ix[i], f[i + R], w[i + R], ix[i + R]);
    } else {
      cx<WEIGHTED>(f[LO], w[LO], ix[LO], f[LO + R], w[LO + R], ix[LO + R]);
    }
  }
};

template <int LO, int N, bool WEIGHTED>
struct OeSort {
  static __device__ __forceinline__ void run(float* f, float* w, int* ix) {
    if constexpr (N > 1) {
      OeSort<LO, N / 2, WEIGHTED>::run(f, w, ix);
      OeSort<LO + N / 2, N / 2, WEIGHTED>::run(f, w, ix);
      OeMerge<LO, N, 1, WEIGHTED>::run(f, w, ix);
    }
  }
};

template <int N, bool WEIGHTED>
__device__ __forceinline__ void oddeven_sort(float* f, float* w, int* ix) {
  OeSort<0, N, WEIGHTED>::run(f, w, ix);
}

// max_k min(sorted(X)_k, c_{o+k}) for a bitonic X[0..M) (ascending then
// descending), c_k = v0 - cc*(2k - W) non-increasing, folded into acc.  A
// half-cleaner splits X into L <= H (both bitonic); since "c_k > X_(k)"
// holds exactly below the crossing k*, one half's contribution is trivial
// -- max(L) = L_(M/2-1) if the crossing lies in H, else c_{o+M/2} -- and
// only the other half is refined: M-1 comparators plus M-1 selects instead
// of the M log M / 2 of a merge followed by a scan.
template <typename T, int M>
__device__ __forceinline__ void bitonic_select(float* X, T& ko, T& acc, T v0,
                                               T cc, T W) {
  if constexpr (M == 1) {
    const T c = v0 - cc * ((T)2 * ko - W);
    acc = fmax(acc, fmin((T)X[0], c));
  } else {
    constexpr int H = M / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const float l = fminf(X[i], X[i + H]);
      X[i + H] = fmaxf(X[i], X[i + H]);
      X[i] = l;
    }
    float mL = X[0];
#pragma unroll
    for (int i = 1; i < H; ++i) mL = fmaxf(mL, X[i]);
    const T cl = v0 - cc * ((T)2 * (ko + (T)(H - 1)) - W);
    const T ch = v0 - cc * ((T)2 * (ko + (T)H) - W);
    const bool inH = cl > (T)mL;
    acc = fmax(acc, inH ? (T)mL : ch);
#pragma unroll
    for (int i = 0; i < H; ++i) X[i] = inH ? X[i + H] : X[i];
    ko = inH ? ko + (T)H : ko;
    bitonic_select<T, H>(X, ko, acc, v0, cc, W);
  }
}

// General weights without carrying them through the sort (NV = 64): the
// breakpoint at sorted position k is c'_k = v0 - cc*(2 S(f_(k)) - W) with
// S(a) = sum of the weights of samples strictly below a (view order).  A
// tie group's first element has S_k = S(a) and later ones only smaller
// breakpoints, so max_k min(f_(k), c'_k) equals the sorted scan's value;
// with dyadic view-tree weights the f64 sums are exact in any order.  The
// selection needs c' only at O(log NV) positions, each an O(NV) pass over
// the leaf's samples (f staged in shared memory, weights from global).
template <typename T, int NV>
struct WeightAt {
  const float* fs;     // s_tile + t: f of view v at fs[v * kTileLeaves]
  const float* wg;     // weights of view v at wg[v * kTileLeaves]
  __device__ __forceinline__ T below(float a) const {
    T S = 0;
#pragma unroll 8
    for (int v = 0; v < NV; ++v) {
      const float wv = __ldg(wg + v * kTileLeaves);
      if (fs[v * kTileLeaves] < a) S += (T)wv;
    }
    return S;
  }
};

template <typename T, int M, int NV>
__device__ __forceinline__ void bitonic_select_w(float* X, T& acc, T v0, T cc,
                                                 T W,
                                                 const WeightAt<T, NV>& wa) {
  if constexpr (M == 1) {
    const T c = v0 - cc * ((T)2 * wa.below(X[0]) - W);
    acc = fmax(acc, fmin((T)X[0], c));
  } else {
    constexpr int H = M / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const float l = fminf(X[i], X[i + H]);
      X[i + H] = fmaxf(X[i], X[i + H]);
      X[i] = l;
    }
    float mL = X[0], mH = X[H];
#pragma unroll
    for (int i = 1; i < H; ++i) {
      mL = fmaxf(mL, X[i]);
      mH = fminf(mH, X[H + i]);
    }
    const T cl = v0 - cc * ((T)2 * wa.below(mL) - W);
    const bool inH = cl > (T)mL;
    const T ch = inH ? (T)0 : v0 - cc * ((T)2 * wa.below(mH) - W);
    acc = fmax(acc, inH ? (T)mL : ch);
#pragma unroll
    for (int i = 0; i < H; ++i) X[i] = inH ? X[i + H] : X[i];
    bitonic_select_w<T, H, NV>(X, acc, v0, cc, W, wa);
  }
}

// shared memory of k_pd_pass: the f tile, then the mask tile (binary
// weights) or the weight tile (NV <= 32; at NV = 64 weights stay in global)
constexpr size_t pd_smem_bytes(int nv, bool binw) {
  return (size_t)nv * kTileLeaves * 4 +
         (binw ? (size_t)kTileLeaves * 4
               : (nv > 32 ? 0 : (size_t)nv * kTileLeaves * 4));
}

// WP: also write the bottom propagate level of the five fields (frozen
// passes over a full leaf-block list)
template <typename T, bool BINW, int NV, bool WP = false>
__global__ void __launch_bounds__(kT, pd_minb(BINW, NV)) k_pd_pass(PdArgs<T> a) {
  static_assert(NV > 0 && (NV & (NV - 1)) == 0, "NV: power of two");
  // NV = 64: general weights selected without sorting them (WeightAt)
  constexpr bool WSEL = NV > 32;
  static_assert(!(WSEL && BINW), "the mask format holds 32 views");
  const int gid = (int)(blockIdx.x * kT + threadIdx.x);
  const int i = gid >> 3;
  const int c = gid & 7;
  const bool inrange = i < (int)a.nlb;
  // samples: the CTA's tile staged by one TMA bulk copy (as k_leaf_pass),
  // read into registers only after the stencil, so the stencil values and
  // the sort network never hold registers at the same time
  extern __shared__ __align__(128) float s_tile[];
  __shared__ __align__(8) uint64_t s_bar;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    const size_t tile = blockIdx.x;
    const unsigned fbytes = NV * kTileLeaves * 4;
    const unsigned abytes = BINW ? kTileLeaves * 4 : (WSEL ? 0 : fbytes);
    mbar_expect_tx(&s_bar, fbytes + abytes);
    bulk_g2s(s_tile, a.F + tile * NV * kTileLeaves, fbytes, &s_bar);
    if (BINW)
      bulk_g2s(s_tile + NV * kTileLeaves, a.M + tile * kTileLeaves, abytes,
               &s_bar);
    else if (!WSEL)
      bulk_g2s(s_tile + NV * kTileLeaves, a.W + tile * NV * kTileLeaves,
               abytes, &s_bar);
  }
  __syncthreads();
  const int4 meta = inrange ? __ldg(a.lmeta + i) : make_int4(0, 0, 0, 0);
  const int32_t b = meta.x;
  const int32_t s = b + c;
  int L, pz;
  unsigned lmask;
  unpack_meta_w(meta.w, pz, lmask, L);
  const int px = meta.y, py = meta.z;
  const bool slot_ok = inrange && !(b == 0 && c != 0);
  const bool active = slot_ok && ((lmask >> c) & 1u);
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

  // samples from the staged tile, view order
  mbar_wait(&s_bar, 0);
  const int t = threadIdx.x;
  float f[NV];
  float w[NV];  // (only the general-weight sort carries them)
  int ix[NV];
  uint32_t mk = 0u;
  T W = 0, num = 0;
  if (BINW) {  // valid views of this leaf; W = their count
    mk = reinterpret_cast<const uint32_t*>(s_tile + NV * kTileLeaves)[t];
    if (a.nv < 32) mk &= (1u << a.nv) - 1u;
    W = (T)__popc(mk);
  }
  // energy numerator in view order; absent samples become +inf (sort last)
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const float fv = s_tile[v * kTileLeaves + t];
    const float wv =
        BINW ? 1.f
             : (WSEL ? __ldg(a.W + (size_t)blockIdx.x * NV * kTileLeaves +
                             v * kTileLeaves + t)
                     : s_tile[(NV + v) * kTileLeaves + t]);
    const bool on = BINW ? ((mk >> v) & 1u) != 0u : (v < a.nv && wv != 0.f);
    if (on) {
      if (!BINW) W += (T)wv;
      num += BINW ? (T)fabs(U0 - (T)fv) : (T)wv * fabs(U0 - (T)fv);
    }
    f[v] = on ? __fadd_rn(fv, 0.f) : __int_as_float(0x7f800000);  // -0 -> +0
    if (!BINW && !WSEL) {
      w[v] = on ? wv : 0.f;
      ix[v] = v;
    }
  }
  const T den = W + a.gamma;
  const T cc = a.tau / den;
  T res0 = -(T)INFINITY;
  if (BINW || WSEL) {
    // two sorted halves, the second read backwards: a bitonic sequence
    // whose order statistics are those of all samples
    oddeven_sort<NV / 2, false>(f, w, ix);
    oddeven_sort<NV / 2, false>(f + NV / 2, w, ix);
#pragma unroll
    for (int i = 0; i < NV / 4; ++i) {
      const float t = f[NV / 2 + i];
      f[NV / 2 + i] = f[NV - 1 - i];
      f[NV - 1 - i] = t;
    }
    if (WSEL) {
      res0 = v0 - cc * W;  // k = NV: f = +inf, S = W
      const WeightAt<T, NV> wa{
          s_tile + t, a.W + (size_t)blockIdx.x * NV * kTileLeaves + t};
      bitonic_select_w<T, NV, NV>(f, res0, v0, cc, W, wa);
    } else {
      res0 = v0 - cc * ((T)2 * (T)NV - W);  // k = NV: f = +inf
      T ko = 0;
      bitonic_select<T, NV>(f, ko, res0, v0, cc, W);
    }
  } else {
    oddeven_sort<NV, true>(f, w, ix);
    // generalised weighted median (oracle/pd_oracle.c wmedian_prox).  With
    // S_k the weight of the first k sorted samples and c_k = v0 - cc*(2 S_k
    // - W), the scan returns at the first k* with c_k* <= f[k*]:
    // max(c_k*, f[k*-1]).  c_k is non-increasing and f non-decreasing, so
    // min(f[k], c_k) is f[k] for k < k* and c_k after, and that value is
    // max_k min(f[k], c_k) (f[NV] = +inf) -- two min/max per sample, no
    // branches.  Absent samples (+inf, weight 0) leave S unchanged.  (With
    // unit weights S_k = k: the BINW branch above, same value.)
    T S = 0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const T cand = v0 - cc * ((T)2 * S - W);
      res0 = fmax(res0, fmin(cand, (T)f[k]));
      S += (T)w[k];
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
      a.epart[blockIdx.x] = tot;
    }
  } else {
    typedef cub::BlockReduce<double, kT> BR;
    __shared__ typename BR::TempStorage tmp;
    const double tot = BR(tmp).Sum(eterm);
    if (threadIdx.x == 0) a.epart[blockIdx.x] = tot;
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
}
