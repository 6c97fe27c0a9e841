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

// compare-swap on (key, weight, view index) with index tie-break
template <bool WEIGHTED>
__device__ __forceinline__ void cas(float& fa, float& wa, int& ia, float& fb,
                                    float& wb, int& ib, bool up) {
  const bool gt = WEIGHTED ? (fa > fb || (fa == fb && ia > ib)) : (fa > fb);
  if (gt == up) {
    float t = fa; fa = fb; fb = t;
    if (WEIGHTED) {
      t = wa; wa = wb; wb = t;
      int u = ia; ia = ib; ib = u;
    }
  }
}

// in-register bitonic sort of N (power of two) entries, ascending
template <int N, bool WEIGHTED>
__device__ __forceinline__ void bitonic(float* f, float* w, int* ix) {
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int l = i ^ j;
        if (l > i) cas<WEIGHTED>(f[i], w[i], ix[i], f[l], w[l], ix[l], (i & k) == 0);
      }
    }
  }
}

template <typename T, bool BINW, int NV>
__global__ void __launch_bounds__(kT) k_pd_pass(PdArgs<T> a) {
  static_assert(NV > 0 && (NV & (NV - 1)) == 0, "NV: power of two");
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
    const unsigned abytes = BINW ? kTileLeaves * 4 : fbytes;
    mbar_expect_tx(&s_bar, fbytes + abytes);
    bulk_g2s(s_tile, a.F + tile * NV * kTileLeaves, fbytes, &s_bar);
    if (BINW)
      bulk_g2s(s_tile + NV * kTileLeaves, a.M + tile * kTileLeaves, abytes,
               &s_bar);
    else
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

  const T U0 = slot_ok ? a.u[s] : (T)0;
  const T B0 = slot_ok ? a.ub[s] : (T)0;
  const T P0 = slot_ok ? a.px[s] : (T)0;
  const T P1 = slot_ok ? a.py[s] : (T)0;
  const T P2 = slot_ok ? a.pz[s] : (T)0;
#define NB(ARR, V0, DX, DY, DZ, MASK, PRED)                                   \
  step_val<DX, DY, DZ>(__shfl_xor_sync(FULL, V0, MASK), c, cx, cy, cz,       \
                       active && (PRED), nb, ARR)
  // ubar at the 13-point stencil
  const T Bx = NB(a.ub, B0, 1, 0, 0, 4, xp);
  const T By = NB(a.ub, B0, 0, 1, 0, 2, yp);
  const T Bz = NB(a.ub, B0, 0, 0, 1, 1, zp);
  const T Bmx = NB(a.ub, B0, -1, 0, 0, 4, xm);
  const T Bmxy = NB(a.ub, B0, -1, 1, 0, 6, xm && yp);
  const T Bmxz = NB(a.ub, B0, -1, 0, 1, 5, xm && zp);
  const T Bmy = NB(a.ub, B0, 0, -1, 0, 2, ym);
  const T Bmyx = NB(a.ub, B0, 1, -1, 0, 6, ym && xp);
  const T Bmyz = NB(a.ub, B0, 0, -1, 1, 3, ym && zp);
  const T Bmz = NB(a.ub, B0, 0, 0, -1, 1, zm);
  const T Bmzx = NB(a.ub, B0, 1, 0, -1, 5, zm && xp);
  const T Bmzy = NB(a.ub, B0, 0, 1, -1, 3, zm && yp);
  // p at the three backward neighbours (all components, for the norms)
  const T Qx0 = NB(a.px, P0, -1, 0, 0, 4, xm), Qx1 = NB(a.py, P1, -1, 0, 0, 4, xm),
          Qx2 = NB(a.pz, P2, -1, 0, 0, 4, xm);
  const T Qy0 = NB(a.px, P0, 0, -1, 0, 2, ym), Qy1 = NB(a.py, P1, 0, -1, 0, 2, ym),
          Qy2 = NB(a.pz, P2, 0, -1, 0, 2, ym);
  const T Qz0 = NB(a.px, P0, 0, 0, -1, 1, zm), Qz1 = NB(a.py, P1, 0, 0, -1, 1, zm),
          Qz2 = NB(a.pz, P2, 0, 0, -1, 1, zm);
  // u at the forward neighbours (energy of the incoming state)
  const T Ux = NB(a.u, U0, 1, 0, 0, 4, xp);
  const T Uy = NB(a.u, U0, 0, 1, 0, 2, yp);
  const T Uz = NB(a.u, U0, 0, 0, 1, 1, zp);
#undef NB

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
  float w[NV];  // (unused with binary weights: the sort carries f only)
  int ix[NV];
  const uint32_t mk =
      BINW ? reinterpret_cast<const uint32_t*>(s_tile + NV * kTileLeaves)[t] : 0u;
  // data: weight sum and energy numerator in view order
  T W = 0, num = 0;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    f[v] = s_tile[v * kTileLeaves + t];
    const float wv = BINW ? ((mk >> v) & 1u ? 1.f : 0.f)
                          : s_tile[(NV + v) * kTileLeaves + t];
    const bool on = v < a.nv && wv != 0.f;
    if (on) {
      W += (T)wv;
      num += (T)wv * fabs(U0 - (T)f[v]);
    }
    if (!on) f[v] = __int_as_float(0x7f800000);  // absent: sorts last
    if (!BINW) {
      w[v] = on ? wv : 0.f;
      ix[v] = v;
    }
  }
  const T den = W + a.gamma;
  bitonic<NV, !BINW>(f, w, ix);
  // generalised weighted median (oracle/pd_oracle.c wmedian_prox); with
  // unit weights the running weight after k sorted samples is simply k
  const T cc = a.tau / den;
  T S = 0, res = v0;
  bool done = false;
#pragma unroll
  for (int k = 0; k <= NV; ++k) {
    const T cand = v0 - cc * ((T)2 * S - W);
    if (!done && k > 0 && cand < (T)f[k - 1]) {
      res = (T)f[k - 1];
      done = true;
    }
    if (!done && (k == NV || cand <= (T)f[k])) {
      res = cand;
      done = true;
    }
    if (k < NV) S += BINW ? (f[k] != __int_as_float(0x7f800000) ? (T)1 : (T)0)
                          : (T)w[k];
  }
  if (a.clamp) res = clamp1(res);
  double eterm = 0.0;
  if (active) {
    a.u_o[s] = res;
    a.ub_o[s] = (T)2 * res - U0;
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
  typedef cub::BlockReduce<double, kT> BR;
  __shared__ typename BR::TempStorage tmp;
  const double tot = BR(tmp).Sum(eterm);
  if (threadIdx.x == 0) a.epart[blockIdx.x] = tot;
}
