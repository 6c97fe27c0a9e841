// The restructuring descent pass, propagate and energy on device.
//
// Included once per precision: solver_f64.cu (T = double, -fmad=false, the
// bit-exact parity mode) and solver_f32.cu (T = float, throughput mode).
// Everything lives in an anonymous namespace so the two instantiations never
// meet at link time.
//
// Semantics follow the reference's recursive visit (_kernels.pyx:256-381),
// restated data-parallel:
//  1. every pre-pass leaf is updated from the immutable snapshot S
//     (k_leaf_pass: 13-point stencil through the block neighbour tables,
//     view samples from the gathered store);
//  2. leaves with |dn| < tau_s split; the cascade below them is evaluated
//     level by level on virtual children that carry the parent's snapshot,
//     which is exactly what the reference's lookups see (a new child's
//     snapshot equals the leaf that contained it), then blocks are
//     allocated in the reference's depth-first order (free list first);
//  3. joins are tested bottom-up level by level on post-update child values;
//  4. joined subtrees are freed in the reference's post-order, which fixes
//     the free-list order; then propagate and energy.
// The pool (value/snap/child/joined/state) therefore ends every pass
// identical to the reference's on live nodes.
#pragma once
#include <chrono>
#include <cooperative_groups.h>
#include <map>
#include <mutex>
#include <set>
#include <cub/cub.cuh>

#include "octf_arith.cuh"
#include "octf_ctx.h"

namespace octf {
namespace {

constexpr int kT = 256;

inline unsigned blocks_for(int64_t n) {
  int64_t g = (n + kT - 1) / kT;
  return (unsigned)(g < 1 ? 1 : g);
}

template <typename T>
struct LeafParams {
  int d_max;
  T lam, eps2, gamma, xi;
  double tau_s, tau_j;
  int clamp;
};

template <typename T>
LeafParams<T> leaf_params(const PassParams& p) {
  LeafParams<T> q;
  q.d_max = p.d_max;
  q.lam = (T)p.lam;
  q.eps2 = (T)p.eps2;
  q.gamma = (T)p.gamma;
  q.xi = (T)p.xi;
  q.tau_s = p.tau_s;
  q.tau_j = p.tau_j;
  q.clamp = p.clamp;
  return q;
}

// exact powers of two built from the exponent field
template <typename T>
__device__ __forceinline__ T pow2(int e);
template <>
__device__ __forceinline__ float pow2<float>(int e) {
  return __int_as_float((e + 127) << 23);
}
template <>
__device__ __forceinline__ double pow2<double>(int e) {
  return __longlong_as_double((long long)(e + 1023) << 52);
}
// 1/h = 2^-(d_max - L) (h = finest-cell units, reference fusion.py:14-15)
template <typename T>
__device__ __forceinline__ T inv_spacing(int d_max, int L) {
  return pow2<T>(L - d_max);
}

template <typename T>
__device__ __forceinline__ T clamp1(T v) {
  return v > (T)1 ? (T)1 : (v < (T)-1 ? (T)-1 : v);
}

// ---------------------------------------------------------------------------
// 1. fast leaf update over leaf blocks (leaf_kernel.cuh)
#include "leaf_kernel.cuh"
#include "pd_kernel.cuh"

// ---------------------------------------------------------------------------
// generic update of one cell at level L from the snapshot by root descents:
// the reference's delta_u (_kernels.pyx:223-253) verbatim in structure.
// Used for split cascades (virtual children) and join candidates.
// dn of one node by root descents (_kernels.pyx:205-253, lookups :193-202),
// by one warp: lane k < 13 resolves stencil point k, lanes cover the views
// (v = lane, lane + 32, ...); every lane then combines the shuffled values
// in the reference's order (flux3 / delta_u, bit for bit), so the dependent
// root-descent chain of one thread is ~1/30 as long.
template <typename T>
__device__ T warp_slow_dn(const int32_t* child, const T* snap, ViewSet vs,
                          const LeafParams<T>& p, int L, int x, int y, int z,
                          T S0, int lane) {
  using A = Arith<T>;
  const unsigned FULL = 0xffffffffu;
  const int m = 1 << L;
  // stencil points: 0 c, 1 +x, 2 +y, 3 +z, 4 -x, 5 -x+y, 6 -x+z, 7 -y,
  // 8 +x-y, 9 -y+z, 10 -z, 11 +x-z, 12 +y-z
  // offsets + 1 packed two bits per point (no local-memory tables)
  constexpr unsigned KX = 0x1u | 2u << 2 | 1u << 4 | 1u << 6 | 0u << 8 |
                          0u << 10 | 0u << 12 | 1u << 14 | 2u << 16 |
                          1u << 18 | 1u << 20 | 2u << 22 | 1u << 24;
  constexpr unsigned KY = 0x1u | 1u << 2 | 2u << 4 | 1u << 6 | 1u << 8 |
                          2u << 10 | 1u << 12 | 0u << 14 | 0u << 16 |
                          0u << 18 | 1u << 20 | 1u << 22 | 2u << 24;
  constexpr unsigned KZ = 0x1u | 1u << 2 | 1u << 4 | 2u << 6 | 1u << 8 |
                          1u << 10 | 2u << 12 | 1u << 14 | 1u << 16 |
                          2u << 18 | 0u << 20 | 0u << 22 | 0u << 24;
  T mine = 0;
  if (lane < 13) {
    const int sh = 2 * lane;
    const int qx = x + (int)((KX >> sh) & 3u) - 1;
    const int qy = y + (int)((KY >> sh) & 3u) - 1;
    const int qz = z + (int)((KZ >> sh) & 3u) - 1;
    if (qx >= 0 && qy >= 0 && qz >= 0 && qx < m && qy < m && qz < m)
      mine = snap[descend(child, L, qx, qy, qz)];
  }
  T P[13];
#pragma unroll
  for (int k = 0; k < 13; ++k) P[k] = __shfl_sync(FULL, mine, k);
  const T ih = inv_spacing<T>(p.d_max, L);
  T q[3], r[3];
  T bx = 0, by = 0, bz = 0;
  {  // flux_at(x, y, z)
    T gx = 0, gy = 0, gz = 0;
    if (x + 1 < m) gx = (P[1] - P[0]) * ih;
    if (y + 1 < m) gy = (P[2] - P[0]) * ih;
    if (z + 1 < m) gz = (P[3] - P[0]) * ih;
    A::flux(gx, gy, gz, p.eps2, q[0], q[1], q[2]);
  }
  if (x > 0) {  // flux_at(x-1, y, z): c = P4, +x = P0, +y = P5, +z = P6
    T gx = (P[0] - P[4]) * ih, gy = 0, gz = 0;
    if (y + 1 < m) gy = (P[5] - P[4]) * ih;
    if (z + 1 < m) gz = (P[6] - P[4]) * ih;
    A::flux(gx, gy, gz, p.eps2, r[0], r[1], r[2]);
    bx = r[0];
  }
  if (y > 0) {  // flux_at(x, y-1, z): c = P7, +x = P8, +y = P0, +z = P9
    T gx = 0, gy = (P[0] - P[7]) * ih, gz = 0;
    if (x + 1 < m) gx = (P[8] - P[7]) * ih;
    if (z + 1 < m) gz = (P[9] - P[7]) * ih;
    A::flux(gx, gy, gz, p.eps2, r[0], r[1], r[2]);
    by = r[1];
  }
  if (z > 0) {  // flux_at(x, y, z-1): c = P10, +x = P11, +y = P12, +z = P0
    T gx = 0, gy = 0, gz = (P[0] - P[10]) * ih;
    if (x + 1 < m) gx = (P[11] - P[10]) * ih;
    if (y + 1 < m) gy = (P[12] - P[10]) * ih;
    A::flux(gx, gy, gz, p.eps2, r[0], r[1], r[2]);
    bz = r[2];
  }
  const T div = ((q[0] - bx) + (q[1] - by) + (q[2] - bz)) * ih;
  T num = 0, den = p.gamma;
  // the first kViewChunks*32 views' nodes by lock-step descents
  constexpr int kViewChunks = 10;
  int32_t nd[kViewChunks];
  descend_views<kViewChunks>(vs.child, vs.n, L, x, y, z, lane, nd);
  // every chunk's (w, f) loaded before the ordered combine (independent
  // loads in flight together: the warp's latency chain is the critical
  // path of a join level)
  float wq[kViewChunks], fq[kViewChunks];
#pragma unroll
  for (int q = 0; q < kViewChunks; ++q) {
    wq[q] = 0.f;
    fq[q] = 0.f;
    if (nd[q] >= 0) {
      const int v = q * 32 + lane;
      wq[q] = vs.w[v][nd[q]];
      fq[q] = vs.val[v][nd[q]];
    }
  }
  for (int v0 = 0; v0 < vs.n; v0 += 32) {
    const int v = v0 + lane;
    float w = 0.f, f = 0.f;
    T g = 0;
    if (v < vs.n) {
      bool got = false;
#pragma unroll
      for (int q = 0; q < kViewChunks; ++q)
        if (v0 == q * 32) {
          w = wq[q];
          f = fq[q];
          got = true;
        }
      if (!got) {
        const int32_t n = descend(vs.child[v], L, x, y, z);
        w = vs.w[v][n];
        f = vs.val[v][n];
      }
      if (w != 0.f) g = A::data_grad((T)w, S0 - (T)f, p.eps2);
    }
    const int nk = vs.n - v0 < 32 ? vs.n - v0 : 32;
    for (int k = 0; k < nk; ++k) {  // view order, as slow_dn
      const float wk = __shfl_sync(FULL, w, k);
      const T gk = __shfl_sync(FULL, g, k);
      if (wk != 0.f) {
        num += gk;
        den += (T)wk;
      }
    }
  }
  const T du = p.lam * div - A::div(num, den);
  return S0 + p.xi * du;
}

// ---------------------------------------------------------------------------
// 2. split cascade on events.  Event = one split, i.e. one block of eight
// children to allocate.  Root events are pre-pass leaves; child events are
// virtual children that split again.
template <typename T>
struct Events {
  int32_t* slot;     // root events: the pre-pass leaf slot; else -1
  int32_t* parent;   // parent event or -1
  int8_t* pc;        // child position inside the parent event's block
  uint64_t* cell;    // packed (level, x, y, z) of the splitting node
  T* S;              // snapshot value every node of this cascade carries
  T* cval;           // [8] final values of non-splitting children
  int32_t* cmask;    // bit c: child c splits further
  uint64_t* key;     // depth-first pre-order key
  int32_t* idx;      // 0..E-1 (sorted alongside key)
  int32_t* rank;     // event -> allocation rank
  int32_t* blk;      // event -> allocated block base
};

__device__ __forceinline__ void slot_cell_of(int32_t s, const int8_t* blevel,
                                             const uint64_t* bcoord, int& L,
                                             int& x, int& y, int& z) {
  if (s == 0) {
    L = x = y = z = 0;
    return;
  }
  const int32_t b = ((s - 1) & ~7) + 1;
  const int c = (s - 1) & 7;
  const int k = block_id(b);
  int pl, px, py, pz;
  unpack_cell(bcoord[k], pl, px, py, pz);
  L = blevel[k];
  x = 2 * px + ((c >> 2) & 1);
  y = 2 * py + ((c >> 1) & 1);
  z = 2 * pz + (c & 1);
}

template <typename T>
__global__ void k_events_init(const int32_t* split_list, int64_t n,
                              const int8_t* blevel, const uint64_t* bcoord,
                              const T* snap, Events<T> ev) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int32_t s = split_list[e];
  int L, x, y, z;
  slot_cell_of(s, blevel, bcoord, L, x, y, z);
  ev.slot[e] = s;
  ev.parent[e] = -1;
  ev.pc[e] = 0;
  ev.cell[e] = pack_cell(L, x, y, z);
  ev.S[e] = snap[s];
  ev.cmask[e] = 0;
}

template <typename T>
__global__ void k_cascade(int64_t e0, int64_t e1, Events<T> ev,
                          const int32_t* __restrict__ child,
                          const T* __restrict__ snap, ViewSet vs,
                          LeafParams<T> p, int32_t* counters, int64_t ev_cap,
                          int64_t buf_cap) {
  // one warp per virtual child (the root descents of its 13 stencil points
  // and of its views spread over the lanes, warp_slow_dn); lane 0 records
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t e = e0 + (gw >> 3);
  const int c = (int)(gw & 7);
  if (e >= e1) return;  // warp-uniform
  int L, x, y, z;
  unpack_cell(ev.cell[e], L, x, y, z);
  const int L1 = L + 1;
  const int x1 = 2 * x + ((c >> 2) & 1), y1 = 2 * y + ((c >> 1) & 1),
            z1 = 2 * z + (c & 1);
  const T S0 = ev.S[e];
  T dn = warp_slow_dn<T>(child, snap, vs, p, L1, x1, y1, z1, S0, lane);
  if (lane != 0) return;
  if (L1 < p.d_max && fabs((double)dn) < p.tau_s) {
    atomicOr(ev.cmask + e, 1 << c);
    const int32_t ne = atomicAdd(counters + 2, 1);
    if (ne >= ev_cap) {  // more blocks than the pool holds
      atomicExch(counters + 3, 1);
      return;
    }
    if (ne >= buf_cap) {  // event buffers too small: the host retries
      atomicExch(counters + 5, 1);
      return;
    }
    ev.slot[ne] = -1;
    ev.parent[ne] = (int32_t)e;
    ev.pc[ne] = (int8_t)c;
    ev.cell[ne] = pack_cell(L1, x1, y1, z1);
    ev.S[ne] = S0;
    ev.cmask[ne] = 0;
  } else {
    if (p.clamp) dn = clamp1(dn);
    ev.cval[e * 8 + c] = dn;
  }
}

template <typename T>
__global__ void k_event_keys(Events<T> ev, int64_t n, int d_max, int reverse) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  int L, x, y, z;
  unpack_cell(ev.cell[e], L, x, y, z);
  ev.key[e] = preorder_key(L, x, y, z, d_max, reverse != 0);
  ev.idx[e] = (int32_t)e;
}

// rank -> block: free-list entries from the head down, then the bump pointer
template <typename T>
__global__ void k_event_alloc(Events<T> ev, int64_t n,
                              const int32_t* free_stack, int64_t nfree,
                              int64_t used) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t e = ev.idx[r];
  ev.rank[e] = (int32_t)r;
  ev.blk[e] = r < nfree ? free_stack[nfree - 1 - r]
                        : (int32_t)(used + 8 * (r - nfree));
}

template <typename T>
__global__ void k_event_materialize(Events<T> ev, int64_t n, int32_t* child,
                                    T* usnap, T* uval, uint8_t* joined) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t e = gid >> 3;
  const int c = (int)(gid & 7);
  if (e >= n) return;
  const int32_t be = ev.blk[e];
  const T S0 = ev.S[e];
  const bool splits = (ev.cmask[e] >> c) & 1;
  const int32_t s = be + c;
  usnap[s] = S0;
  uval[s] = splits ? S0 : ev.cval[e * 8 + c];
  joined[s] = 0;
  if (!splits) child[s] = -1;
  if (c == 0) {
    const int32_t par = ev.parent[e];
    const int32_t ps = par < 0 ? ev.slot[e] : ev.blk[par] + ev.pc[e];
    child[ps] = be;
    if (par < 0) uval[ps] = S0;
  }
}

// ---------------------------------------------------------------------------
// 3. joins, one level at a time from d_max-1 up to the root
template <typename T>
struct JoinRecs {
  int32_t* slot;
  int32_t* blk;
  uint64_t* cell;
  double* vals;   // [8] children's post-update values (log row)
  uint64_t* key;
  int32_t* idx;
};

// candidates of one level: an inner node none of whose children is a live
// inner node (leaf or joined this pass), all with |u| > tau_j and one sign
// (_kernels.pyx:321-354, cheap tests first); its |dn| test follows in
// k_join_dn, one warp per candidate
template <typename T>
__global__ void k_join_cand(const int32_t* __restrict__ blocks, int64_t nblk,
                            const int32_t* child, const uint8_t* joined,
                            const uint8_t* smark, const T* uval,
                            LeafParams<T> p, int32_t* cand, double* cacc,
                            int32_t* ccount) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  if (i >= nblk) return;
  const int32_t b = blocks[i];
  if (b == 0 && c != 0) return;
  const int32_t s = b + c;
  const int32_t cb = child[s];
  if (cb < 0 || smark[s]) return;  // leaf, or a leaf that split this pass
  bool pos = false, neg = false;
  double acc = 0.0;
  for (int q = 0; q < 8; ++q) {
    const int32_t cs = cb + q;
    if (child[cs] >= 0 && !joined[cs]) return;
    const double v = (double)uval[cs];
    if (!(v > p.tau_j || v < -p.tau_j)) return;
    if (v > 0.0)
      pos = true;
    else
      neg = true;
    acc += v;
  }
  if (pos && neg) return;
  const int32_t r = atomicAdd(ccount, 1);
  cand[r] = s;
  cacc[r] = acc;
}

template <typename T>
__global__ void __launch_bounds__(256)
    k_join_dn(const int32_t* __restrict__ cand, const double* __restrict__ cacc,
              const int32_t* __restrict__ ccount, const int8_t* blevel,
              const uint64_t* bcoord, const int32_t* child, uint8_t* joined,
              const T* snap, T* uval, ViewSet vs, LeafParams<T> p,
              JoinRecs<T> rec, int32_t* counters) {
  const int lane = threadIdx.x & 31;
  const int nwarps = (int)(gridDim.x * (blockDim.x >> 5));
  const int n = *ccount;
  for (int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
       w < n; w += nwarps) {
    const int32_t s = cand[w];
    int L, x, y, z;
    slot_cell_of(s, blevel, bcoord, L, x, y, z);
    const T dn = warp_slow_dn<T>(child, snap, vs, p, L, x, y, z, snap[s], lane);
    if (lane == 0 && fabs((double)dn) > p.tau_j) {
      const int32_t cb = child[s];
      joined[s] = 1;
      uval[s] = (T)(cacc[w] / 8.0);
      const int32_t r = atomicAdd(counters + 4, 1);
      rec.slot[r] = s;
      rec.blk[r] = cb;
      rec.cell[r] = pack_cell(L, x, y, z);
      for (int q = 0; q < 8; ++q) rec.vals[r * 8 + q] = (double)uval[cb + q];
    }
  }
}

// All join levels in one cooperative launch (bottom-up, grid barriers
// between the phases), from worklists instead of scans of every level:
// candidates at level L are the parents of the leaf kernel's bottom blocks
// (eight unsplit leaves past tau_j with one sign) that sit at level L, and
// the parents of the nodes joined at level L+1 (proposed once, by the
// highest-index joined sibling).  Every other inner node has a live inner
// child and cannot join (k_join_cand's test), so the candidate sets equal
// the per-level scans'; the test and the update (warp_slow_dn) are the
// same, and the join records are sorted afterwards, so the result does not
// depend on the order candidates are found in.
template <typename T>
struct JoinCoopArgs {
  const int32_t* bot;     // parent slots of the bottom candidate blocks
  int64_t nbot;
  const int8_t* blevel;
  const uint64_t* bcoord;
  const int32_t* bparent;
  const int32_t* child;
  uint8_t* joined;
  const uint8_t* smark;
  const T* snap;
  T* uval;
  ViewSet vs;
  LeafParams<T> p;
  JoinRecs<T> rec;
  int32_t* counters;      // [4]: join records
  int32_t* cand;
  double* cacc;
  int32_t* ccount;        // candidates per round, zeroed
  int d_max;
};

template <typename T>
__device__ __forceinline__ bool join_test(const JoinCoopArgs<T>& a, int32_t s,
                                          double& acc) {
  const int32_t cb = a.child[s];
  if (cb < 0 || a.smark[s]) return false;
  // all loads first (independent), then the reference's test in order
  int32_t ch[8];
  uint8_t jn[8];
  T u[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    ch[q] = a.child[cb + q];
    jn[q] = a.joined[cb + q];
    u[q] = a.uval[cb + q];
  }
  bool pos = false, neg = false;
  acc = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (ch[q] >= 0 && !jn[q]) return false;
    const double v = (double)u[q];
    if (!(v > a.p.tau_j || v < -a.p.tau_j)) return false;
    if (v > 0.0)
      pos = true;
    else
      neg = true;
    acc += v;
  }
  return !(pos && neg);
}

template <typename T>
__global__ void __launch_bounds__(256) k_joins_coop(JoinCoopArgs<T> a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t wid = tid >> 5, nw = nthr >> 5;
  // Rounds instead of levels: round 0 tests every bottom candidate (all
  // levels at once -- their children are leaves, nothing below them can
  // change), round r the parents of the nodes joined in round r-1.  A
  // parent whose inner children join in different rounds is proposed after
  // each of them and passes once the last has joined; `joined` holds the
  // round stamp (round + 1) until the sweep clears it, so "proposed once
  // per round, by the highest-index sibling joined in that round" can be
  // told from siblings joined earlier.  The join set is the same fixpoint
  // as the level order's and a joined node's value depends only on its
  // children's final values, so the pools are identical; the number of
  // barrier pairs drops from the levels holding candidates to the longest
  // join chain.
  int rec_lo = 0;
  for (int round = 0; round < a.d_max; ++round) {
    const int rec_hi = *(volatile int32_t*)(a.counters + 4);
    const int64_t n_in = round == 0 ? a.nbot : rec_hi - rec_lo;
    if (n_in == 0) break;  // the same decision in every thread
    for (int64_t i = tid; i < n_in; i += nthr) {
      int32_t s;
      if (round == 0) {
        s = a.bot[i];
      } else {
        const int32_t j = a.rec.slot[rec_lo + i];
        const int32_t jb = ((j - 1) & ~7) + 1;
        bool later = false;  // a higher sibling joined this round: it proposes
        for (int q = j - jb + 1; q < 8; ++q) later |= a.joined[jb + q] == round;
        if (later) continue;
        s = a.bparent[block_id(jb)];
        if (a.joined[s]) continue;
      }
      double acc;
      if (!join_test(a, s, acc)) continue;
      const int32_t r = atomicAdd(a.ccount + round, 1);
      a.cand[r] = s;
      a.cacc[r] = acc;
    }
    grid.sync();
    const int n = *(volatile int32_t*)(a.ccount + round);
    for (int64_t w = wid; w < n; w += nw) {
      const int32_t s = a.cand[w];
      int Ls, x, y, z;
      slot_cell_of(s, a.blevel, a.bcoord, Ls, x, y, z);
      const T dn = warp_slow_dn<T>(a.child, a.snap, a.vs, a.p, Ls, x, y, z,
                                   a.snap[s], lane);
      if (lane == 0 && fabs((double)dn) > a.p.tau_j) {
        const int32_t cb = a.child[s];
        a.joined[s] = (uint8_t)(round + 1);
        a.uval[s] = (T)(a.cacc[w] / 8.0);
        const int32_t r = atomicAdd(a.counters + 4, 1);
        a.rec.slot[r] = s;
        a.rec.blk[r] = cb;
        a.rec.cell[r] = pack_cell(Ls, x, y, z);
        for (int q = 0; q < 8; ++q)
          a.rec.vals[r * 8 + q] = (double)a.uval[cb + q];
      }
    }
    grid.sync();
    rec_lo = round == 0 ? 0 : rec_hi;
  }
}

template <typename T>
__global__ void k_join_keys(JoinRecs<T> rec, int64_t n, int d_max,
                            int reverse) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int L, x, y, z;
  unpack_cell(rec.cell[r], L, x, y, z);
  rec.key[r] = postorder_key(L, x, y, z, d_max, reverse != 0);
  rec.idx[r] = (int32_t)r;
}

// 4. sweep (_kernels.pyx:357-381): every joined node's child block is freed
// (all inner nodes under a topmost joined node are joined themselves)
// With alternating value buffers (octf_fuse_pass) `mirror` is the other
// buffer: a freed block keeps its last values in the reference's single
// array, so they are copied to the buffer the next pass writes, which never
// touches dead slots again.
template <typename T>
__global__ void k_sweep_clear(JoinRecs<T> rec, int64_t n, int32_t* child,
                              uint8_t* joined, const T* uval, T* mirror) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t s = rec.slot[r], b = rec.blk[r];
  child[s] = -1;
  joined[s] = 0;
  for (int q = 0; q < 8; ++q) {
    joined[b + q] = 0;
    if (q) child[b + q] = -1;
    if (mirror) mirror[b + q] = uval[b + q];
  }
}

// push in post-order: child[b_i] links to the previous head
template <typename T>
__global__ void k_sweep_link(JoinRecs<T> rec, int64_t n, int64_t old_head,
                             int32_t* child, int32_t* free_stack,
                             int64_t nfree) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t b = rec.blk[rec.idx[r]];
  const int32_t prev = r == 0 ? (int32_t)old_head : rec.blk[rec.idx[r - 1]];
  child[b] = prev;
  free_stack[nfree + r] = b;
}

template <typename T>
__global__ void k_join_log(JoinRecs<T> rec, int64_t n, double* jlog) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t j = rec.idx[r];
  int L, x, y, z;
  unpack_cell(rec.cell[j], L, x, y, z);
  double* row = jlog + r * 12;
  row[0] = L;
  row[1] = x;
  row[2] = y;
  row[3] = z;
  for (int q = 0; q < 8; ++q) row[4 + q] = rec.vals[j * 8 + q];
}

__global__ void k_unmark(const int32_t* list, int64_t n, uint8_t* smark) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) smark[list[i]] = 0;
}

// ---------------------------------------------------------------------------
// propagate (_kernels.pyx:80-113): inner = sequential f64 sum of children / 8

// up to five fields at once, one thread per child block: the block's parent
// slot comes from the context's bparent table, and with sector-aligned pools
// (slot 1 on a 32 B / 64 B boundary, _device.py POOL_PAD) the eight children
// are read with 16-byte vector loads.  Same sequential double sum as
// the reference's propagate (_kernels.pyx:80-113, oracle propagate).
template <typename T>
struct FieldSet {
  T* v[5];
};

template <typename T, int NA, bool VEC>
__device__ __forceinline__ void propagate_block(int32_t b, int32_t par,
                                                const FieldSet<T>& f) {
#pragma unroll
  for (int q = 0; q < NA; ++q) {
    T x[8];
    if (VEC) {
      if (sizeof(T) == 4) {
        const float4* p = reinterpret_cast<const float4*>(f.v[q] + b);
        const float4 lo = __ldcs(p), hi = __ldcs(p + 1);
        x[0] = lo.x; x[1] = lo.y; x[2] = lo.z; x[3] = lo.w;
        x[4] = hi.x; x[5] = hi.y; x[6] = hi.z; x[7] = hi.w;
      } else {
        const double2* p = reinterpret_cast<const double2*>(f.v[q] + b);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 d = __ldcs(p + k);
          x[2 * k] = (T)d.x;
          x[2 * k + 1] = (T)d.y;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = f.v[q][b + k];
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += (double)x[k];
    f.v[q][par] = (T)(acc / 8.0);
  }
}

template <typename T, int NA, bool VEC>
__global__ void __launch_bounds__(kT)
    k_propagate_blocks(const int32_t* __restrict__ blocks, int64_t nblk,
                       const int32_t* __restrict__ bparent, FieldSet<T> f) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nblk) return;
  const int32_t b = __ldg(blocks + i);
  propagate_block<T, NA, VEC>(b, __ldg(bparent + ((b + 7) >> 3)), f);
}

// the small levels near the root (each at most one CTA of blocks) in one
// launch: one CTA walks them bottom-up with a barrier in between -- a
// launch per level costs more than its work there
struct TopLevels {
  int n;                      // levels, deepest first
  int32_t off[kMaxDepth + 1];  // start of the level's child-block list
  int32_t cnt[kMaxDepth + 1];
};

template <typename T, int NA, bool VEC>
__global__ void __launch_bounds__(kT)
    k_propagate_top(const int32_t* __restrict__ lvl_blocks, TopLevels tl,
                    const int32_t* __restrict__ bparent, FieldSet<T> f) {
  for (int q = 0; q < tl.n; ++q) {
    if ((int)threadIdx.x < tl.cnt[q]) {
      const int32_t b = __ldg(lvl_blocks + tl.off[q] + threadIdx.x);
      propagate_block<T, NA, VEC>(b, __ldg(bparent + ((b + 7) >> 3)), f);
    }
    __threadfence_block();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// energy (_kernels.pyx:494-533) per leaf, deterministic block sums
template <typename T, bool BINW>
__global__ void __launch_bounds__(kT)
    k_energy(const int32_t* __restrict__ lblocks, int64_t nlb,
             const uint64_t* __restrict__ lkey, const int32_t* __restrict__ nbr,
             const int4* __restrict__ lmeta, const T* __restrict__ u,
             const float* __restrict__ F, const float* __restrict__ W,
             const uint32_t* __restrict__ M, int64_t stride, int nv,
             LeafParams<T> p, double* partials, double* terms,
             const int32_t* __restrict__ tileK,
             const int64_t* __restrict__ tileOff, SDesc sd) {
  using A = Arith<T>;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  bool active = i < nlb;
  const int32_t b = active ? lblocks[i] : 0;
  const int32_t s = b + c;
  if (active && b == 0 && c != 0) active = false;
  // leaf mask of the (possibly rank-restricted) leaf-block list
  if (active && !(((unsigned)lmeta[i].w >> (19 + c)) & 1u)) active = false;
  double term = 0.0;
  if (active) {
    int L, px, py, pz;
    unpack_cell(lkey[i], L, px, py, pz);
    const int cx = (c >> 2) & 1, cy = (c >> 1) & 1, cz = c & 1;
    const int x = 2 * px + cx, y = 2 * py + cy, z = 2 * pz + cz;
    const int m = 1 << L;
    const T ih = inv_spacing<T>(p.d_max, L);
    const T h = pow2<T>(p.d_max - L);
    const int32_t* nb = nbr + i * 12;
    auto U = [&](int dx, int dy, int dz) -> T {
      const int tx = cx + dx, ty = cy + dy, tz = cz + dz;
      const int ox = tx >> 1, oy = ty >> 1, oz = tz >> 1;
      const int cc = ((tx & 1) << 2) | ((ty & 1) << 1) | (tz & 1);
      if ((ox | oy | oz) == 0) return u[b + cc];
      const int32_t r = nb[nbr_dir(ox, oy, oz)];
      return r >= 0 ? u[r + cc] : u[-r - 2];
    };
    const T u0 = u[s];
    const T gx = x + 1 < m ? (U(1, 0, 0) - u0) * ih : (T)0;
    const T gy = y + 1 < m ? (U(0, 1, 0) - u0) * ih : (T)0;
    const T gz = z + 1 < m ? (U(0, 0, 1) - u0) * ih : (T)0;
    const T smooth = p.lam * A::smooth_val(gx, gy, gz, p.eps2);
    T num = 0, den = p.gamma;
    const int64_t slot = i * 8 + c;
    const int4 mt = lmeta[i];
    const SIdx si = sidx(sd, i, c, mt.y, ((unsigned)mt.w >> 19) & 0xffu);
    const uint32_t mk = BINW ? M[si.m] : 0u;
    const int nrow = tileK ? tileK[slot >> 8] : nv;
    for (int v = 0; v < nrow; ++v) {
      const int64_t q = tileK ? ell_idx(tileOff, slot, v) : si.f + (int64_t)v * si.pitch;
      const float w = BINW ? (float)((mk >> v) & 1u) : W[q];
      if (w != 0.f) {
        const T d = u0 - (T)F[q];
        num += A::data_val((T)w, d, p.eps2);
        den += (T)w;
      }
    }
    const T t = (A::div(num, den) + smooth) * (h * h * h);
    term = (double)t;
    if (terms) terms[s] = term;
  }
  typedef cub::BlockReduce<double, kT> BR;
  __shared__ typename BR::TempStorage tmp;
  const double tot = BR(tmp).Sum(term);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// Deterministic two-stage sum of per-CTA energy partials, for several
// passes at once (pass p owns partials[p*n, (p+1)*n)): stage 1 reduces
// kStripes fixed contiguous stripes per pass, stage 2 the stripes.  The
// order depends only on n, so energies are bit-reproducible.
constexpr int kStripes = 128;

__global__ void k_sum_stage1(const double* __restrict__ partials, int64_t n,
                             double* mid) {
  const int64_t len = (n + kStripes - 1) / kStripes;
  const double* p = partials + (int64_t)blockIdx.y * n;
  const int64_t lo = blockIdx.x * len;
  const int64_t hi = lo + len < n ? lo + len : n;
  double acc = 0.0;
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) acc += p[j];
  typedef cub::BlockReduce<double, kT> BR;
  __shared__ typename BR::TempStorage tmp;
  const double tot = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) mid[(int64_t)blockIdx.y * kStripes + blockIdx.x] = tot;
}

__global__ void k_sum_stage2(const double* __restrict__ mid, double* out) {
  const double v = threadIdx.x < kStripes
                       ? mid[(int64_t)blockIdx.x * kStripes + threadIdx.x]
                       : 0.0;
  typedef cub::BlockReduce<double, kT> BR;
  __shared__ typename BR::TempStorage tmp;
  const double tot = BR(tmp).Sum(v);
  if (threadIdx.x == 0) out[blockIdx.x] = tot;
}

// out[p] = sum of partials of pass p, p < npasses (device pointers)
void sum_partials(Ctx& c, const double* partials, int64_t n, int npasses,
                  double* out, cudaStream_t st) {
  c.mid.ensure((size_t)kStripes * (npasses > 32 ? npasses : 32));
  k_sum_stage1<<<dim3(kStripes, npasses), kT, 0, st>>>(partials, n, c.mid.p);
  OCTF_CUDA(cudaGetLastError());
  k_sum_stage2<<<npasses, kT, 0, st>>>(c.mid.p, out);
  OCTF_CUDA(cudaGetLastError());
  c.launches += 2;
}

// ---------------------------------------------------------------------------
// host orchestration
template <typename T>
void ensure_prepared(Ctx& c, const int32_t* child, int64_t cap, int d_max,
                     const int64_t* state, cudaStream_t st) {
  if (!c.valid || c.child_key != child || c.cap != cap || c.d_max != d_max)
    ctx_prepare(c, child, cap, state, d_max, st);
}

// grid of the leaf kernel (also the number of energy partials per pass)
inline unsigned leaf_grid(const Ctx& c) { return blocks_for(c.nlb * 8); }
// energy partials the leaf kernel writes per pass (kLeafParts per CTA)
inline int64_t leaf_parts(const Ctx& c) {
  return (int64_t)leaf_grid(c) * kLeafParts;
}

// resident CTAs of a kernel on the whole GPU (occupancy x SMs), cached
// per kernel and device
inline int resident_ctas(const void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev = 0;
  OCTF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(fn, dev);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0, sms = 0;
  OCTF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads,
                                                          smem));
  OCTF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int n = (per_sm < 1 ? 1 : per_sm) * sms;
  cache[key] = n;
  return n;
}

// opt a kernel in to > 48 KiB of dynamic shared memory, once per device
inline void smem_opt_in(const void* fn, size_t smem) {
  if (smem <= 48 * 1024) return;
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  OCTF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert(std::make_pair(fn, dev)).second)
    OCTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
}

// g = tiles of this launch; staged kernels run persistent (at most the
// resident CTAs, each walking tiles with a grid stride)
template <typename T, bool FZ, int BW, bool EN, int N>
void launch_leaf(unsigned g, cudaStream_t st, LeafArgs<T> a) {
  if constexpr (FZ && N > 0) {  // the packed store: its own instantiation
    if (a.sd.packed) {
      constexpr size_t smem = leaf_smem_bytes(N, BW);
      const void* fn = (const void*)k_leaf_pass<T, FZ, BW, EN, N, true>;
      smem_opt_in(fn, smem);
      a.ntiles = (int)g;
      k_leaf_pass<T, FZ, BW, EN, N, true><<<g, kT, smem, st>>>(a);
      return;
    }
  }
  if constexpr (N == 0) {  // the per-tile ELL store: its own instantiation
    if (a.tileK) {
      a.ntiles = (int)g;
      k_leaf_pass<T, FZ, BW, EN, 0, true><<<g, kT, 0, st>>>(a);
      return;
    }
  }
  constexpr size_t smem = leaf_smem_bytes(N, BW);
  const void* fn = (const void*)k_leaf_pass<T, FZ, BW, EN, N>;
  smem_opt_in(fn, smem);
  a.ntiles = (int)g;
  unsigned grid = g;
  if (OCTF_PERSIST && N > 0) {
    const unsigned res = (unsigned)resident_ctas(fn, kT, smem);
    grid = g < res ? g : res;
  }
  k_leaf_pass<T, FZ, BW, EN, N><<<grid, kT, smem, st>>>(a);
}

template <typename T>
void launch_leaf_pass(Ctx& c, const T* snap, T* uval, const int32_t* child,
                      const LeafParams<T>& lp, bool frozen, double* epart,
                      cudaStream_t st, bool timed = true,
                      int tile0 = 0,
                      int ntiles = -1) {
  const unsigned g = ntiles < 0 ? leaf_grid(c) : (unsigned)ntiles;
  if (g == 0) return;
  LeafArgs<T> a;
  a.tile0 = tile0;
  a.lpar = c.lpar.p;
  a.join_bot = c.join_bot.p;
  a.lblocks = c.lblocks.p;
  a.nlb = c.nlb;
  a.lkey = c.lkey.p;
  a.lmeta = c.lmeta.p;
  a.nbr = c.nbr.p;
  a.child = child;
  a.snap = snap;
  a.uval = uval;
  a.F = c.F.p;
  a.W = c.W.p;
  a.M = c.M.p;
  a.stride = c.sstride;
  a.nv = c.nviews;
  a.p = lp;
  a.smark = c.smark.p;
  a.split_list = c.split_list.p;
  a.counters = c.counters.p;
  a.epart = epart;
  a.tileK = c.ell ? c.tileK.p : nullptr;
  a.tileOff = c.ell ? c.tileOff.p : nullptr;
  a.sd = c.sd;
  const bool en = epart != nullptr;
  if (timed && c.timing) OCTF_CUDA(cudaEventRecord(c.tev[0], st));
#define OCTF_LEAF(FZ, BW, EN)                                         \
  do {                                                                \
    if (c.ell)                                                        \
      launch_leaf<T, FZ, BW, EN, 0>(g, st, a);                        \
    else if (c.nviews == 16)                                          \
      launch_leaf<T, FZ, BW, EN, 16>(g, st, a);                       \
    else if (c.nviews == 32)                                          \
      launch_leaf<T, FZ, BW, EN, 32>(g, st, a);                       \
    else if (c.nviews == 8)                                           \
      launch_leaf<T, FZ, BW, EN, 8>(g, st, a);                        \
    else                                                              \
      launch_leaf<T, FZ, BW, EN, 0>(g, st, a);                        \
  } while (0)
#define OCTF_LEAF_AV(FZ, EN)                                          \
  do {                                                                \
    if (c.nviews == 16)                                               \
      launch_leaf<T, FZ, kAllValid, EN, 16>(g, st, a);                \
    else if (c.nviews == 32)                                          \
      launch_leaf<T, FZ, kAllValid, EN, 32>(g, st, a);                \
    else                                                              \
      launch_leaf<T, FZ, kAllValid, EN, 8>(g, st, a);                 \
  } while (0)
  const bool av = c.allv && !c.ell &&
                  (c.nviews == 8 || c.nviews == 16 || c.nviews == 32);
  if (frozen) {
    if (av) {
      if (en) OCTF_LEAF_AV(true, true); else OCTF_LEAF_AV(true, false);
    } else if (c.binw) {
      if (en) OCTF_LEAF(true, kMask, true); else OCTF_LEAF(true, kMask, false);
    } else {
      if (en) OCTF_LEAF(true, kWeights, true); else OCTF_LEAF(true, kWeights, false);
    }
  } else {
    if (av) {
      if (en) OCTF_LEAF_AV(false, true); else OCTF_LEAF_AV(false, false);
    } else if (c.binw) {
      if (en) OCTF_LEAF(false, kMask, true); else OCTF_LEAF(false, kMask, false);
    } else {
      if (en) OCTF_LEAF(false, kWeights, true); else OCTF_LEAF(false, kWeights, false);
    }
  }
#undef OCTF_LEAF_AV
#undef OCTF_LEAF
  OCTF_CUDA(cudaGetLastError());
  ++c.launches;
  if (timed && c.timing) OCTF_CUDA(cudaEventRecord(c.tev[1], st));
}

// typed scratch kept in a context slot (Ctx::rs_ev / rs_join)
template <typename B>
B& ctx_bufs(std::shared_ptr<void>& slot) {
  if (!slot)
    slot = std::shared_ptr<void>(new B(), [](void* q) { delete (B*)q; });
  return *static_cast<B*>(slot.get());
}

template <typename T>
struct EventBufs {
  DevBuf<int32_t> slot, parent, cmask, idx, rank, blk;
  DevBuf<int8_t> pc;
  DevBuf<uint64_t> cell, key;
  DevBuf<T> S, cval;
  Events<T> view(int64_t cap) {
    Events<T> e;
    e.slot = slot.ensure(cap);
    e.parent = parent.ensure(cap);
    e.pc = pc.ensure(cap);
    e.cell = cell.ensure(cap);
    e.S = S.ensure(cap);
    e.cval = cval.ensure(cap * 8);
    e.cmask = cmask.ensure(cap);
    e.key = key.ensure(cap);
    e.idx = idx.ensure(cap);
    e.rank = rank.ensure(cap);
    e.blk = blk.ensure(cap);
    return e;
  }
};

template <typename T>
struct JoinBufs {
  DevBuf<int32_t> slot, blk, idx, cand, ccount;
  DevBuf<uint64_t> cell, key;
  DevBuf<double> vals, cacc;
  JoinRecs<T> view(int64_t cap) {
    JoinRecs<T> r;
    r.slot = slot.ensure(cap);
    r.blk = blk.ensure(cap);
    r.cell = cell.ensure(cap);
    r.vals = vals.ensure(cap * 8);
    r.key = key.ensure(cap);
    r.idx = idx.ensure(cap);
    return r;
  }
};

template <typename T>
void read_counters(Ctx& c, int n, cudaStream_t st) {
  OCTF_CUDA(cudaMemcpyAsync(c.h_counters, c.counters.p, n * sizeof(int32_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void iterate_pass_impl(Ctx& c, IterArgs& a, cudaStream_t st) {
  const PassParams& prm = a.prm;
  if (prm.d_max < 0 || prm.d_max > kMaxDepth)
    throw Error(kEDepth, "tree depth out of range");
  ensure_prepared<T>(c, a.child, a.cap, prm.d_max, a.state, st);
  if (c.nviews <= 0) throw Error(kEArg, "at least one view is required");
  const int64_t used = a.state[0];
  if (a.snapshot)
    OCTF_CUDA(cudaMemcpyAsync((void*)a.usnap, a.uval, used * sizeof(T),
                              cudaMemcpyDeviceToDevice, st));
  const LeafParams<T> lp = leaf_params<T>(prm);
  const bool frozen = prm.tau_s <= 0.0 && prm.clamp && prm.tau_j >= 1.0;
  if (!frozen && c.ext_F)
    throw Error(kEArg, "per-slot samples need a frozen structure "
                       "(tau_split <= 0, tau_join >= 1, clamp)");
  c.counters.ensure(64);
  c.split_list.ensure(c.nlb * 8 + 1);
  c.join_bot.ensure(c.nlb + 1);
  OCTF_CUDA(cudaMemsetAsync(c.counters.p, 0, 8 * sizeof(int32_t), st));
  double* epart = nullptr;
  if (a.want_energy) {
    c.partials.ensure(leaf_parts(c));
    c.dscalar.ensure(1);
    epart = c.partials.p;
  }
  launch_leaf_pass<T>(c, (const T*)a.usnap, (T*)a.uval, a.child, lp, frozen,
                      epart, st);
  if (epart) {
    sum_partials(c, epart, leaf_parts(c), 1, c.dscalar.p, st);
    OCTF_CUDA(cudaMemcpyAsync(c.h_scalar, c.dscalar.p, sizeof(double),
                              cudaMemcpyDeviceToHost, st));
  }
  read_counters<T>(c, 2, st);
  a.energy_pre = epart ? c.h_scalar[0] : 0.0;
  if (c.timing) {
    float ms = 0.f;
    OCTF_CUDA(cudaEventElapsedTime(&ms, c.tev[0], c.tev[1]));
    c.t_leaf_ms += ms;
    ++c.n_leaf;
  }
  const auto t_restr = std::chrono::steady_clock::now();
  ph_start(c, st);
  const int64_t nsplit = c.h_counters[0];
  const int64_t ncand = c.h_counters[1];
  const T* snap = (const T*)a.usnap;
  T* usnap = (T*)a.usnap;
  T* uval = (T*)a.uval;
  const ViewSet vs = ctx_views(c);
  int64_t splits = 0, joins = 0, jrows = 0;
  bool changed = false;

  // ---- split cascade + allocation in depth-first order
  if (nsplit > 0) {
    EventBufs<T>& eb = ctx_bufs<EventBufs<T>>(c.rs_ev[sizeof(T) == 8]);
    // the pool bound on events (blocks the pool can still hand out) sizes
    // the exhaustion test; the buffers start at a small multiple of the
    // split count and are sized to the bound only when a cascade outgrows
    // them (sizing them to the bound every pass reallocated eleven buffers
    // whenever the free list grew: 0.5 ms for a one-split pass at cfg4)
    const int64_t ev_cap = nsplit + (a.cap - used) / 8 + c.nfree + 8;
    int64_t buf_cap = std::min<int64_t>(ev_cap, 64 * nsplit + 4096);
    Events<T> ev;
    int64_t e1 = nsplit;
    for (;;) {
      ev = eb.view(buf_cap);
      k_events_init<T><<<blocks_for(nsplit), kT, 0, st>>>(
          c.split_list.p, nsplit, c.blevel.p, c.bcoord.p, snap, ev);
      OCTF_CUDA(cudaGetLastError());
      ++c.launches;
      int64_t e0 = 0;
      e1 = nsplit;
      const int32_t init[4] = {(int32_t)nsplit, 0, 0, 0};  // counters 2..5
      OCTF_CUDA(cudaMemcpyAsync(c.counters.p + 2, init, sizeof(init),
                                cudaMemcpyHostToDevice, st));
      bool grow = false;
      while (e1 > e0) {
        k_cascade<T><<<blocks_for((e1 - e0) * 8 * 32), kT, 0, st>>>(
            e0, e1, ev, a.child, snap, vs, lp, c.counters.p, ev_cap, buf_cap);
        OCTF_CUDA(cudaGetLastError());
        ++c.launches;
        read_counters<T>(c, 6, st);
        if (c.h_counters[3])
          throw Error(kEPool, "node pool capacity exhausted");
        if (c.h_counters[5]) {
          grow = true;
          break;
        }
        e0 = e1;
        e1 = c.h_counters[2];
      }
      if (!grow) break;
      buf_cap = ev_cap;  // rerun the cascade with buffers at the bound
    }
    const int64_t E = e1;
    ph_mark(c, kPhSplitCascade, st);
    const int64_t fresh = E > c.nfree ? E - c.nfree : 0;
    if (used + 8 * fresh > a.cap)
      throw Error(kEPool, "node pool capacity exhausted");
    k_event_keys<T><<<blocks_for(E), kT, 0, st>>>(ev, E, prm.d_max,
                                                   prm.reverse);
    OCTF_CUDA(cudaGetLastError());
  ++c.launches;
    sort_u64_i32(c, ev.key, ev.idx, E, st);
    k_event_alloc<T><<<blocks_for(E), kT, 0, st>>>(ev, E, c.free_stack.p,
                                                    c.nfree, used);
    OCTF_CUDA(cudaGetLastError());
  ++c.launches;
    k_event_materialize<T><<<blocks_for(E * 8), kT, 0, st>>>(
        ev, E, a.child, usnap, uval, a.joined);
    OCTF_CUDA(cudaGetLastError());
  ++c.launches;
    // new free-list head
    int64_t head = -1;
    if (E < c.nfree) {
      int32_t h;
      OCTF_CUDA(cudaMemcpyAsync(&h, c.free_stack.p + (c.nfree - 1 - E),
                                sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      OCTF_CUDA(cudaStreamSynchronize(st));
      head = h;
      c.nfree -= E;
    } else {
      c.nfree = 0;
    }
    a.state[0] = used + 8 * fresh;
    a.state[1] = head;
    a.state[2] += 8 * E;
    splits = E;
    changed = true;
    ph_mark(c, kPhSplitAlloc, st);
  }

  // ---- join cascade, bottom-up
  if (ncand > 0) {
    JoinBufs<T>& jb = ctx_bufs<JoinBufs<T>>(c.rs_join[sizeof(T) == 8]);
    const int64_t jcap_rec = c.nblocks * 8 + 8;
    JoinRecs<T> rec = jb.view(jcap_rec);
    // per level (bottom-up): cheap candidate tests over the level's slots,
    // then one warp per candidate for the root-descent update (no host
    // round trip: the dn kernel strides over the device-side count)
    int32_t* cand = jb.cand.ensure(c.nblocks * 8 + 8);
    double* cacc = jb.cacc.ensure(c.nblocks * 8 + 8);
    if (!c.coop_off) {
      // every level in one cooperative launch from the worklists
      int32_t* ccount = jb.ccount.ensure(kMaxDepth + 2);
      OCTF_CUDA(cudaMemsetAsync(ccount, 0, (kMaxDepth + 2) * sizeof(int32_t),
                                st));
      JoinCoopArgs<T> ja;
      ja.bot = c.join_bot.p;
      ja.nbot = ncand;
      ja.blevel = c.blevel.p;
      ja.bcoord = c.bcoord.p;
      ja.bparent = c.bparent.p;
      ja.child = a.child;
      ja.joined = a.joined;
      ja.smark = c.smark.p;
      ja.snap = snap;
      ja.uval = uval;
      ja.vs = vs;
      ja.p = lp;
      ja.rec = rec;
      ja.counters = c.counters.p;
      ja.cand = cand;
      ja.cacc = cacc;
      ja.ccount = ccount;
      ja.d_max = prm.d_max;
      // resident CTAs of the cooperative launch, per device
      static int coop_per_dev[64] = {};
      int dev = 0;
      OCTF_CUDA(cudaGetDevice(&dev));
      int& coop_blocks = coop_per_dev[dev & 63];
      if (!coop_blocks) {
        int per_sm = 0, nsm = 0;
        OCTF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_joins_coop<T>, 256, 0));
        OCTF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount,
                                         dev));
        if (per_sm * nsm < 1) throw Error(kECuda, "joins: no resident CTA");
        coop_blocks = per_sm * nsm;
      }
      void* kargs[] = {&ja};
      OCTF_CUDA(cudaLaunchCooperativeKernel((const void*)k_joins_coop<T>,
                                            coop_blocks, 256, kargs, 0, st));
      ++c.launches;
    }
    for (int L = prm.d_max - 1; L >= 0 && c.coop_off; --L) {
      const int64_t n = c.lvl_cnt[L];
      if (n == 0) continue;
      OCTF_CUDA(cudaMemsetAsync(c.counters.p + 8, 0, sizeof(int32_t), st));
      k_join_cand<T><<<blocks_for(n * 8), kT, 0, st>>>(
          c.lvl_blocks.p + c.lvl_off[L], n, a.child, a.joined, c.smark.p,
          uval, lp, cand, cacc, c.counters.p + 8);
      OCTF_CUDA(cudaGetLastError());
      const int64_t cmax = n * 8;
      const unsigned gw = (unsigned)((cmax + 7) / 8 < 148 * 16 ? (cmax + 7) / 8
                                                                : 148 * 16);
      k_join_dn<T><<<gw, 256, 0, st>>>(cand, cacc, c.counters.p + 8,
                                         c.blevel.p, c.bcoord.p, a.child,
                                         a.joined, snap, uval, vs, lp, rec,
                                         c.counters.p);
      OCTF_CUDA(cudaGetLastError());
      c.launches += 2;
    }
    read_counters<T>(c, 5, st);
    ph_mark(c, kPhJoins, st);
    const int64_t J = c.h_counters[4];
    if (J > 0) {
      // sweep order: forward post-order (sweep ignores `reverse`)
      k_join_keys<T><<<blocks_for(J), kT, 0, st>>>(rec, J, prm.d_max, 0);
      OCTF_CUDA(cudaGetLastError());
  ++c.launches;
      sort_u64_i32(c, rec.key, rec.idx, J, st);
      k_sweep_clear<T><<<blocks_for(J), kT, 0, st>>>(
          rec, J, a.child, a.joined, uval,
          a.snapshot ? (T*)nullptr : (T*)const_cast<void*>(a.usnap));
      OCTF_CUDA(cudaGetLastError());
  ++c.launches;
      c.free_stack.grow_keep(c.nfree + J + 1, c.nfree, st);
      k_sweep_link<T><<<blocks_for(J), kT, 0, st>>>(
          rec, J, a.state[1], a.child, c.free_stack.p, c.nfree);
      OCTF_CUDA(cudaGetLastError());
  ++c.launches;
      int32_t last;
      OCTF_CUDA(cudaMemcpyAsync(&last, c.free_stack.p + c.nfree + J - 1,
                                sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      if (a.jlog && a.jcap > 0) {
        if (prm.reverse) {
          k_join_keys<T><<<blocks_for(J), kT, 0, st>>>(rec, J, prm.d_max, 1);
          OCTF_CUDA(cudaGetLastError());
  ++c.launches;
          sort_u64_i32(c, rec.key, rec.idx, J, st);
        }
        jrows = J < a.jcap ? J : a.jcap;
        k_join_log<T><<<blocks_for(jrows), kT, 0, st>>>(rec, jrows, a.jlog);
        OCTF_CUDA(cudaGetLastError());
  ++c.launches;
      }
      OCTF_CUDA(cudaStreamSynchronize(st));
      c.nfree += J;
      a.state[1] = last;
      a.state[2] -= 8 * J;
      joins = J;
      changed = true;
      ph_mark(c, kPhSweep, st);
    }
  }
  if (nsplit > 0) {
    k_unmark<<<blocks_for(nsplit), kT, 0, st>>>(c.split_list.p, nsplit,
                                                c.smark.p);
    OCTF_CUDA(cudaGetLastError());
  ++c.launches;
  }
  c.hstate[0] = a.state[0];
  c.hstate[1] = a.state[1];
  c.hstate[2] = a.state[2];
  c.nfree_head = a.state[1];  // the free-list mirror was kept in step
  if (changed) {
    c.valid = false;
    c.own_change = true;  // the next rebuild may keep unchanged samples
  }
  a.out3[0] = splits;
  a.out3[1] = joins;
  a.out3[2] = jrows;
  if (c.timing) {
    OCTF_CUDA(cudaStreamSynchronize(st));  // only for the timer
    c.t_restr_ms += std::chrono::duration<double, std::milli>(
                        std::chrono::steady_clock::now() - t_restr).count();
  }
}

// parent levels top .. 0 (default: every level above the finest) of `na`
// fields; level L is filled from the child blocks listed at level L+1
template <typename T>
void launch_propagate_multi(Ctx& c, T* const* vals, int na, cudaStream_t st,
                            int top = -1, int lo = 0) {
  if (na < 1 || na > 5) throw Error(kEArg, "propagate: 1..5 fields");
  FieldSet<T> fs{};
  bool vec = true;
  for (int q = 0; q < na; ++q) {
    fs.v[q] = vals[q];
    vec = vec && ((uintptr_t)(vals[q] + 1) % (8 * sizeof(T)) == 0);
  }
  auto launch = [&](auto kern_top, const int32_t* blk, int64_t n,
                    const TopLevels* tl) {
    (void)kern_top;
    const unsigned g = tl ? 1u : blocks_for(n);
    auto go = [&](auto na_c, auto vec_c, const FieldSet<T>& fset) {
      constexpr int NA = decltype(na_c)::value;
      constexpr bool VEC = decltype(vec_c)::value;
      if (tl)
        k_propagate_top<T, NA, VEC><<<1, kT, 0, st>>>(c.lvl_blocks.p, *tl,
                                                      c.bparent.p, fset);
      else
        k_propagate_blocks<T, NA, VEC><<<g, kT, 0, st>>>(blk, n, c.bparent.p,
                                                         fset);
    };
    using I1 = std::integral_constant<int, 1>;
    using I5 = std::integral_constant<int, 5>;
    if (na == 1) {
      if (vec) go(I1{}, std::true_type{}, fs);
      else go(I1{}, std::false_type{}, fs);
    } else if (na == 5) {
      if (vec) go(I5{}, std::true_type{}, fs);
      else go(I5{}, std::false_type{}, fs);
    } else {
      for (int q = 0; q < na; ++q) {
        FieldSet<T> one{};
        one.v[0] = vals[q];
        go(I1{}, std::false_type{}, one);
      }
    }
    OCTF_CUDA(cudaGetLastError());
    ++c.launches;
  };
  const int L0 = top < 0 ? c.d_max - 1 : top;
  // the levels from `fuse_from` down to `lo` each fit one CTA: one launch
  int fuse_from = lo - 1;
  for (int L = lo; L <= L0; ++L) {
    if (L + 1 >= (int)c.lvl_cnt.size() || c.lvl_cnt[L + 1] > kT) break;
    fuse_from = L;
  }
  for (int L = L0; L > fuse_from; --L) {
    if (L + 1 >= (int)c.lvl_cnt.size()) continue;
    const int64_t n = c.lvl_cnt[L + 1];
    if (n == 0) continue;
    launch(0, c.lvl_blocks.p + c.lvl_off[L + 1], n, nullptr);
  }
  TopLevels tl{};
  for (int L = std::min(fuse_from, L0); L >= lo; --L) {
    if (c.lvl_cnt[L + 1] == 0) continue;
    tl.off[tl.n] = (int32_t)c.lvl_off[L + 1];
    tl.cnt[tl.n] = (int32_t)c.lvl_cnt[L + 1];
    ++tl.n;
  }
  if (tl.n == 1)
    launch(0, c.lvl_blocks.p + tl.off[0], tl.cnt[0], nullptr);
  else if (tl.n > 1)
    launch(0, nullptr, 0, &tl);
}

template <typename T>
void launch_propagate(Ctx& c, T* value, const int32_t* child,
                      cudaStream_t st, int top = -1) {
  (void)child;  // the context's block lists carry the structure
  launch_propagate_multi<T>(c, &value, 1, st, top);
}

template <typename T>
void propagate_impl(Ctx& c, T* value, const int32_t* child, cudaStream_t st) {
  ensure_prepared<T>(c, child, c.cap, c.d_max, c.hstate, st);
  launch_propagate<T>(c, value, child, st);
}

template <typename T>
double energy_impl(Ctx& c, const T* u, const int32_t* child,
                   const PassParams& prm, double* terms, cudaStream_t st) {
  ensure_prepared<T>(c, child, c.cap, prm.d_max, c.hstate, st);
  const LeafParams<T> lp = leaf_params<T>(prm);
  const int64_t n = c.nlb * 8;
  const unsigned g = blocks_for(n);
  c.partials.ensure(g);
  c.dscalar.ensure(1);
  if (c.timing) OCTF_CUDA(cudaEventRecord(c.tev[2], st));
  if (c.binw)
    k_energy<T, true><<<g, kT, 0, st>>>(c.lblocks.p, c.nlb, c.lkey.p, c.nbr.p,
                                        c.lmeta.p, u, c.F.p, c.W.p, c.M.p,
                                        c.sstride, c.nviews, lp, c.partials.p,
                                        terms, c.ell ? c.tileK.p : nullptr,
                                        c.ell ? c.tileOff.p : nullptr,
                                        c.sd);
  else
    k_energy<T, false><<<g, kT, 0, st>>>(c.lblocks.p, c.nlb, c.lkey.p,
                                         c.nbr.p, c.lmeta.p, u, c.F.p, c.W.p,
                                         c.M.p, c.sstride, c.nviews, lp,
                                         c.partials.p, terms,
                                         c.ell ? c.tileK.p : nullptr,
                                         c.ell ? c.tileOff.p : nullptr,
                                         c.sd);
  OCTF_CUDA(cudaGetLastError());
  ++c.launches;
  if (c.timing) OCTF_CUDA(cudaEventRecord(c.tev[3], st));
  sum_partials(c, c.partials.p, g, 1, c.dscalar.p, st);
  OCTF_CUDA(cudaMemcpyAsync(c.h_scalar, c.dscalar.p, sizeof(double),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  if (c.timing) {
    float ms = 0.f;
    OCTF_CUDA(cudaEventElapsedTime(&ms, c.tev[2], c.tev[3]));
    c.t_energy_ms += ms;
    ++c.n_energy;
  }
  return c.h_scalar[0];
}

// K passes of a frozen structure back to back: per pass one leaf kernel
// (update + energy of the incoming state) and the propagate levels; the
// host only waits once, for the K energies.
template <typename T>
void frozen_passes_impl(Ctx& c, FrozenArgs& a, cudaStream_t st) {
  const PassParams& prm = a.prm;
  if (prm.d_max < 0 || prm.d_max > kMaxDepth)
    throw Error(kEDepth, "tree depth out of range");
  if (!(prm.tau_s <= 0.0 && prm.clamp && prm.tau_j >= 1.0))
    throw Error(kEArg, "batched passes need a frozen structure "
                       "(tau_split <= 0, tau_join >= 1, clamp)");
  if (a.npasses < 1) return;
  ensure_prepared<T>(c, a.child, a.cap, prm.d_max, a.state, st);
  if (c.nviews <= 0) throw Error(kEArg, "at least one view is required");
  // fixed-size scratch (no allocation inside a timed loop): energy
  // partials for kChunk passes, one energy slot per pass
  constexpr int kChunk = 32;
  const int64_t g = leaf_parts(c);
  c.partials.ensure((size_t)g * kChunk);
  c.dscalar.ensure(a.npasses > 1024 ? a.npasses : 1024);
  c.counters.ensure(64);
  c.split_list.ensure(c.nlb * 8 + 1);
  if (c.timing && (int)c.pev.size() < 2 * kChunk) {
    for (int k = (int)c.pev.size(); k < 2 * kChunk; ++k) {
      cudaEvent_t e;
      OCTF_CUDA(cudaEventCreate(&e));
      c.pev.push_back(e);
    }
  }
  for (int k0 = 0; k0 < a.npasses; k0 += kChunk) {
    const int nk = a.npasses - k0 < kChunk ? a.npasses - k0 : kChunk;
    for (int j = 0; j < nk; ++j) {
      const int k = k0 + j;
      PassParams pk = prm;
      pk.xi = a.xis[k];
      const LeafParams<T> lp = leaf_params<T>(pk);
      const T* snap = (const T*)a.ubuf[k & 1];
      T* uval = (T*)a.ubuf[(k + 1) & 1];
      if (c.timing) OCTF_CUDA(cudaEventRecord(c.pev[2 * j], st));
      // (the bottom propagate level fused into this kernel, as the
      // primal-dual kernel does for its five fields, was measured slower
      // here: leaf kernel 0.306 -> 0.332 ms on cfg2 for a 17 us launch)
      launch_leaf_pass<T>(c, snap, uval, a.child, lp, true,
                          c.partials.p + (size_t)j * g, st, false);
      if (c.timing) OCTF_CUDA(cudaEventRecord(c.pev[2 * j + 1], st));
      launch_propagate<T>(c, uval, a.child, st);
    }
    // stream order keeps the next chunk from overwriting unsummed partials
    double* eout = a.dev_energies ? a.energies_pre : c.dscalar.p;
    sum_partials(c, c.partials.p, g, nk, eout + k0, st);
    if (c.timing) {  // profiling only: read this chunk's kernel events
      OCTF_CUDA(cudaStreamSynchronize(st));
      for (int j = 0; j < nk; ++j) {
        float ms = 0.f;
        OCTF_CUDA(cudaEventElapsedTime(&ms, c.pev[2 * j], c.pev[2 * j + 1]));
        c.t_leaf_ms += ms;
        ++c.n_leaf;
      }
    }
  }
  if (a.dev_energies) return;  // stays asynchronous
  OCTF_CUDA(cudaMemcpyAsync(a.energies_pre, c.dscalar.p,
                            a.npasses * sizeof(double), cudaMemcpyDeviceToHost,
                            st));
  OCTF_CUDA(cudaStreamSynchronize(st));
}

// npasses of the TV-L1 primal-dual scheme on a frozen tree; set A = a.in,
// set B = a.out; pass k reads the set k%2 and writes the other
template <typename T>
void pd_passes_impl(Ctx& c, PdHostArgs& a, cudaStream_t st);

template <typename T, int BW, int N, bool WP>
void launch_pd_wp(unsigned g, cudaStream_t st, const PdArgs<T>& p) {
  constexpr size_t smem = pd_smem_bytes(N, BW != kWeights) * kStages;
  if (p.sd.packed) {  // the packed store: its own instantiation
    const void* fp = (const void*)k_pd_pass<T, BW, N, WP, true>;
    smem_opt_in(fp, smem);
    k_pd_pass<T, BW, N, WP, true><<<g, kT, smem, st>>>(p);
    return;
  }
  const void* fn = (const void*)k_pd_pass<T, BW, N, WP>;
  smem_opt_in(fn, smem);
  const unsigned res =
      OCTF_PERSIST ? (unsigned)resident_ctas(fn, kT, smem) : g;
  k_pd_pass<T, BW, N, WP><<<g < res ? g : res, kT, smem, st>>>(p);
}
template <typename T, int BW, int N>
void launch_pd(unsigned g, cudaStream_t st, const PdArgs<T>& p, bool wp) {
  if (wp) launch_pd_wp<T, BW, N, true>(g, st, p);
  else launch_pd_wp<T, BW, N, false>(g, st, p);
}
template <typename T>
void pd_passes_impl(Ctx& c, PdHostArgs& a, cudaStream_t st) {
  if (a.d_max < 0 || a.d_max > kMaxDepth)
    throw Error(kEDepth, "tree depth out of range");
  if (a.npasses < 1) return;
  ensure_prepared<T>(c, a.child, a.cap, a.d_max, a.state, st);
  const int nv = c.nviews;
  if (!c.sorted)
    throw Error(kEArg, "solver='pd' needs the sorted sample layout "
                       "(octf_ctx_set_options(ctx, OCTF_CTX_SORTED))");
  // dense store: 4 .. 64 views; more views: the per-tile (ELL) store
  if (!c.ell && (!(nv == 4 || nv == 8 || nv == 16 || nv == 32 || nv == 64) ||
                 c.sstride != nv || (nv == 64 && c.binw)))
    throw Error(kEArg, "solver='pd' with the dense sample store supports 4, "
                       "8, 16, 32 or 64 views (more views: leave "
                       "OCTF_CTX_DENSE off for the per-tile store)");
  constexpr int kChunk = 32;
  const unsigned g = leaf_grid(c);
  // energy partials per pass: one per tile (the primal-dual kernel sums its
  // warps' partials after the barrier its fused parent level needs anyway;
  // per-warp partials without it measured slower, cfg5 3.31 -> 3.79 ms)
  const int64_t gp = g;
  c.partials.ensure((size_t)gp * kChunk);
  c.dscalar.ensure(a.npasses > 1024 ? a.npasses : 1024);
  const bool fused_bottom =
      c.list_full && !c.fuse_off && a.d_max >= 1 && !c.ell;
  for (int k0 = 0; k0 < a.npasses; k0 += kChunk) {
    const int nk = a.npasses - k0 < kChunk ? a.npasses - k0 : kChunk;
    for (int j = 0; j < nk; ++j) {
      const int k = k0 + j;
      void* const* in = (k & 1) ? a.out : a.in;
      void* const* out = (k & 1) ? a.in : a.out;
      PdArgs<T> p;
      p.lblocks = c.lblocks.p;
      p.nlb = c.nlb;
      p.lmeta = c.lmeta.p;
      p.nbr = c.nbr.p;
      p.u = (const T*)in[0];
      p.ub = (const T*)in[1];
      p.px = (const T*)in[2];
      p.py = (const T*)in[3];
      p.pz = (const T*)in[4];
      p.u_o = (T*)out[0];
      p.ub_o = (T*)out[1];
      p.px_o = (T*)out[2];
      p.py_o = (T*)out[3];
      p.pz_o = (T*)out[4];
      p.F = c.F.p;
      p.W = c.W.p;
      p.M = c.M.p;
      p.stride = c.sstride;
      p.nv = nv;
      p.d_max = a.d_max;
      p.lam = (T)a.lam;
      p.tl = (T)(a.tau * a.lam);
      p.sl = (T)(a.sigma * a.lam);
      p.tau = (T)a.tau;
      p.gamma = (T)a.gamma;
      p.clamp = a.clamp;
      p.epart = c.partials.p + (size_t)j * gp;
      p.lpar = c.lpar.p;
      p.sd = c.sd;
      if (c.ell) {
        p.tileK = c.tileK.p;
        p.tileOff = c.tileOff.p;
      }
      if (c.timing && (int)c.pev.size() >= 2 * kChunk)
        OCTF_CUDA(cudaEventRecord(c.pev[2 * j], st));
#define OCTF_PD(BW, N) launch_pd<T, BW, N>(g, st, p, fused_bottom)
      if (c.ell) {
        k_pd_pass<T, kWeights, 1, false, false, true>
            <<<g, kT, pd_smem_bytes(1, false) * kStages, st>>>(p);
      } else if (c.allv && (nv == 8 || nv == 16 || nv == 32)) {
        if (nv == 8) OCTF_PD(kAllValid, 8);
        else if (nv == 16) OCTF_PD(kAllValid, 16); else OCTF_PD(kAllValid, 32);
      } else if (c.binw) {
        if (nv == 4) OCTF_PD(kMask, 4); else if (nv == 8) OCTF_PD(kMask, 8);
        else if (nv == 16) OCTF_PD(kMask, 16); else OCTF_PD(kMask, 32);
      } else {
        if (nv == 4) OCTF_PD(kWeights, 4); else if (nv == 8) OCTF_PD(kWeights, 8);
        else if (nv == 16) OCTF_PD(kWeights, 16);
        else if (nv == 32) OCTF_PD(kWeights, 32); else OCTF_PD(kWeights, 64);
      }
#undef OCTF_PD
      OCTF_CUDA(cudaGetLastError());
      ++c.launches;
      if (c.timing && (int)c.pev.size() >= 2 * kChunk)
        OCTF_CUDA(cudaEventRecord(c.pev[2 * j + 1], st));
      if (!fused_bottom)
        launch_propagate_multi<T>(c, (T* const*)out, 5, st);
      else if (a.d_max >= 2)
        launch_propagate_multi<T>(c, (T* const*)out, 5, st, a.d_max - 2);
    }
    sum_partials(c, c.partials.p, gp, nk,
                 (a.dev_energies ? a.energies : c.dscalar.p) + k0, st);
    if (c.timing && (int)c.pev.size() >= 2 * kChunk) {
      OCTF_CUDA(cudaStreamSynchronize(st));
      for (int j = 0; j < nk; ++j) {
        float ms = 0.f;
        OCTF_CUDA(cudaEventElapsedTime(&ms, c.pev[2 * j], c.pev[2 * j + 1]));
        c.t_leaf_ms += ms;
        ++c.n_leaf;
      }
    }
  }
  if (a.dev_energies) return;  // stays asynchronous
  OCTF_CUDA(cudaMemcpyAsync(a.energies, c.dscalar.p, a.npasses * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------------------
// solver="pd" split/join after a pass (oracle/pd_oracle.c orc_pd_restructure:
// leaves with |u| < tau_s split, children carrying u, ubar, p; inner nodes
// with eight leaf children past tau_j of one sign join; one level per pass).
// Splits claim blocks in depth-first pre-order from the free-list mirror then
// the bump pointer, joins free in post-order -- the descent's allocation.
template <typename T>
__global__ void k_pd_split_flags(const int4* __restrict__ lmeta, int64_t nlb,
                                 const T* __restrict__ u, int d_max,
                                 double tau_s, int32_t* sslot, uint64_t* skey,
                                 int32_t* sidx, int32_t* cnt) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  if (i >= nlb) return;
  const int4 m = lmeta[i];
  int L, pz;
  unsigned mask;
  unpack_meta_w(m.w, pz, mask, L);
  if (!((mask >> c) & 1u) || (m.x == 0 && c != 0)) return;
  const int32_t s = m.x + c;
  if (L >= d_max || !(fabs((double)u[s]) < tau_s)) return;
  const int x = m.x == 0 ? 0 : 2 * meta_px(m.y) + ((c >> 2) & 1);
  const int y = m.x == 0 ? 0 : 2 * m.z + ((c >> 1) & 1);
  const int z = m.x == 0 ? 0 : 2 * pz + (c & 1);
  const int32_t r = atomicAdd(cnt, 1);
  sslot[r] = s;
  skey[r] = preorder_key(L, x, y, z, d_max, false);
  sidx[r] = r;
}

template <typename T>
__global__ void k_pd_join_cand(const int32_t* __restrict__ blocks, int64_t nblk,
                               const int8_t* blevel, const uint64_t* bcoord,
                               const int32_t* __restrict__ child,
                               const T* __restrict__ u, double tau_j,
                               JoinRecs<T> rec, int32_t* cnt) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = gid >> 3;
  const int c = (int)(gid & 7);
  if (i >= nblk) return;
  const int32_t b = blocks[i];
  if (b == 0 && c != 0) return;
  const int32_t s = b + c;
  const int32_t cb = child[s];
  if (cb < 0) return;
  bool pos = false, neg = false;
  for (int q = 0; q < 8; ++q) {
    if (child[cb + q] >= 0) return;
    const double v = (double)u[cb + q];
    if (!(v > tau_j || v < -tau_j)) return;
    if (v > 0.0)
      pos = true;
    else
      neg = true;
  }
  if (pos && neg) return;
  int L, x, y, z;
  slot_cell_of(s, blevel, bcoord, L, x, y, z);
  const int32_t r = atomicAdd(cnt, 1);
  rec.slot[r] = s;
  rec.blk[r] = cb;
  rec.cell[r] = pack_cell(L, x, y, z);
}

template <typename T>
__global__ void k_pd_split_apply(const int32_t* __restrict__ sslot,
                                 const int32_t* __restrict__ sidx, int64_t n,
                                 const int32_t* free_stack, int64_t nfree,
                                 int64_t used, int32_t* child, FieldSet<T> f) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = gid >> 3;
  const int q = (int)(gid & 7);
  if (r >= n) return;
  const int32_t s = sslot[sidx[r]];
  const int32_t nb = r < nfree ? free_stack[nfree - 1 - r]
                               : (int32_t)(used + 8 * (r - nfree));
  child[nb + q] = -1;
#pragma unroll
  for (int k = 0; k < 5; ++k) f.v[k][nb + q] = f.v[k][s];
  if (q == 0) child[s] = nb;
}

template <typename T>
__global__ void k_pd_unlink(JoinRecs<T> rec, int64_t n, int32_t* child) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) child[rec.slot[r]] = -1;
}

template <typename T>
void pd_restructure_impl(Ctx& c, PdRsArgs& a, cudaStream_t st) {
  if (a.d_max < 0 || a.d_max > kMaxDepth)
    throw Error(kEDepth, "tree depth out of range");
  ensure_prepared<T>(c, a.child, a.cap, a.d_max, a.state, st);
  FieldSet<T> fs{};
  for (int k = 0; k < 5; ++k) fs.v[k] = (T*)a.f[k];
  const int64_t used = a.state[0];
  JoinBufs<T>& jb = ctx_bufs<JoinBufs<T>>(c.rs_join[sizeof(T) == 8]);
  DevBuf<int32_t>& sslot = c.rs_slot;
  DevBuf<int32_t>& sidx = c.rs_idx;
  DevBuf<uint64_t>& skey = c.rs_key;
  const int64_t nl = c.nlb * 8 + 1;
  sslot.ensure(nl);
  sidx.ensure(nl);
  skey.ensure(nl);
  JoinRecs<T> rec = jb.view(c.nblocks * 8 + 8);
  c.counters.ensure(64);
  OCTF_CUDA(cudaMemsetAsync(c.counters.p, 0, 2 * sizeof(int32_t), st));
  // candidates on the pre-pass structure (with tau_s < tau_j no node both
  // splits and joins)
  if (c.nlb)
    k_pd_split_flags<T><<<blocks_for(c.nlb * 8), kT, 0, st>>>(
        c.lmeta.p, c.nlb, fs.v[0], a.d_max, a.tau_s, sslot.p, skey.p, sidx.p,
        c.counters.p);
  k_pd_join_cand<T><<<blocks_for(c.nblocks * 8), kT, 0, st>>>(
      c.lvl_blocks.p, c.nblocks, c.blevel.p, c.bcoord.p, a.child, fs.v[0],
      a.tau_j, rec, c.counters.p + 1);
  OCTF_CUDA(cudaGetLastError());
  c.launches += 2;
  read_counters<T>(c, 2, st);
  const int64_t E = c.h_counters[0], J = c.h_counters[1];
  a.out2[0] = E;
  a.out2[1] = J;
  if (E == 0 && J == 0) return;
  if (E > 0) {
    const int64_t fresh = E > c.nfree ? E - c.nfree : 0;
    if (used + 8 * fresh > a.cap)
      throw Error(kEPool, "node pool capacity exhausted");
    sort_u64_i32(c, skey.p, sidx.p, E, st);
    k_pd_split_apply<T><<<blocks_for(E * 8), kT, 0, st>>>(
        sslot.p, sidx.p, E, c.free_stack.p, c.nfree, used, a.child, fs);
    OCTF_CUDA(cudaGetLastError());
    ++c.launches;
    int64_t head = -1;
    if (E < c.nfree) {
      int32_t h;
      OCTF_CUDA(cudaMemcpyAsync(&h, c.free_stack.p + (c.nfree - 1 - E),
                                sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      OCTF_CUDA(cudaStreamSynchronize(st));
      head = h;
      c.nfree -= E;
    } else {
      c.nfree = 0;
    }
    a.state[0] = used + 8 * fresh;
    a.state[1] = head;
    a.state[2] += 8 * E;
  }
  if (J > 0) {
    // free the joined blocks in post-order (forward), as the descent sweep
    k_join_keys<T><<<blocks_for(J), kT, 0, st>>>(rec, J, a.d_max, 0);
    sort_u64_i32(c, rec.key, rec.idx, J, st);
    k_pd_unlink<T><<<blocks_for(J), kT, 0, st>>>(rec, J, a.child);
    c.free_stack.grow_keep(c.nfree + J + 1, c.nfree, st);
    k_sweep_link<T><<<blocks_for(J), kT, 0, st>>>(rec, J, a.state[1], a.child,
                                                   c.free_stack.p, c.nfree);
    OCTF_CUDA(cudaGetLastError());
    c.launches += 3;
    int32_t last;
    OCTF_CUDA(cudaMemcpyAsync(&last, c.free_stack.p + c.nfree + J - 1,
                              sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    OCTF_CUDA(cudaStreamSynchronize(st));
    c.nfree += J;
    a.state[1] = last;
    a.state[2] -= 8 * J;
  }
  c.hstate[0] = a.state[0];
  c.hstate[1] = a.state[1];
  c.hstate[2] = a.state[2];
  c.nfree_head = a.state[1];
  c.valid = false;
  c.own_change = true;
  OCTF_CUDA(cudaStreamSynchronize(st));
}

// leaf kernel of a frozen pass over tiles [tile0, tile0 + ntiles); the
// energy partials land at their tile index, summed by pass_finish_impl
template <typename T>
void pass_tiles_impl(Ctx& c, TileArgs& a, cudaStream_t st) {
  ensure_prepared<T>(c, a.child, a.cap, a.prm.d_max, a.state, st);
  if (c.nviews <= 0) throw Error(kEArg, "at least one view is required");
  const int g = (int)leaf_grid(c);
  if (a.tile0 < 0 || a.ntiles < 0 || a.tile0 + a.ntiles > g)
    throw Error(kEArg, "tile range outside the leaf-block list");
  c.partials.ensure(leaf_parts(c));
  const LeafParams<T> lp = leaf_params<T>(a.prm);
  if (c.timing) {  // an event pair per tile range, read by octf_ctx_profile
    while (c.tile_ev.size() < 2 * c.tile_ev_used + 2) {
      cudaEvent_t e;
      OCTF_CUDA(cudaEventCreate(&e));
      c.tile_ev.push_back(e);
    }
    OCTF_CUDA(cudaEventRecord(c.tile_ev[2 * c.tile_ev_used], st));
  }
  launch_leaf_pass<T>(c, (const T*)a.usnap, (T*)a.uval, a.child, lp, true,
                      c.partials.p, st, false, a.tile0, a.ntiles);
  if (c.timing) OCTF_CUDA(cudaEventRecord(c.tile_ev[2 * c.tile_ev_used++ + 1], st));
}

// propagate every level of the pass's output and sum the pass's energy
// partials (all tiles) into a device double
template <typename T>
void pass_finish_impl(Ctx& c, T* uval, const int32_t* child,
                      double* dev_energy, cudaStream_t st) {
  if (!c.valid) throw Error(kEArg, "context not prepared");
  launch_propagate<T>(c, uval, child, st);
  sum_partials(c, c.partials.p, leaf_parts(c), 1, dev_energy, st);
  if (c.timing) ++c.tile_passes;  // the tile ranges of one pass end here
}

// propagate levels hi-1 .. lo only (the replicated top of a sharded tree)
template <typename T>
void propagate_levels_impl(Ctx& c, T* value, const int32_t* child, int lo,
                           int hi, cudaStream_t st) {
  if (!c.valid) throw Error(kEArg, "context not prepared");
  (void)child;
  if (hi - 1 >= 0 && lo < hi)
    launch_propagate_multi<T>(c, &value, 1, st, hi - 1, lo < 0 ? 0 : lo);
}

}  // namespace
}  // namespace octf
