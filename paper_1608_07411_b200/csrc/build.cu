// Octree construction from depth maps on device: per-view projective TSDF,
// 2x2x2 min/max/mean pyramids, the spread-rule build and readout.
//
// Compiled with -fmad=false: every double expression keeps numpy's operand
// order so the results are bit-identical to the reference's numpy code:
//   TSDF       reference tsdf.py:87-120 (+ volume.py:63-65, 120-128)
//   pyramids   reference octree.py:193-225 (numpy mean of a 2x2x2 block sums
//              ((((b0+b1)+(b2+b3))+(b4+b5))+(b6+b7)), c = x<<2|y<<1|z,
//              pinned by tests/test_oracle_golden.py)
//   build      reference octree.py:243-306 + _kernels.pyx:21-77.  The
//              reference grows the tree depth-first with a LIFO (child 7 is
//              expanded first), so the block of the r-th splitting node in
//              that order lands at slot 1 + 8r.  Here r is computed in
//              parallel: subtree split counts bottom-up, then
//              rank(child c) = rank(parent) + 1 + sum_{c' > c} count(c').
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "octf_build.h"
#include "octf_ctx.h"

namespace octf {
namespace {

constexpr int kB = 256;
inline unsigned nblk(int64_t n) {
  int64_t g = (n + kB - 1) / kB;
  return (unsigned)(g < 1 ? 1 : g);
}

// ------------------------------------------------------------------ TSDF --
struct Cam {
  double fx, fy, cx, cy;
  double r[9];  // camera-to-world rotation, row-major
  double t[3];  // camera centre
};

__global__ void k_view_tsdf(const float* __restrict__ depth, int W, int H,
                            Cam cam, double ox, double oy, double oz,
                            double vox, int n, int i0, int j0, int k0,
                            double delta, double eta, float* f_out,
                            uint8_t* w_out, double* wf_sum, double* w_sum) {
  // the n^3 voxels of the box at global index (i0, j0, k0) (the whole grid:
  // offset 0); outputs indexed box-locally
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n3 = (int64_t)n * n * n;
  if (idx >= n3) return;
  const int k = k0 + (int)(idx % n);
  const int j = j0 + (int)((idx / n) % n);
  const int i = i0 + (int)(idx / ((int64_t)n * n));
  // axis centres minus the camera translation (tsdf.py:93-95)
  const double xs = (ox + ((double)i + 0.5) * vox) - cam.t[0];
  const double ys = (oy + ((double)j + 0.5) * vox) - cam.t[1];
  const double zs = (oz + ((double)k + 0.5) * vox) - cam.t[2];
  const double* r = cam.r;
  const double xc = xs * r[0] + ys * r[3] + zs * r[6];
  const double yc = xs * r[1] + ys * r[4] + zs * r[7];
  const double zc = xs * r[2] + ys * r[5] + zs * r[8];
  const bool front = zc > 0.0;
  const double zsafe = front ? zc : 1.0;
  const double u = cam.fx * xc / zsafe + cam.cx;
  const double v = cam.fy * yc / zsafe + cam.cy;
  const bool inside =
      front && (u >= 0.0) && (u < (double)W) && (v >= 0.0) && (v < (double)H);
  double fu = floor(u + 0.5), fv = floor(v + 0.5);
  fu = fmin(fmax(fu, 0.0), (double)(W - 1));
  fv = fmin(fmax(fv, 0.0), (double)(H - 1));
  const int pu = (int)fu, pv = (int)fv;
  const double d = (double)depth[(int64_t)pv * W + pu];
  const bool observed = inside && (d > 0.0);
  // per-pixel ray norm (volume.py:126-128)
  const double un = ((double)pu - cam.cx) / cam.fx;
  const double vn = ((double)pv - cam.cy) / cam.fy;
  const double norm = sqrt(1.0 + un * un + vn * vn);
  const double dist = sqrt(xc * xc + yc * yc + zc * zc);
  const double phi = d * norm - dist;
  double f = phi / delta;
  f = fmin(fmax(f, -1.0), 1.0);
  const bool w = observed && (phi >= -eta);
  const float fo = w ? __double2float_rn(f) : -1.0f;
  f_out[idx] = fo;
  w_out[idx] = (uint8_t)w;
  if (wf_sum) {  // reference cli.py:148-149 accumulation, view order
    wf_sum[idx] += (double)fo * (double)(w ? 1 : 0);
    w_sum[idx] += (double)(w ? 1 : 0);
  }
}

__global__ void k_initial_field(const double* wf, const double* ws,
                                double gamma, int64_t n, double* u) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double w = ws[i];
  u[i] = w > 0.0 ? wf[i] / (w + gamma) : -1.0;  // fusion.py:149-155
}

// -------------------------------------------------------------- pyramids --
struct Pyr {
  double *mn, *mx, *mean;       // min/max of f64(f); value (mean or weighted)
  uint8_t *wmn, *wmx;           // min/max of w
  double *wm, *wf, *pl;         // means of w, f*w, f (weighted builds)
};

template <typename F>
__global__ void k_pyr_base(const F* __restrict__ f, const uint8_t* w, int64_t n3,
                           Pyr p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const double v = (double)f[i];
  p.mn[i] = v;
  p.mx[i] = v;
  if (w) {
    const uint8_t wi = w[i];
    p.wmn[i] = wi;
    p.wmx[i] = wi;
    p.wm[i] = (double)wi;
    p.wf[i] = v * (double)wi;
    p.pl[i] = v;
    const double wm = (double)wi;
    p.mean[i] = wm > 0.0 ? p.wf[i] / wm : v;
  } else {
    p.mean[i] = v;
  }
}

__device__ __forceinline__ double mean8(const double* a, const int64_t* k) {
  return ((((a[k[0]] + a[k[1]]) + (a[k[2]] + a[k[3]])) + (a[k[4]] + a[k[5]])) +
          (a[k[6]] + a[k[7]])) /
         8.0;
}

// level L (n = 2^L per axis) from level L+1; `off` / `off1` = level offsets
__global__ void k_pyr_level(int64_t off, int64_t off1, int n, Pyr p,
                            int weighted) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n3 = (int64_t)n * n * n;
  if (idx >= n3) return;
  const int k = (int)(idx % n);
  const int j = (int)((idx / n) % n);
  const int i = (int)(idx / ((int64_t)n * n));
  const int n1 = 2 * n;
  int64_t ch[8];
  for (int c = 0; c < 8; ++c)
    ch[c] = off1 + ((int64_t)(2 * i + ((c >> 2) & 1)) * n1 +
                    (2 * j + ((c >> 1) & 1))) *
                       n1 +
            (2 * k + (c & 1));
  const int64_t o = off + idx;
  double mn = p.mn[ch[0]], mx = p.mx[ch[0]];
  for (int c = 1; c < 8; ++c) {
    mn = fmin(mn, p.mn[ch[c]]);
    mx = fmax(mx, p.mx[ch[c]]);
  }
  p.mn[o] = mn;
  p.mx[o] = mx;
  if (weighted) {
    uint8_t a = p.wmn[ch[0]], b = p.wmx[ch[0]];
    for (int c = 1; c < 8; ++c) {
      a = min(a, p.wmn[ch[c]]);
      b = max(b, p.wmx[ch[c]]);
    }
    p.wmn[o] = a;
    p.wmx[o] = b;
    const double wm = mean8(p.wm, ch);
    const double wf = mean8(p.wf, ch);
    const double pl = mean8(p.pl, ch);
    p.wm[o] = wm;
    p.wf[o] = wf;
    p.pl[o] = pl;
    p.mean[o] = wm > 0.0 ? wf / wm : pl;   // octree.py:277-279
  } else {
    p.mean[o] = mean8(p.mean, ch);
  }
}

// ----------------------------------------------------------------- build --
struct BuildScratch {
  uint8_t* split;   // per pyramid cell: splits (if it exists)
  uint8_t* exists;
  int64_t* cnt;     // splitting nodes in the subtree
  int64_t* rank;    // depth-first (child 7 first) rank among splitting nodes
  int32_t* node;    // slot of the cell's node
};

__global__ void k_split_flags(const double* minf, const double* maxf,
                              const uint8_t* wminf, const uint8_t* wmaxf,
                              int has_w, double tau, int64_t off, int64_t n3,
                              int L, int d_max, BuildScratch s) {
  // L, d_max: global levels (a box subtree's level 0 is global level0)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const int64_t k = off + i;
  bool sp = false;
  if (L < d_max) {  // _kernels.pyx:58-63
    if (maxf[k] - minf[k] > tau)
      sp = true;
    else if (has_w && wminf[k] != wmaxf[k])
      sp = true;
  }
  s.split[k] = sp;
  if (n3 == 1) s.exists[k] = 1;  // the (box) root
}

__device__ __forceinline__ int64_t child_index(int64_t off1, int n1, int i,
                                               int j, int k, int c) {
  return off1 + ((int64_t)(2 * i + ((c >> 2) & 1)) * n1 +
                 (2 * j + ((c >> 1) & 1))) *
                    n1 +
         (2 * k + (c & 1));
}

// top-down: children exist iff the parent exists and splits
__global__ void k_exists(int64_t off, int64_t off1, int n, BuildScratch s) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n3 = (int64_t)n * n * n;
  if (idx >= n3) return;
  const int k = (int)(idx % n), j = (int)((idx / n) % n),
            i = (int)(idx / ((int64_t)n * n));
  const uint8_t e = s.exists[off + idx] && s.split[off + idx];
  for (int c = 0; c < 8; ++c) s.exists[child_index(off1, 2 * n, i, j, k, c)] = e;
}

// bottom-up subtree split counts
__global__ void k_counts(int64_t off, int64_t off1, int n, int leaf_level,
                         BuildScratch s) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n3 = (int64_t)n * n * n;
  if (idx >= n3) return;
  const int64_t o = off + idx;
  if (!(s.exists[o] && s.split[o])) {
    s.cnt[o] = 0;
    return;
  }
  int64_t acc = 1;
  if (!leaf_level) {
    const int k = (int)(idx % n), j = (int)((idx / n) % n),
              i = (int)(idx / ((int64_t)n * n));
    for (int c = 0; c < 8; ++c) acc += s.cnt[child_index(off1, 2 * n, i, j, k, c)];
  }
  s.cnt[o] = acc;
}

// top-down ranks and node slots; emits the node arrays of level L+1
template <typename T>
__global__ void k_ranks(int64_t off, int64_t off1, int n, BuildScratch s) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n3 = (int64_t)n * n * n;
  if (idx >= n3) return;
  const int64_t o = off + idx;
  if (!(s.exists[o] && s.split[o])) return;
  const int k = (int)(idx % n), j = (int)((idx / n) % n),
            i = (int)(idx / ((int64_t)n * n));
  const int64_t r = s.rank[o];
  const int64_t base = 1 + 8 * r;
  int64_t later = 0;  // splitting nodes in children c' > c (expanded first)
  for (int c = 7; c >= 0; --c) {
    const int64_t ck = child_index(off1, 2 * n, i, j, k, c);
    s.node[ck] = (int32_t)(base + c);
    if (s.split[ck]) s.rank[ck] = r + 1 + later;
    later += s.cnt[ck];
  }
}

template <typename T>
__global__ void k_emit(int64_t off, int64_t n3, const double* meanf,
                       const double* wmeanf, BuildScratch s, T* value,
                       float* weight, int32_t* child) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n3) return;
  const int64_t o = off + idx;
  if (!s.exists[o]) return;
  const int32_t nd = s.node[o];
  value[nd] = (T)meanf[o];
  if (weight) weight[nd] = (float)wmeanf[o];
  child[nd] = s.split[o] ? (int32_t)(1 + 8 * s.rank[o]) : -1;
}

// propagate over the dense level structure: sequential sum of the 8
// children in order c = 0..7 (_kernels.pyx:104-110)
template <typename T>
__global__ void k_dense_propagate(int64_t off, int64_t off1, int n,
                                  BuildScratch s, T* value) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n3 = (int64_t)n * n * n;
  if (idx >= n3) return;
  const int64_t o = off + idx;
  if (!(s.exists[o] && s.split[o])) return;
  const int k = (int)(idx % n), j = (int)((idx / n) % n),
            i = (int)(idx / ((int64_t)n * n));
  double acc = 0.0;
  for (int c = 0; c < 8; ++c)
    acc += (double)value[s.node[child_index(off1, 2 * n, i, j, k, c)]];
  value[s.node[o]] = (T)(acc / 8.0);
}

template <typename T>
__global__ void k_densify(const T* value, const int32_t* child, int d_max,
                          double* out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = 1 << d_max;
  if (idx >= (int64_t)n * n * n) return;
  const int k = (int)(idx % n), j = (int)((idx / n) % n),
            i = (int)(idx / ((int64_t)n * n));
  out[idx] = (double)value[descend(child, d_max, i, j, k)];
}

std::vector<int64_t> level_offsets(int d_max) {
  std::vector<int64_t> off(d_max + 2);
  int64_t acc = 0;
  for (int l = 0; l <= d_max; ++l) {
    off[l] = acc;
    acc += (int64_t)1 << (3 * l);
  }
  off[d_max + 1] = acc;
  return off;
}

template <typename T>
void build_impl(const BuildIn& in, T* value, float* weight, int32_t* child,
                int64_t* state, bool do_propagate, cudaStream_t st) {
  const int d = in.d_max;
  const std::vector<int64_t> off = in.offs
                                       ? std::vector<int64_t>(in.offs, in.offs + d + 1)
                                       : level_offsets(d);
  const int64_t total = off[d] + ((int64_t)1 << (3 * d));
  DevBuf<uint8_t> split, exists;
  DevBuf<int64_t> cnt, rank;
  DevBuf<int32_t> node;
  BuildScratch s;
  s.split = split.ensure(total);
  s.exists = exists.ensure(total);
  s.cnt = cnt.ensure(total);
  s.rank = rank.ensure(total);
  s.node = node.ensure(total);
  OCTF_CUDA(cudaMemsetAsync(s.exists, 0, total, st));
  for (int L = 0; L <= d; ++L) {
    const int64_t n3 = (int64_t)1 << (3 * L);
    k_split_flags<<<nblk(n3), kB, 0, st>>>(in.minf, in.maxf, in.wminf, in.wmaxf,
                                          in.has_w, in.tau, off[L], n3,
                                          L + in.level0,
                                          in.d_glob >= 0 ? in.d_glob : d, s);
  }
  for (int L = 0; L < d; ++L)
    k_exists<<<nblk((int64_t)1 << (3 * L)), kB, 0, st>>>(off[L], off[L + 1],
                                                         1 << L, s);
  for (int L = d; L >= 0; --L)
    k_counts<<<nblk((int64_t)1 << (3 * L)), kB, 0, st>>>(
        off[L], L < d ? off[L + 1] : 0, 1 << L, L == d, s);
  // the root's depth-first rank and slot: 0 / 0 for a whole tree; a box
  // subtree (octf_build_octree_box) continues the enclosing tree's ranks
  const int64_t root_rank = in.root_rank;
  const int32_t root = in.root_slot;
  OCTF_CUDA(cudaMemcpyAsync(s.rank, &root_rank, sizeof(int64_t),
                            cudaMemcpyHostToDevice, st));
  OCTF_CUDA(cudaMemcpyAsync(s.node, &root, sizeof(int32_t),
                            cudaMemcpyHostToDevice, st));
  for (int L = 0; L < d; ++L)
    k_ranks<T><<<nblk((int64_t)1 << (3 * L)), kB, 0, st>>>(off[L], off[L + 1],
                                                           1 << L, s);
  int64_t nsplit = 0;
  OCTF_CUDA(cudaMemcpyAsync(&nsplit, s.cnt, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
  OCTF_CUDA(cudaStreamSynchronize(st));
  const int64_t used = 1 + 8 * (root_rank + nsplit);
  if (in.nsplit_out) *in.nsplit_out = nsplit;
  if (used > in.cap) throw Error(kEPool, "node pool capacity exhausted");
  for (int L = 0; L <= d; ++L) {
    const int64_t n3 = (int64_t)1 << (3 * L);
    k_emit<T><<<nblk(n3), kB, 0, st>>>(off[L], n3, in.meanf,
                                       in.has_w ? in.wmeanf : nullptr, s, value,
                                       in.has_w ? weight : nullptr, child);
  }
  if (do_propagate)
    for (int L = d - 1; L >= 0; --L)
      k_dense_propagate<T><<<nblk((int64_t)1 << (3 * L)), kB, 0, st>>>(
          off[L], off[L + 1], 1 << L, s, value);
  OCTF_CUDA(cudaGetLastError());
  OCTF_CUDA(cudaStreamSynchronize(st));
  if (state) {
    state[0] = used;
    state[1] = -1;
    state[2] = used;
  }
}

}  // namespace

// ---------------------------------------------------------------- entry --
void view_tsdf(const float* depth, int width, int height, const double* cam,
               const double* origin, double voxel, int n, const int* box,
               double delta, double eta, float* f, uint8_t* w, double* wf_sum,
               double* w_sum, cudaStream_t st) {
  if (delta <= 0 || eta <= 0)
    throw Error(kEArg, "delta and eta must be positive");
  if (n < 1 || (n & (n - 1))) throw Error(kEArg, "resolution must be a power of two");
  Cam c;
  c.fx = cam[0];
  c.fy = cam[1];
  c.cx = cam[2];
  c.cy = cam[3];
  for (int q = 0; q < 9; ++q) c.r[q] = cam[4 + q];
  for (int q = 0; q < 3; ++q) c.t[q] = cam[13 + q];
  // box = {i0, j0, k0, edge} (null: the whole n^3 grid)
  const int nb = box ? box[3] : n;
  if (box && (nb < 1 || box[0] < 0 || box[1] < 0 || box[2] < 0 ||
              box[0] + nb > n || box[1] + nb > n || box[2] + nb > n))
    throw Error(kEArg, "box outside the grid");
  const int64_t n3 = (int64_t)nb * nb * nb;
  k_view_tsdf<<<nblk(n3), kB, 0, st>>>(depth, width, height, c, origin[0],
                                       origin[1], origin[2], voxel, nb,
                                       box ? box[0] : 0, box ? box[1] : 0,
                                       box ? box[2] : 0, delta, eta, f, w,
                                       wf_sum, w_sum);
  OCTF_CUDA(cudaGetLastError());
}

void initial_field(const double* wf, const double* ws, double gamma, int64_t n,
                   double* u, cudaStream_t st) {
  k_initial_field<<<nblk(n), kB, 0, st>>>(wf, ws, gamma, n, u);
  OCTF_CUDA(cudaGetLastError());
}

void pyramids(const void* f, int f_dtype, const uint8_t* w, int d_max,
              double* minf, double* maxf, double* meanf, uint8_t* wminf,
              uint8_t* wmaxf, double* wmeanf, double* wf_tmp, double* pl_tmp,
              cudaStream_t st) {
  if (d_max < 0 || d_max > kMaxDepth) throw Error(kEDepth, "tree depth out of range");
  const std::vector<int64_t> off = level_offsets(d_max);
  Pyr p{minf, maxf, meanf, wminf, wmaxf, wmeanf, wf_tmp, pl_tmp};
  const int64_t n3 = (int64_t)1 << (3 * d_max);
  Pyr pb = p;
  pb.mn += off[d_max];
  pb.mx += off[d_max];
  pb.mean += off[d_max];
  if (w) {
    pb.wmn += off[d_max];
    pb.wmx += off[d_max];
    pb.wm += off[d_max];
    pb.wf += off[d_max];
    pb.pl += off[d_max];
  }
  if (f_dtype == 1)
    k_pyr_base<float><<<nblk(n3), kB, 0, st>>>((const float*)f, w, n3, pb);
  else
    k_pyr_base<double><<<nblk(n3), kB, 0, st>>>((const double*)f, w, n3, pb);
  for (int L = d_max - 1; L >= 0; --L)
    k_pyr_level<<<nblk((int64_t)1 << (3 * L)), kB, 0, st>>>(
        off[L], off[L + 1], 1 << L, p, w != nullptr);
  OCTF_CUDA(cudaGetLastError());
}

void build_tree(const BuildIn& in, void* value, int dtype, float* weight,
                int32_t* child, int64_t* state, bool do_propagate,
                cudaStream_t st) {
  if (in.d_max < 0 || in.d_max > kMaxDepth)
    throw Error(kEDepth, "tree depth out of range");
  if (dtype == 1)
    build_impl<float>(in, (float*)value, weight, child, state, do_propagate, st);
  else
    build_impl<double>(in, (double*)value, weight, child, state, do_propagate,
                       st);
}

void densify(int dtype, const void* value, const int32_t* child, int d_max,
             double* out, cudaStream_t st) {
  if (d_max < 0 || d_max > kMaxDepth) throw Error(kEDepth, "tree depth out of range");
  const int64_t n3 = (int64_t)1 << (3 * d_max);
  if (dtype == 1)
    k_densify<float><<<nblk(n3), kB, 0, st>>>((const float*)value, child, d_max,
                                              out);
  else
    k_densify<double><<<nblk(n3), kB, 0, st>>>((const double*)value, child,
                                               d_max, out);
  OCTF_CUDA(cudaGetLastError());
}

// octree.py:148-166 locate for a batch of cells of one level
__global__ void k_locate(const int32_t* __restrict__ child, int level,
                         const int32_t* __restrict__ cells, int64_t n,
                         int32_t* __restrict__ node, int32_t* __restrict__ lvl) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int l = 0;
  node[i] = descend(child, level, cells[3 * i], cells[3 * i + 1],
                    cells[3 * i + 2], &l);
  lvl[i] = l;
}

void locate(const int32_t* child, int level, const int32_t* cells, int64_t n,
            int32_t* node, int32_t* lvl, cudaStream_t st) {
  if (n <= 0) return;
  k_locate<<<nblk(n), kB, 0, st>>>(child, level, cells, n, node, lvl);
  OCTF_CUDA(cudaGetLastError());
}

}  // namespace octf
