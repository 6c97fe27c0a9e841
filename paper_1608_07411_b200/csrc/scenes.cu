// Ray-marched depth maps of the synthetic scenes (the
// input pipeline on the device).  The reference renders spheres analytically
// (synth.py:80-109); BASELINE configs 2 and 3 need a noisy blob and a room of
// boxes and spheres, which have no closed-form depth, so their pixel rays are
// sphere-traced: conservative steps sd / L until the signed distance bound
// drops under eps, then 40 bisection steps on the last bracket.
//
// One thread per pixel ray, every step in f64 as separate IEEE operations
// (this file is compiled -fmad=false) in the order of the array program in
// scenes.py (`sphere_trace`, `value_noise`, `room_sdf_fn`), which is what the
// golden fixtures' depth maps were made with: the maps are bit-identical.
#include <cuda_runtime.h>

#include <cstdint>

#include "octf_ctx.h"
#include "octf_scenes.h"

namespace octf {
namespace {

struct BlobScene {
  double c[3];
  double radius, amp, base_freq;
  const double* lat[kMaxOctaves];
  int n[kMaxOctaves];
  int noct;
};

struct RoomScene {
  const double* boxes;    // nb x {centre xyz, half extent xyz}
  const double* spheres;  // ns x {centre xyz, radius}
  int nb, ns;
  double size;
};

__device__ __forceinline__ double norm3(double x, double y, double z) {
  return sqrt((x * x + y * y) + z * z);
}

__device__ __forceinline__ double clamp01(double x) {
  return fmin(fmax(x, 0.0), 1.0);
}

// scenes.py value_noise: per octave trilinear interpolation (smoothstep
// fade) of the lattice, amplitude 2^-o, sum divided by the amplitude sum
__device__ double value_noise(const BlobScene& s, const double p[3]) {
  double out = 0.0, amp = 1.0, total = 0.0;
  for (int o = 0; o < s.noct; ++o) {
    const double fr = s.base_freq * (double)(1 << o);
    const int n = s.n[o];
    int i0[3];
    double t[3];
    for (int a = 0; a < 3; ++a) {
      const double q = clamp01(p[a]) * fr;
      const double fl = fmin(floor(q), (double)(n - 2));
      i0[a] = (int)fl;
      const double tt = q - fl;
      t[a] = (tt * tt) * (3.0 - 2.0 * tt);
    }
    const double* tab = s.lat[o];
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dx = (c >> 2) & 1, dy = (c >> 1) & 1, dz = c & 1;
      const double wx = dx ? t[0] : 1.0 - t[0];
      const double wy = dy ? t[1] : 1.0 - t[1];
      const double wz = dz ? t[2] : 1.0 - t[2];
      const double wgt = (wx * wy) * wz;
      const double v =
          __ldg(tab + ((int64_t)(i0[0] + dx) * n + (i0[1] + dy)) * n +
                (i0[2] + dz));
      acc = acc + wgt * v;
    }
    out = out + amp * acc;
    total += amp;
    amp *= 0.5;
  }
  return out * (1.0 / total);  // the array program's form (see sphere_trace)
}

__device__ __forceinline__ double sdf(const BlobScene& s, const double p[3],
                                      const double*) {
  const double r = norm3(p[0] - s.c[0], p[1] - s.c[1], p[2] - s.c[2]);
  return r - (s.radius + s.amp * value_noise(s, p));
}

// scenes.py room_sdf_fn: min over the boxes, the spheres and the six walls.
// `obj` is the CTA's shared-memory copy of the boxes followed by the spheres.
__device__ double sdf(const RoomScene& s, const double p[3],
                      const double* obj) {
  double db = INFINITY, ds = INFINITY;
  const double* b = obj;
  for (int k = 0; k < s.nb; ++k, b += 6) {
    const double qx = fabs(p[0] - b[0]) - b[3];
    const double qy = fabs(p[1] - b[1]) - b[4];
    const double qz = fabs(p[2] - b[2]) - b[5];
    const double outside = norm3(fmax(qx, 0.0), fmax(qy, 0.0), fmax(qz, 0.0));
    const double inside = fmin(fmax(fmax(qx, qy), qz), 0.0);
    db = fmin(db, outside + inside);
  }
  for (int k = 0; k < s.ns; ++k, b += 4)
    ds = fmin(ds, norm3(p[0] - b[0], p[1] - b[1], p[2] - b[2]) - b[3]);
  const double walls =
      fmin(fmin(fmin(p[0], s.size - p[0]), fmin(p[1], s.size - p[1])),
           fmin(p[2], s.size - p[2]));
  return fmin(fmin(db, ds), walls);
}

struct TraceArgs {
  double inv_fx, inv_fy, cx, cy, R[9], o[3];
  int width, height, steps;
  double lipschitz, t_max, eps;
};

template <typename Scene>
__global__ void __launch_bounds__(128)
k_sphere_trace(TraceArgs a, Scene s, int nshared, const double* shared_src,
               double* __restrict__ z) {
  extern __shared__ double obj[];
  for (int q = threadIdx.x; q < nshared; q += blockDim.x)
    obj[q] = shared_src[q];
  __syncthreads();
  // 16 x 8 pixel tiles: neighbouring rays take similar step counts
  const int tiles_x = (a.width + 15) / 16;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int j = tx * 16 + (threadIdx.x & 15), i = ty * 8 + (threadIdx.x >> 4);
  if (i >= a.height || j >= a.width) return;
  const double px = ((double)j - a.cx) * a.inv_fx;
  const double py = ((double)i - a.cy) * a.inv_fy;
  double d[3];
#pragma unroll
  for (int q = 0; q < 3; ++q)
    d[q] = (px * a.R[3 * q] + py * a.R[3 * q + 1]) + 1.0 * a.R[3 * q + 2];
  const double nrm = norm3(d[0], d[1], d[2]);
  const double denom = a.lipschitz * nrm;
  double t = 0.0, t_prev = 0.0;
  bool hit = false;
  for (int it = 0; it < a.steps; ++it) {
    const double p[3] = {a.o[0] + t * d[0], a.o[1] + t * d[1],
                         a.o[2] + t * d[2]};
    const double sd = sdf(s, p, obj);
    if (sd < a.eps) {
      hit = true;
      break;
    }
    t_prev = t;
    t = t + sd / denom;
    if (!(t <= a.t_max)) break;
  }
  double out = 0.0;
  if (hit) {
    double lo = t_prev, hi = t;
    for (int it = 0; it < 40; ++it) {
      const double mid = 0.5 * (lo + hi);
      const double p[3] = {a.o[0] + mid * d[0], a.o[1] + mid * d[1],
                           a.o[2] + mid * d[2]};
      const bool inside = sdf(s, p, obj) < 0.0;
      hi = inside ? mid : hi;
      lo = inside ? lo : mid;
    }
    out = hi;
  }
  z[(int64_t)i * a.width + j] = out;
}

TraceArgs trace_args(const double* cam, int width, int height,
                     double lipschitz, double t_max, int steps, double eps) {
  TraceArgs a;
  a.inv_fx = 1.0 / cam[0];
  a.inv_fy = 1.0 / cam[1];
  a.cx = cam[2];
  a.cy = cam[3];
  for (int q = 0; q < 9; ++q) a.R[q] = cam[4 + q];
  for (int q = 0; q < 3; ++q) a.o[q] = cam[13 + q];
  a.width = width;
  a.height = height;
  a.steps = steps;
  a.lipschitz = lipschitz;
  a.t_max = t_max;
  a.eps = eps;
  return a;
}

unsigned trace_grid(int width, int height) {
  return (unsigned)(((width + 15) / 16) * ((height + 7) / 8));
}

}  // namespace

void trace_blob(const double* cam, int width, int height, const double* centre,
                double radius, double amp, double base_freq,
                const double* const* lattices, const int* lat_n, int noct,
                double lipschitz, double t_max, int steps, double eps,
                double* z, cudaStream_t st) {
  if (noct < 0 || noct > kMaxOctaves)
    throw Error(kEArg, "trace_blob: 0..4 noise octaves");
  BlobScene s;
  for (int q = 0; q < 3; ++q) s.c[q] = centre[q];
  s.radius = radius;
  s.amp = amp;
  s.base_freq = base_freq;
  s.noct = noct;
  for (int o = 0; o < kMaxOctaves; ++o) {
    s.lat[o] = o < noct ? lattices[o] : nullptr;
    s.n[o] = o < noct ? lat_n[o] : 2;
    if (o < noct && (!lattices[o] || lat_n[o] < 2))
      throw Error(kEArg, "trace_blob: lattice of at least 2^3 values");
  }
  const TraceArgs a =
      trace_args(cam, width, height, lipschitz, t_max, steps, eps);
  k_sphere_trace<BlobScene><<<trace_grid(width, height), 128, 0, st>>>(
      a, s, 0, nullptr, z);
  OCTF_CUDA(cudaGetLastError());
}

void trace_room(const double* cam, int width, int height, const double* objects,
                int nb, int ns, double size, double lipschitz, double t_max,
                int steps, double eps, double* z, cudaStream_t st) {
  if (nb < 0 || ns < 0 || (int64_t)nb * 6 + (int64_t)ns * 4 > 5000)
    throw Error(kEArg, "trace_room: at most 5000 object parameters");
  RoomScene s;
  s.boxes = objects;
  s.spheres = objects + (int64_t)nb * 6;
  s.nb = nb;
  s.ns = ns;
  s.size = size;
  const int nsh = nb * 6 + ns * 4;
  const TraceArgs a =
      trace_args(cam, width, height, lipschitz, t_max, steps, eps);
  k_sphere_trace<RoomScene>
      <<<trace_grid(width, height), 128, nsh * sizeof(double), st>>>(
          a, s, nsh, objects, z);
  OCTF_CUDA(cudaGetLastError());
}

}  // namespace octf
