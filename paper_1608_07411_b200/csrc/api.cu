// extern "C" boundary (include/octfuse_b200.h): argument checks, error
// mapping and precision dispatch.  No compute happens here.
#include <cstring>
#include <string>

#include "../../include/octfuse_b200.h"
#include "octf_build.h"
#include "octf_scenes.h"
#include "octf_mesh_diff.h"
#include "octf_ctx.h"

struct octf_ctx {
  octf::Ctx c;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return OCTF_OK;
  } catch (const octf::Error& e) {
    return fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(OCTF_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(OCTF_ECUDA, e.what());
  }
}

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

void need_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw octf::Error(octf::kECuda, "no CUDA device available");
  }
  octf::pool_keep();
}

void check_dtype(int dtype) {
  if (dtype != OCTF_F64 && dtype != OCTF_F32)
    throw octf::Error(octf::kEArg, "dtype must be OCTF_F64 or OCTF_F32");
}

octf::PassParams make_params(int d_max, double lam, double eps, double gamma,
                             double xi, double tau_s, double tau_j, int clamp,
                             int reverse) {
  octf::PassParams p;
  p.d_max = d_max;
  p.lam = lam;
  p.eps2 = eps * eps;  // _kernels.pyx:405
  p.gamma = gamma;
  p.xi = xi;
  p.tau_s = tau_s;
  p.tau_j = tau_j;
  p.clamp = clamp;
  p.reverse = reverse;
  return p;
}

}  // namespace

extern "C" {

const char* octf_last_error(void) { return g_err.c_str(); }

int octf_version(void) { return 100; }

int octf_selftest(void) {
  using namespace octf;
  // Morton order == x-major child index at every level
  for (int x = 0; x < 4; ++x)
    for (int y = 0; y < 4; ++y)
      for (int z = 0; z < 4; ++z) {
        uint64_t k = morton3(x, y, z);
        uint64_t ref = ((uint64_t)octant(x >> 1, y >> 1, z >> 1) << 3) |
                       (uint64_t)octant(x, y, z);
        if (k != ref) return 1;
      }
  // neighbour directions round-trip
  for (int d = 0; d < 12; ++d) {
    int ox, oy, oz;
    dir_offset(d, ox, oy, oz);
    if (nbr_dir(ox, oy, oz) != d) return 2;
  }
  int used = 0;
  for (int ox = -1; ox <= 1; ++ox)
    for (int oy = -1; oy <= 1; ++oy)
      for (int oz = -1; oz <= 1; ++oz) used += nbr_dir(ox, oy, oz) >= 0;
  if (used != 12) return 3;
  // every stencil point of the reference's delta_u (_kernels.pyx:205-242)
  // maps to its own block or one of the 12 tabled neighbours
  const int pts[13][3] = {{0, 0, 0},  {1, 0, 0},  {0, 1, 0},  {0, 0, 1},
                          {-1, 0, 0}, {-1, 1, 0}, {-1, 0, 1}, {0, -1, 0},
                          {1, -1, 0}, {0, -1, 1}, {0, 0, -1}, {1, 0, -1},
                          {0, 1, -1}};
  for (int c = 0; c < 8; ++c)
    for (auto& p : pts) {
      int tx = ((c >> 2) & 1) + p[0], ty = ((c >> 1) & 1) + p[1],
          tz = (c & 1) + p[2];
      int ox = tx >> 1, oy = ty >> 1, oz = tz >> 1;
      if ((ox | oy | oz) != 0 && nbr_dir(ox, oy, oz) < 0) return 4;
    }
  // pack/unpack
  int L, x, y, z;
  unpack_cell(pack_cell(19, 524287, 3, 524000), L, x, y, z);
  if (L != 19 || x != 524287 || y != 3 || z != 524000) return 5;
  // pre/post-order keys: parent before child, child before parent
  if (!(preorder_key(1, 1, 0, 0, 3, false) < preorder_key(2, 2, 0, 0, 3, false)))
    return 6;
  if (!(postorder_key(2, 3, 1, 1, 3, false) < postorder_key(1, 1, 0, 0, 3, false)))
    return 7;
  if (!(postorder_key(1, 0, 1, 1, 3, false) < postorder_key(2, 2, 0, 0, 3, false)))
    return 8;
  return 0;
}

int octf_ctx_create(octf_ctx** out) {
  return guard([&] {
    if (!out) throw octf::Error(octf::kEArg, "null output pointer");
    need_device();
    *out = new octf_ctx();
  });
}

int octf_ctx_destroy(octf_ctx* ctx) {
  delete ctx;
  return OCTF_OK;
}

int octf_ctx_invalidate(octf_ctx* ctx) {
  if (ctx) {
    ctx->c.valid = false;
    ctx->c.free_ok = false;
    ctx->c.own_change = false;
    ctx->c.store_ok = false;
    ctx->c.vkey.clear();
    if (!ctx->c.ext_F) ctx->c.nviews = 0;
  }
  return OCTF_OK;
}

int octf_ctx_set_options(octf_ctx* ctx, int flags) {
  return guard([&] {
    if (!ctx) throw octf::Error(octf::kEArg, "null context");
    const bool dense = (flags & OCTF_CTX_DENSE) != 0;
    const bool ell = (flags & OCTF_CTX_ELL) != 0;
    const bool sorted = (flags & OCTF_CTX_SORTED) != 0;
    if (dense && ell)
      throw octf::Error(octf::kEArg, "ELL excludes the dense layout");
    ctx->c.defer_gather = (flags & OCTF_CTX_DEFER) != 0;
    const bool pack = (flags & OCTF_CTX_PACKED) != 0;
    if (pack != ctx->c.pack_opt) {
      ctx->c.pack_opt = pack;
      ctx->c.store_ok = false;
      ctx->c.valid = false;  // regather at packed positions
    }
    if (dense != ctx->c.dense_only || ell != ctx->c.force_ell ||
        sorted != ctx->c.sorted) {
      ctx->c.dense_only = dense;
      ctx->c.force_ell = ell;
      ctx->c.sorted = sorted;
      ctx->c.store_ok = false;
      ctx->c.valid = false;  // regather in the requested layout
    }
  });
}

int octf_ctx_info(octf_ctx* ctx, int64_t* out) {
  return guard([&] {
    if (!ctx || !out) throw octf::Error(octf::kEArg, "null argument");
    const octf::Ctx& c = ctx->c;
    out[0] = c.nlb;
    out[1] = c.nleaves;
    out[2] = c.nblocks;
    out[3] = c.nfree;
    out[4] = c.binw;
    out[5] = c.sstride;
    out[6] = c.nviews;
    out[7] = c.valid;
    out[8] = (c.nlb * 8 + 255) / 256;  // leaf tiles (one CTA each)
    out[9] = c.ell ? 1 : 0;
    out[10] = c.allv ? 1 : 0;
    out[11] = c.packed ? 1 : 0;
  });
}

int octf_ctx_profile(octf_ctx* ctx, int enable, double* out) {
  return guard([&] {
    if (!ctx) throw octf::Error(octf::kEArg, "null context");
    octf::Ctx& c = ctx->c;
    if (enable && !c.tev[0])
      for (auto& e : c.tev) OCTF_CUDA(cudaEventCreate(&e));
    while (enable && c.pev.size() < 64) {  // per-pass pairs, batched passes
      cudaEvent_t e;
      OCTF_CUDA(cudaEventCreate(&e));
      c.pev.push_back(e);
    }
    if (c.tile_ev_used) {  // tile-range launches: all of a pass's ranges
      OCTF_CUDA(cudaEventSynchronize(c.tile_ev[2 * c.tile_ev_used - 1]));
      for (size_t k = 0; k < c.tile_ev_used; ++k) {
        float ms = 0.f;
        OCTF_CUDA(cudaEventElapsedTime(&ms, c.tile_ev[2 * k], c.tile_ev[2 * k + 1]));
        c.t_leaf_ms += ms;
      }
      c.n_leaf += c.tile_passes;
    }
    c.tile_ev_used = 0;
    c.tile_passes = 0;
    if (out) {
      out[0] = c.t_leaf_ms;
      out[1] = (double)c.n_leaf;
      out[2] = c.t_energy_ms;
      out[3] = (double)c.n_energy;
      out[4] = (double)c.launches;
    }
    c.t_leaf_ms = c.t_energy_ms = 0;
    c.n_leaf = c.n_energy = c.launches = 0;
    c.t_prep_ms = c.t_gather_ms = c.t_restr_ms = 0;
    for (double& t : c.t_ph) t = 0;
    c.n_prep = c.n_gather = 0;
    c.timing = enable != 0;
  });
}

int octf_ctx_phases(octf_ctx* ctx, double* out) {
  return guard([&] {
    if (!ctx || !out) throw octf::Error(octf::kEArg, "null argument");
    const octf::Ctx& c = ctx->c;
    out[0] = c.t_prep_ms;
    out[1] = (double)c.n_prep;
    out[2] = c.t_gather_ms;
    out[3] = (double)c.n_gather;
    out[4] = c.t_restr_ms;
    for (int k = 0; k < octf::kPhCount; ++k) out[5 + k] = c.t_ph[k];
  });
}

int octf_iterate_pass(octf_ctx* ctx, int dtype, void* usnap, void* uval,
                      int32_t* uchild, uint8_t* ujoined, int64_t* ustate,
                      int64_t cap, int nviews, const float* const* vvals,
                      const float* const* vws, const int32_t* const* vchilds,
                      int d_max, double lam, double eps, double gamma,
                      double xi, double tau_s, double tau_j, int clamp,
                      int reverse, int snapshot, double* jlog, int64_t jcap,
                      int64_t* out3, void* stream) {
  return guard([&] {
    if (!ctx || !usnap || !uval || !uchild || !ujoined || !ustate || !out3)
      throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (d_max > 60 || d_max > OCTF_MAX_DEPTH || d_max < 0)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (nviews < 1 && !ctx->c.ext_F)
      throw octf::Error(octf::kEArg, "at least one view is required");
    octf::ctx_set_views(ctx->c, nviews, vvals, vws, vchilds, S(stream));
    octf::IterArgs a;
    a.usnap = usnap;
    a.uval = uval;
    a.child = uchild;
    a.joined = ujoined;
    a.state = ustate;
    a.cap = cap;
    a.prm = make_params(d_max, lam, eps, gamma, xi, tau_s, tau_j, clamp,
                        reverse);
    a.jlog = jlog;
    a.jcap = jlog ? jcap : 0;
    a.snapshot = snapshot;
    if (dtype == OCTF_F64)
      octf::iterate_pass_f64(ctx->c, a, S(stream));
    else
      octf::iterate_pass_f32(ctx->c, a, S(stream));
    out3[0] = a.out3[0];
    out3[1] = a.out3[1];
    out3[2] = a.out3[2];
  });
}

int octf_fuse_pass(octf_ctx* ctx, int dtype, void* usnap, void* uval,
                   int32_t* uchild, uint8_t* ujoined, int64_t* ustate,
                   int64_t cap, int nviews, const float* const* vvals,
                   const float* const* vws, const int32_t* const* vchilds,
                   int d_max, double lam, double eps, double gamma, double xi,
                   double tau_s, double tau_j, int clamp, int reverse,
                   double* jlog, int64_t jcap, int64_t* out3,
                   double* energy_pre, void* stream) {
  return guard([&] {
    if (!ctx || !usnap || !uval || !uchild || !ujoined || !ustate || !out3 ||
        !energy_pre)
      throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (nviews < 1 && !ctx->c.ext_F)
      throw octf::Error(octf::kEArg, "at least one view is required");
    octf::ctx_set_views(ctx->c, nviews, vvals, vws, vchilds, S(stream));
    octf::IterArgs a;
    a.usnap = usnap;
    a.uval = uval;
    a.child = uchild;
    a.joined = ujoined;
    a.state = ustate;
    a.cap = cap;
    a.prm = make_params(d_max, lam, eps, gamma, xi, tau_s, tau_j, clamp,
                        reverse);
    a.jlog = jlog;
    a.jcap = jlog ? jcap : 0;
    a.snapshot = 0;
    a.want_energy = 1;
    if (dtype == OCTF_F64) {
      octf::iterate_pass_f64(ctx->c, a, S(stream));
      octf::propagate_ctx_f64(ctx->c, (double*)uval, uchild, S(stream));
    } else {
      octf::iterate_pass_f32(ctx->c, a, S(stream));
      octf::propagate_ctx_f32(ctx->c, (float*)uval, uchild, S(stream));
    }
    out3[0] = a.out3[0];
    out3[1] = a.out3[1];
    out3[2] = a.out3[2];
    *energy_pre = a.energy_pre;
  });
}

int octf_fuse_passes(octf_ctx* ctx, int dtype, void* ubuf0, void* ubuf1,
                     int32_t* uchild, uint8_t* ujoined, int64_t* ustate,
                     int64_t cap, int nviews, const float* const* vvals,
                     const float* const* vws, const int32_t* const* vchilds,
                     int d_max, double lam, double eps, double gamma,
                     double tau_s, double tau_j, int clamp, int reverse,
                     const double* xis, int npasses, int64_t* out3,
                     double* energies_pre, int* done, void* stream) {
  if (done) *done = 0;
  return guard([&] {
    if (!ctx || !ubuf0 || !ubuf1 || !uchild || !ujoined || !ustate || !xis ||
        !out3 || !energies_pre || !done)
      throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (nviews < 1 && !ctx->c.ext_F)
      throw octf::Error(octf::kEArg, "at least one view is required");
    octf::ctx_set_views(ctx->c, nviews, vvals, vws, vchilds, S(stream));
    void* buf[2] = {ubuf0, ubuf1};
    for (int k = 0; k < npasses; ++k) {
      octf::IterArgs a;
      a.usnap = buf[k & 1];
      a.uval = buf[(k + 1) & 1];
      a.child = uchild;
      a.joined = ujoined;
      a.state = ustate;
      a.cap = cap;
      a.prm = make_params(d_max, lam, eps, gamma, xis[k], tau_s, tau_j, clamp,
                          reverse);
      a.jlog = nullptr;
      a.jcap = 0;
      a.snapshot = 0;
      a.want_energy = 1;
      // a pass that runs out of pool capacity throws before any structural
      // write: *done passes are complete, buffer (done & 1) holds the state
      if (dtype == OCTF_F64) {
        octf::iterate_pass_f64(ctx->c, a, S(stream));
        octf::propagate_ctx_f64(ctx->c, (double*)a.uval, uchild, S(stream));
      } else {
        octf::iterate_pass_f32(ctx->c, a, S(stream));
        octf::propagate_ctx_f32(ctx->c, (float*)a.uval, uchild, S(stream));
      }
      out3[3 * k] = a.out3[0];
      out3[3 * k + 1] = a.out3[1];
      out3[3 * k + 2] = ustate[2];
      energies_pre[k] = a.energy_pre;
      *done = k + 1;
    }
  });
}

int octf_fuse_passes_frozen(octf_ctx* ctx, int dtype, void* ubuf0, void* ubuf1,
                            const int32_t* uchild, const int64_t* ustate,
                            int64_t cap, int nviews, const float* const* vvals,
                            const float* const* vws,
                            const int32_t* const* vchilds, int d_max,
                            double lam, double eps, double gamma,
                            double tau_s, double tau_j, int clamp,
                            const double* xis, int npasses,
                            double* energies_pre, int device_energies,
                            void* stream) {
  return guard([&] {
    if (!ctx || !ubuf0 || !ubuf1 || !uchild || !ustate || !xis ||
        !energies_pre)
      throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (nviews < 1 && !ctx->c.ext_F)
      throw octf::Error(octf::kEArg, "at least one view is required");
    octf::ctx_set_views(ctx->c, nviews, vvals, vws, vchilds, S(stream));
    octf::FrozenArgs a;
    a.ubuf[0] = ubuf0;
    a.ubuf[1] = ubuf1;
    a.child = uchild;
    a.state = ustate;
    a.cap = cap;
    a.prm = make_params(d_max, lam, eps, gamma, 0.0, tau_s, tau_j, clamp, 0);
    a.xis = xis;
    a.npasses = npasses;
    a.energies_pre = energies_pre;
    a.dev_energies = device_energies != 0;
    if (dtype == OCTF_F64)
      octf::frozen_passes_f64(ctx->c, a, S(stream));
    else
      octf::frozen_passes_f32(ctx->c, a, S(stream));
  });
}

int octf_marching_cubes(const double* values, const uint8_t* mask, int n,
                        const int8_t* tri_table, const int8_t* tri_count,
                        const int8_t* edge_axis, const int8_t* edge_offset,
                        const double* origin, double voxel_size, int world,
                        octf_mesh** out, int64_t* nverts, int64_t* nfaces,
                        void* stream) {
  return guard([&] {
    if (!values || !tri_table || !tri_count || !edge_axis || !edge_offset ||
        !origin || !out || !nverts || !nfaces)
      throw octf::Error(octf::kEArg, "null argument");
    need_device();
    octf_mesh* m = new octf_mesh();
    try {
      octf::marching_cubes(values, mask, n, tri_table, tri_count, edge_axis,
                           edge_offset, origin, voxel_size, world, m, S(stream));
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
    *nverts = m->nv;
    *nfaces = m->nf;
  });
}

int octf_marching_cubes_tree(octf_ctx* ctx, int dtype, const void* value,
                             const int32_t* child, const int64_t* state,
                             int64_t cap, int d_max, int seen_dtype,
                             const void* seen_value, const int32_t* seen_child,
                             const int8_t* tri_table, const int8_t* tri_count,
                             const int8_t* edge_axis, const int8_t* edge_offset,
                             const double* origin, double voxel_size,
                             int world, int64_t slab0, int64_t slab1,
                             octf_mesh** out, int64_t* nverts,
                             int64_t* nfaces, void* stream) {
  return guard([&] {
    check_dtype(dtype);
    check_dtype(seen_dtype);
    if (!value || !child || !state || !tri_table || !tri_count || !edge_axis ||
        !edge_offset || !origin || !out || !nverts || !nfaces)
      throw octf::Error(octf::kEArg, "null argument");
    if ((seen_value == nullptr) != (seen_child == nullptr))
      throw octf::Error(octf::kEArg, "seen tree: values and children");
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    need_device();
    octf_ctx tmp;
    octf::Ctx& c = ctx ? ctx->c : tmp.c;
    if (!c.valid || c.child_key != child || c.cap != cap || c.d_max != d_max ||
        c.hstate[0] != state[0] || c.hstate[1] != state[1])
      octf::ctx_prepare(c, child, cap, state, d_max, S(stream));
    octf_mesh* m = new octf_mesh();
    try {
      octf::marching_cubes_tree(c, dtype, value, child, d_max, seen_dtype,
                                seen_value, seen_child, tri_table, tri_count,
                                edge_axis, edge_offset, origin, voxel_size,
                                world, slab0, slab1, m, S(stream));
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
    *nverts = m->nv;
    *nfaces = m->nf;
  });
}

int octf_mesh_copy(octf_mesh* m, double* verts, int32_t* faces, void* stream) {
  return guard([&] {
    if (!m) throw octf::Error(octf::kEArg, "null mesh");
    if (m->nv && verts)
      OCTF_CUDA(cudaMemcpyAsync(verts, m->verts, m->nv * 3 * sizeof(double),
                                cudaMemcpyDeviceToDevice, S(stream)));
    if (m->nf && faces)
      OCTF_CUDA(cudaMemcpyAsync(faces, m->faces, m->nf * 3 * sizeof(int32_t),
                                cudaMemcpyDeviceToDevice, S(stream)));
    OCTF_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int octf_mesh_free(octf_mesh* m) {
  delete m;
  return OCTF_OK;
}

int octf_pass_tiles(octf_ctx* ctx, int dtype, const void* usnap, void* uval,
                    const int32_t* uchild, const int64_t* ustate, int64_t cap,
                    int nviews, const float* const* vvals,
                    const float* const* vws, const int32_t* const* vchilds,
                    int d_max, double lam, double eps, double gamma, double xi,
                    int clamp, int tile0, int ntiles, void* stream) {
  return guard([&] {
    if (!ctx || !usnap || !uval || !uchild || !ustate)
      throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (!clamp) throw octf::Error(octf::kEArg, "tile passes are frozen: clamp");
    octf::ctx_set_views(ctx->c, nviews, vvals, vws, vchilds, S(stream));
    octf::TileArgs a;
    a.usnap = usnap;
    a.uval = uval;
    a.child = uchild;
    a.state = ustate;
    a.cap = cap;
    a.prm = make_params(d_max, lam, eps, gamma, xi, 0.0, 2.0, clamp, 0);
    a.tile0 = tile0;
    a.ntiles = ntiles;
    if (dtype == OCTF_F64)
      octf::pass_tiles_f64(ctx->c, a, S(stream));
    else
      octf::pass_tiles_f32(ctx->c, a, S(stream));
  });
}

int octf_pass_finish(octf_ctx* ctx, int dtype, void* uval,
                     const int32_t* uchild, double* dev_energy, void* stream) {
  return guard([&] {
    if (!ctx || !uval || !uchild || !dev_energy)
      throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (dtype == OCTF_F64)
      octf::pass_finish_f64(ctx->c, uval, uchild, dev_energy, S(stream));
    else
      octf::pass_finish_f32(ctx->c, uval, uchild, dev_energy, S(stream));
  });
}

int octf_pd_passes(octf_ctx* ctx, int dtype, void* const* set_a,
                   void* const* set_b, const int32_t* uchild,
                   const int64_t* ustate, int64_t cap, int nviews,
                   const float* const* vvals, const float* const* vws,
                   const int32_t* const* vchilds, int d_max, double lam,
                   double tau, double sigma, double gamma, int clamp,
                   int npasses, double* energies_pre, int device_energies,
                   void* stream) {
  return guard([&] {
    if (!ctx || !set_a || !set_b || !uchild || !ustate || !energies_pre)
      throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (nviews < 1 && !ctx->c.ext_F)
      throw octf::Error(octf::kEArg, "at least one view is required");
    if (!(tau > 0 && sigma > 0 && lam > 0 && gamma > 0))
      throw octf::Error(octf::kEArg, "tau, sigma, lam, gamma must be positive");
    octf::ctx_set_views(ctx->c, nviews, vvals, vws, vchilds, S(stream));
    octf::PdHostArgs a;
    for (int q = 0; q < 5; ++q) {
      a.in[q] = set_a[q];
      a.out[q] = set_b[q];
    }
    a.child = uchild;
    a.state = ustate;
    a.cap = cap;
    a.d_max = d_max;
    a.lam = lam;
    a.tau = tau;
    a.sigma = sigma;
    a.gamma = gamma;
    a.clamp = clamp;
    a.npasses = npasses;
    a.dev_energies = device_energies != 0;
    a.energies = energies_pre;
    if (dtype == OCTF_F64)
      octf::pd_passes_f64(ctx->c, a, S(stream));
    else
      octf::pd_passes_f32(ctx->c, a, S(stream));
  });
}

int octf_pd_restructure(octf_ctx* ctx, int dtype, void* const* set,
                        int32_t* uchild, int64_t* ustate, int64_t cap,
                        int d_max, double tau_split, double tau_join,
                        int64_t* out2, void* stream) {
  return guard([&] {
    if (!ctx || !set || !uchild || !ustate || !out2)
      throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (!ctx->c.valid)
      throw octf::Error(octf::kEArg, "context not prepared (run a pass first)");
    octf::PdRsArgs a;
    for (int q = 0; q < 5; ++q) a.f[q] = set[q];
    a.child = uchild;
    a.state = ustate;
    a.cap = cap;
    a.d_max = d_max;
    a.tau_s = tau_split;
    a.tau_j = tau_join;
    if (dtype == OCTF_F64)
      octf::pd_restructure_f64(ctx->c, a, S(stream));
    else
      octf::pd_restructure_f32(ctx->c, a, S(stream));
    out2[0] = a.out2[0];
    out2[1] = a.out2[1];
  });
}

int octf_ctx_prepare(octf_ctx* ctx, const int32_t* uchild,
                     const int64_t* ustate, int64_t cap, int d_max, int nviews,
                     const float* const* vvals, const float* const* vws,
                     const int32_t* const* vchilds, void* stream) {
  return guard([&] {
    if (!ctx || !uchild || !ustate) throw octf::Error(octf::kEArg, "null argument");
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (nviews > 0)
      octf::ctx_set_views(ctx->c, nviews, vvals, vws, vchilds, S(stream));
    octf::ctx_prepare(ctx->c, uchild, cap, ustate, d_max, S(stream));
  });
}

int octf_ctx_set_samples(octf_ctx* ctx, const float* f_slot,
                         const float* w_slot, int nviews, int64_t cap,
                         void* stream) {
  return guard([&] {
    if (!ctx || !f_slot) throw octf::Error(octf::kEArg, "null argument");
    if (nviews < 1) throw octf::Error(octf::kEArg, "at least one view is required");
    octf::ctx_set_samples(ctx->c, f_slot, w_slot, nviews, cap, S(stream));
  });
}

int octf_ctx_select(octf_ctx* ctx, const int32_t* sel, const uint8_t* masks,
                    int64_t nsel, void* stream) {
  return guard([&] {
    if (!ctx || (nsel && (!sel || !masks)))
      throw octf::Error(octf::kEArg, "null argument");
    octf::ctx_select(ctx->c, sel, masks, nsel, S(stream));
  });
}

int octf_propagate_levels(octf_ctx* ctx, int dtype, void* value,
                          const int32_t* child, int lo, int hi, void* stream) {
  return guard([&] {
    if (!ctx || !value || !child) throw octf::Error(octf::kEArg, "null argument");
    check_dtype(dtype);
    if (dtype == OCTF_F64)
      octf::propagate_levels_f64(ctx->c, (double*)value, child, lo, hi,
                                 S(stream));
    else
      octf::propagate_levels_f32(ctx->c, (float*)value, child, lo, hi,
                                 S(stream));
  });
}

int octf_halo_pack(int dtype, void* const* fields, int nfields,
                   const int32_t* idx, int64_t n, void* buf, int unpack,
                   void* stream) {
  return guard([&] {
    check_dtype(dtype);
    if (!fields || (n && (!idx || !buf)))
      throw octf::Error(octf::kEArg, "null argument");
    for (int k = 0; k < nfields; ++k)
      if (!fields[k]) throw octf::Error(octf::kEArg, "null field");
    if (dtype == OCTF_F64)
      octf::halo_pack<double>((double* const*)fields, nfields, idx, n,
                              (double*)buf, unpack != 0, S(stream));
    else
      octf::halo_pack<float>((float* const*)fields, nfields, idx, n,
                             (float*)buf, unpack != 0, S(stream));
  });
}

int octf_propagate(octf_ctx* ctx, int dtype, void* value, const int32_t* child,
                   const int64_t* state, int64_t cap, int d_max, void* stream) {
  return guard([&] {
    check_dtype(dtype);
    if (!value || !child) throw octf::Error(octf::kEArg, "null argument");
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    need_device();
    octf_ctx tmp;
    octf::Ctx& c = ctx ? ctx->c : tmp.c;
    int64_t st3[3] = {cap, -1, cap};
    const int64_t* stp = state ? state : st3;
    if (!c.valid || c.child_key != child || c.cap != cap || c.d_max != d_max)
      octf::ctx_prepare(c, child, cap, stp, d_max, S(stream));
    if (dtype == OCTF_F64)
      octf::propagate_ctx_f64(c, (double*)value, child, S(stream));
    else
      octf::propagate_ctx_f32(c, (float*)value, child, S(stream));
    if (!ctx) OCTF_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int octf_node_order(octf_ctx* ctx, const int32_t* child, const int64_t* state,
                    int64_t cap, int d_max, int leaves_only, int32_t* slots,
                    uint64_t* keys, int64_t* count, void* stream) {
  return guard([&] {
    if (!child || !state || !count)
      throw octf::Error(octf::kEArg, "null argument");
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    need_device();
    octf_ctx tmp;
    octf::Ctx& c = ctx ? ctx->c : tmp.c;
    if (!c.valid || c.child_key != child || c.cap != cap || c.d_max != d_max ||
        c.hstate[0] != state[0] || c.hstate[1] != state[1])
      octf::ctx_prepare(c, child, cap, state, d_max, S(stream));
    *count = octf::ctx_node_order(c, child, d_max, leaves_only != 0, slots,
                                  keys, S(stream));
  });
}

int octf_tree_energy(octf_ctx* ctx, int dtype, const void* uval,
                     const int32_t* uchild, const int64_t* ustate, int64_t cap,
                     int nviews, const float* const* vvals,
                     const float* const* vws, const int32_t* const* vchilds,
                     int d_max, double lam, double eps, double gamma,
                     double* out, double* terms, void* stream) {
  return guard([&] {
    check_dtype(dtype);
    if (!uval || !uchild || !out) throw octf::Error(octf::kEArg, "null argument");
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    need_device();
    octf_ctx tmp;
    octf::Ctx& c = ctx ? ctx->c : tmp.c;
    int64_t st3[3] = {cap, -1, cap};
    const int64_t* stp = ustate ? ustate : st3;
    octf::ctx_set_views(c, nviews, vvals, vws, vchilds, S(stream));
    if (!c.valid || c.child_key != uchild || c.cap != cap || c.d_max != d_max)
      octf::ctx_prepare(c, uchild, cap, stp, d_max, S(stream));
    const octf::PassParams p =
        make_params(d_max, lam, eps, gamma, 0.0, 0.0, 1.0, 1, 0);
    *out = dtype == OCTF_F64
               ? octf::energy_f64(c, (const double*)uval, uchild, p, terms,
                                  S(stream))
               : octf::energy_f32(c, (const float*)uval, uchild, p, terms,
                                  S(stream));
  });
}

int octf_densify(int dtype, const void* value, const int32_t* child, int d_max,
                 double* out, void* stream) {
  return guard([&] {
    check_dtype(dtype);
    need_device();
    octf::densify(dtype, value, child, d_max, out, S(stream));
    OCTF_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int octf_build_tree(const double* meanf, const double* minf,
                    const double* maxf, const int64_t* offs, int has_w,
                    const uint8_t* wminf, const uint8_t* wmaxf,
                    const double* wmeanf, double tau, void* value, int dtype,
                    float* weight, int32_t* child, int64_t* state, int64_t cap,
                    int d_max, void* stream) {
  return guard([&] {
    check_dtype(dtype);
    if (d_max > 60) throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (!meanf || !minf || !maxf || !value || !child || !state)
      throw octf::Error(octf::kEArg, "null argument");
    if (has_w && (!wminf || !wmaxf || !wmeanf || !weight))
      throw octf::Error(octf::kEArg, "weighted build needs weight pyramids");
    need_device();
    octf::BuildIn in{meanf, minf, maxf, offs, has_w, wminf, wmaxf, wmeanf,
                     tau, d_max, cap};
    octf::build_tree(in, value, dtype, weight, child, state, false, S(stream));
  });
}

int octf_pyramids(const void* f, int f_dtype, const uint8_t* w, int d_max,
                  double* minf, double* maxf, double* meanf, uint8_t* wminf,
                  uint8_t* wmaxf, double* wmeanf, double* wf_tmp,
                  double* pl_tmp, void* stream) {
  return guard([&] {
    check_dtype(f_dtype);
    if (w && (!wminf || !wmaxf || !wmeanf || !wf_tmp || !pl_tmp))
      throw octf::Error(octf::kEArg, "weighted pyramids need all outputs");
    need_device();
    octf::pyramids(f, f_dtype, w, d_max, minf, maxf, meanf, wminf, wmaxf,
                   wmeanf, wf_tmp, pl_tmp, S(stream));
  });
}

int octf_build_octree(const void* f, int f_dtype, const uint8_t* w, int d_max,
                      double tau, void* value, int dtype, float* weight,
                      int32_t* child, int64_t* state, int64_t cap,
                      void* stream) {
  return guard([&] {
    check_dtype(f_dtype);
    check_dtype(dtype);
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (w && !weight) throw octf::Error(octf::kEArg, "weighted build needs weight");
    need_device();
    int64_t total = 0;
    for (int l = 0; l <= d_max; ++l) total += (int64_t)1 << (3 * l);
    octf::DevBuf<double> mn, mx, mean, wm, wf, pl;
    octf::DevBuf<uint8_t> wmn, wmx;
    mn.ensure(total);
    mx.ensure(total);
    mean.ensure(total);
    if (w) {
      wm.ensure(total);
      wf.ensure(total);
      pl.ensure(total);
      wmn.ensure(total);
      wmx.ensure(total);
    }
    octf::pyramids(f, f_dtype, w, d_max, mn.p, mx.p, mean.p, wmn.p, wmx.p,
                   wm.p, wf.p, pl.p, S(stream));
    octf::BuildIn in{mean.p, mn.p, mx.p, nullptr, w != nullptr, wmn.p, wmx.p,
                     wm.p, tau, d_max, cap};
    // weighted trees keep their pyramid values (octree.py:302-305)
    octf::build_tree(in, value, dtype, w ? weight : nullptr, child, state,
                     w == nullptr, S(stream));
  });
}

int octf_view_tsdf(const float* depth, int width, int height,
                   const double* cam, const double* origin, double voxel,
                   int n, double delta, double eta, float* f, uint8_t* w,
                   double* wf_sum, double* w_sum, void* stream) {
  return octf_view_tsdf_box(depth, width, height, cam, origin, voxel, n,
                            nullptr, delta, eta, f, w, wf_sum, w_sum, stream);
}

int octf_view_tsdf_box(const float* depth, int width, int height,
                       const double* cam, const double* origin, double voxel,
                       int n, const int32_t* box, double delta, double eta,
                       float* f, uint8_t* w, double* wf_sum, double* w_sum,
                       void* stream) {
  return guard([&] {
    if (!depth || !cam || !origin || !f || !w)
      throw octf::Error(octf::kEArg, "null argument");
    if ((wf_sum == nullptr) != (w_sum == nullptr))
      throw octf::Error(octf::kEArg, "wf_sum and w_sum go together");
    need_device();
    int b[4];
    if (box)
      for (int q = 0; q < 4; ++q) b[q] = box[q];
    octf::view_tsdf(depth, width, height, cam, origin, voxel, n,
                    box ? b : nullptr, delta, eta, f, w, wf_sum, w_sum,
                    S(stream));
  });
}

int octf_build_octree_box(const void* f, int f_dtype, const uint8_t* w,
                          int d_box, int level0, int d_max, double tau,
                          void* value, int dtype, float* weight,
                          int32_t* child, int64_t cap, int64_t root_rank,
                          int32_t root_slot, int propagate, int64_t* nsplit,
                          double* root_stats, void* stream) {
  return guard([&] {
    check_dtype(f_dtype);
    check_dtype(dtype);
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH || d_box < 0 || level0 < 0 ||
        level0 + d_box != d_max)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (w && !weight) throw octf::Error(octf::kEArg, "weighted build needs weight");
    if (!f || !value || !child || !nsplit || !root_stats)
      throw octf::Error(octf::kEArg, "null argument");
    need_device();
    int64_t total = 0;
    for (int l = 0; l <= d_box; ++l) total += (int64_t)1 << (3 * l);
    octf::DevBuf<double> mn, mx, mean, wm, wf, pl;
    octf::DevBuf<uint8_t> wmn, wmx;
    mn.ensure(total);
    mx.ensure(total);
    mean.ensure(total);
    if (w) {
      wm.ensure(total);
      wf.ensure(total);
      pl.ensure(total);
      wmn.ensure(total);
      wmx.ensure(total);
    }
    octf::pyramids(f, f_dtype, w, d_box, mn.p, mx.p, mean.p, wmn.p, wmx.p,
                   wm.p, wf.p, pl.p, S(stream));
    // the box root's pyramid statistics, for the enclosing levels
    double st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint8_t wb[2] = {0, 0};
    OCTF_CUDA(cudaMemcpyAsync(&st[0], mn.p, 8, cudaMemcpyDeviceToHost, S(stream)));
    OCTF_CUDA(cudaMemcpyAsync(&st[1], mx.p, 8, cudaMemcpyDeviceToHost, S(stream)));
    OCTF_CUDA(cudaMemcpyAsync(&st[2], mean.p, 8, cudaMemcpyDeviceToHost, S(stream)));
    if (w) {
      OCTF_CUDA(cudaMemcpyAsync(&wb[0], wmn.p, 1, cudaMemcpyDeviceToHost, S(stream)));
      OCTF_CUDA(cudaMemcpyAsync(&wb[1], wmx.p, 1, cudaMemcpyDeviceToHost, S(stream)));
      OCTF_CUDA(cudaMemcpyAsync(&st[5], wm.p, 8, cudaMemcpyDeviceToHost, S(stream)));
      OCTF_CUDA(cudaMemcpyAsync(&st[6], wf.p, 8, cudaMemcpyDeviceToHost, S(stream)));
      OCTF_CUDA(cudaMemcpyAsync(&st[7], pl.p, 8, cudaMemcpyDeviceToHost, S(stream)));
    }
    OCTF_CUDA(cudaStreamSynchronize(S(stream)));
    st[3] = wb[0];
    st[4] = wb[1];
    for (int q = 0; q < 8; ++q) root_stats[q] = st[q];
    octf::BuildIn in{mean.p, mn.p, mx.p, nullptr, w != nullptr, wmn.p, wmx.p,
                     wm.p, tau, d_box, cap};
    in.level0 = level0;
    in.d_glob = d_max;
    in.root_rank = root_rank;
    in.root_slot = root_slot;
    in.nsplit_out = nsplit;
    octf::build_tree(in, value, dtype, w ? weight : nullptr, child, nullptr,
                     propagate != 0, S(stream));
  });
}

int octf_initial_field(const double* wf_sum, const double* w_sum, double gamma,
                       int64_t n, double* u, void* stream) {
  return guard([&] {
    need_device();
    octf::initial_field(wf_sum, w_sum, gamma, n, u, S(stream));
  });
}

int octf_trace_blob(const double* cam, int width, int height,
                    const double* centre, double radius, double amp,
                    double base_freq, const double* const* lattices,
                    const int32_t* lat_n, int n_oct, double lipschitz,
                    double t_max, int steps, double eps, double* z,
                    void* stream) {
  return guard([&] {
    if (!cam || !centre || !z || (n_oct > 0 && (!lattices || !lat_n)))
      throw octf::Error(octf::kEArg, "null argument");
    if (width < 1 || height < 1 || steps < 0 || !(lipschitz > 0.0))
      throw octf::Error(octf::kEArg, "bad image size, steps or lipschitz");
    need_device();
    int n[octf::kMaxOctaves] = {};
    for (int o = 0; o < n_oct && o < octf::kMaxOctaves; ++o) n[o] = lat_n[o];
    octf::trace_blob(cam, width, height, centre, radius, amp, base_freq,
                     lattices, n, n_oct, lipschitz, t_max, steps, eps, z,
                     S(stream));
  });
}

int octf_trace_room(const double* cam, int width, int height,
                    const double* objects, int n_box, int n_sph, double size,
                    double lipschitz, double t_max, int steps, double eps,
                    double* z, void* stream) {
  return guard([&] {
    if (!cam || !z || (!objects && n_box + n_sph > 0))
      throw octf::Error(octf::kEArg, "null argument");
    if (width < 1 || height < 1 || steps < 0 || !(lipschitz > 0.0))
      throw octf::Error(octf::kEArg, "bad image size, steps or lipschitz");
    need_device();
    octf::trace_room(cam, width, height, objects, n_box, n_sph, size,
                     lipschitz, t_max, steps, eps, z, S(stream));
  });
}

int octf_nearest_vertex(const double* a, int64_t na, const double* b,
                        int64_t nb, double* dist, void* stream) {
  return guard([&] {
    if (na < 1 || nb < 1)
      throw octf::Error(octf::kEArg, "cannot compare empty meshes");
    if (!a || !b || !dist) throw octf::Error(octf::kEArg, "null argument");
    need_device();
    octf::nearest_vertex(a, na, b, nb, dist, S(stream));
  });
}

int octf_locate(const int32_t* child, int d_max, int level,
                const int32_t* cells, int64_t n, int32_t* node,
                int32_t* node_level, void* stream) {
  return guard([&] {
    if (d_max < 0 || d_max > OCTF_MAX_DEPTH)
      throw octf::Error(octf::kEDepth, "tree depth out of range");
    if (level < 0 || level > d_max)
      throw octf::Error(octf::kEArg, "level outside [0, d_max]");
    if (n < 0 || (n > 0 && (!child || !cells || !node || !node_level)))
      throw octf::Error(octf::kEArg, "null argument");
    need_device();
    octf::locate(child, level, cells, n, node, node_level, S(stream));
  });
}

}  // extern "C"
