/*
 * octfuse_b200 -- C ABI of the B200 (sm_100a) octree range-fusion hot path.
 *
 * This is the drop-in boundary for the reference's native kernel module
 * (/root/reference/pkg/src/octfuse/_kernels.pyx, selected through
 * _backend.get(), _backend.py:24-26).  Each entry point below names the
 * reference routine it replaces.  Conventions:
 *
 *  - Node pools keep the reference layout (octree.py:49-71): node 0 = root,
 *    children = 8 contiguous slots at child[n] (-1 for a leaf), blocks start
 *    at slots b with b % 8 == 1, state = {slots used, free-list head, live
 *    nodes}.  Pool arrays (value, snap, child, joined, weight, grids,
 *    pyramids, jlog) are DEVICE pointers; `state`, `out3`, `offs`, `cam`,
 *    `origin` and the per-view pointer tables are HOST pointers (the
 *    tables hold device pointers).
 *  - dtype selects the value pool type: OCTF_F64 (parity mode, bit-exact
 *    with the reference) or OCTF_F32 (throughput mode).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls that
 *    return host values synchronise that stream.
 *  - Return value: OCTF_OK or an error code mirroring the reference's
 *    exceptions (_kernels.pyx:26-27 ValueError, :84-87 MemoryError,
 *    :454-455 RuntimeError); octf_last_error() has the message.
 *  - There is no CPU fallback: without a CUDA device every call fails with
 *    OCTF_ECUDA.
 */
#ifndef OCTFUSE_B200_H
#define OCTFUSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCTF_OK 0
#define OCTF_EDEPTH 1 /* ValueError("tree depth out of range")          */
#define OCTF_ENOMEM 2 /* MemoryError                                     */
#define OCTF_EPOOL 3  /* RuntimeError("node pool capacity exhausted")    */
#define OCTF_EARG 4   /* ValueError (bad argument)                       */
#define OCTF_ECUDA 5  /* RuntimeError (CUDA failure / no device)         */

#define OCTF_F64 0
#define OCTF_F32 1

#define OCTF_MAX_DEPTH 19

typedef struct octf_ctx octf_ctx;
typedef struct octf_mesh octf_mesh;

/* message of the last failed call on this thread */
const char *octf_last_error(void);
/* ABI version (major * 100 + minor) */
int octf_version(void);
/* host-only consistency checks of the index helpers (no GPU needed):
 * returns 0 when every check passes */
int octf_selftest(void);

/* Solver context: device structures derived from one pool (level lists,
 * leaf blocks, stencil neighbour tables, gathered per-leaf view samples,
 * free-list mirror).  The reference keeps none (it re-descends from the
 * root on every lookup, _kernels.pyx:193-202).  Call octf_ctx_invalidate
 * after modifying a pool or view tree outside this library. */
int octf_ctx_create(octf_ctx **out);
int octf_ctx_destroy(octf_ctx *ctx);
int octf_ctx_invalidate(octf_ctx *ctx);
/* out[0..11] = leaf blocks, leaves, live blocks, free blocks, mask-format
 * samples (0/1), sample stride, views, valid, leaf tiles, ELL layout (0/1),
 * every leaf has every sample (0/1; kernels then read no mask), packed
 * sample positions in use (0/1, OCTF_CTX_PACKED) (int64[12]) */
int octf_ctx_info(octf_ctx *ctx, int64_t *out);

/* Context options.  By default more than 64 views use the ELL sample
 * layout -- per 256-leaf tile only as many rows as its most-observed leaf
 * has observed views, each leaf's observed samples in view order (the
 * zero-weight views the reference skips, _kernels.pyx:244-252, are not
 * stored).  OCTF_CTX_DENSE keeps the dense [leaf][view] layout at any view
 * count; OCTF_CTX_ELL uses ELL from 33 views. */
#define OCTF_CTX_DENSE 1
#define OCTF_CTX_ELL 2
/* OCTF_CTX_SORTED: each leaf's samples are sorted once by (f, view index)
 * when gathered, absent ones last as +inf -- the layout the solver="pd"
 * kernel selects its generalised-median prox on.  With OCTF_CTX_DENSE: 4, 8,
 * 16, 32 or 64 views; without it more than 64 views -- with OCTF_CTX_ELL
 * any number of views -- use the per-tile store (each leaf's observed rows
 * sorted). */
#define OCTF_CTX_SORTED 4
/* OCTF_CTX_DEFER: octf_ctx_prepare / set_samples build the structure but
 * gather no samples; the next octf_ctx_select gathers its subset only (and
 * clears the flag) -- a shard never holds the whole tree's samples. */
#define OCTF_CTX_DEFER 8
/* OCTF_CTX_PACKED (frozen trees only): a leaf's samples sit at its rank
 * among the leaves of its 256-slot tile, so the kernels stream only the
 * tile's leaves' samples, not the rows of the inner siblings a leaf block
 * spans.  The context then never patches its leaf list in place: a pass
 * that restructures gets a full rebuild. */
#define OCTF_CTX_PACKED 16
int octf_ctx_set_options(octf_ctx *ctx, int flags);

/* Live profiling: enable != 0 brackets the leaf-update and energy kernels
 * with CUDA events on their launch stream.  out[0..4] (optional) receives
 * {leaf-update ms, leaf-update launches, energy ms, energy launches, kernel
 * launches} accumulated since the previous call, which resets them. */
int octf_ctx_profile(octf_ctx *ctx, int enable, double *out);

/* Host-side phase times since the last octf_ctx_profile call (which resets
 * them; recorded only while profiling is enabled): out[0..4] = {context
 * rebuild ms (incl. gathers), rebuilds, sample gather ms, gathers,
 * restructuring ms after the leaf kernel (events, cascade, joins, sweep)},
 * out[5..18] = phases (only with env OCTF_PHASES=1: each mark synchronises
 * the stream): rebuild -- level walk, list diff, tables, ELL grow, ELL
 * update, new-leaf gather, ELL tile moves, full list rebuild, full gather,
 * rest -- and restructuring -- split cascade, split allocation, joins,
 * sweep.  out holds 19 doubles. */
int octf_ctx_phases(octf_ctx *ctx, double *out);

/* _kernels.pyx:384-461 iterate_pass -- one Jacobi descent pass with the
 * in-pass split cascade, join cascade and sweep.  snapshot=1 reproduces the
 * reference's own first step (copy uval into usnap, :390-393); snapshot=0
 * lets a caller that ping-pongs two buffers skip that copy (usnap must then
 * hold the pass-start values; uval's old contents are not read).
 * out3 = {splits, joins, join-log rows}.  jlog: jcap rows of 12 doubles. */
int octf_iterate_pass(octf_ctx *ctx, int dtype, void *usnap, void *uval,
                      int32_t *uchild, uint8_t *ujoined, int64_t *ustate,
                      int64_t cap, int nviews, const float *const *vvals,
                      const float *const *vws, const int32_t *const *vchilds,
                      int d_max, double lam, double eps, double gamma,
                      double xi, double tau_s, double tau_j, int clamp,
                      int reverse, int snapshot, double *jlog, int64_t jcap,
                      int64_t *out3, void *stream);

/* One pass of the reference's fuse loop (fusion.py:221-228) in one call:
 * iterate_pass in ping-pong mode (snapshot=0) + propagate of uval.  The
 * energy of the incoming (snapshot) state -- i.e. the previous pass's
 * post-propagate energy, _kernels.pyx:536-578 -- is evaluated by the same
 * leaf kernel from the same stencil values and returned in *energy_pre. */
int octf_fuse_pass(octf_ctx *ctx, int dtype, void *usnap, void *uval,
                   int32_t *uchild, uint8_t *ujoined, int64_t *ustate,
                   int64_t cap, int nviews, const float *const *vvals,
                   const float *const *vws, const int32_t *const *vchilds,
                   int d_max, double lam, double eps, double gamma, double xi,
                   double tau_s, double tau_j, int clamp, int reverse,
                   double *jlog, int64_t jcap, int64_t *out3,
                   double *energy_pre, void *stream);

/* npasses passes of that loop (fusion.py:204-229) without returning to the
 * caller in between: pass k reads buffer k % 2 and writes the other, its step
 * scale is xis[k] (fusion.py:124-126); out3 = npasses x {splits, joins, live
 * nodes after the pass}, energies_pre[k] = the energy of pass k's incoming
 * state.  *done = passes completed: a pass that runs out of pool capacity
 * (OCTF_EPOOL) stops the run before any structural write, with buffer
 * (*done % 2) holding the current state, so the caller can grow the pools
 * and go on.  No join log (use octf_fuse_pass for that). */
int octf_fuse_passes(octf_ctx *ctx, int dtype, void *ubuf0, void *ubuf1,
                     int32_t *uchild, uint8_t *ujoined, int64_t *ustate,
                     int64_t cap, int nviews, const float *const *vvals,
                     const float *const *vws, const int32_t *const *vchilds,
                     int d_max, double lam, double eps, double gamma,
                     double tau_s, double tau_j, int clamp, int reverse,
                     const double *xis, int npasses, int64_t *out3,
                     double *energies_pre, int *done, void *stream);

/* npasses passes of a frozen structure (tau_s <= 0, tau_j >= 1 with clamp:
 * no split or join can happen) without any host round trip.  Buffers
 * alternate: pass k reads ubuf[k%2] and writes ubuf[(k+1)%2];
 * energies_pre[k] (host) = energy before pass k.  xis: host step sizes. */
int octf_fuse_passes_frozen(octf_ctx *ctx, int dtype, void *ubuf0, void *ubuf1,
                            const int32_t *uchild, const int64_t *ustate,
                            int64_t cap, int nviews, const float *const *vvals,
                            const float *const *vws,
                            const int32_t *const *vchilds, int d_max,
                            double lam, double eps, double gamma,
                            double tau_s, double tau_j, int clamp,
                            const double *xis, int npasses,
                            double *energies_pre, int device_energies,
                            void *stream);

/* Zero-isosurface readout (reference
 * octfuse/mesh.py:63-125 extract_zero_surface / marching_cubes): marching
 * cubes over the dense cell-centred grid `values` (device f64, n^3, x-major)
 * with the observed mask `mask` (device u8 n^3, or NULL = all observed).  A
 * cube emits its case's triangles only if all eight corners are observed;
 * vertices are the grid edges' zero crossings, t = v0 / (v0 - v1), sorted by
 * edge key ((axis*n + x)*n + y)*n + z; faces index them in cube order then
 * table order -- the reference's vertex and face arrays bit for bit.  The
 * case tables (tri_table int8[256][32], tri_count int8[256], edge_axis
 * int8[12], edge_offset int8[12][3]; host) come from the caller
 * (paper_1608_07411_b200/mesh.py generates them).  world != 0 maps vertices
 * to origin + (p + 1/2) * voxel_size.  The result lives on the device until
 * octf_mesh_copy (device destinations) / octf_mesh_free. */
int octf_marching_cubes(const double *values, const uint8_t *mask, int n,
                        const int8_t *tri_table, const int8_t *tri_count,
                        const int8_t *edge_axis, const int8_t *edge_offset,
                        const double *origin, double voxel_size, int world,
                        octf_mesh **out, int64_t *nverts, int64_t *nfaces,
                        void *stream);
/* Mesh readout from the leaf store: the mesh of
 * octf_marching_cubes(densify(value), seen) (mesh.py:63-125,
 * octree.py:327-342) -- same vertices, faces and order -- without the dense
 * (2^d)^3 grid: only 8^3-cube bricks whose corner cells meet leaves of both
 * signs are evaluated.  seen_value / seen_child (optional, dtype
 * seen_dtype): an observed-mask tree over the same domain, node value != 0 =
 * observed (NULL: every cell observed).  Tables, origin, voxel_size, world
 * and the result as octf_marching_cubes.  slab0 / slab1 (-1: all) restrict
 * the readout to the cubes with x in [8 slab0, 8 slab1) -- a mesh too large
 * for one call is read slab by slab (vertices on a slab's end plane then
 * appear in both).  ctx may be NULL. */
int octf_marching_cubes_tree(octf_ctx *ctx, int dtype, const void *value,
                             const int32_t *child, const int64_t *state,
                             int64_t cap, int d_max, int seen_dtype,
                             const void *seen_value, const int32_t *seen_child,
                             const int8_t *tri_table, const int8_t *tri_count,
                             const int8_t *edge_axis, const int8_t *edge_offset,
                             const double *origin, double voxel_size,
                             int world, int64_t slab0, int64_t slab1,
                             octf_mesh **out, int64_t *nverts,
                             int64_t *nfaces, void *stream);
int octf_mesh_copy(octf_mesh *m, double *verts, int32_t *faces, void *stream);
int octf_mesh_free(octf_mesh *m);

/* Sharded overlap: one frozen descent pass split into
 * leaf-tile ranges, so a rank updates its interior tiles while the halo of
 * the previous pass is in flight and its boundary tiles afterwards.
 * octf_pass_tiles runs the leaf kernel (snapshot usnap -> uval, step xi) on
 * tiles [tile0, tile0+ntiles) of the context's leaf-block list (256 leaves
 * per tile; octf_ctx_info out[8] = tiles), energy partials per tile;
 * octf_pass_finish propagates uval and sums the pass's energy partials into
 * *dev_energy (a device double).  Same arithmetic as octf_fuse_passes_frozen. */
int octf_pass_tiles(octf_ctx *ctx, int dtype, const void *usnap, void *uval,
                    const int32_t *uchild, const int64_t *ustate, int64_t cap,
                    int nviews, const float *const *vvals,
                    const float *const *vws, const int32_t *const *vchilds,
                    int d_max, double lam, double eps, double gamma, double xi,
                    int clamp, int tile0, int ntiles, void *stream);
int octf_pass_finish(octf_ctx *ctx, int dtype, void *uval,
                     const int32_t *uchild, double *dev_energy, void *stream);

/* solver="pd" (north_star; no reference counterpart,
 * definition in oracle/pd_oracle.c): npasses TV-L1 primal-dual passes on a
 * frozen tree.  set_a / set_b: host tables of 5 device pools {u, ubar, px,
 * py, pz}; pass k reads set_a (k even) or set_b (k odd) and writes the
 * other, then propagates all five.  energies_pre (host): E(u) before each
 * pass (exact TV + L1 data, same normalisation as the descent's data term).
 * 4, 8, 16 or 32 views. */
int octf_pd_passes(octf_ctx *ctx, int dtype, void *const *set_a,
                   void *const *set_b, const int32_t *uchild,
                   const int64_t *ustate, int64_t cap, int nviews,
                   const float *const *vvals, const float *const *vws,
                   const int32_t *const *vchilds, int d_max, double lam,
                   double tau, double sigma, double gamma, int clamp,
                   int npasses, double *energies_pre, int device_energies,
                   void *stream);

/* solver="pd" split/join on the current set {u, ubar, px, py, pz} after a
 * pass (north_star item (d); definition oracle/pd_oracle.c
 * orc_pd_restructure -- the reference has no primal-dual mode): leaves with
 * |u| < tau_split and level < d_max get eight children carrying their u,
 * ubar, p; inner nodes whose eight children are leaves past tau_join with one
 * sign become leaves (their propagated means stay).  Splits claim blocks in
 * depth-first order from the free list then the bump pointer, joined blocks
 * are freed in post-order, as the descent pass (_kernels.pyx:277-381).
 * ustate is updated; out2 = {splits, joins}.  The context must hold the
 * structure of the last pass (octf_pd_passes); OCTF_EPOOL leaves the pool
 * untouched. */
int octf_pd_restructure(octf_ctx *ctx, int dtype, void *const *set,
                        int32_t *uchild, int64_t *ustate, int64_t cap,
                        int d_max, double tau_split, double tau_join,
                        int64_t *out2, void *stream);

/* Build the context's structures for a pool (and views) up front. */
int octf_ctx_prepare(octf_ctx *ctx, const int32_t *uchild,
                     const int64_t *ustate, int64_t cap, int d_max, int nviews,
                     const float *const *vvals, const float *const *vws,
                     const int32_t *const *vchilds, void *stream);

/* Per-leaf samples supplied directly instead of view trees (BASELINE
 * config 5: "N fp32 TSDF samples per leaf"): f_slot / w_slot are device
 * [nviews][cap] arrays indexed by node slot (w_slot NULL = every sample has
 * weight 1).  Frozen trees only; view-taking calls then pass nviews = 0. */
int octf_ctx_set_samples(octf_ctx *ctx, const float *f_slot,
                         const float *w_slot, int nviews, int64_t cap,
                         void *stream);

/* Sharding: restrict the context's leaf-block list to the
 * blocks `sel` (host int32 indices into the current list) with per-block
 * owned-leaf masks (host u8, bit c = sibling c is updated by this rank);
 * samples are regathered for the subset.  Frozen structures only. */
int octf_ctx_select(octf_ctx *ctx, const int32_t *sel, const uint8_t *masks,
                    int64_t nsel, void *stream);

/* Propagate only levels hi-1 .. lo (the replicated top of a sharded tree). */
/* Halo staging for the sharded solver (shard.py HaloExchange; SURVEY.md
 * §8(e) -- no reference counterpart, the reference is single-process):
 * pack (unpack = 0) copies fields[k][idx[j]] to buf[k*n + j] for k < nfields
 * (1..5: u, or u, ubar, px, py, pz in pd mode), unpack (1) the reverse.  All
 * pointers are device pointers; enqueued on `stream`. */
int octf_halo_pack(int dtype, void *const *fields, int nfields,
                   const int32_t *idx, int64_t n, void *buf, int unpack,
                   void *stream);
int octf_propagate_levels(octf_ctx *ctx, int dtype, void *value,
                          const int32_t *child, int lo, int hi, void *stream);

/* _kernels.pyx:80-113 propagate -- inner value = (sequential sum of the 8
 * children)/8, bottom-up.  ctx may be NULL (a temporary one is built). */
int octf_propagate(octf_ctx *ctx, int dtype, void *value,
                   const int32_t *child, const int64_t *state, int64_t cap,
                   int d_max, void *stream);

/* _kernels.pyx:536-578 tree_energy -- leaf-summed energy.  The per-leaf
 * terms equal the reference's bit for bit in OCTF_F64; the sum is a
 * deterministic tree reduction.  terms (optional, device, cap doubles)
 * receives every leaf's term at its slot. */
int octf_tree_energy(octf_ctx *ctx, int dtype, const void *uval,
                     const int32_t *uchild, const int64_t *ustate, int64_t cap,
                     int nviews, const float *const *vvals,
                     const float *const *vws, const int32_t *const *vchilds,
                     int d_max, double lam, double eps, double gamma,
                     double *out, double *terms, void *stream);

/* The reference's canonical node order on the device (octree.py:168-181
 * leaves(), :413-431 serialize(): depth-first pre-order, children in index
 * order): every live node -- or every leaf, leaves_only != 0 -- as its slot
 * (slots, device, int32) and preorder key (keys, device, optional:
 * Morton key of its first finest-level cell << 5 | level), sorted by a
 * radix sort of the keys.  slots / keys must hold state[2] entries;
 * *count (host) receives the number written.  ctx may be NULL. */
int octf_node_order(octf_ctx *ctx, const int32_t *child, const int64_t *state,
                    int64_t cap, int d_max, int leaves_only, int32_t *slots,
                    uint64_t *keys, int64_t *count, void *stream);

/* _kernels.pyx:116-158 densify -- leaves to a dense (2^d)^3 f64 grid */
int octf_densify(int dtype, const void *value, const int32_t *child,
                 int d_max, double *out, void *stream);

/* _kernels.pyx:21-77 build_tree -- spread-rule build from flattened
 * pyramids (offs: host level offsets; NULL = sum_{l<L} 8^l).  Produces the
 * reference's exact pool layout (depth-first, child 7 expanded first). */
int octf_build_tree(const double *meanf, const double *minf,
                    const double *maxf, const int64_t *offs, int has_w,
                    const uint8_t *wminf, const uint8_t *wmaxf,
                    const double *wmeanf, double tau, void *value, int dtype,
                    float *weight, int32_t *child, int64_t *state, int64_t cap,
                    int d_max, void *stream);

/* octree.py:193-225 reduce_pyramid/flatten_pyramid on device (numpy's
 * summation order).  f: dense (2^d)^3 grid, f_dtype OCTF_F32/OCTF_F64;
 * w (optional) u8 weights.  Outputs are flattened, root first, sized
 * sum_{l<=d} 8^l.  wm_tmp..pl_tmp: scratch of the same size when w given. */
int octf_pyramids(const void *f, int f_dtype, const uint8_t *w, int d_max,
                  double *minf, double *maxf, double *meanf, uint8_t *wminf,
                  uint8_t *wmaxf, double *wmeanf, double *wf_tmp,
                  double *pl_tmp, void *stream);

/* octree.py:243-306 build_octree -- pyramids + build (+ propagate_means
 * when unweighted) in one call; scratch is allocated internally. */
int octf_build_octree(const void *f, int f_dtype, const uint8_t *w, int d_max,
                      double tau, void *value, int dtype, float *weight,
                      int32_t *child, int64_t *state, int64_t cap,
                      void *stream);

/* tsdf.py:87-120 build_view_tsdf -- per-voxel projective TSDF in f64 with
 * numpy's operand order.  cam = {fx, fy, cx, cy, R (3x3 camera-to-world,
 * row-major), t (camera centre)}; origin = volume minimum corner.  When
 * wf_sum/w_sum are given the view is also accumulated into them
 * (cli.py:148-149). */
int octf_view_tsdf(const float *depth, int width, int height,
                   const double *cam, const double *origin, double voxel,
                   int n, double delta, double eta, float *f, uint8_t *w,
                   double *wf_sum, double *w_sum, void *stream);

/* The same TSDF for the n_b^3 voxels of a box of the n^3 grid, box =
 * {i0, j0, k0, n_b} (host): global voxel (i0 + i, j0 + j, k0 + k) -- the
 * same arithmetic -- at box-local index (i*n_b + j)*n_b + k of f, w and the
 * optional accumulators. */
int octf_view_tsdf_box(const float *depth, int width, int height,
                       const double *cam, const double *origin, double voxel,
                       int n, const int32_t *box, double delta, double eta,
                       float *f, uint8_t *w, double *wf_sum, double *w_sum,
                       void *stream);

/* octree.py:243-306 build_octree for a BOX subtree of a tree of depth
 * d_max: f (and w) the (2^d_box)^3 grid of the box, whose root is the node
 * at global level level0 = d_max - d_box and pool slot root_slot; split
 * decisions use global levels, and the box's splitting nodes continue the
 * enclosing tree's depth-first ranks from root_rank (rank of the box root if
 * it splits), so the subtree lands at the slots the whole-tree build gives
 * it.  *nsplit (host) = splitting nodes of the box; root_stats (host,
 * double[8]) = the box root's pyramid entries {min f, max f, value mean,
 * min w, max w, mean w, mean f*w, mean f} for the enclosing levels.
 * propagate != 0: unweighted build's child means inside the box.
 * OCTF_EPOOL if the pool is too small (nothing written past cap). */
int octf_build_octree_box(const void *f, int f_dtype, const uint8_t *w,
                          int d_box, int level0, int d_max, double tau,
                          void *value, int dtype, float *weight,
                          int32_t *child, int64_t cap, int64_t root_rank,
                          int32_t root_slot, int propagate, int64_t *nsplit,
                          double *root_stats, void *stream);

/* fusion.py:149-155 initial_field */
int octf_initial_field(const double *wf_sum, const double *w_sum, double gamma,
                       int64_t n, double *u, void *stream);

/* Scene generators on the device (the reference
 * renders its spheres analytically, synth.py:80-109): camera-frame depth z
 * of every pixel ray's first hit, 0 on a miss, by sphere tracing (steps
 * sd / lipschitz until sd < eps, then 40 bisections) in f64 -- the array
 * program of the package's scenes.py, operation for operation.  cam as in
 * octf_view_tsdf (host); z = height x width doubles (device).
 * Blob: sd(p) = |p - centre| - (radius + amp * noise(p)), noise = n_oct
 * octaves of lattice value noise (lattices[o] = n_o^3 doubles on the
 * device, frequency base_freq * 2^o, amplitude 2^-o). */
int octf_trace_blob(const double *cam, int width, int height,
                    const double *centre, double radius, double amp,
                    double base_freq, const double *const *lattices,
                    const int32_t *lat_n, int n_oct, double lipschitz,
                    double t_max, int steps, double eps, double *z,
                    void *stream);

/* Room: union of n_box axis-aligned boxes {centre, half extents}, n_sph
 * spheres {centre, radius} (objects = the boxes then the spheres, device)
 * and the six walls of the size^3 cube seen from inside. */
int octf_trace_room(const double *cam, int width, int height,
                    const double *objects, int n_box, int n_sph, double size,
                    double lipschitz, double t_max, int steps, double eps,
                    double *z, void *stream);

/* mesh.py:162-167 vertex_diff -- dist[i] = Euclidean distance from vertex
 * a[i] to the nearest vertex of b (what the reference gets from scipy's k-d
 * tree, bit for bit); a = na x 3, b = nb x 3 doubles, dist = na doubles, all
 * on the device.  Call it both ways for the symmetric statistics. */
int octf_nearest_vertex(const double *a, int64_t na, const double *b,
                        int64_t nb, double *dist, void *stream);

/* octree.py:148-166 locate, batched: for each of n cells (x, y, z) at
 * `level` (int32 triples, device) the deepest node on the root path of the
 * cell and that node's level (device outputs). */
int octf_locate(const int32_t *child, int d_max, int level,
                const int32_t *cells, int64_t n, int32_t *node,
                int32_t *node_level, void *stream);

#ifdef __cplusplus
}
#endif
#endif
