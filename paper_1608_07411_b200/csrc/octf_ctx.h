// Host-side solver context: device acceleration structures derived from a
// reference-layout node pool, kept across passes so a pass only streams the
// leaves.  Everything here is an implementation detail behind the C ABI in
// include/octfuse_b200.h.
#pragma once
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "octf_common.cuh"

// extracted zero surface (octf_marching_cubes), device arrays
struct octf_mesh {
  int64_t nv = 0, nf = 0;
  double* verts = nullptr;   // nv x 3
  int32_t* faces = nullptr;  // nf x 3
  ~octf_mesh() {
    if (verts) cudaFree(verts);
    if (faces) cudaFree(faces);
  }
};

namespace octf {

// error kinds mirror the reference's three exceptions (_kernels.pyx:26-27,
// :84-87, :454-455) plus argument and CUDA failures
enum Err : int {
  kOk = 0,
  kEDepth = 1,  // ValueError("tree depth out of range")
  kENoMem = 2,  // MemoryError
  kEPool = 3,   // RuntimeError("node pool capacity exhausted")
  kEArg = 4,    // ValueError (bad argument)
  kECuda = 5,   // RuntimeError (CUDA failure)
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check_cuda(cudaError_t e, const char* what);
struct Ctx;
// phase stopwatch of context rebuilds (no-ops unless timing is on)
void ph_start(Ctx& c, cudaStream_t st);
void ph_mark(Ctx& c, int phase, cudaStream_t st);
#define OCTF_CUDA(call) ::octf::check_cuda((call), #call)

// owning device buffer (grow-only)
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void swap(DevBuf& o) {
    T* tp = p;
    p = o.p;
    o.p = tp;
    size_t tn = n;
    n = o.n;
    o.n = tn;
  }
  // Allocations come from the device's default stream-ordered pool on the
  // legacy stream (kept cached: see pool_keep() in ctx.cu), so contexts
  // created per fuse() call do not pay cudaMalloc/cudaFree each time.
  // (a reallocation is rare: the device is synchronised first, so no
  // kernel on any stream still uses the old block and the new one is ready
  // for every stream)
  void release() {
    if (p) {
      cudaDeviceSynchronize();
      cudaFreeAsync(p, cudaStreamLegacy);
    }
    p = nullptr;
    n = 0;
  }
  // grow keeping the first `keep` elements (stream-ordered copy)
  T* grow_keep(size_t count, size_t keep, cudaStream_t st) {
    if (count <= n && p) return p;
    T* q = nullptr;
    size_t c = count > 2 * n ? count : 2 * n;
    if (cudaMallocAsync((void**)&q, c * sizeof(T), cudaStreamLegacy) !=
            cudaSuccess ||
        cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess) {
      cudaGetLastError();
      throw Error(kENoMem, "device allocation failed");
    }
    if (p && keep)
      check_cuda(cudaMemcpyAsync(q, p, keep * sizeof(T),
                                 cudaMemcpyDeviceToDevice, st),
                 "grow_keep");
    if (p) {
      cudaDeviceSynchronize();
      cudaFreeAsync(p, cudaStreamLegacy);
    }
    p = q;
    n = c;
    return p;
  }
  T* ensure(size_t count) {
    if (count <= n && p) return p;
    // a buffer that has to grow again gets 1/8 headroom, so structures that
    // creep up pass by pass (patched leaf lists) do not reallocate each time
    const size_t grown = p ? count + count / 8 : count;
    release();
    size_t c = grown ? grown : 1;
    cudaError_t e = cudaMallocAsync((void**)&p, c * sizeof(T), cudaStreamLegacy);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      throw Error(kENoMem, "device allocation of " +
                               std::to_string(c * sizeof(T)) + " bytes failed");
    }
    n = c;
    return p;
  }
};

// rebuild phases (Ctx::t_ph)
enum Phase : int {
  kPhWalk = 0,     // level walk (block lists per level)
  kPhListDiff,     // patched list: holes and appended blocks
  kPhTables,       // neighbour tables of touched entries
  kPhEllGrow,      // ELL rows for appended tiles (counts, scan, offsets)
  kPhEllUpdate,    // ELL: queue the new leaves
  kPhFresh,        // gather of the new leaves' samples
  kPhMove,         // ELL: tiles moved to bigger row ranges
  kPhFull,         // full rebuild (sorted list, tables) instead of a patch
  kPhGather,       // full sample gather
  kPhTail,         // free-list mirror, marks, rest of the rebuild
  kPhSplitCascade, // restructuring pass: split events and their cascade
  kPhSplitAlloc,   // ... pre-order keys, sort, block allocation
  kPhJoins,        // ... join candidates and updates, level by level
  kPhSweep,        // ... post-order sweep, free list, join log
  kPhCount
};

struct Ctx {
  // ---- identity of the pool / views the cached structures describe
  const int32_t* child_key = nullptr;
  int64_t cap = 0;
  int d_max = -1;
  bool valid = false;
  int64_t hstate[3] = {1, -1, 1};  // last known pool state
  std::vector<const void*> vkey;
  int nviews = 0;

  // ---- structure (rebuilt by prepare())
  DevBuf<int8_t> blevel;      // per block id: level of its nodes (-1 free)
  DevBuf<uint64_t> bcoord;    // per block id: packed parent cell
  DevBuf<int32_t> bparent;    // per block id: parent node slot
  std::vector<int64_t> lvl_off, lvl_cnt;  // per level ranges in lvl_blocks
  DevBuf<int32_t> lvl_blocks;             // live block bases, level-major
  int64_t nblocks = 0;
  bool fuse_off = false;
  bool no_morton = false;     // env OCTF_NO_MORTON=1: frozen lists by base
  bool list_morton = false;   // the leaf-block list is in Morton order  // env OCTF_NO_FUSED_PARENT=1: pd bottom level apart
  DevBuf<int32_t> lblocks;    // blocks holding >= 1 leaf, ascending base
  DevBuf<uint64_t> lkey;      // per leaf block: packed (level, parent cell)
  DevBuf<int4> lmeta;         // per leaf block: {base, px, py, pz|mask|L}
  DevBuf<int32_t> lpar;       // per leaf block: parent node slot (-1 root)
  DevBuf<int32_t> nbr;        // per leaf block: 12 neighbour refs
  int64_t nlb = 0;
  int64_t nleaves = 0;

  // ---- per-leaf samples, leaf index i*8+c over the leaf-block list
  DevBuf<float> F;            // [leaf][view], sstride floats per leaf
  DevBuf<float> W;            // [leaf][view] (general weights)
  DevBuf<uint32_t> M;         // [sample] bit v = weight of view v is 1
  bool binw = false;          // samples use the mask format
  bool allv = false;          // ... and every leaf has all of them (no mask
                              // read; set with 8/16/32 views)
  int64_t sstride = 0;        // views per leaf vector, padded to 4
  // packed store (OCTF_CTX_PACKED, frozen trees; octf_common.cuh SDesc):
  // a leaf's samples at its rank among its tile's leaves
  bool pack_opt = false;      // requested
  bool packed = false;        // in use (some block is not 8 leaves)
  SDesc sd;                   // the dense store's layout
  // ELL layout (views > 64, unless dense_only): F/W hold per tile K_t rows
  // of the leaves' observed samples (octf_common.cuh ell_idx)
  bool ell = false;
  bool dense_only = false;    // octf_ctx_set_options: keep the dense layout
  bool force_ell = false;     // ... or use ELL from 33 views (default: 65)
  bool defer_gather = false;  // OCTF_CTX_DEFER: prepare builds structure
                              // only; ctx_select gathers (shards)
  bool sorted = false;        // OCTF_CTX_SORTED: each leaf's samples sorted
                              // by (f, view) once when gathered (pd prox)
  DevBuf<int32_t> tileK;      // per tile: rows
  DevBuf<int64_t> tileOff;    // per tile: first float of its rows
  int64_t ell_tiles = 0, ell_size = 0;
  int64_t ell_waste = 0;      // rows of tiles moved to bigger ranges
  bool store_ok = false;      // F/W/M describe the current leaf-block list
  bool own_change = false;    // invalid only because our pass restructured
  bool no_regather = false;   // env OCTF_FULL_GATHER=1: always rebuild all
  // stable leaf-block list (ctx_list_update): after our own restructure the
  // list is patched in place -- blocks that lost their leaves become holes,
  // new leaf blocks are appended -- so unchanged leaves keep their list
  // position and samples; a full sorted rebuild compacts it when holes or
  // appended entries pass a quarter of the list
  DevBuf<int32_t> lpos;       // per block id: list position or -1
  int64_t lpos_n = 0;         // block ids lpos covers
  int64_t nholes = 0;
  bool list_full = false;     // list = every leaf block (not a shard subset)
  DevBuf<int32_t> app_buf;    // appended blocks scratch
  DevBuf<int32_t> vmap;       // per-level view maps (gather), chunk x cap

  // ---- or samples supplied per slot by the caller (frozen trees only)
  const float* ext_F = nullptr;  // [view][ext_cap]
  const float* ext_W = nullptr;  // [view][ext_cap] or null (all weight 1)
  int64_t ext_cap = 0;

  // ---- views (device arrays of device pointers)
  DevBuf<const float*> dv_val, dv_w;
  DevBuf<const int32_t*> dv_child;

  // ---- free list mirror: stack of free block bases, top = free-list head
  DevBuf<int32_t> free_stack;
  int64_t nfree = 0;
  bool free_ok = false;       // mirror matches the pool's free list
  int64_t nfree_head = -1;    // pool free-list head the mirror ends at

  // ---- pass scratch
  DevBuf<uint8_t> smark;      // per slot: leaf split this pass
  DevBuf<int32_t> counters;   // device counters
  DevBuf<int32_t> split_list;
  DevBuf<int32_t> join_bot;   // parent slots of bottom join candidates
  bool coop_off = false;      // env OCTF_LEVEL_JOINS=1: per-level join scans
  bool walk_coop = false;     // env OCTF_COOP_WALK=1: the level walk as one cooperative launch
  DevBuf<uint8_t> cub_tmp;
  DevBuf<uint64_t> sort_k64;  // sort scratch (persistent)
  DevBuf<int32_t> sort_k32, sort_v32;
  DevBuf<uint8_t> flags;
  DevBuf<double> partials;
  DevBuf<double> mid;       // stripe sums of the two-stage energy reduction
  DevBuf<double> dscalar;
  // restructuring scratch of the typed solver (solver_impl.cuh: split
  // events, join records) per value type, and the pd split keys: owned by
  // the context, so two contexts (or devices) never share device buffers
  std::shared_ptr<void> rs_ev[2], rs_join[2];
  DevBuf<int32_t> rs_slot, rs_idx;
  DevBuf<uint64_t> rs_key;

  // live profiling (octf_ctx_profile): CUDA events on the launch stream
  bool timing = false;
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> pev;  // per-pass pairs for batched passes
  // tile-range launches (sharded overlap): event pairs read at the next
  // octf_ctx_profile call, so timing never synchronises the pass
  std::vector<cudaEvent_t> tile_ev;
  size_t tile_ev_used = 0;
  int64_t tile_passes = 0;
  double t_leaf_ms = 0, t_energy_ms = 0;
  // host wall clock (timing on): context rebuilds, sample gathers, the
  // restructuring tail of a pass (after the leaf kernel)
  double t_prep_ms = 0, t_gather_ms = 0, t_restr_ms = 0;
  int64_t n_prep = 0, n_gather = 0, n_regather = 0;
  // finer phases of a context rebuild (timing on and OCTF_PHASES=1; each mark synchronises):
  // kPh* indices, exported by octf_ctx_phases after the five totals
  double t_ph[16] = {};
  bool phase_marks = false;  // env OCTF_PHASES=1 (the marks synchronise)
  std::chrono::steady_clock::time_point ph_t0;
  int64_t n_leaf = 0, n_energy = 0, launches = 0;

  // host pinned staging for small readbacks
  int32_t* h_counters = nullptr;
  double* h_scalar = nullptr;

  Ctx();
  ~Ctx();
};

// structure rebuild from the pool (BFS over levels, leaf-block list,
// neighbour tables); views gather when given.  Syncs the stream.
void ctx_prepare(Ctx& c, const int32_t* child, int64_t cap,
                 const int64_t* state, int d_max, cudaStream_t st);
// halo staging of shard.HaloExchange: buf[k*n + j] <-> fields[k][idx[j]]
// (pack: fields -> buf; unpack: buf -> fields), k < nf <= kMaxHaloFields
constexpr int kMaxHaloFields = 5;
template <typename T>
void halo_pack(T* const* fields, int nf, const int32_t* idx, int64_t n,
               T* buf, bool unpack, cudaStream_t st);

// sort the sample vectors of store slots list[0 .. *nlist) (list null: all
// slots) -- solver="pd" (sample_sort.cuh); no-op unless c.sorted
void ctx_sort_samples(Ctx& c, const int32_t* list, const int32_t* nlist,
                      cudaStream_t st);
void ctx_set_views(Ctx& c, int nviews, const float* const* vval,
                   const float* const* vw, const int32_t* const* vchild,
                   cudaStream_t st);
void ctx_gather(Ctx& c, cudaStream_t st);
void pool_keep();  // the default memory pool keeps freed blocks (per device)
int64_t ctx_node_order(Ctx& c, const int32_t* child, int d_max,
                       bool leaves_only, int32_t* out_slots,
                       uint64_t* out_keys, cudaStream_t st);
void ctx_gather_ell(Ctx& c, cudaStream_t st);
void ctx_list_full(Ctx& c, const int32_t* child, int64_t total, int64_t nbid,
                   int d_max, cudaStream_t st);
bool ctx_list_update(Ctx& c, const int32_t* child, int64_t total, int64_t nbid,
                     cudaStream_t st);  // false: rebuild with ctx_list_full
void ctx_set_samples(Ctx& c, const float* F, const float* W, int nviews,
                     int64_t cap, cudaStream_t st);
void ctx_free_stack(Ctx& c, const int32_t* child, const int64_t* state,
                    cudaStream_t st);
ViewSet ctx_views(const Ctx& c);

// cub wrappers (ctx.cu)
void sort_u64_i32(Ctx& c, uint64_t* keys, int32_t* vals, int64_t n,
                  cudaStream_t st);
void sort_i32(Ctx& c, int32_t* keys, int64_t n, cudaStream_t st);

struct IterArgs {
  const void* usnap;  // pass-start values (+ new children's snapshots)
  void* uval;         // post-pass values
  int32_t* child;
  uint8_t* joined;
  int64_t* state;     // host int64[3]
  int64_t cap;
  PassParams prm;
  double* jlog;       // device rows of 12 doubles (may be null)
  int64_t jcap;
  int snapshot;       // 1: copy uval -> usnap first (_kernels.pyx:390-393)
  int want_energy = 0;      // also evaluate the energy of the snapshot state
  double energy_pre = 0.0;  // ... returned here
  int64_t out3[3];    // splits, joins, log rows
};

// K passes on a frozen structure (no split or join can occur) with no host
// round trip: buffers alternate, energies_pre[k] = energy before pass k
struct FrozenArgs {
  void* ubuf[2];
  const int32_t* child;
  const int64_t* state;
  int64_t cap;
  PassParams prm;     // xi is taken from xis[]
  const double* xis;  // host, npasses
  int npasses;
  double* energies_pre;  // host (or device with dev_energies), npasses
  bool dev_energies = false;
};

// per precision entry points (solver_f64.cu / solver_f32.cu)
void iterate_pass_f64(Ctx& c, IterArgs& a, cudaStream_t st);
void iterate_pass_f32(Ctx& c, IterArgs& a, cudaStream_t st);
void propagate_ctx_f64(Ctx& c, double* value, const int32_t* child,
                       cudaStream_t st);
void propagate_ctx_f32(Ctx& c, float* value, const int32_t* child,
                       cudaStream_t st);
double energy_f64(Ctx& c, const double* u, const int32_t* child,
                  const PassParams& p, double* terms, cudaStream_t st);
double energy_f32(Ctx& c, const float* u, const int32_t* child,
                  const PassParams& p, double* terms, cudaStream_t st);
// solver="pd": TV-L1 primal-dual passes (frozen tree), 5 arrays per set
// {u, ubar, px, py, pz}; pass k reads in (k even) / out (k odd)
struct PdHostArgs {
  void* in[5];
  void* out[5];
  const int32_t* child;
  const int64_t* state;
  int64_t cap;
  int d_max;
  double lam, tau, sigma, gamma;
  int clamp;
  int npasses;
  double* energies;  // npasses: energy of u before each pass (host, or
  bool dev_energies = false;  // a device array: then fully asynchronous)
};
// sharded overlap: one frozen pass split into tile ranges (interior tiles
// while the halo is in flight, then boundary tiles), then the finish
struct TileArgs {
  const void* usnap;
  void* uval;
  const int32_t* child;
  const int64_t* state;
  int64_t cap;
  PassParams prm;
  int tile0, ntiles;
};
void pass_tiles_f64(Ctx& c, TileArgs& a, cudaStream_t st);
void pass_tiles_f32(Ctx& c, TileArgs& a, cudaStream_t st);
void pass_finish_f64(Ctx& c, void* uval, const int32_t* child,
                     double* dev_energy, cudaStream_t st);
void pass_finish_f32(Ctx& c, void* uval, const int32_t* child,
                     double* dev_energy, cudaStream_t st);

// solver="pd" split/join on the current set after a pass
struct PdRsArgs {
  void* f[5];          // u, ubar, px, py, pz of the current set
  int32_t* child;
  int64_t* state;      // host int64[3]
  int64_t cap;
  int d_max;
  double tau_s, tau_j;
  int64_t out2[2];     // splits, joins
};
void pd_restructure_f64(Ctx& c, PdRsArgs& a, cudaStream_t st);
void pd_restructure_f32(Ctx& c, PdRsArgs& a, cudaStream_t st);
void pd_passes_f64(Ctx& c, PdHostArgs& a, cudaStream_t st);
void pd_passes_f32(Ctx& c, PdHostArgs& a, cudaStream_t st);
void frozen_passes_f64(Ctx& c, FrozenArgs& a, cudaStream_t st);
void frozen_passes_f32(Ctx& c, FrozenArgs& a, cudaStream_t st);
void propagate_levels_f64(Ctx& c, double* v, const int32_t* child, int lo,
                          int hi, cudaStream_t st);
void propagate_levels_f32(Ctx& c, float* v, const int32_t* child, int lo,
                          int hi, cudaStream_t st);
// marching cubes over a dense cell-centred grid (mesh.cu)
void marching_cubes_tree(Ctx& c, int dtype, const void* value,
                         const int32_t* child, int d_max, int seen_dtype,
                         const void* seen_v, const int32_t* seen_c,
                         const int8_t* tri_table, const int8_t* tri_count,
                         const int8_t* edge_axis, const int8_t* edge_off,
                         const double* origin, double voxel, int world,
                         int64_t bx0, int64_t bx1, octf_mesh* out,
                         cudaStream_t st);
void marching_cubes(const double* values, const uint8_t* mask, int n,
                    const int8_t* tri_table, const int8_t* tri_count,
                    const int8_t* edge_axis, const int8_t* edge_off,
                    const double* origin, double voxel, int world,
                    octf_mesh* out, cudaStream_t st);

// restrict the leaf-block list to a subset with per-block leaf masks
// (sharding); host arrays; regathers samples
void ctx_select(Ctx& c, const int32_t* sel, const uint8_t* masks,
                int64_t nsel, cudaStream_t st);

}  // namespace octf
