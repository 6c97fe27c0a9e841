"""ctypes binding of the C ABI in include/octfuse_b200.h.

The shared library is built in-tree (``liboctfuse_b200.so`` next to this
file, see ``csrc/Makefile``).  There is no fallback: if the library or a CUDA
device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OCTF_LIB_PATH") or os.path.join(_HERE,
                                                           "liboctfuse_b200.so")

OCTF_F64 = 0
OCTF_F32 = 1
MAX_DEPTH = 19

_ERRORS = {1: ValueError, 2: MemoryError, 3: RuntimeError, 4: ValueError,
           5: RuntimeError}

P = ctypes.c_void_p
I32 = ctypes.c_int
I64 = ctypes.c_int64
DBL = ctypes.c_double

_SIGS = {
    "octf_last_error": ([], ctypes.c_char_p),
    "octf_version": ([], I32),
    "octf_selftest": ([], I32),
    "octf_ctx_create": ([P], I32),
    "octf_ctx_destroy": ([P], I32),
    "octf_ctx_invalidate": ([P], I32),
    "octf_ctx_info": ([P, P], I32),
    "octf_ctx_profile": ([P, I32, P], I32),
    "octf_ctx_set_options": ([P, I32], I32),
    "octf_ctx_phases": ([P, P], I32),
    "octf_iterate_pass": ([P, I32, P, P, P, P, P, I64, I32, P, P, P, I32, DBL,
                           DBL, DBL, DBL, DBL, DBL, I32, I32, I32, P, I64, P,
                           P], I32),
    "octf_fuse_pass": ([P, I32, P, P, P, P, P, I64, I32, P, P, P, I32, DBL,
                        DBL, DBL, DBL, DBL, DBL, I32, I32, P, I64, P, P, P],
                       I32),
    "octf_fuse_passes": ([P, I32, P, P, P, P, P, I64, I32, P, P, P, I32, DBL,
                          DBL, DBL, DBL, DBL, I32, I32, P, I32, P, P, P, P],
                         I32),
    "octf_fuse_passes_frozen": ([P, I32, P, P, P, P, I64, I32, P, P, P, I32,
                                 DBL, DBL, DBL, DBL, DBL, I32, P, I32, P, I32,
                                 P], I32),
    "octf_ctx_prepare": ([P, P, P, I64, I32, I32, P, P, P, P], I32),
    "octf_node_order": ([P, P, P, I64, I32, I32, P, P, P, P], I32),
    "octf_view_tsdf_box": ([P, I32, I32, P, P, DBL, I32, P, DBL, DBL, P, P, P,
                            P, P], I32),
    "octf_build_octree_box": ([P, I32, P, I32, I32, I32, DBL, P, I32, P, P,
                               I64, I64, I32, I32, P, P, P], I32),
    "octf_pd_restructure": ([P, I32, P, P, P, I64, I32, DBL, DBL, P, P], I32),
    "octf_marching_cubes": ([P, P, I32, P, P, P, P, P, DBL, I32, P, P, P, P],
                            I32),
    "octf_mesh_copy": ([P, P, P, P], I32),
    "octf_marching_cubes_tree": ([P, I32, P, P, P, I64, I32, I32, P, P, P, P,
                                  P, P, P, DBL, I32, I64, I64, P, P, P, P],
                                 I32),
    "octf_mesh_free": ([P], I32),
    "octf_pass_tiles": ([P, I32, P, P, P, P, I64, I32, P, P, P, I32, DBL, DBL,
                         DBL, DBL, I32, I32, I32, P], I32),
    "octf_pass_finish": ([P, I32, P, P, P, P], I32),
    "octf_pd_passes": ([P, I32, P, P, P, P, I64, I32, P, P, P, I32, DBL, DBL,
                        DBL, DBL, I32, I32, P, I32, P], I32),
    "octf_ctx_select": ([P, P, P, I64, P], I32),
    "octf_ctx_set_samples": ([P, P, P, I32, I64, P], I32),
    "octf_propagate_levels": ([P, I32, P, P, I32, I32, P], I32),
    "octf_halo_pack": ([I32, P, I32, P, I64, P, I32, P], I32),
    "octf_propagate": ([P, I32, P, P, P, I64, I32, P], I32),
    "octf_tree_energy": ([P, I32, P, P, P, I64, I32, P, P, P, I32, DBL, DBL,
                          DBL, P, P, P], I32),
    "octf_densify": ([I32, P, P, I32, P, P], I32),
    "octf_build_tree": ([P, P, P, P, I32, P, P, P, DBL, P, I32, P, P, P, I64,
                         I32, P], I32),
    "octf_pyramids": ([P, I32, P, I32, P, P, P, P, P, P, P, P, P], I32),
    "octf_build_octree": ([P, I32, P, I32, DBL, P, I32, P, P, P, I64, P], I32),
    "octf_view_tsdf": ([P, I32, I32, P, P, DBL, I32, DBL, DBL, P, P, P, P, P],
                       I32),
    "octf_initial_field": ([P, P, DBL, I64, P, P], I32),
    "octf_trace_blob": ([P, I32, I32, P, DBL, DBL, DBL, P, P, I32, DBL, DBL,
                         I32, DBL, P, P], I32),
    "octf_locate": ([P, I32, I32, P, I64, P, P, P], I32),
    "octf_nearest_vertex": ([P, I64, P, I64, P, P], I32),
    "octf_trace_room": ([P, I32, I32, P, I32, I32, DBL, DBL, DBL, I32, DBL, P,
                         P], I32),
}

_lib = None


def build(force: bool = False) -> str:
    """Compile the CUDA library for sm_100a (nvcc cross-compiles, no GPU
    needed)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-j8", "-C",
                               os.path.join(_HERE, "csrc")])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with "
                "`make -C paper_1608_07411_b200/csrc` (there is no CPU "
                "fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc:
        msg = lib().octf_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr_table(ptrs):
    return (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)


# octf_ctx_set_options flags (include/octfuse_b200.h)
CTX_DENSE, CTX_ELL, CTX_SORTED, CTX_DEFER, CTX_PACKED = 1, 2, 4, 8, 16

# context rebuild phases (octf_ctx.h Phase), in export order
PHASES = ("walk", "list_diff", "tables", "ell_grow", "ell_update", "fresh",
          "move", "full_list", "full_gather", "tail", "split_cascade",
          "split_alloc", "joins", "sweep")


class Ctx:
    """Owning handle of an ``octf_ctx`` (solver acceleration structures)."""

    def __init__(self):
        h = ctypes.c_void_p()
        call("octf_ctx_create", ctypes.byref(h))
        self.h = h

    def invalidate(self):
        call("octf_ctx_invalidate", self.h)

    def info(self) -> dict:
        import numpy as np
        out = np.zeros(12, dtype=np.int64)
        call("octf_ctx_info", self.h, out.ctypes.data)
        keys = ("leaf_blocks", "leaves", "blocks", "free_blocks", "mask_samples",
                "sample_stride", "views", "valid", "tiles", "ell", "all_valid",
                "packed")
        return dict(zip(keys, (int(v) for v in out)))

    def set_dense(self, dense: bool = True) -> None:
        """Keep the dense sample layout at any view count (solver='pd')."""
        call("octf_ctx_set_options", self.h, 1 if dense else 0)

    def set_options(self, flags: int) -> None:
        """octf_ctx_set_options: CTX_DENSE (1) dense samples, CTX_ELL (2)
        ELL from 33 views, CTX_SORTED (4) samples sorted per leaf (pd),
        CTX_DEFER (8) no sample gather before ctx_select (shards),
        CTX_PACKED (16) leaf-rank sample positions (frozen trees)."""
        call("octf_ctx_set_options", self.h, int(flags))

    def profile(self, enable: bool = True) -> dict:
        """Read and reset the live kernel timers; (re)arm them if enable."""
        import numpy as np
        ph = np.zeros(5 + len(PHASES), dtype=np.float64)
        call("octf_ctx_phases", self.h, ph.ctypes.data)  # before the reset
        out = np.zeros(5, dtype=np.float64)
        call("octf_ctx_profile", self.h, int(bool(enable)), out.ctypes.data)
        return {"leaf_ms": float(out[0]), "leaf_launches": int(out[1]),
                "energy_ms": float(out[2]), "energy_launches": int(out[3]),
                "launches": int(out[4]),
                "prepare_ms": float(ph[0]), "prepares": int(ph[1]),
                "gather_ms": float(ph[2]), "gathers": int(ph[3]),
                "restructure_ms": float(ph[4]),
                "rebuild_phases_ms": {k: float(v)
                                      for k, v in zip(PHASES, ph[5:])}}

    def close(self):
        if self.h:
            lib().octf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
