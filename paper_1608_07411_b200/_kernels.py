"""The kernel module behind ``_backend.get()`` -- the reference's plugin
boundary (reference ``_backend.py:24-26``, ``_kernels.pyx``) on the GPU.

Same function names, argument order, return values and exception types as
the reference's compiled module, with pools as CUDA tensors (torch is only
the allocator here) instead of numpy arrays; ``state`` stays a host int64[3]
array exactly like the reference.  Every call goes through the C ABI of
``liboctfuse_b200.so``; there is no CPU path.

The reference's kernels are stateless, so by default each call here starts
from a fresh view of the pool (the solver context is rebuilt).  ``fusion.fuse``
passes a persistent ``ctx`` so structure is only rebuilt when a pass changes
it.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._device import ptr, stream_handle
from ._lib import OCTF_F32, OCTF_F64, call, ptr_table

_shared_ctx = None


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return OCTF_F64
    if t.dtype == torch.float32:
        return OCTF_F32
    raise TypeError(f"unsupported pool dtype {t.dtype}")


def _fresh_ctx():
    global _shared_ctx
    if _shared_ctx is None:
        _shared_ctx = _lib.Ctx()
    _shared_ctx.invalidate()
    return _shared_ctx


def _state_ptr(state: np.ndarray) -> int:
    if not (isinstance(state, np.ndarray) and state.dtype == np.int64
            and state.flags.c_contiguous and state.shape[0] >= 3):
        raise TypeError("state must be a contiguous host int64[3] array")
    return state.ctypes.data


_view_cache = None   # (vvals, vws, vchilds, first/last pointers, tables)


def drop_view_cache() -> None:
    """Forget the cached pointer tables (and the references to the view
    pools they keep alive); solvers call it when they close."""
    global _view_cache
    _view_cache = None


def _views(vvals, vws, vchilds):
    """Pointer tables of the view pools.  A solver passes the same three
    lists every pass: the tables of the last call are reused while the list
    objects (and their end pointers) are unchanged -- 900 data_ptr() calls
    per pass at 300 views otherwise (0.2 ms of host time per pass)."""
    global _view_cache
    if not (len(vvals) == len(vws) == len(vchilds)):
        raise ValueError("view pool lists differ in length")
    ends = ((ptr(vvals[0]), ptr(vvals[-1]), ptr(vws[0]), ptr(vws[-1]),
             ptr(vchilds[0]), ptr(vchilds[-1])) if len(vvals) else ())
    c = _view_cache
    if (c is not None and c[0] is vvals and c[1] is vws and c[2] is vchilds
            and c[3] == (len(vvals),) + ends):
        return c[4]
    for v in vvals:
        if v.dtype != torch.float32:
            raise TypeError("view values must be float32 pools")
    tabs = (ptr_table([ptr(v) for v in vvals]),
            ptr_table([ptr(v) for v in vws]),
            ptr_table([ptr(v) for v in vchilds]))
    _view_cache = (vvals, vws, vchilds, (len(vvals),) + ends, tabs)
    return tabs


def build_tree(meanf, minf, maxf, offs, has_w, wminf, wmaxf, wmeanf, tau,
               value, weight, child, state, d_max):
    """_kernels.pyx:21-77 (pyramids and pools on device, offs/state host)."""
    if d_max > 60:
        raise ValueError("tree depth out of range")
    offs = np.ascontiguousarray(np.asarray(offs, dtype=np.int64))
    call("octf_build_tree", ptr(meanf), ptr(minf), ptr(maxf), offs.ctypes.data,
         int(bool(has_w)), ptr(wminf) if has_w else None,
         ptr(wmaxf) if has_w else None, ptr(wmeanf) if has_w else None,
         float(tau), ptr(value), _dtype_code(value),
         ptr(weight) if has_w else None, ptr(child), _state_ptr(state),
         value.shape[0], int(d_max), stream_handle())


def propagate(value, child, *, state=None, d_max=_lib.MAX_DEPTH, ctx=None):
    """_kernels.pyx:80-113."""
    c = ctx if ctx is not None else _fresh_ctx()
    call("octf_propagate", c.h, _dtype_code(value), ptr(value), ptr(child),
         _state_ptr(state) if state is not None else None, child.shape[0],
         int(d_max), stream_handle())


def node_order(child, state, d_max, *, leaves_only=False, ctx=None):
    """Every live node (or leaf) in the reference's canonical depth-first
    order (octree.py:168-181, :413-431), computed on the device: (slots
    int32, preorder keys int64) CUDA tensors -- see decode_keys."""
    c = ctx if ctx is not None else _fresh_ctx()
    st = np.ascontiguousarray(np.asarray(state, dtype=np.int64)[:3])
    n = int(st[2])
    slots = torch.empty(max(n, 1), dtype=torch.int32, device=child.device)
    keys = torch.empty(max(n, 1), dtype=torch.int64, device=child.device)
    cnt = np.zeros(1, dtype=np.int64)
    call("octf_node_order", c.h, ptr(child), st.ctypes.data, child.shape[0],
         int(d_max), 1 if leaves_only else 0, ptr(slots), ptr(keys),
         cnt.ctypes.data, stream_handle())
    k = int(cnt[0])
    return slots[:k], keys[:k]


def decode_keys(keys, d_max):
    """(level, x, y, z) int64 tensors of preorder keys (Morton key of the
    node's first finest-level cell << 5 | level)."""
    level = keys & 31
    first = keys >> 5
    x = torch.zeros_like(first)
    y = torch.zeros_like(first)
    z = torch.zeros_like(first)
    for bit in range(d_max):
        x |= ((first >> (3 * bit + 2)) & 1) << bit
        y |= ((first >> (3 * bit + 1)) & 1) << bit
        z |= ((first >> (3 * bit)) & 1) << bit
    sh = d_max - level
    return level, x >> sh, y >> sh, z >> sh


def densify(value, child, d_max, out):
    """_kernels.pyx:116-158 (out: device (2^d)^3 float64)."""
    if d_max > 60:
        raise ValueError("tree depth out of range")
    call("octf_densify", _dtype_code(value), ptr(value), ptr(child),
         int(d_max), ptr(out), stream_handle())


def iterate_pass(uval, usnap, uchild, ujoined, ustate, vvals, vws, vchilds,
                 d_max, lam, eps, gamma, xi, tau_s, tau_j, clamp, reverse,
                 jlog, *, ctx=None, snapshot=True):
    """_kernels.pyx:384-461; returns (splits, joins, jrows)."""
    if d_max > 60:
        raise ValueError("tree depth out of range")
    c = ctx if ctx is not None else _fresh_ctx()
    tv, tw, tc = _views(vvals, vws, vchilds)
    out3 = np.zeros(3, dtype=np.int64)
    jcap = 0 if jlog is None else int(jlog.shape[0])
    call("octf_iterate_pass", c.h, _dtype_code(uval), ptr(usnap), ptr(uval),
         ptr(uchild), ptr(ujoined), _state_ptr(ustate), uval.shape[0],
         len(vvals), tv, tw, tc, int(d_max), float(lam), float(eps),
         float(gamma), float(xi), float(tau_s), float(tau_j), int(bool(clamp)),
         int(bool(reverse)), int(bool(snapshot)),
         ptr(jlog) if jcap else None, jcap, out3.ctypes.data, stream_handle())
    return int(out3[0]), int(out3[1]), int(out3[2])


def fuse_pass(usnap, uval, uchild, ujoined, ustate, vvals, vws, vchilds,
              d_max, lam, eps, gamma, xi, tau_s, tau_j, clamp, reverse, jlog,
              *, ctx):
    """One pass of the fuse loop (iterate + propagate) with the energy of the
    incoming state; returns (splits, joins, jrows, energy_pre)."""
    tv, tw, tc = _views(vvals, vws, vchilds)
    out3 = np.zeros(3, dtype=np.int64)
    e = np.zeros(1, dtype=np.float64)
    jcap = 0 if jlog is None else int(jlog.shape[0])
    call("octf_fuse_pass", ctx.h, _dtype_code(uval), ptr(usnap), ptr(uval),
         ptr(uchild), ptr(ujoined), _state_ptr(ustate), uval.shape[0],
         len(vvals), tv, tw, tc, int(d_max), float(lam), float(eps),
         float(gamma), float(xi), float(tau_s), float(tau_j), int(bool(clamp)),
         int(bool(reverse)), ptr(jlog) if jcap else None, jcap,
         out3.ctypes.data, e.ctypes.data, stream_handle())
    return int(out3[0]), int(out3[1]), int(out3[2]), float(e[0])


def fuse_passes(ubuf0, ubuf1, uchild, ujoined, ustate, vvals, vws, vchilds,
                d_max, lam, eps, gamma, tau_s, tau_j, clamp, reverse, xis, *,
                ctx):
    """len(xis) passes of the fuse loop with split/join in one call (pass k
    reads buffer k % 2); returns (done, out3[done, 3] = splits / joins / live
    nodes, energies_pre[done], error): ``error`` is the RuntimeError of a
    pass that ran out of pool capacity (None otherwise) -- the first
    ``done`` passes are complete and the caller may grow the pools."""
    import ctypes
    tv, tw, tc = _views(vvals, vws, vchilds)
    xis = np.ascontiguousarray(np.asarray(xis, dtype=np.float64))
    k = len(xis)
    out3 = np.zeros((max(k, 1), 3), dtype=np.int64)
    en = np.zeros(max(k, 1), dtype=np.float64)
    done = ctypes.c_int(0)
    err = None
    try:
        call("octf_fuse_passes", ctx.h, _dtype_code(ubuf0), ptr(ubuf0),
             ptr(ubuf1), ptr(uchild), ptr(ujoined), _state_ptr(ustate),
             ubuf0.shape[0], len(vvals), tv, tw, tc, int(d_max), float(lam),
             float(eps), float(gamma), float(tau_s), float(tau_j),
             int(bool(clamp)), int(bool(reverse)), xis.ctypes.data, k,
             out3.ctypes.data, en.ctypes.data, ctypes.byref(done),
             stream_handle())
    except RuntimeError as exc:
        if "capacity" not in str(exc):
            raise
        err = exc
    n = int(done.value)
    return n, out3[:n], en[:n], err


def fuse_passes_frozen(ubuf0, ubuf1, uchild, ustate, vvals, vws, vchilds,
                       d_max, lam, eps, gamma, tau_s, tau_j, clamp, xis, *,
                       ctx, energies_out=None):
    """len(xis) passes of a frozen structure in one call; returns the
    energies before each pass.  Pass k reads buffer k%2."""
    tv, tw, tc = _views(vvals, vws, vchilds)
    xis = np.ascontiguousarray(np.asarray(xis, dtype=np.float64))
    if energies_out is None:
        en = np.zeros(len(xis), dtype=np.float64)
        eptr, dev = en.ctypes.data, 0
    else:  # device tensor: the call stays asynchronous
        en = energies_out
        eptr, dev = ptr(energies_out), 1
    call("octf_fuse_passes_frozen", ctx.h, _dtype_code(ubuf0), ptr(ubuf0),
         ptr(ubuf1), ptr(uchild), _state_ptr(ustate), ubuf0.shape[0],
         len(vvals), tv, tw, tc, int(d_max), float(lam), float(eps),
         float(gamma), float(tau_s), float(tau_j), int(bool(clamp)),
         xis.ctypes.data, len(xis), eptr, dev, stream_handle())
    return en


def pd_passes(set_a, set_b, uchild, ustate, vvals, vws, vchilds, d_max, lam,
              tau, sigma, gamma, clamp, npasses, *, ctx, energies_out=None):
    """solver='pd': npasses primal-dual passes; set_a/set_b = 5 pools
    (u, ubar, px, py, pz).  Returns the energies before each pass (host), or
    writes them to ``energies_out`` (a float64 CUDA tensor; asynchronous)."""
    tv, tw, tc = _views(vvals, vws, vchilds)
    ta = ptr_table([ptr(t) for t in set_a])
    tb = ptr_table([ptr(t) for t in set_b])
    dev = energies_out is not None
    if dev and (energies_out.dtype != torch.float64 or not energies_out.is_cuda
                or energies_out.numel() < npasses):
        raise TypeError("energies_out must be a float64 CUDA tensor")
    en = None if dev else np.zeros(max(int(npasses), 1), dtype=np.float64)
    call("octf_pd_passes", ctx.h, _dtype_code(set_a[0]), ta, tb, ptr(uchild),
         _state_ptr(ustate), uchild.shape[0], len(vvals), tv, tw, tc,
         int(d_max), float(lam), float(tau), float(sigma), float(gamma),
         int(bool(clamp)), int(npasses),
         ptr(energies_out) if dev else en.ctypes.data, int(dev),
         stream_handle())
    return energies_out if dev else en[:npasses]


def pass_tiles(usnap, uval, uchild, ustate, vvals, vws, vchilds, d_max, lam,
               eps, gamma, xi, clamp, tile0, ntiles, *, ctx):
    """Leaf kernel of one frozen pass on leaf tiles [tile0, tile0+ntiles)
    (sharded overlap: interior tiles while the halo is in flight)."""
    tv, tw, tc = _views(vvals, vws, vchilds)
    call("octf_pass_tiles", ctx.h, _dtype_code(uval), ptr(usnap), ptr(uval),
         ptr(uchild), _state_ptr(ustate), uchild.shape[0], len(vvals), tv, tw,
         tc, int(d_max), float(lam), float(eps), float(gamma), float(xi),
         int(bool(clamp)), int(tile0), int(ntiles), stream_handle())


def pass_finish(uval, uchild, dev_energy, *, ctx):
    """Propagate the pass output and sum its energy partials into
    ``dev_energy`` (a one-element float64 CUDA tensor)."""
    if dev_energy.dtype != torch.float64 or not dev_energy.is_cuda:
        raise TypeError("dev_energy must be a float64 CUDA tensor")
    call("octf_pass_finish", ctx.h, _dtype_code(uval), ptr(uval), ptr(uchild),
         ptr(dev_energy), stream_handle())


def pd_restructure(fields, uchild, ustate, d_max, tau_split, tau_join, *,
                   ctx):
    """solver='pd' split/join on the current set (u, ubar, px, py, pz) after
    a pass; updates uchild/ustate in place.  Returns (splits, joins)."""
    tf = ptr_table([ptr(t) for t in fields])
    out = np.zeros(2, dtype=np.int64)
    call("octf_pd_restructure", ctx.h, _dtype_code(fields[0]), tf,
         ptr(uchild), _state_ptr(ustate), uchild.shape[0], int(d_max),
         float(tau_split), float(tau_join), out.ctypes.data, stream_handle())
    return int(out[0]), int(out[1])


def ctx_prepare(ctx, uchild, ustate, d_max, vvals, vws, vchilds):
    tv, tw, tc = _views(vvals, vws, vchilds)
    call("octf_ctx_prepare", ctx.h, ptr(uchild), _state_ptr(ustate),
         uchild.shape[0], int(d_max), len(vvals), tv, tw, tc, stream_handle())


def ctx_set_samples(ctx, f_slot, w_slot=None):
    """Per-slot samples [nviews][cap] (device float32) instead of views."""
    if f_slot.dtype != torch.float32 or f_slot.dim() != 2:
        raise TypeError("samples must be a [nviews, cap] float32 tensor")
    f_slot = f_slot.contiguous()
    if w_slot is not None:
        w_slot = w_slot.contiguous()
    call("octf_ctx_set_samples", ctx.h, ptr(f_slot), ptr(w_slot),
         f_slot.shape[0], f_slot.shape[1], stream_handle())


def ctx_select(ctx, sel, masks):
    sel = np.ascontiguousarray(np.asarray(sel, dtype=np.int32))
    masks = np.ascontiguousarray(np.asarray(masks, dtype=np.uint8))
    call("octf_ctx_select", ctx.h, sel.ctypes.data if sel.size else None,
         masks.ctypes.data if masks.size else None, sel.size, stream_handle())


def propagate_levels(value, child, lo, hi, *, ctx):
    call("octf_propagate_levels", ctx.h, _dtype_code(value), ptr(value),
         ptr(child), int(lo), int(hi), stream_handle())


def tree_energy(uval, uchild, vvals, vws, vchilds, d_max, lam, eps, gamma, *,
                state=None, ctx=None, terms=None):
    """_kernels.pyx:536-578; returns the energy as a Python float."""
    c = ctx if ctx is not None else _fresh_ctx()
    tv, tw, tc = _views(vvals, vws, vchilds)
    out = np.zeros(1, dtype=np.float64)
    call("octf_tree_energy", c.h, _dtype_code(uval), ptr(uval), ptr(uchild),
         _state_ptr(state) if state is not None else None, uchild.shape[0],
         len(vvals), tv, tw, tc, int(d_max), float(lam), float(eps),
         float(gamma), out.ctypes.data, ptr(terms), stream_handle())
    return float(out[0])


def halo_pack(fields, idx, buf, unpack=False):
    """buf[k*n + j] <-> fields[k][idx[j]] on the current stream (shard.py
    halo staging; idx an int32 CUDA tensor, buf a flat CUDA tensor)."""
    fields = list(fields)
    n = idx.shape[0]
    if idx.dtype != torch.int32 or not idx.is_cuda:
        raise TypeError("idx must be an int32 CUDA tensor")
    if buf.numel() < len(fields) * n or buf.dtype != fields[0].dtype:
        raise ValueError("halo buffer too small or of another dtype")
    call("octf_halo_pack", _dtype_code(fields[0]),
         ptr_table([ptr(f) for f in fields]), len(fields), ptr(idx), n,
         ptr(buf), int(bool(unpack)), stream_handle())
