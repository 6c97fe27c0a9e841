"""The C-ABI library: builds, loads, exports every declared symbol, passes its
host self-test and refuses to compute without a GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from tests.conftest import REPO, has_gpu

HEADER = os.path.join(REPO, "include", "octfuse_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(octf_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1608_07411_b200 import _lib
    path = _lib.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", path]).decode()
    exported = set(re.findall(r"\bT (octf_[a-z_0-9]+)", out))
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    L = _lib.lib()
    for s in declared():
        assert getattr(L, s) is not None
    # the python binding declares a signature for every entry point
    assert set(_lib._SIGS) == set(declared())


def test_selftest_and_version():
    from paper_1608_07411_b200 import _lib
    assert _lib.lib().octf_selftest() == 0
    assert _lib.lib().octf_version() >= 100


def test_library_is_built_for_sm100a():
    from paper_1608_07411_b200 import _lib
    out = subprocess.check_output(["cuobjdump", "--list-elf", _lib.LIB_PATH]).decode()
    assert "sm_100a" in out


@pytest.mark.skipif(has_gpu(), reason="checks the no-device error path")
def test_no_cpu_fallback_without_device():
    from paper_1608_07411_b200 import _lib
    h = ctypes.c_void_p()
    rc = _lib.lib().octf_ctx_create(ctypes.byref(h))
    assert rc == 5
    assert b"no CUDA device" in _lib.lib().octf_last_error()
    with pytest.raises(RuntimeError):
        _lib.call("octf_densify", 0, None, None, 3, None, None)


def test_backend_module_mirrors_reference_plugin():
    from paper_1608_07411_b200 import _backend
    kern = _backend.get()
    for fn in ("build_tree", "propagate", "densify", "iterate_pass",
               "tree_energy"):
        assert callable(getattr(kern, fn))
    assert _backend.name() == "cuda"


def test_params_validation_mirrors_reference():
    from paper_1608_07411_b200.fusion import FusionParams, step_scale
    FusionParams()
    FusionParams(tau=-1.0)
    for bad in (dict(delta=0.0), dict(eta=0.0), dict(eta=0.001), dict(lam=0.0),
                dict(eps=0.0), dict(gamma=0.0), dict(xi0=0.0),
                dict(halve_every=0), dict(iterations=-1), dict(tau_split=-0.1),
                dict(tau_split=0.5), dict(tau_join=0.05)):
        with pytest.raises(ValueError):
            FusionParams(**bad)
    p = FusionParams(xi0=0.1, halve_every=20)
    assert step_scale(0, p) == 0.1 and step_scale(20, p) == 0.05
