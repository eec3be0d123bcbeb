"""The C-ABI library builds, loads and exports every symbol include/*.h declares
(CPU: no kernel launches), and rejects bad arguments with IG_EINVAL."""

import ctypes
import glob
import os
import re

import pytest

from tests.conftest import ROOT


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        with open(h) as f:
            names |= set(re.findall(r"^(?:int|const char\*)\s+(ig_\w+)\s*\(", f.read(), re.M))
    return names


@pytest.fixture(scope="module")
def lib():
    import torch  # noqa: F401  (loads the CUDA runtime the library links against)
    from paper_2406_19707_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.load(require_gpu=False)


def test_every_declared_symbol_is_exported_and_bound(lib):
    from paper_2406_19707_b200 import _lib
    declared = _declared()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)


def test_abi_version_and_status_strings(lib):
    assert lib.ig_abi_version() == 2
    assert lib.ig_status_string(0) == b"ok"
    assert b"invalid" in lib.ig_status_string(1)


def test_argument_validation_without_gpu(lib):
    from paper_2406_19707_b200 import _lib
    P = None
    assert lib.ig_rehearse(P, 0, P, P, P, 0, 1, 1, 1, 4, 1.0, P, P, P) == _lib.IG_EINVAL
    assert lib.ig_select(P, P, P, 1, 1, 1, 4, 1, 0.2, 1, P, P, P, None, P) == _lib.IG_EINVAL
    assert lib.ig_fetch(P, P, P, 1, 1, 4, 1, 512, P, 1, 256, P) == _lib.IG_EINVAL
    assert lib.ig_attend(P, 0, P, P, 0, P, 0, P, P, P, P, 1, 1, 128, 4, P, P, P, 0, P) == _lib.IG_EINVAL
    assert lib.ig_count(P, P, P, 1, 1, 4, -1.0, P, P, P) == _lib.IG_EINVAL
    sz, tk = ctypes.c_size_t(), ctypes.c_size_t()
    assert lib.ig_attend_scratch(2, 3, 128, 300, ctypes.byref(sz), ctypes.byref(tk)) == 0
    assert sz.value == 2 * 3 * 3 * 130 and tk.value == 6


def test_status_mapping_to_reference_exceptions(lib):
    from paper_2406_19707_b200 import _lib
    with pytest.raises(ValueError):
        _lib.check(_lib.IG_EINVAL, "x")
    with pytest.raises(IndexError):
        _lib.check(_lib.IG_ERANGE, "x")
    with pytest.raises(_lib.ArtifactConsistencyError):
        _lib.check(_lib.IG_ECONSISTENCY, "x")


def test_sass_is_sm100a(lib):
    """The fatbin carries sm_100a SASS only (no PTX JIT, no other arch)."""
    import subprocess
    from paper_2406_19707_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches
