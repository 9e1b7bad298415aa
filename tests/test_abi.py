"""CPU checks of the drop-in boundary: libgfcuda.so loads and exports every
symbol declared in include/gatefit_b200.h; the product has no CPU fallback."""

import ctypes
import os
import re

from conftest import ROOT


def _header_functions():
    src = open(os.path.join(ROOT, "include", "gatefit_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2506_23775_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTS)
    assert lib.gf_abi_version() == 100


def test_library_is_sm100a_cubin():
    import subprocess

    from paper_2506_23775_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_map_to_value_error():
    import pytest

    from paper_2506_23775_b200 import _lib

    rc = _lib.lib.gf_apply_gate(None, None, 4, 0, 1, None, 0, 1, None)
    assert rc == _lib.GF_EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc)
    rc = _lib.lib.gf_sector_unrank(None, 5, 0, None, None)
    assert rc == _lib.GF_EINVAL


def test_compute_without_gpu_fails_loudly():
    import numpy as np
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2506_23775_b200 import kernels as K

    with pytest.raises(RuntimeError):
        K.apply_gate(np.ones(4, complex), K.Gate(np.eye(4), (0, 1)))
