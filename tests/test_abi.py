"""The C-ABI library loads and exports every symbol include/stb200.h declares;
without a GPU the product fails loudly (no CPU fallback).  CPU only."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "stb200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(stb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2010_10248_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == names


def test_abi_version_and_error_channel():
    from paper_2010_10248_b200 import _lib
    lib = _lib.lib()
    assert lib.stb_abi_version() == 1
    # an argument error is reported through the status + thread-local message
    rc = lib.stb_support_info(None, None, None)
    assert rc == _lib.STB_ERR_ARG
    assert b"NULL" in lib.stb_last_error()


def test_cubins_are_sm100a():
    from paper_2010_10248_b200 import _lib
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    from paper_2010_10248_b200 import _lib, errors
    import paper_2010_10248_b200 as stb
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    grid = stb.GridSpec((8, 8, 8), (10.0,) * 3)
    cfg = stb.RunConfig(physics="acoustic", grid=grid, space_order=4, nt=2,
                        medium={"velocity": 1500.0})
    with pytest.raises(errors.DeviceError):
        stb.run(cfg)
    with pytest.raises(Exception):
        stb.interp_stencil((10.0, 10.0, 10.0), grid)
    with pytest.raises(errors.DeviceError):        # page-locked arrays need the driver too
        stb.pinned_empty((16, 16))
    assert stb.pinned_empty((0, 4)).shape == (0, 4)   # empty: plain NumPy, no device call


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2010_10248_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*", "", src).replace('"""', "") or \
                    "import oracle" not in src, f
                assert "import oracle" not in src and "from oracle" not in src, f
