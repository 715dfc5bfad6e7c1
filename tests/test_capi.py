"""The C-ABI library builds, loads without a GPU and exports every declared symbol."""

import os
import re

from paper_2112_06396_b200 import _lib
from paper_2112_06396_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ckks_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ck_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    build()
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)


def test_error_strings_and_version_without_device():
    lib = _lib.load()
    assert lib.ck_version() >= 1
    assert lib.ck_error_string(-1) == b"invalid argument"
    assert lib.ck_error_string(-2) == b"invalid modulus"


def test_plan_create_fails_loudly_without_device():
    import ctypes as C
    import torch
    if torch.cuda.is_available():
        return
    lib = _lib.load()
    h = C.c_void_p()
    ch = (C.c_uint64 * 1)(params_first_prime())
    rc = lib.ck_plan_create(12, ch, 1, None, 0, 1, C.byref(h))
    assert rc == -4  # CK_ERR_DEVICE: no silent CPU fallback


def params_first_prime():
    from paper_2112_06396_b200.params import config
    return config("C1").params.chain[0]


def test_sass_is_sm100a():
    """The shipped .so contains sm_100a SASS (cross-compiled here)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
