"""ctypes binding of libckks_b200.so (include/ckks_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
product entry point raises.  The binding is the same one a maintainer would
add to the reference package.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libckks_b200.so")

u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
vp = C.c_void_p

# (name, restype, argtypes) -- mirrors include/ckks_b200.h
_SIGS = [
    ("ck_version", C.c_int, []),
    ("ck_error_string", C.c_char_p, [C.c_int]),
    ("ck_launch_count", C.c_int64, []),
    ("ck_plan_create", C.c_int, [C.c_int, vp, C.c_int, vp, C.c_int, C.c_int, C.POINTER(vp)]),
    ("ck_plan_destroy", C.c_int, [vp]),
    ("ck_plan_info", C.c_int, [vp, vp]),
    ("ck_plan_psi", C.c_int, [vp, vp]),
    ("ck_plan_twiddles", C.c_int, [vp, C.c_int, C.c_int, vp]),
    ("ck_ntt", C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int64, C.c_int, vp]),
    ("ck_poly_op", C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, C.c_int, vp]),
    ("ck_automorph", C.c_int, [vp, vp, vp, C.c_int, C.c_uint64, vp]),
    ("ck_bconv_create", C.c_int, [vp, vp, C.c_int, vp, C.c_int, C.c_int, C.POINTER(vp)]),
    ("ck_bconv_destroy", C.c_int, [vp]),
    ("ck_bconv_apply", C.c_int, [vp, vp, vp, vp, vp]),
    ("ck_workspace_bytes", C.c_size_t, [vp, C.c_int, C.c_int]),
    ("ck_modup", C.c_int, [vp, vp, C.c_int, vp, vp, C.c_int, vp]),
    ("ck_kskip", C.c_int, [vp, vp, vp, vp, C.c_int, C.c_uint64, vp, vp, vp, C.c_int, vp]),
    ("ck_moddown", C.c_int, [vp, vp, C.c_int, C.c_int, vp, vp, C.c_uint64, vp, C.c_int, vp]),
    ("ck_rotate", C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.c_uint64, vp, C.c_int, vp, vp, vp,
                            C.c_int, vp]),
    ("ck_keyswitch_workspace_bytes", C.c_size_t, [vp, C.c_int, C.c_int, C.c_int]),
    ("ck_keyswitch", C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.c_uint64, vp, C.c_int, vp, vp, vp,
                               C.c_int, vp]),
    ("ck_relin_workspace_bytes", C.c_size_t, [vp, C.c_int, C.c_int]),
    ("ck_relin", C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, vp, vp, vp, C.c_int, vp]),
    ("ck_hrotate_workspace_bytes", C.c_size_t, [vp, C.c_int, C.c_int]),
    ("ck_hrotate", C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, vp, vp, vp, vp]),
    ("ck_xof_uniform", C.c_int, [vp, vp, C.c_int64, vp, C.c_int, C.c_int, vp, vp]),
    ("ck_expand_key_a", C.c_int, [vp, vp, vp, C.c_int64, C.c_int, vp, vp]),
    ("ck_pt_matvec_workspace_bytes", C.c_size_t, [vp, C.c_int, C.c_int]),
    ("ck_pt_matvec", C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, vp,
                               vp]),
    ("ck_bsgs_workspace_bytes", C.c_size_t, [vp, C.c_int, C.c_int, C.c_int]),
    ("ck_bsgs", C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp,
                          vp, vp]),
    ("ck_fill_uniform", C.c_int, [vp, C.c_int64, C.c_int, vp, vp, vp]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None


class CkError(RuntimeError):
    pass


def load(path: str | None = None):
    """Load the shared library (no device needed) and bind every symbol.
    CKB200_LIB overrides the path (A/B builds of the same sources)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("CKB200_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise CkError(f"{path} missing: run `python -m paper_2112_06396_b200.build` "
                      "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in _SIGS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


CK_ERR_ARG, CK_ERR_MODULUS, CK_ERR_ALLOC, CK_ERR_DEVICE = -1, -2, -3, -4


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().ck_error_string(rc).decode()
        if rc == -1:
            raise AssertionError(f"{what}: {msg}")  # reference raises AssertionError on bad args
        raise CkError(f"{what}: {msg} (code {rc})")
