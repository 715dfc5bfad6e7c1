"""Plans (C-ABI handles) and device-side helpers for the Python mirror.

A plan owns the per-basis device tables (twiddles with Shoup companions,
per-level base-conversion tables); it plays the role of the reference's
module-level caches `_CTX_CACHE`, `_BC_CACHE`, `_BC_CENTER_CACHE`,
`_PARAMS_CACHE` (rnspoly.py:19-21, 245, 287; ckks.py:68), but is immutable
after creation and shared read-only.
"""

from __future__ import annotations

import ctypes as C
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _lib
from ._lib import CkError, check

_REG: dict[tuple, "Plan"] = {}
_REG_LOCK = threading.Lock()


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise CkError("CUDA device required: the B200 path has no CPU fallback")


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda, "device tensor expected"
    return t.data_ptr()


def to_dev(x) -> torch.Tensor:
    """numpy uint64 / torch tensor -> contiguous cuda uint64 tensor."""
    if isinstance(x, torch.Tensor):
        t = x if x.dtype == torch.uint64 else x.to(torch.uint64)
        return t.contiguous().cuda() if not t.is_cuda else t.contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
    return torch.from_numpy(a).cuda()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


class Plan:
    def __init__(self, logn: int, chain: tuple[int, ...], special: tuple[int, ...], dnum: int):
        require_cuda()
        lib = _lib.load()
        self.logn, self.n = logn, 1 << logn
        self.chain, self.special, self.dnum = tuple(chain), tuple(special), dnum
        self.moduli = self.chain + self.special
        self.index = {q: i for i, q in enumerate(self.moduli)}
        ch = (C.c_uint64 * len(chain))(*chain)
        sp = (C.c_uint64 * max(1, len(special)))(*special) if special else None
        h = C.c_void_p()
        torch.cuda.current_device()  # make sure the primary context exists
        check(lib.ck_plan_create(logn, ch, len(chain), sp, len(special), dnum, C.byref(h)),
              "ck_plan_create")
        self.h = h
        self._lib = lib
        self._idx: dict[tuple, torch.Tensor] = {}
        self._bc: dict[tuple, C.c_void_p] = {}
        self._lock = threading.Lock()
        info = (C.c_int64 * 5)()
        check(lib.ck_plan_info(h, info))
        self.alpha = int(info[4])

    def __del__(self):
        try:
            for b in self._bc.values():
                self._lib.ck_bconv_destroy(b)
            self._lib.ck_plan_destroy(self.h)
        except Exception:
            pass

    # ------------------------------------------------------------ helpers
    def prime_idx(self, moduli) -> torch.Tensor:
        key = tuple(moduli)
        t = self._idx.get(key)
        if t is None:
            t = torch.tensor([self.index[q] for q in key], dtype=torch.int32, device="cuda")
            self._idx[key] = t
        return t

    def workspace(self, level: int, batch: int) -> torch.Tensor:
        """Scratch for one ck_rotate / ck_modup / ck_moddown call, allocated per
        call from torch's stream-ordered caching allocator: concurrent callers
        on different streams or threads never share it."""
        nbytes = self._lib.ck_workspace_bytes(self.h, level, batch)
        if nbytes == 0:
            raise AssertionError(f"bad level {level}")
        return torch.empty(nbytes // 8, dtype=torch.uint64, device="cuda")

    def bconv(self, src, dst, centered: bool) -> C.c_void_p:
        key = (tuple(src), tuple(dst), bool(centered))
        with self._lock:
            b = self._bc.get(key)
            if b is None:
                si = (C.c_int32 * len(src))(*[self.index[q] for q in src])
                di = (C.c_int32 * len(dst))(*[self.index[q] for q in dst])
                b = C.c_void_p()
                check(self._lib.ck_bconv_create(self.h, si, len(src), di, len(dst),
                                                int(centered), C.byref(b)), "ck_bconv_create")
                self._bc[key] = b
        return b

    def psi(self) -> list[int]:
        out = (C.c_uint64 * len(self.moduli))()
        check(self._lib.ck_plan_psi(self.h, out))
        return [int(v) for v in out]

    def twiddles(self, q: int, inverse: bool = False) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.uint64)
        check(self._lib.ck_plan_twiddles(self.h, self.index[q], int(inverse),
                                         out.ctypes.data_as(C.c_void_p)))
        return out

    def covers(self, moduli) -> bool:
        return all(q in self.index for q in moduli)


def plan_for(params) -> Plan:
    key = ("p", params.logn, tuple(params.chain), tuple(params.special), params.dnum)
    with _REG_LOCK:
        p = _REG.get(key)
        if p is None:
            p = Plan(params.logn, tuple(params.chain), tuple(params.special), params.dnum)
            _REG[key] = p
    return p


def plan_covering(moduli, n: int) -> Plan:
    """Any registered plan of ring degree n whose basis contains `moduli`."""
    logn = n.bit_length() - 1
    with _REG_LOCK:
        for p in _REG.values():
            if p.logn == logn and p.covers(moduli):
                return p
        key = ("m", logn, tuple(moduli))
        p = Plan(logn, tuple(moduli), (), 1)
        _REG[key] = p
        return p


_CONST: "OrderedDict[tuple, torch.Tensor]" = OrderedDict()
_CONST_LOCK = threading.Lock()
_CONST_MAX = 512


def const_tensor(values, dtype=torch.uint64) -> torch.Tensor:
    """A small immutable device array (Galois elements, key / diagonal pointer
    arrays, Shoup constants), uploaded once per distinct content and reused:
    no host-to-device copy on repeat calls.  Keyed by the values themselves,
    so an entry can never go stale; callers must not write to it."""
    key = (dtype, tuple(int(v) for v in values))
    with _CONST_LOCK:
        t = _CONST.get(key)
        if t is not None:
            _CONST.move_to_end(key)
            return t
    np_dt = {torch.uint64: np.uint64, torch.int64: np.int64, torch.int32: np.int32}[dtype]
    t = torch.from_numpy(np.array(key[1], dtype=np_dt)).to("cuda")
    with _CONST_LOCK:
        _CONST[key] = t
        while len(_CONST) > _CONST_MAX:
            _CONST.popitem(last=False)
    return t


def ptr_array(tensors) -> torch.Tensor:
    """DEVICE array of the tensors' data pointers (the C ABI's key_ptrs[] / diags[])."""
    return const_tensor([ptr(t) for t in tensors], torch.int64)


def shoup_pairs(vals, moduli) -> torch.Tensor:
    """[(c, floor(c*2^64/q))] per row as a flat cuda uint64 tensor (cached on the device)."""
    out = []
    for c, q in zip(vals, moduli):
        c = int(c) % q
        out += [c, (c << 64) // q]
    return const_tensor(out)


def fill_uniform(out: torch.Tensor, keys: np.ndarray, qs: np.ndarray, logn: int) -> None:
    """Device twin of synth.uniform_row for len(keys) rows of out."""
    k = to_dev(np.asarray(keys, dtype=np.uint64))
    q = to_dev(np.asarray(qs, dtype=np.uint64))
    check(_lib.load().ck_fill_uniform(ptr(out), len(keys), logn, ptr(k), ptr(q),
                                      stream_handle()), "ck_fill_uniform")
