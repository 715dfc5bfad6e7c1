"""GPU mirror of ckkslab.rnspoly (/root/reference/pkg/src/ckkslab/rnspoly.py).

Same names, argument meaning and error behaviour (AssertionError on basis /
representation mismatch); ``data`` is a (limbs, N) torch.uint64 CUDA tensor
instead of a numpy array.  Every arithmetic op runs in libckks_b200.so.
Pure functions: outputs are fresh tensors, inputs are never mutated
(rnspoly.py:49, 65, 178).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check
from .device import plan_covering, ptr, shoup_pairs, stream_handle, to_dev

OP_ADD, OP_SUB, OP_MUL, OP_NEG, OP_MULC, OP_COPY, OP_ADDC = range(7)


def _poly_op(op: int, moduli, x: torch.Tensor, y: torch.Tensor | None = None,
             cst: torch.Tensor | None = None) -> torch.Tensor:
    n = x.shape[1]
    plan = plan_covering(moduli, n)
    out = torch.empty_like(x)
    if len(moduli) == 0:
        return out
    check(_lib.load().ck_poly_op(plan.h, op, ptr(out), ptr(x), ptr(y), ptr(plan.prime_idx(moduli)),
                                 ptr(cst), len(moduli), stream_handle()), "ck_poly_op")
    return out


def ntt_rows(data: torch.Tensor, moduli, inverse: bool) -> torch.Tensor:
    """_ntt_rows (ckks.py:359-364) / to_eval / to_coeff on a (limbs, N) tensor."""
    out = data.clone()
    if len(moduli) == 0:
        return out
    n = data.shape[1]
    plan = plan_covering(moduli, n)
    check(_lib.load().ck_ntt(plan.h, ptr(out), ptr(plan.prime_idx(moduli)), len(moduli), 1, 0,
                             int(inverse), stream_handle()), "ck_ntt")
    return out


class NttContext:
    """NttContext (rnspoly.py:24-98) for one (q, n); tables live in a plan."""

    def __init__(self, q: int, n: int):
        self.q, self.n = q, n
        self.plan = plan_covering((q,), n)
        self.psi = self.plan.psi()[self.plan.index[q]]

    @property
    def tw(self):
        return self.plan.twiddles(self.q, False)

    @property
    def itw(self):
        return self.plan.twiddles(self.q, True)

    def ntt(self, a) -> torch.Tensor:
        return ntt_rows(to_dev(a).reshape(1, -1), (self.q,), False)[0]

    def intt(self, a) -> torch.Tensor:
        return ntt_rows(to_dev(a).reshape(1, -1), (self.q,), True)[0]


_CTX: dict = {}


def get_ctx(q: int, n: int) -> NttContext:
    key = (q, n)
    if key not in _CTX:
        _CTX[key] = NttContext(q, n)
    return _CTX[key]


@dataclass
class RnsPoly:
    moduli: tuple[int, ...]
    data: torch.Tensor
    rep: str  # "coeff" | "eval"

    def __post_init__(self):
        self.moduli = tuple(int(q) for q in self.moduli)
        self.data = to_dev(self.data)

    @property
    def n(self) -> int:
        return self.data.shape[1]

    @classmethod
    def zeros(cls, moduli, n: int, rep: str) -> "RnsPoly":
        return cls(tuple(moduli), torch.zeros((len(moduli), n), dtype=torch.uint64, device="cuda"), rep)

    def copy(self) -> "RnsPoly":
        return RnsPoly(self.moduli, self.data.clone(), self.rep)

    def _check(self, other: "RnsPoly") -> None:
        assert self.moduli == other.moduli and self.rep == other.rep

    def add(self, other: "RnsPoly") -> "RnsPoly":
        self._check(other)
        return RnsPoly(self.moduli, _poly_op(OP_ADD, self.moduli, self.data, other.data), self.rep)

    def sub(self, other: "RnsPoly") -> "RnsPoly":
        self._check(other)
        return RnsPoly(self.moduli, _poly_op(OP_SUB, self.moduli, self.data, other.data), self.rep)

    def neg(self) -> "RnsPoly":
        return RnsPoly(self.moduli, _poly_op(OP_NEG, self.moduli, self.data), self.rep)

    def mul(self, other: "RnsPoly") -> "RnsPoly":
        self._check(other)
        assert self.rep == "eval"
        return RnsPoly(self.moduli, _poly_op(OP_MUL, self.moduli, self.data, other.data), self.rep)

    def mul_scalars(self, scalars) -> "RnsPoly":
        cst = shoup_pairs(scalars, self.moduli)
        return RnsPoly(self.moduli, _poly_op(OP_MULC, self.moduli, self.data, cst=cst), self.rep)

    def add_scalars(self, scalars) -> "RnsPoly":
        """self + (per-row constant in every slot): pt_add of encode_const's
        degree-0 polynomial (ckks.py:557-568) without materialising it."""
        assert self.rep == "eval"
        cst = shoup_pairs(scalars, self.moduli)
        return RnsPoly(self.moduli, _poly_op(OP_ADDC, self.moduli, self.data, cst=cst), self.rep)

    def to_eval(self) -> "RnsPoly":
        if self.rep == "eval":
            return self.copy()
        return RnsPoly(self.moduli, ntt_rows(self.data, self.moduli, False), "eval")

    def to_coeff(self) -> "RnsPoly":
        if self.rep == "coeff":
            return self.copy()
        return RnsPoly(self.moduli, ntt_rows(self.data, self.moduli, True), "coeff")

    def automorph(self, t: int) -> "RnsPoly":
        assert self.rep == "eval", "GPU path implements the eval-domain automorphism"
        return RnsPoly(self.moduli, automorph_rows(self.data, t, self.moduli), self.rep)


def automorph_rows(data: torch.Tensor, t: int, moduli=None) -> torch.Tensor:
    n = data.shape[1]
    out = torch.empty_like(data)
    if data.shape[0] == 0:
        return out
    plan = plan_covering(moduli if moduli else (), n) if moduli else _any_plan(n)
    check(_lib.load().ck_automorph(plan.h, ptr(out), ptr(data), data.shape[0], t % (2 * n),
                                   stream_handle()), "ck_automorph")
    return out


def _any_plan(n: int):
    from .device import _REG
    logn = n.bit_length() - 1
    for p in _REG.values():
        if p.logn == logn:
            return p
    raise AssertionError("no plan for this ring degree; create one via plan_for(params)")


def bc_convert(x: RnsPoly, dst) -> RnsPoly:
    """rnspoly.bc_convert (rnspoly.py:264-284)."""
    assert x.rep == "coeff"
    src = x.moduli
    dst = tuple(dst)
    assert len(src) * max(dst) < (1 << 64)
    plan = plan_covering(src + dst, x.n)
    out = torch.empty((len(dst), x.n), dtype=torch.uint64, device="cuda")
    check(_lib.load().ck_bconv_apply(plan.h, plan.bconv(src, dst, False), ptr(x.data), ptr(out),
                                     stream_handle()), "ck_bconv_apply")
    return RnsPoly(dst, out, "coeff")


def bc_convert_centered(x: RnsPoly, dst) -> RnsPoly:
    """rnspoly.bc_convert_centered (rnspoly.py:303-331), float64 estimate replicated."""
    assert x.rep == "coeff"
    src = x.moduli
    dst = tuple(dst)
    assert len(src) * max(dst) < (1 << 64)
    plan = plan_covering(src + dst, x.n)
    out = torch.empty((len(dst), x.n), dtype=torch.uint64, device="cuda")
    check(_lib.load().ck_bconv_apply(plan.h, plan.bconv(src, dst, True), ptr(x.data), ptr(out),
                                     stream_handle()), "ck_bconv_apply")
    return RnsPoly(dst, out, "coeff")


def modup_coeff(x: RnsPoly, extra) -> RnsPoly:
    conv = bc_convert(x, extra)
    return RnsPoly(x.moduli + tuple(extra), torch.cat([x.data, conv.data]), "coeff")


def moddown_coeff(x: RnsPoly, keep: int) -> RnsPoly:
    """rnspoly.moddown_coeff (rnspoly.py:341-359)."""
    assert x.rep == "coeff"
    drop, base = x.moduli[keep:], x.moduli[:keep]
    conv = bc_convert_centered(RnsPoly(drop, x.data[keep:], "coeff"), base)
    big_p = 1
    for p in drop:
        big_p *= p
    diff = RnsPoly(base, x.data[:keep], "coeff").sub(conv)
    return diff.mul_scalars([pow(big_p % q, -1, q) for q in base])


def rescale_coeff(x: RnsPoly) -> RnsPoly:
    return moddown_coeff(x, len(x.moduli) - 1)
