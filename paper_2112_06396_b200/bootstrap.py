"""GPU mirror of the reference bootstrapping driver (ckkslab/bootstrap.py).

Covers SURVEY 8(f) rows 2-3: the CoeffToSlot / SlotToCoeff linear transforms
(``pt_matvec`` stages, ckks.py) and the sine evaluation -- the
baby-step/giant-step Chebyshev evaluator built on ``new_mult``'s fused
variants plus the double-angle steps (bootstrap.py:158-210, 290-297) -- and
``bootstrap`` itself (bootstrap.py:300-333).  Every ciphertext operation runs
on the device through libckks_b200.so; only the Chebyshev coefficient
algebra (numpy.polynomial, float64 on a few dozen coefficients, exactly as
the reference) and the constant encodings run on the host.

Plans are built by the reference's host encoder (diagonals encoded on the
raised basis, bootstrap.py:236-240); ``BootstrapPlan`` holds the same fields.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from numpy.polynomial import chebyshev as C

from . import ckks
from .ckks import Ciphertext, CkksParams, KeySet, MatvecStage


@dataclass
class BootstrapPlan:
    """bootstrap.BootstrapPlan (bootstrap.py:219-233); `cts`/`stc` are
    MatvecStage lists with device diagonals."""

    params: CkksParams
    doublings: int
    degree: int
    cheb: np.ndarray
    const_shift: float
    cts: list
    stc: list
    input_limbs: int
    output_limbs: int


class ChebEvaluator:
    """bootstrap._ChebEvaluator (bootstrap.py:158-210).

    T_1 = ct_w; T_2,4,..,32 by doubling (new_mult(ct, ct, value_mult=2,
    const=-1)); T_3,5,6,7 as 2 T_a T_b - T_|a-b| via new_mult's addend;
    the BSGS recursion splits at the largest power-of-two giant <= degree
    with chebdiv and recombines with new_mult(q, T_giant, addend=r).
    """

    def __init__(self, params: CkksParams, keys: KeySet, ct_w: Ciphertext, degree: int):
        self.params, self.keys = params, keys
        self.t: dict[int, Ciphertext] = {1: ct_w}
        for k in (2, 4, 8, 16, 32):
            if k <= degree:
                self.t[k] = self._double(self.t[k // 2])
        for k in (3, 5, 6, 7):
            if k <= min(degree, 7):
                a, b = (2, 1) if k == 3 else (4, k - 4)
                self.t[k] = ckks.new_mult(params, keys, self.t[a], self.t[b], value_mult=2,
                                          addend=self.t[abs(2 * a - k)], addend_sign=-1)

    def _double(self, ct: Ciphertext) -> Ciphertext:
        return ckks.new_mult(self.params, self.keys, ct, ct, value_mult=2, const=-1.0)

    def run(self, coeffs) -> Ciphertext:
        return self._eval(np.asarray(coeffs, dtype=float))

    def _eval(self, coeffs: np.ndarray) -> Ciphertext:
        deg = len(coeffs) - 1
        if deg <= 7:
            terms = [(self.t[j], float(coeffs[j])) for j in range(1, deg + 1)
                     if abs(coeffs[j]) > 1e-300]
            return ckks.pt_combo(self.params, terms, float(coeffs[0]))
        giant = 8
        while giant * 2 <= deg:
            giant *= 2
        tg = np.zeros(giant + 1)
        tg[giant] = 1.0
        quo, rem = C.chebdiv(coeffs, tg)
        q_ct = self._eval(quo)
        r_ct = self._eval(rem)
        return ckks.new_mult(self.params, self.keys, q_ct, self.t[giant], addend=r_ct,
                             addend_sign=1)


def sine_eval(params: CkksParams, keys: KeySet, plan: BootstrapPlan,
              ct: Ciphertext) -> Ciphertext:
    """bootstrap._sine_eval (bootstrap.py:290-297)."""
    ct_w = ckks.const_add(params, ct, plan.const_shift)
    ev = ChebEvaluator(params, keys, ct_w, plan.degree)
    out = ev.run(plan.cheb)
    for _ in range(plan.doublings):
        out = ev._double(out)
    return out


def bootstrap(params: CkksParams, keys: KeySet, plan: BootstrapPlan,
              ct: Ciphertext) -> Ciphertext:
    """bootstrap.bootstrap (bootstrap.py:300-333): raise, CoeffToSlot,
    conjugate split, two sine evaluations, SlotToCoeff."""
    assert ct.limbs >= plan.input_limbs
    half = params.n_ring // 2
    eps = ct.delta / params.delta - 1
    assert abs(eps) < 1e-4, eps
    ct = Ciphertext(ct.a, ct.b, params.delta)
    ct = ckks.coeff_to_slot_entry(params, ct, plan.input_limbs)
    ct = ckks.matvec_stages(params, keys, ct, plan.cts)
    cj = ckks.conjugate(params, keys, ct)
    lo = ckks.add(ct, cj)
    hi = ckks.negate(ckks.mult_monomial(params, ckks.sub(ct, cj), half))
    lo = sine_eval(params, keys, plan, lo)
    hi = sine_eval(params, keys, plan, hi)
    out = ckks.add(lo, ckks.mult_monomial(params, hi, half))
    out = ckks.matvec_stages(params, keys, out, plan.stc)
    assert out.limbs == plan.output_limbs
    return out


__all__ = ["BootstrapPlan", "ChebEvaluator", "MatvecStage", "sine_eval", "bootstrap"]
