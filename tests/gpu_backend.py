"""Adapter: run the parity cases (tests/golden/cases.py) through the GPU product.

Inputs arrive as numpy arrays, are uploaded once, and every operation goes
through the Python mirror -> C ABI -> CUDA kernels.  Outputs are copied back
for comparison against the reference goldens and the oracle.
"""

import numpy as np

from paper_2112_06396_b200 import ckks, rnspoly
from paper_2112_06396_b200.device import to_dev, to_host
from paper_2112_06396_b200.rnspoly import RnsPoly


def _keys(p, keys):
    return ckks.KeySet(p, None, None, rot={r: ckks.SwitchingKey(p.full_moduli, kb, a=ka)
                                           for r, (kb, ka) in keys.items()})


def _ct(p, a, b):
    mods = p.chain[:a.shape[0]]
    return ckks.Ciphertext(RnsPoly(mods, a, "eval"), RnsPoly(mods, b, "eval"), p.delta)


class GpuBackend:
    def ntt(self, x, mods):
        return to_host(rnspoly.ntt_rows(to_dev(x), tuple(mods), False))

    def intt(self, x, mods):
        return to_host(rnspoly.ntt_rows(to_dev(x), tuple(mods), True))

    def ntt_batch(self, xs, mods, inverse):
        """The whole [batch][limbs][N] array in ONE ck_ntt call (batch indexing)."""
        from paper_2112_06396_b200._lib import check, load
        from paper_2112_06396_b200.device import plan_covering, ptr, stream_handle
        x = to_dev(xs)
        B, L, n = x.shape
        plan = plan_covering(tuple(mods), n)
        idx = plan.prime_idx(tuple(mods))
        check(load().ck_ntt(plan.h, ptr(x), ptr(idx), L, B, L * n, int(inverse), stream_handle()),
              "ck_ntt")
        return list(to_host(x))

    def bc_convert(self, x, src, dst):
        return to_host(rnspoly.bc_convert(RnsPoly(src, x, "coeff"), dst).data)

    def bc_convert_centered(self, x, src, dst):
        return to_host(rnspoly.bc_convert_centered(RnsPoly(src, x, "coeff"), dst).data)

    def decomp_modup(self, p, a, mods):
        return [to_host(d.data) for d in ckks._decomp_modup(p, RnsPoly(mods, a, "eval"))]

    def kskip(self, p, digits, kb, ka, limbs):
        raised = p.raised_moduli(limbs)
        key = ckks.SwitchingKey(p.full_moduli, kb, a=ka)
        u, v = ckks._kskip(p, [RnsPoly(raised, d, "eval") for d in digits], key)
        return to_host(u.data), to_host(v.data)

    def moddown_pair(self, p, u, v, limbs):
        raised = p.raised_moduli(limbs)
        du, dv = ckks._moddown_pair(p, RnsPoly(raised, u, "eval"), RnsPoly(raised, v, "eval"), limbs)
        return to_host(du.data), to_host(dv.data)

    def hrotate(self, p, a, b, keys, rots):
        outs = ckks.hrotate(p, _keys(p, keys), _ct(p, a, b), tuple(rots))
        return [(to_host(o.a.data), to_host(o.b.data)) for o in outs]

    def rotate(self, p, a, b, keys, r):
        o = ckks.rotate(p, _keys(p, keys), _ct(p, a, b), r)
        return to_host(o.a.data), to_host(o.b.data)

    def conjugate(self, p, a, b, kb, ka):
        ks = ckks.KeySet(p, None, None, conj=ckks.SwitchingKey(p.full_moduli, kb, a=ka))
        o = ckks.conjugate(p, ks, _ct(p, a, b))
        return to_host(o.a.data), to_host(o.b.data)

    def mult(self, p, ct1, ct2, relin):
        ks = ckks.KeySet(p, None, ckks.SwitchingKey(p.full_moduli, relin[0], a=relin[1]))
        o = ckks.mult(p, ks, _ct(p, *ct1), _ct(p, *ct2))
        return to_host(o.a.data), to_host(o.b.data)

    def new_mult(self, p, ct1, ct2, relin, vm, cres):
        ks = ckks.KeySet(p, None, ckks.SwitchingKey(p.full_moduli, relin[0], a=relin[1]))
        const = 0.0
        if cres is not None:
            integer = int(cres[0])
            const = integer / (p.delta * p.delta)
        o = ckks.new_mult(p, ks, _ct(p, *ct1), _ct(p, *ct2), value_mult=vm, const=const)
        return to_host(o.a.data), to_host(o.b.data)

    def new_mult_add(self, p, ct1, ct2, relin, vm, add, add_delta, sign):
        ks = ckks.KeySet(p, None, ckks.SwitchingKey(p.full_moduli, relin[0], a=relin[1]))
        ad = ckks.Ciphertext(RnsPoly(p.chain[:add[0].shape[0]], add[0], "eval"),
                             RnsPoly(p.chain[:add[1].shape[0]], add[1], "eval"), add_delta)
        o = ckks.new_mult(p, ks, _ct(p, *ct1), _ct(p, *ct2), value_mult=vm, addend=ad,
                          addend_sign=sign)
        return to_host(o.a.data), to_host(o.b.data)

    def pt_matvec(self, p, a, b, keys, diags):
        raised = p.raised_moduli(a.shape[0])
        d = {o: RnsPoly(raised, m, "eval") for o, m in diags.items()}
        o = ckks.pt_matvec(p, _keys(p, keys), _ct(p, a, b), d, p.delta)
        return to_host(o.a.data), to_host(o.b.data)

    def bsgs(self, p, a, b, keys, diags, baby, giant):
        raised = p.raised_moduli(a.shape[0])
        d = {jk: RnsPoly(raised, m, "eval") for jk, m in diags.items()}
        o = ckks.bsgs(p, _keys(p, keys), _ct(p, a, b), d, p.delta, baby, giant)
        return to_host(o.a.data), to_host(o.b.data)


class GpuRotateBackend(GpuBackend):
    """Routes single-rotation hrotate calls through the fused ck_rotate entry."""

    def hrotate(self, p, a, b, keys, rots):
        if len(rots) == 1:
            return [self.rotate(p, a, b, keys, rots[0])]
        return super().hrotate(p, a, b, keys, rots)
