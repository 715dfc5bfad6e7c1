"""Generate golden fixtures by running the REFERENCE itself (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--only PREFIX] [--skip-big]

Imports ckkslab from /root/reference/pkg/src (read-only), feeds it the seeded
inputs of tests/golden/cases.py through its own public functions
(ckks.hrotate / conjugate / mult / new_mult / pt_matvec, rnspoly NTT and basis
conversions, ckks._decomp_modup / _kskip / _moddown_pair) and writes

    tests/golden/golden.json   {case: sha256 digest of the outputs}
    tests/golden/toy.npz       full outputs of the toy-size cases
    tests/golden/tables.json   digests of reference twiddle tables / psi

The GPU box never runs this (no /root/reference there); it only reads the
committed fixtures.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from ckkslab import ckks, rnspoly  # noqa: E402  (the reference)

import cases  # noqa: E402
from paper_2112_06396_b200.digest import digest  # noqa: E402


def _ref_params(p):
    return ckks.CkksParams(p.logn, tuple(p.chain), tuple(p.special), p.dnum, p.delta, p.seed)


def _poly(mods, data, rep="eval"):
    return rnspoly.RnsPoly(tuple(mods), np.ascontiguousarray(data, dtype=np.uint64), rep)


def _swk(p, kb, ka):
    return ckks.SwitchingKey(tuple(p.full_moduli), kb, seed=None, a=ka)


def _keyset(p, keys=None, conj=None, relin=None):
    rp = _ref_params(p)
    dummy = _poly(p.full_moduli, np.zeros((len(p.full_moduli), p.n_ring), np.uint64))
    ks = ckks.KeySet(rp, dummy, relin if relin is not None else None)
    if keys:
        for r, (kb, ka) in keys.items():
            ks.rot[r] = _swk(p, kb, ka)
    if conj is not None:
        ks.conj = conj
    return ks


class RefBackend:
    def ntt(self, x, mods):
        return np.stack([rnspoly.get_ctx(q, x.shape[1]).ntt(x[i]) for i, q in enumerate(mods)])

    def intt(self, x, mods):
        return np.stack([rnspoly.get_ctx(q, x.shape[1]).intt(x[i]) for i, q in enumerate(mods)])

    def bc_convert(self, x, src, dst):
        return rnspoly.bc_convert(_poly(src, x, "coeff"), tuple(dst)).data

    def bc_convert_centered(self, x, src, dst):
        return rnspoly.bc_convert_centered(_poly(src, x, "coeff"), tuple(dst)).data

    def decomp_modup(self, p, a, mods):
        return [d.data for d in ckks._decomp_modup(_ref_params(p), _poly(mods, a))]

    def kskip(self, p, digits, kb, ka, limbs):
        raised = p.raised_moduli(limbs)
        u, v = ckks._kskip(_ref_params(p), [_poly(raised, d) for d in digits], _swk(p, kb, ka))
        return u.data, v.data

    def moddown_pair(self, p, u, v, limbs):
        raised = p.raised_moduli(limbs)
        du, dv = ckks._moddown_pair(_ref_params(p), _poly(raised, u), _poly(raised, v), limbs)
        return du.data, dv.data

    def _ct(self, p, a, b):
        mods = p.chain[:a.shape[0]]
        return ckks.Ciphertext(_poly(mods, a), _poly(mods, b), p.delta)

    def hrotate(self, p, a, b, keys, rots):
        outs = ckks.hrotate(_ref_params(p), _keyset(p, keys), self._ct(p, a, b), tuple(rots))
        return [(o.a.data, o.b.data) for o in outs]

    def conjugate(self, p, a, b, kb, ka):
        o = ckks.conjugate(_ref_params(p), _keyset(p, conj=_swk(p, kb, ka)), self._ct(p, a, b))
        return o.a.data, o.b.data

    def mult(self, p, ct1, ct2, relin):
        ks = _keyset(p, relin=_swk(p, *relin))
        o = ckks.mult(_ref_params(p), ks, self._ct(p, *ct1), self._ct(p, *ct2))
        return o.a.data, o.b.data

    def new_mult(self, p, ct1, ct2, relin, vm, cres):
        ks = _keyset(p, relin=_swk(p, *relin))
        const = 0.0
        if cres is not None:
            # encode_const rounds const*delta1*delta2 (ckks.py:530-537); choose
            # const so that the rounded integer is exactly the case's integer
            c1, c2 = self._ct(p, *ct1), self._ct(p, *ct2)
            integer = cres_integer(p, cres)
            const = integer / (c1.delta * c2.delta)
            assert round(const * c1.delta * c2.delta) == integer
        o = ckks.new_mult(_ref_params(p), ks, self._ct(p, *ct1), self._ct(p, *ct2),
                          value_mult=vm, const=const)
        return o.a.data, o.b.data

    def new_mult_add(self, p, ct1, ct2, relin, vm, add, add_delta, sign):
        ks = _keyset(p, relin=_swk(p, *relin))
        ad = ckks.Ciphertext(_poly(p.chain[:add[0].shape[0]], add[0]),
                             _poly(p.chain[:add[1].shape[0]], add[1]), add_delta)
        o = ckks.new_mult(_ref_params(p), ks, self._ct(p, *ct1), self._ct(p, *ct2),
                          value_mult=vm, addend=ad, addend_sign=sign)
        return o.a.data, o.b.data

    def pt_matvec(self, p, a, b, keys, diags):
        raised = p.raised_moduli(a.shape[0])
        d = {o: _poly(raised, m) for o, m in diags.items()}
        o = ckks.pt_matvec(_ref_params(p), _keyset(p, keys), self._ct(p, a, b), d, p.delta)
        return o.a.data, o.b.data

    def bsgs(self, p, a, b, keys, diags, baby, giant):
        """Oracle form of a19: sum_j rotate(pt_matvec(ct, group_j), -baby*j)."""
        rp = _ref_params(p)
        ks = _keyset(p, keys)
        ct = self._ct(p, a, b)
        raised = p.raised_moduli(a.shape[0])
        acc = None
        for j in range(1, giant + 1):
            grp = {k: _poly(raised, diags[(j, k)]) for k in range(1, baby + 1)}
            mv = ckks.pt_matvec(rp, ks, ct, grp, p.delta)
            rj = ckks.rotate(rp, ks, mv, -baby * j)
            acc = rj if acc is None else ckks.add(acc, rj)
        return acc.a.data, acc.b.data


def cres_integer(p, cres):
    """The small integer whose residues are cres (cases use const < all q)."""
    vals = set(int(c) for c in cres)
    assert len(vals) == 1
    return vals.pop()


def table_digests():
    from paper_2112_06396_b200.params import config
    out = {}
    for name in ("C1", "C3", "C5"):
        p = config(name).params
        for q in p.full_moduli:
            ctx = rnspoly.get_ctx(q, p.n_ring)
            out[f"{p.n_ring}:{q}"] = {"psi": int(ctx.psi), "tw": digest(ctx.tw),
                                      "itw": digest(ctx.itw), "n_inv": int(ctx.n_inv)}
    # eval-domain automorphism permutations (empirical, rnspoly.py:127-135)
    perms = {}
    for logn in (5, 6, 12):
        n = 1 << logn
        q = cases.make_params(cases.TOY_C).chain[0] if logn == 5 else None
        from paper_2112_06396_b200.params import ntt_prime_below
        q = ntt_prime_below(50, n)
        ctx = rnspoly.get_ctx(q, n)
        for t in (5, 25, 2 * n - 1, pow(5, -3, 2 * n), 77 % (2 * n) | 1):
            rnspoly._AUTO_EVAL_CACHE.clear()
            perms[f"{n}:{t}"] = digest(rnspoly.automorph_eval_perm(n, t, ctx).astype(np.uint64))
    return out, perms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--skip-big", action="store_true")
    args = ap.parse_args()
    gpath = os.path.join(HERE, "golden.json")
    golden = json.load(open(gpath)) if os.path.exists(gpath) else {}
    npz_path = os.path.join(HERE, "toy.npz")
    toy = dict(np.load(npz_path)) if os.path.exists(npz_path) else {}
    be = RefBackend()
    if args.only is None or args.only == "tables":
        tw, perms = table_digests()
        json.dump({"tables": tw, "perms": perms}, open(os.path.join(HERE, "tables.json"), "w"),
                  indent=1, sort_keys=True)
        print("tables done", flush=True)
    for case in cases.all_cases():
        if args.only and not case.name.startswith(args.only):
            continue
        if args.skip_big and case.pspec[0] == "cfg" and case.pspec[1] in ("C4", "C5"):
            continue
        t0 = time.time()
        out = cases.run_case(case, be)
        golden[case.name] = {"digest": digest(*out), "shapes": [list(o.shape) for o in out]}
        if case.full:
            for i, o in enumerate(out):
                toy[f"{case.name}/{i}"] = o
        print(f"{case.name}: {time.time() - t0:.1f}s", flush=True)
        json.dump(golden, open(gpath, "w"), indent=1, sort_keys=True)
        np.savez_compressed(npz_path, **toy)


if __name__ == "__main__":
    main()
