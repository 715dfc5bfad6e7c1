"""Parity cases shared by the golden generator, the oracle test and the GPU tests.

Every case is fully determined by (params spec, seed, op, args); inputs are
regenerated from the counter-based generator in paper_2112_06396_b200.synth,
so the fixtures only store outputs (full arrays for toy sizes, sha256
digests for everything).

A *backend* is any object with the methods used below (``ntt``, ``intt``,
``bc_convert``, ``bc_convert_centered``, ``decomp_modup``, ``kskip``,
``moddown_pair``, ``hrotate``, ``conjugate``, ``mult``, ``new_mult``,
``pt_matvec``, ``bsgs``), taking and returning numpy uint64 arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2112_06396_b200 import synth
from paper_2112_06396_b200.params import CkksParams, config, galois_exponents, prime_chain_below

SEED = 20211212


@dataclass(frozen=True)
class Case:
    name: str
    pspec: tuple           # ("toy", logn, chain_bits, L, special_bits, K, dnum) or ("cfg", "C3")
    op: str
    args: tuple = ()
    full: bool = False     # store full output arrays (toy sizes only)


def make_params(pspec) -> CkksParams:
    if pspec[0] == "cfg":
        return config(pspec[1]).params
    _, logn, cb, L, sb, K, dnum = pspec
    chain, special = prime_chain_below(1 << logn, cb, L, sb, K)
    return CkksParams(logn, chain, special, dnum, float(2 ** 40), 1)


TOY_A = ("toy", 6, 50, 5, 60, 3, 2)      # alpha=3, spans (0,3),(3,5)
TOY_B = ("toy", 7, 54, 6, 60, 2, 3)      # alpha=2
TOY_C = ("toy", 5, 50, 4, 51, 1, 4)      # alpha=1 (C1 shape)
TOY_D = ("toy", 8, 54, 6, 60, 2, 3)


def _toy_cases():
    out = []
    for tag, ps in (("A", TOY_A), ("B", TOY_B), ("C", TOY_C), ("D", TOY_D)):
        out += [
            Case(f"{tag}_ntt", ps, "ntt", (), True),
            Case(f"{tag}_intt", ps, "intt", (), True),
            Case(f"{tag}_bc", ps, "bc_convert", (), True),
            Case(f"{tag}_bcc", ps, "bc_convert_centered", (), True),
            Case(f"{tag}_bcc_edge", ps, "bc_centered_edge", (), True),
            Case(f"{tag}_modup", ps, "decomp_modup", (None,), True),
            Case(f"{tag}_modup_lo", ps, "decomp_modup", (-1,), True),
            Case(f"{tag}_kskip", ps, "kskip", (None,), True),
            Case(f"{tag}_moddown", ps, "moddown_pair", (None,), True),
            Case(f"{tag}_hrot", ps, "hrotate", ((1, -1, 3, -7), None), True),
            Case(f"{tag}_hrot_lo", ps, "hrotate", ((2, -5), -1), True),
            Case(f"{tag}_conj", ps, "conjugate", (None,), True),
            Case(f"{tag}_mult", ps, "mult", (), True),
            Case(f"{tag}_new_mult", ps, "new_mult", (1, None), True),
            Case(f"{tag}_new_mult_vc", ps, "new_mult", (3, 12345), True),
            Case(f"{tag}_new_mult_add", ps, "new_mult_add", (1, 1, 0), True),
            Case(f"{tag}_new_mult_sub_lo", ps, "new_mult_add", (5, -1, 1), True),
            Case(f"{tag}_matvec", ps, "pt_matvec", ((0, 1, 3, 5),), True),
        ]
    out.append(Case("B_bsgs", TOY_B, "bsgs", (4, 2), True))
    out.append(Case("D_bsgs", TOY_D, "bsgs", (3, 3), True))
    # more than 32 diagonals / baby steps (chunked accumulation): a radix-32
    # CoeffToSlot stage has 2*32-1 = 63 diagonals (bootstrap.py:128-133)
    out.append(Case("B_matvec63", TOY_B, "pt_matvec", (tuple(range(-31, 32)),), True))
    out.append(Case("D_bsgs40", TOY_D, "bsgs", (40, 2), True))
    return out


def full_cases():
    c3k = galois_exponents(1 << 16, 64, SEED)
    c5k = galois_exponents(1 << 17, 256, SEED)
    return [
        Case("C1_rot", ("cfg", "C1"), "rotate_k", (0, 1)),
        Case("C2_ntt", ("cfg", "C2"), "ntt", ()),
        Case("C2_intt", ("cfg", "C2"), "intt", ()),
        # the whole C2 batch (16 polynomials x 24 limbs) forward and inverse
        Case("C2_ntt_b16", ("cfg", "C2"), "ntt_batch", (16, False)),
        Case("C2_intt_b16", ("cfg", "C2"), "ntt_batch", (16, True)),
        Case("C3_rot0", ("cfg", "C3"), "rotate_k", (0, c3k[0])),
        Case("C3_rot1", ("cfg", "C3"), "rotate_k", (1, c3k[1])),
        Case("C3_rot63", ("cfg", "C3"), "rotate_k", (63, c3k[63])),
        Case("C3_conj", ("cfg", "C3"), "conjugate", (None,)),
        # hoisted: the 16 baby rotations of C4 (k = 1..16) from one shared ModUp
        Case("C3_hrot16", ("cfg", "C3"), "hrotate", (tuple(-k for k in range(1, 17)), None)),
        Case("C3_new_mult", ("cfg", "C3"), "new_mult", (1, None)),
        Case("C4_bsgs", ("cfg", "C4"), "bsgs", (16, 8)),
        Case("C5_rot0", ("cfg", "C5"), "rotate_k", (0, c5k[0])),
        Case("C5_rot255", ("cfg", "C5"), "rotate_k", (255, c5k[255])),
    ]


def all_cases():
    return _toy_cases() + full_cases()


# ------------------------------------------------------------------ inputs

def _rows(p: CkksParams, unit: int, tag: int, mods, digit: int = 0, rows=None):
    return synth.uniform_poly(SEED, unit, tag, mods, p.n_ring, digit=digit, rows=rows)


ADDEND_DELTA = float(2 ** 30)  # ct deltas are 2^40: lift = round(2^80 / 2^30) = 2^50


def _level(p: CkksParams, lv):
    return p.limbs if lv is None else p.limbs + lv


def _keys(p: CkksParams, rs):
    """{r: (key_b, key_a)} with a distinct generator unit per rotation r."""
    return {r: synth.switching_key(p, SEED, 1000 + (r % (4 * p.n_ring))) for r in rs}


def edge_inputs(p: CkksParams, src, count: int = 16):
    """Coefficients sitting on the centered-rounding boundary (x ~ Q/2, k*Q+Q/2)."""
    big_q = 1
    for q in src:
        big_q *= q
    vals = []
    for i in range(count):
        base = (big_q // 2) if i % 2 == 0 else (big_q * (i % len(src) + 1) // 2)
        vals.append(base + (i // 2 - count // 4))
    rng_fill = synth.uniform_poly(SEED, 7, synth.TAG_NTT, src, p.n_ring)
    x = rng_fill.copy()
    for c, v in enumerate(vals):
        for i, q in enumerate(src):
            x[i, c] = v % q
    return x


def run_case(case: Case, be):
    """Execute one case on backend `be`; returns a tuple of uint64 arrays."""
    p = make_params(case.pspec)
    n = p.n_ring
    full = p.full_moduli
    op = case.op
    if op in ("ntt", "intt"):
        mods = full if case.pspec[0] == "toy" else p.chain
        x = _rows(p, 0, synth.TAG_NTT, mods)
        return (be.ntt(x, mods) if op == "ntt" else be.intt(x, mods),)
    if op == "ntt_batch":
        units, inverse = case.args
        xs = np.stack([_rows(p, u, synth.TAG_NTT, p.chain) for u in range(units)])
        if hasattr(be, "ntt_batch"):
            return tuple(be.ntt_batch(xs, p.chain, inverse))
        f = be.intt if inverse else be.ntt
        return tuple(f(x, p.chain) for x in xs)
    if op == "bc_convert":
        src, dst = p.chain[:p.alpha], p.chain[p.alpha:] + p.special
        return (be.bc_convert(_rows(p, 0, synth.TAG_NTT, src), src, dst),)
    if op == "bc_convert_centered":
        src, dst = p.special, p.chain
        return (be.bc_convert_centered(_rows(p, 0, synth.TAG_NTT, src), src, dst),)
    if op == "bc_centered_edge":
        src, dst = p.special + p.chain[-1:], p.chain[:-1]
        return (be.bc_convert_centered(edge_inputs(p, src), src, dst),)
    if op == "decomp_modup":
        lim = _level(p, case.args[0])
        a = _rows(p, 0, synth.TAG_CT_A, p.chain[:lim])
        return tuple(be.decomp_modup(p, a, p.chain[:lim]))
    if op in ("kskip", "moddown_pair"):
        lim = _level(p, case.args[0])
        raised = p.raised_moduli(lim)
        ndig = len(p.digit_spans(lim))
        if op == "kskip":
            digits = [_rows(p, 0, synth.TAG_CT_A, raised, digit=j) for j in range(ndig)]
            kb, ka = synth.switching_key(p, SEED, 0)
            return be.kskip(p, digits, kb, ka, lim)
        u = _rows(p, 0, synth.TAG_CT_A, raised)
        v = _rows(p, 0, synth.TAG_CT_B, raised)
        return be.moddown_pair(p, u, v, lim)
    if op == "hrotate":
        rots, lv = case.args
        lim = _level(p, lv)
        a = _rows(p, 0, synth.TAG_CT_A, p.chain[:lim])
        b = _rows(p, 0, synth.TAG_CT_B, p.chain[:lim])
        outs = be.hrotate(p, a, b, _keys(p, rots), rots)
        return tuple(x for pair in outs for x in pair)
    if op == "rotate_k":
        unit, k = case.args
        a, b, kb, ka = synth.rotation_inputs(p, SEED, unit)
        return tuple(be.hrotate(p, a, b, {-k: (kb, ka)}, (-k,))[0])
    if op == "conjugate":
        lim = _level(p, case.args[0])
        a = _rows(p, 0, synth.TAG_CT_A, p.chain[:lim])
        b = _rows(p, 0, synth.TAG_CT_B, p.chain[:lim])
        kb, ka = synth.switching_key(p, SEED, 999)
        return tuple(be.conjugate(p, a, b, kb, ka))
    if op in ("mult", "new_mult"):
        mods = p.chain
        ct1 = (_rows(p, 0, synth.TAG_CT_A, mods), _rows(p, 0, synth.TAG_CT_B, mods))
        ct2 = (_rows(p, 0, synth.TAG_CT2_A, mods), _rows(p, 0, synth.TAG_CT2_B, mods))
        relin = synth.switching_key(p, SEED, 998)
        if op == "mult":
            return tuple(be.mult(p, ct1, ct2, relin))
        vm, const = case.args
        cres = None if const is None else [const % q for q in mods]
        return tuple(be.new_mult(p, ct1, ct2, relin, vm, cres))
    if op == "new_mult_add":
        # addend folded in after an integer scale lift (ckks.py:624-636); ct2 may
        # sit `drop` limbs lower (lim = min, drop_limbs on ct1 and the addend)
        vm, sign, drop = case.args
        mods = p.chain
        ct1 = (_rows(p, 0, synth.TAG_CT_A, mods), _rows(p, 0, synth.TAG_CT_B, mods))
        m2 = mods[:len(mods) - drop]
        ct2 = (_rows(p, 0, synth.TAG_CT2_A, m2), _rows(p, 0, synth.TAG_CT2_B, m2))
        add = (_rows(p, 3, synth.TAG_CT_A, mods), _rows(p, 3, synth.TAG_CT_B, mods))
        relin = synth.switching_key(p, SEED, 998)
        return tuple(be.new_mult_add(p, ct1, ct2, relin, vm, add, ADDEND_DELTA, sign))
    if op == "pt_matvec":
        offs = case.args[0]
        mods = p.chain
        raised = p.raised_moduli(p.limbs)
        a = _rows(p, 0, synth.TAG_CT_A, mods)
        b = _rows(p, 0, synth.TAG_CT_B, mods)
        diags = {o: _rows(p, 0, synth.TAG_DIAG, raised, digit=o) for o in offs}
        keys = _keys(p, [-o for o in offs if o % p.slots])
        return tuple(be.pt_matvec(p, a, b, keys, diags))
    if op == "bsgs":
        baby, giant = case.args
        mods = p.chain
        raised = p.raised_moduli(p.limbs)
        a = _rows(p, 0, synth.TAG_CT_A, mods)
        b = _rows(p, 0, synth.TAG_CT_B, mods)
        diags = {(j, k): _rows(p, j, synth.TAG_DIAG, raised, digit=k)
                 for j in range(1, giant + 1) for k in range(1, baby + 1)}
        rs = sorted({-k for k in range(1, baby + 1)} | {-baby * j for j in range(1, giant + 1)})
        return tuple(be.bsgs(p, a, b, _keys(p, rs), diags, baby, giant))
    raise KeyError(op)


class OracleBackend:
    """The numpy restatement in oracle/ (test infrastructure)."""

    def new_mult_add(self, p, ct1, ct2, relin, vm, add, add_delta, sign):
        from oracle import ckks_np
        lift = sign * round(p.delta * p.delta / add_delta)  # ckks.py:632-634
        return ckks_np.new_mult(p, ct1, ct2, relin, vm, None, addend=(add[0], add[1], lift))

    def __getattr__(self, name):
        from oracle import ckks_np
        if name == "moddown_pair":
            return ckks_np.moddown_pair
        return getattr(ckks_np, name)
