"""Host parameter plumbing vs the reference (psi, twiddles, primes, generator)."""

import json
import os

import numpy as np

import cases
from oracle import ckks_np
from paper_2112_06396_b200 import params, synth
from paper_2112_06396_b200.digest import digest

TABLES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tables.json")))


def test_primes_are_largest_below_bound():
    for name in ("C1", "C3", "C5"):
        p = params.config(name).params
        n = p.n_ring
        for q in p.full_moduli:
            assert params.is_prime(q) and q % (2 * n) == 1 and q < 2 ** 60
        assert len(set(p.full_moduli)) == len(p.full_moduli)
        top = p.chain[0]
        bits = top.bit_length()
        # nothing between chain[0] and 2^bits qualifies
        step = 2 * n
        c = ((1 << bits) - 1) // step * step + 1
        while c > top:
            assert not params.is_prime(c)
            c -= step


def test_psi_and_tables_match_reference():
    """psi (smallest primitive root rule, zq.py:79-84) and bit-reversed twiddles."""
    for name in ("C1", "C3", "C5"):
        p = params.config(name).params
        for q in p.full_moduli:
            ref = TABLES["tables"][f"{p.n_ring}:{q}"]
            assert params.primitive_root_2n(q, p.n_ring) == ref["psi"]
            if p.n_ring <= 1 << 16 and q == p.full_moduli[0]:
                tw, itw, ninv = ckks_np.twiddles(q, p.n_ring)
                assert digest(tw) == ref["tw"] and digest(itw) == ref["itw"]
                assert ninv == ref["n_inv"]


def test_automorph_closed_form_matches_reference_permutation():
    for key, d in TABLES["perms"].items():
        n, t = map(int, key.split(":"))
        assert digest(ckks_np.automorph_perm(n, t).astype(np.uint64)) == d


def test_smallest_primitive_root_matches_sympy():
    import sympy
    for q in params.config("C3").params.full_moduli[:6]:
        assert params.smallest_primitive_root(q) == sympy.primitive_root(q)


def test_galois_exponents_distinct_in_range():
    ks = params.galois_exponents(1 << 16, 64, cases.SEED)
    assert len(set(ks)) == 64 and all(1 <= k < (1 << 15) for k in ks)


def test_uniform_generator_in_range_and_deterministic():
    q = params.config("C3").params.special[0]
    a = synth.uniform_row(7, 3, q, 4096)
    b = synth.uniform_row(7, 3, q, 4096)
    assert np.array_equal(a, b) and int(a.max()) < q
    # scalar twin
    key = synth.stream_key(7, 3)
    for k in (0, 1, 4095):
        x = synth.splitmix64_scalar((key + k) % 2 ** 64)
        assert int(a[k]) == (x * q) >> 64
    # roughly uniform
    assert abs(float(a.astype(np.float64).mean()) / q - 0.5) < 0.02
