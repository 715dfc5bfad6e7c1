"""Extreme residues on the GPU, bit-exact against the oracle.

Uniform random inputs rarely reach the worst cases of the lazy reductions
(NTT butterflies in [0, 16q), the byte-sliced tensor-core contractions whose
plane sums are bounded by 255^2 per term, the FP64-quotient epilogues, the
30-bit-split MAC accumulators).  These tests drive every kernel of the fused
key-switch with all-(q-1) residues, all zeros and a mixed 0 / q-1 / 1 pattern,
at the benchmark shapes (C3, C1) and through the NTT at C2 and C5 sizes.
"""

import numpy as np
import pytest
import torch

from oracle import ckks_np
from paper_2112_06396_b200 import ckks, rnspoly
from paper_2112_06396_b200.device import to_dev, to_host
from paper_2112_06396_b200.params import config
from paper_2112_06396_b200.rnspoly import RnsPoly

pytestmark = pytest.mark.gpu

PATTERNS = ["max", "zero", "mixed"]


def _fill(mods, n, pattern, salt=0):
    out = np.empty((len(mods), n), dtype=np.uint64)
    for i, q in enumerate(mods):
        if pattern == "max":
            out[i] = q - 1
        elif pattern == "zero":
            out[i] = 0
        else:  # q-1 / 0 / 1 / q-2 cycling, shifted per limb and per operand
            cyc = np.array([q - 1, 0, 1, q - 2], dtype=np.uint64)
            out[i] = cyc[(np.arange(n) + i + salt) % 4]
    return out


def _key(p, pattern, salt):
    dn = len(p.digit_spans(p.limbs))
    full = p.full_moduli
    kb = np.stack([_fill(full, p.n_ring, pattern, salt + 10 * j) for j in range(dn)])
    ka = np.stack([_fill(full, p.n_ring, pattern, salt + 10 * j + 5) for j in range(dn)])
    return kb, ka


@pytest.mark.parametrize("cfg,pattern", [(c, pt) for c in ("C1", "C3") for pt in PATTERNS] +
                         [("C5", "max"), ("C5", "mixed")])
def test_rotation_extremes(cfg, pattern):
    p = config(cfg).params
    a = _fill(p.chain, p.n_ring, pattern, 1)
    b = _fill(p.chain, p.n_ring, pattern, 2)
    kb, ka = _key(p, pattern, 3)
    want_a, want_b = ckks_np.rotate(p, a, b, {-1: (kb, ka)}, -1)
    # mirror API (hoisted path) ...
    keys = ckks.KeySet(p, None, None, rot={-1: ckks.SwitchingKey(p.full_moduli, kb, a=ka)})
    ct = ckks.Ciphertext(RnsPoly(p.chain, a, "eval"), RnsPoly(p.chain, b, "eval"), p.delta)
    out = ckks.rotate(p, keys, ct, -1)
    assert np.array_equal(to_host(out.a.data), want_a)
    assert np.array_equal(to_host(out.b.data), want_b)
    # ... and the fused batched benchmark entry (ck_rotate)
    gal = torch.tensor([pow(5, 1, 2 * p.n_ring)], dtype=torch.uint64, device="cuda")
    oa = torch.empty((1, p.limbs, p.n_ring), dtype=torch.uint64, device="cuda")
    ob = torch.empty_like(oa)
    ckks.rotate_batch(p, to_dev(a[None]), to_dev(b[None]), to_dev(kb[None]), to_dev(ka[None]),
                      gal, oa, ob)
    assert np.array_equal(to_host(oa[0]), want_a)
    assert np.array_equal(to_host(ob[0]), want_b)


@pytest.mark.parametrize("cfg", ["C2", "C5"])
@pytest.mark.parametrize("pattern", PATTERNS)
def test_ntt_extremes(cfg, pattern):
    p = config(cfg).params
    mods = tuple(p.chain[:4]) + tuple(p.special[:2])
    x = _fill(mods, p.n_ring, pattern, 7)
    fwd = to_host(rnspoly.ntt_rows(to_dev(x), mods, False))
    assert np.array_equal(fwd, ckks_np.ntt(x, mods))
    inv = to_host(rnspoly.ntt_rows(to_dev(x), mods, True))
    assert np.array_equal(inv, ckks_np.intt(x, mods))
