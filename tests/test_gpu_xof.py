"""On-device compressed-key expansion (ck_xof_uniform / ck_expand_key_a) against
the reference goldens of tests/golden/xof.json (make_golden_xof.py)."""

import json
import os

import numpy as np
import pytest
import torch

import cases
import xof_cases
from paper_2112_06396_b200 import _lib, ckks, synth
from paper_2112_06396_b200.device import to_host
from paper_2112_06396_b200.digest import digest
from paper_2112_06396_b200.params import config
from paper_2112_06396_b200.rnspoly import RnsPoly

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLD = json.load(open(os.path.join(HERE, "xof.json")))
ARR = np.load(os.path.join(HERE, "xof.npz"))


@pytest.mark.parametrize("i", range(len(xof_cases.XOF_ROWS)))
def test_xof_row_matches_reference(i):
    seed, tag, q, n = xof_cases.XOF_ROWS[i]
    row = to_host(ckks._xof_uniform(seed, tag, q, n))
    assert digest(row) == GOLD[f"row{i}"]


@pytest.mark.parametrize("name", ["toyA", "C3"])
def test_expand_key_batch_matches_reference(name):
    p = cases.make_params(cases.TOY_A) if name == "toyA" else config("C3").params
    a = ckks.expand_key_a(p, list(xof_cases.KEY_SEEDS))
    for k in range(len(xof_cases.KEY_SEEDS)):
        got = to_host(a[k])
        assert digest(got) == GOLD[f"key_{name}_{k}"], k
        if name == "toyA":
            assert np.array_equal(got, ARR[f"key_toyA_{k}"])


def test_switching_key_from_seed_matches_batch_expansion():
    p = cases.make_params(cases.TOY_A)
    dn = len(p.digit_spans(p.limbs))
    b = np.zeros((dn, len(p.full_moduli), p.n_ring), dtype=np.uint64)
    key = ckks.SwitchingKey(p.full_moduli, b, seed=xof_cases.KEY_SEEDS[1])
    assert np.array_equal(to_host(key.a), ARR["key_toyA_1"])


def test_hrotate_with_compressed_key_matches_reference():
    p = cases.make_params(cases.TOY_A)
    a = cases._rows(p, 0, synth.TAG_CT_A, p.chain)
    b = cases._rows(p, 0, synth.TAG_CT_B, p.chain)
    kb, _ = synth.switching_key(p, cases.SEED, 1005)
    ks = ckks.KeySet(p, None, None,
                     rot={5: ckks.SwitchingKey(p.full_moduli, kb, seed=xof_cases.KEY_SEEDS[0])})
    ct = ckks.Ciphertext(RnsPoly(p.chain, a, "eval"), RnsPoly(p.chain, b, "eval"), p.delta)
    for out in (ckks.hrotate(p, ks, ct, (5,))[0], ckks.rotate(p, ks, ct, 5)):
        assert digest(to_host(out.a.data), to_host(out.b.data)) == GOLD["hrot_compressed_toyA"]


def test_xof_argument_errors():
    lib = _lib.load()
    out = torch.empty(4, dtype=torch.uint64, device="cuda")
    assert lib.ck_xof_uniform(None, None, 0, None, -1, 4, out.data_ptr(), None) == _lib.CK_ERR_ARG
    assert lib.ck_xof_uniform(None, None, 0, None, 1, 4, out.data_ptr(), None) == _lib.CK_ERR_ARG
    assert lib.ck_expand_key_a(None, None, None, 0, 1, None, None) == _lib.CK_ERR_ARG


def test_expand_key_both_kernel_forms_agree():
    """ck_expand_key_a picks one warp per row up to ~3,000 rows and one thread per
    row above: the same keys expanded in a large batch (thread form) and alone
    (warp form) must agree, and the reference-pinned keys sit in both."""
    p = config("C3").params
    seeds = list(xof_cases.KEY_SEEDS) + [b"rot%d" % k + (7).to_bytes(8, "little") for k in range(40)]
    big = ckks.expand_key_a(p, seeds)            # > 40 keys x 96 rows -> thread per row
    for k in (0, 1, 20, len(seeds) - 1):
        small = ckks.expand_key_a(p, [seeds[k]])  # 96 rows -> warp per row
        assert torch.equal(big[k], small[0]), k
    for k in range(len(xof_cases.KEY_SEEDS)):
        assert digest(to_host(big[k])) == GOLD[f"key_C3_{k}"], k
