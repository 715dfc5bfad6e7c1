"""Batched relinearisation (ck_relin, the fused key-switch pipeline with a shared
relin key) bit-exact against the CPU oracle's new_mult relinearisation
(oracle/ckks_np.py, pinned to the reference's ckks.py:639-651)."""

import numpy as np
import pytest
import torch

from oracle import ckks_np
from paper_2112_06396_b200 import synth
from paper_2112_06396_b200._lib import check, load
from paper_2112_06396_b200.device import plan_for, ptr, stream_handle, to_dev, to_host
from paper_2112_06396_b200.params import CkksParams, config, prime_chain_below
from paper_2112_06396_b200.workload import RelinBatch

pytestmark = pytest.mark.gpu


def _oracle_relin(p, a3, b3, c3, kb, ka):
    lim = a3.shape[0]
    mods = p.chain[:lim]
    digits = ckks_np.decomp_modup(p, a3, mods)
    u, v = ckks_np.kskip(p, digits, kb, ka, lim)
    qr = ckks_np._qcol(p.raised_moduli(lim), 2)
    u = ckks_np.addmod(u, ckks_np.pmodup(p, b3, mods), qr)
    v = ckks_np.addmod(v, ckks_np.pmodup(p, c3, mods), qr)
    return ckks_np.moddown_merged(p, u, lim), ckks_np.moddown_merged(p, v, lim)


def _relin(p, x, kb, ka, lim, B):
    plan = plan_for(p)
    n = p.n_ring
    out_a = torch.empty((B, lim - 1, n), dtype=torch.uint64, device="cuda")
    out_b = torch.empty_like(out_a)
    ws = torch.empty(load().ck_relin_workspace_bytes(plan.h, lim, B) // 8, dtype=torch.uint64,
                     device="cuda")
    check(load().ck_relin(plan.h, ptr(x[0]), ptr(x[1]), ptr(x[2]), ptr(kb), ptr(ka), lim,
                          ptr(out_a), ptr(out_b), ptr(ws), B, stream_handle()), "ck_relin")
    return out_a, out_b


@pytest.mark.parametrize("logn,L,K,dnum,lim", [(12, 6, 2, 3, 6), (12, 6, 2, 3, 4), (13, 5, 3, 2, 5),
                                               (6, 5, 3, 2, 5)])
def test_batched_relin_matches_oracle(logn, L, K, dnum, lim):
    chain, special = prime_chain_below(1 << logn, 54, L, 60, K)
    p = CkksParams(logn, chain, special, dnum, 2.0 ** 40, 1)
    B = 3
    mods = p.chain[:lim]
    xs = np.stack([np.stack([synth.uniform_poly(5, u, tag, mods, p.n_ring) for u in range(B)])
                   for tag in (synth.TAG_CT_A, synth.TAG_CT_B, synth.TAG_CT2_A)])
    kb, ka = synth.switching_key(p, 5, 998)
    out_a, out_b = _relin(p, to_dev(xs), to_dev(kb), to_dev(ka), lim, B)
    for u in range(B):
        wa, wb = _oracle_relin(p, xs[0, u], xs[1, u], xs[2, u], kb, ka)
        assert np.array_equal(to_host(out_a[u]), wa), u
        assert np.array_equal(to_host(out_b[u]), wb), u


def test_c3_relin_batch_items_equal_single_calls():
    """C3 (the C3M bench unit): every item of a batch of 5 equals ck_relin on it alone
    (batch 1 is pinned to the reference through the C3_new_mult golden)."""
    p = config("C3M").params
    rb = RelinBatch(p, 20211212, [0, 1, 2, 3, 4])
    rb.run()
    for u in (0, 4):
        x1 = rb.x[:, u:u + 1].contiguous()
        a1, b1 = _relin(p, x1, rb.key_b, rb.key_a, p.limbs, 1)
        assert torch.equal(a1[0], rb.out_a[u]) and torch.equal(b1[0], rb.out_b[u]), u


def test_c3_relin_item_matches_oracle():
    p = config("C3M").params
    rb = RelinBatch(p, 20211212, [7, 8])
    rb.run()
    x = to_host(rb.x[:, 1])
    wa, wb = _oracle_relin(p, x[0], x[1], x[2], to_host(rb.key_b), to_host(rb.key_a))
    assert np.array_equal(to_host(rb.out_a[1]), wa)
    assert np.array_equal(to_host(rb.out_b[1]), wb)
