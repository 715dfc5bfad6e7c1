"""ck_keyswitch (SURVEY 8(b)'s single key-switch entry): every mode equals the
dedicated entry it dispatches to -- mode 0/1 == ck_rotate (pinned to the
reference through the C*_rot / conj goldens), mode 2 with (b3, c3) interleaved
per item == ck_relin and the oracle relinearisation (ckks.py:639-651)."""

import numpy as np
import pytest
import torch

from paper_2112_06396_b200 import synth
from paper_2112_06396_b200._lib import check, load
from paper_2112_06396_b200.device import plan_for, ptr, stream_handle, to_dev, to_host
from paper_2112_06396_b200.params import CkksParams, prime_chain_below

from test_gpu_relin import _oracle_relin, _relin

pytestmark = pytest.mark.gpu


def _params(logn=12, L=6, K=2, dnum=3):
    chain, special = prime_chain_below(1 << logn, 54, L, 60, K)
    return CkksParams(logn, chain, special, dnum, 2.0 ** 40, 1)


def _ws(plan, lim, mode, B):
    nbytes = load().ck_keyswitch_workspace_bytes(plan.h, lim, mode, B)
    assert nbytes > 0
    return torch.empty(nbytes // 8, dtype=torch.uint64, device="cuda")


def _ks(p, a, b, kb, ka, lim, t, mode, B, out_rows):
    plan = plan_for(p)
    n = p.n_ring
    out_a = torch.empty((B, out_rows, n), dtype=torch.uint64, device="cuda")
    out_b = torch.empty_like(out_a)
    ws = _ws(plan, lim, mode, B)
    check(load().ck_keyswitch(plan.h, ptr(a), ptr(b), ptr(kb), ptr(ka), lim, t, None, mode,
                              ptr(out_a), ptr(out_b), ptr(ws), B, stream_handle()), "ck_keyswitch")
    return out_a, out_b


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("lim", [6, 3])
def test_keyswitch_rotation_modes_equal_ck_rotate(mode, lim):
    p = _params()
    n = p.n_ring
    B = 2
    mods = p.chain[:lim]
    a = to_dev(np.stack([synth.uniform_poly(9, u, synth.TAG_CT_A, mods, n) for u in range(B)]))
    b = to_dev(np.stack([synth.uniform_poly(9, u, synth.TAG_CT_B, mods, n) for u in range(B)]))
    # modes 0/1: one switching key per batch item ([batch][dnum][L+K][N])
    keys = [synth.switching_key(p, 9, 17 + u) for u in range(B)]
    kb = to_dev(np.stack([k[0] for k in keys]))
    ka = to_dev(np.stack([k[1] for k in keys]))
    t = (2 * n - 1) if mode == 1 else pow(5, 3, 2 * n)
    ga, gb = _ks(p, a, b, kb, ka, lim, t, mode, B, lim)
    plan = plan_for(p)
    ra, rb = torch.empty_like(ga), torch.empty_like(gb)
    ws = plan.workspace(lim, B)
    check(load().ck_rotate(plan.h, ptr(a), ptr(b), ptr(kb), ptr(ka), lim, t, None, mode, ptr(ra),
                           ptr(rb), ptr(ws), B, stream_handle()), "ck_rotate")
    assert torch.equal(ga, ra) and torch.equal(gb, rb)


@pytest.mark.parametrize("lim", [6, 2])
def test_keyswitch_relin_mode_interleaved(lim):
    p = _params()
    n = p.n_ring
    B = 3
    mods = p.chain[:lim]
    xs = np.stack([np.stack([synth.uniform_poly(4, u, tag, mods, n) for u in range(B)])
                   for tag in (synth.TAG_CT_A, synth.TAG_CT_B, synth.TAG_CT2_A)])
    kb, ka = synth.switching_key(p, 4, 998)
    a3 = to_dev(xs[0])
    bc = to_dev(np.ascontiguousarray(np.stack([xs[1], xs[2]], axis=1)))   # [B][2][lim][N]
    ga, gb = _ks(p, a3, bc, to_dev(kb), to_dev(ka), lim, 1, 2, B, lim - 1)
    ra, rb = _relin(p, to_dev(xs), to_dev(kb), to_dev(ka), lim, B)
    assert torch.equal(ga, ra) and torch.equal(gb, rb)
    wa, wb = _oracle_relin(p, xs[0, 1], xs[1, 1], xs[2, 1], kb, ka)
    assert np.array_equal(to_host(ga[1]), wa) and np.array_equal(to_host(gb[1]), wb)


def test_keyswitch_rejects_bad_mode():
    p = _params()
    plan = plan_for(p)
    assert load().ck_keyswitch_workspace_bytes(plan.h, 4, 7, 1) == 0
    assert load().ck_keyswitch(plan.h, None, None, None, None, 4, 1, None, 7, None, None, None, 1,
                               None) == -1
