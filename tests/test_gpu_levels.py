"""Fused ck_rotate / conjugate at levels below the top, batched, and error behaviour.

The reference supports key-switching at any level l <= L (ckks.py:421-465 use
the digit spans and key rows of level l).  The oracle is pinned to the
reference at the top level and at l-1 (tests/test_oracle_golden.py); here the
GPU fused path is checked against it at several levels and batch sizes.
"""

import numpy as np
import pytest
import torch

import cases
import gpu_backend
from oracle import ckks_np
from paper_2112_06396_b200 import ckks, synth
from paper_2112_06396_b200.device import plan_for, to_dev, to_host
from paper_2112_06396_b200.params import CkksParams, config, prime_chain_below
from paper_2112_06396_b200.rnspoly import RnsPoly

pytestmark = pytest.mark.gpu


def _params(logn, L, K, dnum, cb=54, sb=60):
    chain, special = prime_chain_below(1 << logn, cb, L, sb, K)
    return CkksParams(logn, chain, special, dnum, 2.0 ** 40, 1)


@pytest.mark.parametrize("logn,L,K,dnum,level", [
    (12, 6, 2, 3, 6), (12, 6, 2, 3, 5), (12, 6, 2, 3, 1), (13, 7, 3, 2, 4),
    (14, 5, 5, 1, 3), (16, 24, 8, 3, 23), (16, 24, 8, 3, 17)])
def test_fused_rotate_below_top_level(logn, L, K, dnum, level):
    p = _params(logn, L, K, dnum)
    a, b, kb, ka = synth.rotation_inputs(p, 77, 0, limbs=level)
    k = 9
    t = pow(5, k, 2 * p.n_ring)
    want_a, want_b = ckks_np.rotate_galois(p, a, b, kb, ka, t)
    ks = ckks.KeySet(p, None, None, rot={-k: ckks.SwitchingKey(p.full_moduli, kb, a=ka)})
    ct = ckks.Ciphertext(RnsPoly(p.chain[:level], a, "eval"), RnsPoly(p.chain[:level], b, "eval"), 1.0)
    out = ckks.rotate(p, ks, ct, -k)
    assert np.array_equal(to_host(out.a.data), want_a)
    assert np.array_equal(to_host(out.b.data), want_b)


@pytest.mark.parametrize("level", [23, 17])
def test_fused_rotate_repeatable(level):
    """The same single key-switch eight times on a nearly empty GPU: ks_row's key stage is
    refilled by a TMA bulk copy as soon as the key words are in registers; without the proxy
    fence before that refill the copy overtook in-flight shared-memory loads and these
    launches (not the full batches) produced sporadic mismatches."""
    p = _params(16, 24, 8, 3)
    a, b, kb, ka = synth.rotation_inputs(p, 77, 0, limbs=level)
    k = 9
    want_a, want_b = ckks_np.rotate_galois(p, a, b, kb, ka, pow(5, k, 2 * p.n_ring))
    ks = ckks.KeySet(p, None, None, rot={-k: ckks.SwitchingKey(p.full_moduli, kb, a=ka)})
    ct = ckks.Ciphertext(RnsPoly(p.chain[:level], a, "eval"), RnsPoly(p.chain[:level], b, "eval"), 1.0)
    for _ in range(8):
        out = ckks.rotate(p, ks, ct, -k)
        assert np.array_equal(to_host(out.a.data), want_a)
        assert np.array_equal(to_host(out.b.data), want_b)


@pytest.mark.parametrize("batch", [1, 3, 5])
def test_batched_rotate_distinct_galois_small_ring(batch):
    p = _params(12, 6, 2, 3)
    units = list(range(batch))
    ins = [synth.rotation_inputs(p, 5, u) for u in units]
    ks = [3 + 2 * u for u in units]
    a = to_dev(np.stack([x[0] for x in ins])); b = to_dev(np.stack([x[1] for x in ins]))
    kb = to_dev(np.stack([x[2] for x in ins])); ka = to_dev(np.stack([x[3] for x in ins]))
    gal = torch.tensor(np.array([pow(5, k, 2 * p.n_ring) for k in ks], dtype=np.uint64), device="cuda")
    oa, ob = torch.empty_like(a), torch.empty_like(b)
    ckks.rotate_batch(p, a, b, kb, ka, gal, oa, ob)
    for i, (x, k) in enumerate(zip(ins, ks)):
        wa, wb = ckks_np.rotate_galois(p, *x, pow(5, k, 2 * p.n_ring))
        assert np.array_equal(to_host(oa[i]), wa) and np.array_equal(to_host(ob[i]), wb)


def test_conjugate_below_top_level():
    p = _params(13, 6, 2, 3)
    level = 4
    a, b, kb, ka = synth.rotation_inputs(p, 3, 1, limbs=level)
    want = ckks_np.conjugate(p, a, b, kb, ka)
    ks = ckks.KeySet(p, None, None, conj=ckks.SwitchingKey(p.full_moduli, kb, a=ka))
    ct = ckks.Ciphertext(RnsPoly(p.chain[:level], a, "eval"), RnsPoly(p.chain[:level], b, "eval"), 1.0)
    out = ckks.conjugate(p, ks, ct)
    assert np.array_equal(to_host(out.a.data), want[0]) and np.array_equal(to_host(out.b.data), want[1])


def test_error_behaviour_matches_reference():
    p = _params(12, 4, 1, 4)
    a, b, kb, ka = synth.rotation_inputs(p, 1, 0)
    ks = ckks.KeySet(p, None, None, rot={-1: ckks.SwitchingKey(p.full_moduli, kb, a=ka)})
    ct = ckks.Ciphertext(RnsPoly(p.chain, a, "eval"), RnsPoly(p.chain, b, "eval"), 1.0)
    with pytest.raises(KeyError):               # missing rotation key (ckks.py:664)
        ckks.hrotate(p, ks, ct, (5,))
    x = RnsPoly(p.chain, a, "eval")
    y = RnsPoly(p.chain[:3], a[:3], "eval")
    with pytest.raises(AssertionError):         # basis mismatch (rnspoly.py:174)
        x.add(y)
    with pytest.raises(AssertionError):         # rep mismatch
        x.add(RnsPoly(p.chain, a, "coeff"))
    with pytest.raises(AssertionError):         # mul needs eval rep (rnspoly.py:199)
        RnsPoly(p.chain, a, "coeff").mul(RnsPoly(p.chain, a, "coeff"))
    from paper_2112_06396_b200 import _lib
    lib = _lib.load()
    plan = plan_for(p)
    assert lib.ck_rotate(plan.h, None, None, None, None, 0, 1, None, 0, None, None, None, 1, None) == -1
    assert lib.ck_workspace_bytes(plan.h, 99, 1) == 0


def test_plan_rejects_bad_modulus():
    import ctypes as C
    from paper_2112_06396_b200 import _lib
    lib = _lib.load()
    h = C.c_void_p()
    ch = (C.c_uint64 * 1)(2 ** 40 + 1)            # not 1 mod 2N prime
    assert lib.ck_plan_create(12, ch, 1, None, 0, 1, C.byref(h)) == -2
    ch = (C.c_uint64 * 1)(prime_chain_below(1 << 12, 61, 1, 61, 0)[0][0])  # >= 2^60
    assert lib.ck_plan_create(12, ch, 1, None, 0, 1, C.byref(h)) == -2


@pytest.mark.parametrize("offs", [(0,), (2, 6), (0, 1, 2, 3, 4, 5, 6, 7, 9, 11), (-3, 4)])
def test_pt_matvec_diagonal_sets(offs):
    """ck_pt_matvec: identity-only, rotations-only, many diagonals, negative offsets."""
    p = cases.make_params(cases.TOY_A)
    mods, raised = p.chain, p.raised_moduli(p.limbs)
    a = cases._rows(p, 0, synth.TAG_CT_A, mods)
    b = cases._rows(p, 0, synth.TAG_CT_B, mods)
    diags = {o: cases._rows(p, 0, synth.TAG_DIAG, raised, digit=o % 64) for o in offs}
    keys = cases._keys(p, [-o for o in offs if o % p.slots])
    want = cases.OracleBackend().pt_matvec(p, a, b, keys, diags)
    got = gpu_backend.GpuBackend().pt_matvec(p, a, b, keys, diags)
    for w, g in zip(want, got):
        assert np.array_equal(w, g)


def test_relin_argument_errors():
    """ck_relin (new_mult's fused relinearisation key-switch) rejects bad levels
    and null operands with CK_ERR_ARG instead of launching."""
    from paper_2112_06396_b200 import _lib
    from paper_2112_06396_b200.device import plan_for
    p = _params(12, 4, 1, 4)
    lib = _lib.load()
    h = plan_for(p).h
    assert lib.ck_relin_workspace_bytes(h, 1, 1) == 0          # merged ModDown needs l >= 2
    assert lib.ck_relin_workspace_bytes(h, p.limbs, 0) == 0    # empty batch
    assert lib.ck_relin_workspace_bytes(h, p.limbs, 1) > 0
    x = torch.zeros((p.limbs, p.n_ring), dtype=torch.uint64, device="cuda")
    assert lib.ck_relin(h, x.data_ptr(), x.data_ptr(), x.data_ptr(), None, None, p.limbs,
                        x.data_ptr(), x.data_ptr(), x.data_ptr(), 1, None) == _lib.CK_ERR_ARG
    assert lib.ck_relin(h, x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(), 1,
                        x.data_ptr(), x.data_ptr(), x.data_ptr(), 1, None) == _lib.CK_ERR_ARG
    assert lib.ck_relin(h, x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(),
                        p.limbs, x.data_ptr(), x.data_ptr(), x.data_ptr(), 0, None) == _lib.CK_ERR_ARG


@pytest.mark.parametrize("kind", ["pt_matvec", "bsgs", "hrotate"])
def test_hoisted_paths_fused_ring_match_oracle(kind):
    """hrotate / pt_matvec / BSGS at N = 2^12 run the fused ModDown (md_row) path;
    bit-exact against the oracle (the toy goldens cover the small-ring path)."""
    p = _params(12, 6, 2, 3)
    mods, raised = p.chain, p.raised_moduli(p.limbs)
    a = cases._rows(p, 0, synth.TAG_CT_A, mods)
    b = cases._rows(p, 0, synth.TAG_CT_B, mods)
    ob, gb = cases.OracleBackend(), gpu_backend.GpuBackend()
    if kind == "pt_matvec":
        offs = (0, 1, 5, -3, 40)
        diags = {o: cases._rows(p, 0, synth.TAG_DIAG, raised, digit=o % 64) for o in offs}
        keys = cases._keys(p, [-o for o in offs if o % p.slots])
        want, got = ob.pt_matvec(p, a, b, keys, diags), gb.pt_matvec(p, a, b, keys, diags)
    elif kind == "bsgs":
        baby, giant = 5, 3
        diags = {(j, k): cases._rows(p, j, synth.TAG_DIAG, raised, digit=k)
                 for j in range(1, giant + 1) for k in range(1, baby + 1)}
        rs = sorted({-k for k in range(1, baby + 1)} | {-baby * j for j in range(1, giant + 1)})
        keys = cases._keys(p, rs)
        want = ob.bsgs(p, a, b, keys, diags, baby, giant)
        got = gb.bsgs(p, a, b, keys, diags, baby, giant)
    else:
        rots = (1, -2, 7, 100)
        keys = cases._keys(p, rots)
        want = [x for pair in ob.hrotate(p, a, b, keys, rots) for x in pair]
        got = [x for pair in gb.hrotate(p, a, b, keys, rots) for x in pair]
    for w, g in zip(want, got):
        assert np.array_equal(w, g)


def test_many_digits_beyond_fused_limit():
    """dnum = 12 (beta = 12 > 8 digits): the KSKIP runs in digit chunks that
    accumulate; rotation, hoisted rotations and relinearisation stay bit-exact
    against the oracle (the reference has no dnum cap, ckks.py:31-65)."""
    p = _params(12, 12, 1, 12, cb=50, sb=51)
    assert len(p.digit_spans(p.limbs)) == 12
    a, b, kb, ka = synth.rotation_inputs(p, 5, 0)
    want = ckks_np.rotate_galois(p, a, b, kb, ka, pow(5, 3, 2 * p.n_ring))
    ks = ckks.KeySet(p, None, None, rot={-3: ckks.SwitchingKey(p.full_moduli, kb, a=ka)})

    def ct(x, y):
        return ckks.Ciphertext(RnsPoly(p.chain, to_dev(x), "eval"), RnsPoly(p.chain, to_dev(y), "eval"),
                               p.delta)

    c1 = ct(a, b)
    got = ckks.rotate(p, ks, c1, -3)
    assert np.array_equal(to_host(got.a.data), want[0])
    assert np.array_equal(to_host(got.b.data), want[1])
    gh = ckks.hrotate(p, ks, c1, (-3,))[0]
    assert np.array_equal(to_host(gh.a.data), want[0])
    assert np.array_equal(to_host(gh.b.data), want[1])
    a2 = synth.uniform_poly(5, 1, synth.TAG_CT2_A, p.chain, p.n_ring)
    b2 = synth.uniform_poly(5, 1, synth.TAG_CT2_B, p.chain, p.n_ring)
    rk = synth.switching_key(p, 5, 998)
    wa, wb = ckks_np.new_mult(p, (a, b), (a2, b2), rk)
    ksr = ckks.KeySet(p, None, ckks.SwitchingKey(p.full_moduli, rk[0], a=rk[1]))
    o = ckks.new_mult(p, ksr, c1, ct(a2, b2))
    assert np.array_equal(to_host(o.a.data), wa) and np.array_equal(to_host(o.b.data), wb)


@pytest.mark.parametrize("logn", [18, 19, 20])
def test_large_rings_ntt_match_oracle(logn):
    """N = 2^18 .. 2^20 (column/row splits 512x512 .. 1024x1024): forward NTT of one limb
    bit-exact against the oracle, and INTT(NTT(x)) == x on two limbs."""
    from paper_2112_06396_b200.rnspoly import ntt_rows
    chain, _ = prime_chain_below(1 << logn, 54, 2, 60, 0)
    x = synth.uniform_poly(9, 0, synth.TAG_NTT, chain, 1 << logn)
    f = ntt_rows(to_dev(x), tuple(chain), False)
    assert np.array_equal(to_host(f[:1]), ckks_np.ntt(x[:1], chain[:1]))
    assert np.array_equal(to_host(ntt_rows(f, tuple(chain), True)), x)


def test_large_ring_rotation_matches_oracle():
    """A fused rotation key-switch at N = 2^18 (the reference has no ring-size cap)."""
    p = _params(18, 3, 1, 3, cb=54, sb=60)
    a, b, kb, ka = synth.rotation_inputs(p, 5, 0)
    t = pow(5, 7, 2 * p.n_ring)
    want = ckks_np.rotate_galois(p, a, b, kb, ka, t)
    ks = ckks.KeySet(p, None, None, rot={-7: ckks.SwitchingKey(p.full_moduli, kb, a=ka)})
    ct = ckks.Ciphertext(RnsPoly(p.chain, to_dev(a), "eval"), RnsPoly(p.chain, to_dev(b), "eval"),
                         p.delta)
    got = ckks.rotate(p, ks, ct, -7)
    assert np.array_equal(to_host(got.a.data), want[0])
    assert np.array_equal(to_host(got.b.data), want[1])


@pytest.mark.parametrize("kind,count", [("bsgs", 20), ("bsgs", 33), ("pt_matvec", 33), ("pt_matvec", 65)])
def test_chunk_boundaries_fused_ring(kind, count):
    """Chunked accumulation across launches at N = 2^12: BSGS with 20 / 33 babies (fused
    kernel in chunks of 16), pt_matvec with 33 / 65 diagonals (chunks of 32)."""
    p = _params(12, 4, 2, 2)
    mods, raised = p.chain, p.raised_moduli(p.limbs)
    a = cases._rows(p, 0, synth.TAG_CT_A, mods)
    b = cases._rows(p, 0, synth.TAG_CT_B, mods)
    ob, gb = cases.OracleBackend(), gpu_backend.GpuBackend()
    if kind == "bsgs":
        baby, giant = count, 2
        diags = {(j, k): cases._rows(p, j, synth.TAG_DIAG, raised, digit=k)
                 for j in range(1, giant + 1) for k in range(1, baby + 1)}
        rs = sorted({-k for k in range(1, baby + 1)} | {-baby * j for j in range(1, giant + 1)})
        keys = cases._keys(p, rs)
        want = ob.bsgs(p, a, b, keys, diags, baby, giant)
        got = gb.bsgs(p, a, b, keys, diags, baby, giant)
    else:
        offs = tuple(range(-(count // 2), count - count // 2))
        assert len(offs) == count and 0 in offs
        diags = {o: cases._rows(p, 0, synth.TAG_DIAG, raised, digit=o % 64) for o in offs}
        keys = cases._keys(p, [-o for o in offs if o % p.slots])
        want, got = ob.pt_matvec(p, a, b, keys, diags), gb.pt_matvec(p, a, b, keys, diags)
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
