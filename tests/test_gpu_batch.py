"""Batched key-switch (the benchmark's unit) and device input generation."""

import json
import os

import numpy as np
import pytest
import torch

import cases
from paper_2112_06396_b200 import ckks, synth
from paper_2112_06396_b200.device import to_dev, to_host
from paper_2112_06396_b200.digest import digest
from paper_2112_06396_b200.params import config, galois_exponents
from paper_2112_06396_b200 import workload

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def test_device_generator_matches_host():
    p = config("C3").params
    units = [0, 5]
    dev = workload.RotationBatch(p, cases.SEED, units)
    a, b, kb, ka = synth.rotation_inputs(p, cases.SEED, 5)
    assert np.array_equal(to_host(dev.a[1]), a)
    assert np.array_equal(to_host(dev.b[1]), b)
    assert np.array_equal(to_host(dev.key_b[1]), kb)
    assert np.array_equal(to_host(dev.key_a[1]), ka)


def test_batched_rotations_match_reference_digests():
    p = config("C3").params
    ks = galois_exponents(p.n_ring, 64, cases.SEED)
    units = [0, 1, 63]
    wb = workload.RotationBatch(p, cases.SEED, units, ks=[ks[u] for u in units])
    wb.run()
    torch.cuda.synchronize()
    for i, u in enumerate(units):
        got = digest(to_host(wb.out_a[i]), to_host(wb.out_b[i]))
        assert got == GOLD[{0: "C3_rot0", 1: "C3_rot1", 63: "C3_rot63"}[u]]["digest"], u


def test_c2_ntt_roundtrip_full_batch_identity():
    """Size-independent property at BASELINE size: INTT(NTT(x)) == x on 16 x 24 limbs."""
    nb = workload.NttBatch(config("C2").params, cases.SEED, 16)
    x0 = nb.x.clone()
    nb.run()
    torch.cuda.synchronize()
    assert torch.equal(nb.x, x0)


def test_c2_ntt_linearity():
    from paper_2112_06396_b200.rnspoly import ntt_rows
    p = config("C2").params
    mods = p.chain[:4]
    x = synth.uniform_poly(1, 0, 0, mods, p.n_ring)
    y = synth.uniform_poly(1, 0, 1, mods, p.n_ring)
    q = np.array(mods, dtype=np.uint64)[:, None]
    s = (x + y) % q
    fx, fy, fs = (to_host(ntt_rows(to_dev(v), mods, False)) for v in (x, y, s))
    assert np.array_equal((fx + fy) % q, fs)
