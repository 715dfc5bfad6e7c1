"""Limb-sharded key-switch orchestration on the GPU (world size 1, NCCL).

Multi-rank coverage is tests/test_multiproc_gloo.py (CPU); this runs the same
orchestration through the CUDA library and an NCCL process group.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

import cases
from oracle import ckks_np
from paper_2112_06396_b200 import shard, synth
from paper_2112_06396_b200.device import plan_for, to_dev, to_host
from paper_2112_06396_b200.digest import digest
from paper_2112_06396_b200.params import galois_exponents

GOLD = __import__("json").load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("pspec", [cases.TOY_B, ("cfg", "C5")])
def test_limb_sharded_world1_matches_oracle(nccl1, pspec):
    p = cases.make_params(pspec)
    plan_for(p)
    full = pspec[0] == "cfg"
    # C5: unit 0 with the benchmark's first Galois exponent = the reference golden C5_rot0
    unit, k = (0, galois_exponents(p.n_ring, 256, cases.SEED)[0]) if full else (3, 11)
    a, b, kb, ka = synth.rotation_inputs(p, cases.SEED, unit)
    L = p.limbs
    sh = shard.LimbShard(p, L, 1, 0)
    rows = sh.rows()
    krows = [i for i in rows]
    ndig = len(p.digit_spans(L))
    t = pow(5, k, 2 * p.n_ring)
    oa, ob = shard.keyswitch_limb_sharded(
        p, sh, to_dev(a), to_dev(b), to_dev(kb[:ndig][:, krows]), to_dev(ka[:ndig][:, krows]), t,
        shard.TorchOps(p.n_ring))
    torch.cuda.synchronize()
    if full:
        # C5: pinned to the reference itself (tests/golden/golden.json, produced by
        # running ckkslab's hrotate on these inputs) and to the fused single-GPU rotation
        assert digest(to_host(oa), to_host(ob)) == GOLD["C5_rot0"]["digest"]
        from paper_2112_06396_b200 import ckks
        from paper_2112_06396_b200.rnspoly import RnsPoly
        key = ckks.SwitchingKey(p.full_moduli, kb, a=ka)
        ct = ckks.Ciphertext(RnsPoly(p.chain, a, "eval"), RnsPoly(p.chain, b, "eval"), p.delta)
        ks = ckks.KeySet(p, None, None, rot={-k: key})
        ref = ckks.rotate(p, ks, ct, -k)
        assert torch.equal(oa, ref.a.data) and torch.equal(ob, ref.b.data)
    else:
        want_a, want_b = ckks_np.rotate_galois(p, a, b, kb, ka, t)
        assert np.array_equal(to_host(oa), want_a)
        assert np.array_equal(to_host(ob), want_b)
