"""Concurrent callers: the reference's operations are pure and must give bit-identical
results under parallel execution.  Four host threads, each on its own
CUDA stream, run rotations, conjugations and hoisted rotations on different ciphertexts of
the SAME plan at the same time; every result must equal the one the same call produced
alone.  (Scratch is allocated per call from the stream-ordered allocator; plan tables are
read-only.)"""

import threading

import numpy as np
import pytest
import torch

from paper_2112_06396_b200 import ckks, synth
from paper_2112_06396_b200.device import to_host
from paper_2112_06396_b200.params import CkksParams, prime_chain_below
from paper_2112_06396_b200.rnspoly import RnsPoly

pytestmark = pytest.mark.gpu


def _params(logn, L, K, dnum, cb=54, sb=60):
    chain, special = prime_chain_below(1 << logn, cb, L, sb, K)
    return CkksParams(logn, chain, special, dnum, 2.0 ** 40, 1)


@pytest.mark.parametrize("logn,L,K,dnum", [(12, 6, 2, 3), (14, 8, 4, 2)])
def test_parallel_streams_bit_identical(logn, L, K, dnum):
    p = _params(logn, L, K, dnum)
    T, REPS = 4, 12
    rots = (-3, -7)
    work = []
    for u in range(T):
        a, b, _, _ = synth.rotation_inputs(p, 11, u)
        keys = {}
        for j, k in enumerate(rots):
            _, _, kb, ka = synth.rotation_inputs(p, 11, 10 * u + j + 1)
            keys[k] = ckks.SwitchingKey(p.full_moduli, kb, a=ka)
        _, _, cb_, ca_ = synth.rotation_inputs(p, 11, 100 + u)
        ks = ckks.KeySet(p, None, None, rot=keys, conj=ckks.SwitchingKey(p.full_moduli, cb_, a=ca_))
        ct = ckks.Ciphertext(RnsPoly(p.chain, a, "eval"), RnsPoly(p.chain, b, "eval"), 1.0)
        work.append((ks, ct))

    def ops(ks, ct):
        outs = [ckks.rotate(p, ks, ct, rots[0]), ckks.conjugate(p, ks, ct)]
        outs += list(ckks.hrotate(p, ks, ct, list(rots)))
        return [(to_host(o.a.data), to_host(o.b.data)) for o in outs]

    alone = [ops(ks, ct) for ks, ct in work]
    torch.cuda.synchronize()
    bad, errs = [], []
    start = threading.Barrier(T)

    def worker(u):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                start.wait()
                for r in range(REPS):
                    got = ops(*work[u])
                    for i, ((ga, gb), (wa, wb)) in enumerate(zip(got, alone[u])):
                        if not (np.array_equal(ga, wa) and np.array_equal(gb, wb)):
                            bad.append((u, r, i))
        except Exception as e:  # surfaced below: a thread's exception would otherwise be lost
            errs.append(repr(e))

    ts = [threading.Thread(target=worker, args=(u,)) for u in range(T)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert not bad, bad[:8]
