"""Device-resident BASELINE.json workloads (inputs generated on the GPU).

* RotationBatch: B independent rotation key-switches (configs C1/C3/C5): per
  unit u a ciphertext (a, b) at top level, an expanded switching key and a
  Galois element 5^k mod 2N.  Inputs come from the counter-based generator
  (synth.py); ``ck_fill_uniform`` reproduces the host generator bit-for-bit.
* NttBatch: config C2, a batch of polynomials NTT'd then INTT'd in place.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ckks, synth
from ._lib import check, load
from .device import fill_uniform, plan_for, ptr, stream_handle
from .params import galois_exponents


def _row_keys(seed: int, unit: int, tag: int, moduli, digit: int = 0):
    keys = [synth.stream_key(seed, synth.stream_id(unit, tag, digit, r)) for r in range(len(moduli))]
    return keys, list(moduli)


class RotationBatch:
    def __init__(self, params, seed: int, units, ks=None, limbs: int | None = None):
        self.params = params
        self.units = list(units)
        B = len(self.units)
        n = params.n_ring
        L = params.limbs if limbs is None else limbs
        self.limbs = L
        full = params.full_moduli
        dn = len(params.digit_spans(params.limbs))
        self.plan = plan_for(params)
        dev = dict(dtype=torch.uint64, device="cuda")
        self.a = torch.empty((B, L, n), **dev)
        self.b = torch.empty((B, L, n), **dev)
        self.key_b = torch.empty((B, dn, len(full), n), **dev)
        self.key_a = torch.empty((B, dn, len(full), n), **dev)
        ka, qa, kb, qb, kkb, qkb, kka, qka = ([] for _ in range(8))
        for u in self.units:
            k, q = _row_keys(seed, u, synth.TAG_CT_A, params.chain[:L]); ka += k; qa += q
            k, q = _row_keys(seed, u, synth.TAG_CT_B, params.chain[:L]); kb += k; qb += q
            for j in range(dn):
                k, q = _row_keys(seed, u, synth.TAG_KEY_B, full, j); kkb += k; qkb += q
                k, q = _row_keys(seed, u, synth.TAG_KEY_A, full, j); kka += k; qka += q
        fill_uniform(self.a, ka, qa, params.logn)
        fill_uniform(self.b, kb, qb, params.logn)
        fill_uniform(self.key_b, kkb, qkb, params.logn)
        fill_uniform(self.key_a, kka, qka, params.logn)
        if ks is None:
            allk = galois_exponents(n, max(self.units) + 1, seed)
            ks = [allk[u] for u in self.units]
        self.ks = list(ks)
        self.galois = torch.tensor(np.array([pow(5, k, 2 * n) for k in self.ks], dtype=np.uint64),
                                   device="cuda")
        self.out_a = torch.empty_like(self.a)
        self.out_b = torch.empty_like(self.b)
        self.ws = self.plan.workspace(L, B, "batch")

    def run(self) -> None:
        ckks.rotate_batch(self.params, self.a, self.b, self.key_b, self.key_a, self.galois,
                          self.out_a, self.out_b, self.ws)

    def input_bytes(self) -> int:
        return sum(t.numel() * 8 for t in (self.a, self.b, self.key_b, self.key_a))

    def output_bytes(self) -> int:
        return 2 * self.out_a.numel() * 8


class NttBatch:
    def __init__(self, params, seed: int, batch: int):
        self.params = params
        n, L = params.n_ring, params.limbs
        self.plan = plan_for(params)
        self.x = torch.empty((batch, L, n), dtype=torch.uint64, device="cuda")
        keys, qs = [], []
        for u in range(batch):
            k, q = _row_keys(seed, u, synth.TAG_NTT, params.chain)
            keys += k
            qs += q
        fill_uniform(self.x, keys, qs, params.logn)
        self.idx = self.plan.prime_idx(params.chain)
        self.batch = batch

    def run(self) -> None:
        lib = load()
        L, n = self.params.limbs, self.params.n_ring
        for inv in (0, 1):
            check(lib.ck_ntt(self.plan.h, ptr(self.x), ptr(self.idx), L, self.batch, L * n, inv,
                             stream_handle()), "ck_ntt")
