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
from .device import fill_uniform, plan_for, ptr, ptr_array, stream_handle
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
        self.ws = self.plan.workspace(L, B)

    def run(self) -> None:
        ckks.rotate_batch(self.params, self.a, self.b, self.key_b, self.key_a, self.galois,
                          self.out_a, self.out_b, self.ws)

    def release_inputs(self) -> None:
        """Drop the device-resident keys (8 GB at C3) -- outputs are kept."""
        self.key_b = self.key_a = None
        torch.cuda.empty_cache()

    def input_bytes(self) -> int:
        return sum(t.numel() * 8 for t in (self.a, self.b, self.key_b, self.key_a))

    def output_bytes(self) -> int:
        return 2 * self.out_a.numel() * 8


class RelinBatch:
    """B independent relinearisations of new_mult (ckks.py:639-651) through one
    batched ck_relin: per unit u the tensor-product rows (a3, b3, c3) at `limbs`
    levels (TAG_CT_A / TAG_CT_B / TAG_CT2_A of unit u), ONE relinearisation key
    (KeySet.relin is shared by every product, ckks.py:230)."""

    def __init__(self, params, seed: int, units, limbs: int | None = None):
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
        self.x = torch.empty((3, B, L, n), **dev)  # a3, b3, c3
        keys, qs = [], []
        for tag in (synth.TAG_CT_A, synth.TAG_CT_B, synth.TAG_CT2_A):
            for u in self.units:
                k, q = _row_keys(seed, u, tag, params.chain[:L]); keys += k; qs += q
        fill_uniform(self.x, keys, qs, params.logn)
        self.key_b = torch.empty((dn, len(full), n), **dev)
        self.key_a = torch.empty((dn, len(full), n), **dev)
        kkb, qkb, kka, qka = [], [], [], []
        for j in range(dn):
            k, q = _row_keys(seed, 998, synth.TAG_KEY_B, full, j); kkb += k; qkb += q
            k, q = _row_keys(seed, 998, synth.TAG_KEY_A, full, j); kka += k; qka += q
        fill_uniform(self.key_b, kkb, qkb, params.logn)
        fill_uniform(self.key_a, kka, qka, params.logn)
        self.out_a = torch.empty((B, L - 1, n), **dev)
        self.out_b = torch.empty((B, L - 1, n), **dev)
        nbytes = load().ck_relin_workspace_bytes(self.plan.h, L, B)
        self.ws = torch.empty(nbytes // 8, **dev)

    def run(self) -> None:
        check(load().ck_relin(self.plan.h, ptr(self.x[0]), ptr(self.x[1]), ptr(self.x[2]),
                              ptr(self.key_b), ptr(self.key_a), self.limbs, ptr(self.out_a),
                              ptr(self.out_b), ptr(self.ws), len(self.units), stream_handle()),
              "ck_relin")

    def algorithmic_bytes_per_unit(self) -> int:
        return relin_bytes(self.params, self.limbs, len(self.units))


def relin_bytes(p, l: int, batch: int) -> int:
    """Compulsory HBM bytes per relinearisation in a batch sharing one key: read
    a3, b3, c3 (3 l limbs), write two (l-1)-limb outputs, and the key's
    2 beta (l+K) rows once per batch."""
    beta = len(p.digit_spans(l))
    key = 2 * beta * (l + len(p.special))
    return 8 * p.n_ring * (3 * l + 2 * (l - 1)) + 8 * p.n_ring * key // batch


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


class BsgsWorkload:
    """Config C4 on the device: one hoisted BSGS transform per run().

    Inputs follow tests/golden/cases.py's C4 case exactly (same stream ids), so
    the output digest can be checked against the reference golden.
    """

    def __init__(self, params, seed: int, baby: int = 16, giant: int = 8):
        self.params, self.baby, self.giant = params, baby, giant
        n, L = params.n_ring, params.limbs
        full = params.full_moduli
        raised = params.raised_moduli(L)
        dn = len(params.digit_spans(L))
        self.plan = plan_for(params)
        dev = dict(dtype=torch.uint64, device="cuda")
        self.a = torch.empty((L, n), **dev)
        self.b = torch.empty((L, n), **dev)
        k, q = _row_keys(seed, 0, synth.TAG_CT_A, params.chain)
        fill_uniform(self.a, k, q, params.logn)
        k, q = _row_keys(seed, 0, synth.TAG_CT_B, params.chain)
        fill_uniform(self.b, k, q, params.logn)

        def keys_for(rs):
            kb = torch.empty((len(rs), dn, len(full), n), **dev)
            ka = torch.empty((len(rs), dn, len(full), n), **dev)
            kkb, qkb, kka, qka = [], [], [], []
            for r in rs:
                unit = 1000 + (r % (4 * n))
                for j in range(dn):
                    k, q = _row_keys(seed, unit, synth.TAG_KEY_B, full, j); kkb += k; qkb += q
                    k, q = _row_keys(seed, unit, synth.TAG_KEY_A, full, j); kka += k; qka += q
            fill_uniform(kb, kkb, qkb, params.logn)
            fill_uniform(ka, kka, qka, params.logn)
            return kb, ka

        self.bkb, self.bka = keys_for([-k for k in range(1, baby + 1)])
        self.gkb, self.gka = keys_for([-baby * j for j in range(1, giant + 1)])
        self.diags = torch.empty((giant, baby, len(raised), n), **dev)
        kk, qq = [], []
        for j in range(1, giant + 1):
            for kb_ in range(1, baby + 1):
                k, q = _row_keys(seed, j, synth.TAG_DIAG, raised, kb_)
                kk += k
                qq += q
        fill_uniform(self.diags, kk, qq, params.logn)
        self.out = (torch.empty((L - 1, n), **dev), torch.empty((L - 1, n), **dev))
        # the C ABI takes per-key / per-diagonal pointer arrays (built once)
        self.ptrs = (ptr_array(list(self.bkb)), ptr_array(list(self.bka)),
                     ptr_array(list(self.gkb)), ptr_array(list(self.gka)),
                     ptr_array([self.diags[j, k] for j in range(giant) for k in range(baby)]))
        nbytes = load().ck_bsgs_workspace_bytes(self.plan.h, L, baby, giant)
        self.ws = torch.empty(nbytes // 8, **dev)

    def run(self) -> None:
        ckks.bsgs_raw(self.params, self.a, self.b, *self.ptrs, self.baby, self.giant,
                      out=self.out, ws=self.ws)

    def algorithmic_bytes(self) -> int:
        """a, b; baby keys; diagonals; giant keys (at l-1); output."""
        p = self.params
        L, K = p.limbs, len(p.special)
        beta = len(p.digit_spans(L))
        beta1 = len(p.digit_spans(L - 1))
        limbs = (2 * L + self.baby * 2 * beta * (L + K) + self.giant * self.baby * (L + K)
                 + self.giant * 2 * beta1 * (L - 1 + K) + 2 * (L - 1))
        return limbs * p.n_ring * 8
