"""Multi-GPU partitioning of the key-switch path.

Two modes, one process per GPU (torch.distributed, NCCL on B200, gloo in the
CPU tests):

* batch partitioning (throughput mode, configs C3/C5): units (independent
  (ciphertext, key, Galois element) triples) are split across ranks; there is
  no data-path collective -- only the timing barrier / max-reduction.
* limb sharding (config C5 variant): ONE key-switch with its raised-basis
  limbs and key rows block-partitioned across ranks.  Exactly two exchange
  steps, both all-gathers of coefficient-form rows:
    1. the INTT'd chain limbs of `a` (every rank needs a whole digit to
       base-convert it to its own target limbs, ckks.py:427-431);
    2. the INTT'd special rows of u and v (every rank needs all of them for
       the centered ModDown conversion to its own chain limbs, ckks.py:409-410).
  Everything else (BC to own targets, NTT, automorphism, KSKIP on own rows,
  ModDown epilogue on own chain rows) is rank-local.

The limb-sharded algorithm is written once against a small `ops` interface
(`TorchOps`: the CUDA library on the GPU; the CPU tests bind the same interface
to the numpy checker in tests/numpy_ops.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def units_for_rank(rank: int, per_rank: int) -> list[int]:
    """Weak-scaling unit assignment: rank r owns units [r*B, (r+1)*B)."""
    return [rank * per_rank + i for i in range(per_rank)]


def block_partition(total: int, world: int, rank: int) -> range:
    """Balanced contiguous block of [0, total) for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


@dataclass
class LimbShard:
    """Ownership of the raised basis chain[:l] + special by one rank."""

    params: object
    limbs: int
    world: int
    rank: int

    @property
    def R(self) -> int:
        return self.limbs + len(self.params.special)

    def rows(self, rank: int | None = None) -> list[int]:
        return list(block_partition(self.R, self.world, self.rank if rank is None else rank))

    def chain_rows(self, rank: int | None = None) -> list[int]:
        return [i for i in self.rows(rank) if i < self.limbs]

    def special_rows(self, rank: int | None = None) -> list[int]:
        return [i for i in self.rows(rank) if i >= self.limbs]

    def moduli(self, rows) -> tuple[int, ...]:
        raised = self.params.raised_moduli(self.limbs)
        return tuple(raised[i] for i in rows)


def _all_gather_rows(local, owners: list[list[int]], total_rows: int, ops, group=None):
    """All-gather variable-size row blocks (padded to the largest block)."""
    import torch.distributed as dist
    world = len(owners)
    width = max(len(o) for o in owners)
    padded = ops.pad_rows(local, width)
    parts = [ops.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    out = ops.empty_rows(total_rows, padded)
    for r, rows in enumerate(owners):
        for k, row in enumerate(rows):
            ops.set_row(out, row, parts[r], k)
    return out


def keyswitch_limb_sharded(params, shard: LimbShard, a_rows, b_rows, key_b_rows, key_a_rows,
                           galois_t: int, ops, group=None):
    """Rotation key-switch (hrotate order: ModUp then automorph) on a limb shard.

    a_rows, b_rows: this rank's chain rows of the eval-rep ciphertext
    (shard.chain_rows() order); key_b_rows / key_a_rows: (beta, len(rows), N)
    key rows for this rank's raised rows.  Returns this rank's chain rows of
    (out_a, out_b), bit-identical to the unsharded rotation.
    """
    l, R = shard.limbs, shard.R
    raised = params.raised_moduli(l)
    my_rows = shard.rows()
    my_chain = shard.chain_rows()
    owners_chain = [shard.chain_rows(r) for r in range(shard.world)]
    owners_spec = [[i - l for i in shard.special_rows(r)] for r in range(shard.world)]

    # ---- exchange 1: coefficient-form chain limbs of a
    a_coeff_local = ops.intt(a_rows, shard.moduli(my_chain))
    a_coeff = _all_gather_rows(a_coeff_local, owners_chain, l, ops, group)

    # ---- ModUp digits restricted to my rows; automorph; KSKIP on my rows
    spans = params.digit_spans(l)
    my_mods = shard.moduli(my_rows)
    u = v = None
    for d, (lo, hi) in enumerate(spans):
        own = tuple(raised[lo:hi])
        tgt_rows = [i for i in my_rows if not (lo <= i < hi)]
        conv = ops.bc_convert(ops.take_rows(a_coeff, list(range(lo, hi))), own,
                              tuple(raised[i] for i in tgt_rows))
        conv = ops.ntt(conv, tuple(raised[i] for i in tgt_rows))
        parts = []
        for i in my_rows:
            if lo <= i < hi:
                parts.append(ops.take_rows(a_rows, [my_chain.index(i)]))
            else:
                parts.append(ops.take_rows(conv, [tgt_rows.index(i)]))
        digit = ops.automorph(ops.cat_rows(parts), galois_t)
        pu = ops.mul(digit, key_a_rows[d], my_mods)
        pv = ops.mul(digit, key_b_rows[d], my_mods)
        u = pu if u is None else ops.add(u, pu, my_mods)
        v = pv if v is None else ops.add(v, pv, my_mods)

    # ---- exchange 2: coefficient-form special rows of u and v
    my_spec = shard.special_rows()
    spec_idx = [my_rows.index(i) for i in my_spec]
    spec_mods = shard.moduli(my_spec)
    uv_spec_local = ops.cat_rows([ops.intt(ops.take_rows(u, spec_idx), spec_mods),
                                  ops.intt(ops.take_rows(v, spec_idx), spec_mods)])
    K = len(params.special)
    owners_uv = [o + [k + K for k in o] for o in owners_spec]
    uv_spec = _all_gather_rows(uv_spec_local, owners_uv, 2 * K, ops, group)

    # ---- ModDown to my chain rows (centered BC from all specials), epilogue
    special = tuple(params.special)
    keep = shard.moduli(my_chain)
    chain_idx = [my_rows.index(i) for i in my_chain]
    big_p = 1
    for p in special:
        big_p *= p
    pinv = [pow(big_p % q, -1, q) for q in keep]
    outs = []
    for w, x in ((0, u), (1, v)):
        conv = ops.bc_convert_centered(ops.take_rows(uv_spec, list(range(w * K, (w + 1) * K))),
                                       special, keep)
        conv = ops.ntt(conv, keep)
        y = ops.mul_scalars(ops.sub(ops.take_rows(x, chain_idx), conv, keep), pinv, keep)
        outs.append(y)
    out_b = ops.add(outs[1], ops.automorph(b_rows, galois_t), keep)
    return outs[0], out_b


class TorchOps:
    """CUDA-library row ops on torch.uint64 device tensors (NCCL on the wire)."""

    def __init__(self, n: int):
        self.n = n

    def _rp(self):
        from . import rnspoly
        return rnspoly

    def intt(self, x, mods):
        return self._rp().ntt_rows(x.contiguous(), tuple(mods), True)

    def ntt(self, x, mods):
        return self._rp().ntt_rows(x.contiguous(), tuple(mods), False)

    def bc_convert(self, x, src, dst):
        import torch
        if len(dst) == 0:
            return torch.zeros((0, x.shape[1]), dtype=torch.uint64, device=x.device)
        rp = self._rp()
        return rp.bc_convert(rp.RnsPoly(tuple(src), x.contiguous(), "coeff"), tuple(dst)).data

    def bc_convert_centered(self, x, src, dst):
        import torch
        if len(dst) == 0:
            return torch.zeros((0, x.shape[1]), dtype=torch.uint64, device=x.device)
        rp = self._rp()
        return rp.bc_convert_centered(rp.RnsPoly(tuple(src), x.contiguous(), "coeff"),
                                      tuple(dst)).data

    def automorph(self, x, t):
        return self._rp().automorph_rows(x.contiguous(), t)

    def _op(self, op, x, y, mods):
        return self._rp()._poly_op(op, tuple(mods), x.contiguous(), y.contiguous())

    def mul(self, x, y, mods):
        return self._op(self._rp().OP_MUL, x, y, mods)

    def add(self, x, y, mods):
        return self._op(self._rp().OP_ADD, x, y, mods)

    def sub(self, x, y, mods):
        return self._op(self._rp().OP_SUB, x, y, mods)

    def mul_scalars(self, x, s, mods):
        rp = self._rp()
        return rp.RnsPoly(tuple(mods), x.contiguous(), "eval").mul_scalars(s).data

    def take_rows(self, x, idx):
        import torch
        if not len(idx):
            return x[:0]
        sel = torch.tensor(list(idx), dtype=torch.long, device=x.device)
        return x.view(torch.int64)[sel].view(torch.uint64)  # no uint64 gather kernel in torch

    def cat_rows(self, parts):
        import torch
        return torch.cat(parts, dim=0)

    def pad_rows(self, x, width):
        import torch
        out = torch.zeros((width, x.shape[1]), dtype=torch.uint64, device=x.device)
        out[:x.shape[0]] = x
        return out.view(torch.int64)

    def empty_like(self, t):
        import torch
        return torch.empty_like(t)

    def empty_rows(self, rows, like):
        import torch
        return torch.empty((rows, like.shape[1]), dtype=torch.uint64, device=like.device)

    def set_row(self, out, row, part, k):
        import torch
        out[row] = part[k].view(torch.uint64)
