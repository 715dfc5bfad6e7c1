"""Multi-process (N>1) paths on CPU with the gloo backend (world sizes 2 and 3).

* batch partitioning: every rank processes its own units; the union of the
  per-rank results equals the single-process results (bit-exact digests);
* limb sharding (C5 variant): one key-switch split by raised
  limbs across ranks with exactly two all-gathers; the gathered output rows
  are bit-identical to the unsharded rotation.
Compute here is the CPU oracle; the GPU runs the same orchestration with
the CUDA library and NCCL.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup(rank, world, port):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)


def _batch_worker(rank, world, port, per_rank, out_q):
    _setup(rank, world, port)
    import cases
    from oracle import ckks_np
    from paper_2112_06396_b200 import shard, synth
    from paper_2112_06396_b200.digest import digest
    from paper_2112_06396_b200.params import galois_exponents
    p = cases.make_params(cases.TOY_B)
    units = shard.units_for_rank(rank, per_rank)
    ks = galois_exponents(p.n_ring, per_rank * world, cases.SEED)
    local = {}
    for u in units:
        a, b, kb, ka = synth.rotation_inputs(p, cases.SEED, u)
        oa, ob = ckks_np.rotate_galois(p, a, b, kb, ka, pow(5, ks[u], 2 * p.n_ring))
        local[u] = digest(oa, ob)
    got = [None] * world
    dist.all_gather_object(got, local)
    if rank == 0:
        merged = {}
        for g in got:
            assert not (set(g) & set(merged)), "units assigned twice"
            merged.update(g)
        out_q.put(merged)
    dist.destroy_process_group()


def _limb_worker(rank, world, port, pspec, k, out_q):
    _setup(rank, world, port)
    import cases
    from numpy_ops import NumpyOps
    from paper_2112_06396_b200 import shard, synth
    p = cases.make_params(pspec)
    a, b, kb, ka = synth.rotation_inputs(p, cases.SEED, 3)
    L = p.limbs
    sh = shard.LimbShard(p, L, world, rank)
    rows = sh.rows()
    chain = sh.chain_rows()
    krows = [i if i < L else p.limbs + (i - L) for i in rows]  # full-basis key rows
    ndig = len(p.digit_spans(L))
    t = pow(5, k, 2 * p.n_ring)
    oa, ob = shard.keyswitch_limb_sharded(
        p, sh, a[chain], b[chain], kb[:ndig][:, krows], ka[:ndig][:, krows], t, NumpyOps())
    got = [None] * world
    dist.all_gather_object(got, (chain, oa, ob))
    if rank == 0:
        out_q.put(got)
    dist.destroy_process_group()


def _run(fn, world, *args):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tmp.start_processes(fn, args=(world, port, *args, q), nprocs=world, join=True,
                        start_method="spawn")
    return q.get(timeout=60)


@pytest.mark.parametrize("world", [2, 3])
def test_batch_partition_matches_single_process(world):
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import cases
    from oracle import ckks_np
    from paper_2112_06396_b200 import synth
    from paper_2112_06396_b200.digest import digest
    from paper_2112_06396_b200.params import galois_exponents
    per_rank = 2
    merged = _run(_batch_worker, world, per_rank)
    p = cases.make_params(cases.TOY_B)
    ks = galois_exponents(p.n_ring, per_rank * world, cases.SEED)
    assert sorted(merged) == list(range(per_rank * world))
    for u in range(per_rank * world):
        a, b, kb, ka = synth.rotation_inputs(p, cases.SEED, u)
        oa, ob = ckks_np.rotate_galois(p, a, b, kb, ka, pow(5, ks[u], 2 * p.n_ring))
        assert merged[u] == digest(oa, ob)


@pytest.mark.parametrize("world,pspec", [(2, ("toy", 7, 54, 6, 60, 2, 3)),
                                         (3, ("toy", 6, 50, 5, 60, 3, 2)),
                                         (2, ("toy", 8, 50, 8, 60, 2, 4))])
def test_limb_sharded_keyswitch_bit_exact(world, pspec):
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import cases
    from oracle import ckks_np
    from paper_2112_06396_b200 import synth
    k = 7
    got = _run(_limb_worker, world, pspec, k)
    p = cases.make_params(pspec)
    a, b, kb, ka = synth.rotation_inputs(p, cases.SEED, 3)
    want_a, want_b = ckks_np.rotate_galois(p, a, b, kb, ka, pow(5, k, 2 * p.n_ring))
    seen = []
    for chain, oa, ob in got:
        for i, row in enumerate(chain):
            assert np.array_equal(oa[i], want_a[row]), (row, "a")
            assert np.array_equal(ob[i], want_b[row]), (row, "b")
            seen.append(row)
    assert sorted(seen) == list(range(p.limbs))


def test_block_partition_covers_evenly():
    from paper_2112_06396_b200.shard import block_partition
    for total in (1, 7, 45, 64):
        for world in (1, 2, 3, 8):
            parts = [list(block_partition(total, world, r)) for r in range(world)]
            flat = [x for p in parts for x in p]
            assert flat == list(range(total))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
