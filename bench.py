"""Benchmark: CKKS rotation key-switches/s at N=2^16, L=24, dnum=3 (BASELINE config C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = the BASELINE C3 workload on each GPU: 64 independent rotation
key-switches (distinct ciphertexts, keys and Galois elements 5^k), batched
through ck_rotate (C ABI).  Inputs are generated on the device (counter-based
generator, bit-identical to the host generator the oracle uses) and exceed L2
(8 GB per step), so no L2 flush is needed between steps.

Multi-GPU (torchrun): every rank processes its own 64 units (weak scaling,
no data-path collective); time = max over ranks of CUDA-event time.

--impl reference times the reference algorithm's CPU implementation (the
numpy port in oracle/, the only CPU form of the reference that can run on
the GPU box) on all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "key-switches/sec at N=2^16,L=24,dnum=3; achieved HBM GB/s vs B200 peak"
UNIT = "key-switches/s"
SEED = 20211212
CPU_WORKERS_MAX = 32


def _peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ks_bytes(params, limbs=None) -> int:
    """Compulsory HBM bytes per rotation key-switch:
    8 N (l [a] + l [b] + 2 beta (l+K) [evk a,b rows] + 2 l [out])."""
    l = params.limbs if limbs is None else limbs
    beta = len(params.digit_spans(l))
    K = len(params.special)
    return 8 * params.n_ring * (l + l + 2 * beta * (l + K) + 2 * l)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.QUERY}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except Exception:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- CPU oracle
def _cpu_task(args):
    unit, k = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import ckks_np
    from paper_2112_06396_b200 import synth
    from paper_2112_06396_b200.digest import digest
    from paper_2112_06396_b200.params import config
    p = config("C3").params
    a, b, kb, ka = synth.rotation_inputs(p, SEED, unit)
    t0 = time.perf_counter()
    oa, ob = ckks_np.rotate_galois(p, a, b, kb, ka, pow(5, k, 2 * p.n_ring))
    return unit, time.perf_counter() - t0, digest(oa, ob)


def _warm(name="C3"):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import ckks_np
    from paper_2112_06396_b200.params import config
    p = config(name).params
    for q in p.full_moduli:
        ckks_np.twiddles(q, p.n_ring)
    return True


# ---- per-config CPU baseline units (the oracle port of the reference, one unit per
# task; bench.py's cpu_baseline leg is the only product-side caller of oracle/)
def _cpu_unit(args):
    """(config, unit, extra) -> (unit, seconds, digest of the unit's outputs)."""
    name, unit, extra = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import ckks_np
    from paper_2112_06396_b200 import synth
    from paper_2112_06396_b200.digest import digest
    from paper_2112_06396_b200.params import config
    p = config(name).params
    if name in ("C1", "C3", "C5"):
        a, b, kb, ka = synth.rotation_inputs(p, SEED, unit)
        t0 = time.perf_counter()
        out = ckks_np.rotate_galois(p, a, b, kb, ka, pow(5, extra, 2 * p.n_ring))
    elif name == "C2":  # one polynomial (all limbs) forward, then its inverse
        x = synth.uniform_poly(SEED, unit, synth.TAG_NTT, p.chain, p.n_ring)
        t0 = time.perf_counter()
        f = ckks_np.ntt(x, p.chain)
        inv = ckks_np.intt(x, p.chain)
        out = (f,)
        assert inv.shape == x.shape
    elif name == "C3M":  # relinearisation of unit `unit`, shared relin key (unit 998)
        mods = p.chain
        a3, b3, c3 = (synth.uniform_poly(SEED, unit, tag, mods, p.n_ring)
                      for tag in (synth.TAG_CT_A, synth.TAG_CT_B, synth.TAG_CT2_A))
        kb, ka = synth.switching_key(p, SEED, 998)
        t0 = time.perf_counter()
        lim = len(mods)
        digits = ckks_np.decomp_modup(p, a3, mods)
        u, v = ckks_np.kskip(p, digits, kb, ka, lim)
        qr = ckks_np._qcol(p.raised_moduli(lim), 2)
        u = ckks_np.addmod(u, ckks_np.pmodup(p, b3, mods), qr)
        v = ckks_np.addmod(v, ckks_np.pmodup(p, c3, mods), qr)
        out = (ckks_np.moddown_merged(p, u, lim), ckks_np.moddown_merged(p, v, lim))
    else:
        raise KeyError(name)
    return unit, time.perf_counter() - t0, digest(*out)


def _c4_stage(args):
    """One stage of the hoisted C4 BSGS transform on the CPU (oracle port), with
    intermediates in a RAM-backed directory (numpy files, memory-mapped by the
    next stage's workers instead of pickled through pipes):
    ('modup', dir) -> digits; ('baby', dir, k) -> (u_k, v_k + P b_k);
    ('giant', dir, j) -> rotate(ModDown(sum_k diag[j][k] (u_k, v_k)), -16 j)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np
    from oracle import ckks_np
    from paper_2112_06396_b200 import synth
    from paper_2112_06396_b200.params import config
    p = config("C4").params
    n, L = p.n_ring, p.limbs
    mods, raised = p.chain, p.raised_moduli(L)
    qr = ckks_np._qcol(raised, 2)
    kind, d = args[0], args[1]
    if kind == "modup":
        a = synth.uniform_poly(SEED, 0, synth.TAG_CT_A, mods, n)
        np.save(os.path.join(d, "digits.npy"), np.stack(ckks_np.decomp_modup(p, a, mods)))
        return True
    if kind == "baby":
        k = args[2]
        digits = np.load(os.path.join(d, "digits.npy"), mmap_mode="r")
        b = synth.uniform_poly(SEED, 0, synth.TAG_CT_B, mods, n)
        kb, ka = synth.switching_key(p, SEED, 1000 + ((-k) % (4 * n)))
        perm = ckks_np.automorph_perm(n, ckks_np.galois_rot(n, -k))
        u, v = ckks_np.kskip(p, [np.asarray(x)[:, perm] for x in digits], kb, ka, L)
        v = ckks_np.addmod(v, ckks_np.pmodup(p, b[:, perm], mods), qr)
        np.save(os.path.join(d, f"baby{k}.npy"), np.stack([u, v]))
        return True
    j = args[2]
    acc_u = np.zeros((len(raised), n), dtype=np.uint64)
    acc_v = np.zeros_like(acc_u)
    for k in range(1, 17):
        uv = np.load(os.path.join(d, f"baby{k}.npy"), mmap_mode="r")
        m = synth.uniform_poly(SEED, j, synth.TAG_DIAG, raised, n, digit=k)
        acc_u = ckks_np.addmod(acc_u, ckks_np.mulmod(m, np.asarray(uv[0]), qr), qr)
        acc_v = ckks_np.addmod(acc_v, ckks_np.mulmod(m, np.asarray(uv[1]), qr), qr)
    ga, gb = ckks_np.moddown_merged(p, acc_u, L), ckks_np.moddown_merged(p, acc_v, L)
    r = -16 * j
    kb, ka = synth.switching_key(p, SEED, 1000 + (r % (4 * n)))
    return ckks_np.rotate_galois(p, ga, gb, kb, ka, ckks_np.galois_rot(n, r))


def cpu_c4_transform(pool):
    """One C4 transform, hoisted, stages parallel across the pool (ModUp; 16 babies;
    8 giant groups each MAC + ModDown + rotation; sum).  Returns (seconds, digest)."""
    import shutil
    from oracle import ckks_np
    from paper_2112_06396_b200.digest import digest
    from paper_2112_06396_b200.params import config
    p = config("C4").params
    d = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    try:
        t0 = time.perf_counter()
        pool.apply(_c4_stage, (("modup", d),))
        pool.map(_c4_stage, [("baby", d, k) for k in range(1, 17)], chunksize=1)
        giants = pool.map(_c4_stage, [("giant", d, j) for j in range(1, 9)], chunksize=1)
        ql = ckks_np._qcol(p.chain[:p.limbs - 1], 2)
        oa, ob = giants[0]
        for ga, gb in giants[1:]:
            oa, ob = ckks_np.addmod(oa, ga, ql), ckks_np.addmod(ob, gb, ql)
        return time.perf_counter() - t0, digest(oa, ob)
    finally:
        shutil.rmtree(d, ignore_errors=True)


def _init_worker():
    os.environ["OMP_NUM_THREADS"] = "1"


def cpu_pool(wait: bool = True, name: str = "C3"):
    """Fork the CPU workers BEFORE CUDA is initialised in this process."""
    workers = max(1, min(os.cpu_count() or 1, CPU_WORKERS_MAX))
    ctx = mp.get_context("fork")
    pool = ctx.Pool(workers, initializer=_init_worker)
    warm = pool.map_async(_warm, [name] * workers)
    if wait:
        warm.wait()
    return pool, workers


def cpu_sample(pool, workers, units, ks):
    t0 = time.perf_counter()
    res = pool.map(_cpu_task, list(zip(units, ks)), chunksize=1)
    wall = time.perf_counter() - t0
    return wall, res


# --------------------------------------------------------------- reference
def run_reference(args, rank: int):
    if rank != 0:
        return
    from paper_2112_06396_b200.params import config, galois_exponents
    wl = config("C3")
    p = wl.params
    allk = galois_exponents(p.n_ring, 64, SEED)
    pool, workers = cpu_pool()
    units = list(range(workers))
    ks = [allk[u % 64] for u in units]
    for _ in range(args.warmup):
        cpu_sample(pool, workers, units[:1], ks[:1])
    times = []
    for _ in range(args.steps):
        wall, _ = cpu_sample(pool, workers, units, ks)
        times.append(wall)
    pool.close()
    total = sum(times)
    value = workers * args.steps / total
    sample = f"{workers} C3 rotation key-switches per step (one per worker process), numpy port of the reference (oracle/ckks_np.py)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded counter-based residues)",
        # the same workload identification as our arm's line (run_ours)
        "config": {"workload": wl.desc, "limbs": p.limbs, "special": len(p.special), "dnum": p.dnum,
                   "log_n": p.logn, "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    from paper_2112_06396_b200 import _lib
    from paper_2112_06396_b200.digest import digest
    from paper_2112_06396_b200.params import config, galois_exponents
    from paper_2112_06396_b200.workload import RotationBatch

    pool = None
    if rank == 0 and world == 1 and not args.no_cpu:
        pool, workers = cpu_pool(wait=False)
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    lib = _lib.load()
    wl = config("C3")
    p = wl.params
    B = args.batch
    units = [rank * B + i for i in range(B)]
    allk = galois_exponents(p.n_ring, B * world, SEED)
    ks = [allk[u] for u in units]
    wb = RotationBatch(p, SEED, units, ks=ks)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        wb.run()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local_rank)
    clk.start()
    n0 = lib.ck_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        wb.run()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = lib.ck_launch_count() - n0
    barrier()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms / args.steps
    value = B * world * args.steps / (ms / 1000.0)

    # ---- roofline of the key-switch (per GPU)
    peak, peak_kind = _peaks()
    bytes_ks = ks_bytes(p)
    achieved = bytes_ks * B / (ms_step / 1000.0) / 1e9
    traffic, tr_src = args.traffic, "--traffic"
    tr_all = {}
    try:
        tr_all = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json"))).get("C3", {})
    except Exception:
        pass
    if traffic is None and tr_all:
        traffic, tr_src = tr_all["dram_bytes_per_unit"] * B, "profiles/r02_traffic.json: " + tr_all["source"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": tr_src,
                "kernel": "ck_rotate pipeline (batched key-switch, all launches of one step)",
                "algorithmic_bytes_per_unit": bytes_ks, "units_per_launch": B,
                "peak_kind": peak_kind}
    # The path is bound by the fma-heavy (IMAD) pipe, not by HBM:
    # its MEASURED utilisation, time-weighted over the step's kernels (ncu
    # sm__pipe_fmaheavy_cycles_active, committed with the launch list).
    if tr_all.get("fmaheavy_time_weighted_pct") is not None:
        roofline["int_pipe"] = {"bound": "fma-heavy pipe (IMAD)",
                                "frac": tr_all["fmaheavy_time_weighted_pct"] / 100.0,
                                "source": "ncu sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_"
                                          "elapsed per kernel, weighted by kernel time (profiles/r02_traffic.json)"}

    # ---- end to end through the public API with host buffers
    e2e = None
    ok, why = 1.0, "pinned host buffers could not be allocated on every rank"
    if not args.no_e2e:
        ins = [wb.a, wb.b, wb.key_b, wb.key_a]
        # pinned host buffers filled straight from the device (no pageable copy:
        # at N=8 every rank holds ~10 GB of inputs)
        host_in, host_out = [], []
        try:
            for t in ins:
                h = torch.empty(t.shape, dtype=torch.uint64, pin_memory=True)
                h.copy_(t)
                host_in.append(h)
            host_out = [torch.empty(wb.out_a.shape, dtype=torch.uint64, pin_memory=True) for _ in range(2)]
        except RuntimeError as exc:  # e.g. pinned host memory exhausted with many ranks
            ok, why = 0.0, "pinned host buffers: " + str(exc).splitlines()[0][:160]
        # every rank must agree before the (barrier-synchronised) e2e run
        if world > 1:
            flag = torch.tensor([ok], dtype=torch.float64, device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            ok = float(flag.item())
        del ins
    if not args.no_e2e and ok == 0.0:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "unavailable": why}
    elif not args.no_e2e:
        from paper_2112_06396_b200.ckks import HostRotationPipeline
        wb.release_inputs()  # the host pipeline owns its own device buffers
        pipe = HostRotationPipeline(p, B, chunk=args.e2e_chunk, nbuf=args.e2e_nbuf)
        ke = max(1, min(args.steps, args.e2e_steps))
        pipe.run(*host_in, wb.galois, *host_out)  # warm-up
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            pipe.run(*host_in, wb.galois, *host_out)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": B * world * ke / (ems / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": sum(t.numel() * 8 for t in host_in),
               "d2h_bytes_per_step": sum(t.numel() * 8 for t in host_out),
               "steps": ke,
               "note": ("ciphertexts AND per-rotation evaluation keys copied H2D every step "
                        f"(HostRotationPipeline, chunks of {args.e2e_chunk}, {args.e2e_nbuf} buffers, overlap PCIe with compute)")}
        # bit-exact: host outputs equal the device-resident outputs
        e2e["matches_device_outputs"] = bool(
            torch.equal(host_out[0], wb.out_a.cpu()) and torch.equal(host_out[1], wb.out_b.cpu()))
        if not args.no_compressed:
            # (chunk sizes re-measured with the faster kernels, tools/e2e_sweep.sh: chunks of 4 with
            # 6 buffers 613, 8/4 599, 16/3 569, 32/2 524 key-switches/s -- the link carries ~60 GB/s
            # for both directions together, so 4.83 GB in + 1.61 GB out bound it near 600)
            if args.e2e_chunk_compressed != args.e2e_chunk:
                del pipe
                pipe = HostRotationPipeline(p, B, chunk=args.e2e_chunk_compressed, nbuf=args.e2e_nbuf)
            comp = e2e_compressed(args, p, B, world, wb, host_in, host_out, pipe,
                                  stream, max_over_ranks, barrier, units)
            # The reference's keygen keeps rotation keys PRNG-compressed (b-rows + seed,
            # ckkslab ckks.py:308-316), so that is what a user of the public API holds on
            # the host: the compressed-key pipeline is the headline e2e, the run with
            # fully expanded (a, b) key rows over PCIe is reported beside it.
            if comp.get("value") and comp.get("matches_device_outputs"):
                comp["key_format"] = ("compressed rotation keys (b-rows + seed): the reference "
                                      "keygen's default, ckkslab ckks.py:308-316")
                comp["expanded_keys"] = e2e
                e2e = comp
            else:
                e2e["compressed_keys"] = comp

    # ---- CPU baseline (oracle port on host cores), rank 0 at N=1
    cpu = None
    if pool is not None:
        n_s = min(workers, B)
        wall, res = cpu_sample(pool, workers, units[:n_s], ks[:n_s])
        pool.close()
        torch.cuda.synchronize()
        parity = all(dg == digest(wb.out_a[i].cpu().numpy(), wb.out_b[i].cpu().numpy())
                     for i, (_, _, dg) in enumerate(res))
        cpu = {"value": n_s / wall, "unit": UNIT, "cores": workers, "kind": "port",
               "sample": f"{n_s} of the {B} C3 rotations, one per worker process (numpy port, oracle/ckks_np.py)",
               "parity_vs_gpu_bit_exact": parity}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded counter-based residues, generated on device)",
            "config": {"workload": wl.desc, "units_per_gpu_per_step": B,
                       "global_units_per_step": B * world, "limbs": p.limbs,
                       "special": len(p.special), "dnum": p.dnum, "log_n": p.logn,
                       "l2": "inputs larger than L2 (8 GB/step/GPU), no flush",
                       "parallelism": f"batch-partitioned x{world}"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()



def e2e_compressed(args, p, B, world, wb, host_in, host_out, pipe, stream, max_over_ranks,
                   barrier, units):
    """End to end with COMPRESSED rotation keys (the reference's keygen default,
    ckkslab ckks.py:310-312): per unit the host holds (a, b, key b-rows, key
    seed); only those cross PCIe and the key a-rows are expanded on the device
    with SHAKE256 (ck_expand_key_a) inside the timed region.  Same key-switch
    count and shapes as the headline e2e; the key a-rows are different values
    (XOF output instead of the counter generator), so parity is checked against
    a device-resident rotate_batch of the same compressed keys."""
    import torch
    from paper_2112_06396_b200 import ckks
    seed_root = int(p.seed).to_bytes(8, "little")
    two_n = 2 * p.n_ring
    seeds = [b"rot%d" % ((-k) % two_n) + seed_root for k in wb.ks]
    a_h, b_h, kb_h = host_in[0], host_in[1], host_in[2]
    ke = max(1, min(args.steps, args.e2e_steps))
    pipe.run(a_h, b_h, kb_h, None, wb.galois, *host_out, key_seeds=seeds)  # warm-up
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ke):
        pipe.run(a_h, b_h, kb_h, None, wb.galois, *host_out, key_seeds=seeds)
    e1.record(stream)
    torch.cuda.synchronize()
    ems = max_over_ranks(e0.elapsed_time(e1))
    seed_bytes = sum(len(x) for x in seeds) + 4 * len(seeds)
    out = {"value": B * world * ke / (ems / 1000.0), "unit": UNIT,
           "h2d_bytes_per_step": sum(t.numel() * 8 for t in (a_h, b_h, kb_h)) + seed_bytes,
           "d2h_bytes_per_step": sum(t.numel() * 8 for t in host_out), "steps": ke,
           "note": ("key b-rows + seeds over PCIe; a-rows SHAKE256-expanded on device in the timed "
                    f"region (HostRotationPipeline, chunks of {pipe.chunk})")}
    # parity: first 4 units through the device-resident path with the same keys
    m = min(4, B)
    ka = ckks.expand_key_a(p, seeds[:m])
    dev = [t[:m].cuda() for t in (a_h, b_h, kb_h)]
    oa, ob = torch.empty_like(dev[0]), torch.empty_like(dev[1])
    ckks.rotate_batch(p, dev[0], dev[1], dev[2], ka, wb.galois[:m], oa, ob)
    torch.cuda.synchronize()
    out["matches_device_outputs"] = bool(torch.equal(oa.cpu(), host_out[0][:m]) and
                                         torch.equal(ob.cpu(), host_out[1][:m]))
    return out

def _traffic(name: str):
    """ncu DRAM bytes per unit of a config from the committed launch-list summary
    (profiles/r02_traffic.json, written by tools/traffic_json.py), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
        return d[name]["dram_bytes_per_unit"], d[name]["source"]
    except Exception:
        return None, None


def run_config(args, rank: int, world: int, local_rank: int):
    """BASELINE configs C1, C2, C4, C5 and the relinearisation workload C3M: device-
    resident throughput, roofline, clocks and the CPU baseline (oracle port of the
    reference on the host cores, rank 0 at N=1) in one line."""
    pool = None
    if rank == 0 and world == 1 and not args.no_cpu:
        pool, workers = cpu_pool(wait=False, name=args.config)
    import torch
    import torch.distributed as dist
    from paper_2112_06396_b200 import _lib
    from paper_2112_06396_b200.digest import digest
    from paper_2112_06396_b200.params import config, galois_exponents
    from paper_2112_06396_b200 import workload as W

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    lib = _lib.load()
    wl = config(args.config)
    p = wl.params
    ks = None
    if wl.kind == "rotate":
        B = args.batch if args.batch_set else {"C1": 1, "C5": 32}.get(args.config, 64)
        units = [rank * B + i for i in range(B)]
        allk = galois_exponents(p.n_ring, B * world, SEED)
        # C1 is "HRotate by k=1 (Galois element 5)" (BASELINE.json configs[0])
        ks = [1] * B if args.config == "C1" else [allk[u] for u in units]
        job = W.RotationBatch(p, SEED, units, ks=ks)
        per_step, unit, bytes_unit = B, "key-switches/s", ks_bytes(p)
    elif wl.kind == "relin":
        B = args.batch
        units = [rank * B + i for i in range(B)]
        job = W.RelinBatch(p, SEED, units)
        per_step, unit, bytes_unit = B, "relinearisations/s", job.algorithmic_bytes_per_unit()
    elif wl.kind == "ntt":
        units = list(range(16))
        job = W.NttBatch(p, SEED, 16)
        per_step, unit = 16 * p.limbs, "limb NTT+INTT round trips/s"
        bytes_unit = 4 * 8 * p.n_ring
    else:
        units = [0]
        job = W.BsgsWorkload(p, SEED)
        per_step, unit, bytes_unit = 1, "BSGS transforms/s", job.algorithmic_bytes()
    for _ in range(args.warmup):
        job.run()
    torch.cuda.synchronize()
    # Launch-bound configs (C1: one N=2^12 key-switch is ~10 short kernels) replay
    # one step captured as a CUDA graph; every replay runs the full step.
    graph = None
    use_graph = args.graph if args.graph is not None else args.config == "C1"
    if use_graph:
        n_cap = lib.ck_launch_count()
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                job.run()
        torch.cuda.current_stream().wait_stream(cap)
        launches_per_step = lib.ck_launch_count() - n_cap
        if hasattr(job, "out_a"):  # the replay must redo the work: clear, replay, compare
            ref = (job.out_a.clone(), job.out_b.clone())
            job.out_a.zero_()
            job.out_b.zero_()
            graph.replay()
            torch.cuda.synchronize()
            assert torch.equal(job.out_a, ref[0]) and torch.equal(job.out_b, ref[1]), \
                "CUDA-graph replay does not reproduce the step"
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
    # inputs smaller than L2 (C1: 1.8 MB per step) -> flush L2 between timed steps
    # (a 256 MB write outside the per-step event pairs)
    in_bytes = getattr(job, "input_bytes", lambda: 1 << 40)()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if in_bytes < (256 << 20) else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local_rank)
    clk.start()
    n0 = lib.ck_launch_count()
    step = (lambda: graph.replay()) if graph is not None else job.run
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    else:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for e0, e1 in evs:
            flush.add_(1)
            e0.record()
            step()
            e1.record()
        torch.cuda.synchronize()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    launches = (launches_per_step * args.steps if graph is not None
                else lib.ck_launch_count() - n0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = clk.stop()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    peak, peak_kind = _peaks()
    ms_step = ms / args.steps
    achieved = bytes_unit * per_step / (ms_step / 1000.0) / 1e9
    tr_unit, tr_src = _traffic(args.config)
    extra = {}
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    if wl.kind == "bsgs" and rank == 0:
        extra["parity_vs_reference_digest"] = (
            digest(job.out[0].cpu().numpy(), job.out[1].cpu().numpy()) == gold["C4_bsgs"]["digest"])

    # ---- CPU baseline: the oracle port of the reference on the host cores (bounded sample)
    cpu = None
    if pool is not None:
        if wl.kind == "bsgs":
            wall, dg = cpu_c4_transform(pool)
            cpu = {"value": 1.0 / wall, "unit": unit, "cores": workers, "kind": "port",
                   "sample": "one C4 transform, hoisted (ModUp; 16 baby KSKIPs in parallel; 8 giant "
                             "groups (MAC + merged ModDown + rotation) in parallel; sum), numpy port",
                   "parity_vs_gpu_bit_exact": dg == gold["C4_bsgs"]["digest"]}
        else:
            n_s = {"C1": 8 * workers, "C2": workers}.get(args.config, workers)
            if wl.kind == "rotate":
                tasks = [(args.config, units[i % len(units)], ks[i % len(units)]) for i in range(n_s)]
            else:
                tasks = [(args.config, units[i % len(units)], None) for i in range(n_s)]
            t0 = time.perf_counter()
            res = pool.map(_cpu_unit, tasks, chunksize=1)
            wall = time.perf_counter() - t0
            per_task = p.limbs if wl.kind == "ntt" else 1
            if wl.kind == "ntt":
                parity = res[0][2] == gold["C2_ntt"]["digest"]
                what = "polynomials of 24 limbs (forward NTT then inverse, one per task)"
            else:
                outs = {u: digest(job.out_a[i].cpu().numpy(), job.out_b[i].cpu().numpy())
                        for i, u in enumerate(units)}
                parity = all(dg == outs[u] for u, _, dg in res)
                what = {"rotate": "rotation key-switches", "relin": "relinearisations"}[wl.kind]
            cpu = {"value": n_s * per_task / wall, "unit": unit, "cores": workers, "kind": "port",
                   "sample": f"{n_s} {what} of this workload, one per task on {workers} worker "
                             "processes (numpy port of the reference, oracle/ckks_np.py)",
                   "parity_vs_gpu_bit_exact": parity}
        pool.close()
    if rank == 0:
        print(json.dumps({
            "metric": f"{unit} ({args.config})", "value": per_step * world * args.steps / (ms / 1000.0),
            "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded, generated on device)",
            "config": {"workload": wl.desc, "units_per_gpu_per_step": per_step,
                       "global_units_per_step": per_step * world, "cuda_graph": graph is not None,
                       "l2": ("flushed between timed steps (256 MB write outside the events)"
                              if flush is not None else "inputs larger than L2, no flush")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": tr_unit * per_step if tr_unit else None, "traffic_source": tr_src,
                         "algorithmic_bytes_per_unit": bytes_unit, "units_per_launch": per_step,
                         "peak_kind": peak_kind},
            "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clocks, **extra}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without torchrun: start N ranks of this script, one per
    GPU (RANK / LOCAL_RANK = 0..N-1, rendezvous on 127.0.0.1), exactly as
    `torch.distributed.run --nproc-per-node N` would; rank 0 prints the line."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    return max(abs(pr.wait()) for pr in procs)


def run_selftest(args, rank: int, world: int):
    """CPU stand-in for the multi-rank harness (gloo): the same rank layout,
    barrier-bracketed timed region, max-over-ranks reduction and JSON line as
    run_ours, with each rank's 'step' a fixed host delay instead of the GPU
    key-switch.  Lets a CPU test check the launcher and the aggregation."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    B = args.batch
    units = [rank * B + i for i in range(B)]
    for _ in range(args.warmup):
        time.sleep(0.001)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(0.002 * (1 + rank))  # ranks differ: the max must win
    ms = 1000 * (time.perf_counter() - t0)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        seen = torch.tensor([len(units)], dtype=torch.int64)
        dist.all_reduce(seen)
        total_units = int(seen.item())
    else:
        total_units = len(units)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": total_units * args.steps / (ms / 1000.0),
                          "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms / args.steps, "selftest": True,
                          "config": {"units_per_gpu_per_step": B, "global_units_per_step": total_units,
                                     "parallelism": f"batch-partitioned x{world}"}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C3M", "C4", "C5"])
    ap.add_argument("--graph", type=int, default=None,
                    help="replay a CUDA-graph capture of one step (non-C3 configs; default: C1 only)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=4)
    ap.add_argument("--e2e-chunk-compressed", type=int, default=4)
    ap.add_argument("--e2e-nbuf", type=int, default=6, help="device chunk buffers in the host pipeline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-compressed", action="store_true",
                    help="skip the compressed-key variant of the end-to-end measurement")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch (default: profiles/r01_traffic.json x units)")
    ap.add_argument("--selftest-cpu", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to "
                         "report a world size that was not launched")
    args.batch_set = args.batch is not None
    if args.batch is None:
        args.batch = 64
    if args.selftest_cpu:
        run_selftest(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if args.config != "C3":
        run_config(args, rank, world, local_rank)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
