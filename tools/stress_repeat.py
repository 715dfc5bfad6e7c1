"""Determinism stress (race detection by repetition; compute-sanitizer is closed on the GPU pool).

Runs each device workload R times from identical inputs and compares every output with the
first run's, bit for bit, on the device.  The first run's correctness is the parity tests'
job; a data race (e.g. a missing proxy fence in front of a TMA refill, a stale TMEM read)
shows up here as a run that differs.  Single launches on an otherwise idle GPU and full
batches both run, because the two expose different interleavings.

    python tools/stress_repeat.py [R]
"""
import os
import sys
import time

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import torch

from paper_2112_06396_b200 import workload
from paper_2112_06396_b200.params import config

R = int(sys.argv[1]) if len(sys.argv) > 1 else 200
SEED = 20211206


def outs(job):
    if hasattr(job, "out_a"):
        return (job.out_a, job.out_b)
    if hasattr(job, "out"):
        return tuple(job.out)
    return (job.x,)


def stress(name, job, reps, restore=None):
    job.run()
    torch.cuda.synchronize()
    first = [o.clone() for o in outs(job)]
    bad = 0
    t0 = time.time()
    for _ in range(reps):
        if restore is not None:
            restore()
        for o in outs(job):
            if restore is None:
                o.zero_()
        job.run()
        torch.cuda.synchronize()
        bad += 0 if all(torch.equal(o, f) for o, f in zip(outs(job), first)) else 1
    print(f"{name:34s} runs={reps:4d} differing={bad}  ({time.time() - t0:.1f} s)", flush=True)
    return bad


def main():
    bad = 0
    for cfg in ("C3", "C5"):
        p = config(cfg).params
        for units in ([0], [0, 1], list(range(5)), list(range(16))):
            reps = R if len(units) < 16 else max(R // 8, 10)
            bad += stress(f"{cfg} rotate batch={len(units)}", workload.RotationBatch(p, SEED, units), reps)
            torch.cuda.empty_cache()
        for units in ([0], list(range(4))):
            bad += stress(f"{cfg} relin batch={len(units)}", workload.RelinBatch(p, SEED, units), R)
            torch.cuda.empty_cache()
    p = config("C3").params
    bad += stress("C3 rotate batch=64", workload.RotationBatch(p, SEED, list(range(64))), max(R // 10, 10))
    torch.cuda.empty_cache()
    bad += stress("C4 bsgs 16x8", workload.BsgsWorkload(config("C4").params, SEED), max(R // 4, 10))
    torch.cuda.empty_cache()
    nb = workload.NttBatch(config("C2").params, SEED, 16)
    x0 = nb.x.clone()
    bad += stress("C2 ntt+intt batch=16", nb, R, restore=lambda: nb.x.copy_(x0))
    p1 = config("C1").params
    bad += stress("C1 rotate batch=1", workload.RotationBatch(p1, SEED, [0]), 4 * R)
    print("TOTAL differing runs:", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
