"""Where does the host-pipeline time go?  PCIe alone vs the pipeline (C3, 64 units)."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2112_06396_b200 import ckks
from paper_2112_06396_b200.params import config
from paper_2112_06396_b200.workload import RotationBatch

cfg = config("C3")
p = cfg.params
B = 64
wb = RotationBatch(p, 1, range(B))
host = {k: torch.empty(t.shape, dtype=torch.uint64, pin_memory=True).copy_(t)
        for k, t in (("a", wb.a), ("b", wb.b), ("kb", wb.key_b), ("ka", wb.key_a))}
outs = [torch.empty(wb.out_a.shape, dtype=torch.uint64, pin_memory=True) for _ in range(2)]
dev = {k: torch.empty_like(wb.a if k in "ab" else wb.key_b) for k in host}
wb.release_inputs()


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d(names):
    def f():
        for n in names:
            dev[n].copy_(host[n], non_blocking=True)
    return f


for names in (("a", "b", "kb"), ("a", "b", "kb", "ka")):
    ms = timed(h2d(names))
    gb = sum(host[n].numel() * 8 for n in names) / 1e9
    print(f"H2D {names}: {ms:.1f} ms  {gb / ms * 1e3:.1f} GB/s", flush=True)
ms = timed(lambda: [o.copy_(wb.out_a, non_blocking=True) for o in outs])
print(f"D2H outs: {ms:.1f} ms {2 * wb.out_a.numel() * 8 / ms / 1e6:.1f} GB/s", flush=True)
s2 = torch.cuda.Stream()


def both():
    with torch.cuda.stream(s2):
        for o in outs:
            o.copy_(wb.out_a, non_blocking=True)
    h2d(("a", "b", "kb"))()
    torch.cuda.current_stream().wait_stream(s2)


ms = timed(both)
print(f"H2D(a,b,kb) || D2H(outs): {ms:.1f} ms", flush=True)
seeds = [b"rot%d" % k for k in range(B)]
ms = timed(lambda: ckks.expand_key_a(p, seeds))
print(f"expand 64 keys: {ms:.1f} ms", flush=True)
for chunk, nb in ((8, 4), (4, 8)):
    pipe = ckks.HostRotationPipeline(p, B, chunk=chunk, nbuf=nb)
    ms = timed(lambda: pipe.run(host["a"], host["b"], host["kb"], None, wb.galois, *outs,
                                key_seeds=seeds))
    print(f"pipeline compressed chunk={chunk} nbuf={nb}: {ms:.1f} ms -> {B / ms * 1e3:.0f} ks/s", flush=True)
    ms = timed(lambda: pipe.run(host["a"], host["b"], host["kb"], host["ka"], wb.galois, *outs))
    print(f"pipeline expanded   chunk={chunk} nbuf={nb}: {ms:.1f} ms -> {B / ms * 1e3:.0f} ks/s", flush=True)
    del pipe
