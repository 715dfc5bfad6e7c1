"""Time on-device compressed-key expansion (ck_expand_key_a) at C3 shapes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2112_06396_b200 import ckks
from paper_2112_06396_b200.params import config

p = config("C3").params
for nk in (1, 8, 64):
    seeds = [b"rot%d" % k + (1).to_bytes(8, "little") for k in range(nk)]
    out = ckks.expand_key_a(p, seeds)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 3
    for _ in range(reps):
        ckks.expand_key_a(p, seeds, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"keys={nk} rows={nk * 96} ms={ms:.2f} keys/s={nk / ms * 1e3:.0f} "
          f"GB/s_out={out.numel() * 8 / ms / 1e6:.1f}", flush=True)
