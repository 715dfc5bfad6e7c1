"""Reference wire-format blobs (serialize.py) for the GPU ingestion tests.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_wire.py

Writes tests/golden/wire.npz: byte blobs produced by the REFERENCE's
serialize.{poly,ciphertext,switching_key}_to_bytes for seeded toy objects
(a compressed and an expanded switching key), plus the arrays they hold.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from ckkslab import ckks, rnspoly, serialize  # noqa: E402  (the reference)

import cases  # noqa: E402
import xof_cases  # noqa: E402
from paper_2112_06396_b200 import synth  # noqa: E402


def main():
    p = cases.make_params(cases.TOY_A)
    a = cases._rows(p, 0, synth.TAG_CT_A, p.chain)
    b = cases._rows(p, 0, synth.TAG_CT_B, p.chain)
    poly = rnspoly.RnsPoly(tuple(p.chain), a, "eval")
    ct = ckks.Ciphertext(poly, rnspoly.RnsPoly(tuple(p.chain), b, "eval"), 1099511627776.0 * 3)
    kb, ka = synth.switching_key(p, cases.SEED, 1005)
    comp = ckks.SwitchingKey(tuple(p.full_moduli), kb, seed=xof_cases.KEY_SEEDS[0])
    full = ckks.SwitchingKey(tuple(p.full_moduli), kb, seed=None, a=ka)
    blobs = {"poly": serialize.poly_to_bytes(poly), "ct": serialize.ciphertext_to_bytes(ct),
             "ksk_comp": serialize.switching_key_to_bytes(comp),
             "ksk_full": serialize.switching_key_to_bytes(full)}
    out = {f"blob/{k}": np.frombuffer(v, dtype=np.uint8) for k, v in blobs.items()}
    out.update({"a": a, "b": b, "kb": kb, "ka": ka, "ka_comp": comp.expand().a})
    np.savez_compressed(os.path.join(HERE, "wire.npz"), **out)
    print({k: len(v) for k, v in blobs.items()})


if __name__ == "__main__":
    main()
