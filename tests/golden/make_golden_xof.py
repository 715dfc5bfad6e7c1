"""Generate the compressed-key golden fixtures by running the REFERENCE itself.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_xof.py

Writes tests/golden/xof.json (sha256 digests) and tests/golden/xof.npz (small
rows): ckks._xof_uniform for every XOF_ROWS case, SwitchingKey(seed).expand()
for the toy basis and the C3 basis, and a reference hrotate with a COMPRESSED
rotation key (the a-rows regenerated inside _kskip via a_row, ckks.py:450-465).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from ckkslab import ckks  # noqa: E402  (the reference)

import cases  # noqa: E402
import make_golden  # noqa: E402
import xof_cases  # noqa: E402
from paper_2112_06396_b200 import synth  # noqa: E402
from paper_2112_06396_b200.digest import digest  # noqa: E402
from paper_2112_06396_b200.params import config  # noqa: E402


def main():
    gold, arrs = {}, {}
    for i, (seed, tag, q, n) in enumerate(xof_cases.XOF_ROWS):
        row = ckks._xof_uniform(seed, tag, q, n)
        gold[f"row{i}"] = digest(row)
        if n <= 5000:
            arrs[f"row{i}"] = row
    for name, p in (("toyA", cases.make_params(cases.TOY_A)), ("C3", config("C3").params)):
        dn = len(p.digit_spans(p.limbs))
        b = np.zeros((dn, len(p.full_moduli), p.n_ring), dtype=np.uint64)
        for k, seed in enumerate(xof_cases.KEY_SEEDS):
            key = ckks.SwitchingKey(tuple(p.full_moduli), b, seed=seed)
            assert key.compressed
            a = key.expand().a
            gold[f"key_{name}_{k}"] = digest(a)
            if name == "toyA":
                arrs[f"key_{name}_{k}"] = a
    # hrotate with a compressed key on TOY_A at the top level
    p = cases.make_params(cases.TOY_A)
    a = cases._rows(p, 0, synth.TAG_CT_A, p.chain)
    bb = cases._rows(p, 0, synth.TAG_CT_B, p.chain)
    kb, _ = synth.switching_key(p, cases.SEED, 1005)
    ks = make_golden._keyset(p)
    ks.rot[5] = ckks.SwitchingKey(tuple(p.full_moduli), kb, seed=xof_cases.KEY_SEEDS[0])
    out = ckks.hrotate(make_golden._ref_params(p), ks, RefCt(p, a, bb), (5,))[0]
    gold["hrot_compressed_toyA"] = digest(out.a.data, out.b.data)
    arrs["hrot_compressed_toyA/0"] = out.a.data
    arrs["hrot_compressed_toyA/1"] = out.b.data
    json.dump(gold, open(os.path.join(HERE, "xof.json"), "w"), indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "xof.npz"), **arrs)
    print("wrote", len(gold), "digests")


def RefCt(p, a, b):
    return make_golden.RefBackend()._ct(p, a, b)


if __name__ == "__main__":
    main()
