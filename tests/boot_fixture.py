"""Shared loader for tests/golden/boot.npz (make_golden_boot.py): a real
reference BootstrapPlan's CoeffToSlot / SlotToCoeff stages with reference keys."""

import json
import os

import numpy as np

from paper_2112_06396_b200.params import CkksParams

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Boot:
    def __init__(self):
        self.meta = json.load(open(os.path.join(HERE, "boot.json")))
        self.z = np.load(os.path.join(HERE, "boot.npz"))
        m = self.meta
        self.params = CkksParams(m["logn"], tuple(m["chain"]), tuple(m["special"]), m["dnum"],
                                 m["delta"], m["seed"])
        self.seed_root = int(m["seed"]).to_bytes(8, "little")

    def key_seed(self, r: int) -> bytes:
        return b"rot%d" % (r % (2 * self.params.n_ring)) + self.seed_root

    def key_b(self, r) -> np.ndarray:
        return self.z[f"key_b/{r}"]

    def stage_diags(self, kind: str, si: int) -> dict:
        st = self.meta[kind][si]
        return {o: self.z[f"{kind}{si}/diag/{o}"] for o in st["offsets"]}
