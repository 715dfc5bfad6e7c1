"""Shared loader for tests/golden/polyeval.npz (make_golden_polyeval.py): the
reference's sine evaluation, full bootstrap and new_mult unit cases on the
same BootstrapPlan / keys as tests/golden/boot.npz."""

import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class PolyEval:
    def __init__(self):
        self.meta = json.load(open(os.path.join(HERE, "polyeval.json")))
        self.z = np.load(os.path.join(HERE, "polyeval.npz"))

    def pair(self, name):
        return self.z[name + "/a"], self.z[name + "/b"]

    def delta(self, name) -> float:
        return self.meta["deltas"][name]
