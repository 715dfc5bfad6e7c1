"""GPU product vs the reference goldens and the CPU oracle (bit-exact).

Every call goes Python mirror -> C ABI (libckks_b200.so) -> CUDA kernels.
"""

import json
import os

import numpy as np
import pytest

import cases
from gpu_backend import GpuBackend, GpuRotateBackend
from paper_2112_06396_b200.digest import digest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLD = json.load(open(os.path.join(HERE, "golden.json")))
TOY = np.load(os.path.join(HERE, "toy.npz"))

TOY_CASES = [c for c in cases.all_cases() if c.full]
FULL = {c.name: c for c in cases.all_cases() if not c.full}


def _check_toy(case, out):
    for i, o in enumerate(out):
        want = TOY[f"{case.name}/{i}"]
        if not np.array_equal(o, want):
            bad = np.argwhere(o != want)
            raise AssertionError(f"{case.name}[{i}]: {len(bad)} mismatches, first {bad[:3].tolist()}")
    assert digest(*out) == GOLD[case.name]["digest"]


@pytest.mark.parametrize("case", TOY_CASES, ids=lambda c: c.name)
def test_toy_case_bit_exact(case):
    _check_toy(case, cases.run_case(case, GpuBackend()))


@pytest.mark.parametrize("case", [c for c in TOY_CASES if c.op in ("hrotate", "conjugate")],
                         ids=lambda c: c.name)
def test_toy_case_fused_rotate_entry(case):
    _check_toy(case, cases.run_case(case, GpuRotateBackend()))


@pytest.mark.parametrize("name", ["C1_rot", "C2_ntt", "C2_intt", "C2_ntt_b16", "C2_intt_b16",
                                  "C3_rot0", "C3_rot1", "C3_rot63", "C3_conj", "C3_hrot16",
                                  "C3_new_mult", "C5_rot0", "C5_rot255"])
def test_full_config_digest(name):
    out = cases.run_case(FULL[name], GpuRotateBackend())
    assert digest(*out) == GOLD[name]["digest"], name


def test_c3_hrotate_shared_modup_digest():
    """hrotate path (shared ModUp + per-rotation KSKIP/ModDown) at full C3 size."""
    out = cases.run_case(FULL["C3_rot1"], GpuBackend())
    assert digest(*out) == GOLD["C3_rot1"]["digest"]


def test_c4_bsgs_digest():
    out = cases.run_case(FULL["C4_bsgs"], GpuBackend())
    assert digest(*out) == GOLD["C4_bsgs"]["digest"]
