"""Every NTT column-phase implementation stays bit-exact: the tcgen05 kernels
(default: forward and inverse), forward-only (CKB200_NTTTC=2) and the CUDA-core
butterflies (CKB200_NTTTC=0).  The mode is read at plan creation, so each runs
in a fresh process on the full-size C2/C3/C5 golden digests."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, os, sys
sys.path[:0] = [{root!r}, os.path.join({root!r}, "tests"), os.path.join({root!r}, "tests", "golden")]
import cases
from gpu_backend import GpuRotateBackend
from paper_2112_06396_b200.digest import digest
gold = json.load(open(os.path.join({root!r}, "tests", "golden", "golden.json")))
full = {{c.name: c for c in cases.all_cases() if not c.full}}
bad = [n for n in ("C2_ntt", "C2_intt", "C3_rot0", "C3_rot63", "C3_new_mult", "C5_rot0")
       if digest(*cases.run_case(full[n], GpuRotateBackend())) != gold[n]["digest"]]
print("BAD", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("mode", ["0", "2", "1"])
def test_column_phase_modes_bit_exact(mode):
    env = dict(os.environ, CKB200_NTTTC=mode)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
