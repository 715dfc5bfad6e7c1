"""Every implementation variant stays bit-exact on the full-size C2/C3/C5 golden
digests: the NTT column phase on tcgen05 (default: forward and inverse),
forward-only (CKB200_NTTTC=2) or on CUDA-core butterflies (CKB200_NTTTC=0,
also with FP64-assisted twiddles, CKB200_FPNTT=1); and the opt-in pipeline
variants kept for measurement: unfused key-switch (CKB200_UNFUSED=1),
warp-specialised ks_row (CKB200_KSWS=1), special-row INTT inside ks_row
(CKB200_KSINTT=1), BC fused with the column phase (CKB200_BCCOL=1), CUDA-core
BC (CKB200_BCTC=0), chunked multi-stream batches (CKB200_CHUNK/STREAMS),
plain launches instead of programmatic dependent launch (CKB200_PDL=0).
Variants are read at plan creation, so each runs in a fresh process."""

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


VARIANTS = {
    "ntt_tc": {},
    "ntt_tc_fwd_only": {"CKB200_NTTTC": "2"},
    "butterflies": {"CKB200_NTTTC": "0"},
    "butterflies_fp64_twiddles": {"CKB200_NTTTC": "0", "CKB200_FPNTT": "1"},
    "unfused": {"CKB200_UNFUSED": "1"},
    "ks_row_warp_specialised": {"CKB200_KSWS": "1"},
    "ks_row_inline_special_intt": {"CKB200_KSINTT": "1"},
    "bc_fused_with_column_phase": {"CKB200_BCCOL": "1", "CKB200_NTTTC": "0"},
    "bc_cuda_cores": {"CKB200_BCTC": "0"},
    "chunked_two_streams": {"CKB200_CHUNK": "16", "CKB200_STREAMS": "2"},
    "no_programmatic_dependent_launch": {"CKB200_PDL": "0"},
}


@pytest.mark.parametrize("name", list(VARIANTS))
def test_variant_bit_exact(name):
    env = dict(os.environ, **VARIANTS[name])
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
