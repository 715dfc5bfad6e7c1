"""The roofline accounting bench.py reports (CPU-only): compulsory bytes per
key-switch must equal SURVEY 8(d)'s figures, and the IMAD-slot model must stay
positive and scale with the ring."""

import importlib.util
import os

from paper_2112_06396_b200.params import config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)


def test_compulsory_bytes_match_survey():
    # 8 N (l [a] + l [b] + 2 beta (l+K) [evk a,b rows] + 2 l [out]) -- SURVEY 8(d)
    assert bench.ks_bytes(config("C1").params) == 1_835_008
    assert bench.ks_bytes(config("C3").params) == 150_994_944
    assert bench.ks_bytes(config("C5").params) == 528_482_304


def test_int_slot_model_scales():
    c3 = bench.int_slots_per_ks(config("C3").params)
    c5 = bench.int_slots_per_ks(config("C5").params)
    assert 1e9 < c3 < 1e10
    assert c5 > 3 * c3
