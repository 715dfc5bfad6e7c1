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


def test_relin_bytes():
    from paper_2112_06396_b200.workload import relin_bytes
    p = config("C3M").params
    # (3 x 24 + 2 x 23) limbs of 512 KiB + the 192-limb key shared by 64 units
    assert relin_bytes(p, 24, 64) == 118 * 524_288 + 192 * 524_288 // 64
    assert relin_bytes(p, 24, 1) == (118 + 192) * 524_288


def test_traffic_summary_tool(tmp_path):
    """tools/traffic_json.py: the last K launches of an ncu list are one step."""
    import csv
    import json
    import subprocess
    import sys
    path = tmp_path / "l.csv"
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"])
        for i in range(4):
            w.writerow([i, f"k{i % 2}(Args)", "gpu__time_duration.sum", "ns", "1000"])
            w.writerow([i, f"k{i % 2}(Args)", "dram__bytes_read.sum", "byte", str(100 * (i + 1))])
            w.writerow([i, f"k{i % 2}(Args)", "dram__bytes_write.sum", "byte", "10"])
    out = tmp_path / "t.json"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "traffic_json.py"), str(out),
                    f"X:{path}:2:4"], check=True, capture_output=True)
    d = json.load(open(out))["X"]
    assert d["dram_bytes_per_unit"] == (300 + 400 + 20) / 4
    assert d["step_time_us"] == 2.0
