"""Run full-size golden cases by name (for compute-sanitizer runs): python tools/sanitize_case.py C2_ntt ..."""
import os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"), os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")]
import json, cases
from gpu_backend import GpuRotateBackend
from paper_2112_06396_b200.digest import digest
gold = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "golden.json")))
full = {c.name: c for c in cases.all_cases() if not c.full}
for n in sys.argv[1:]:
    ok = digest(*cases.run_case(full[n], GpuRotateBackend())) == gold[n]["digest"]
    print(n, ok)
