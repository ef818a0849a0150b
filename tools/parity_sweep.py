"""Runs the config parity sweep (tests/sweep.py) on cuda:0 against the literal
reference and writes the JSON report: python tools/parity_sweep.py OUT.json"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import paper_2012_10802_b200 as pkg  # noqa: E402
from paper_2012_10802_b200.api import Library  # noqa: E402
from sweep import run_sweep, sweep_cases  # noqa: E402

gpu = pkg.load_library().context(0)
ref = Library(str(ROOT / "oracle" / "_ref" / "librpd_ref.so"))
report = run_sweep(gpu, ref, sweep_cases())
Path(sys.argv[1]).write_text(json.dumps(report, indent=1))
print(json.dumps(report["summary"]))
