"""Randomised parity regression (tools/fuzz_parity.py with a fixed seed, small sizes):
random N, D = 1..8, parameters across their valid ranges, ties, clustered / spread /
offset locations, both precisions, both decompositions and emulated worlds, each against
the oracle under the tolerance rule."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_fuzz_parity_fixed_seed():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"), "--cases", "60",
                          "--seed", "11", "--nmax", "1500"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    summary = lines[-1]
    assert summary.get("summary") and summary["fails"] == 0, lines[:-1]
