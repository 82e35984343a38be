"""A short randomised differential run (tools/fuzz_parity.py) as a GPU test:
20 s of random lane products / closures and Boolean products / closures through
the public classes, each compared bit for bit with the CPU oracle."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_fuzz_parity_short():
    r = subprocess.run([sys.executable, str(REPO / "tools" / "fuzz_parity.py"), "20", "5"], cwd=REPO,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    summary = json.loads(lines[-1])
    assert summary["failures"] == 0, "\n".join(lines[-10:])
    assert sum(summary["cases"].values()) > 100
