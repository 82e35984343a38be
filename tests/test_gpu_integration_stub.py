"""The reference-side binding in INTEGRATION.md, executed as written: the
ctypes stubs a maintainer would drop into semimat/antidist.py in place of
_mul_vector (antidist.py:361-371) and _close_vector (:390-398, the device
copy and the one-call host-buffer versions) must give the oracle's bytes on
the reference's own numpy storage.
"""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from paper_1705_08743_b200 import _build, workloads

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent


def _stub_blocks():
    text = (REPO / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    return [b for b in blocks if "_close_vector" in b]


def test_integration_stubs_match_oracle(oracle_lib):
    first, host = _stub_blocks()
    ns: dict = {}
    exec(first.replace("/path/to/libsemimat_b200.so", str(_build.LIB)), ns)
    cfg = workloads.CONFIGS["c4_fw_u16"]
    (t,) = workloads.make_inputs(cfg, 1100)
    want = oracle_lib.semiring_close(t, 16, "anti")

    dev = t.copy()
    ns["_close_vector"](dev, 1100, 65535)                  # device-copy stub
    np.testing.assert_array_equal(dev, want)

    c3 = workloads.CONFIGS["c3_mul_u16"]
    a, b = workloads.make_inputs(c3, 600)
    got = ns["_mul_vector"](a, b, 600, 65535)
    np.testing.assert_array_equal(got, oracle_lib.semiring_mul(a, b, 600, 16, "anti"))

    exec(host, ns)                                          # one-call host-buffer stub
    hb = t.copy()
    ns["_close_vector"](hb, 1100, 65535)
    np.testing.assert_array_equal(hb, want)
