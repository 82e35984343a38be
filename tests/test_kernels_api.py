"""The device-backed `kernels` module keeps the reference's list API and its
validation (pkg/src/semimat/kernels.py:41-204).  CPU only: every case here
raises before any device work, or only queries path state."""

from __future__ import annotations

import pytest

from paper_1705_08743_b200 import kernels


def test_lane_geometry():
    assert [kernels.lane_count(w) for w in (8, 16, 32)] == [16, 8, 4]
    assert kernels.dtype_for(16).__name__ == "uint16"
    with pytest.raises(ValueError):
        kernels.lane_count(12)


def test_validation_messages_match_reference():
    with pytest.raises(ValueError, match=r"lane value outside \[0, 255\]"):
        kernels.subsat([256] + [0] * 15, [0] * 16, 8)
    with pytest.raises(ValueError, match=r"lane value outside \[0, 255\]"):
        kernels.addsat([0] * 16, [-1] + [0] * 15, 8)
    with pytest.raises(ValueError, match="expected a flat sequence of a multiple of 8 lanes"):
        kernels.maxlanes([1, 2, 3], [1, 2, 3], 16)
    with pytest.raises(ValueError, match="lane count mismatch: 16 vs 8"):
        kernels.minlanes([0] * 16, [0] * 8, 16)
    with pytest.raises(ValueError, match="count must be a positive multiple of 4, got 6"):
        kernels.clonenot(1, 32, count=6)
    with pytest.raises(ValueError, match=r"lane value 300 outside \[0, 255\]"):
        kernels.clonenot(300, 8)


def test_path_state_mirrors_reference(monkeypatch):
    monkeypatch.delenv(kernels.FORCE_SCALAR_ENV, raising=False)
    assert kernels.use_vector() == kernels.vector_supported()
    monkeypatch.setenv(kernels.FORCE_SCALAR_ENV, "1")
    assert kernels.use_vector() is False
    with kernels.forced_vector():
        assert kernels.use_vector() is True
        with kernels.forced_scalar():
            assert kernels.use_vector() is False
        assert kernels.use_vector() is True
    monkeypatch.setenv(kernels.FORCE_SCALAR_ENV, "0")
    assert kernels.use_vector() == kernels.vector_supported()


def test_np_addsat_requires_the_lane_limit():
    import numpy as np
    with pytest.raises(ValueError, match="lane limit"):
        kernels.np_addsat(np.zeros(4, np.uint8), np.zeros(4, np.uint8), 100)
