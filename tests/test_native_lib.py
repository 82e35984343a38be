"""The C-ABI library builds for sm_100a, loads, and exports every declared
symbol (CPU only: nothing here launches a kernel)."""

from __future__ import annotations

import re
import subprocess

from paper_1705_08743_b200 import _build, _native

from conftest import REPO


def header_symbols():
    text = (REPO / "include" / "semimat_b200.h").read_text()
    return sorted(set(re.findall(r"\b(smx_\w+)\s*\(", text)))


def test_library_builds_and_loads():
    path = _build.build()
    assert path.exists()
    lib = _native.lib()
    assert lib.smx_version() >= 100


def test_exports_every_header_symbol():
    _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_build.LIB)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (smx_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, f"declared in include/semimat_b200.h but not exported: {missing}"


def test_binding_covers_header():
    assert set(header_symbols()) <= set(_native.declared_symbols())


def test_error_strings():
    lib = _native.lib()
    assert lib.smx_error_string(0) == b"ok"
    assert b"aligned" in lib.smx_error_string(-2)


def test_sm100a_cubin_and_native_instructions():
    """The library carries sm_100a SASS with the native packed-integer ops."""
    _build.build()
    sass = subprocess.run(["cuobjdump", "-sass", str(_build.LIB)], capture_output=True, text=True,
                          check=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(_build.LIB)], capture_output=True,
                                       text=True).stdout or "SM100" in sass.upper()
    assert "VIADDMNMX.U16x2" in sass
    assert "VIMNMX.U16x2" in sass


def test_hot_kernels_use_blackwell_paths():
    """Per-kernel SASS: the packed semiring kernel streams tiles with bulk
    async copies and mbarriers and updates with VIADDMNMX.U16x2; the Boolean
    tensor-core kernel issues tcgen05 MMAs fed by TMA and reads TMEM."""
    _build.build()
    import sys
    sys.path.insert(0, str(_build.REPO / "tools"))
    from sass_census import census
    funcs = census(_build.LIB)
    packed = [c for name, c in funcs.items() if "packed_gemm_kernelIt" in name]
    tc = [c for name, c in funcs.items() if "bool_i8_gemm_kernel" in name]
    assert packed and tc
    for c in packed:
        assert c["UBLKCP"] > 0 and c["SYNCS.PHASECHK.TRANS64.TRYWAIT"] > 0 and c["VIADDMNMX.U16x2"] > 0
    for c in tc:
        # kind::i8 instantiations issue UTCIMMA, the E2M1 (kind::mxf4) ones UTCOMMA
        assert c["UTCIMMA"] + c["UTCOMMA"] > 0 and c["UTMALDG"] > 0 and c["LDTM"] > 0
    assert any(c["UTCIMMA"] for c in tc) and any(c["UTCOMMA"] for c in tc)
