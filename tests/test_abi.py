"""CPU-side checks of the C-ABI boundary: the library builds, loads, and exports every symbol include/gwas.h
declares (no compute calls without a GPU)."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gwas.h")).read()
    return sorted(set(re.findall(r"GWAS_API[^;{]*?\b(gwas_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ["gwas_setup", "gwas_attach", "gwas_run", "gwas_state_bytes", "gwas_workspace_bytes",
                     "gwas_timings", "gwas_destroy", "gwas_last_error"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1207_2169_b200 import build
    lib = build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(gwas_\w+)\b", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    from paper_1207_2169_b200 import _lib
    assert sorted(_lib.EXPORTS) == _declared()
    for n in _declared():
        assert hasattr(_lib.lib, n)


def test_library_is_sm100a_and_uses_dmma_and_tma():
    from paper_1207_2169_b200 import build
    lib = build.build()
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", lib], capture_output=True, text=True).stdout or "sm_100a" in sass
    assert "DMMA" in sass          # FP64 tensor-core MMA (K1/K2)
    assert "UTMALDG" in sass       # TMA tile loads


def test_pure_host_calls_without_gpu():
    import ctypes as C
    from paper_1207_2169_b200 import _lib
    o = _lib.default_options()
    assert o.block_cols == 8192 and o.xr_dtype == _lib.XR_U8 and abs(o.eps_spd - 1e-10) < 1e-25
    n, p, t = 10_000, 5, 1000
    sb = _lib.lib.gwas_state_bytes(n, p, t, C.byref(o))
    # Z + B2 dominate: 8 (kpad^2 + n2 kpad)
    assert sb >= 8 * (10_000 ** 2 + (1000 * 6 + 1000) * 10_000)
    assert _lib.lib.gwas_state_bytes(3, 5, 1, C.byref(o)) == 0        # n < p + 1
    assert b"n = 3" in _lib.lib.gwas_last_error()
    assert _lib.lib.gwas_version().startswith(b"gwas")
