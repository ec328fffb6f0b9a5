"""C-ABI boundary checks that need no GPU: the library builds for sm_100a, loads, and exports every
entry point include/lpfem.h declares; context creation without a device fails loudly (no CPU fallback)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lpfem.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lpfem_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def built():
    from paper_2311_05170_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("lpfem_create", "lpfem_step", "lpfem_get_fields", "lpfem_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (lpfem_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    import paper_2311_05170_b200 as P
    assert sorted(P.SYMBOLS) == declared_symbols()


def test_library_is_sm100a(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_loads_and_reports_status_strings(built):
    import paper_2311_05170_b200 as P
    L = P.lib()
    assert L.lpfem_status_string(0) == b"ok"
    assert L.lpfem_status_string(4) == b"solver did not converge"


def test_create_without_gpu_fails_loudly(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import lpfem_inputs as I
    import paper_2311_05170_b200 as P
    with pytest.raises(P.LPFEMError):
        P.LPFEM(I.config(0))


def test_create_rejects_bad_sizes(built):
    import lpfem_inputs as I
    import paper_2311_05170_b200 as P
    with pytest.raises(P.LPFEMError) as e:
        P.LPFEM(I.config(0, h=1 / 16.5))
    assert e.value.status in (1, 2, 3, 5)
