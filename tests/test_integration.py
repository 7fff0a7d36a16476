"""The reference-side adapter (integration/kinetics_b200_adapter.cpp) compiles
against the reference's own headers and the C ABI (CPU only)."""
import shutil
import subprocess
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
REF_INC = Path("/root/reference/proj/include")


@pytest.mark.skipif(not REF_INC.exists(), reason="reference headers not present")
def test_adapter_compiles_against_reference_headers(tmp_path):
    cxx = shutil.which("g++") or "g++"
    r = subprocess.run([cxx, "-std=c++20", "-fsyntax-only", f"-I{REF_INC}", f"-I{REPO / 'include'}",
                        str(REPO / "integration" / "kinetics_b200_adapter.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_abi_header_is_plain_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "kin_abi.h"\nint main(void){kin_sweep_desc d; (void)d; return kin_abi_version() == KIN_ABI_VERSION ? 0 : 1;}\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", f"-I{REPO / 'include'}", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
