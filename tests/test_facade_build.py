"""The C++ facade compiles against the reference headers (CPU-only check)."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT

REF_INC = "/root/reference/proj/core/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_facade_compiles_against_reference_headers(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "uot/cuda.hpp"\nint main() { return 0; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                        f"-I{REF_INC}", f"-I{os.path.join(ROOT, 'include')}", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
