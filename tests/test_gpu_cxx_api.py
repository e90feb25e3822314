"""GPU: the reference-shaped C++ API (include/gmi_b200/gmi.hpp over
libgmi_b200_cxx.so) — restated reference unit tests compiled as a C++
program against the drop-in library (tests/cxx/test_cxx_api.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cxx_api_program(gmi, tmp_path):
    lib = os.path.join(ROOT, "paper_2012_13257_b200", "lib")
    exe = str(tmp_path / "test_cxx_api")
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cxx", "test_cxx_api.cpp"), "-o", exe,
                    f"-L{lib}", "-lgmi_b200_cxx", "-lgmi_b200", f"-Wl,-rpath,{lib}"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cxx api ok" in r.stdout
