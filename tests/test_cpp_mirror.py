"""The C++ mirror of the reference API (include/volsr_b200/volsr.hpp): it
compiles against the reference-style test code here, and on a GPU the
restated reference tests pass through it."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "tests" / "cpp" / "_build" / "test_volsr_b200"


def build():
    EXE.parent.mkdir(parents=True, exist_ok=True)
    lib = ROOT / "paper_2010_15491_b200" / "_lib"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "test_volsr_b200.cpp"),
           f"-L{lib}", "-lvsr_b200", f"-Wl,-rpath,{lib}", "-o", str(EXE)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_mirror_compiles():
    build()
    assert EXE.exists()


@pytest.mark.gpu
def test_cpp_mirror_reference_tests_on_gpu():
    build()
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
