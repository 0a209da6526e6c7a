"""The C++ mirror of the reference API (include/volsr_b200/volsr.hpp).

1. tests/cpp/test_volsr_b200.cpp: restated reference tests through the mirror.
2. The reference's OWN doctest suites (proj/tests/test_volume.cpp,
   test_operators.cpp, test_spectral.cpp, test_solvers.cpp) compiled
   UNCHANGED against the mirror: the include path resolves "volsr/*.hpp" to
   tests/cpp/refshim/volsr/ (each forwards to the mirror), doctest and Eigen
   come from oracle/shim, the dense-matrix builders are the reference's own
   src/dense.cpp and the dense oracles / metrics / phantom generators are
   test-infrastructure restatements (tests/cpp/refshim/refshim_extras.cpp).
   Everything on the hot path runs through libvsr_b200.so on the GPU.

The suites are compiled where /root/reference exists (this container, and
__graft_entry__.build()); the binaries in tests/cpp/_build travel to the GPU
box, which has no /root/reference.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BUILD = ROOT / "tests" / "cpp" / "_build"
EXE = BUILD / "test_volsr_b200"
LIB = ROOT / "paper_2010_15491_b200" / "_lib"
REF = Path("/root/reference/proj")
SUITES = ["test_volume", "test_operators", "test_spectral", "test_solvers"]
# Reference test cases excluded on the B200 mirror, with the reason:
EXCLUDED = {}


def build():
    BUILD.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "test_volsr_b200.cpp"),
           f"-L{LIB}", "-lvsr_b200", "-Wl,-rpath,$ORIGIN/../../../paper_2010_15491_b200/_lib", "-o", str(EXE)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def build_reference_suites():
    """Compile the reference's suites against the mirror (needs /root/reference)."""
    if not (REF / "tests").exists():
        return False
    BUILD.mkdir(parents=True, exist_ok=True)
    flags = ["-std=c++20", "-O2", "-w", "-include", "algorithm", "-include", "cstring",
             f"-I{ROOT / 'tests' / 'cpp' / 'refshim'}", f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'shim'}",
             f"-I{REF / 'tests'}"]
    objs = []
    for src, name in ((REF / "src" / "dense.cpp", "ref_dense.o"),
                      (ROOT / "tests" / "cpp" / "refshim" / "refshim_extras.cpp", "refshim_extras.o")):
        o = BUILD / name
        subprocess.run(["g++", *flags, "-c", str(src), "-o", str(o)], check=True, capture_output=True, text=True)
        objs.append(str(o))
    for s in SUITES:
        subprocess.run(["g++", *flags, str(REF / "tests" / f"{s}.cpp"), *objs, f"-L{LIB}", "-lvsr_b200",
                        "-Wl,-rpath,$ORIGIN/../../../paper_2010_15491_b200/_lib", "-o", str(BUILD / f"ref_{s}")],
                       check=True, capture_output=True, text=True)
    return True


def test_cpp_mirror_compiles():
    build()
    assert EXE.exists()


def test_reference_suites_compile_unchanged_against_mirror():
    if not build_reference_suites():
        pytest.skip("/root/reference absent (prebuilt binaries are used on the GPU box)")
    for s in SUITES:
        assert (BUILD / f"ref_{s}").exists()


@pytest.mark.gpu
def test_cpp_mirror_reference_tests_on_gpu():
    build()
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_b200(suite):
    exe = BUILD / f"ref_{suite}"
    if not exe.exists():
        build_reference_suites()
    if not exe.exists():
        pytest.skip("reference suite binaries not built (no /root/reference and none shipped)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    failed = {ln[len("[FAIL] "):].strip() for ln in r.stderr.splitlines() if ln.startswith("[FAIL] ")}
    assert failed <= set(EXCLUDED.get(suite, {})), r.stdout[-2000:] + r.stderr[-4000:]
    assert "test cases:" in r.stdout, r.stdout + r.stderr
