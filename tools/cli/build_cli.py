"""CLI relink: the reference's own command-line tool (proj/tools/volsr_main.cpp,
with its selftest src/selftest.cpp) compiled UNCHANGED against the B200
library, so `volsr tikhonov|tv|bench|...` runs the hot path on the GPU.

  tools/cli/_build/volsr    the reference CLI on libvsr_b200.so: "volsr/*.hpp"
                            resolves to tests/cpp/refshim (forwarding to the C++
                            mirror include/volsr_b200/volsr.hpp), CLI11 to the
                            API subset in tools/cli/CLI11.hpp
  oracle/_ref/volsr_ref     the same sources on the reference library itself
                            (oracle/_ref objects), for side-by-side tests
  tests/cpp/_build/ref_test_cli
                            the reference's CLI test suite (proj/tests/test_cli.cpp)
                            compiled unchanged; it runs the binary named by $VOLSR_CLI
  tests/cpp/_build/ref_acceptance
                            the reference's acceptance suite (proj/tests/acceptance_main.cpp)
                            compiled unchanged against the mirror

Needs /root/reference (this container, __graft_entry__.build()); the
binaries travel to the GPU box with the repo.
"""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/proj")
OUT = ROOT / "tools" / "cli" / "_build"
LIB = ROOT / "paper_2010_15491_b200" / "_lib"
CPP_BUILD = ROOT / "tests" / "cpp" / "_build"
REF_OBJ = ROOT / "oracle" / "_ref"
VERSION = '-DVOLSR_VERSION="0.1.0"'  # CMakeLists.txt:2,35 (project version)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(map(str, cmd)) + "\n" + r.stdout + r.stderr)


def build() -> bool:
    if not (REF / "tools" / "volsr_main.cpp").exists():
        return False
    OUT.mkdir(parents=True, exist_ok=True)
    CPP_BUILD.mkdir(parents=True, exist_ok=True)
    shim = [f"-I{ROOT / 'tests' / 'cpp' / 'refshim'}", f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'shim'}",
            f"-I{ROOT / 'tools' / 'cli'}"]
    flags = ["-std=c++20", "-O2", "-w", "-include", "algorithm", "-include", "cstring", VERSION]
    # objects shared with the reference suites (tests/test_cpp_mirror.py)
    objs = []
    for src, name in ((REF / "src" / "dense.cpp", "ref_dense.o"),
                      (ROOT / "tests" / "cpp" / "refshim" / "refshim_extras.cpp", "refshim_extras.o"),
                      (REF / "src" / "selftest.cpp", "ref_selftest.o")):
        o = CPP_BUILD / name
        _run(["g++", *flags, *shim, "-c", str(src), "-o", str(o)])
        objs.append(str(o))
    rpath = "-Wl,-rpath," + "$ORIGIN/../../../paper_2010_15491_b200/_lib"
    _run(["g++", *flags, *shim, str(REF / "tools" / "volsr_main.cpp"), *objs, f"-L{LIB}", "-lvsr_b200", rpath,
          "-o", str(OUT / "volsr")])
    # the reference's CLI tests, unchanged (doctest from oracle/shim)
    _run(["g++", *flags, *shim, f"-I{REF / 'tests'}", str(REF / "tests" / "test_cli.cpp"), objs[1], objs[0],
          f"-L{LIB}", "-lvsr_b200", "-Wl,-rpath,$ORIGIN/../../../paper_2010_15491_b200/_lib",
          "-o", str(CPP_BUILD / "ref_test_cli")])
    # the reference's acceptance suite (proj/tests/acceptance_main.cpp), unchanged
    _run(["g++", *flags, *shim, f"-I{REF / 'tests'}", str(REF / "tests" / "acceptance_main.cpp"), *objs,
          f"-L{LIB}", "-lvsr_b200", "-Wl,-rpath,$ORIGIN/../../../paper_2010_15491_b200/_lib",
          "-o", str(CPP_BUILD / "ref_acceptance")])
    # the same CLI on the reference library (oracle/_ref, built by oracle/Makefile)
    ref_objs = [REF_OBJ / f"{n}.o" for n in ("volume", "fft", "operators", "spectral", "solvers", "dense", "sim",
                                             "metrics", "volume_io", "fftw_shim")]
    if all(o.exists() for o in ref_objs):
        _run(["g++", *flags, f"-I{REF / 'include'}", f"-I{ROOT / 'oracle' / 'shim'}", f"-I{ROOT / 'tools' / 'cli'}",
              str(REF / "tools" / "volsr_main.cpp"), str(REF / "src" / "selftest.cpp"), *map(str, ref_objs),
              "-lpthread", "-o", str(REF_OBJ / "volsr_ref")])
    return True


if __name__ == "__main__":
    ok = build()
    print("built" if ok else "skipped (no /root/reference)")
    sys.exit(0)
