"""CLI relink (reference tools/volsr_main.cpp): the
reference's own command-line tool compiled UNCHANGED against the B200 library
(tools/cli/build_cli.py: "volsr/*.hpp" -> the C++ mirror, CLI11 -> the API
subset in tools/cli/CLI11.hpp).

GPU: the reference's CLI test suite (proj/tests/test_cli.cpp, compiled
unchanged) run against the relinked binary, and the relinked binary against
the same CLI built on the reference library (oracle/_ref/volsr_ref) on one
pipeline: phantom -> degrade -> tikhonov / tv -> psnr.
CPU: the binaries exist and parse (usage errors exit 2, --help exits 0)."""
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "tools" / "cli" / "_build" / "volsr"
REF_CLI = ROOT / "oracle" / "_ref" / "volsr_ref"
SUITE = ROOT / "tests" / "cpp" / "_build" / "ref_test_cli"
# reference test cases that fail on the reference's own build too (oracle/_ref/volsr_ref), with the reason
EXCLUDED = {
    "degrade with trivial operators reproduces the input":
        "asserts a bit-exact FFT round trip (FFTW codelets); neither the FFTW-API shim nor the B200 engine "
        "reproduces FFTW's rounding",
    "selftest passes clean and fails under fault injection":
        "the reference selftest itself throws (src/selftest.cpp:161-166 builds a 3^3 PSF on a 6x4x2 grid: "
        "'make_gaussian_psf: kernel size 3 exceeds volume axis 3 of length 2')",
}


def _need(p):
    if not p.exists():
        pytest.skip(f"{p.name} not built (tools/cli/build_cli.py needs /root/reference)")


def _run(exe, args, cwd, env=None):
    r = subprocess.run([str(exe), *args], cwd=cwd, capture_output=True, text=True, timeout=900,
                       env={**os.environ, **(env or {})})
    return r.returncode, r.stdout + r.stderr


def _manifest(text):
    return dict(ln.split("=", 1) for ln in text.splitlines() if "=" in ln and not ln.startswith("error"))


def test_cli_parses(tmp_path):
    _need(CLI)
    code, out = _run(CLI, [], tmp_path)
    assert code == 2 and "subcommand" in out
    code, out = _run(CLI, ["--help"], tmp_path)
    assert code == 0 and "tikhonov" in out
    code, out = _run(CLI, ["tikhonov", "--in", "a"], tmp_path)  # --out is required
    assert code == 2 and "--out" in out
    code, out = _run(CLI, ["tv", "--in", "a", "--out", "b", "--lambda", "abc"], tmp_path)
    assert code == 2


@pytest.mark.gpu
def test_reference_cli_suite_on_b200(tmp_path):
    _need(CLI)
    _need(SUITE)
    r = subprocess.run([str(SUITE)], cwd=tmp_path, capture_output=True, text=True, timeout=1800,
                       env={**os.environ, "VOLSR_CLI": str(CLI)})
    failed = {ln[len("[FAIL] "):].strip() for ln in (r.stdout + r.stderr).splitlines() if ln.startswith("[FAIL] ")}
    assert "test cases:" in r.stdout, r.stdout + r.stderr
    assert failed <= set(EXCLUDED), r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.gpu
def test_cli_b200_matches_reference_cli(tmp_path):
    """The same command lines through both builds: outputs within the parity bar."""
    _need(CLI)
    _need(REF_CLI)
    import ref_binding as R
    assert R.available()
    for exe, tag in ((CLI, "b"), (REF_CLI, "r")):
        for args in (["phantom", "--out", f"x_{tag}", "--dims", "64,64,32"],
                     ["degrade", "--in", f"x_{tag}", "--out", f"y_{tag}", "--decim", "2", "--psf-size", "9",
                      "--psf-sigma", "1.5", "--bsnr", "30", "--seed", "4"],
                     ["tikhonov", "--in", f"y_{tag}", "--out", f"t_{tag}", "--decim", "2", "--psf-size", "9",
                      "--psf-sigma", "1.5", "--lambda", "1e-3", "--ref", f"x_{tag}"],
                     ["tv", "--in", f"y_{tag}", "--out", f"v_{tag}", "--decim", "2", "--psf-size", "9",
                      "--psf-sigma", "1.5", "--iters", "5", "--tol", "0", "--tau", "5e-5", "--ref", f"x_{tag}",
                      "--manifest", f"m_{tag}.txt"]):
            code, out = _run(exe, args, tmp_path)
            assert code == 0, (tag, args, out)
    # the phantom (input synthesis, restated host code) is bit-identical; degrade
    # (blur by FFT on the GPU vs the FFTW-API shim) agrees to rounding
    assert (tmp_path / "x_b.vol").read_bytes() == (tmp_path / "x_r.vol").read_bytes()
    for name in ("y", "t", "v"):
        got, want = R.load_volume(str(tmp_path / f"{name}_b")), R.load_volume(str(tmp_path / f"{name}_r"))
        assert rel_err(got, want) < 1e-10, name
    mb = _manifest((tmp_path / "m_b.txt").read_text())
    mr = _manifest((tmp_path / "m_r.txt").read_text())
    for k in ("iterations_run", "lambda", "mu", "tau", "hr_dims", "lr_dims"):
        assert mb[k] == mr[k], k
    for k in ("initial_objective", "final_objective", "psnr"):
        assert abs(float(mb[k]) - float(mr[k])) <= 1e-9 * abs(float(mr[k])), k


ACCEPTANCE = ROOT / "tests" / "cpp" / "_build" / "ref_acceptance"


@pytest.mark.gpu
def test_reference_acceptance_suite_on_b200(tmp_path):
    """proj/tests/acceptance_main.cpp compiled unchanged against the mirror.
    The reference's own build of it stops after criterion 1: criterion 2 draws
    a 3^3 random PSF on a grid with an axis of length 2 and the uncaught
    'make_gaussian_psf: kernel size 3 exceeds volume axis 3 of length 2'
    aborts the suite (reproduced on oracle/_ref).  The B200 build must behave
    the same: criterion 1 passes, then the same abort.  Criterion 3 is run on
    its own in tests/test_acceptance.py."""
    _need(ACCEPTANCE)
    _need(CLI)
    r = subprocess.run([str(ACCEPTANCE)], cwd=tmp_path, capture_output=True, text=True, timeout=2400,
                       env={**os.environ, "VOLSR_CLI": str(CLI)})
    out = r.stdout + r.stderr
    print(out[-2000:])
    assert "[PASS] criterion 1:" in r.stdout
    assert "[FAIL]" not in r.stdout
    assert "kernel size 3 exceeds volume axis 3 of length 2" in out
