"""The drop-in boundary: libvsr_b200.so loads and exports every entry point
include/vsr.h declares; without a GPU the product path fails loudly (no CPU
fallback).  CPU only: no compute calls."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2010_15491_b200" / "_lib" / "libvsr_b200.so"


def declared():
    txt = (ROOT / "include" / "vsr.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vsr_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_boundary():
    names = declared()
    for must in ("vsr_tikhonov_create", "vsr_tikhonov_solve", "vsr_admm_tv", "vsr_tv_x_update",
                 "vsr_tv_shrink", "vsr_make_gamma", "vsr_objective_tv", "vsr_fft3", "vsr_ifft3_real",
                 "vsr_folded_apply", "vsr_alias_fold", "vsr_fft_counters"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert LIB.exists(), "build first: python -c 'import __graft_entry__ as g; g.build()'"
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    missing = [n for n in declared() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(LIB)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_loads_and_fails_loudly_without_gpu():
    import torch
    from paper_2010_15491_b200 import volsr as V
    assert V.launch_count() >= 0
    assert V.tikhonov_algorithmic_bytes((256, 256, 256), (2, 2, 2)) == (72 + 40 / 8) * 256 ** 3
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(V.DeviceError):
        V.Context(0)
