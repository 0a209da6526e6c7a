"""Volume files (.volhdr/.vol), reference src/volume_io.cpp:17-131.

The golden (tests/golden/volio.npz, tools/make_golden.py volio) holds the
REFERENCE's own bytes for a saved f64 and f32 volume and its error text for
every malformed case of volio_cases.py.  CPU tests exercise the library's
host entry points (vsr_load_volume / vsr_save_volume: no device needed);
GPU tests the streamed device variants (vsr_load_volume_d / _save_volume_d),
including a multi-chunk volume."""
from pathlib import Path

import numpy as np
import pytest

import volio_cases as VC

G = Path(__file__).resolve().parent / "golden" / "volio.npz"


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(G))


def test_golden_values_match_cases(gold):
    assert np.array_equal(gold["vals"], VC.VALS)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_save_is_byte_identical_to_reference(V, gold, tmp_path, dtype):
    V.save_volume(VC.VALS, str(tmp_path / "w"), dtype=dtype)
    assert (tmp_path / "w.volhdr").read_bytes() == bytes(gold[f"{dtype}_hdr"])
    assert (tmp_path / "w.vol").read_bytes() == bytes(gold[f"{dtype}_raw"])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_load_reference_files(V, gold, tmp_path, dtype):
    (tmp_path / "r.volhdr").write_bytes(bytes(gold[f"{dtype}_hdr"]))
    (tmp_path / "r.vol").write_bytes(bytes(gold[f"{dtype}_raw"]))
    for p in ("r", "r.vol", "r.volhdr"):  # strip_volume_extension (volume_io.cpp:27-31)
        v = V.load_volume(str(tmp_path / p))
        want = VC.VALS if dtype == "f64" else VC.VALS.astype(np.float32).astype(np.float64)
        assert v.shape == (3, 4, 5) and np.array_equal(v, want)
    assert V.volume_header(str(tmp_path / "r")) == ((5, 4, 3), dtype)


def test_malformed_cases_match_reference_text(V, gold, tmp_path):
    for name, base in VC.cases(tmp_path).items():
        want = str(gold[f"case_{name}"])
        if want == "OK":
            assert np.array_equal(V.load_volume(str(base)), gold[f"case_{name}_vals"]), name
            continue
        with pytest.raises(V.VolumeIOError) as ei:
            V.load_volume(str(base))
        assert VC.norm(str(ei.value), tmp_path) == want, name


def test_save_non_finite_matches_reference(V, gold, tmp_path):
    bad = VC.VALS.copy()
    bad[2, 0, 1] = np.inf
    with pytest.raises(V.NumericError) as ei:
        V.save_volume(bad, str(tmp_path / "b"))
    assert str(ei.value) == str(gold["save_non_finite"])
    assert not (tmp_path / "b.volhdr").exists()


def test_buffer_size_mismatch_is_shape_error(V, tmp_path):
    V.save_volume(VC.VALS, str(tmp_path / "w"))
    import ctypes as C
    out = np.empty(10)
    rc = V._lib.vsr_load_volume(str(tmp_path / "w").encode(), out.ctypes.data_as(C.c_void_p), out.size)
    assert rc == V.VSR_ERR_SHAPE


# ------------------------------------------------------------------ device streaming
class _Dev:
    def __init__(self, t):
        import ctypes as C
        self.t = t
        self.ptr = C.c_void_p(t.data_ptr())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("dims", [(5, 4, 3), (256, 256, 72)])  # the second spans several 32 MB chunks
def test_device_stream_round_trip(V, tmp_path, dtype, dims):
    import torch
    m, n, s = dims
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, (s, n, m))
    V.save_volume(v, str(tmp_path / "h"), dtype=dtype)           # host writer
    dev = torch.empty(s * n * m, dtype=torch.float64, device="cuda")
    assert V.load_volume_device(str(tmp_path / "h"), _Dev(dev)) == dims
    V.default_context().synchronize()
    want = v if dtype == "f64" else v.astype(np.float32).astype(np.float64)
    assert np.array_equal(dev.cpu().numpy().reshape(s, n, m), want)
    V.save_volume_device(_Dev(dev), dims, str(tmp_path / "d"), dtype=dtype)
    for ext in (".volhdr", ".vol"):
        assert (tmp_path / f"d{ext}").read_bytes() == (tmp_path / f"h{ext}").read_bytes()


@pytest.mark.gpu
def test_device_stream_errors_match_reference(V, gold, tmp_path):
    import torch
    dev = torch.empty(60, dtype=torch.float64, device="cuda")
    for name, base in VC.cases(tmp_path).items():
        want = str(gold[f"case_{name}"])
        if want == "OK":
            V.load_volume_device(str(base), _Dev(dev))
            V.default_context().synchronize()
            assert np.array_equal(dev.cpu().numpy().reshape(3, 4, 5), gold[f"case_{name}_vals"]), name
            continue
        with pytest.raises(V.VolumeIOError) as ei:
            V.load_volume_device(str(base), _Dev(dev))
        assert VC.norm(str(ei.value), tmp_path) == want, name
    bad = torch.from_numpy(VC.VALS.reshape(-1).copy()).cuda()
    bad[41] = float("inf")
    with pytest.raises(V.NumericError) as ei:
        V.save_volume_device(_Dev(bad), (5, 4, 3), str(tmp_path / "b"))
    assert str(ei.value) == str(gold["save_non_finite"])
