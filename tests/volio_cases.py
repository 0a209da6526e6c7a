"""Malformed / edge-case volume files for the .volhdr/.vol parity tests
(reference src/volume_io.cpp:17-131).  Each case writes files under `d` and
returns the base path; tools/make_golden.py records the REFERENCE's error
text for every case (tests/golden/volio.npz) and tests/test_volio.py checks
the library's text against it.  Paths in messages are normalised to <dir>."""
import numpy as np

GOOD = "dims=5,4,3\ndtype=f64\norder=lex\n"
VALS = np.arange(60, dtype=np.float64).reshape(3, 4, 5) * 0.25 - 3.0


def _write(d, name, hdr, payload=None):
    base = d / name
    if hdr is not None:
        (d / f"{name}.volhdr").write_bytes(hdr.encode())
    if payload is not None:
        (d / f"{name}.vol").write_bytes(payload)
    return base


def cases(d):
    raw = VALS.tobytes()
    bad = VALS.copy()
    bad[1, 2, 3] = np.nan
    return {
        "missing_header": _write(d, "missing_header", None, raw),
        "malformed_line": _write(d, "malformed_line", "dims=5,4,3\nxyz\n", raw),
        "duplicate_dims": _write(d, "duplicate_dims", "dims=5,4,3\ndims=5,4,3\ndtype=f64\norder=lex\n", raw),
        "malformed_dims": _write(d, "malformed_dims", "dims=5,4\ndtype=f64\norder=lex\n", raw),
        "zero_dims": _write(d, "zero_dims", "dims=0,4,3\ndtype=f64\norder=lex\n", raw),
        "bad_dtype": _write(d, "bad_dtype", "dims=5,4,3\ndtype=f16\norder=lex\n", raw),
        "duplicate_dtype": _write(d, "duplicate_dtype", "dims=5,4,3\ndtype=f64\ndtype=f64\norder=lex\n", raw),
        "bad_order": _write(d, "bad_order", "dims=5,4,3\ndtype=f64\norder=col\n", raw),
        "unknown_key": _write(d, "unknown_key", GOOD + "foo=1\n", raw),
        "incomplete": _write(d, "incomplete", "dims=5,4,3\ndtype=f64\n", raw),
        "missing_payload": _write(d, "missing_payload", GOOD, None),
        "short_payload": _write(d, "short_payload", GOOD, raw[:-8]),
        "non_finite": _write(d, "non_finite", GOOD, bad.tobytes()),
        "crlf_ok": _write(d, "crlf_ok", GOOD.replace("\n", "\r\n"), raw),
        "f32_ok": _write(d, "f32_ok", "dims=5,4,3\ndtype=f32\norder=lex\n", VALS.astype(np.float32).tobytes()),
    }


def norm(msg, d):
    return msg.replace(str(d), "<dir>")
