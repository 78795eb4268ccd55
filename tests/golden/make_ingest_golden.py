"""Golden expectations for dataset ingest (csv / tsv / binary-f64), produced by the
UNMODIFIED reference's ingest_dataset (proj/src/io.cpp:15-106) through
oracle/_ref/libknnjoin_ref.so (ref_ingest in oracle/ref_capi.cpp).

    python tests/golden/make_ingest_golden.py      # writes tests/golden/ingest_cases.json

`cases()` builds every input deterministically, so tests/test_io.py regenerates the
same files and compares the engine's ingest with the stored outcome: the sizes and a
SHA-256 of the parsed coordinates, or the error kind and message (the file path is
stored as "{path}").
"""
import ctypes as C
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "ingest_cases.json")


def _big(rows, cols, seed, sep, bad=None):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((rows, cols)) * 10.0 ** rng.integers(-5, 6, (rows, 1))
    lines = [sep.join("%.17g" % v for v in r) for r in X]
    for row, text in (bad or {}).items():
        lines[row - 1] = text
    return ("\n".join(lines) + "\n").encode()


def cases():
    """(name, format, file bytes) of every ingest case."""
    c = [
        ("csv_simple", "csv", b"1,2\n3,4\n5,6\n"),
        ("csv_no_final_newline", "csv", b"1,2\n3,4"),
        ("csv_spaces_tabs", "csv", b" 1.5 ,\t2\n  -3e2,4.25  \n"),
        ("csv_crlf", "csv", b"1,2\r\n3,4\r\n"),
        ("csv_empty_lines", "csv", b"\n1,2\n\n\n3,4\n\n"),
        ("csv_cr_only_line", "csv", b"1,2\n\r\n3,4\n"),
        ("csv_trailing_sep", "csv", b"1,2,\n3,4,\n"),
        ("csv_nan", "csv", b"1,2\n3,nan\n"),
        ("csv_inf", "csv", b"1,2\n-inf,4\n"),
        ("csv_overflow", "csv", b"1,2\n1e400,4\n"),
        ("csv_subnormal", "csv", b"1e-320,-0\n.5,5.\n"),
        ("csv_plus_sign", "csv", b"1,2\n+1,2\n"),
        ("csv_hex", "csv", b"0x1p3,2\n"),
        ("csv_word", "csv", b"1,2\n3,abc\n"),
        ("csv_fewer_cols", "csv", b"1,2,3\n4,5\n"),
        ("csv_more_cols", "csv", b"1,2\n3,4,5\n"),
        ("csv_more_cols_bad", "csv", b"1,2\n3,4,x\n"),
        ("csv_empty_file", "csv", b""),
        ("csv_only_newlines", "csv", b"\n\n\n"),
        ("csv_single", "csv", b"42\n"),
        ("tsv_simple", "tsv", b"1\t2\t3\n4\t5\t6\n"),
        ("tsv_spaces", "tsv", b" 1 \t 2\n3\t4 \n"),
        ("tsv_comma_inside", "tsv", b"1,5\t2\n"),
        ("tsv_empty_field", "tsv", b"1\t\t2\n"),
        ("csv_big", "csv", _big(60000, 7, 1, ",")),
        ("tsv_big", "tsv", _big(50000, 9, 2, "\t")),
        ("csv_big_error_deep", "csv", _big(60000, 7, 3, ",", {45001: "1,2,3,4,5,6,oops"})),
        ("csv_big_two_errors", "csv", _big(60000, 7, 4, ",", {20000: "1,2,3,4,5,6", 50000: "x"})),
        ("csv_big_nan_deep", "csv", _big(60000, 7, 5, ",", {59999: "1,2,3,4,5,6,nan"})),
        ("csv_big_cols_late", "csv", _big(60000, 7, 6, ",", {30001: "1,2,3,4,5,6,7,8"})),
        ("csv_big_first_line_short", "csv", _big(60000, 7, 7, ",", {1: "1,2,3"})),
    ]
    X = np.random.default_rng(9).standard_normal((123, 5))
    hdr = np.array([123, 5], "<u8").tobytes()
    c += [
        ("bin_ok", "bin", hdr + X.astype("<f8").tobytes()),
        ("bin_short", "bin", hdr + X.astype("<f8").tobytes()[:800]),
        ("bin_truncated_header", "bin", bytes(7)),
        ("bin_empty_header", "bin", np.array([0, 5], "<u8").tobytes()),
    ]
    bad = X.copy()
    bad[77, 3] = np.inf
    bad[100, 1] = np.nan
    c.append(("bin_nonfinite", "bin", hdr + bad.astype("<f8").tobytes()))
    return c


def sha(X):
    return hashlib.sha256(np.ascontiguousarray(X, "<f8").tobytes()).hexdigest()


def main():
    lib = C.CDLL(os.path.join(HERE, "..", "..", "oracle", "_ref", "libknnjoin_ref.so"))
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_ingest.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_uint64,
                               C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    kinds = {1: "UsageError", 2: "IngestError"}
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, fmt, data in cases():
            path = os.path.join(d, name + "." + fmt)
            with open(path, "wb") as f:
                f.write(data)
            N, n = C.c_uint64(), C.c_uint64()
            rc = lib.ref_ingest(path.encode(), fmt.encode(), None, 0, C.byref(N), C.byref(n))
            if rc:
                out[name] = {"format": fmt, "error": kinds.get(rc, str(rc)),
                             "message": lib.ref_last_error().decode().replace(path, "{path}")}
                continue
            X = np.zeros((N.value, n.value))
            rc = lib.ref_ingest(path.encode(), fmt.encode(), X.ctypes.data, X.size, C.byref(N),
                                C.byref(n))
            assert rc == 0
            out[name] = {"format": fmt, "points": N.value, "dims": n.value, "sha256": sha(X)}
        N, n = C.c_uint64(), C.c_uint64()
        rc = lib.ref_ingest(os.path.join(d, "missing.csv").encode(), b"csv", None, 0, C.byref(N),
                            C.byref(n))
        out["missing_file"] = {"format": "csv", "error": kinds.get(rc, str(rc)),
                               "message": lib.ref_last_error().decode().replace(
                                   os.path.join(d, "missing.csv"), "{path}")}
        rc = lib.ref_ingest(b"x", b"xml", None, 0, C.byref(N), C.byref(n))
        out["unknown_format"] = {"format": "xml", "error": kinds.get(rc, str(rc)),
                                 "message": lib.ref_last_error().decode()}
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(f"wrote {len(out)} cases to {OUT}")


if __name__ == "__main__":
    sys.exit(main())
