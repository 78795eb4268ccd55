"""CPU: the host I/O of the engine library (no GPU): the native TSV writer is
byte-identical to io::tsv_string's "%u\\t%u\\t%.17g" (proj/src/io.cpp:141-154), and
binary-f64 ingest behaves like ingest_binary (proj/src/io.cpp:69-91)."""
import os

import numpy as np
import pytest

from paper_1810_04758_b200 import KnnjError
from paper_1810_04758_b200.engine import (KnnRunResult, read_binary_f64, tsv_bytes, tsv_string,
                                          write_tsv)


def _result(nq, k, seed):
    rng = np.random.default_rng(seed)
    d = np.sort(rng.exponential(1.0, (nq, k)) * 10.0 ** rng.integers(-8, 6, (nq, 1)), axis=1)
    d[0, :min(k, 6)] = [0.0, 5e-324, 1e-300, 0.1, 1.0 / 3, 2.0 ** 52 + 0.5][:min(k, 6)]
    ids = rng.integers(0, 2 ** 32 - 1, (nq, k), dtype=np.uint64).astype(np.uint32)
    q = np.sort(rng.choice(10 ** 6, nq, replace=False)).astype(np.uint32)
    return KnnRunResult(queries=q, ids=ids, dist=d, provenance=np.zeros(nq, np.uint8),
                        k_effective=k, info={})


@pytest.mark.parametrize("nq,k,threads", [(1, 1, 1), (37, 5, 0), (3000, 32, 3), (200001, 2, 0)])
def test_tsv_matches_printf(nq, k, threads):
    r = _result(nq, k, nq + k)
    want = tsv_string(r).encode()
    assert tsv_bytes(r, threads) == want


def test_tsv_file(tmp_path):
    r = _result(5000, 7, 3)
    p = str(tmp_path / "out.tsv")
    n = write_tsv(p, r, threads=4)
    data = open(p, "rb").read()
    assert n == len(data) and data == tsv_string(r).encode()


def test_tsv_reference_bytes():
    """known lines from the reference's %.17g formatting (printf semantics)"""
    r = KnnRunResult(queries=np.array([3], np.uint32), ids=np.array([[7, 9, 11]], np.uint32),
                     dist=np.array([[5.0, 3.7416573867739413, 0.1]]), provenance=np.zeros(1, np.uint8),
                     k_effective=3, info={})
    assert tsv_bytes(r) == b"3\t7\t5\n3\t9\t3.7416573867739413\n3\t11\t0.10000000000000001\n"


def test_binary_roundtrip_and_errors(tmp_path):
    X = np.random.default_rng(1).standard_normal((123, 5))
    p = tmp_path / "d.bin"
    with open(p, "wb") as f:
        f.write(np.array([123, 5], "<u8").tobytes())
        f.write(X.astype("<f8").tobytes())
    assert np.array_equal(read_binary_f64(str(p)), X)
    bad = X.copy()
    bad[4, 2] = np.nan
    with open(p, "wb") as f:
        f.write(np.array([123, 5], "<u8").tobytes())
        f.write(bad.astype("<f8").tobytes())
    with pytest.raises(KnnjError) as e:
        read_binary_f64(str(p))
    assert e.value.kind == "IngestError" and "row 5, column 3: non-finite value" in str(e.value)
    with open(p, "wb") as f:
        f.write(np.array([123, 5], "<u8").tobytes())
        f.write(X.astype("<f8").tobytes()[:800])
    with pytest.raises(KnnjError) as e:
        read_binary_f64(str(p))
    assert "body shorter than header promises (123 x 5)" in str(e.value)
    with open(p, "wb") as f:
        f.write(bytes(7))
    with pytest.raises(KnnjError) as e:
        read_binary_f64(str(p))
    assert "truncated header" in str(e.value)
    with pytest.raises(KnnjError):
        read_binary_f64(str(tmp_path / "missing.bin"))


# ---- dataset ingest (csv / tsv / binary-f64) against the reference's own outcomes
import hashlib  # noqa: E402
import json  # noqa: E402
import sys  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
from make_ingest_golden import cases as _ingest_cases  # noqa: E402

from paper_1810_04758_b200 import ingest_dataset  # noqa: E402

_GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                    "ingest_cases.json")))
_CASES = _ingest_cases()


@pytest.mark.parametrize("threads", [1, 8])
@pytest.mark.parametrize("name,fmt,data", _CASES, ids=[c[0] for c in _CASES])
def test_ingest_matches_reference(tmp_path, name, fmt, data, threads):
    """ingest_dataset (proj/src/io.cpp:15-106): sizes and coordinates, or the error kind
    and message, equal the unmodified reference's (tests/golden/make_ingest_golden.py);
    multi-threaded parsing reports the first error in file order."""
    want = _GOLD[name]
    p = str(tmp_path / f"{name}.{fmt}")
    with open(p, "wb") as f:
        f.write(data)
    if "error" in want:
        with pytest.raises(KnnjError) as e:
            ingest_dataset(p, fmt, threads=threads)
        assert e.value.kind == want["error"]
        assert str(e.value) == f"{want['error']}: " + want["message"].replace("{path}", p)
        return
    X = ingest_dataset(p, fmt, threads=threads)
    assert X.shape == (want["points"], want["dims"])
    assert hashlib.sha256(np.ascontiguousarray(X, "<f8").tobytes()).hexdigest() == want["sha256"]


def test_ingest_missing_and_unknown_format(tmp_path):
    p = str(tmp_path / "missing.csv")
    with pytest.raises(KnnjError) as e:
        ingest_dataset(p, "csv")
    assert str(e.value) == "IngestError: " + _GOLD["missing_file"]["message"].replace("{path}", p)
    with pytest.raises(KnnjError) as e:
        ingest_dataset("x", "xml")
    assert e.value.kind == "UsageError" and _GOLD["unknown_format"]["message"] in str(e.value)
