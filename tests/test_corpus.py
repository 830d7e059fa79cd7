"""Sparse corpus text format (dataset.cpp:80-198): the host reader/writer against
the unmodified reference's reader (CPU); the device path over a parsed corpus is
in test_gpu_sparse.py."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1602_02350_b200 import skridge as sk

CORPUS = """# a comment line
1.5 1:0.5 3:-2 7:1e-3   # trailing comment
-2 2:4

0 1:0 4:2.5
3.25e0 5:1 6:-0.75 9:0.125
"""


@pytest.fixture()
def corpus_path(tmp_path):
    p = tmp_path / "c.txt"
    p.write_text(CORPUS)
    return str(p)


def _parse_host(path):
    """The reader's arrays without touching a device (the DataMatrix needs one)."""
    import paper_1602_02350_b200.skridge as m
    captured = {}
    real = m.DataMatrix.from_csr

    def fake(rp, ci, va, d, ctx=None):
        captured.update(rp=rp, ci=ci, va=va, d=d)
        return None

    m.DataMatrix.from_csr = staticmethod(fake)
    try:
        ds = m.read_sparse_corpus(path)
    finally:
        m.DataMatrix.from_csr = real
    return captured, ds.labels


def test_reader_matches_reference(corpus_path):
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    got, y = _parse_host(corpus_path)
    (rp, ci, va, d), yr = oracle.ref().read_sparse_corpus(corpus_path)
    assert got["d"] == d == 9
    assert np.array_equal(got["rp"], rp) and np.array_equal(got["ci"], ci) and np.array_equal(got["va"], va)
    assert np.array_equal(y, yr)


@pytest.mark.parametrize("bad,line", [("1 2:1 2:3\n", 1), ("x 1:1\n", 1), ("1 0:1\n", 1), ("1 1:nan\n", 1),
                                      ("1 1:\n", 1), ("\n1 1:1\n2 a:1\n", 3), ("1 3:1 2:1\n", 1)])
def test_reader_errors_carry_line_numbers(tmp_path, bad, line):
    p = tmp_path / "bad.txt"
    p.write_text(bad)
    with pytest.raises(sk.ParseError) as e:
        _parse_host(str(p))
    assert e.value.line == line
    if oracle.ref_available():
        with pytest.raises(oracle.OracleError):
            oracle.ref().read_sparse_corpus(str(p))


def test_reader_empty_and_featureless(tmp_path):
    p = tmp_path / "e.txt"
    p.write_text("# nothing\n\n")
    with pytest.raises(sk.InputError):
        _parse_host(str(p))
    p.write_text("1\n2\n")
    with pytest.raises(sk.DegenerateDataError):
        _parse_host(str(p))
    with pytest.raises(sk.InputError):
        _parse_host(str(tmp_path / "missing.txt"))


def test_writer_round_trip(corpus_path, tmp_path):
    got, y = _parse_host(corpus_path)
    out = str(tmp_path / "w.txt")
    sk.write_sparse_corpus(got["rp"], got["ci"], got["va"], y, out)
    again, y2 = _parse_host(out)
    assert np.array_equal(again["rp"], got["rp"]) and np.array_equal(again["va"], got["va"])
    assert np.array_equal(y2, y)


def test_cpp_parser_matches_reference_reader(tmp_path):
    """include/skridge_b200.hpp parse_sparse_corpus against the unmodified reference
    reader (dataset.cpp:87-162) on valid corpora and every malformed-line class
    (tests/cpp/corpus_parse.cpp, built by __graft_entry__.build())."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cpp", "corpus_parse")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/corpus_parse not built (needs /root/reference at build time)")
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 of 19 cases differ" in r.stdout
