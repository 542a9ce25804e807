"""Matrix Market exchange (proj/include/semikern/matio.hpp, proj/src/matio.cpp):
the device-built reader and the writer against the reference library on the
same texts -- results bitwise, error messages (with line numbers) identical."""
import io
import os

import numpy as np
import pytest

from oracle.oracle import Csr

pytestmark = pytest.mark.gpu

H = "%%MatrixMarket matrix coordinate real general\n"
A = "%%MatrixMarket matrix array real general\n"

VALID = {
    "simple": H + "3 4 3\n1 1 1.5\n2 4 -2\n3 2 0.25\n",
    "unsorted_comments_blank_crlf": ("%%MatrixMarket Matrix Coordinate REAL General\r\n% c\r\n"
                                     "\r\n  3   3  4 \r\n3 3 1e-3\r\n\r\n1 2 +7\r\n2\t1\t-0\r\n"
                                     "1 1 3.5e+2\r\n"),
    "zero_values_elided": H + "2 2 2\n1 1 0\n2 2 0.0\n",
    "empty": H + "5 6 0\n",
    "no_final_newline": H + "2 2 1\n2 2 9",
    "subnormal_and_big": H + "1 3 3\n1 1 1e-40\n1 2 3.4028234e38\n1 3 -1.17549435e-38\n",
    "array": A + "2 3\n1\n2\n3\n4\n5\n6\n",
    "array_comments": A + "% x\n\n2 2\n1.5\n\n-2\n0\n+8\n",
    "array_empty": A + "0 3\n",
}

BAD = {
    "empty_file": "",
    "no_banner": "%%Matrix matrix coordinate real general\n",
    "short_header": "%%MatrixMarket matrix coordinate real\n",
    "not_matrix": "%%MatrixMarket vector coordinate real general\n",
    "format": "%%MatrixMarket matrix sparse real general\n1 1 0\n",
    "type": "%%MatrixMarket matrix coordinate integer general\n1 1 0\n",
    "symmetry": "%%MatrixMarket matrix coordinate real symmetric\n1 1 0\n",
    "eof_before_size": H + "% only comments\n\n",
    "size_fields": H + "2 2\n",
    "size_token": H + "2 x 1\n",
    "negative_count": H + "-2 2 1\n",
    "entry_fields": H + "2 2 1\n1 1\n",
    "row_token": H + "2 2 1\n1.0 1 1\n",
    "value_token": H + "2 2 1\n1 1 abc\n",
    "value_overflow": H + "2 2 1\n1 1 1e50\n",
    "row_range": H + "2 2 1\n3 1 1\n",
    "col_zero": H + "2 2 1\n1 0 1\n",
    "truncated": H + "2 2 3\n1 1 1\n\n2 2 2\n",
    "extra_content": H + "2 2 1\n1 1 1\n\n1 2 1\n",
    "duplicate": H + "3 3 4\n1 1 1\n2 2 2\n1 1 3\n1 1 4\n",
    "duplicate_order": H + "3 3 4\n3 3 1\n2 2 2\n3 3 5\n2 2 3\n",
    "array_size": A + "2 2 4\n",
    "array_two_values": A + "2 1\n1 2\n",
    "array_truncated": A + "2 2\n1\n2\n",
    "array_extra": A + "1 1\n1\n2\n",
    "array_value": A + "1 1\nx\n",
}


def refmsg(e):
    return str(e).split(": ", 1)[1]


def check_same(got, want):
    kind, w = want
    if kind == "csr":
        assert got.is_sparse()
        rp, ci, v = got.csr().extract()
        assert got.rows() == w.rows and got.cols() == w.cols
        assert np.array_equal(rp, w.row_ptr) and np.array_equal(ci, w.col_idx)
        assert np.array_equal(np.asarray(v, np.float32).view(np.uint32),
                              w.values.view(np.uint32))
    else:
        assert not got.is_sparse()
        d = got.dense().numpy()
        assert d.shape == w.shape
        assert np.array_equal(d.view(np.uint32), w.view(np.uint32))


@pytest.mark.parametrize("name", sorted(VALID))
def test_read_valid_matches_reference(sk, ref, name):
    text = VALID[name]
    check_same(sk.read_matrix(io.StringIO(text)), ref.read_matrix_text(text))


@pytest.mark.parametrize("name", sorted(BAD))
def test_read_errors_match_reference(sk, ref, name):
    text = BAD[name]
    with pytest.raises(Exception) as want:
        ref.read_matrix_text(text)
    with pytest.raises(sk.Error) as got:
        sk.read_matrix(io.StringIO(text))
    assert str(got.value) == refmsg(want.value)
    assert type(got.value).__name__ == want.value.kind


def test_write_matches_reference_and_round_trips(sk, ref, tmp_path):
    rng = np.random.default_rng(4)
    flat = rng.choice(300 * 200, size=2000, replace=False)
    r, c = (flat // 200).astype(np.uint32), (flat % 200).astype(np.uint32)
    v = (rng.standard_normal(2000) * 10.0 ** rng.integers(-30, 30, 2000)).astype(np.float32)
    a = sk.csr_from_triples(300, 200, (r, c, v))
    rp, ci, vals = a.extract()
    host = Csr(300, 200, np.asarray(rp, np.uint32), np.asarray(ci, np.uint32),
               np.asarray(vals, np.float32))
    buf = io.StringIO()
    info = sk.write_matrix(a, buf)
    assert buf.getvalue() == ref.format_matrix(host)
    assert (info.kind, info.rows, info.cols, info.entries) == (sk.MatrixFileKind.coordinate,
                                                               300, 200, a.nnz())
    check_same(sk.read_matrix(io.StringIO(buf.getvalue())), ("csr", host))  # %.9g round trips
    d = (rng.standard_normal((7, 5)) * 1e3).astype(np.float32)
    buf = io.StringIO()
    sk.write_matrix(sk.DenseMatrix.from_numpy(d), buf)
    assert buf.getvalue() == ref.format_matrix(d)
    # the path overloads
    p = os.path.join(str(tmp_path), "w.mtx")
    info = sk.write_matrix(a, p)
    assert info.path == p and open(p).read() == ref.format_matrix(host)
    check_same(sk.read_matrix(p), ("csr", host))
    with pytest.raises(sk.Error, match="cannot open"):
        sk.read_matrix(os.path.join(str(tmp_path), "missing.mtx"))
