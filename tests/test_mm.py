"""CPU: Matrix Market I/O -- libdpt_b200.so's
multithreaded reader/writer against the reference's own read_matrix_market /
write_matrix_market (proj/src/matrix_market.cpp, compiled in oracle/_ref).

Parity is bitwise: the same CSR (row offsets, column indices, every value's
bits), the same dense values, the same IoError messages, byte-identical
output files.  The reference's known-answer tests
(proj/tests/test_matrix_market.cpp) are restated first."""
import os

import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import ReferenceMatrixMarket, available
from paper_2002_12872_b200.dpt import CsrMatrix

pytestmark = pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def R():
    return ReferenceMatrixMarket()


def write(tmp_path, name, text, mode="w"):
    p = tmp_path / name
    with open(p, mode) as f:
        f.write(text)
    return str(p)


def bits(a):
    return np.ascontiguousarray(a).view(np.int64)


def assert_same(R, path, threads=0):
    rc, msg, ref = R.read(path)
    if rc != 0:
        with pytest.raises(P.IoError) as e:
            P.read_matrix_market(path, threads)
        assert str(e.value) == msg
        return None
    got = P.read_matrix_market(path, threads)
    if ref[0] == "dense":
        assert isinstance(got, np.ndarray) and got.shape == ref[1].shape
        g = got.astype(np.complex128)
        assert np.array_equal(bits(g), bits(ref[1]))
    else:
        _, rp, ci, vals, ncols = ref
        assert isinstance(got, CsrMatrix)
        assert (got.ncols or got.n) == ncols
        assert np.array_equal(got.rowptr, rp) and np.array_equal(got.cols.astype(np.int64), ci)
        assert np.array_equal(bits(np.asarray(got.vals).astype(np.complex128)), bits(vals))
    return got


# ---- the reference's known-answer tests (test_matrix_market.cpp) ----------
def test_dense_complex_round_trip_bitwise(tmp_path):
    rng = np.random.default_rng(31)
    m = rng.uniform(-1, 1, (3, 4)) + 1j * rng.uniform(-1, 1, (3, 4))
    p = str(tmp_path / "dense.mtx")
    P.write_matrix_market(m, p)
    back = P.read_matrix_market(p)
    assert back.shape == (3, 4) and np.array_equal(bits(back), bits(m))


def test_sparse_round_trip_keeps_sparsity(tmp_path):
    m = CsrMatrix(5, np.array([0, 1, 1, 2, 2, 3]), np.array([0, 1, 4], np.int32), np.array([1.25, -0.5, 3.0]))
    p = str(tmp_path / "sparse.mtx")
    P.write_matrix_market(m, p)
    s = P.read_matrix_market(p)
    assert s.nnz == 3 and np.array_equal(s.todense(), m.todense())


def test_field_choice(tmp_path):
    p = str(tmp_path / "real.mtx")
    P.write_matrix_market(np.array([[1.0, 0.0], [0.0, -2.0]], dtype=complex), p)
    assert " real " in open(p).readline()
    P.write_matrix_market(np.array([[0.0, 1j], [0.0, 0.0]]), p)
    assert " complex " in open(p).readline()


def test_symmetric_coordinate_expands(tmp_path):
    p = write(tmp_path, "sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 2.0\n2 1 5.0\n"
                                    "3 2 -1.0\n")
    s = P.read_matrix_market(p)
    assert s.nnz == 5
    d = s.todense()
    assert d[0, 0] == 2.0 and d[1, 0] == d[0, 1] == 5.0 and d[2, 1] == d[1, 2] == -1.0


def test_array_column_major(tmp_path):
    p = write(tmp_path, "array.mtx", "%%MatrixMarket matrix array real general\n% comment line\n2 2\n1\n2\n3\n4\n")
    assert np.array_equal(P.read_matrix_market(p), np.array([[1.0, 3.0], [2.0, 4.0]]))


@pytest.mark.parametrize("text", [
    "%%NotMatrixMarket nonsense\n1 1 1\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
])
def test_malformed_raises_ioerror_with_reference_message(R, tmp_path, text):
    assert assert_same(R, write(tmp_path, "bad.mtx", text)) is None
    with pytest.raises(P.IoError):
        P.read_matrix_market(str(tmp_path / "definitely_missing.mtx"))


# ---- parity corpus --------------------------------------------------------
def _fmt(x, style):
    return {"g": "%.17g" % x, "e": "%.6e" % x, "f": "%.9f" % x, "plus": "+%.17g" % x if x >= 0 else "%.17g" % x,
            "E": ("%.12E" % x)}[style]


@pytest.mark.parametrize("seed", range(6))
def test_coordinate_corpus_bitwise(R, tmp_path, seed):
    rng = np.random.default_rng(seed)
    rows, cols = int(rng.integers(1, 60)), int(rng.integers(1, 60))
    sym = seed % 3 == 1
    if sym:
        cols = rows
    cplx = seed % 2 == 1
    ne = int(rng.integers(0, 400))
    lines = [f"%%MatrixMarket matrix coordinate {'complex' if cplx else 'real'} "
             f"{'symmetric' if sym else 'general'}", "% generated", "", f"{rows} {cols} {ne}"]
    styles = ["g", "e", "f", "plus", "E"]
    for k in range(ne):
        i, j = int(rng.integers(1, rows + 1)), int(rng.integers(1, cols + 1))
        if sym and j > i:
            i, j = j, i
        v = float(rng.normal() * 10.0 ** rng.integers(-8, 8))
        s = styles[k % len(styles)]
        line = f"{i} {j} {_fmt(v, s)}"
        if cplx:
            line += " " + _fmt(float(rng.normal()), styles[(k + 2) % len(styles)])
        if k % 17 == 3:
            line = "  \t" + line + "   extra tokens"
        lines.append(line)
        if k % 29 == 5:
            lines.append("% interleaved comment")
        if k % 31 == 7:
            lines.append("   ")
    text = "\n".join(lines) + ("\n" if seed % 2 else "")
    path = write(tmp_path, "c.mtx", text)
    a = assert_same(R, path, threads=1)
    b = assert_same(R, path, threads=8)
    if a is not None:
        assert np.array_equal(bits(np.asarray(a.vals).astype(complex)), bits(np.asarray(b.vals).astype(complex)))


@pytest.mark.parametrize("seed", range(4))
def test_array_corpus_bitwise(R, tmp_path, seed):
    rng = np.random.default_rng(100 + seed)
    sym = seed % 2 == 1
    rows = int(rng.integers(1, 40))
    cols = rows if sym else int(rng.integers(1, 40))
    cplx = seed >= 2
    lines = [f"%%MatrixMarket matrix array {'complex' if cplx else 'real'} {'symmetric' if sym else 'general'}",
             f"{rows} {cols}"]
    for j in range(cols):
        for i in range(j if sym else 0, rows):
            v = "%.17g" % float(rng.normal())
            lines.append(v + (" %.17g" % float(rng.normal()) if cplx else ""))
    path = write(tmp_path, "a.mtx", "\r\n".join(lines) + "\r\n")  # CRLF: '\r' is whitespace to istream
    assert_same(R, path, threads=1)
    assert_same(R, path, threads=8)


def test_duplicates_and_unsorted_entries(R, tmp_path):
    # the reference sums duplicates in std::sort's order; the same sort on the
    # same sequence reproduces it
    rng = np.random.default_rng(5)
    lines = ["%%MatrixMarket matrix coordinate complex general", "7 5 300"]
    for _ in range(300):
        lines.append(f"{rng.integers(1, 8)} {rng.integers(1, 6)} {rng.normal():.17g} {rng.normal():.17g}")
    assert_same(R, write(tmp_path, "dup.mtx", "\n".join(lines) + "\n"), threads=8)


@pytest.mark.parametrize("body", [
    "2 2 1\n1 1 1e400\n",            # overflow fails like num_get
    "2 2 1\n1 1 1e-400\n",           # underflow gives strtod's 0
    "2 2 1\n1 1 4.9e-324\n",         # smallest denormal
    "2 2 1\n1 1 inf\n",
    "2 2 1\n1 1 nan\n",
    "2 2 1\n1 1 1e\n",
    "2 2 1\n1 1 .5\n",
    "2 2 1\n1 1 5.\n",
    "2 2 1\n1 1 0x10\n",             # num_get stops at 'x': value 0
    "2 2 1\n1.5 1 2.0\n",
    "2 2 1\n+1 +2 -3.25\n",
    "2 2 1\n1 1\n",
    "2 2 x\n1 1 1.0\n",              # failed count extraction stores 0: an empty matrix
    "2 x 1\n1 1 1.0\n",
    "2 2\n1 1 1.0\n",
    "-1 2 1\n1 1 1.0\n",
    "2 2 1\n1 0 1.0\n",
    "2 2 0\n",
    "2 2 1\n\n\n% c\n2 2 7\nignored tail line\n",
])
def test_edge_cases_match_reference(R, tmp_path, body):
    assert_same(R, write(tmp_path, "e.mtx", "%%MatrixMarket matrix coordinate real general\n" + body))


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix array real general\n2 x\n",
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
    "%%MatrixMarket matrix array real general\n2 2\n1\nfoo\n3\n4\n",
    "%%MatrixMarket matrix array real symmetric\n2 3\n1\n",
    "%%MatrixMarket matrix array complex general\n1 1\n1\n",
    "%%MatrixMarket matrix array real general\n0 0\n",
    "%%matrixmarket MATRIX Array REAL General\n1 1\n7\n",
    "%%MatrixMarket matrix\n",
    "\n",
])
def test_array_and_banner_edge_cases(R, tmp_path, text):
    assert_same(R, write(tmp_path, "b.mtx", text))


def test_writers_byte_identical(R, tmp_path):
    rng = np.random.default_rng(9)
    dense_r = rng.normal(size=(13, 7)) * 1e-3
    dense_c = rng.normal(size=(5, 9)) + 1j * rng.normal(size=(5, 9))
    special = np.array([[0.0, -0.0, 5e-324, 1e-300], [1e300, -1.7976931348623157e308, 123456789012345678.0, 0.1],
                        [np.inf, -np.inf, 1e-5, 1e16], [2.5e-7, 1e21, 1e-7, 33.0]])
    special_c = special + 1j * special[::-1]
    for a in (dense_r, dense_c, np.zeros((0, 3)), dense_r.astype(complex), special, special_c):
        ours, ref = str(tmp_path / "o.mtx"), str(tmp_path / "r.mtx")
        P.write_matrix_market(a, ours, threads=8)
        R.write_dense(a, ref)
        assert open(ours, "rb").read() == open(ref, "rb").read()
    n = 200
    d = rng.normal(size=(n, n + 3))
    d[rng.uniform(size=d.shape) < 0.9] = 0.0
    rows, cols = np.nonzero(d)
    rp = np.searchsorted(rows, np.arange(n + 1)).astype(np.int64)
    for vals in (d[rows, cols], d[rows, cols] + 1j * rng.normal(size=rows.size)):
        m = CsrMatrix(n, rp, cols.astype(np.int32), vals, ncols=n + 3)
        ours, ref = str(tmp_path / "o.mtx"), str(tmp_path / "r.mtx")
        P.write_matrix_market(m, ours, threads=8)
        R.write_csr(n, n + 3, rp, cols, vals, ref)
        assert open(ours, "rb").read() == open(ref, "rb").read()
        assert_same(R, ours, threads=8)


def test_large_file_threads_agree(R, tmp_path):
    """300k entries: the threaded parse equals the single-threaded one and the reference."""
    rng = np.random.default_rng(1)
    n, ne = 20000, 300000
    i = rng.integers(1, n + 1, ne)
    j = rng.integers(1, n + 1, ne)
    v = rng.normal(size=ne)
    path = str(tmp_path / "big.mtx")
    with open(path, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate real general\n{n} {n} {ne}\n")
        f.write("\n".join(f"{a} {b} {c:.17g}" for a, b, c in zip(i, j, v)))
        f.write("\n")
    a = assert_same(R, path, threads=1)
    b = P.read_matrix_market(path, threads=16)
    assert np.array_equal(a.rowptr, b.rowptr) and np.array_equal(a.cols, b.cols)
    assert np.array_equal(bits(a.vals), bits(b.vals))
    os.remove(path)
