"""MatrixMarket ingestion, host side: the examples the
spec lists plus the hex system round trip that feeds build_hierarchy."""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2506_08284_b200 import mmio
from paper_2506_08284_b200.inputs import discretize_hex


def test_round_trip_random_bit_stable(tmp_path):
    rng = np.random.default_rng(0)
    A = sp.random(10, 7, density=0.4, random_state=rng, format="csr")
    A.data = rng.standard_normal(A.nnz) * np.exp(20 * rng.standard_normal(A.nnz))
    p = tmp_path / "a.mtx"
    mmio.write_matrix_market(A, p)
    B = mmio.read_matrix_market(p)
    assert B.shape == (10, 7)
    assert np.array_equal(B.indptr, A.indptr) and np.array_equal(B.indices, A.indices)
    assert np.array_equal(B.data.view(np.uint64), A.data.view(np.uint64))
    assert open(p).readline().strip() == mmio.BANNER


def test_zero_based_entry_rejected(tmp_path):
    p = tmp_path / "z.mtx"
    p.write_text(mmio.BANNER + "\n2 2 1\n0 1 1.0\n")
    with pytest.raises(ValueError, match="out of range"):
        mmio.read_matrix_market(p)


@pytest.mark.parametrize("banner,msg", [
    ("%%MatrixMarket matrix coordinate real symmetric", "symmetric-format"),
    ("%%MatrixMarket matrix array real general", "only 'coordinate real general'"),
    ("%%MatrixMarket matrix coordinate pattern general", "only 'coordinate real general'"),
    ("%MatrixMarket matrix coordinate real general", "malformed"),
])
def test_unsupported_formats(tmp_path, banner, msg):
    p = tmp_path / "f.mtx"
    p.write_text(banner + "\n2 2 1\n1 1 1.0\n")
    with pytest.raises(ValueError, match=msg):
        mmio.read_matrix_market(p)


def test_bad_counts_and_comments(tmp_path):
    p = tmp_path / "c.mtx"
    p.write_text(mmio.BANNER + "\n% exported\n%\n3 3 2\n1 1 2.5\n3 2 -1\n")
    A = mmio.read_matrix_market(p)
    assert A.toarray().tolist() == [[2.5, 0, 0], [0, 0, 0], [0, -1.0, 0]]
    p.write_text(mmio.BANNER + "\n3 3 3\n1 1 2.5\n3 2 -1\n")
    with pytest.raises(ValueError, match="expected 3 entries"):
        mmio.read_matrix_market(p)
    p.write_text(mmio.BANNER + "\n3 x 3\n")
    with pytest.raises(ValueError, match="size line"):
        mmio.read_matrix_market(p)


def test_duplicates_summed(tmp_path):
    p = tmp_path / "d.mtx"
    p.write_text(mmio.BANNER + "\n2 2 3\n1 2 1.0\n1 2 0.5\n2 1 4\n")
    A = mmio.read_matrix_market(p)
    assert A.nnz == 2 and A[0, 1] == 1.5 and A[1, 0] == 4.0


def test_gradient_entries_are_pm1(tmp_path):
    s = discretize_hex(2, 1.0, False)
    mmio.write_matrix_market(s.D, tmp_path / "D.mtx")
    lines = open(tmp_path / "D.mtx").read().splitlines()[2:]
    assert len(lines) == s.D.nnz == 2 * s.D.shape[0]
    assert {float(x.split()[2]) for x in lines} == {-1.0, 1.0}


def test_load_system_round_trip_and_dims(tmp_path):
    s = discretize_hex(4, 1e-2, True)
    paths = []
    for name in ("A_e", "S", "A_n", "D"):
        paths.append(tmp_path / f"{name}.mtx")
        mmio.write_matrix_market(getattr(s, name), paths[-1])
    A_e, S, A_n, D = mmio.load_system(*paths)
    for M, ref in ((A_e, s.A_e), (S, s.S), (A_n, s.A_n), (D, s.D)):
        ref = sp.csr_matrix(ref)
        ref.sort_indices()
        assert np.array_equal(M.indices, ref.indices)
        assert np.array_equal(M.data.view(np.uint64), ref.data.view(np.uint64))
    with pytest.raises(ValueError, match="inconsistent import: A_n"):
        mmio.load_system(paths[0], paths[1], paths[0], paths[3])
