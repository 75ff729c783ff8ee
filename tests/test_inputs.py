"""The input generator reproduces the reference's assembly bit for bit."""

import pytest

from golden_util import csr_hash, inputs_table
from paper_2506_08284_b200.inputs import discretize_hex

TABLE = inputs_table()


@pytest.mark.parametrize("key", sorted(TABLE))
def test_assembly_bitwise(key):
    N, dirichlet, sigma = key.split("_")
    N = int(N)
    if N > 16:
        pytest.skip("covered by the N=32 slow test")
    s = discretize_hex(N, float(sigma), bool(int(dirichlet)))
    for k in ("A_e", "S", "A_n", "D"):
        assert csr_hash(getattr(s, k)) == TABLE[key][k], k


@pytest.mark.slow
def test_assembly_bitwise_n32():
    for key in [k for k in TABLE if k.startswith("32_")]:
        _, dirichlet, sigma = key.split("_")
        s = discretize_hex(32, float(sigma), bool(int(dirichlet)))
        for k in ("A_e", "S", "A_n", "D"):
            assert csr_hash(getattr(s, k)) == TABLE[key][k], (key, k)
