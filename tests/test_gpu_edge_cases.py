"""Degenerate but valid inputs against the unmodified reference
(tests/edge_cases.py, golden tests/golden/edge_cases.json): zero right-hand
side (multigrid.py:232-233), a hierarchy that is only its coarsest level
(multigrid.py:119, 136-138), max_levels 1 and 2, maxit 0 and 1
(multigrid.py:243, 270), a loose tolerance, the 2^3 meshes and extreme sigma --
including the two on which the reference itself raises because the coarse
curl-curl operator is pure round-off (multigrid.py:114). The device runs the
reference's smoother; level sizes, statuses and iteration counts must be
equal, histories to 1e-6 (plus 1e-10 of |b| where the reference's own value
is round-off)."""

import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

import edge_cases
from golden_util import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.inputs import discretize_hex
    with open(os.path.join(GOLDEN, "edge_cases.json")) as f:
        golden = json.load(f)
    m = SimpleNamespace(mg=mg, system=discretize_hex,
                        config=lambda **kw: mg.SolverConfig(smoother="gauss_seidel", **kw))
    return m, golden


@pytest.mark.parametrize("name", sorted(edge_cases.CASES))
def test_edge_case_matches_reference(env, name):
    m, golden = env
    ref = golden[name]
    got = edge_cases.run(m, name)
    if "error" in ref:
        # the reference raises; the numbers in its message are round-off
        assert "error" in got, got
        assert got["error"][0] == ref["error"][0]
        head = ref["error"][1].split(": max|S D|")[0]
        assert got["error"][1].startswith(head), got["error"][1]
        return
    assert "error" not in got, got
    for k in ("n_levels", "n_edges", "status", "iterations", "x_size"):
        assert got[k] == ref[k], k
    assert abs(got["operator_complexity"] - ref["operator_complexity"]) < 1e-14
    b0 = ref["residual_history"][0]
    for k in ("residual_history", "precond_history"):
        assert len(got[k]) == len(ref[k]), k
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-6, atol=1e-10 * max(b0, 1e-300),
                                   err_msg=k)
    np.testing.assert_allclose(got["x_norm"], ref["x_norm"], rtol=1e-6)
    assert abs(got["relative_residual"] - ref["relative_residual"]) <= 1e-6 * ref[
        "relative_residual"] + 1e-10
