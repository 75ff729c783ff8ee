"""Error parity: the inputs on which the reference raises (tests/error_inputs.py,
run on the unmodified reference by tests/golden/make_golden.py error_inputs)
raise the same exception type with the same message on the device path --
malformed gradients, non-positive / zero diagonals, a violated null-space
identity, an all-zero curl-curl operator, Algorithm 1's empty rows and
columns, zero row sums, shape mismatches and the EminConfig validation
(reference file:line per case in error_inputs.json's order: edge_prolongator.py:
40-44, nodal_amg.py:43, emin_setup.py:73, multigrid.py:114, edge_prolongator.py:
163, multigrid.py:40, nodal_amg.py:133,146,149, coarse_gradient.py:81,49).
The device reports the lowest failing row through a status slot; the host
raises with the reference's text at the next readback."""

import json
import os
from types import SimpleNamespace

import pytest

import error_inputs
from golden_util import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    from paper_2506_08284_b200 import coarse_gradient as cgm
    from paper_2506_08284_b200 import edge_prolongator as epm
    from paper_2506_08284_b200 import emin_setup as es
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200 import nodal_amg as na
    from paper_2506_08284_b200.inputs import discretize_hex
    with open(os.path.join(GOLDEN, "error_inputs.json")) as f:
        golden = json.load(f)
    return SimpleNamespace(na=na, cgm=cgm, es=es, epm=epm, mg=mg), discretize_hex(4, 1.0, False), golden


@pytest.mark.parametrize("name", sorted(error_inputs.CASES))
def test_error_matches_reference(env, name):
    from paper_2506_08284_b200 import device as dv
    m, s, golden = env
    assert golden[name] is not None, "the reference raises on every case"
    try:
        got = error_inputs.run(m, s, name)
        if got is None:
            # device checks are deferred to the next readback
            try:
                dv.flush_checks()
            except Exception as e:      # noqa: BLE001
                got = [type(e).__name__, str(e)]
    finally:
        try:
            dv.flush_checks()
        except Exception:               # noqa: BLE001 -- leave no pending check behind
            pass
    assert got == golden[name]
