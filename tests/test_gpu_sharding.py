"""Sharded setup on the B200: every row-block phase (emin constraints and
sweeps, all SpGEMMs of the hierarchy) run block by block with the ranks
emulated in one process must give a hierarchy BITWISE equal to the
unsharded one (the per-row arithmetic does not depend on the partition)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    from paper_2506_08284_b200.build import build_library
    build_library()


def _eq(A, B):
    return (A.shape == B.shape and torch.equal(A.rowptr, B.rowptr) and torch.equal(A.col, B.col)
            and torch.equal(A.val, B.val))


def _inputs(case):
    from paper_2506_08284_b200 import device as dv
    from paper_2506_08284_b200.inputs import make_config
    if case == "C4dev":
        from paper_2506_08284_b200.assembly import make_device_config
        s, rhs, _ = make_device_config("C4", 12)
        return (s.A_e, s.S, s.A_n, s.D), rhs, 200
    s, rhs, _ = make_config("C1")
    return tuple(dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D)), rhs, 200


@pytest.mark.parametrize("case", ["C1", "C4dev"])
@pytest.mark.parametrize("world", [2, 3, 7])
def test_sharded_hierarchy_is_bitwise_identical(case, world):
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.sharding import Sharding
    ins, rhs, cs = _inputs(case)
    cfg = mg.SolverConfig(coarse_size=cs)
    h0 = mg.build_hierarchy(*ins, cfg)
    h1 = mg.build_hierarchy(*ins, cfg, shard=Sharding.emulated(world))
    assert len(h0.levels) == len(h1.levels) >= 2
    for a, b in zip(h0.levels, h1.levels):
        for k in ("A_e", "S_e", "D", "nodal_aux"):
            assert _eq(getattr(a, k), getattr(b, k)), k
        if a.P_e is not None:
            assert _eq(a.P_e, b.P_e)
            assert a.emin_energy == b.emin_energy
            assert a.commutator_residual == b.commutator_residual
            assert a.subproblem_dims == b.subproblem_dims
    assert torch.equal(h0.coarse_factorization, h1.coarse_factorization)
    r0 = mg.pcg_solve(h0.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h0))
    r1 = mg.pcg_solve(h1.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h1))
    assert r0.iterations == r1.iterations and r0.residual_history == r1.residual_history


def test_single_rank_group_nccl():
    """The collective path with a real 1-rank NCCL group (world 1: no-ops)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.sharding import Sharding
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        ins, rhs, cs = _inputs("C1")
        sh = Sharding.from_group()
        h = mg.build_hierarchy(*ins, mg.SolverConfig(coarse_size=cs), shard=sh)
        r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h))
        assert r.status == "converged"
    finally:
        dist.destroy_process_group()
