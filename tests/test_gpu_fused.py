"""Fused multi-step Chebyshev passes (csrc/sell.cu k_sell_cheb_fused): the
same buffers and arithmetic as the step-by-step launches, so results must be
BITWISE equal; checked on a streamed operator (A_e of a 48^3 hex mesh,
345,744 rows) and on its Hiptmair / V-cycle use."""

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


def _sweepers(A, fuse):
    from paper_2506_08284_b200 import multigrid as mg
    old = mg.FUSE_L2_BYTES
    mg.FUSE_L2_BYTES = 64 * 2**20          # fusion is opt-in
    try:
        sw = mg.ChebyshevSweeper(A, 3)
        mg.finalize_sweepers()
    finally:
        mg.FUSE_L2_BYTES = old
    if fuse is not None:
        if fuse and not sw.fuse:
            pytest.skip("operator too small / window too large for fusion")
        if fuse:
            sw.fuse = fuse
            nblk = (A.shape[0] + mg.FUSE_ROWS - 1) // mg.FUSE_ROWS
            sw.fuse_sync = torch.empty(1 + fuse * nblk, dtype=torch.int32, device="cuda")
        else:
            sw.fuse = 0
    return sw


@pytest.mark.parametrize("jitter", [False, True])
def test_fused_steps_bitwise_equal(jitter):
    from paper_2506_08284_b200.assembly import assemble_hex
    N = 48
    jit = None
    if jitter:
        rng = np.random.default_rng(3)
        jit = rng.uniform(-0.2 / N, 0.2 / N, ((N - 1) ** 3, 3))
    s = assemble_hex(N, 1e-2, False, jit)
    A = s.A_e
    n = A.shape[0]
    ref = _sweepers(A, 0)
    b = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
    x0 = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, n)).cuda()
    want_z = ref.symmetric(None, b, x_zero=True).clone()
    want_x = ref.symmetric(x0.clone(), b).clone()
    dref = ref.d.clone()
    for ks in (3, 2):
        sw = _sweepers(A, ks)
        assert sw.coefs == ref.coefs
        got_z = sw.symmetric(None, b, x_zero=True)
        assert torch.equal(got_z, want_z), ks
        got_x = sw.symmetric(x0.clone(), b)
        assert torch.equal(got_x, want_x), ks
        assert torch.equal(sw.d, dref), ks
        # input aliasing one of the sweeper's own buffers (the Hiptmair
        # post-smoothing case)
        sw.buf[1].copy_(x0)
        ref.buf[1].copy_(x0)
        assert torch.equal(sw.symmetric(sw.buf[1], b), ref.symmetric(ref.buf[1], b)), ks


def test_fused_hierarchy_solve_matches_unfused(monkeypatch):
    """A whole setup + solve with fused passes on every eligible level
    returns the bitwise-same iterate and histories as with fusion off."""
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.assembly import assemble_hex
    s = assemble_hex(48, 1.0, False)
    b = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, s.A_e.shape[0])).cuda()
    cfg = mg.SolverConfig(coarse_size=1000)
    out = []
    for mb in ("0", "64"):
        monkeypatch.setattr(mg, "FUSE_L2_BYTES", float(mb) * 2**20)
        h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, cfg)
        fused = [lv.edge_sweeper.fuse for lv in h.levels[:-1]]
        r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
        out.append((fused, r))
    assert out[0][0][0] == 0 and out[1][0][0] >= 2
    r0, r1 = out[0][1], out[1][1]
    assert r0.iterations == r1.iterations and r0.status == r1.status == "converged"
    assert r0.residual_history == r1.residual_history
    assert torch.equal(r0.x, r1.x)


@pytest.mark.parametrize("config,N,dirichlet_like", [("C4", 20, False), ("C2", 16, True)])
def test_hiptmair_mid_step_matches_unfused(config, N, dirichlet_like):
    """sphc_sell_hipt_mid (x + D c and the next sweep's first step from
    r - (A D) c) against the separate D pass and A pass: the same iterate to
    round-off (the two residuals differ only in summation order), the same
    PCG iteration count +-1, on a jittered natural-BC recipe and a
    Dirichlet one (D rows with a single entry)."""
    from paper_2506_08284_b200 import multigrid as mg, device as dv
    if config == "C4":
        from paper_2506_08284_b200.assembly import make_device_config
        s, rhs, cfg = make_device_config(config, N)
        A_e, S, A_n, D = s.A_e, s.S, s.A_n, s.D
    else:
        from paper_2506_08284_b200.inputs import make_config
        s, rhs, cfg = make_config(config, N)
        A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
    old = mg.HIPT_MID_MIN_ROWS
    try:
        mg.HIPT_MID_MIN_ROWS = -1
        h0 = mg.build_hierarchy(A_e, S, A_n, D, mg.SolverConfig(coarse_size=300))
        mg.HIPT_MID_MIN_ROWS = 0
        h1 = mg.build_hierarchy(A_e, S, A_n, D, mg.SolverConfig(coarse_size=300))
    finally:
        mg.HIPT_MID_MIN_ROWS = old
    assert all(lv.mid is None for lv in h0.levels)
    assert all(lv.mid is not None for lv in h1.levels[:-1])
    b = torch.from_numpy(rhs).cuda()
    x0 = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, rhs.size)).cuda()
    for xz in (True, False):
        w = mg.hiptmair_smooth(h0.levels[0], None if xz else x0.clone(), b, x_zero=xz).clone()
        g = mg.hiptmair_smooth(h1.levels[0], None if xz else x0.clone(), b, x_zero=xz).clone()
        err = float((w - g).abs().max() / w.abs().max())
        assert err < 1e-12, (xz, err)
    v0 = mg.v_cycle(h0, None, b).clone()
    v1 = mg.v_cycle(h1, None, b).clone()
    # the whole V-cycle amplifies the round-off difference through the
    # near-singular coarsest operators of the lognormal recipe (1e-8 there)
    assert float((v0 - v1).abs().max() / v0.abs().max()) < 1e-6
    r0 = mg.pcg_solve(h0.levels[0].A_e, b, mg.v_cycle_preconditioner(h0))
    r1 = mg.pcg_solve(h1.levels[0].A_e, b, mg.v_cycle_preconditioner(h1))
    assert r0.status == r1.status == "converged"
    assert abs(r0.iterations - r1.iterations) <= 1, (r0.iterations, r1.iterations)


def test_delta_coded_sell_kernels_are_bitwise():
    """sphc_sell_spmv16 / sphc_sell_cheb_step16 (16-bit column differences)
    against the 32-bit SELL kernels on a streamed operator (A_e of a 48^3
    jittered mesh): same entries, order and fma chain, so bitwise equal; a
    matrix with a column jump beyond 16 bits is reported as not
    representable and keeps its 32-bit columns."""
    from paper_2506_08284_b200 import device as dv
    from paper_2506_08284_b200._lib import call
    from paper_2506_08284_b200.assembly import assemble_hex
    N = 48
    rng = np.random.default_rng(3)
    s = assemble_hex(N, 1e-2, False, rng.uniform(-0.2 / N, 0.2 / N, ((N - 1) ** 3, 3)))
    A = dv.own_csr(s.A_e)
    n = A.shape[0]
    old = dv.SELL16_MIN_BYTES
    try:
        dv.SELL16_MIN_BYTES = 0
        m = dv.sell(A)
    finally:
        dv.SELL16_MIN_BYTES = old
    assert m.d16 is not None and m.c0 is not None
    x = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    b = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    dinv = dv.reciprocal(dv.diagonal(A))
    y0, y1 = torch.empty_like(x), torch.empty_like(x)
    call("sphc_sell_spmv", n, m.slice_ptr, m.col, m.val, x, -1.0, 1.0, b, y0, m.padded)
    call("sphc_sell_spmv16", n, m.slice_ptr, m.d16, m.c0, m.val, x, -1.0, 1.0, b, y1, m.nbase)
    assert torch.equal(y0, y1)
    d0 = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    d1 = d0.clone()
    o0, o1 = torch.empty_like(x), torch.empty_like(x)
    call("sphc_sell_cheb_step", n, m.slice_ptr, m.col, m.val, dinv, b, x, o0, d0, 0.3, 0.7, 0,
         m.padded)
    call("sphc_sell_cheb_step16", n, m.slice_ptr, m.d16, m.c0, m.val, dinv, b, x, o1, d1, 0.3,
         0.7, m.nbase)
    assert torch.equal(o0, o1) and torch.equal(d0, d1)
    # the fused Hiptmair mid step on delta-coded columns of A D
    D = dv.own_csr(s.D)
    AD = dv.spgemm(A, D, drop=False)
    old16 = dv.SELL16
    try:
        dv.SELL16 = False
        m32 = dv.sell_rect(AD)
        dv.SELL16, dv.SELL16_MIN_BYTES = True, 0
        m16 = dv.sell_rect(AD)
    finally:
        dv.SELL16, dv.SELL16_MIN_BYTES = old16, old
    assert m32.d16 is None and m16.d16 is not None
    c = torch.from_numpy(rng.uniform(-1, 1, D.shape[1])).cuda()
    r = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    o0, o1 = torch.empty_like(x), torch.empty_like(x)
    e0, e1 = torch.empty_like(x), torch.empty_like(x)
    call("sphc_sell_hipt_mid", n, m32.slice_ptr, m32.col, m32.val, D.rowptr, D.col, D.val, dinv,
         r, c, x, o0, e0, 0.7, m32.padded)
    call("sphc_sell_hipt_mid16", n, m16.slice_ptr, m16.d16, m16.c0, m16.val, D.rowptr, D.col,
         D.val, dinv, r, c, x, o1, e1, 0.7, m16.nbase)
    assert torch.equal(o0, o1) and torch.equal(e0, e1)
    assert m.nbase == 1 and m16.nbase == 1
    # jumps beyond 16 bits: up to three per row restart from the row's next
    # 32-bit base (the plane jumps of a 256^3 numbering); more are not
    # representable and the mirror keeps its 32-bit columns
    import scipy.sparse as sp
    nb = 300_000
    rows = np.repeat(np.arange(nb), 5)
    off = np.tile(np.array([0, 3, 70_000, 140_001, 210_500]), nb)
    cols = rows + off
    keep = cols < nb                       # no wrap-around: at most 3 far jumps per row
    rows, cols = rows[keep], cols[keep]
    Bs = sp.csr_matrix((rng.uniform(-1, 1, rows.size), (rows, cols)), shape=(nb, nb))
    Bs.sum_duplicates()
    Bs.sort_indices()
    dB = dv.DeviceCSR.from_scipy(Bs)
    try:
        dv.SELL16_MIN_BYTES = 0
        mb = dv.sell(dB)
    finally:
        dv.SELL16_MIN_BYTES = old
    assert mb.d16 is not None and mb.nbase == 4
    xb = torch.from_numpy(rng.uniform(-1, 1, nb)).cuda()
    y0, y1 = torch.empty_like(xb), torch.empty_like(xb)
    call("sphc_sell_spmv", nb, mb.slice_ptr, mb.col, mb.val, xb, 1.0, 0.0, None, y0, mb.padded)
    call("sphc_sell_spmv16", nb, mb.slice_ptr, mb.d16, mb.c0, mb.val, xb, 1.0, 0.0, None, y1,
         mb.nbase)
    assert torch.equal(y0, y1)
    assert np.allclose(y1.cpu().numpy(), Bs @ xb.cpu().numpy(), rtol=1e-12, atol=1e-12)
    off6 = np.tile(np.array([0, 66_000, 132_001, 198_002, 264_003, 299_000]), nb)
    rows6 = np.repeat(np.arange(nb), 6)
    cols6 = rows6 + off6
    k6 = cols6 < nb                        # row 0 keeps all six: four far jumps
    B6 = sp.csr_matrix((np.ones(int(k6.sum())), (rows6[k6], cols6[k6])), shape=(nb, nb))
    B6.sum_duplicates()
    B6.sort_indices()
    try:
        dv.SELL16_MIN_BYTES = 0
        m6 = dv.sell(dv.DeviceCSR.from_scipy(B6))
    finally:
        dv.SELL16_MIN_BYTES = old
    assert m6.d16 is None
