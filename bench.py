"""Benchmark: SpHcurlAMG setup + PCG solve to 1e-8 on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A step is one pass of the hot path over one synthetic problem: build_hierarchy
(constrained-energy-minimisation prolongators, Galerkin products, coarse
gradients) followed by pcg_solve with the Chebyshev-Hiptmair V-cycle, rtol 1e-8.
The default workload is the largest BASELINE.json config that fits one GPU
with the reference's settings, configs[3] ("C4": 128^3 hex, natural BC,
lognormal per-element sigma, jittered isoparametric hexes, RHS U[-1,1], all
from default_rng(3), coarse_size 1000). Inputs are synthetic, assembled on
the device (csrc/assemble.cu); the reference arm runs on the bit-identical
host build of the same rows (oracle/host_assembly.py).

value = edge DOFs/s of setup + solve with the inputs resident in HBM; e2e = the
same through the public API with host (scipy / numpy) inputs and the solution
copied back, host<->device copies inside the timed region. Multi-GPU (torchrun,
--gpus N): ONE problem, row-block sharded setup + row-block partitioned solve
(strong scaling; neighbour halo exchanges and all-reduced PCG scalars over
NCCL -- DESIGN.md "Multi-GPU"); --replicas runs N independent replicas instead
(weak scaling, no data-path collective). Timing is the max over ranks.

--impl reference times the reference algorithm's CPU implementation (the
oracle port in oracle/, Gauss-Seidel smoother as in the reference) on rank 0,
re-executed under the survey's pin (OPENBLAS_CORETYPE=Haswell,
OPENBLAS_NUM_THREADS=1, ``taskset -c 0``: one host core) before numpy loads.
"""

import os
import sys

_PIN_ENV = {"OPENBLAS_CORETYPE": "Haswell", "OPENBLAS_NUM_THREADS": "1",
            "OMP_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"}


def _pinned_cmd(argv):
    """argv under ``taskset -c 0`` (when available) for the 1-core CPU legs."""
    import shutil
    cmd = [sys.executable] + list(argv)
    if shutil.which("taskset"):
        cmd = ["taskset", "-c", "0"] + cmd
    return cmd


def _reexec_pinned():
    """The CPU arms (--impl reference, --cpu-sample) must see the BLAS pin
    before numpy is imported, and run on one core: re-exec once."""
    argv = sys.argv[1:]
    cpu_leg = ("--cpu-sample" in argv or
               any(a == "--impl=reference" for a in argv) or
               ("--impl" in argv and argv[argv.index("--impl") + 1:][:1] == ["reference"]))
    if cpu_leg and os.environ.get("SPHC_CPU_PINNED") != "1":
        env = dict(os.environ, SPHC_CPU_PINNED="1", **_PIN_ENV)
        cmd = _pinned_cmd(sys.argv)
        os.execvpe(cmd[0], cmd, env)


if __name__ == "__main__":
    _reexec_pinned()

import argparse
import json
import math
import statistics
import subprocess
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


_NVML_POLL = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
    nv.nvmlDeviceGetCurrentClocksThrottleReasons
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
while True:
    try:
        print(time.time(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx, int(get_r(h)),
              flush=True)
    except Exception:
        pass
    time.sleep(0.005)
"""


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region by a
    separate process (NVML polled every 5 ms; nvidia-smi -lms 200 if pynvml
    is missing), so sampling never contends for this process's GIL while
    the host drives the setup."""

    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None
        self.kind = None

    def __enter__(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
        try:
            import pynvml  # noqa: F401
            # samples go to a file, not a pipe: a pipe nobody drains fills
            # up after ~5 s and blocks the poller (long C4/C5 runs)
            self.out = tempfile.TemporaryFile(mode="w+")
            self.p = subprocess.Popen([sys.executable, "-c", _NVML_POLL, str(idx)],
                                      stdout=self.out, stderr=subprocess.DEVNULL,
                                      text=True)
            self.kind = "nvml"
            time.sleep(0.2)        # first samples before the timed region
        except Exception:   # noqa: BLE001
            try:
                self.out = tempfile.TemporaryFile(mode="w+")
                self.p = subprocess.Popen(
                    ["nvidia-smi", "-i", str(idx), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits", "-lms", "200"],
                    stdout=self.out, stderr=subprocess.DEVNULL, text=True)
                self.kind = "nvidia-smi"
            except OSError:
                self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            self.p.terminate()
            self.p.wait(timeout=10)
            self.out.seek(0)
            self.lines = [l for l in self.out.read().splitlines() if l.strip()]
            self.out.close()

    def mark(self, which):
        """Wall-clock bounds of the timed region (samples outside are dropped)."""
        setattr(self, which, time.time())

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            if self.kind == "nvml":
                f = l.split()
                try:
                    ts, clk, cmax, bits = float(f[0]), float(f[1]), float(f[2]), int(f[3])
                except (ValueError, IndexError):
                    continue
                if t0 is not None and t1 is not None and not (t0 <= ts <= t1):
                    continue
                sm.append(clk)
                mx = max(mx, cmax)
                reasons |= {k for k, b in self.BITS.items() if bits & b}
                continue
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm), "source": self.kind}


def vcycle_bytes(h, degree=3):
    """Algorithmic bytes of one V-cycle: per level
    p_A beta(A_e) + p_X beta(D^T A D) + p_D beta(D) + p_P beta(P_e), plus the
    dense coarsest GEMV; beta(M) = 12 nnz + 8 (rows + 1) + 8 (rows + cols)."""
    def beta(M):
        r, c = M.shape
        return 12 * M.nnz + 8 * (r + 1) + 8 * (r + c)
    pA, pX, pD, pP = 4 * degree + 3, 2 * degree, 4, 2
    tot = 0
    for lv in h.levels[:-1]:
        tot += pA * beta(lv.A_e) + pX * beta(lv.nodal_aux) + pD * beta(lv.D) + pP * beta(lv.P_e)
    nc = h.levels[-1].A_e.shape[0]
    return tot + 8 * nc * nc + 16 * nc


def cheb_kernel_bytes(A):
    """Algorithmic bytes of one fused Chebyshev step on A by SURVEY.md 8(d)'s
    formula: the CSR pass (12 nnz + 8 (n + 1)) plus x gather, b, dinv, d
    (read + write), x_out."""
    n = A.shape[0]
    return 12 * A.nnz + 8 * (n + 1) + 8 * 6 * n


def cheb_kernel_bytes_coded(A, nbase=1):
    """The same step on delta-coded columns (csrc/sell.cu k_sell_cheb16): 8 B
    of value + 2 B of column difference per entry, 4 B of first column per
    row, the slice pointers, the same six vector passes."""
    n = A.shape[0]
    return 10 * A.nnz + 4 * nbase * n + 8 * (n // 32 + 2) + 8 * 6 * n


def vcycle_bytes_moved(h, degree=3):
    """Compulsory bytes of one V-cycle in the formats the kernels actually
    read (delta-coded SELL where built, the fused Hiptmair mid step: one A D
    pass instead of a D and an A_e pass per sweep, no pass for a zero initial
    guess), for the hardware-utilisation figure next to the survey's
    algorithmic one."""
    def sell_pass(M, m, vecs):
        r, c = M.shape
        per = 10 if (m is not None and getattr(m, "d16", None) is not None) else 12
        return per * M.nnz + 8 * (r + 1) + 8 * vecs * r
    def csr_pass(M):
        r, c = M.shape
        return 12 * M.nnz + 8 * (r + 1) + 8 * (r + c)
    tot = 0
    for lv in h.levels[:-1]:
        es, ax = lv.edge_sweeper, lv.aux_sweeper
        me = getattr(es, "sell", None)
        ma = getattr(ax, "sell", None)
        mid = getattr(lv, "mid", None)
        # per V-cycle: two Hiptmair sweeps; each = edge Chebyshev (degree
        # steps), residual, D^T r, nodal Chebyshev from zero, x += D c, edge
        # Chebyshev; plus the residual / restriction / prolongation between
        a_cheb = 4 * degree - 1 - (2 if mid is not None else 0)   # steps with an A pass
        tot += a_cheb * sell_pass(lv.A_e, me, 6)
        tot += 3 * sell_pass(lv.A_e, me, 3)                       # residuals
        if mid is not None:
            n = lv.A_e.shape[0]
            per = 10 if mid.d16 is not None else 12
            # A D entries + D's CSR + r, dinv, x_in, x_out, d and the c gathers
            tot += 2 * (per * mid.val.numel() + 12 * lv.D.nnz + 16 * (n + 1) + 8 * 6 * n)
        else:
            tot += 2 * csr_pass(lv.D)
        tot += 2 * (degree - 1) * sell_pass(lv.nodal_aux, ma, 6)
        tot += 2 * csr_pass(lv.Dt) + csr_pass(lv.P_e) + csr_pass(lv.R_e)
    nc = h.levels[-1].A_e.shape[0]
    return tot + 8 * nc * nc + 16 * nc


def ncu_traffic_file(config):
    """The committed ncu --set full summary of the roofline kernel for this
    workload: profiles/*_<config>_k_sell_cheb_full.txt (newest round)."""
    import glob
    files = sorted(glob.glob(os.path.join(REPO, "profiles",
                                          f"r*_{config.lower()}_k_sell_cheb_full.txt")))
    return os.path.relpath(files[-1], REPO) if files else None


def ncu_traffic(config):
    """DRAM bytes (read + write) per launch of the roofline kernel from that
    summary, or None."""
    f = ncu_traffic_file(config)
    if f is None:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    found = 0
    for line in open(os.path.join(REPO, f)):
        x = line.split()
        if len(x) == 3 and x[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(x[1]) * scale.get(x[2], 1)
            found += 1
    return tot if found == 2 else None


_FLUSH_R = None


def cold_flush(flush, v):
    """Untimed: write 256 MB (> 126 MB L2), then read a clean 256 MB buffer."""
    flush.fill_(v)
    if _FLUSH_R is not None:
        _FLUSH_R.sum()


def scale_roofline(args, flush):
    """The same kernel (fused SELL Chebyshev step) on the finest A_e of a
    config larger than L2 (default C3: 811k edges, 26M nonzeros, 313 MB),
    each launch timed alone after an L2 flush."""
    import torch
    from paper_2506_08284_b200 import _lib, device as dv
    if args.scale_config in DEVICE_INPUTS:
        A = make_device_problem(args.scale_config)[0].A_e
    else:
        A = dv.DeviceCSR.from_scipy(make_problem(args.scale_config)[0].A_e)
    n = A.shape[0]
    m = dv.sell(A)
    dinv = dv.reciprocal(dv.diagonal(A))
    g = torch.Generator(device="cpu").manual_seed(0)
    b = torch.rand(n, generator=g, dtype=torch.float64).cuda()
    x = torch.rand(n, generator=g, dtype=torch.float64).cuda()
    out, d = torch.empty_like(x), torch.zeros_like(x)

    def k():
        _lib.call("sphc_sell_cheb_step", n, m.slice_ptr, m.col, m.val, dinv, b, x, out, d,
                  0.3, 0.7, 0, m.padded)

    for _ in range(3):
        k()
    nk = 20
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(nk)]
    for i in range(nk):
        cold_flush(flush, 100.0 + i)
        ev[i][0].record()
        k()
        ev[i][1].record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(bb) for a, bb in ev)[nk // 2]
    byts = cheb_kernel_bytes(A)
    pk, kind = peaks()
    ach = byts / (t * 1e-3) / 1e9
    return {"config": f"{args.scale_config} finest A_e ({n} rows, {A.nnz} nnz)",
            "kernel": "k_sell_cheb", "launch_ms_median": t, "algorithmic_bytes": byts,
            "achieved": ach, "peak": float(pk["hbm_gbs"]), "unit": "GB/s",
            "frac": ach / float(pk["hbm_gbs"]), "sell_padding": m.padded / A.nnz,
            "traffic": ncu_traffic(args.scale_config),
            "traffic_source": ncu_traffic_file(args.scale_config)}


DEVICE_INPUTS = ("C3", "C4", "C5")


def make_problem(config, N=None):
    """Host (scipy) inputs: bit-identical to the reference's assembly for
    C1/C2; C3-C5 are generated on the device (csrc/assemble.cu: per-element
    sigma, jittered hexes for C4) and downloaded."""
    if config in DEVICE_INPUTS:
        sysd, rhs, cfg = make_device_problem(config, N)
        from types import SimpleNamespace
        return SimpleNamespace(**{k: getattr(sysd, k).to_scipy()
                                  for k in ("A_e", "S", "A_n", "D")}), rhs, cfg
    from paper_2506_08284_b200.inputs import make_config
    sysm, rhs, cfg = make_config(config, N)
    return sysm, rhs, cfg


def make_device_problem(config, N=None):
    from paper_2506_08284_b200.assembly import make_device_config
    return make_device_config(config, N)


def run_ours(args):
    import torch
    import torch.distributed as tdist
    from paper_2506_08284_b200 import _lib, device as dv, multigrid as mg
    from paper_2506_08284_b200.build import build_library

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    build_library()
    dev = torch.device("cuda", torch.cuda.current_device())
    # inputs resident in HBM for the device-timed value
    if args.config in DEVICE_INPUTS:
        sysd, rhs, cfg = make_device_problem(args.config, args.N)
        A_e, S, A_n, D = sysd.A_e, sysd.S, sysd.A_n, sysd.D
        # host copies for the e2e leg (skipped above ~10M edges: C5's
        # host matrices alone are ~50 GB)
        sysm = None
        if sysd.n_edges <= 10_000_000 and not args.no_e2e:
            from types import SimpleNamespace
            sysm = SimpleNamespace(**{k: getattr(sysd, k).to_scipy()
                                      for k in ("A_e", "S", "A_n", "D")})
    else:
        sysm, rhs, cfg = make_problem(args.config, args.N)
        A_e = dv.DeviceCSR.from_scipy(sysm.A_e)
        S = dv.DeviceCSR.from_scipy(sysm.S)
        A_n = dv.DeviceCSR.from_scipy(sysm.A_n)
        D = dv.DeviceCSR.from_scipy(sysm.D)
        if args.no_e2e:
            sysm = None
    n_e = A_e.shape[0]
    if args.coarse_size is None:
        args.coarse_size = cfg.get("coarse_size", 1000)
    scfg = mg.SolverConfig(coarse_size=args.coarse_size, smoother=args.smoother)
    b = torch.from_numpy(rhs).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    # the per-launch roofline timings also read a second, never-written
    # 256 MB buffer after the write flush: the flush's dirty L2 lines are
    # written back before the timed launch instead of during it (ncu's
    # clean-cache replay measures the same way)
    global _FLUSH_R
    _FLUSH_R = torch.zeros(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    # N > 1: one problem, row-block sharded setup + partitioned solve
    # (strong scaling) unless --replicas; N = 1: the single-GPU path
    # (--partitioned runs the partitioned code on a one-rank group)
    partitioned = args.partitioned or (ws > 1 and not args.replicas)
    if partitioned and ws == 1 and not tdist.is_initialized():
        # one-rank group: exercises the sharded / partitioned path on 1 GPU
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            os.environ.setdefault("MASTER_PORT", str(so.getsockname()[1]))
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        tdist.init_process_group("nccl", rank=0, world_size=1)
    if partitioned:
        from paper_2506_08284_b200 import distributed as dist_mod

    shard = None
    if partitioned:
        from paper_2506_08284_b200.sharding import Sharding
        shard = Sharding.from_group()

    def step():
        h = mg.build_hierarchy(A_e, S, A_n, D, scfg, shard=shard)
        if partitioned:
            # row-block sharded setup, row-block partitioned solve (strong scaling)
            dh = dist_mod.distribute_hierarchy(h)
            part = dh.levels[0].edge_part
            res = dist_mod.dist_pcg_solve(dh, b[part.lo(rank):part.hi(rank)].contiguous())
            return h, res
        res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
        return h, res

    def barrier():
        if ws > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    h = res = None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    # the sampler starts before the warm-up (no idle gap that would let the
    # clocks drop before the timed steps); only samples inside the timed
    # region are summarised
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            h = res = None            # free the previous hierarchy first (C5: ~140 GB)
            h, res = step()
        barrier()
        l0 = _lib.launch_count()
        clk.mark("t0")
        for k in range(args.steps):
            flush.fill_(float(k))          # L2 flush (256 MB > 126 MB L2), untimed
            h = res = None
            ev[k][0].record()
            h, res = step()
            ev[k][1].record()
        barrier()
        clk.mark("t1")
    launches = (_lib.launch_count() - l0) // args.steps
    step_ms = [a.elapsed_time(bb) for a, bb in ev]
    from paper_2506_08284_b200 import trace
    if trace.ENABLED:
        print("step ms:", step_ms, "\n" + trace.report(), file=sys.stderr)
    t_step = sum(step_ms) / args.steps
    if ws > 1:
        t = torch.tensor([t_step], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        t_step = float(t.item())
    iters = res.iterations
    assert res.status == "converged", res.status

    # setup / solve split and V-cycle bandwidth (device events, untimed region)
    h = res = None
    flush.fill_(1.0)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    h = mg.build_hierarchy(A_e, S, A_n, D, scfg)
    e1.record()
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    e2.record()
    torch.cuda.synchronize()
    t_setup, t_solve = e0.elapsed_time(e1), e1.elapsed_time(e2)
    pre = mg.v_cycle_preconditioner(h)
    nv = 20
    for _ in range(3):
        pre(b)
    # the V-cycle as the solve runs it: captured once, replayed (device time,
    # no host launch gaps); each replay after an L2 flush at C4/C5 sizes is
    # the same as back to back since the working set exceeds L2 there
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        vgraph = mg.PcgGraph(lambda: pre(b))
    torch.cuda.current_stream().wait_stream(cap)
    vgraph.replay()
    flush.fill_(2.0)
    v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    v0.record()
    for _ in range(nv):
        vgraph.replay()
    v1.record()
    torch.cuda.synchronize()
    del vgraph
    t_vc = v0.elapsed_time(v1) / nv
    vbytes = vcycle_bytes(h, scfg.cheb_degree)

    # dominant solve kernel: the fused Chebyshev step on the finest A_e (SELL
    # layout). Each launch is timed alone after an L2 flush (cold HBM), and a
    # back-to-back warm loop is reported beside it.
    sw = h.levels[0].edge_sweeper
    A0 = h.levels[0].A_e
    x0 = torch.zeros(n_e, dtype=torch.float64, device=dev)
    gs_mode = not hasattr(sw, "coefs")
    if gs_mode:
        # the reference smoother: the lower Gauss-Seidel half sweep
        def kstep():
            _lib.call("sphc_gs_half_sweep", n_e, A0.rowptr, A0.col, A0.val, b, x0, sw.buf[0],
                      sw.y, sw.ticket, 1, sw.status.t)
    else:
        m0 = sw.sell
        cd, cr = sw.coefs[1]
        coded = getattr(m0, "d16", None) is not None     # the kernel the solve runs

        def kstep():
            if coded:
                _lib.call("sphc_sell_cheb_step16", n_e, m0.slice_ptr, m0.d16, m0.c0, m0.val,
                          sw.dinv, b, x0, sw.buf[0], sw.d, cd, cr, m0.nbase)
            else:
                _lib.call("sphc_sell_cheb_step", n_e, m0.slice_ptr, m0.col, m0.val, sw.dinv, b,
                          x0, sw.buf[0], sw.d, cd, cr, 0, m0.padded)

    for _ in range(3):
        kstep()
    nk = 30
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(nk)]
    for k in range(nk):
        cold_flush(flush, 10.0 + k)
        kev[k][0].record()
        kstep()
        kev[k][1].record()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record()
    for _ in range(nk):
        kstep()
    k1.record()
    torch.cuda.synchronize()
    t_k = sum(a.elapsed_time(bb) for a, bb in kev) / nk
    t_k_warm = k0.elapsed_time(k1) / nk
    kbytes = (12 * A0.nnz + 8 * (n_e + 1) + 32 * n_e) if gs_mode else cheb_kernel_bytes(A0)
    # hardware utilisation is judged on the bytes of the format the kernel
    # reads (delta-coded columns: 10 B per entry); the survey's 12 B formula
    # is reported beside it
    kbytes_fmt = (cheb_kernel_bytes_coded(A0, m0.nbase) if (not gs_mode and coded) else kbytes)
    vmoved = vcycle_bytes_moved(h, scfg.cheb_degree) if not gs_mode else vbytes
    # the main roofline is already at scale (> L2) for C3-C5
    at_scale = (None if args.no_scale_roofline or args.config in DEVICE_INPUTS
                else scale_roofline(args, flush))

    # e2e: public API with host inputs, solution back to host
    e2e = None
    if sysm is not None:
        e2e_ms, first_ms = [], None
        for k in range(-2, max(2, min(args.steps, 5))):    # k < 0: untimed warm-up
            flush.fill_(3.0 + k)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            he = mg.build_hierarchy(sysm.A_e, sysm.S, sysm.A_n, sysm.D, scfg, shard=shard)
            if partitioned:
                dh = dist_mod.distribute_hierarchy(he)
                part = dh.levels[0].edge_part
                bo = torch.from_numpy(rhs[part.lo(rank):part.hi(rank)]).to(dev)
                re = dist_mod.dist_pcg_solve(dh, bo)
                re.x = re.x.cpu().numpy()          # the owned block back to the host
                del dh
            else:
                # the reference's own usage: pcg_solve(h.levels[0].A_e, b, V(h))
                re = mg.pcg_solve(he.levels[0].A_e, rhs, mg.v_cycle_preconditioner(he))
            torch.cuda.synchronize()
            if k >= 0:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
            elif first_ms is None:
                # first public-API call on these host arrays (staging buffers,
                # graph capture and instantiation included)
                first_ms = (time.perf_counter() - t0) * 1e3
            assert isinstance(re.x, np.ndarray)
            del he, re
        t_e2e = sum(e2e_ms) / len(e2e_ms)
        if ws > 1:
            t = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            t_e2e = float(t.item())

        # build_hierarchy uploads (A_e, S, A_n, D); pcg_solve uploads b
        # (int64 row pointers and int32 columns on the device)
        def dev_bytes(M):
            return M.data.size * 8 + M.indices.size * 4 + M.indptr.size * 8
        # every rank uploads the whole system (replicated / sharded setup)
        h2d = ws * sum(dev_bytes(M) for M in (sysm.A_e, sysm.S, sysm.A_n, sysm.D)) + \
            (1 if partitioned else ws) * rhs.nbytes
        e2e = {"value": (1 if partitioned else ws) * n_e / (t_e2e * 1e-3),
               "unit": "edge DOFs/s",
               "ms": t_e2e, "first_call_ms": first_ms, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int((1 if partitioned else ws) * n_e * 8),
               "host_memory": "caller arrays staged through a pinned buffer "
                              "(no page-locking of caller memory; SPHC_PIN=1 opts in)"}

    pk, pk_kind = peaks()
    peak = float(pk["hbm_gbs"])
    achieved = kbytes_fmt / (t_k * 1e-3) / 1e9
    line = None
    if rank == 0:
        cpu = cpu_baseline(args) if (ws == 1 and not args.no_cpu_baseline) else None
        line = {
            "metric": "edge DOFs/s for setup + PCG solve to 1e-8",
            "value": (1 if partitioned else ws) * n_e / (t_step * 1e-3),
            "unit": "edge DOFs/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step,
            "higher_is_better": True, "scaling": "strong" if partitioned else "weak",
            "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (reference model problem, seeded RHS)",
            "config": workload_config(args.config, cfg, n_e, args.coarse_size),
            "run": {"levels": [lv.A_e.shape[0] for lv in h.levels],
                    "operator_complexity": h.operator_complexity,
                    "pcg_iterations": iters,
                    "smoother": ("chebyshev-3 hiptmair" if args.smoother == "chebyshev"
                                 else "symmetric gauss-seidel hiptmair (reference smoother)"),
                    "parallelism": (f"row-block sharded setup + partitioned solve x{ws}"
                                    if partitioned else f"replicas x{ws}"),
                    "l2": "256 MB flush before every timed step (inputs > L2 at C3-C5)"},
            "step_ms": [round(x, 3) for x in step_ms],
            "setup_ms": t_setup, "solve_ms": t_solve,
            "setup_dofs_per_s": n_e / (t_setup * 1e-3),
            "solve_dofs_per_s": n_e / (t_solve * 1e-3),
            "vcycle": {"ms": t_vc, "bytes": vbytes,
                       "achieved_gbs": vbytes / (t_vc * 1e-3) / 1e9,
                       "frac_of_peak": vbytes / (t_vc * 1e-3) / 1e9 / peak,
                       "bytes_note": "bytes = SURVEY.md 8(d)'s algorithmic formula (15 A_e "
                                     "passes of 12 B per entry); bytes_moved = what the "
                                     "kernels' formats read (fused mid step, delta-coded "
                                     "columns)",
                       "bytes_moved": vmoved,
                       "moved_gbs": vmoved / (t_vc * 1e-3) / 1e9,
                       "moved_frac_of_peak": vmoved / (t_vc * 1e-3) / 1e9 / peak},
            "roofline": {"bound": "hbm",
                         "kernel": ("k_gs_half<lower> (sync-free Gauss-Seidel half sweep, "
                                    "level-0 A_e; latency bound)" if gs_mode else
                                    ("k_sell_cheb16 (fused Chebyshev step, SELL-32 with "
                                     "delta-coded 16-bit columns, level-0 A_e)" if coded else
                                     "k_sell_cheb (fused Chebyshev step, SELL-32, level-0 A_e)")),
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "bytes_per_launch": kbytes_fmt,
                         "survey_formula": {"bytes": kbytes,
                                            "achieved": kbytes / (t_k * 1e-3) / 1e9,
                                            "frac": kbytes / (t_k * 1e-3) / 1e9 / peak},
                         "traffic": None if gs_mode else ncu_traffic(args.config),
                         "traffic_source": None if gs_mode else ncu_traffic_file(args.config),
                         "peak_source": pk_kind, "launch_ms": t_k,
                         "launch_ms_l2_warm": t_k_warm,
                         "l2_flushed_per_launch": "256 MB write + 256 MB clean read",
                         "sell_padding": None if gs_mode else m0.padded / max(A0.nnz, 1),
                         "algorithmic_bytes": kbytes_fmt},
            "roofline_at_scale": at_scale,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if tdist.is_initialized():
        tdist.barrier()
        tdist.destroy_process_group()
    return line


def host_problem(config, N=None):
    """Host (scipy) inputs for the CPU legs, no GPU needed: inputs.py for
    C1/C2 (bit-identical to the reference's assembly); for C3-C5 the host
    build of the device assembly rows (oracle/host_assembly.py; bit-identical
    to what the GPU arm assembles, tests/test_gpu_assembly.py)."""
    from types import SimpleNamespace
    if config in DEVICE_INPUTS:
        from oracle.host_assembly import config_host
        A_e, S, A_n, D, rhs, cfg = config_host(config, N)
        return SimpleNamespace(A_e=A_e, S=S, A_n=A_n, D=D), rhs, cfg
    from paper_2506_08284_b200.inputs import make_config
    return make_config(config, N)


def _oracle_step(sysm, rhs, coarse_size, smoother):
    from oracle import hcurl_oracle as O
    t0 = time.perf_counter()
    h = O.build_hierarchy(sysm.A_e, sysm.S, sysm.A_n, sysm.D, coarse_size=coarse_size,
                          smoother=smoother)
    t1 = time.perf_counter()
    res = O.solve(h, rhs)
    t2 = time.perf_counter()
    return t2 - t0, res, t1 - t0, t2 - t1


def host_info():
    """What the CPU legs ran on: lscpu model, os.cpu_count(), the affinity
    actually used (taskset -c 0 -> 1) and the BLAS pin."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for l in out.splitlines():
            if l.startswith("Model name:"):
                model = l.split(":", 1)[1].strip()
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = None
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "affinity_cores": aff,
            "openblas": {k: os.environ.get(k) for k in ("OPENBLAS_CORETYPE",
                                                        "OPENBLAS_NUM_THREADS")}}


# cpu_baseline sample per bench workload: the same recipe at a size whose
# port setup + solve takes ~10-20 s on one core
CPU_SAMPLE_N = {"C1": None, "C2": None, "C3": 32, "C4": 32, "C5": 32}


def cpu_sample(args):
    """--cpu-sample (re-executed pinned, one core): the oracle port's setup +
    solve on a bounded sample of the workload; prints one JSON line."""
    sysm, rhs, cfg = host_problem(args.config, args.N)
    t, res, ts, tv = _oracle_step(sysm, rhs, args.coarse_size or cfg.get("coarse_size", 1000),
                                  "gs")
    print(json.dumps({"t": t, "t_setup": ts, "t_solve": tv, "n_e": sysm.A_e.shape[0],
                      "N": cfg["N"], "its": res.iterations, "status": res.status,
                      "host": host_info()}), flush=True)


def cpu_baseline(args):
    """The oracle port (reference algorithm, Gauss-Seidel) on a bounded
    sample of the workload -- the same recipe at CPU_SAMPLE_N[config] --
    in a pinned one-core subprocess (this process has numpy loaded already)."""
    nsamp = CPU_SAMPLE_N.get(args.config)
    cmd = _pinned_cmd([os.path.abspath(__file__), "--cpu-sample", "--config", args.config] +
                      (["--N", str(nsamp)] if nsamp else []))
    env = dict(os.environ, SPHC_CPU_PINNED="1", **_PIN_ENV)
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, check=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    return {"value": r["n_e"] / r["t"], "unit": "edge DOFs/s",
            "cores": r["host"]["affinity_cores"] or 1, "kind": "port",
            "sample": f"{args.config} recipe at {r['N']}^3 ({r['n_e']} edges): oracle port "
                      f"setup {r['t_setup']:.2f} s + Gauss-Seidel PCG {r['its']} its "
                      f"{r['t_solve']:.2f} s, one core (taskset -c 0, OpenBLAS Haswell x1)",
            "host": r["host"]}


def host_cfg(config, N=None):
    """The config dict of a workload without building it."""
    from paper_2506_08284_b200.inputs import CONFIGS
    cfg = dict(CONFIGS[config])
    if N is not None:
        cfg["N"] = int(N)
    if cfg["sigma"] == "lognormal":
        cfg["geometry"] = "jittered isoparametric trilinear hexes (|dx| <= 0.2 h)"
    return cfg


def full_n_edges(cfg):
    """Edge count of the hex mesh."""
    N = cfg["N"]
    return 3 * N * (N - 1) ** 2 if cfg["dirichlet"] else 3 * N * (N + 1) ** 2


def workload_config(config, cfg, n_e, coarse_size):
    """The ``config`` object both arms print (identical for the same run)."""
    sig = cfg["sigma"]
    sig = sig if isinstance(sig, (int, float, str)) else "per-element"
    return {"workload": f"{config}: {cfg['N']}^3 hex, "
                        f"{'Dirichlet' if cfg['dirichlet'] else 'natural'} BC, sigma={sig}"
                        + (", jittered hexes" if cfg.get("geometry", "").startswith("jitter")
                           else "")
                        + f", rhs U[-1,1] seed {cfg['seed']}, coarse_size {coarse_size}, "
                          "PCG rtol 1e-8",
            "n_edges": int(n_e)}


# reference-arm sample per workload (--ref-N overrides; 0 = the full size):
# the full C4 setup + solve takes ~1 h on one core (the reference package
# itself ~3 h), far beyond a bench run, so each step runs the
# same recipe at 32^3
REF_SAMPLE_N = {"C3": 32, "C4": 32, "C5": 32}
REF_BUDGET_S = 150


def run_reference(args):
    """The reference's CPU path (the oracle port with the reference's
    Gauss-Seidel smoother; the reference package itself cannot travel to
    the GPU box) on one pinned core, rank 0 only. Each step is one full
    setup + solve of a bounded sample of the workload: the same recipe at
    REF_SAMPLE_N; --steps of them, or as many as fit REF_BUDGET_S."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    full_cfg = host_cfg(args.config, args.N)
    nsamp = REF_SAMPLE_N.get(args.config) if args.ref_N is None else (args.ref_N or None)
    sysm, rhs, cfg = host_problem(args.config, nsamp or args.N)
    n_e = sysm.A_e.shape[0]
    cs = args.coarse_size or cfg.get("coarse_size", 1000)
    wu = args.warmup
    s1, r1, _ = host_problem("C1")
    for _ in range(wu):        # warm-up on a small instance (imports, page-in)
        _oracle_step(s1, r1, 1000, "gs")
    # K timed steps, as many as fit REF_BUDGET_S of CPU time (or --ref-steps)
    kmax = args.steps if args.ref_steps is None else min(args.steps, args.ref_steps)
    times, res, t0 = [], None, time.perf_counter()
    while len(times) < max(1, kmax):
        t, res, ts, tv = _oracle_step(sysm, rhs, cs, "gs")
        times.append((t, ts, tv))
        if args.ref_steps is None and time.perf_counter() - t0 + t > REF_BUDGET_S:
            break
    k = len(times)
    tm = sum(x[0] for x in times) / k
    v = n_e / tm
    hi = host_info()
    line = {"impl": "reference", "metric": "edge DOFs/s for setup + PCG solve to 1e-8",
            "value": v, "unit": "edge DOFs/s", "n_gpus": ws, "steps": k,
            "warmup": wu, "ms_per_step": tm * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (reference model problem, seeded RHS)",
            "config": workload_config(args.config, full_cfg, full_n_edges(full_cfg), cs),
            "run": {"pcg_iterations": res.iterations, "status": res.status,
                    "sample": {"N": cfg["N"], "n_edges": int(n_e)},
                    "smoother": "symmetric gauss-seidel hiptmair (reference)",
                    "setup_s": [round(x[1], 3) for x in times],
                    "solve_s": [round(x[2], 3) for x in times]},
            "cpu_baseline": {"value": v, "unit": "edge DOFs/s",
                             "cores": hi["affinity_cores"] or 1, "kind": "port",
                             "sample": f"{args.config} recipe at {cfg['N']}^3 ({n_e} edges): "
                                       f"full setup + Gauss-Seidel PCG, {k} of the "
                                       f"{args.steps} requested steps (CPU budget "
                                       f"{REF_BUDGET_S} s), one core",
                             "host": hi},
            "e2e": {"value": v, "unit": "edge DOFs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--coarse-size", type=int, default=None,
                    help="default: the config's (1000; 10000 for C5)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--smoother", default="chebyshev", choices=["chebyshev", "gauss_seidel"])
    ap.add_argument("--ref-steps", type=int, default=None,
                    help="cap on the reference arm's timed steps (default: as many of "
                         "--steps as fit its CPU time budget)")
    ap.add_argument("--ref-N", type=int, default=None,
                    help="reference-arm sample size (default REF_SAMPLE_N; 0: full size)")
    ap.add_argument("--cpu-sample", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-scale-roofline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent replicas (weak scaling) instead of the "
                         "partitioned solve")
    ap.add_argument("--partitioned", action="store_true",
                    help="N=1: run the partitioned path on a one-rank group; "
                         "N>1: one problem, row-block sharded setup + partitioned solve "
                         "(strong scaling)")
    ap.add_argument("--scale-config", default="C3")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.cpu_sample:
        cpu_sample(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
