"""Collective layer of the sharded setup (paper_2506_08284_b200/sharding.py)
on CPU with gloo, world size 2 and 3: range all-gathers with padding for
every dtype the setup exchanges, and the max / min / sum reductions of the
emin statistics and status slots. The row-block kernels themselves are
checked on the B200 (tests/test_gpu_sharding.py)."""

import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_08284_b200.sharding import Sharding

DTYPES = (torch.int64, torch.int32, torch.float64, torch.uint8)


def _expected(n, world, dtype):
    g = torch.Generator().manual_seed(n)
    full = (torch.rand(n, generator=g, dtype=torch.float64) * 250).to(dtype)
    return full


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = Sharding.from_group()
    res = {}
    for n in (0, 1, 7, 1000):
        for dt in DTYPES:
            full = _expected(n, world, dt)
            # uneven value ranges (a CSR's rows differ in length)
            offs = sorted(set([0, n] + [(n * (r * r + 1)) // (world * world + 1)
                                        for r in range(1, world)]))
            while len(offs) < world + 1:
                offs.insert(1, offs[0])
            buf = torch.zeros(n, dtype=dt)
            a, b = offs[rank], offs[rank + 1]
            buf[a:b] = full[a:b]
            sh.gather_ranges(buf, offs)
            res[(n, str(dt))] = bool(torch.equal(buf, full))
    t = torch.tensor([float(rank), -float(rank)], dtype=torch.float64)
    sh.max_(t)
    m = torch.tensor([10 + rank], dtype=torch.int64)
    sh.min_(m)
    s = torch.ones(3, dtype=torch.int64) * (rank + 1)
    sh.sum_(s)
    res["max"] = t.tolist()
    res["min"] = int(m.item())
    res["sum"] = s.tolist()
    res["bounds"] = sh.bounds(10)
    objs = [None] * world
    dist.all_gather_object(objs, res)
    if rank == 0:
        with open(out_path, "wb") as f:
            pickle.dump(objs, f)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_gather_ranges_and_reductions_gloo(world):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.pkl")
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        with open(out, "rb") as f:
            objs = pickle.load(f)
    for r, res in enumerate(objs):
        for k, v in res.items():
            if isinstance(k, tuple):
                assert v, (r, k)
        assert res["max"] == [world - 1.0, 0.0]
        assert res["min"] == 10
        assert res["sum"] == [world * (world + 1) // 2] * 3
        assert res["bounds"] == [(10 * q) // world for q in range(world + 1)]


def test_emulated_and_single_rank_blocks():
    sh = Sharding.emulated(3)
    assert [b for b in sh.blocks(10)] == [(0, 0, 3), (1, 3, 6), (2, 6, 10)]
    assert not sh.collective
    one = Sharding()
    assert list(one.blocks(5)) == [(0, 0, 5)] and not one.active
