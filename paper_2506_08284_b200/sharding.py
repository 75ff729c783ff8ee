"""Row-block sharded setup: the setup's row-parallel work is
split over the ranks of a process group, every rank ending with the same
(replicated) hierarchy.

The setup's heavy phases are independent per output row:

* the emin constraint pass and sweeps, one warp per fine edge
  (emin_setup.py:256-336, edge_prolongator.py:154-181);
* every sparse product of the hierarchy -- A D / S D for the null-space
  check, D^T (A D), the Galerkin pairs A P / S P and R (A P) / R (S P), the
  nodal P^T (A P) (multigrid.py:103,111,150-152) -- whose rows are
  independent (Gustavson row-wise SpGEMM).

Each such phase runs in the GLOBAL index space: rank r computes the rows of
its contiguous block [lo_r, hi_r) (counts first, then values at their global
CSR positions), and the blocks are exchanged with one all-gather per array
(NCCL over NVLink; the rows' value ranges are contiguous in CSR, so a block
is a single range). Because every kernel's per-row arithmetic is unchanged,
the sharded hierarchy is BITWISE identical to the single-GPU one
(tests/test_gpu_sharding.py checks this with the ranks emulated on one GPU).

The nodal chain (strength, aggregation, P_n, Algorithm 1, the coarse
gradient) stays replicated: its sequential greedy passes and summation
orders are global ("replicas only").

``Sharding(world, rank, group)`` is the real collective layer;
``Sharding.emulated(world)`` runs every rank's block in one process (the
single-GPU test of the row-range logic: no collectives needed, since all
blocks land in the same buffers).
"""

import numpy as np
import torch
import torch.distributed as dist


class Sharding:
    def __init__(self, world=1, rank=0, group=None, emulate=False):
        self.world = int(world)
        self.rank = int(rank)
        self.group = group
        self.emulate = bool(emulate)

    @staticmethod
    def from_group(group=None):
        return Sharding(dist.get_world_size(group), dist.get_rank(group), group)

    @staticmethod
    def emulated(world):
        return Sharding(world, 0, None, emulate=True)

    @property
    def active(self):
        return self.world > 1

    @property
    def collective(self):
        return self.world > 1 and not self.emulate

    def ranks(self):
        """The ranks whose row blocks this process computes."""
        return range(self.world) if self.emulate else (self.rank,)

    def bounds(self, n):
        """Row offsets [world + 1] of the balanced contiguous partition of n."""
        return [(n * r) // self.world for r in range(self.world + 1)]

    def blocks(self, n):
        b = self.bounds(n)
        return [(r, b[r], b[r + 1]) for r in self.ranks()]

    # ---- collectives (no-ops when emulated or world == 1)

    def gather_ranges(self, buf, offsets):
        """buf: global 1-D buffer; rank r owns buf[offsets[r]:offsets[r+1]].
        After the call every rank holds every range."""
        if not self.collective:
            return buf
        offsets = [int(o) for o in offsets]
        sizes = [offsets[r + 1] - offsets[r] for r in range(self.world)]
        m = max(sizes)
        if m == 0:
            return buf
        send = torch.zeros(m, dtype=buf.dtype, device=buf.device)
        a, b = offsets[self.rank], offsets[self.rank + 1]
        send[:b - a].copy_(buf[a:b])
        recv = torch.empty(m * self.world, dtype=buf.dtype, device=buf.device)
        dist.all_gather_into_tensor(recv, send, group=self.group)
        for r in range(self.world):
            if r != self.rank and sizes[r]:
                buf[offsets[r]:offsets[r + 1]].copy_(recv[r * m:r * m + sizes[r]])
        return buf

    def _reduce(self, t, op):
        if self.collective:
            dist.all_reduce(t, op=op, group=self.group)
        return t

    def max_(self, t):
        return self._reduce(t, dist.ReduceOp.MAX)

    def min_(self, t):
        return self._reduce(t, dist.ReduceOp.MIN)

    def sum_(self, t):
        return self._reduce(t, dist.ReduceOp.SUM)


NONE = Sharding()


def host_offsets(rowptr, bounds):
    """rowptr values at the partition bounds (one small device->host copy)."""
    idx = torch.tensor(bounds, dtype=torch.int64, device=rowptr.device)
    return np.asarray(rowptr[idx].cpu().numpy(), dtype=np.int64)
