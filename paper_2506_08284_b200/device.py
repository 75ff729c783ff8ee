"""Device CSR container and thin wrappers over the libsphcurl C ABI.

B200 replacement of the reference's scipy-CSR substrate (sparse_ops.py):
int64 row pointers, int32 columns, fp64 values, all resident in HBM as torch
tensors (torch is the allocator / stream plumbing; every numeric operation is
a libsphcurl kernel).
"""

import functools
import os
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib

INT64_MAX = np.iinfo(np.int64).max
SLOTS = 32
ST = dict(ZERO_DIAG=0, NONPOS_DIAG=1, NODAL_ZERO_DIAG=2, ZERO_ROWSUM=3,
          MALFORMED_GRAD=4, EMPTY_I=5, REDUCIBLE=6, RANK_LOW=7, EMIN_CAPACITY=8,
          EMPTY_J=9, SPGEMM_CAPACITY=10, SORT_CAPACITY=11, TRSV_STALL=12,
          PC_EMPTY_COLUMN=13, PC_EMPTY_ROW=14, PC_NO_DONOR=15, AGG_CAPACITY=16,
          PC_NO_FIXPOINT=17)


_DEVICE = None


def device():
    global _DEVICE
    if _DEVICE is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2506_08284_b200 needs a CUDA device (B200); "
                               "there is no CPU path")
        _DEVICE = torch.device("cuda", torch.cuda.current_device())
    return _DEVICE


def call(name, *args):
    return _lib.call(name, *args)


class Status:
    """Device error slots: slot k holds the lowest row failing check k.

    Slots come out of pooled blocks (one fill launch per 64 statuses). A
    check is either read now (``rows()``) or deferred (``defer(handler)``):
    deferred checks ride along with the next host readback of any kind
    (``readback``, ``scan``), run in program order before that readback's
    own values are used, so an error surfaces with the reference's message
    and order at the cost of no extra synchronisation."""

    _block = None
    _next = 0

    def __init__(self):
        blk = Status._block
        if blk is None or Status._next >= blk.shape[0] or blk.device != device():
            blk = Status._block = torch.full((64, SLOTS), INT64_MAX, dtype=torch.int64,
                                             device=device())
            Status._next = 0
        self.t = blk[Status._next]
        Status._next += 1

    def rows(self):
        return _decode(readback(self.t)[0])

    def defer(self, handler):
        _PENDING.append((self, handler))


def _decode(h):
    return {k: int(h[v]) for k, v in ST.items() if h[v] != INT64_MAX}


_PENDING = []


_PIN = [None]


def _staging(nbytes):
    buf = _PIN[0]
    if buf is None or buf.numel() < nbytes:
        buf = _PIN[0] = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, pin_memory=True)
    return buf


_RB_LOCK = __import__("threading").RLock()


def readback(*tensors):
    """Small device tensors -> numpy arrays after ONE stream synchronisation,
    first running every deferred status check (Status.defer) in order. Each
    part is DMA'd straight into a page-locked staging buffer (no gather
    kernel, no pageable bounce through the driver's staging copy). The
    staging buffer is shared: serialised across host threads."""
    with _RB_LOCK:
        return _readback(tensors)


def _readback(tensors):
    pend = list(_PENDING)
    _PENDING.clear()
    parts = [st.t for st, _ in pend] + [t.reshape(-1) for t in tensors]
    if not parts:
        return []
    parts = [p if p.is_contiguous() else p.contiguous() for p in parts]
    sizes = [p.numel() * p.element_size() for p in parts]
    offs, o = [], 0
    for nb in sizes:
        offs.append(o)
        o += (nb + 15) & ~15
    buf = _staging(o)
    base = buf.data_ptr()
    rng = [(p.data_ptr(), nb, off) for p, nb, off in zip(parts, sizes, offs) if nb]
    if len(rng) <= 16 and all(nb % 4 == 0 for _, nb, _ in rng):
        # one kernel writes every range into the mapped staging buffer
        call("sphc_readback_gather", len(rng), np.array(rng, dtype=np.int64).reshape(-1),
             base)
    else:
        for src, nb, off in rng:
            call("sphc_copy_d2h", base + off, src, nb)
    call("sphc_stream_sync")
    raw = buf.numpy()
    hs = [raw[off:off + nb].view(_NP[p.dtype]).copy() for p, nb, off in zip(parts, sizes, offs)]
    for (st, handler), h in zip(pend, hs):
        handler(_decode(h))
    return hs[len(pend):]


def flush_checks():
    """Run the deferred status checks now (end of a public entry point)."""
    if _PENDING:
        readback()


_DEPTH = [0]


def checked(fn):
    """Public entry points: the outermost one runs every check deferred
    inside it before returning. If it exits by an exception, the deferred
    checks still run first, so an earlier device-detected error wins, as it
    would in the reference's sequential code."""
    @functools.wraps(fn)
    def wrap(*args, **kwargs):
        _DEPTH[0] += 1
        try:
            out = fn(*args, **kwargs)
        except BaseException:
            _DEPTH[0] -= 1
            if _DEPTH[0] == 0:
                try:
                    flush_checks()
                finally:
                    _PENDING.clear()
            raise
        _DEPTH[0] -= 1
        if _DEPTH[0] == 0:
            flush_checks()
        return out
    return wrap


_NP = {torch.int64: np.int64, torch.int32: np.int32, torch.float64: np.float64,
       torch.uint8: np.uint8, torch.bool: np.bool_}


_PINNED = {}
_INFLIGHT = []        # (host array, event): direct DMAs whose source must stay alive


def _retire_inflight():
    while _INFLIGHT and _INFLIGHT[0][1].query():
        _INFLIGHT.pop(0)


_COPY_POOL = []


def parallel_copyto(dst, src, nthreads=8):
    """np.copyto(dst, src, casting="unsafe") split over a few threads for
    large arrays (numpy releases the GIL; a fresh destination's page faults
    spread over the threads too)."""
    n = dst.size
    if n * dst.itemsize < (8 << 20):
        np.copyto(dst, src, casting="unsafe")
        return
    if not _COPY_POOL:
        from concurrent.futures import ThreadPoolExecutor
        _COPY_POOL.append(ThreadPoolExecutor(nthreads))
    step = -(-n // nthreads)
    list(_COPY_POOL[0].map(lambda k: np.copyto(dst[k:k + step], src[k:k + step],
                                               casting="unsafe"), range(0, n, step)))


def to_host(t):
    """Device tensor -> new numpy array through a pinned staging buffer (one
    DMA at pinned-memory bandwidth, then a threaded copy out); waits for the
    current stream."""
    t = t.contiguous()
    nbytes = t.numel() * t.element_size()
    if nbytes < (1 << 20):
        return t.cpu().numpy()
    buf = _PINNED.get("d2h")
    if buf is None or buf.numel() < nbytes:
        buf = _PINNED["d2h"] = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    buf[:nbytes].copy_(t.view(-1).view(torch.uint8), non_blocking=True)
    call("sphc_stream_sync")
    out = np.empty(t.numel(), dtype=_NP[t.dtype])
    parallel_copyto(out, buf[:nbytes].numpy().view(_NP[t.dtype]))
    return out.reshape(tuple(t.shape))


def upload(a, dtype, dev=None, owned=True):
    """Host array -> new device tensor through a reused pinned staging buffer
    (one cast on the host, one DMA at pinned-memory bandwidth).

    With page-locking enabled (SPHC_PIN=1, opt-in) an array the CALLER owns
    (``owned``; never a temporary made here) that already has the device
    dtype is DMA'd straight from its own memory; it is kept alive until that
    copy's event completes, so neither the caller dropping it nor its
    registration being released can race the copy."""
    dev = dev or device()
    a0 = a
    a = np.asarray(a)
    n = a.size
    t = torch.empty(n, dtype=torch.from_numpy(np.zeros(0, dtype=dtype)).dtype, device=dev)
    if n == 0:
        return t
    nbytes = n * np.dtype(dtype).itemsize
    _retire_inflight()
    if owned and a is a0 and a.dtype == np.dtype(dtype) and pinned_in_place(a):
        call("sphc_copy_h2d", t, a, nbytes)     # stream ordered, no staging / sync
        ev = torch.cuda.Event()
        ev.record()
        _INFLIGHT.append((a, ev))
        return t
    # the staging buffer is reused: the next upload waits for this copy's
    # event (normally long done) instead of this one syncing the stream
    ev = _PINNED.get("event")
    if ev is not None:
        ev.synchronize()
    buf = _PINNED.get("buf")
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 24), dtype=torch.uint8, pin_memory=True)
        _PINNED["buf"] = buf
    host = buf[:nbytes].numpy().view(dtype)
    parallel_copyto(host, a.reshape(-1))
    t.view(torch.uint8).copy_(buf[:nbytes], non_blocking=True)
    if ev is None:
        ev = _PINNED["event"] = torch.cuda.Event()
    ev.record()
    return t


@dataclass
class DeviceCSR:
    rowptr: torch.Tensor          # int64 [n_rows + 1]
    col: torch.Tensor             # int32 [nnz]
    val: torch.Tensor             # float64 [nnz] (None for a pure pattern)
    shape: tuple

    @property
    def nnz(self):
        return int(self.col.numel())

    @property
    def n_rows(self):
        return self.shape[0]

    @staticmethod
    def from_scipy(A, dev=None):
        dev = dev or device()
        A0 = A = host_csr(A)
        if not A.has_canonical_format:
            A = A.copy()
            A.sum_duplicates()
            A.sort_indices()
        owned = A is A0          # a canonicalised temporary is always staged
        return DeviceCSR(rowptr=upload(A.indptr, np.int64, dev, owned),
                         col=upload(A.indices, np.int32, dev, owned),
                         val=upload(A.data, np.float64, dev, owned),
                         shape=tuple(int(s) for s in A.shape))

    def to_scipy(self):
        val = self.val.cpu().numpy() if self.val is not None else np.ones(self.nnz)
        return sp.csr_matrix((val, self.col.cpu().numpy(), self.rowptr.cpu().numpy()),
                             shape=self.shape)

    def lanes(self):
        """Lanes per row for the row-grouped SpMV (mean row length)."""
        m = self.nnz / max(self.shape[0], 1)
        for L, lim in ((2, 3), (4, 6), (8, 14), (16, 40)):
            if m <= lim:
                return L
        return 32


def host_csr(A):
    """A scipy CSR as is (so scipy's cached canonical-format flag survives
    repeated calls with the same matrix object); anything else converted."""
    if sp.issparse(A) and A.format == "csr":
        return A
    return sp.csr_matrix(A)


def own_csr(A):
    """A solver-owned DeviceCSR for a caller's matrix: a caller DeviceCSR is
    re-wrapped (same tensors, new object), so caches and pattern sharing the
    solver attaches to its own matrices never touch the caller's object."""
    if isinstance(A, DeviceCSR):
        return DeviceCSR(A.rowptr, A.col, A.val, A.shape)
    return as_device_csr(A)


def as_device_csr(A):
    if isinstance(A, DeviceCSR):
        return A
    if isinstance(A, PendingCSR):
        return A.get()
    return DeviceCSR.from_scipy(A)


_STAGE = {}
import threading as _threading  # noqa: E402
_STAGE_LOCK = _threading.Lock()
_REG = {}      # (address, bytes) -> weakref of the page-locked host array


PIN_CALLER_MEMORY = os.environ.get("SPHC_PIN", "0") == "1"


def pinned_in_place(a):
    """True if host array ``a`` is page-locked for direct DMA. Opt-in
    (SPHC_PIN=1): page-locking is a process-wide side effect on the caller's
    memory, so by default every upload is staged. When enabled, each array
    object is registered once (sphc_host_register) and released when it is
    garbage collected (its in-flight copies keep it alive until they finish,
    ``upload``); small, strided or overlapping arrays return False (the
    caller stages them instead)."""
    if not PIN_CALLER_MEMORY or a.nbytes < (1 << 20) or not a.flags.c_contiguous:
        return False
    import weakref
    key = (a.ctypes.data, a.nbytes)
    ref = _REG.get(key)
    if ref is not None:
        if ref() is a:
            return True
        return False          # an older array at this address: let it be released first
    try:
        call("sphc_host_register", a, a.nbytes)
    except RuntimeError:
        return False

    def release(_, ptr=key[0], key=key):
        _REG.pop(key, None)
        try:
            _lib.lib().sphc_host_unregister(ctypes_void(ptr))
        except Exception:     # noqa: BLE001 - interpreter shutdown
            pass
    _REG[key] = weakref.ref(a, release)
    return True


def ctypes_void(p):
    import ctypes
    return ctypes.c_void_p(p)


class AsyncUpload:
    """Host -> device upload of scipy CSR matrices in the background: a
    helper thread casts / copies the arrays chunk by chunk into a ring of
    pinned staging slots with a small pool of threads (numpy releases the
    GIL) and queues each chunk's DMA on a side stream; ``get(k)`` makes the
    caller's stream wait on matrix k's copy event (no host sync). The caller
    keeps launching device work meanwhile (build_hierarchy runs the nodal
    chain while S and A_e arrive)."""

    def __init__(self, mats, nthreads=8):
        dev = device()
        self.mats, owned = [], []
        for A in mats:
            A0 = A = host_csr(A)
            if not A.has_canonical_format:
                A = A.copy()
                A.sum_duplicates()
                A.sort_indices()
            self.mats.append(A)
            owned += [A is A0] * 3
        self.specs = []
        for A in self.mats:
            self.specs += [(A.indptr, np.int64), (A.indices, np.int32), (A.data, np.float64)]
        self.owned = owned
        tdt = {np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}
        self.dst = [torch.empty(a.size, dtype=tdt[d], device=dev) for a, d in self.specs]
        self.offs, o = [], 0
        for a, d in self.specs:
            self.offs.append(o)
            o += (a.size * np.dtype(d).itemsize + 255) // 256 * 256
        self.nbytes = o
        self.nthreads = nthreads
        self.dev = dev
        self.stream = torch.cuda.Stream(device=dev)
        import threading
        nm = len(self.mats)
        self.events = [torch.cuda.Event() for _ in range(nm)]
        self.ready = [threading.Event() for _ in range(nm)]
        self.event = self.events[-1] if nm else torch.cuda.Event()
        self.err = None
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()
        self.csr = [None] * nm

    CHUNK = 1 << 25          # staging granularity (bytes)
    SLOTS = 16               # ring of pinned chunks (512 MB, whatever the inputs' size)

    def _run(self):
        # one upload at a time owns the staging ring
        with _STAGE_LOCK:
            self._run_locked()

    def _run_locked(self):
        try:
            torch.cuda.set_device(self.dev)
            ring = _STAGE.get("ring")
            if ring is None:
                ring = _STAGE["ring"] = torch.empty(self.SLOTS * self.CHUNK, dtype=torch.uint8,
                                                    pin_memory=True)
                _STAGE["slot_events"] = [None] * self.SLOTS
            slot_ev = _STAGE["slot_events"]
            hv = ring.numpy()
            # arrays already in the device dtype DMA straight from the
            # caller's page-locked memory (opt-in); the rest are cast into
            # the ring chunk by chunk by a small pool of threads, and each
            # chunk's DMA is queued as soon as its host copy is done, so the
            # copies of later chunks (and of A_e) overlap the transfers of
            # earlier ones (and of S). A slot is reused once its DMA is done.
            direct = [own and a.dtype == np.dtype(d) and pinned_in_place(a)
                      for (a, d), own in zip(self.specs, self.owned)]
            chunks = []              # (array index, first element, elements, last of array)
            for idx, ((a, d), dr) in enumerate(zip(self.specs, direct)):
                if dr or not a.size:
                    chunks.append((idx, 0, 0, True))
                    continue
                per = max(1, self.CHUNK // np.dtype(d).itemsize)
                for k in range(0, a.size, per):
                    n = min(per, a.size - k)
                    chunks.append((idx, k, n, k + n == a.size))
            from concurrent.futures import ThreadPoolExecutor
            # small systems: one copy thread (a pool costs more than it saves)
            nthreads = self.nthreads if self.nbytes >= (64 << 20) else 1
            depth = min(self.SLOTS, 2 * nthreads)

            def stage(c, slot):
                idx, k, n, _ = chunks[c]
                a, d = self.specs[idx]
                dstv = hv[slot * self.CHUNK:slot * self.CHUNK + n * np.dtype(d).itemsize].view(d)
                np.copyto(dstv, a[k:k + n], casting="unsafe")

            with ThreadPoolExecutor(nthreads) as ex, torch.cuda.stream(self.stream):
                futs = {}
                submitted = issued = 0
                nslot = 0                      # staged chunks so far (slot = nslot % SLOTS)
                slot_of = {}
                while issued < len(chunks):
                    while submitted < len(chunks) and submitted - issued < depth:
                        if chunks[submitted][2]:
                            slot = nslot % self.SLOTS
                            nslot += 1
                            if slot_ev[slot] is not None:
                                slot_ev[slot].synchronize()      # its last DMA is done
                            slot_of[submitted] = slot
                            futs[submitted] = ex.submit(stage, submitted, slot)
                        submitted += 1
                    idx, k, n, last = chunks[issued]
                    a, d = self.specs[idx]
                    if n:
                        futs.pop(issued).result()
                        slot = slot_of.pop(issued)
                        isz = np.dtype(d).itemsize
                        self.dst[idx].view(torch.uint8)[k * isz:(k + n) * isz].copy_(
                            ring[slot * self.CHUNK:slot * self.CHUNK + n * isz],
                            non_blocking=True)
                        ev = slot_ev[slot]
                        if ev is None:
                            ev = slot_ev[slot] = torch.cuda.Event()
                        ev.record(self.stream)
                    elif a.size:               # direct (page-locked caller array)
                        call("sphc_copy_h2d", self.dst[idx], a, a.nbytes)
                    if last and idx % 3 == 2:  # a matrix's last array is queued
                        m = idx // 3
                        self.events[m].record(self.stream)
                        self.ready[m].set()
                    issued += 1
            # direct sources stay referenced (self.mats) until get() has
            # made the compute stream wait on the copies; keep them alive
            # past that too, until the copies are done
            _INFLIGHT.extend((a, self.event) for (a, _), dr in zip(self.specs, direct) if dr)
        except BaseException as e:   # noqa: BLE001 - re-raised by get()
            self.err = e
        finally:
            for r in self.ready:
                r.set()

    def get(self, k):
        if self.csr[k] is None:
            self.ready[k].wait()
            if self.err is not None:
                self.thread.join()
                raise self.err
            torch.cuda.current_stream().wait_event(self.events[k])
            A = self.mats[k]
            self.csr[k] = DeviceCSR(self.dst[3 * k], self.dst[3 * k + 1], self.dst[3 * k + 2],
                                    tuple(int(x) for x in A.shape))
        return self.csr[k]


class PendingCSR:
    """A matrix of an AsyncUpload; its shape is known before the data lands."""

    def __init__(self, up, k):
        self.up, self.k = up, k
        self.shape = tuple(int(x) for x in up.mats[k].shape)

    def get(self):
        return self.up.get(self.k)


def empty_f64(n):
    return torch.empty(int(n), dtype=torch.float64, device=device())


def zeros_f64(n):
    return torch.zeros(int(n), dtype=torch.float64, device=device())


def zeros_i64(n):
    return torch.zeros(int(n), dtype=torch.int64, device=device())


def scan(counts, with_max=False):
    """Exclusive scan -> (rowptr [n+1], total) (one host sync for the total,
    shared with any deferred status checks); with_max: (rowptr, total,
    max count) from the same readback."""
    n = counts.numel()
    rp = torch.empty(n + 1, dtype=torch.int64, device=counts.device)
    call("sphc_scan_i64", n, counts, rp)
    if not with_max:
        return rp, int(readback(rp[n:n + 1])[0][0])
    mx = torch.amax(counts).reshape(1) if n else torch.zeros(1, dtype=torch.int64,
                                                             device=counts.device)
    tot, m = readback(rp[n:n + 1], mx)
    return rp, int(tot[0]), int(m[0])


def scan_many(*counts):
    """Several exclusive scans, one host sync for all totals."""
    rps = []
    for c in counts:
        n = c.numel()
        rp = torch.empty(n + 1, dtype=torch.int64, device=c.device)
        call("sphc_scan_i64", n, c, rp)
        rps.append(rp)
    tot = readback(torch.stack([rp[-1] for rp in rps]))[0]
    return [(rp, int(t)) for rp, t in zip(rps, tot)]


def dot(x, y, out=None):
    out = out if out is not None else empty_f64(1)
    call("sphc_dot", x.numel(), x, y, out)
    return out


def vsum(x, out=None):
    out = out if out is not None else empty_f64(1)
    call("sphc_sum", x.numel(), x, out)
    return out


def maxabs(x, out=None):
    out = out if out is not None else empty_f64(1)
    call("sphc_maxabs", x.numel(), x, out)
    return out


def diagonal(A, status=None):
    d = empty_f64(A.shape[0])
    call("sphc_csr_diag", A.shape[0], A.rowptr, A.col, A.val, d,
         status.t if status is not None else None)
    return d


def reciprocal(x, zero_sub=None):
    y = empty_f64(x.numel())
    call("sphc_reciprocal", x.numel(), x, zero_sub, y)
    return y


@checked
def transpose(A, status=None):
    st = status or Status()
    nr, nc = A.shape
    trp = torch.empty(nc + 1, dtype=torch.int64, device=A.rowptr.device)
    tci = torch.empty(A.nnz, dtype=torch.int32, device=A.rowptr.device)
    tv = empty_f64(A.nnz) if A.val is not None else None
    call("sphc_csr_transpose", nr, nc, A.nnz, A.rowptr, A.col, A.val, trp, tci, tv, st.t)
    if status is None:
        st.defer(capacity_check)
    return DeviceCSR(trp, tci, tv, (nc, nr))


def _raise_capacity(st):
    capacity_check(st.rows())


def capacity_check(rows):
    for k in ("SORT_CAPACITY", "SPGEMM_CAPACITY", "EMIN_CAPACITY"):
        if k in rows:
            raise RuntimeError(f"device kernel capacity exceeded ({k}) at row {rows[k]}")


@checked
def drop_zeros(A):
    """compress(A, 0.0): remove stored exact zeros (sparse_ops.py:107-113)."""
    return drop_zeros_many(A)[0]


def drop_zeros_many(*mats):
    """drop_zeros of several matrices with one host sync for all counts."""
    cnts = []
    for A in mats:
        cnt = torch.empty(A.shape[0], dtype=torch.int64, device=A.rowptr.device)
        call("sphc_csr_count_nonzero", A.shape[0], A.rowptr, A.val, cnt)
        cnts.append(cnt)
    return [_compact(A, rp, nnz) for A, (rp, nnz) in zip(mats, scan_many(*cnts))]


@checked
def csr_add(A, B, alpha=1.0, beta=1.0):
    """alpha A + beta B on the union pattern (scipy's csr_binop_csr)."""
    if A.shape != B.shape:
        raise ValueError(f"shape mismatch {A.shape} vs {B.shape}")
    n = A.shape[0]
    cnt = torch.empty(n, dtype=torch.int64, device=A.rowptr.device)
    call("sphc_csr_add_count", n, A.rowptr, A.col, B.rowptr, B.col, cnt)
    rp, nnz = scan(cnt)
    ci = torch.empty(nnz, dtype=torch.int32, device=A.rowptr.device)
    v = empty_f64(nnz)
    call("sphc_csr_add_fill", n, A.rowptr, A.col, A.val, B.rowptr, B.col, B.val, float(alpha),
         float(beta), rp, ci, v)
    return DeviceCSR(rp, ci, v, A.shape)


def _compact(A, rp, nnz):
    n = A.shape[0]
    if nnz == A.nnz:
        return A
    ci = torch.empty(nnz, dtype=torch.int32, device=A.rowptr.device)
    v = empty_f64(nnz)
    call("sphc_csr_compact", n, A.rowptr, A.col, A.val, rp, ci, v)
    return DeviceCSR(rp, ci, v, A.shape)


LONG_ROW = int(os.environ.get("SPHC_LONG_ROW", "64"))


def _long_rows(A):
    """Average A row length at which the CTA-per-row SpGEMM takes over (the
    R (A P) Galerkin products; no host sync: nnz and shape are known)."""
    return A.shape[0] > 0 and A.nnz >= LONG_ROW * A.shape[0]


THIN_PRODUCTS = float(os.environ.get("SPHC_THIN_PRODUCTS", "160"))


def _thin_rows(A, B):
    """Products with few multiplications per output row (A_e D, S_e D,
    D^T (A D): mean row products nnz(A)/rows(A) x nnz(B)/rows(B) below
    THIN_PRODUCTS) go to the thread-per-row kernels (sphc_spgemm_*_thin);
    no host sync: sizes are known."""
    if A.shape[0] == 0 or B.shape[0] == 0 or THIN_PRODUCTS <= 0:
        return False
    return (A.nnz / A.shape[0]) * (B.nnz / B.shape[0]) <= THIN_PRODUCTS


_ANY_OVER = {}


def _any_over(dev):
    """One-int device scratch of the thin count pass, per (device, stream):
    virtual-rank threads drive their own streams."""
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    t = _ANY_OVER.get(key)
    if t is None:
        t = _ANY_OVER[key] = torch.zeros(1, dtype=torch.int32, device=dev)
    return t


def _rows(A, lo):
    """Row-pointer view starting at row lo (absolute positions into A's
    column / value arrays, so a kernel launched on it computes rows lo..)."""
    return A.rowptr[lo:]


class _Overflow:
    """Deferred status handler of the SpGEMM count passes: rows beyond the
    on-chip capacity (count -1) are noted for the global-memory path;
    every other capacity status still raises."""

    def __init__(self):
        self.hit = False

    def __call__(self, rows):
        if "SPGEMM_CAPACITY" in rows:
            self.hit = True
        capacity_check({k: v for k, v in rows.items() if k != "SPGEMM_CAPACITY"})


def _global_rows_count(A, B, cnt):
    """Rows the count kernels marked -1: their true counts by the
    global-memory kernel (one CTA per row, hash tables in global scratch).
    Rare (imported matrices with very long rows); a few host syncs."""
    dev = A.rowptr.device
    rows = torch.nonzero(cnt < 0).flatten()
    nr = rows.numel()
    STATS["spgemm_global_rows"] += nr
    prods = torch.empty(nr, dtype=torch.int64, device=dev)
    call("sphc_spgemm_global_products", nr, rows, A.rowptr, A.col, B.rowptr, prods)
    sz = torch.clamp(2 * prods, min=64)
    sz = torch.pow(2, torch.ceil(torch.log2(sz.to(torch.float64)))).to(torch.int64)
    hoff = torch.zeros(nr + 1, dtype=torch.int64, device=dev)
    hoff[1:] = torch.cumsum(sz, 0)
    tot = int(readback(hoff[nr:nr + 1])[0][0])
    hkeys = torch.empty(tot, dtype=torch.int32, device=dev)
    hslot = torch.empty(tot, dtype=torch.int32, device=dev)
    st = Status()
    call("sphc_spgemm_global", nr, rows, hoff, hkeys, hslot, A.rowptr, A.col, None, None,
         B.rowptr, B.col, None, None, cnt, None, None, None, None, st.t)
    return (rows, hoff, hkeys, hslot)


def _global_rows_fill(g, A, B, rp, ci, v, A2=None, B2=None, v2=None):
    rows, hoff, hkeys, hslot = g
    st = Status()
    call("sphc_spgemm_global", rows.numel(), rows, hoff, hkeys, hslot, A.rowptr, A.col, A.val,
         None if A2 is None else A2.val, B.rowptr, B.col, B.val,
         None if B2 is None else B2.val, None, rp, ci, v, v2, st.t)
    st.defer(capacity_check)


# rows of more output columns than this also take the global-memory path
# (0 = only the rows the on-chip kernels cannot hold; tests lower it to
# drive whole hierarchies through the global path)
GLOBAL_ROWS_ABOVE = int(os.environ.get("SPHC_SPGEMM_GLOBAL_ABOVE", "0"))
STATS = {"spgemm_global_rows": 0}


def _count_with_overflow(A, B, cnt, st, shard, n):
    """scan of the count pass; rows beyond the on-chip capacity go to the
    global-memory path (their counts fixed, then a second scan)."""
    ov = _Overflow()
    st.defer(ov)
    if GLOBAL_ROWS_ABOVE > 0:
        cnt.masked_fill_(cnt > GLOBAL_ROWS_ABOVE, -1)
        ov.hit = True
    rp, nnz, mcols = scan(cnt, with_max=True)
    g = None
    if ov.hit:
        g = _global_rows_count(A, B, cnt)
        rp, nnz, mcols = scan(cnt, with_max=True)
    return rp, nnz, mcols, g


@checked
def spgemm(A, B, drop=True, ordered=False, shard=None):
    """C = A B; exact zeros dropped like scipy's product (drop=True).
    ordered=True reproduces scipy csr_matmat's accumulation bit for bit.
    shard: rows computed by row blocks over a ``sharding.Sharding``.
    Rows beyond the on-chip kernels' capacity (> 256 distinct columns) take
    the global-memory path (sphc_spgemm_global, same ordered sums)."""
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"spgemm dimension mismatch: {A.shape} @ {B.shape}")
    n = A.shape[0]
    st = Status()
    cnt = torch.empty(n, dtype=torch.int64, device=A.rowptr.device)
    blocks = shard.blocks(n) if shard is not None else [(0, 0, n)]
    long_rows = _long_rows(A) and not ordered
    thin = not long_rows and _thin_rows(A, B)
    for _, lo, hi in blocks:
        if thin:
            call("sphc_spgemm_count_thin", hi - lo, _rows(A, lo), A.col, B.rowptr, B.col,
                 cnt[lo:], _any_over(cnt.device), st.t)
        else:
            call("sphc_spgemm_count_long" if long_rows else "sphc_spgemm_count", hi - lo,
                 _rows(A, lo), A.col, B.rowptr, B.col, cnt[lo:], st.t)
    if shard is not None:
        shard.gather_ranges(cnt, shard.bounds(n))
        shard.min_(st.t)
    rp, nnz, mcols, g = _count_with_overflow(A, B, cnt, st, shard, n)
    ci = torch.empty(nnz, dtype=torch.int32, device=A.rowptr.device)
    v = empty_f64(nnz)
    for _, lo, hi in blocks:
        if thin:
            call("sphc_spgemm_fill_thin", hi - lo, _rows(A, lo), A.col, A.val, None, B.rowptr,
                 B.col, B.val, None, rp[lo:], ci, v, None, int(ordered), mcols, st.t)
        elif long_rows:
            call("sphc_spgemm_fill_long", hi - lo, _rows(A, lo), A.col, A.val, None, B.rowptr,
                 B.col, B.val, None, rp[lo:], ci, v, None)
        else:
            call("sphc_spgemm_fill", hi - lo, _rows(A, lo), A.col, A.val, B.rowptr, B.col,
                 B.val, rp[lo:], ci, v, int(ordered), mcols, st.t)
    if g is not None:
        _global_rows_fill(g, A, B, rp, ci, v)
    if shard is not None and shard.collective:
        from .sharding import host_offsets
        off = host_offsets(rp, shard.bounds(n))
        shard.gather_ranges(ci, off)
        shard.gather_ranges(v, off)
    C = DeviceCSR(rp, ci, v, (A.shape[0], B.shape[1]))
    return drop_zeros(C) if drop else C


def same_pattern(A, B):
    if A.shape != B.shape or A.nnz != B.nnz:
        return False
    if A.rowptr is B.rowptr and A.col is B.col:      # shared index arrays: no sync
        return True
    eq = (A.rowptr == B.rowptr).all() & (A.col == B.col).all()
    if not bool(readback(eq)[0][0]):
        return False
    # equal patterns: share one copy of the index arrays, so later checks
    # of the pair (and of their Galerkin products) need no readback
    B.rowptr, B.col = A.rowptr, A.col
    return True


@checked
def spgemm_pair(A1, A2, B1, B2, drop=True, shard=None):
    """(A1 B1, A2 B2) for A1/A2 and B1/B2 with shared patterns, one pass.
    Stored exact zeros are dropped per product (drop=True)."""
    n = A1.shape[0]
    st = Status()
    cnt = torch.empty(n, dtype=torch.int64, device=A1.rowptr.device)
    blocks = shard.blocks(n) if shard is not None else [(0, 0, n)]
    long_rows = _long_rows(A1)
    thin = not long_rows and _thin_rows(A1, B1)
    for _, lo, hi in blocks:
        if thin:
            call("sphc_spgemm_count_thin", hi - lo, _rows(A1, lo), A1.col, B1.rowptr, B1.col,
                 cnt[lo:], _any_over(cnt.device), st.t)
        else:
            call("sphc_spgemm_count_long" if long_rows else "sphc_spgemm_count", hi - lo,
                 _rows(A1, lo), A1.col, B1.rowptr, B1.col, cnt[lo:], st.t)
    if shard is not None:
        shard.gather_ranges(cnt, shard.bounds(n))
        shard.min_(st.t)
    rp, nnz, mcols, g = _count_with_overflow(A1, B1, cnt, st, shard, n)
    ci = torch.empty(nnz, dtype=torch.int32, device=A1.rowptr.device)
    v1, v2 = empty_f64(nnz), empty_f64(nnz)
    for _, lo, hi in blocks:
        if thin:
            call("sphc_spgemm_fill_thin", hi - lo, _rows(A1, lo), A1.col, A1.val, A2.val,
                 B1.rowptr, B1.col, B1.val, B2.val, rp[lo:], ci, v1, v2, 0, mcols, st.t)
        elif long_rows:
            call("sphc_spgemm_fill_long", hi - lo, _rows(A1, lo), A1.col, A1.val, A2.val,
                 B1.rowptr, B1.col, B1.val, B2.val, rp[lo:], ci, v1, v2)
        else:
            call("sphc_spgemm_fill_pair", hi - lo, _rows(A1, lo), A1.col, A1.val, A2.val,
                 B1.rowptr, B1.col, B1.val, B2.val, rp[lo:], ci, v1, v2, mcols, st.t)
    if g is not None:
        _global_rows_fill(g, A1, B1, rp, ci, v1, A2, B2, v2)
    if shard is not None and shard.collective:
        from .sharding import host_offsets
        off = host_offsets(rp, shard.bounds(n))
        for t in (ci, v1, v2):
            shard.gather_ranges(t, off)
    shape = (A1.shape[0], B1.shape[1])
    C1, C2 = DeviceCSR(rp, ci, v1, shape), DeviceCSR(rp, ci, v2, shape)
    return tuple(drop_zeros_many(C1, C2)) if drop else (C1, C2)


@dataclass
class SellMirror:
    """SELL-32 copy of a square operator for the solve (csrc/sell.cu)."""

    slice_ptr: torch.Tensor   # int64 [n_slices + 1]
    col: torch.Tensor         # int32 [padded entries]
    val: torch.Tensor         # float64 [padded entries]
    n: int
    # streamed operators: 16-bit column differences + first column per row
    # (sphc_sell_fill16), None when not built / not representable
    d16: torch.Tensor = None
    c0: torch.Tensor = None   # int32 [n * nbase]: the rows' 32-bit bases
    nbase: int = 1

    @property
    def padded(self):
        return int(self.val.numel())


def _sell_key(A):
    return (A.rowptr.data_ptr(), A.col.data_ptr(), A.val.data_ptr(), A.val._version)


def sell_mirror(A):
    """A's cached SELL mirror if it still matches A's arrays (an in-place
    update of A.val bumps its version and retires the mirror), else None."""
    m = getattr(A, "_sell", None)
    if m is not None and A._sell_key == _sell_key(A):
        return m
    return None


def sell(A):
    """SELL-32 mirror of A (built once per array version, cached on A; the
    solver builds it on its own wrappers, never on a caller's DeviceCSR)."""
    m = sell_mirror(A)
    if m is not None:
        return m
    n = A.shape[0]
    ns = (n + 31) // 32
    sz = torch.empty(ns, dtype=torch.int64, device=A.rowptr.device)
    call("sphc_sell_sizes", n, A.rowptr, sz)
    sp_, tot = scan(sz)
    ci = torch.empty(tot, dtype=torch.int32, device=A.rowptr.device)
    v = empty_f64(tot)
    call("sphc_sell_fill", n, A.rowptr, A.col, A.val, sp_, ci, v)
    m = SellMirror(sp_, ci, v, n)
    if SELL16 and tot * 12 > SELL16_MIN_BYTES and ns >= 148 * 48:
        # operators streamed from HBM by one warp per slice: delta-coded
        # columns (10 instead of 12 bytes per entry), if they fit 16 bits
        _delta_code(m, A, sp_, tot, 0)
    A._sell, A._sell_key = m, _sell_key(A)
    return m


def _delta_code(m, A, sp_, tot, rect):
    """Attach delta-coded columns to mirror ``m`` if A's rows can be coded:
    with one 32-bit base per row, else with four (escapes for the jumps
    beyond 16 bits: the plane-to-plane jumps of a 256^3 numbering)."""
    n, dev = A.shape[0], A.rowptr.device
    d16 = torch.empty(tot, dtype=torch.int16, device=dev)
    big = torch.empty(1, dtype=torch.int32, device=dev)
    for nbase in (1, 4):
        c0 = torch.empty(n * nbase, dtype=torch.int32, device=dev)
        call("sphc_sell_fill16", n, A.rowptr, A.col, sp_, d16, c0, big, rect, nbase)
        if int(readback(big)[0][0]) == 0:
            m.d16, m.c0, m.nbase = d16, c0, nbase
            return True
    return False


def sell_rect(A):
    """Uncached SELL-32 copy of a rectangular operator (A_e D for the fused
    Hiptmair mid step): padding repeats a valid column of the row."""
    n = A.shape[0]
    ns = (n + 31) // 32
    sz = torch.empty(ns, dtype=torch.int64, device=A.rowptr.device)
    call("sphc_sell_sizes", n, A.rowptr, sz)
    sp_, tot = scan(sz)
    ci = torch.empty(tot, dtype=torch.int32, device=A.rowptr.device)
    v = empty_f64(tot)
    call("sphc_sell_fill_rect", n, A.rowptr, A.col, A.val, sp_, ci, v)
    m = SellMirror(sp_, ci, v, n)
    if SELL16 and tot * 12 > SELL16_MIN_BYTES and ns >= 148 * 48:
        if _delta_code(m, A, sp_, tot, 1):
            m.col = None          # only the delta-coded kernel reads this mirror
    return m


SELL16 = os.environ.get("SPHC_SELL16", "1") != "0"
SELL16_MIN_BYTES = 48 << 20          # the kernels' streaming threshold (csrc/sell.cu)


CTA_ROW_MAX_ROWS = int(os.environ.get("SPHC_CTA_ROW_MAX_ROWS", "4096"))
CTA_ROW_MIN_LEN = 96


def spmv(A, x, y, alpha=1.0, beta=0.0, z=None, lanes=None):
    """y = alpha A x + beta z (on A's SELL mirror when it has a current one)."""
    m = sell_mirror(A)
    if m is not None:
        if m.d16 is not None:
            call("sphc_sell_spmv16", m.n, m.slice_ptr, m.d16, m.c0, m.val, x, alpha, beta, z, y,
                 m.nbase)
        else:
            call("sphc_sell_spmv", m.n, m.slice_ptr, m.col, m.val, x, alpha, beta, z, y,
                 m.padded)
        return y
    if lanes is None:
        lanes = A.lanes()
        if lanes == 32 and A.shape[0] <= CTA_ROW_MAX_ROWS and \
                A.nnz >= CTA_ROW_MIN_LEN * A.shape[0]:
            lanes = 256       # one CTA per row (coarse-level restrictions)
    call("sphc_spmv", A.shape[0], A.rowptr, A.col, A.val, lanes, x, alpha, beta, z, y)
    return y


def to_dense(A):
    out = torch.empty(A.shape, dtype=torch.float64, device=A.rowptr.device)
    call("sphc_csr_to_dense", A.shape[0], A.shape[1], A.rowptr, A.col, A.val, out)
    return out
