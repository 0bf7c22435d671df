"""Device-resident WHFF step executor, single GPU or row-sharded over N GPUs.

One step (pipeline.py:199-205 + thermal.py:98-117, for a whole field):
    u_k      = source term of the light step            (thermal.py:81-88)
    T_{k+1}  = fp32(A64 T_k + B u_k)                     (thermal.py:98-109)
    S_{k+1}  = fp32(P64 T_{k+1})                         (thermal.py:112-117)
    D_d      = C_d,field S_{k+1}, d in {x, y, z}         (pipeline.py:199-205)
with C_d,field held as compressed slit streams in HBM and the three products
issued as ONE persistent fused decode+GEMV launch over every (slit, block-row)
job (whff_gemv_plan_*).

Sharding (multi-GPU): the (axis, slit, block-row) units of the field are
split into N contiguous ranges of equal count (FixedRate: equal bytes) or of
equal compressed bytes (variable-rate modes, `weights`); rank r decodes only its range
(its streams are the only ones it holds), so the step needs no data-path
collective except the tiny S broadcast (or a replicated thermal step) and the
all-gather of the per-rank deformation rows.  The rows never split a
reduction, so there is no all-reduce.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import CorruptStreamError


class GemvPlan:
    """Batched fused decode+GEMV over many (stream, vector, output, rows) jobs."""

    def __init__(self, jobs, policy="mixed", evaluation="exact"):
        # jobs: list of (DeviceStream, v_tensor, y_tensor, row_begin, row_end)
        n = len(jobs)
        self._keep = jobs
        H = (ctypes.c_void_p * n)(*[j[0].handle for j in jobs])
        V = (ctypes.c_void_p * n)(*[j[1].data_ptr() for j in jobs])
        Y = (ctypes.c_void_p * n)(*[j[2].data_ptr() for j in jobs])
        RB = (ctypes.c_uint64 * n)(*[int(j[3]) for j in jobs])
        RE = (ctypes.c_uint64 * n)(*[int(j[4]) for j in jobs])
        h = ctypes.c_void_p()
        _lib.call("whff_gemv_plan_create", n, H, V, Y, RB, RE, _lib.POLICY[policy],
                  _lib.EVAL[evaluation], ctypes.byref(h))
        self._h = h
        br, bw, nb = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _lib.call("whff_gemv_plan_traffic", h, ctypes.byref(br), ctypes.byref(bw), ctypes.byref(nb))
        self.bytes_read, self.bytes_written, self.n_blocks = br.value, bw.value, nb.value
        self.flops = sum((j[4] - j[3]) * (2 * j[0].cols - 1) for j in jobs)

    def launch(self, status):
        _lib.call("whff_gemv_plan_launch", self._h, _lib.ptr(status), _lib.cur_stream())

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().whff_gemv_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Unit:
    axis: int
    slit: int
    brow: int


def unit_bounds(n_units, world, weights=None):
    """Contiguous split of n_units ordered units over `world` ranks:
    boundaries b[0] = 0 <= b[1] <= ... <= b[world] = n_units.  Equal counts
    without weights; with per-unit weights (compressed bytes of each block-
    row: variable-rate modes are balanced by bytes) rank r starts
    at the first unit whose preceding weight reaches r/world of the total."""
    if weights is None:
        return [n_units * r // world for r in range(world + 1)]
    w = np.asarray(weights, dtype=np.int64).reshape(-1)
    if w.size != n_units or (w < 0).any():
        raise ValueError("weights: one nonnegative value per unit")
    excl = np.concatenate([[0], np.cumsum(w)[:-1]]) if n_units else np.zeros(0, np.int64)
    total = int(w.sum())
    b = [0]
    for r in range(1, world):
        # first u whose preceding weight reaches floor(total * r / world)
        b.append(int(np.searchsorted(excl, (total * r) // world, side="left")))
    b.append(n_units)
    return [max(b[i], b[i - 1]) if i else b[i] for i in range(len(b))]


def shard_units(n_axes, n_slits, rows_per_slit, world, rank, weights=None):
    """Contiguous split of the (axis, slit, block-row) units: equal counts,
    or balanced by `weights` (one per unit, in unit order, e.g. the
    compressed bytes of each block-row from DeviceStream.block_row_bytes).

    Returns, for this rank, a list of (axis, slit, row_begin, row_end) jobs and
    the global unit range.  Concatenating every rank's rows in rank order
    gives, per axis, the field rows in order.
    """
    bpr = (rows_per_slit + 3) // 4
    total = n_axes * n_slits * bpr
    bounds = unit_bounds(total, world, weights)
    u0, u1 = bounds[rank], bounds[rank + 1]
    jobs = []
    u = u0
    while u < u1:
        axis, rem = divmod(u, n_slits * bpr)
        slit, brow = divmod(rem, bpr)
        take = min(u1 - u, bpr - brow)          # stay inside the slit
        r0 = brow * 4
        r1 = min(rows_per_slit, (brow + take) * 4)
        jobs.append((axis, slit, r0, r1))
        u += take
    return jobs, (u0, u1)


def shard_row_counts(n_axes, n_slits, rows_per_slit, world, weights=None):
    """Rows owned by each rank, per axis (for un-padding the all-gather)."""
    out = []
    for r in range(world):
        jobs, _ = shard_units(n_axes, n_slits, rows_per_slit, world, r, weights)
        counts = [0] * n_axes
        for axis, _, r0, r1 in jobs:
            counts[axis] += r1 - r0
        out.append(counts)
    return out


def unit_weights(streams, n_axes, n_slits):
    """Per-unit compressed bytes (axis, slit, block-row order) from device
    streams (every streams[axis][slit] must be present)."""
    return np.concatenate([streams[a][s].block_row_bytes() for a in range(n_axes)
                           for s in range(n_slits)])


class FieldStep:
    """Thermal step + fused field products on this rank's share of the field.

    streams[axis][slit] -> DeviceStream for slits this rank needs (others may
    be None).  A, P: thermal.DeviceCSR; B, dark, footprint: CUDA tensors.
    """

    def __init__(self, A, B, P, streams, rows_per_slit, n_slits, dark, footprint, dose=1.0,
                 policy="mixed", evaluation="exact", world=1, rank=0, group=None,
                 vector_mode="broadcast", weights=None):
        torch = _lib.require_cuda()
        self.A, self.B, self.P = A, B, P
        self.dark, self.footprint, self.dose = dark, footprint, dose
        self.world, self.rank, self.group = world, rank, group
        self.vector_mode = vector_mode
        self.n_axes = len(streams)
        self.rows_per_slit, self.n_slits = rows_per_slit, n_slits
        dev = torch.device("cuda", torch.cuda.current_device())
        T, S = A.shape[0], P.shape[0]
        self.T = torch.zeros(T, dtype=torch.float32, device=dev)
        self.T_next = torch.zeros(T, dtype=torch.float32, device=dev)
        self.u = torch.zeros(T, dtype=torch.float32, device=dev)
        self.S = torch.zeros(S, dtype=torch.float32, device=dev)
        self.status = _lib.status_word(dev)
        jobs, self.unit_range = shard_units(self.n_axes, n_slits, rows_per_slit, world, rank, weights)
        self.jobs = jobs
        self.local_rows = sum(r1 - r0 for _, _, r0, r1 in jobs)
        counts = shard_row_counts(self.n_axes, n_slits, rows_per_slit, world, weights)
        self.rank_rows = [sum(c) for c in counts]
        self.max_rows = max(self.rank_rows)
        self.local = torch.zeros(self.max_rows, dtype=torch.float32, device=dev)
        plan_jobs, off = [], 0
        for axis, slit, r0, r1 in jobs:
            ds = streams[axis][slit]
            plan_jobs.append((ds, self.S, self.local[off:off + (r1 - r0)], r0, r1))
            off += r1 - r0
        self.plan = GemvPlan(plan_jobs, policy, evaluation) if plan_jobs else None
        self.gathered = torch.zeros(self.max_rows * world, dtype=torch.float32, device=dev)
        self.graph = None

    # -- pieces ---------------------------------------------------------------
    def thermal(self):
        from .thermal import csr_matvec, source_term_device
        source_term_device(self.footprint, self.dark, self.dose, out=self.u)
        csr_matvec(self.A, self.T, self.B, self.u, out=self.T_next)
        csr_matvec(self.P, self.T_next, out=self.S)
        self.T.copy_(self.T_next)   # fixed buffers: the step is graph-capturable

    def products(self):
        if self.plan is not None:
            self.plan.launch(self.status)

    def step_local(self):
        """One step without collectives (capturable in a CUDA graph)."""
        self.status.fill_(-1)
        if self.world == 1 or self.vector_mode == "replicate" or self.rank == 0:
            self.thermal()
        if self.world > 1 and self.vector_mode == "broadcast":
            import torch.distributed as dist
            dist.broadcast(self.S, src=0, group=self.group)
        self.products()

    _list_gather = False

    def gather(self):
        """All-gather the per-rank deformation rows (padded to max_rows): one
        all_gather_into_tensor on every backend that has it (NCCL; gloo
        where it supports the tensor's device), the list form otherwise."""
        import torch.distributed as dist
        if not self._list_gather:
            try:
                dist.all_gather_into_tensor(self.gathered, self.local, group=self.group)
                return
            except (RuntimeError, NotImplementedError, ValueError):
                if dist.get_backend(self.group) == "nccl":
                    raise
                self._list_gather = True
        parts = list(self.gathered.view(self.world, self.max_rows).unbind(0))
        dist.all_gather(parts, self.local, group=self.group)

    def step(self):
        self.step_local()
        if self.world > 1:
            self.gather()

    def check(self):
        if _lib.read_status(self.status) is not None:
            raise CorruptStreamError("decoded array contains non-finite values")

    def deformations(self):
        """Per-axis field deformation rows (host numpy), rank order = row order."""
        torch = _lib.require_cuda()
        if self.world == 1:
            flat = self.local[: self.local_rows]
        else:
            parts = [self.gathered[r * self.max_rows: r * self.max_rows + self.rank_rows[r]]
                     for r in range(self.world)]
            flat = torch.cat(parts)
        flat = flat.cpu().numpy()
        per_axis = self.n_slits * self.rows_per_slit
        return {a: flat[a * per_axis:(a + 1) * per_axis] for a in range(self.n_axes)}

    # -- CUDA graph -------------------------------------------------------------
    def capture(self):
        """Capture step_local (N=1 or replicate mode) into a CUDA graph."""
        torch = _lib.require_cuda()
        if self.world > 1 and self.vector_mode == "broadcast":
            return False
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                self.step_local()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step_local()
        self.graph = g
        return True

    def replay(self):
        if self.graph is None:
            self.step_local()
        else:
            self.graph.replay()
