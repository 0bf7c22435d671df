"""Device-resident scan: the reference's two-stage pipeline (pipeline.py:164-289)
executed on the B200, with the firm-deadline accounting measured on the
device instead of simulated.

Reference semantics kept (pipeline.py:1-8): the per-millisecond thermal state
advances through every schedule step (thermal.py:120-140); on light steps the
three per-axis deformation products of the illuminated slit are evaluated
(pipeline.py:199-205); values never depend on timing; deadline misses are
recorded, never fatal; the trace and its CSV export have the reference's
fields and format (pipeline.py:369-381).

What changes:
  * everything runs on one CUDA stream: source term, T' = A T + B u and
    S = P T' (bit-identical CSR kernels), then ONE fused decode+GEMV launch
    per light step over the slit's three compressed streams;
  * stage 1 (transfer + decode) is not a separate stage: the compressed slit
    streams are resident in HBM and decoded inside the GEMV, so t_transfer
    and t_decode are 0 and bytes_in keeps the reference's meaning (payload
    bytes moved per light step, pipeline.py:147);
  * stage-2 start/end times are CUDA events on the stream; with
    ``step_period_s`` set, each schedule step is held until its millisecond
    on the device clock (%globaltimer, whff_wait_until), so the trace is a
    real-time run; without it steps run back to back (throughput mode);
  * ``streaming=True`` reproduces the reference's stage 1 for fields larger
    than HBM: the slits' compressed (device-layout) payloads and index arrays
    live in pinned host memory and a ring of ``queue_depth`` device slots is
    refilled by H2D copies on a second CUDA stream, bounded by the consumer exactly like
    the reference's queue (pipeline.py:225-238); the trace then carries the
    measured transfer times;
  * a field's latency is its last delivery (end of its last light step)
    minus the field's start, judged against its budget as the reference's
    simulated clock does (pipeline.py:269-270, 285-289).

Evaluations: "reference" decodes the slit words and runs the sequential mixed
GEMV (bit-identical to the reference's decompress + gemv), "exact" and
"coefficient" are the fused kernels (within the reference's error bound).
Without compression the binary32 slits are resident and the sequential mixed
GEMV is used (bit-identical).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import codec as codec_mod
from .errors import CorruptStreamError, WhffError
from .model import AXES


@dataclass
class PipelineConfig:
    """pipeline.py:26-53 plus the device-execution knobs."""
    interconnect_bandwidth: float = 16e9
    use_compression: bool = False
    codec_mode: object = None                  # default FixedAccuracy(1e-12)
    decode_throughput: float = 33e9
    queue_depth: int = 2
    axis_workers: int = 1
    time_source: str = "device"                # "device" (= "real"): CUDA events /
                                               # %globaltimer; "simulated": the reference's
                                               # cost-model clock (pipeline.py:208-289)
    compute_flops_per_s: float = 50e9
    transfer_time_override: float = None
    compute_time_override: float = None
    decode_time_override: float = None
    decode_stall_s: dict = field(default_factory=dict)
    # B200 additions
    evaluation: str = "exact"                  # "reference" | "exact" | "coefficient"
    policy: str = "mixed"
    layout: str = None                         # device layout of resident slits: "packed"
                                               # (default: the tile-packed copy read by
                                               # k_pk_gemv2), "skeleton-first", "reference";
                                               # streaming stages a stream layout
                                               # (default "skeleton-first")
    step_period_s: float = None                # pace steps on the device clock
    streaming: bool = False                    # stage 1 = H2D of the slit streams (ring of
                                               # queue_depth device slots)

    def __post_init__(self):
        if self.interconnect_bandwidth <= 0:
            raise WhffError("interconnect bandwidth must be positive")
        if self.queue_depth < 2:
            raise WhffError("queue_depth must be >= 2 (double buffering)")
        if not 1 <= self.axis_workers <= 3:
            raise WhffError("axis_workers must be in 1..3")
        if self.time_source not in ("device", "real", "simulated"):
            raise WhffError(f"unknown time source {self.time_source!r}")
        if self.evaluation not in ("reference", "exact", "coefficient"):
            raise WhffError(f"unknown evaluation {self.evaluation!r}")
        if self.step_period_s is not None and self.step_period_s <= 0:
            raise WhffError("step_period_s must be positive")
        if self.codec_mode is None:
            self.codec_mode = codec_mod.FixedAccuracy(1e-12)
        if self.layout is None:
            self.layout = "skeleton-first" if self.streaming else "packed"
        if self.layout not in ("packed", "skeleton-first", "reference"):
            raise WhffError(f"unknown layout {self.layout!r}")
        if self.streaming and self.layout == "packed":
            raise WhffError("streaming stages the stream layouts (skeleton-first or reference); "
                            "the packed copy is built on the device for resident slits")
        if self.streaming and not self.use_compression:
            raise WhffError("streaming stages compressed slit streams (use_compression=True)")


@dataclass
class StepRecord:
    field_id: int
    k: int
    phase: str
    slit: int
    bytes_in: int
    t_transfer: float
    t_decode: float
    t_compute: float
    stage1_start: float
    stage1_end: float
    stage2_start: float
    stage2_end: float


@dataclass
class FieldRecord:
    field_id: int
    start: float
    end: float
    latency_s: float
    budget_s: float
    deadline_met: bool


@dataclass
class PipelineTrace:
    steps: list
    fields: list


@dataclass
class ScanResult:
    deformations: dict
    trace: PipelineTrace


@dataclass
class DeadlineReport:
    verdicts: list
    miss_rate: float
    worst_latency_s: float


# ---------------------------------------------------------------------------
# slit preparation (pipeline.py:128-152): compress once, keep in HBM
# ---------------------------------------------------------------------------

class _Slit:
    """One (field, slit): the three axis operators on the device (streaming:
    their device-layout payloads in pinned host memory instead)."""

    def __init__(self, model, f, s, cfg, dev, keep_template=False):
        import torch
        self.streams, self.mats, self.host = [], [], []
        self.nbytes = 0
        self.raw_bytes = 3 * model.spec.M * model.S * 4    # sum of c_slit.nbytes
        for axis in AXES:
            if hasattr(model, "slit_rows"):
                rows = model.slit_rows(axis, f, s, device=dev)
            else:                            # the reference's WaferModel (model.py:94-112)
                rows = model.fetch_slit_submatrix(model.fetch_field_submatrix(axis, f), f, s)
                rows = torch.from_numpy(np.ascontiguousarray(rows, np.float32)).to(dev)
            if cfg.use_compression:
                ds = codec_mod.compress_device(rows, cfg.codec_mode)
                self.nbytes += ds.payload_bytes
                if cfg.layout == "packed":
                    ds.pack()
                elif cfg.evaluation != "reference" and cfg.layout != "reference":
                    ds.relayout(cfg.layout)
                if cfg.streaming:
                    self.host.append(ds.export(pinned=True))
                    if keep_template:
                        self.streams.append(ds)
                    else:
                        ds.close()
                else:
                    self.streams.append(ds)
            else:
                m = rows if isinstance(rows, torch.Tensor) else torch.from_numpy(
                    np.ascontiguousarray(rows))
                m = m.to(dev).contiguous()
                self.nbytes += m.numel() * 4
                self.mats.append(m)
            del rows


def _prepare(model, schedule, cfg, dev):
    need = {}
    for fs in schedule.fields:
        n_slits = model.n_slits(fs.field_id)
        for i in range(fs.t_l):
            need.setdefault((fs.field_id, fs.slit_for_light_step(i, n_slits)), None)
    return {key: _Slit(model, key[0], key[1], cfg, dev, keep_template=(i == 0))
            for i, key in enumerate(need)}


# ---------------------------------------------------------------------------
# scan execution
# ---------------------------------------------------------------------------

def run_scan(model, schedule, heatload, cfg=None, resampler=None, backend=None):
    """pipeline.py:164-181 on the device.  Returns ScanResult with per-axis
    (n_light_total, M) binary32 deformations and the measured trace."""
    torch = _lib.require_cuda()
    from .executor import GemvPlan
    from .mpgemv import gemv_device
    from .thermal import DeviceCSR, DeviceHeatLoad, csr_matvec

    if backend not in (None, "b200"):
        raise WhffError(f"unknown backend {backend!r} (the B200 pipeline has no other)")
    cfg = cfg or PipelineConfig()
    if len(schedule.fields) > model.n_fields:
        raise WhffError(f"schedule has {len(schedule.fields)} fields, model only {model.n_fields}")
    dev = torch.device("cuda", torch.cuda.current_device())
    M, T_, S_ = model.spec.M, model.T, model.S

    slits = _prepare(model, schedule, cfg, dev)
    A = DeviceCSR(model.A_f64(), device=dev)
    P = DeviceCSR(model.P_f64(), device=dev)
    B = torch.from_numpy(np.ascontiguousarray(model.B, np.float32)).to(dev)
    fps = {}
    for key in slits:
        fps[key] = heatload.light_load(*key)
    hl = DeviceHeatLoad(heatload.dark_load, fps, heatload.dose_scale)

    # enumerate the steps (deterministic, timing-independent)
    steps = []                       # (field_schedule, k_in_field, phase, slit)
    for fs in schedule.fields:
        n_slits = model.n_slits(fs.field_id)
        for i in range(fs.t_l + fs.t_d):
            if i < fs.t_l:
                steps.append((fs, i, "light", fs.slit_for_light_step(i, n_slits)))
            else:
                steps.append((fs, i, "dark", -1))
    n_light = sum(1 for s in steps if s[2] == "light")

    T = torch.zeros(T_, dtype=torch.float32, device=dev)
    T_next = torch.empty_like(T)
    u = torch.empty_like(T)
    S = torch.zeros(S_, dtype=torch.float32, device=dev)
    D = torch.zeros((max(n_light, 1), 3, M), dtype=torch.float32, device=dev)
    status = _lib.status_word(dev)

    # streaming: a ring of queue_depth slots, each three device streams of the
    # field's geometry, refilled by H2D copies on their own CUDA stream
    ring = None
    light_keys = [(fs.field_id, slit) for fs, i, phase, slit in steps if phase == "light"]
    if cfg.streaming:
        template = next(sl for sl in slits.values() if sl.streams)
        cap = [max(int(sl.host[a][0].numel()) for sl in slits.values()) for a in range(3)]
        ring = [[template.streams[a].clone() for a in range(3)] for _ in range(cfg.queue_depth)]
        for slot in ring:
            for a in range(3):
                slot[a].reserve(cap[a])

    # one plan per light item: the slit's three streams -> D[item, axis]
    plans, scratch = [], None
    item = 0
    for fs, i, phase, slit in steps:
        if phase != "light":
            continue
        sl = slits[(fs.field_id, slit)]
        if cfg.use_compression and cfg.evaluation != "reference":
            src = ring[item % cfg.queue_depth] if cfg.streaming else sl.streams
            if cfg.streaming:                # the item's payload sizes, for its plan
                for a in range(3):
                    src[a].rebind(sl.host[a][0].numel())
            plans.append(GemvPlan([(src[a], S, D[item, a], 0, M) for a in range(3)],
                                  cfg.policy, cfg.evaluation))
        else:
            plans.append(None)
        item += 1
    if cfg.use_compression and cfg.evaluation == "reference":
        scratch = torch.empty((M, S_), dtype=torch.float32, device=dev)

    cur = torch.cuda.current_stream(dev)
    n = len(steps)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    t_base = torch.zeros(1, dtype=torch.int64, device=dev)
    period_ns = None if cfg.step_period_s is None else int(round(cfg.step_period_s * 1e9))

    cstream = torch.cuda.Stream(dev) if cfg.streaming else None
    up_s = [torch.cuda.Event(enable_timing=True) for _ in range(n_light)] if cfg.streaming else []
    up_e = [torch.cuda.Event(enable_timing=True) for _ in range(n_light)] if cfg.streaming else []
    done = [torch.cuda.Event() for _ in range(n_light)] if cfg.streaming else []

    def upload(it):                          # stage 1 of light item `it` (copy stream)
        slot = ring[it % cfg.queue_depth]
        with torch.cuda.stream(cstream):
            if it >= cfg.queue_depth:        # the slot's previous item has been consumed
                cstream.wait_event(done[it - cfg.queue_depth])
            up_s[it].record(cstream)
            for a in range(3):
                slot[a].import_async(*slits[light_keys[it]].host[a])
            up_e[it].record(cstream)

    status.fill_(-1)
    torch.cuda.synchronize(dev)
    ev0.record(cur)
    if cfg.streaming:
        cstream.wait_event(ev0)
        for it in range(min(cfg.queue_depth, n_light)):
            upload(it)
    if period_ns is not None:
        _lib.call("whff_device_timestamp", _lib.ptr(t_base), _lib.cur_stream())
    item = 0
    for j, (fs, i, phase, slit) in enumerate(steps):
        if period_ns is not None:    # step j may not start before its millisecond
            _lib.call("whff_wait_until", _lib.ptr(t_base), j * period_ns, _lib.cur_stream())
        ev_s[j].record(cur)
        hl.source(fs.field_id, phase, slit if phase == "light" else None, out=u)
        csr_matvec(A, T, B, u, out=T_next)
        csr_matvec(P, T_next, out=S)
        T, T_next = T_next, T
        if phase == "light":
            sl = slits[(fs.field_id, slit)]
            if cfg.streaming:                # stage 1 of this item must have landed
                cur.wait_event(up_e[item])
            if not cfg.use_compression:
                for a in range(3):
                    gemv_device(sl.mats[a], S, "mixed", "sequential", out=D[item, a])
            elif cfg.evaluation == "reference":
                src = ring[item % cfg.queue_depth] if cfg.streaming else sl.streams
                for a in range(3):
                    src[a].decode(out=scratch, check=False)
                    gemv_device(scratch, S, "mixed", "sequential", out=D[item, a])
            else:
                plans[item].launch(status)
            if cfg.streaming:                # release the slot, refill it with item + depth
                done[item].record(cur)
                if item + cfg.queue_depth < n_light:
                    upload(item + cfg.queue_depth)
            item += 1
        ev_e[j].record(cur)
    torch.cuda.synchronize(dev)
    if _lib.read_status(status) is not None:
        raise CorruptStreamError("decoded array contains non-finite values")

    # ---- trace (seconds since the scan started, device clock) ---------------
    t_s = [ev0.elapsed_time(e) / 1e3 for e in ev_s]
    t_e = [ev0.elapsed_time(e) / 1e3 for e in ev_e]
    t_up = [(ev0.elapsed_time(up_s[i]) / 1e3, ev0.elapsed_time(up_e[i]) / 1e3)
            for i in range(n_light)] if cfg.streaming else []
    records, fields = [], []
    k = 0
    j = 0
    li = 0
    for fs in schedule.fields:
        nsteps = fs.t_l + fs.t_d
        field_start = t_s[j]
        last_delivery = field_start
        for _ in range(nsteps):
            _, i, phase, slit = steps[j]
            k += 1
            nbytes = slits[(fs.field_id, slit)].nbytes if phase == "light" else 0
            if phase == "light" and cfg.streaming:
                s1, e1 = t_up[li]
                records.append(StepRecord(fs.field_id, k, phase, slit, nbytes, e1 - s1, 0.0,
                                          t_e[j] - t_s[j], s1, e1, t_s[j], t_e[j]))
            else:
                records.append(StepRecord(fs.field_id, k, phase, slit, nbytes, 0.0, 0.0,
                                          t_e[j] - t_s[j], t_s[j], t_s[j], t_s[j], t_e[j]))
            li += phase == "light"
            if phase == "light":             # a delivery (pipeline.py:269-270, 287)
                last_delivery = t_e[j]
            j += 1
        latency = last_delivery - field_start
        budget = fs.time_budget_ms / 1e3
        fields.append(FieldRecord(fs.field_id, field_start, t_e[j - 1], latency, budget,
                                  latency <= budget))

    if cfg.time_source == "simulated":       # the reference's clock, same values
        records, fields = _simulated_trace(model, schedule, cfg, slits)

    Dh = D[:n_light].cpu().numpy()
    deformations = {}
    for a, axis in enumerate(AXES):
        rows = Dh[:, a, :] if n_light else np.zeros((0, M), np.float32)
        if resampler is not None:
            rows = np.stack([np.asarray(resampler(axis, r), dtype=np.float32) for r in rows]) \
                if n_light else rows
        deformations[axis] = np.ascontiguousarray(rows, dtype=np.float32)
    for p in plans:
        if p is not None:
            p.close()
    if ring is not None:
        for slot in ring:
            for ds in slot:
                ds.close()
    return ScanResult(deformations, PipelineTrace(records, fields))


# ---------------------------------------------------------------------------
# the reference's simulated clock (pipeline.py:155-162, 184-196, 208-289)
# ---------------------------------------------------------------------------

def _step_flops(model, light):
    """pipeline.py:155-162: sparse update + diagonal input + interpolation,
    plus the three per-axis products on light steps."""
    flops = 2 * model.A.nnz + 2 * model.T + 2 * model.P.nnz
    if light:
        flops += 3 * model.spec.M * (2 * model.S - 1)
    return flops


def _stage1_times(cfg, field_id, nbytes, raw_bytes):
    """pipeline.py:184-196."""
    if cfg.transfer_time_override is not None:
        t_transfer = cfg.transfer_time_override
    else:
        t_transfer = nbytes / cfg.interconnect_bandwidth
    if cfg.decode_time_override is not None:
        t_decode = cfg.decode_time_override
    elif cfg.use_compression:
        t_decode = raw_bytes / cfg.decode_throughput
    else:
        t_decode = 0.0
    t_decode += cfg.decode_stall_s.get(field_id, 0.0)
    return t_transfer, t_decode


def _simulated_trace(model, schedule, cfg, slits):
    """The trace of the reference's simulated two-stage pipeline
    (pipeline.py:208-289): a producer that may run queue_depth light items
    ahead of the consumer, consumer steps costed by the flop model.  Pure host
    arithmetic over the deterministic step list, evaluated in the reference's
    order so the times are identical."""
    items = []
    for fs in schedule.fields:
        n_slits = model.n_slits(fs.field_id)
        for i in range(fs.t_l):
            slit = fs.slit_for_light_step(i, n_slits)
            sl = slits[(fs.field_id, slit)]
            items.append((slit, sl.nbytes) + _stage1_times(cfg, fs.field_id, sl.nbytes,
                                                           sl.raw_bytes))
    p_finish, c_start = [], []
    last = [0.0]

    def produce_through(i):
        while len(p_finish) <= i:
            j = len(p_finish)
            start = last[0]
            if j >= cfg.queue_depth:         # bounded queue
                start = max(start, c_start[j - cfg.queue_depth])
            last[0] = start + items[j][2] + items[j][3]
            p_finish.append((start, last[0]))

    steps, fields = [], []
    c_time, item, k = 0.0, 0, 0
    for fs in schedule.fields:
        field_start = c_time
        last_delivery = c_time
        for i in range(fs.t_l + fs.t_d):
            k += 1
            light = i < fs.t_l
            if cfg.compute_time_override is not None:
                t_comp = cfg.compute_time_override
            else:
                t_comp = _step_flops(model, light) / cfg.compute_flops_per_s
                if light:
                    t_comp /= min(cfg.axis_workers, 3)
            if light:
                produce_through(item)
                slit, nbytes, t_tr, t_dec = items[item]
                s1_start, s1_end = p_finish[item]
                s2_start = max(c_time, s1_end)
                c_start.append(s2_start)
                s2_end = s2_start + t_comp
                steps.append(StepRecord(fs.field_id, k, "light", slit, nbytes, t_tr, t_dec, t_comp,
                                        s1_start, s1_end, s2_start, s2_end))
                last_delivery = s2_end
                item += 1
            else:
                s2_start, s2_end = c_time, c_time + t_comp
                steps.append(StepRecord(fs.field_id, k, "dark", -1, 0, 0.0, 0.0, t_comp,
                                        s2_start, s2_start, s2_start, s2_end))
            c_time = s2_end
        latency = last_delivery - field_start
        budget = fs.time_budget_ms / 1e3
        fields.append(FieldRecord(fs.field_id, field_start, c_time, latency, budget,
                                  latency <= budget))
    return steps, fields


# ---------------------------------------------------------------------------
# reporting (pipeline.py:348-381)
# ---------------------------------------------------------------------------

def deadline_report(trace, budgets=None):
    verdicts = []
    for fr in trace.fields:
        budget = fr.budget_s if budgets is None else budgets[fr.field_id]
        verdicts.append((fr.field_id, fr.latency_s <= budget, fr.latency_s))
    misses = sum(1 for _, met, _ in verdicts if not met)
    return DeadlineReport(verdicts, misses / len(verdicts) if verdicts else 0.0,
                          max((lat for _, _, lat in verdicts), default=0.0))


TRACE_HEADER = ("field,k,phase,slit,bytes_in,t_transfer_s,t_decode_s,"
                "t_compute_s,latency_s,deadline_met")


def export_trace_csv(trace, path):
    by_field = {fr.field_id: fr for fr in trace.fields}
    with open(path, "w", newline="") as fh:
        fh.write(TRACE_HEADER + "\n")
        for s in trace.steps:
            fr = by_field[s.field_id]
            fh.write(f"{s.field_id},{s.k},{s.phase},{s.slit},{s.bytes_in},"
                     f"{s.t_transfer!r},{s.t_decode!r},{s.t_compute!r},"
                     f"{fr.latency_s!r},{str(fr.deadline_met).lower()}\n")


def pipeline_period(t_transfer, t_compute, t_decode, r, compressed):
    """Table-1 period algebra (pipeline.py:100-108)."""
    _check_table1(t_transfer, t_compute, t_decode, r)
    if compressed:
        return max(t_transfer / r, t_compute + t_decode)
    return max(t_transfer, t_compute)


def pipeline_latency(t_transfer, t_compute, t_decode, r, compressed):
    _check_table1(t_transfer, t_compute, t_decode, r)
    if compressed:
        return t_compute + t_transfer / r + t_decode
    return t_compute + t_transfer


def _check_table1(t_transfer, t_compute, t_decode, r):
    if min(t_transfer, t_compute, t_decode) < 0:
        raise WhffError("stage times must be nonnegative")
    if r < 1:
        raise WhffError(f"compression factor must be >= 1, got {r}")
