#!/usr/bin/env python
"""WHFF paper-scale step benchmark (BASELINE.json configs[2], N=1; configs[3]
under torchrun N>1).

One step = thermal update + interpolation (T = 608^2, S = 256,000, nnz 7) and
the x/y/z field products D_d = C_d,field S, C_d,field = 52 slits x 378 rows x
256,000 columns per axis held as FixedRate(8) WHFZ streams in HBM (15.18 GB;
~30.2 GFLOP per step), decoded on the fly by the fused kernel.

Prints one JSON line (rank 0).  `value` is compressed GB/s over the whole job
(payload + device index bytes of every slit stream / step time, max over
ranks); GFLOP/s, decoded-equivalent GB/s and the per-step p50/p99 latency
against the 50 ms firm deadline ride along.  `--impl reference` times the
reference's own CPU path (oracle/_ref: whff.codec.decompress + mpgemv.gemv)
on a bounded sample of the same workload with all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused decompress+GEMV GB/s and GFLOP/s per GPU; p99 step latency vs 50 ms"
DEADLINE_MS = 50.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N>1 path with several ranks sharing one GPU (a "
                         "functional check; numbers are not NVLink numbers)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mode", default="rate:8", help="rate:BPV | precision:P | accuracy:TOL")
    ap.add_argument("--evaluation", default="coefficient", choices=["exact", "coefficient"],
                    help="coefficient: accumulate 2^k Q (G^T v) per block and apply the inverse "
                         "lift G once per block-row (SURVEY 7, hard part 2); exact: decoded "
                         "binary32 words x v, the reference's products")
    ap.add_argument("--layout", default="packed", choices=["reference", "skeleton-first", "packed"],
                    help="packed: the tile-packed device copy (whff_dstream_pack: the decoded "
                         "coefficients as fixed-width fields per segment, bit-exact words) is "
                         "what the kernel reads; reference / skeleton-first: the fused kernel "
                         "parses the WHFZ bitstream (or its per-block bit permutation) itself")
    ap.add_argument("--policy", default="mixed", choices=["mixed", "single", "double"])
    ap.add_argument("--slits", type=int, default=52)
    ap.add_argument("--rows", type=int, default=378)
    ap.add_argument("--S", type=int, default=256000)
    ap.add_argument("--grid", type=int, default=608)
    ap.add_argument("--preset", choices=["paper", "mesh4x"], default=None,
                    help="paper: configs[2]/[3] (S = 256,000, T = 608^2, the defaults); "
                         "mesh4x: the configs[4] sustained workload (S = 1,024,000, "
                         "T = 1216^2, 1000 latency steps), unchanged at --gpus 8")
    ap.add_argument("--distinct", type=int, default=0,
                    help="distinct slit contents per axis (0 = all); the rest are "
                         "physically distinct HBM copies")
    ap.add_argument("--vector-mode", default="replicate", choices=["broadcast", "replicate"],
                    help="replicate: every rank runs the deterministic thermal step (~25 MB), "
                         "so the step needs no broadcast and stays CUDA-graph captured; "
                         "broadcast: rank 0 computes S and broadcasts it")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variants", default="exact,accuracy:1e-12,precision:17",
                    help="extra lines measured after the headline (N=1): 'exact' = the same "
                         "streams with the reference's products (exact evaluation); "
                         "'<mode>' = the same step over streams of another codec mode "
                         "(accuracy:1e-12 is the reference pipeline's default, pipeline.py:50-51); "
                         "'' = none")
    ap.add_argument("--cpu-sample-cols", type=int, default=8192)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--latency-steps", type=int, default=1000,
                    help="extra back-to-back steps (after the timed region) whose per-step "
                         "CUDA-event times give latency p50/p99/max (SURVEY 8d: >= 1000)")
    args = ap.parse_args()
    if args.preset == "mesh4x":
        args.S, args.grid, args.latency_steps = 1024000, 1216, max(args.latency_steps, 1000)
    elif args.preset == "paper":
        args.S, args.grid = 256000, 608
    return args


def parse_mode(s):
    from paper_1902_08018_b200 import codec
    kind, p = s.split(":")
    if kind == "rate":
        return codec.FixedRate(int(p))
    if kind == "precision":
        return codec.FixedPrecision(int(p))
    return codec.FixedAccuracy(float(p))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class Clocks:
    """nvidia-smi clocks/throttle sampling during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        if sm:
            out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                   "reasons": sorted(reasons), "samples": len(sm)}
        return out


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# workload construction
# ---------------------------------------------------------------------------

def build_field(args, world, rank):
    import numpy as np
    import torch
    from paper_1902_08018_b200 import codec, synth, thermal
    from paper_1902_08018_b200.executor import FieldStep, shard_units

    K = args.slits * args.rows
    spec = synth.Spec(grid_rows=args.grid, grid_cols=args.grid, S=args.S, K=K, M=args.rows,
                      nnz_target=7, seed=7, n_fields=1)
    t0 = time.time()
    ops = synth.generate(spec)
    dark, fps, dose = synth.heatload(spec, 1, args.slits, seed=0)
    t_ops = time.time() - t0
    mode = parse_mode(args.mode)
    jobs, _ = shard_units(3, args.slits, args.rows, world, rank)
    need = sorted({(a, s) for a, s, _, _ in jobs})
    distinct = args.distinct if args.distinct > 0 else args.slits
    streams = [[None] * args.slits for _ in range(3)]
    made = {}
    t0 = time.time()
    for a, s in need:
        src = s % distinct
        if (a, src) not in made:
            rows = synth.deformation_rows(spec, a, ops.phases[synth.AXES[a]], src * args.rows,
                                          (src + 1) * args.rows, device="cuda")
            made[(a, src)] = codec.compress_device(rows, mode)
            if args.layout == "packed":
                made[(a, src)].pack()
            elif args.layout != "reference":
                made[(a, src)].relayout(args.layout)
            del rows
            streams[a][src] = made[(a, src)]
        if streams[a][s] is None:
            streams[a][s] = made[(a, src)].clone()
    torch.cuda.synchronize()
    t_enc = time.time() - t0
    A = thermal.DeviceCSR(ops.A64())
    P = thermal.DeviceCSR(ops.P64())
    B = torch.from_numpy(ops.B).cuda()
    fs = FieldStep(A, B, P, streams, args.rows, args.slits, torch.from_numpy(dark).cuda(),
                   torch.from_numpy(fps[(0, 0)]).cuda(), dose, policy=args.policy,
                   evaluation=args.evaluation, world=world, rank=rank,
                   vector_mode=args.vector_mode)
    # compressed bytes this rank decodes per step: the block-rows of its jobs
    # (a slit split across two ranks is held by both but decoded once)
    stream_bytes = 0
    packed_bytes, exceptions, blocks = 0, 0, 0
    for a, s_, r0, r1 in jobs:
        ds = streams[a][s_]
        nbr = (r1 + 3) // 4 - r0 // 4
        stream_bytes += (ds.payload_bytes + ds.index_bytes) * nbr / ds.block_rows
        if getattr(ds, "packed", False):
            packed_bytes += ds.packed_bytes * nbr / ds.block_rows
            exceptions += ds.packed_exceptions
        blocks += nbr * ds.block_cols
    stream_bytes = int(round(stream_bytes))
    info = {"t_ops_s": round(t_ops, 2), "t_encode_s": round(t_enc, 2),
            "streams": sum(1 for row in streams for ds in row if ds is not None),
            "distinct_per_axis": distinct, "stream_bytes_rank": stream_bytes,
            "index_kind": streams[need[0][0]][need[0][1]].index_kind if need else None,
            "packed_bytes_rank": int(round(packed_bytes)),
            "packed_bits_per_block": round(8 * packed_bytes / max(blocks, 1), 2),
            "reference_bits_per_block": round(8 * stream_bytes / max(blocks, 1), 2),
            "packed_exceptions": exceptions}
    return fs, spec, ops, mode, streams, info


# ---------------------------------------------------------------------------
# CPU reference leg
# ---------------------------------------------------------------------------

def _ref_task(payload_path):
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    from whff import codec as rc
    from whff import mpgemv as rm
    d = np.load(payload_path, allow_pickle=True)
    kind, p = str(d["kind"]), d["param"].item()
    mode = {"rate": rc.FixedRate, "precision": rc.FixedPrecision, "accuracy": rc.FixedAccuracy}[kind](
        int(p) if kind != "accuracy" else float(p))
    s = rc.CompressedStream(mode=mode, rows=int(d["rows"]), cols=int(d["cols"]), payload=d["payload"],
                            block_index=d["index"], total_bits=int(d["total_bits"]))
    t0 = time.perf_counter()
    C = rc.decompress(s)
    y = rm.gemv(rm.GemvRequest(C, d["v"], "mixed", "sequential"))
    return time.perf_counter() - t0, int(d["payload"].size), int(C.size), float(y.sum())


def _port_task(payload_path):
    import numpy as np
    from oracle import oracle as orc
    from types import SimpleNamespace
    d = np.load(payload_path, allow_pickle=True)
    kind, p = str(d["kind"]), d["param"].item()
    s = SimpleNamespace(mode=(kind, p), rows=int(d["rows"]), cols=int(d["cols"]),
                        payload=d["payload"], block_index=d["index"])
    t0 = time.perf_counter()
    C = orc.decompress(s)
    y = orc.gemv_kernel(C, d["v"], "mixed", "sequential")
    return time.perf_counter() - t0, int(d["payload"].size), int(C.size), float(y.sum())


def _sample_task(job):
    """Compress one sample chunk on the host with the reference's own encoder
    (oracle/_ref whff.codec.compress; the C port when it is absent) -- no
    CUDA, no libwhff_b200.so in the reference arm."""
    import numpy as np
    from paper_1902_08018_b200 import synth      # host path: numpy only
    (grid, S, K, rows, cols, kind, param, a, path) = job
    spec = synth.Spec(grid_rows=grid, grid_cols=grid, S=S, K=K, M=rows, nnz_target=7, seed=7, n_fields=1)
    # the first `cols` columns of slit 0 of axis a (model.py:258-268, host expression)
    C = synth.deformation_rows(spec, a, 0.5 + a, 0, rows, ncols=cols)
    ref = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "whff")):
        sys.path.insert(0, ref)
        from whff import codec as rc
        mode = {"rate": rc.FixedRate, "precision": rc.FixedPrecision, "accuracy": rc.FixedAccuracy}[kind](
            int(param) if kind != "accuracy" else float(param))
        s = rc.compress(C, mode)
        payload, index, total_bits = s.payload, s.block_index, s.total_bits
    else:
        from oracle import oracle as orc
        s = orc.compress(C, (kind, int(param) if kind != "accuracy" else float(param)))
        payload, index, total_bits = s.payload, s.block_index, s.total_bits
    v = np.random.default_rng(a).random(cols).astype(np.float32)
    np.savez(path, kind=kind, param=np.array(param), rows=rows, cols=cols,
             payload=payload, index=index, total_bits=total_bits, v=v)
    return path


def make_cpu_samples(args, tmpdir):
    """Bounded sample of the workload: the first `--cpu-sample-cols` columns
    of one slit per axis, compressed on the host by the reference encoder
    (in a process pool: ~2.5 s per FixedRate(8) chunk)."""
    import multiprocessing as mp
    kind, param = args.mode.split(":")
    param = float(param)
    K = args.slits * args.rows
    jobs = [(args.grid, args.S, K, args.rows, args.cpu_sample_cols, kind, param, a,
             os.path.join(tmpdir, f"sample{a}.npz")) for a in range(3)]
    with mp.get_context("fork").Pool(3) as pool:
        return pool.map(_sample_task, jobs)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_cpu_leg(paths, reps, warmup=0):
    """Run the CPU path over `reps` x samples with all host cores; returns
    (GB/s compressed, seconds, cores, kind, per-sample seconds)."""
    import multiprocessing as mp
    have_ref = os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "whff"))
    task = _ref_task if have_ref else _port_task
    kind = "reference" if have_ref else "port"
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    work = [p for _ in range(reps) for p in paths]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        if warmup:
            pool.map(task, paths[:1] * min(cores, warmup))
        t0 = time.perf_counter()
        res = pool.map(task, work, chunksize=1)
        wall = time.perf_counter() - t0
    nbytes = sum(r[1] for r in res)
    per = statistics.median(r[0] for r in res)
    return nbytes / wall / 1e9, wall, cores, kind, per, sum(r[2] for r in res)


# ---------------------------------------------------------------------------
# main legs
# ---------------------------------------------------------------------------

def workload_config(args, world):
    """The workload both arms report (`config`): what is computed, not how."""
    if (args.S, args.grid) == (256000, 608):
        name = "paper-scale WHFF step (configs[2])" if world == 1 else \
            f"paper-scale WHFF step row-sharded over {world} GPUs (configs[3])"
    elif args.S == 1024000:
        name = "4x paper mesh step (configs[4] workload)"
    else:
        name = "WHFF step"
    return {"workload": name + f": thermal T={args.grid}^2 nnz7 + 3 axes x {args.slits} slits x "
                               f"{args.rows}x{args.S}",
            "mode": args.mode, "policy": args.policy,
            "parallelism": f"row-shard{world}" if world > 1 else "single",
            "l2": "inputs (compressed field) far larger than L2; no flush needed"}


def step_stream_bytes(args):
    """Compressed bytes of the whole step's slit streams at FixedRate (the
    other modes' sizes depend on the data: None)."""
    kind, p = args.mode.split(":")
    if kind != "rate":
        return None
    blocks = 3 * args.slits * ((args.rows + 3) // 4) * ((args.S + 3) // 4)
    return blocks * 16 * int(p) // 8


def reference_main(args, world, rank):
    """The reference's own CPU path (oracle/_ref: whff.codec.decompress +
    whff.mpgemv.gemv(mixed, sequential), codec.py:296-314, mpgemv.py:54-61) on
    all host cores, on a bounded sample of this workload; no CUDA context and
    no repository .so (sample streams come from the reference encoder)."""
    if rank != 0:
        return 0
    tmp = tempfile.mkdtemp()
    paths = make_cpu_samples(args, tmp)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    reps = max(1, (5 * cores) // 6)          # ~2.5 chunks per core per step
    for _ in range(min(args.warmup, 1)):
        run_cpu_leg(paths, 1)
    total_bytes, t_all, per_chunk, kind = 0.0, 0.0, [], None
    for _ in range(args.steps):
        v, wall, cores, kind, per, _ = run_cpu_leg(paths, reps)
        t_all += wall
        total_bytes += v * wall * 1e9
        per_chunk.append(per)
    value = total_bytes / t_all / 1e9
    full = step_stream_bytes(args)
    # the full step at this sustained all-core rate (the sample is a labelled
    # subset of the same workload: ms_per_step is extrapolated linearly)
    ms_full = 1e3 * full / (value * 1e9) if full else None
    chunk = f"{args.rows}x{args.cpu_sample_cols}"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_full, 1) if ms_full else round(1e3 * t_all / args.steps, 3),
        "ms_per_step_kind": ("full step extrapolated linearly from the sample's all-core rate"
                             if ms_full else "one sample pass"),
        "sample_ms_per_step": round(1e3 * t_all / args.steps, 3),
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 products, f64 accumulate",
        "data": "synthetic (reference smooth-C formula, model.py:252-268)",
        "config": workload_config(args, 1),
        "cpu_baseline": {"value": round(value, 6), "unit": "GB/s", "cores": cores, "kind": kind,
                         "value_1core": round(statistics.mean(
                             int(__import__("numpy").load(p)["payload"].size) for p in paths)
                             / statistics.median(per_chunk) / 1e9, 6),
                         "cpu_model": cpu_model(),
                         "sample": f"reference codec.decompress + mpgemv.gemv(mixed, sequential) on "
                                   f"{3 * reps} chunks of {chunk} ({args.mode}; first {args.cpu_sample_cols} "
                                   f"columns of one slit per axis, streams from the reference encoder) per step"},
        "e2e": {"value": round(value, 6), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def measure_variant(fs, steps, warmup, use_graph):
    """ms per step (graph replays, CUDA events on the current stream) and the
    fused launch alone, for one more FieldStep over resident streams."""
    import torch
    cur = torch.cuda.current_stream()
    if use_graph:
        fs.capture()
    for _ in range(max(3, warmup)):
        fs.replay()
    torch.cuda.synchronize()
    fs.check()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(steps):
        fs.replay()
    e1.record(cur)
    torch.cuda.synchronize()
    fs.check()
    step_ms = e0.elapsed_time(e1) / steps
    e0.record(cur)
    for _ in range(steps):
        fs.plan.launch(fs.status)
    e1.record(cur)
    torch.cuda.synchronize()
    return step_ms, e0.elapsed_time(e1) / steps


def run_variants(args, fs, streams, info, use_graph, hbm):
    """The driver-visible extra lines: the exact
    evaluation over the headline's streams and other codec modes."""
    import copy
    import torch
    from paper_1902_08018_b200.executor import FieldStep
    out = []
    for spec_ in [s.strip() for s in args.variants.split(",") if s.strip()]:
        try:
            if spec_ == "exact":
                if args.evaluation == "exact":
                    continue
                v = FieldStep(fs.A, fs.B, fs.P, streams, args.rows, args.slits, fs.dark, fs.footprint,
                              fs.dose, policy=args.policy, evaluation="exact")
                step_ms, kms = measure_variant(v, args.steps, args.warmup, use_graph)
                vinfo, vmode, veval = info, args.mode, "exact"
                v.plan.close()
                del v
            else:
                a2 = copy.copy(args)
                a2.mode = spec_
                v, _, _, _, vstreams, vinfo = build_field(a2, 1, 0)
                step_ms, kms = measure_variant(v, args.steps, args.warmup, use_graph)
                vmode, veval = spec_, args.evaluation
            kbytes = float(v.plan.bytes_read + v.plan.bytes_written) if spec_ != "exact" else \
                float(fs.plan.bytes_read + fs.plan.bytes_written)
            sb = vinfo["stream_bytes_rank"]
            K = args.slits * args.rows
            out.append({"mode": vmode, "evaluation": veval, "ms_per_step": round(step_ms, 4),
                        "value": round(sb / (step_ms / 1e3) / 1e9, 3), "unit": "GB/s",
                        "gflops": round(3 * K * (2 * args.S - 1) / (step_ms / 1e3) / 1e9, 2),
                        "stream_bytes": sb, "kernel_ms": round(kms, 4),
                        "kernel_bytes": int(kbytes),
                        "frac": round(kbytes / (kms / 1e3) / 1e9 / hbm, 4),
                        "reference_stream_frac": round(sb / (kms / 1e3) / 1e9 / hbm, 4),
                        "packed_bits_per_block": vinfo.get("packed_bits_per_block"),
                        "reference_bits_per_block": vinfo.get("reference_bits_per_block")})
            if spec_ != "exact":
                v.plan.close()
                del v, vstreams
                torch.cuda.empty_cache()
        except Exception as exc:   # a variant never hides the headline line
            out.append({"variant": spec_, "error": f"{type(exc).__name__}: {exc}"})
    return out


def b200_main(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    dev_index = local % torch.cuda.device_count()     # == local on a multi-GPU box
    torch.cuda.set_device(dev_index)
    group = None
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:   # functional check of the N>1 path with several ranks on one GPU
            dist.init_process_group("gloo")
    from paper_1902_08018_b200 import _lib
    _lib.lib()

    fs, spec, ops, mode, streams, info = build_field(args, world, rank)
    plan = fs.plan
    cur = torch.cuda.current_stream()

    use_graph = (world == 1 or args.vector_mode == "replicate") and not args.no_graph
    if use_graph:
        fs.capture()

    def step():
        if use_graph:
            fs.replay()
        else:
            fs.step_local()
        if world > 1:
            fs.gather()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    fs.check()

    # ---- timed region: K steps, per-step events -----------------------------
    clocks = Clocks(dev_index)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev[0].record(cur)
    for i in range(args.steps):
        step()
        ev[i + 1].record(cur)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    fs.check()

    # ---- dominant kernel alone (fused decode+GEMV plan launch), right after
    # the timed steps (before the long latency sample heats the board) -------
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nk = max(3, args.steps // 2)
    plan.launch(fs.status)
    torch.cuda.synchronize()
    k0.record(cur)
    for _ in range(nk):
        plan.launch(fs.status)
    k1.record(cur)
    torch.cuda.synchronize()
    kernel_ms = k0.elapsed_time(k1) / nk

    # ---- latency sample: >= 1000 back-to-back steps, per-step events ---------
    lat_ms = list(step_ms)
    if args.latency_steps > 0:
        evl = [torch.cuda.Event(enable_timing=True) for _ in range(args.latency_steps + 1)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evl[0].record(cur)
        for i in range(args.latency_steps):
            step()
            evl[i + 1].record(cur)
        torch.cuda.synchronize()
        lat_ms = [evl[i].elapsed_time(evl[i + 1]) for i in range(args.latency_steps)]
        fs.check()

    # ---- e2e through the public API with host buffers ------------------------
    T = spec.T
    u_host = torch.from_numpy((ops.B * 0 + 1e-3).astype(np.float32)).pin_memory()
    out_rows = fs.gathered.numel() if world > 1 else fs.local.numel()
    d_host = torch.empty(out_rows, dtype=torch.float32).pin_memory()
    from paper_1902_08018_b200.thermal import csr_matvec

    def e2e_step():
        fs.u.copy_(u_host, non_blocking=True)
        fs.status.fill_(-1)
        if world == 1 or args.vector_mode == "replicate" or rank == 0:
            csr_matvec(fs.A, fs.T, fs.B, fs.u, out=fs.T_next)
            csr_matvec(fs.P, fs.T_next, out=fs.S)
            fs.T.copy_(fs.T_next)
        if world > 1 and args.vector_mode == "broadcast":
            dist.broadcast(fs.S, src=0)
        fs.products()
        if world > 1:
            fs.gather()
            d_host.copy_(fs.gathered, non_blocking=True)
        else:
            d_host.copy_(fs.local, non_blocking=True)
        cur.synchronize()

    for _ in range(2):
        e2e_step()
    e2e_drain = None
    if world == 1 and use_graph:
        # The same API calls as a real-time loop issues them: step k's input
        # is copied from pinned host memory on a copy stream while step k - 1
        # computes (two device input buffers), step k runs as one CUDA graph
        # (thermal update, interpolation, fused products, result copy to
        # pinned host) and the host waits for step k - 1's result.
        u_dev = [fs.u, torch.empty_like(fs.u)]
        d_pair = [d_host, torch.empty_like(d_host).pin_memory()]

        def e2e_body(b):
            fs.status.fill_(-1)
            csr_matvec(fs.A, fs.T, fs.B, u_dev[b], out=fs.T_next)
            csr_matvec(fs.P, fs.T_next, out=fs.S)
            fs.T.copy_(fs.T_next)
            fs.products()
            d_pair[b].copy_(fs.local, non_blocking=True)

        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            e2e_body(0)
        cur.wait_stream(side)
        torch.cuda.synchronize()
        g_pair = []
        for b in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                e2e_body(b)
            g_pair.append(g)
        copy_stream = torch.cuda.Stream()
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        st = {"k": 0}

        def h2d(b):   # step input into buffer b, once the step that last read it is done
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(ev_done[b])
                u_dev[b].copy_(u_host, non_blocking=True)
                ev_in[b].record(copy_stream)

        for b in range(2):
            ev_done[b].record(cur)
        h2d(0)

        def e2e_step():
            k = st["k"]
            b = k & 1
            h2d(b ^ 1)                     # step k + 1's input, overlapping step k
            cur.wait_event(ev_in[b])
            g_pair[b].replay()
            ev_done[b].record(cur)
            if k > 0:
                ev_done[b ^ 1].synchronize()   # step k - 1's result is on the host
            st["k"] = k + 1

        def e2e_drain():
            ev_done[(st["k"] - 1) & 1].synchronize()

        for _ in range(2):
            e2e_step()
        e2e_drain()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e0.record(cur)
    for _ in range(args.steps):
        e2e_step()
    if e2e_drain is not None:
        e2e_drain()
    e1.record(cur)
    torch.cuda.synchronize()
    e2e_ms = max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)) / args.steps

    # ---- reduce over ranks -------------------------------------------------
    stats = torch.tensor([total_ms, e2e_ms, kernel_ms, float(info["stream_bytes_rank"]),
                          float(plan.bytes_read + plan.bytes_written) if plan else 0.0],
                         dtype=torch.float64, device="cuda")
    per_step = torch.tensor(lat_ms, dtype=torch.float64, device="cuda")
    if world > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        dist.all_reduce(per_step, op=dist.ReduceOp.MAX)
        total_ms, e2e_ms, kernel_ms = mx[0].item(), mx[1].item(), mx[2].item()
        job_bytes, kernel_bytes = sm[3].item(), mx[4].item()
    else:
        job_bytes, kernel_bytes = float(info["stream_bytes_rank"]), stats[4].item()
    lat_ms = per_step.cpu().tolist()

    # ---- CPU baseline beside it (rank 0, N=1) --------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tmp = tempfile.mkdtemp()
        paths = make_cpu_samples(args, tmp)
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        reps = max(1, (5 * cores) // 6)          # ~2.5 chunks per core: 10-30 core-seconds
        v, wall, cores, kind, per, _ = run_cpu_leg(paths, reps)
        pb = [int(np.load(pth)["payload"].size) for pth in paths]
        cpu = {"value": round(v, 6), "unit": "GB/s", "cores": cores, "kind": kind,
               "value_1core": round(statistics.mean(pb) / per / 1e9, 6),
               "cpu_model": cpu_model(),
               "sample": f"{3 * reps} chunks of {args.rows}x{args.cpu_sample_cols} "
                         f"({args.mode}), reference codec.decompress + mpgemv.gemv(mixed, sequential); "
                         f"{wall:.1f}s wall; value_1core: the median chunk on one core"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    pk, pk_kind = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    variants = run_variants(args, fs, streams, info, use_graph, hbm) if world == 1 else []
    K = args.slits * args.rows
    flops = 3 * K * (2 * args.S - 1)
    decoded_bytes = 3 * K * args.S * 4
    steps_s = total_ms / 1e3
    value = job_bytes * args.steps / steps_s / 1e9
    achieved = kernel_bytes / (kernel_ms / 1e3) / 1e9
    traffic = None
    instr = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tj = json.load(fh)
        for e in (tj if isinstance(tj, list) else [tj]):
            if (e.get("mode") == args.mode and e.get("evaluation") == args.evaluation
                    and e.get("layout", "reference") == args.layout
                    and e.get("slits", 52) == args.slits and e.get("S", 256000) == args.S):
                traffic = e.get("dram_bytes_per_launch")
                if "thread_instr_per_block" in e:
                    # instruction roofline: the SM issue budget per block
                    # at HBM speed is 128 lane-instr/clk * clk / (blocks/s at peak);
                    # a block is 16 bytes at FixedRate(8), fewer in variable modes
                    bpb = kernel_bytes / e.get("blocks_per_launch", kernel_bytes / 16)
                    budget = 128 * 148 * 1.965e9 / (hbm * 1e9 / bpb)
                    instr = {"thread_instr_per_block": e["thread_instr_per_block"],
                             "budget_at_hbm_peak": round(budget, 1),
                             "alu_pipe_pct": e.get("alu_pipe_pct"),
                             "issue_active_pct": e.get("issue_active_pct"),
                             "source": "ncu --set full (profiles/r2_ncu_summary.md, profiles/ncu_traffic.json)"}
    except Exception:
        pass
    p50 = statistics.median(lat_ms)
    p99 = sorted(lat_ms)[min(len(lat_ms) - 1, int(0.99 * len(lat_ms)))]
    # source term, 2 CSR products, the fused kernel; the vector prologue
    # (U = G^T v, or v padded for the packed exact evaluation); the packed
    # layout's band combine
    packed = args.layout == "packed"
    launches_per_step = 4 + (1 if args.evaluation == "coefficient" or packed else 0) + (1 if packed else 0)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": (("f32 coefficient-domain products, f64 accumulate" if args.evaluation == "coefficient"
                   else "f32 products, f64 accumulate") if args.policy == "mixed" else args.policy),
        "data": "synthetic (reference smooth-C formula model.py:252-268, seed 7); "
                f"{info['distinct_per_axis']} distinct slits/axis",
        "config": workload_config(args, world),
        "impl_config": {"evaluation": args.evaluation, "layout": args.layout,
                        "vector_mode": args.vector_mode if world > 1 else None,
                        "cuda_graph": use_graph, "index_kind": info["index_kind"]},
        "gflops": round(flops * args.steps / steps_s / 1e9, 2),
        "decoded_gbs": round(decoded_bytes * args.steps / steps_s / 1e9, 2),
        "per_gpu_gbs": round(value / world, 3),
        "latency_ms": {"p50": round(p50, 4), "p99": round(p99, 4), "max": round(max(lat_ms), 4),
                       "samples": len(lat_ms),
                       "deadline": DEADLINE_MS, "deadline_met": max(lat_ms) <= DEADLINE_MS},
        "e2e": {"value": round(job_bytes / (e2e_ms / 1e3) / 1e9, 3), "unit": "GB/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": T * 4,
                "d2h_bytes_per_step": out_rows * 4,
                "issue": "one CUDA graph per step; each step's input copied from pinned host on a "
                         "copy stream while the previous step computes; the host waits for every "
                         "step's result" if world == 1 and use_graph
                         else "eager API calls, host waits for each result"},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "hbm", "kernel": "k_pk_gemv2 + k_pk_combine" if args.layout == "packed" else "k_decode_gemv",
                     "bytes": ("tile-packed copy read by the launch (body + segment headers + "
                               "exception list) + vector + output" if args.layout == "packed" else
                               "WHFZ payload + device index + vector + output"),
                     "reference_stream_gbs": round(job_bytes / (kernel_ms / 1e3) / 1e9, 2),
                     "reference_stream_frac": round(job_bytes / (kernel_ms / 1e3) / 1e9 / hbm, 4),
                     "achieved": round(achieved, 2),
                     "peak": hbm, "peak_kind": f"{pk_kind} hbm_gbs (burst copy)", "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "bytes_per_launch": int(kernel_bytes), "kernel_ms": round(kernel_ms, 4),
                     "share_of_step": round(kernel_ms / (total_ms / args.steps), 3),
                     "instruction_roofline": instr},
        "variants": variants,
        "cpu_baseline": cpu,
        "clocks": clk,
        "setup": info,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        return reference_main(args, world, rank)
    return b200_main(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
