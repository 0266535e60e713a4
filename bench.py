#!/usr/bin/env python
"""Benchmark: corrected-key Mbps of the batched quantized LDPC syndrome decoder on B200.

Workload (BASELINE.json configs[4], "C5"): 65536 frames of the config-3 code (n=51200,
R~0.84, QBER 2%) plus 65536 frames of the config-2 code (n=8192, R=0.5, QBER 8%), split
evenly across ranks by global frame id (strong scaling), max 50 iterations, early stop.
One step = for both workloads: Alice's syndrome, Bob's int8 LLRs, the fused layered
decode, scoring against Alice's key (counters) -- then one NCCL allreduce of the int64
counters when N > 1.  Inputs are synthetic (synth/, seeded BSC frames on seeded QC codes).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload C5|C1|..]

--impl reference times the CPU oracle (the reference arm of this tier; oracle/) on a bounded
sample per step on the host cores and extrapolates to the same workload and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "corrected-key Mbps at QBER 1-8% (1/2/4/8 GPU); % of HBM roofline per iteration"
UNIT = "Mbps"
# The paper's own CPU figures (Table 2): context only -- its codes, frame length and
# workload are unpublished, so no ratio is formed (vs_baseline stays null).
PAPER_CONTEXT = {"value": 57.60, "unit": "Mbps", "hardware": "Intel i7-6700HQ, 4 cores (P:54, P:211)",
                 "also": "122.17 Mbps on an Intel i9-9900K (P:209)", "efficiency": 1.108,
                 "note": "paper's unpublished ~100 kb codes, bi-directional protocol; not this workload"}

WORKLOADS = {"C5": ["C5a", "C5b"], "C1": ["C1"], "C2": ["C2"], "C3": ["C3"],
             "C4": [f"C4@{q:g}" for q in synth.C4_QBERS]}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def shard(F: int, rank: int, world: int) -> tuple[int, int]:
    """Global frame ids [a, b) decoded by `rank` (contiguous, even split)."""
    return rank * F // world, (rank + 1) * F // world


def reduce_counters(counters, world: int):
    """The one collective of the path: SUM all-reduce of the int64 counters."""
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(counters)
    return counters


def payload_bits(w):
    d, p, s = w.rate_adaptive_counts()
    return w.n - p - s


# ------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        t0 = time.time()   # a timed region shorter than nvidia-smi's start-up: take the first sample after it
        while not self.rows and time.time() - t0 < 3.0 and self.proc.poll() is None:
            time.sleep(0.02)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------- oracle arm
def oracle_sample(names, frames_per, nthreads):
    """Decode a bounded sample with the CPU oracle.  Returns per-workload dicts with the
    wall time, frames, corrected frames."""
    import oracle

    out = {}
    for name in names:
        w = synth.workload(name)
        F = frames_per[name]
        x, y, _ = w.gen(0, F, nthreads)
        kind = w.pos_kind()
        oc = oracle.Code(w.shifts(), w.Z)
        syn = oc.syndrome(x)
        t0 = time.perf_counter()
        llr = oc.build_llr(w.qber, y, kind, x)
        r = oc.decode(llr, syn, w.max_iter, w.early_stop, want_state=False, nthreads=nthreads)
        dt = time.perf_counter() - t0
        ok = (r["success"] == 1) & (r["bits"] == x).all(axis=1) if kind is None else (r["success"] == 1) & (
            ((r["bits"] ^ x) & np.packbits(kind == 0, bitorder="little")[None, :]) == 0).all(axis=1)
        out[name] = dict(seconds=dt, frames=F, corrected=int(ok.sum()), iters=float(r["iters"].mean()))
    return out


def extrapolate(names, sample, frames_total):
    """Corrected-key Mbps of the whole step (all workloads, full frame counts) from the sample."""
    bits = 0.0
    secs = 0.0
    for name in names:
        w = synth.workload(name)
        s = sample[name]
        per_frame = s["seconds"] / s["frames"]
        secs += per_frame * frames_total[name]
        bits += (s["corrected"] / s["frames"]) * frames_total[name] * payload_bits(w)
    return bits / secs / 1e6, secs


def default_sample(names, cores):
    per = {}
    for name in names:
        w = synth.workload(name)
        edges_iter = w.max_iter * (w.shifts() >= 0).sum() * w.Z       # worst-case work per frame
        # ~3e7 scalar edge updates per second per core for the plain -O2 oracle
        per_frame_s = edges_iter / 3e7
        per[name] = int(max(cores, min(w.frames, cores * max(1, round(12.0 / per_frame_s)))))
    return per


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    names = WORKLOADS[args.workload]
    cores = host_cores()
    frames_total = {n: synth.workload(n).frames for n in names}
    per = default_sample(names, cores)
    per = {k: max(1, v // 4) for k, v in per.items()}          # ~1 s of CPU per step
    vals, secs = [], []
    for i in range(args.warmup + args.steps):
        s = oracle_sample(names, per, cores)
        v, _ = extrapolate(names, s, frames_total)
        if i >= args.warmup:
            vals.append(v)
            secs.append(sum(x["seconds"] for x in s.values()))
    value = statistics.median(vals)
    sample_desc = ", ".join(f"first {per[n]} frames of {n}" for n in names)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.median(secs),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic", "config": workload_config(args.workload, args.gpus, args.scaling),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample_desc + " per step, extrapolated to the full workload"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_efficiency(name):
    """R20: f = (m - p) / ((n - p - s) h2(q)) of a workload (the reference it is quoted against)."""
    import math

    w = synth.workload(name)
    d, p, s = w.rate_adaptive_counts()
    q = w.qber
    h2 = -q * math.log2(q) - (1 - q) * math.log2(1 - q)
    return (w.m - p) / ((w.n - p - s) * h2)


def workload_config(wl, gpus=1, scaling="strong"):
    """The config dict -- identical in both arms (native and --impl reference)."""
    names = WORKLOADS[wl]
    cfg = {"workload": wl + " = " + " + ".join(
        f"{n}({synth.workload(n).Mb}x{synth.workload(n).Nb} Z={synth.workload(n).Z} n={synth.workload(n).n} "
        f"QBER={synth.workload(n).qber:g} frames={synth.workload(n).frames} T={synth.workload(n).max_iter})"
        for n in names),
        "frames_per_workload": {n: synth.workload(n).frames for n in names},
        "max_iter": {n: synth.workload(n).max_iter for n in names},
        "early_stop": True, "frames_per_group": 4,
        "efficiency_f": {n: round(workload_efficiency(n), 4) for n in names},
        "parallelism": f"frames sharded over {gpus} rank(s), {scaling} scaling",
        "l2": "inputs larger than L2 (C5a LLR alone is 3.4 GB); no flush needed"}
    return cfg


# ------------------------------------------------------------------------------- GPU arm
class NativeEngine:
    """The product: this rank's shard of every workload decoded by libqkdldpc.so on its GPU.
    The rank/step/timing control flow around it (run_ranks) is shared with the CPU test stub
    (tests/bench_stub.py), which is how the multi-rank path is tested without GPUs."""

    backend = "nccl"

    def __init__(self, args, world, rank, local):
        import torch

        import paper_1903_10107_b200 as qkd

        self.torch, self.qkd, self.args = torch, qkd, args
        self.world, self.rank, self.local = world, rank, local
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream()
        self.device_id = self.dev

    def prepare(self):
        torch, qkd, args, dev = self.torch, self.qkd, self.args, self.dev
        world, rank = self.world, self.rank
        nthreads = max(1, host_cores() // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world))))
        W = []
        for name in WORKLOADS[args.workload]:
            w = synth.workload(name)
            F = w.frames * (world if args.scaling == "weak" else 1)   # weak: BASELINE's count on every rank
            a, b = shard(F, rank, world)
            t0 = time.perf_counter()
            x, y, _ = w.gen(a, b - a, nthreads)
            kind = w.pos_kind()
            code = qkd.QCCode(w.shifts(), w.Z, kind)
            Fr = b - a
            st = dict(name=name, w=w, code=code, F=Fr, x_host=x, y_host=y,
                      x=torch.from_numpy(x).to(dev), y=torch.from_numpy(y).to(dev))
            st["syn"] = torch.empty((Fr, code.mb8), dtype=torch.uint8, device=dev)
            st["llr"] = torch.empty((Fr, code.n), dtype=torch.int8, device=dev)
            st["ws"] = torch.empty(code.workspace_bytes(Fr), dtype=torch.uint8, device=dev)
            st["out"] = dict(bits=torch.empty((Fr, code.nb8), dtype=torch.uint8, device=dev),
                             iters=torch.empty(Fr, dtype=torch.int32, device=dev),
                             success=torch.empty(Fr, dtype=torch.uint8, device=dev))
            st["info"] = code.launch_info(Fr)
            st["known"] = st["x"] if kind is not None else None
            st["ev"] = []
            log(f"[rank {rank}] {name}: frames [{a},{b}) generated in {time.perf_counter() - t0:.1f}s, "
                f"launch {st['info']}")
            W.append(st)
        self.W = W
        self.launches_per_step = 4 * len(W)   # syndrome, LLR, decode, score per workload
        return [s["name"] for s in W]

    def zeros(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.int64, device=self.dev)

    def step(self, counters, record):
        torch, stream = self.torch, self.stream
        counters.zero_()
        for i, s in enumerate(self.W):
            code = s["code"]
            code.syndrome(s["x"], out=s["syn"])                       # Alice (a3)
            code.build_llr(s["w"].qber, s["y"], s["known"], out=s["llr"])   # Bob (a2)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            code.decode(s["llr"], s["syn"], s["w"].max_iter, True, counters=counters[i], workspace=s["ws"],
                        out=s["out"])                                  # a4-a8
            e1.record(stream)
            if record:
                s["ev"].append((e0, e1))
            code.score(s["out"]["bits"], s["x"], s["out"]["success"], counters=counters[i])   # a9

    def sync(self):
        self.torch.cuda.synchronize()

    def clear_records(self):
        for s in self.W:
            s["ev"].clear()

    def start_timer(self):
        self.t_start = self.torch.cuda.Event(enable_timing=True)
        self.t_end = self.torch.cuda.Event(enable_timing=True)
        self.clk = ClockSampler(self.local)
        self.clk.start()
        self.t_start.record(self.stream)

    def stop_timer(self):
        """Device time of the timed steps on this rank (ms), taken after a synchronize."""
        self.t_end.record(self.stream)
        self.torch.cuda.synchronize()
        self.clocks = self.clk.stop()
        return self.t_start.elapsed_time(self.t_end)

    def decode_ms(self, i):
        return statistics.mean(a.elapsed_time(b) for a, b in self.W[i]["ev"])

    def payload_bits(self, i):
        return payload_bits(self.W[i]["w"])

    def extras(self, c, ms_total, per_wl):
        """roofline, e2e, cpu_baseline: the GPU-specific parts of the line."""
        torch, args, world, rank = self.torch, self.args, self.world, self.rank
        W = self.W
        peak, peak_kind = peaks()
        for i, s in enumerate(W):
            code = s["code"]
            # this rank's algorithmic bytes: per frame-iteration 2|E| (every int8
            # message read and rewritten once), per frame once n + ceil(m/8) + ceil(n/8) + 5.
            frames_g, iters_g = int(c[i, 0]), int(c[i, 4])
            frac = s["F"] / max(1, frames_g)
            b_it = 2 * code.n_edges
            once = code.n + code.mb8 + code.nb8 + 5
            bytes_rank = frac * (iters_g * b_it + frames_g * once)
            t = per_wl[s["name"]]["decode_ms"]
            per_wl[s["name"]].update(alg_bytes=bytes_rank, alg_GBps=bytes_rank / (t / 1000) / 1e9, launch=s["info"])
        dom = max(per_wl, key=lambda k: per_wl[k]["decode_ms"])
        achieved = per_wl[dom]["alg_GBps"]
        traffic, ncu = None, None
        clocks = self.clocks
        try:   # from the committed ncu capture of this launch (profiles/traffic.json)
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tj = json.load(f)
            if tj.get("workload", "C5a") != dom:   # the capture is of another workload's launch
                raise LookupError
            traffic = tj.get("decode_dram_bytes_per_launch")
            ncu = dict(tj.get("ncu") or {}, source=tj.get("source"))
            if world > 1:   # the capture is of the 1-GPU launch (all frames of the workload)
                traffic = None
            elif ncu.get("warp_instructions") and clocks and clocks.get("sm_mhz"):
                # SURVEY §8(d) co-bound: integer-issue fraction inst_executed / (SMs * 4 * clk * t), with the
                # captured launch's instruction count (deterministic for this workload) and the live time/clock
                sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
                ncu["int_issue_frac_live"] = ncu["warp_instructions"] / (
                    sms * 4 * clocks["sm_mhz"] * 1e6 * per_wl[dom]["decode_ms"] / 1000)
        except Exception:
            pass
        sec_per_step = ms_total / 1000.0 / args.steps
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "ncu": ncu,
                    "kernel": f"decode_kernel ({dom} launch: {per_wl[dom]['decode_ms']:.1f} ms of "
                              f"{1000 * sec_per_step:.1f} ms per step)",
                    "algorithmic_bytes_per_launch": per_wl[dom]["alg_bytes"],
                    "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs"}
        e2e = run_e2e(args, W, world, rank, self.dev)   # end to end through the C ABI, host buffers
        cpu = None
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            names = [s["name"] for s in W]
            cores = host_cores()
            per = default_sample(names, cores)
            t0 = time.perf_counter()
            sm = oracle_sample(names, per, cores)
            v, _ = extrapolate(names, sm, {n: synth.workload(n).frames for n in names})
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": ", ".join(f"first {per[n]} frames of {n}" for n in names)
                   + f" ({time.perf_counter() - t0:.1f}s of CPU work), extrapolated to the full workload",
                   "cpu_model": cpu_model()}
            # single-thread figure beside the all-core one (small sample, ~2-4 s)
            per1 = {n: max(1, per[n] // max(1, cores) // 4) for n in names}
            sm1 = oracle_sample(names, per1, 1)
            cpu["single_thread_value"], _ = extrapolate(names, sm1, {n: synth.workload(n).frames for n in names})
            cpu["single_thread_sample"] = ", ".join(f"first {per1[n]} frames of {n}" for n in names)
        return {"roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks, "dtype": "int8",
                "paper_context": PAPER_CONTEXT}


def load_engine(spec):
    """--engine module:Class (default: the native engine); the tests plug in a CPU stub."""
    if not spec:
        return NativeEngine
    import importlib

    mod, cls = spec.split(":")
    return getattr(importlib.import_module(mod), cls)


def run_ranks(args, engine_cls):
    """One process per GPU (rank): prepare this rank's shards, W untimed steps, a barrier, K timed
    steps, a barrier; time = MAX over ranks; counters = SUM over ranks (the path's one collective).
    Rank 0 prints the JSON line."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a wrong n_gpus")
        return 2
    eng = engine_cls(args, world, rank, local)
    import torch
    import torch.distributed as dist

    if world > 1:
        kw = {"device_id": eng.device_id} if getattr(eng, "device_id", None) is not None else {}
        dist.init_process_group(eng.backend, **kw)
    names = eng.prepare()
    counters = eng.zeros((len(names), 5))
    for _ in range(args.warmup):
        eng.step(counters, False)
        reduce_counters(counters, world)
    eng.sync()
    eng.clear_records()
    if world > 1:
        dist.barrier()
    eng.sync()
    eng.start_timer()
    for _ in range(args.steps):
        eng.step(counters, True)
        reduce_counters(counters, world)                              # a9: the only collective
    ms_local = eng.stop_timer()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([ms_local], dtype=torch.float64, device=counters.device)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_total = float(ms.item())
    c = counters.cpu().numpy()      # last step (identical every step)

    # ---- metric: corrected = syndrome matched and no payload bit error
    corrected_bits = sum(int(c[i, 1] - c[i, 3]) * eng.payload_bits(i) for i in range(len(names)))
    processed_bits = sum(int(c[i, 0]) * eng.payload_bits(i) for i in range(len(names)))
    sec_per_step = ms_total / 1000.0 / args.steps
    value = corrected_bits / sec_per_step / 1e6
    processed = processed_bits / sec_per_step / 1e6
    per_wl = {}
    for i, name in enumerate(names):
        frames_g = int(c[i, 0])
        d = {"decode_ms": eng.decode_ms(i), "frames": frames_g, "fer": 1 - c[i, 1] / max(1, frames_g),
             "mean_iters": c[i, 4] / max(1, frames_g), "undetected": int(c[i, 3]),
             "frames_with_errors": int(c[i, 2]),
             "corrected_key_mbps": int(c[i, 1] - c[i, 3]) * eng.payload_bits(i) / sec_per_step / 1e6,
             "processed_key_mbps": frames_g * eng.payload_bits(i) / sec_per_step / 1e6}
        try:
            d["efficiency_f"] = workload_efficiency(name)
        except Exception:
            pass
        per_wl[name] = d
    extra = eng.extras(c, ms_total, per_wl)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": extra.pop("dtype", "int8"),
                "data": "synthetic", "config": workload_config(args.workload, args.gpus, args.scaling),
                "processed_key_mbps": processed,
                "frames_total": {name: int(c[i, 0]) for i, name in enumerate(names)},
                "per_workload": per_wl,
                "gpu_launches": eng.launches_per_step * args.steps}
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_gpu(args):
    return run_ranks(args, load_engine(args.engine))


def run_e2e(args, W, world, rank, dev):
    import torch
    import torch.distributed as dist

    steps = max(1, min(args.steps, 3))
    for s in W:
        code = s["code"]
        Fr = s["F"]
        s["pin_y"] = torch.from_numpy(s["y_host"]).pin_memory()
        s["pin_known"] = torch.from_numpy(s["x_host"]).pin_memory() if s["known"] is not None else None
        s["pin_syn"] = s["syn"].cpu().pin_memory()
        s["pin_out"] = (torch.empty((Fr, code.nb8), dtype=torch.uint8).pin_memory(),
                        torch.empty(Fr, dtype=torch.int32).pin_memory(),
                        torch.empty(Fr, dtype=torch.uint8).pin_memory())
        s["dbuf"] = torch.empty(code.reconcile_device_bytes(Fr), dtype=torch.uint8, device=dev)
    h2d = sum(s["F"] * (s["code"].nb8 * (2 if s["known"] is not None else 1) + s["code"].mb8) for s in W) * world
    d2h = sum(s["F"] * (s["code"].nb8 + 5) for s in W) * world

    def one():
        for s in W:
            s["code"].reconcile_host(s["w"].qber, s["pin_y"], s["pin_syn"], s["w"].max_iter, True,
                                     known_bits=s["pin_known"], device_buffer=s["dbuf"], out=s["pin_out"])

    one()   # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = torch.tensor([(time.perf_counter() - t0) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    corrected = 0
    for s in W:
        bits, iters, succ = (t.numpy() for t in s["pin_out"])
        kind = s["w"].pos_kind()
        diff = bits ^ s["x_host"]
        if kind is not None:
            diff &= np.packbits(kind == 0, bitorder="little")[None, :]
        ok = (succ == 1) & (diff == 0).all(axis=1)
        corrected += int(ok.sum()) * payload_bits(s["w"])
    cb = torch.tensor([corrected], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(cb)
    return {"value": float(cb.item()) / float(dt.item()) / 1e6, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "note": "qkd_reconcile_host per workload: H2D(Bob bits, syndrome) + LLR + decode + D2H(bits, iters, "
                    "success) on pinned host buffers, host wall clock, max over ranks"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default, BASELINE configs[4]: 65536 frames per workload in total, split "
                         "across ranks) or weak (65536 frames per workload on every rank)")
    ap.add_argument("--engine", default="", help=argparse.SUPPRESS)   # module:Class (tests' CPU stub)
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


def relaunch(n):
    """`bench.py --gpus N` without a launcher: re-run this command as N ranks (one process per GPU)
    under torch.distributed.run on this node; rank 0's line is the output."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log("bench.py: launching " + " ".join(cmd[1:]))
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
