#!/usr/bin/env python
"""Benchmark of the Wire-Cell signal-simulation hot path (raster + scatter + FFT-conv).

Metric (BASELINE.json): depositions/s (and events/s) for raster + scatter +
FFT-convolution on a MicroBooNE-scale event (configs[1]): 100k depositions on
straight 3D tracks projected onto U/V (induction, 2400 wires) and W
(collection, 3456 wires) planes x 9600 ticks, pad 100/100, pitch 3 mm, tick
0.5 us, fluctuation off, field + electronics response. One step = one event.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  python bench.py --workload sigproc ...   (the paper's Listing 1 chain, §8(f))
  python bench.py --workload c4 ...        (configs[3]: ProtoDUNE-SP 6-APA event, 36 (face, plane) units)
  python bench.py --workload c5 ...        (configs[4]: 64-event batches, 1k-1M depos/event sweep)

N > 1 runs one rank per GPU (torchrun; `--gpus N` without torchrun's
environment re-launches itself under torch.distributed.run). event: weak
scaling, every rank simulates its own events; c4 / c5: strong scaling, the
36 units / 64 events of a step are sharded over the ranks (LPT / round
robin). No data-path collective; value = all ranks' depositions / max-over-
ranks device time.

Timing: CUDA events on the library's stream around exactly K steps, barrier +
synchronize on both sides, max over ranks. Inputs rotate over 10 distinct
pre-generated events (144 MB of depos > 126 MB L2; every step also writes
347 MB of frames). `e2e` measures the same workload through the
reference-facing host-buffer call, ws_run_events (run_simulation's output:
SimResult::adc, digitized codes in uint16): pinned depos H2D and the ADC
frames D2H inside the timed region, pipelined.

--impl reference times the reference's own CPU implementation (the
unmodified library compiled into oracle/_ref) on the host cores, one plane of
the event per step (rotating U, V, W), response kernels built once outside
the timed region; events/s = 1 / (3 x mean plane time).
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_DEPOS = 100_000
N_EVENTS_ROTATE = 10
WORKLOAD = "microboone_event: 100k depos, U/V/W 2400/2400/3456 wires x 9600 ticks, pad 100/100, fluct off"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every ~2 ms while the
    timed region runs (nvidia-smi's 100 ms floor would miss short regions)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:  # no NVML: report unsampled
            self.nvml = None
        return self

    def _sample(self):
        p = self.nvml
        sm = p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM)
        try:
            r = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = p.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, r))

    def _run(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                break
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.thread.join(timeout=1)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s for s, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("WS_BENCH_SHARED_GPU") == "1":
        # test mode for the multi-rank path on a box with fewer GPUs than
        # ranks: ranks share devices (use WS_BENCH_BACKEND=gloo: NCCL refuses
        # two ranks on one GPU); never for a reported number
        import torch
        local = local % max(1, torch.cuda.device_count())
    return world, rank, local


def init_dist(local: int):
    import torch
    import torch.distributed as dist
    backend = os.environ.get("WS_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return backend


def relaunch_distributed(n: int) -> int:
    """`--gpus N` without a torchrun environment: run this script under
    torch.distributed.run with N ranks (one per GPU) and pass its output through."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def make_events(rank: int):
    from paper_2104_08265_b200.workloads import microboone_event
    return [microboone_event(N_DEPOS, seed=1000 * rank + e + 1) for e in range(N_EVENTS_ROTATE)]


def cpu_reference_plane_times(events, planes_idx, workers):
    """Time the unmodified reference (oracle/_ref) fluctuation-off path, one plane
    per step; each plane's response kernel is built once (cached, reported apart)."""
    from oracle.oracle import Reference, build_ref, make_grid, make_response, ref_available
    from paper_2104_08265_b200.workloads import microboone_grids
    if not ref_available():
        build_ref()
    ref = Reference()
    grids, resps = microboone_grids()
    cache = {}
    out = []
    for step, pi in enumerate(planes_idx):
        if pi not in cache:
            g, r = grids[pi], resps[pi]
            og = make_grid(g.n_wires, g.n_ticks, g.pad_wires, g.pad_ticks, g.pitch, g.tick)
            orr = make_response(r.plane_kind, r.field_sigma_t, r.shaper_peaking, r.shaper_order, r.gain)
            cache[pi] = ref.plane(og, orr)
        t = cache[pi].time_fluct_off(events[step % len(events)][pi], workers=workers)
        out.append(dict(plane=pi, sample_s=t["sample_s"], scatter_s=t["scatter_s"], convolve_s=t["convolve_s"],
                        build_response_s=cache[pi].build_s))
    return out


def cpu_baseline_event(events, cores):
    """The GPU arm's cpu_baseline: the unmodified reference on ALL three planes
    of one event at `cores` threads (stage breakdown per plane), plus the U
    plane at one worker; build_response excluded (cached, reported)."""
    t_all = cpu_reference_plane_times(events, [0, 1, 2], cores)
    t_one = cpu_reference_plane_times(events, [0], 1)[0]
    stages = {k: sum(x[k] for x in t_all) for k in ("sample_s", "scatter_s", "convolve_s")}
    ev_s = sum(stages.values())
    return {"value": N_DEPOS / ev_s, "unit": "depos/s", "cores": cores, "kind": "reference",
            "sample": f"all three planes (U, V, W) of one 100k-depo event through the unmodified reference at "
                      f"{cores} threads, build_response excluded (cached); stage seconds summed over planes",
            "event_s": ev_s, "stages_s": stages,
            "per_plane_s": [round(x["sample_s"] + x["scatter_s"] + x["convolve_s"], 4) for x in t_all],
            "build_response_s": [round(x["build_response_s"], 2) for x in t_all],
            "workers_1": {"plane": "U", "plane_s": t_one["sample_s"] + t_one["scatter_s"] + t_one["convolve_s"],
                          "stages_s": {k: t_one[k] for k in ("sample_s", "scatter_s", "convolve_s")},
                          "depos_per_s_event_equiv": N_DEPOS / (3 * (t_one["sample_s"] + t_one["scatter_s"] +
                                                                      t_one["convolve_s"]))}}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    from paper_2104_08265_b200.workloads import microboone_event
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    ev = [microboone_event(N_DEPOS, seed=1)]
    seq = [(i % 3) for i in range(args.warmup + args.steps)]
    t = cpu_reference_plane_times(ev, seq, cores)
    timed = t[args.warmup:]
    plane_s = [x["sample_s"] + x["scatter_s"] + x["convolve_s"] for x in timed]
    mean_plane = sum(plane_s) / len(plane_s)
    ev_s = 3 * mean_plane
    value = N_DEPOS / ev_s
    line = {
        "impl": "reference", "metric": "depositions_per_sec", "value": value, "unit": "depos/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_plane * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic line tracks",
        "config": {"workload": WORKLOAD, "events_per_sec": 1.0 / ev_s, "step": "one plane (U,V,W rotating)",
                   "workers": cores},
        "cpu_baseline": {"value": value, "unit": "depos/s", "cores": cores, "kind": "reference",
                         "sample": "one plane per step rotating U/V/W of a 100k-depo event; build_response cached"},
        "e2e": {"value": value, "unit": "depos/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def pipe_summary(kernel: str):
    """North star: rasterization (k_sample_off's erfc + FMA work) as a fraction
    of the FP32 / SFU (XU) peaks; % of peak over active cycles from the
    committed ncu capture (inst-executed rates per pipe)."""
    p = profile_facts(kernel).get("pipes") or {}
    keys = {"fp32_fma": "inst_fma", "sfu_xu": "inst_xu", "fp64": "inst_fp64", "alu": "inst_alu", "lsu": "inst_lsu"}
    out = {k: round(p[v] / 100.0, 4) for k, v in keys.items() if v in p}
    if out:
        out["kernel"] = kernel
        out["source"] = profile_facts(kernel).get("source")
    return out or None


def profile_facts(kernel: str):
    """Per-launch counters of `kernel` from the committed ncu captures
    (profiles/traffic_<kernel>.json): DRAM bytes, warp instructions, pipes."""
    prof = ROOT / "profiles" / f"traffic_{kernel}.json"
    return json.loads(prof.read_text()) if prof.exists() else {}


SP_ROWS, SP_COLS, SP_PAD, SP_OUT = 960, 6000, 80, 800
SP_WORKLOAD = (f"sigproc_chain: {SP_ROWS} signals x {SP_COLS} samples (complex128 spectra), complex filter, "
               f"block rows [{SP_PAD}, {SP_PAD + SP_OUT}), per-row medians")


def sigproc_inputs(seed: int):
    """Spectra of real waveforms (Hermitian rows) and a real, even low-pass
    filter, as in Listing 1's ROI filtering, so the output is real."""
    rng = np.random.default_rng(seed)
    data = np.fft.fft(rng.normal(size=(SP_ROWS, SP_COLS)), axis=1)
    k = np.arange(SP_COLS)
    filt = np.exp(-(np.minimum(k, SP_COLS - k) / 1000.0) ** 2).astype(np.complex128)
    return data, filt


def sigproc_reference_times(steps: int, workers: int):
    """The unmodified reference's sigproc_chain (oracle/_ref), one batch per step."""
    from oracle.oracle import Reference, build_ref, ref_available
    if not ref_available():
        build_ref()
    ref = Reference()
    data, filt = sigproc_inputs(1)
    return [ref.sigproc_chain(data, filt, SP_PAD, SP_OUT, workers=workers)[3] for _ in range(steps)]


def run_sigproc(args, world, rank, local):
    """--workload sigproc: the paper's Listing 1 chain.
    One step = one batch of 960 x 6000 signals; device-resident inputs rotate
    over two batches (184 MB > 126 MB L2)."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    bytes_per_batch = SP_ROWS * SP_COLS * 16 + SP_OUT * SP_COLS * 8 + SP_OUT * 8
    if args.impl == "reference":
        if rank != 0:
            return
        t = sigproc_reference_times(args.warmup + args.steps, cores)[args.warmup:]
        mean = sum(t) / len(t)
        value = SP_ROWS / mean
        print(json.dumps({
            "impl": "reference", "metric": "signals_per_sec", "value": value, "unit": "signals/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (spectra of seeded normal waveforms, Gaussian low-pass)", "config": {"workload": SP_WORKLOAD, "workers": cores},
            "cpu_baseline": {"value": value, "unit": "signals/s", "cores": cores, "kind": "reference",
                             "sample": "one full batch per step"},
            "e2e": {"value": value, "unit": "signals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
            flush=True)
        return
    import torch
    import torch.distributed as dist
    from paper_2104_08265_b200 import Context, sigproc_chain, sigproc_chain_device
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    batches = [sigproc_inputs(100 * rank + i + 1) for i in range(2)]
    dd = [torch.from_numpy(b[0]).cuda() for b in batches]
    fd = [torch.from_numpy(b[1]).cuda() for b in batches]
    blk = torch.empty((SP_OUT, SP_COLS), dtype=torch.float64, device="cuda")
    med = torch.empty(SP_OUT, dtype=torch.float64, device="cuda")

    def step(i):
        sigproc_chain_device(ctx, dd[i % 2], SP_ROWS, SP_COLS, fd[i % 2], blk, med, pad_rows=SP_PAD,
                             out_rows=SP_OUT)

    for i in range(args.warmup):
        step(i)
    ctx.synchronize()
    l0 = ctx.launch_count
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(args.steps):
            step(i)
        end.record(stream)
        ctx.synchronize()
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = ctx.launch_count - l0
    kernel_ms = ms / args.steps
    value = world * SP_ROWS * args.steps / (ms * 1e-3)
    peak, peak_kind = peaks()
    achieved = bytes_per_batch / (kernel_ms * 1e-3) / 1e9
    prof = ROOT / "profiles" / "traffic_k_sigproc.json"
    traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch") if prof.exists() else None
    e2e = None
    if not args.no_e2e:  # host buffers (pinned), pipelined H2D / chain / D2H inside ws_sigproc_chain
        pin_in = torch.from_numpy(batches[0][0]).pin_memory().numpy()
        pin_blk = torch.empty((SP_OUT, SP_COLS), dtype=torch.float64).pin_memory().numpy()
        pin_med = torch.empty(SP_OUT, dtype=torch.float64).pin_memory().numpy()
        for _ in range(2):
            sigproc_chain(pin_in, batches[0][1], SP_PAD, SP_OUT, ctx=ctx, block_out=pin_blk, medians_out=pin_med)
        k = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(k):
            sigproc_chain(pin_in, batches[0][1], SP_PAD, SP_OUT, ctx=ctx, block_out=pin_blk, medians_out=pin_med)
        e2e_s = (time.perf_counter() - t0) / k
        e2e = {"value": world * SP_ROWS / e2e_s, "unit": "signals/s",
               "h2d_bytes_per_step": SP_ROWS * SP_COLS * 16 + SP_COLS * 16,
               "d2h_bytes_per_step": SP_OUT * SP_COLS * 8 + SP_OUT * 8, "steps": k, "ms_per_step": e2e_s * 1e3}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t = sigproc_reference_times(2, cores)
        cpu = {"value": SP_ROWS / min(t), "unit": "signals/s", "cores": cores, "kind": "reference",
               "sample": "one 960 x 6000 batch through the unmodified reference sigproc_chain, best of 2"}
    if rank == 0:
        print(json.dumps({
            "metric": "signals_per_sec", "value": value, "unit": "signals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": kernel_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (spectra of seeded normal waveforms, Gaussian low-pass)",
            "config": {"workload": SP_WORKLOAD, "l2": "inputs rotate over 2 batches (184 MB > 126 MB L2)",
                       "parallelism": f"batch-sharded x{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": "k_sigproc", "kernel_ms": kernel_ms,
                         "algorithmic_bytes": bytes_per_batch, "peak_kind": peak_kind},
            "clocks": clocks.summary(), "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_reference_units(units, workers):
    """The unmodified reference's fluctuation-off path on (grid, response,
    depos) units, one plane run each (response built once per geometry,
    excluded): seconds per unit (sample + scatter + convolve)."""
    from oracle.oracle import Reference, build_ref, make_grid, make_response, ref_available
    if not ref_available():
        build_ref()
    ref = Reference()
    cache, out = {}, []
    for g, r, d in units:
        key = (g.n_wires, g.n_ticks, g.pad_wires, g.pad_ticks, g.pitch, r.plane_kind, tuple(r.wire_weights))
        if key not in cache:
            og = make_grid(g.n_wires, g.n_ticks, g.pad_wires, g.pad_ticks, g.pitch, g.tick)
            orr = make_response(r.plane_kind, r.field_sigma_t, r.shaper_peaking, r.shaper_order, r.gain,
                                tuple(r.wire_weights))
            cache[key] = ref.plane(og, orr)
        t = cache[key].time_fluct_off(d, workers=workers)
        out.append(t["sample_s"] + t["scatter_s"] + t["convolve_s"])
    return out


C4_DEPOS = 20_000      # per (face, plane) unit
C4_ROTATE = 4          # distinct events (4 x 36 units x 20k x 48 B = 138 MB of depos > L2)
C5_EVENTS = 64
C5_ROTATE = 8          # distinct events per size (rotating over the 64 of a step)
C5_SIZES = (1_000, 10_000, 100_000, 1_000_000)


C1_DEPOS = 10_000
C1_IMPACTS = 10


def c1_plane():
    """configs[0]: one plane of 480 wires x 6000 ticks (pad 100/100, pitch 5 mm,
    tick 0.5 us: 680 x 6200 padded), collection response."""
    from paper_2104_08265_b200 import GridSpec, ResponseParams
    return GridSpec(n_wires=480, n_ticks=6000, pad_wires=100, pad_ticks=100, pitch=5.0, tick=0.5), \
        ResponseParams(plane_kind="collection")


def workload_desc(args):
    if args.workload == "c1":
        return (f"single plane (configs[0]): {C1_DEPOS} line-track depos, 480 wires x 6000 ticks (680 x 6200 padded), "
                f"{C1_IMPACTS} impacts/pitch (identical per-impact responses: the case the reference pins), "
                f"fluct off")
    if args.workload == "c3":
        return ("microboone_event with fluctuation (configs[2]): 100k depos, U/V/W 2400/2400/3456 wires x 9600 "
                "ticks, exact binomial walk on the shared Philox stream (seed 12345), field + electronics response "
                "(shaper 2 us, order 2, gain 14)")
    if args.workload == "c4":
        return (f"protodune_event (configs[3]): 12 faces x U/V/W (800/800/480 wires) x 6000 ticks, pad 100/100, "
                f"pitch 5 mm, {C4_DEPOS} depos per (face, plane) unit (720k per event), fluct off; 36 units "
                f"LPT-sharded over the ranks")
    if args.workload == "c5":
        return (f"batched events (configs[4]): {C5_EVENTS} MicroBooNE-geometry events of {args.depos} depos per "
                f"step, round-robin over the ranks, fluct off")
    return WORKLOAD


def c3_reference(cores):
    """configs[2] on the CPU: the unmodified reference's run_simulation (it
    always fluctuates; substream mode, the reference's own stream) on the three
    planes of the event at `cores` threads; the time of build_response (rebuilt
    inside every run_simulation call, pipeline.cpp:417) is measured apart and
    subtracted, so the CPU is credited with a cached response."""
    from oracle.oracle import Reference, build_ref, make_grid, make_response, ref_available
    from paper_2104_08265_b200.workloads import microboone_event, microboone_grids
    if not ref_available():
        build_ref()
    ref = Reference()
    grids, resps = microboone_grids()
    ev = microboone_event(N_DEPOS, seed=1)
    total, parts = 0.0, []
    for g, r, d in zip(grids, resps, ev):
        og = make_grid(g.n_wires, g.n_ticks, g.pad_wires, g.pad_ticks, g.pitch, g.tick)
        orr = make_response(r.plane_kind, r.field_sigma_t, r.shaper_peaking, r.shaper_order, r.gain)
        t0 = time.perf_counter()
        ref.build_response(og, orr, values=True)
        build_s = time.perf_counter() - t0
        t = ref.run_simulation(og, orr, d, rng_mode=2, seed=12345, workers=cores)["timing"]
        plane_s = float(t[0]) + float(t[3]) + max(0.0, float(t[4]) - build_s)  # raster + scatter + (ft - build)
        parts.append(round(plane_s, 3))
        total += plane_s
    return N_DEPOS / total, (f"the three planes of one 100k-depo event through the unmodified reference's "
                             f"run_simulation (substream fluctuation) at {cores} threads, build_response time "
                             f"subtracted; per-plane s {parts}")


def reference_sample(args, cores):
    """CPU reference (oracle/_ref) on a bounded sample of the c4 / c5 step, scaled
    to the step by unit counts; returns (depos/s, description)."""
    from paper_2104_08265_b200.workloads import microboone_event, microboone_grids, protodune_event, protodune_specs
    if args.workload == "c3":
        return c3_reference(cores)
    if args.workload == "c1":
        from paper_2104_08265_b200.workloads import line_tracks
        g, r = c1_plane()
        t = cpu_reference_units([(g, r, line_tracks(C1_DEPOS, g, seed=1))] * 3, cores)
        return C1_DEPOS / min(t), (f"the C1 plane (10k depos) through the unmodified reference at {cores} threads, "
                                   f"best of 3; the reference bins per wire (the degenerate impact case)")
    if args.workload == "c4":
        specs = protodune_specs()
        plane_of, depos = protodune_event(C4_DEPOS, seed=1)
        t = cpu_reference_units([(specs[0][0], specs[0][1], depos[0]), (specs[2][0], specs[2][1], depos[2])], cores)
        step_s = 24 * t[0] + 12 * t[1]  # 12 U + 12 V (same geometry as U) + 12 W units
        return 36 * C4_DEPOS / step_s, (f"face 0's U and W units timed at {cores} threads ({t[0]:.2f} s, {t[1]:.2f} s), "
                                        f"scaled by unit count to the 36-unit event; build_response excluded")
    grids, resps = microboone_grids()
    ev = microboone_event(args.depos, seed=1)
    t = cpu_reference_units([(grids[i], resps[i], ev[i]) for i in range(3)], cores)
    return args.depos / sum(t), (f"one {args.depos}-depo event (3 planes) timed at {cores} threads "
                                 f"({sum(t):.2f} s); depos/s of the 64-event step equals the per-event rate")


def run_sim(args, world, rank, local):
    """The simulation workloads (event / c4 / c5) on this rank's GPU."""
    import torch
    import torch.distributed as dist
    from paper_2104_08265_b200 import AdcConfig, Context, Plane, SimConfig, run_events, simulate_event_device
    from paper_2104_08265_b200._lib import TimingC
    from paper_2104_08265_b200.sharding import shard_units, unit_cost
    from paper_2104_08265_b200.workloads import microboone_event, microboone_grids, protodune_event, protodune_specs

    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    if args.impl == "reference":
        if rank == 0:
            value, sample = reference_sample(args, cores)
            print(json.dumps({
                "impl": "reference", "metric": "depositions_per_sec", "value": value, "unit": "depos/s",
                "n_gpus": args.gpus, "steps": 1, "warmup": 0, "ms_per_step": None, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic line tracks",
                "config": {"workload": workload_desc(args), "workers": cores},
                "cpu_baseline": {"value": value, "unit": "depos/s", "cores": cores, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": value, "unit": "depos/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
                flush=True)
        return

    torch.cuda.set_device(local)
    backend = init_dist(local) if world > 1 else "nccl"

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda" if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    from paper_2104_08265_b200 import RngConfig
    cfg = SimConfig(fluctuate=args.workload == "c3", rng=RngConfig(mode="philox", seed=12345),
                    adc=AdcConfig(1.0, 2048.0, 12))
    # calls[r] = list of (planes, [host depo arrays]) for rotation slot r; one
    # step runs every call of one slot
    if args.workload == "c1":
        from paper_2104_08265_b200.workloads import line_tracks
        g, r = c1_plane()
        planes = [Plane(ctx, g, r, impacts_per_pitch=C1_IMPACTS)]
        calls = [[(planes, [line_tracks(C1_DEPOS, g, seed=1000 * rank + e + 1)])] for e in range(N_EVENTS_ROTATE)]
        scaling = "weak"
        step_depos_all = world * C1_DEPOS
        parallel = f"plane-sharded x{world}"
    elif args.workload in ("event", "c3"):
        grids, resps = microboone_grids()
        planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
        calls = [[(planes, ev)] for ev in make_events(rank)]
        scaling = "weak"
        step_depos_all = world * N_DEPOS
        parallel = f"event-sharded x{world}"
    elif args.workload == "c5":
        grids, resps = microboone_grids()
        planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
        distinct = [microboone_event(args.depos, seed=50 + e) for e in range(C5_ROTATE)]
        mine = list(range(rank, C5_EVENTS, world))
        calls = [[(planes, distinct[(e + k) % C5_ROTATE]) for e in mine] for k in range(2)]
        scaling = "strong"
        step_depos_all = C5_EVENTS * args.depos
        parallel = f"{C5_EVENTS} events round-robin over {world} rank(s)"
    else:
        specs = protodune_specs()
        plane_of, _ = protodune_event(1, seed=1)
        costs = [unit_cost(specs[p][0].padded_wires(), specs[p][0].padded_ticks(), C4_DEPOS) for p in plane_of]
        mine = shard_units(costs, world)[rank]
        planes = [Plane(ctx, *specs[plane_of[u]]) for u in mine]
        calls = []
        for k in range(C4_ROTATE):
            _, depos = protodune_event(C4_DEPOS, seed=1 + k)
            calls.append([(planes, [depos[u] for u in mine])])
        scaling = "strong"
        step_depos_all = 36 * C4_DEPOS
        parallel = f"36 (face, plane) units LPT-sharded over {world} rank(s)"
    n_rot = len(calls)
    dev = [[([torch.from_numpy(d.view(np.uint8)).cuda() for d in ds], [len(d) for d in ds]) for _, ds in slot]
           for slot in calls]
    frames = {}
    for slot in calls:
        for pl, _ in slot:
            for p in pl:
                if id(p) not in frames:
                    frames[id(p)] = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    step_cells = sum(p.shape[0] * p.shape[1] for pl, _ in calls[0] for p in pl)
    torch.cuda.synchronize()

    def step(i, timing=None):
        for j, (pl, _) in enumerate(calls[i % n_rot]):
            dd, nd = dev[i % n_rot][j]
            simulate_event_device(ctx, pl, dd, nd, cfg, [frames[id(p)] for p in pl],
                                  timing=timing if j == 0 else None)

    from paper_2104_08265_b200._lib import WsError
    for attempt in range(4):  # the warm-up also sizes the workspace: a device call that
        try:                  # overflowed it returns WS_ERANGE (it grew), so warm up again
            for i in range(args.warmup):
                step(i)
            ctx.synchronize()
            break
        except WsError as e:
            if e.code != 2 or attempt == 3:  # WS_ERANGE
                raise
    stage = TimingC()  # per-stage device times of one call (outside the timed region)
    step(0, timing=stage)
    ctx.synchronize()

    launches0 = ctx.launch_count
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    if args.workload == "c1":
        # the step's working set (5 MB of depos, 17 MB of frame) fits in L2:
        # each step timed alone, L2 flushed (256 MB written) between steps
        flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        with ClockSampler(local) as clocks:
            for i in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.fill_(float(i))
                evs[i][0].record(stream)
                step(i)
                evs[i][1].record(stream)
            ctx.synchronize()
            torch.cuda.synchronize()
        ms_local = sum(a.elapsed_time(b) for a, b in evs)
    else:
        with ClockSampler(local) as clocks:
            start.record(stream)
            for i in range(args.steps):
                step(i)
            end.record(stream)
            ctx.synchronize()
            torch.cuda.synchronize()
        ms_local = start.elapsed_time(end)
    barrier()
    gpu_launches = ctx.launch_count - launches0
    ms = max_over_ranks(ms_local)
    ms_per_step = ms / args.steps
    value = step_depos_all * args.steps / (ms * 1e-3)
    clk = clocks.summary()

    # dominant kernel roofline: the convolution stage of one call (k_direct on
    # time-domain planes, k_conv on row-FFT planes), timed by stage events on
    # the library's stream. Algorithmic traffic = SURVEY.md §8(d) K3's floor,
    # 8 B/cell (read S + write M), x the call's cells.
    call_planes = calls[0][0][0][:8]
    call_cells = sum(p.shape[0] * p.shape[1] for p in call_planes)
    conv_ms = max_over_ranks(float(stage.convolve_ms))
    n_direct = int(stage.direct_planes)
    conv_kernel = "k_direct" if n_direct == len(call_planes) else ("k_conv" if n_direct == 0 else "k_direct+k_conv")
    if args.workload == "c3":
        conv_kernel = "k_conv_tc2"  # fluctuation counts: the grid convolution on tcgen05 (ws_conv_tc.cu)
    alg_bytes = 8.0 * call_cells
    peak, peak_kind = peaks()
    achieved = alg_bytes / (conv_ms * 1e-3) / 1e9
    facts = profile_facts(conv_kernel.split("+")[0])
    binding = None
    if facts.get("warp_inst_per_launch") and args.workload in ("event", "c4", "c5"):
        # k_direct is bound by instruction issue (shared-memory REDs and their
        # address / rounding arithmetic), not by HBM: its issue roofline
        sm_hz = 1e6 * float(clk.get("sm_mhz") or 1965.0)
        issue_peak = 148 * 4 * sm_hz  # warp instructions / s (4 schedulers per SM, 1 issue / clk)
        issue_ach = facts["warp_inst_per_launch"] / (conv_ms * 1e-3)
        binding = {"resource": "instruction issue (warp instr/s)", "achieved": issue_ach, "peak": issue_peak,
                   "frac": issue_ach / issue_peak, "warp_inst_per_launch": facts["warp_inst_per_launch"],
                   "source": facts.get("source")}

    # end to end through the reference-facing call: ws_run_events (SimResult::adc
    # as uint16 codes) with pinned host depos in and ADC frames out, pipelined
    e2e = e2e_f32 = None
    if not args.no_e2e:
        slot_planes = calls[0][0][0]
        host_events = []
        for k in range(min(2, n_rot)):
            for _, ds in calls[k]:
                row = []
                for d in ds:
                    t = torch.empty(d.nbytes, dtype=torch.uint8).pin_memory()
                    t.numpy()[:] = d.view(np.uint8)
                    row.append(t.numpy().view(d.dtype))
                host_events.append(row)
        per_step = len(calls[0])
        k_e2e = max(3, min(args.steps, 20)) if args.workload in ("event", "c3", "c1") else max(1, min(args.steps, 3))
        batch = [host_events[i % len(host_events)] for i in range(k_e2e * per_step)]
        adc_bufs = [[torch.empty(p.shape, dtype=torch.uint16).pin_memory().numpy() for p in slot_planes]
                    for _ in range(2)]
        adcs = [adc_bufs[i % 2] for i in range(len(batch))]
        run_events(ctx, slot_planes, batch[:2], cfg, adc_type="u16", adcs=adcs[:2])  # warm-up
        barrier()
        t0 = time.perf_counter()
        run_events(ctx, slot_planes, batch, cfg, adc_type="u16", adcs=adcs)
        t1 = time.perf_counter()
        barrier()
        e2e_s = max_over_ranks(t1 - t0)
        h2d = int(sum(d.nbytes for d in host_events[0]))
        d2h = int(sum(p.shape[0] * p.shape[1] * 2 for p in slot_planes))
        e2e = {"value": step_depos_all * k_e2e / e2e_s, "unit": "depos/s",
               "h2d_bytes_per_step": h2d * per_step, "d2h_bytes_per_step": d2h * per_step,
               "steps": k_e2e, "ms_per_step": 1e3 * e2e_s / k_e2e,
               "call": "ws_run_events (run_simulation's SimResult::adc, uint16 codes, digitize fused; pinned host "
                       "buffers, pipelined H2D / compute / D2H)"}
        if args.workload == "event":
            from paper_2104_08265_b200 import simulate_events
            fr_bufs = [[torch.empty(p.shape, dtype=torch.float32).pin_memory().numpy() for p in slot_planes]
                       for _ in range(2)]
            outs = [fr_bufs[i % 2] for i in range(len(batch))]
            simulate_events(ctx, slot_planes, batch[:2], cfg, frames=outs[:2])
            barrier()
            t0 = time.perf_counter()
            simulate_events(ctx, slot_planes, batch, cfg, frames=outs)
            t1 = time.perf_counter()
            barrier()
            s2 = max_over_ranks(t1 - t0)
            e2e_f32 = {"value": step_depos_all * k_e2e / s2, "unit": "depos/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": int(sum(p.shape[0] * p.shape[1] * 4 for p in slot_planes)),
                       "steps": k_e2e, "ms_per_step": 1e3 * s2 / k_e2e,
                       "call": "ws_simulate_events (fp32 pre-noise frames M)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.workload == "event":
            cpu = cpu_baseline_event([calls[0][0][1]], cores)
        elif args.workload in ("c3", "c1"):
            v, sample = reference_sample(args, cores)
            cpu = {"value": v, "unit": "depos/s", "cores": cores, "kind": "reference", "sample": sample}
        else:
            v, sample = reference_sample(args, cores)
            cpu = {"value": v, "unit": "depos/s", "cores": cores, "kind": "reference", "sample": sample}

    if rank == 0:
        line = {
            "metric": "depositions_per_sec", "value": value, "unit": "depos/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (straight line tracks, fixed seeds)",
            "config": {"workload": workload_desc(args), "events_per_sec": None if args.workload in ("c4", "c1") else
                       (world if args.workload in ("event", "c3") else C5_EVENTS) * 1e3 / ms_per_step,
                       "depos_per_step": step_depos_all, "cells_per_call": call_cells,
                       "l2": "inputs rotate over distinct events (> 126 MB L2); every step writes the frames",
                       "parallelism": parallel,
                       "stage_ms": {k: round(getattr(stage, k), 4) for k in
                                    ("prepare_ms", "bin_ms", "convolve_ms", "total_ms")},
                       "conv_path": f"{n_direct}/{len(call_planes)} planes of a call time-domain (k_direct), "
                                    f"rest row-FFT (k_conv)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": facts.get("dram_bytes_per_launch"),
                         "kernel": conv_kernel, "kernel_ms": conv_ms, "algorithmic_bytes": alg_bytes,
                         "peak_kind": peak_kind, "binding": binding,
                         "raster_pipes": pipe_summary("k_sample_off"),
                         "note": (None if achieved <= peak else
                                  "frac > 1: the fused time-domain kernel never materialises S, so on sparse events it "
                                  "beats the unfused 8 B/cell floor of SURVEY 8(d); its own floor is the 4 B/cell "
                                  f"frame write ({4.0 * call_cells / (conv_ms * 1e-3) / 1e9 / peak:.2f} of peak here)")},
            "fluctuation": None if args.workload != "c3" else {
                "kernels": "k_fluct_prep (per-bin draw records) + k_fluct_walk (CDF walk, dominant)",
                "kernel": "k_fluct_walk", "stage_ms": float(stage.fluctuate_ms),
                "share_of_event": float(stage.fluctuate_ms) / float(stage.total_ms),
                "pipes": pipe_summary("k_fluct_walk"), "prep_pipes": pipe_summary("k_fluct_prep")},
            "clocks": clk,
            "gpu_launches": gpu_launches,
            "e2e": e2e,
            "e2e_frames_f32": e2e_f32,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="event", choices=["event", "sigproc", "c1", "c3", "c4", "c5"],
                    help="event: the headline metric (configs[1]); c1: configs[0] (10 impacts/pitch); c3: configs[2]; "
                         "c4: configs[3]; c5: configs[4]; "
                         "sigproc: the Listing 1 chain (§8(f))")
    ap.add_argument("--depos", type=int, default=100_000, help="c5: depositions per event (1k-1M sweep)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    world, rank, local = dist_setup()
    if args.workload == "sigproc":
        run_sigproc(args, world, rank, local)
        return
    if args.impl == "reference" and args.workload == "event":
        run_reference_arm(args, world, rank)
        return
    run_sim(args, world, rank, local)


if __name__ == "__main__":
    main()
