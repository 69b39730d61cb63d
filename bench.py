#!/usr/bin/env python
"""Benchmark of the sliding super-point path (BASELINE.json metric: Mpps of
the SRE+SLE packet scan with per-slide estimation).

One *step* = one pass of the window engine over the whole synthetic trace of
the workload (default C2: 100M packets in 600 slices, k=300, paper geometry):
every slice is scanned (K1), every completed slice from k-1 on runs the full
per-slide detection (hot extraction, reconstruction, setting factors,
per-candidate estimates -> a DetectionReport on the host), then the window
slides. Inputs are resident in HBM for `value`; `e2e` drives the same engine
through the C ABI with the trace in pinned HOST memory (H2D inside the timed
region) and the reports read back to the host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 runs under torchrun: one process per GPU, each rank scans its own
edge-router stream (weak scaling); per-slide merging is reported in DESIGN.md.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Mpps packet scan (SRE+SLE update) at 1/2/4/8 B200; per-slide estimate latency"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--packets", type=int, default=None, help="override packets (testing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-slices", type=int, default=24,
                    help="slices per reference-arm / cpu_baseline sample step")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, rank):
    from paper_1805_09246_b200 import synth

    w = synth.WORKLOADS[args.workload]
    spec = dict(w.spec)
    if args.packets:
        spec["packets"] = args.packets
    # one independent edge-router stream per rank (weak scaling)
    spec["seed"] = spec["seed"] + 1000 * rank
    return synth.Workload(w.name, spec, dict(w.params), w.k, w.reinit)


def config_json(w, packets, world):
    p = w.params
    return {
        "workload": w.name,
        "packets_per_step_per_gpu": int(packets),
        "slices": int(w.spec["n_slices"]),
        "packets_per_slice": int(packets // w.spec["n_slices"]),
        "k": w.k,
        "reinit_per_window": w.reinit,
        "sketch": (f"q={p['q']} r={p['r']} delta={p['delta']} eta={p['eta']} "
                   f"q'={p['q_prime']} r'={p['r_prime']} delta'={p['delta_prime']} "
                   f"eta'={p['eta_prime']} theta={p['theta']}"),
        "l2": "inputs larger than L2 (8 B/packet trace per step >> 126 MB); sketch state "
              "stays resident by design",
        "parallelism": f"dp{world} (one edge-router stream per GPU)",
    }


class NvmlSampler(threading.Thread):
    """SM clock and throttle reasons sampled through NVML (in-process, every
    100 ms) during the timed region: far lighter than an nvidia-smi process,
    whose start-up and per-query driver traffic stalled short timed regions."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index, interval=0.1):
        super().__init__(daemon=True)
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.interval = interval
        self.samples = []
        self.reasons = set()
        self.stop_ev = threading.Event()

    def sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for n, bit in self.REASONS.items():
            if r & bit:
                self.reasons.add(n)

    def run(self):
        while not self.stop_ev.wait(self.interval):
            self.sample()

    def __enter__(self):
        self.sample()
        self.start()
        time.sleep(0.05)  # thread start-up outside the timed region
        return self

    def mark(self):
        """the timed region starts: keep only samples taken from here on"""
        self.samples.clear()
        self.reasons.clear()
        self.sample()

    def __exit__(self, *a):
        self.stop_ev.set()
        self.join()
        self.sample()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "NVML (in-process, 100 ms)"}


def clock_sampler(index):
    try:
        return NvmlSampler(index)
    except Exception:
        return ClockSampler(index)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region
    (fallback when NVML is unavailable)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        # nvidia-smi's start-up (NVML init) contends with the CUDA driver: let it
        # reach its first sample before the timed region starts
        t0 = time.time()
        while self.proc and time.time() - t0 < 3.0:
            self.file.flush()
            if os.path.getsize(self.file.name) > 0:
                break
            time.sleep(0.02)
        return self

    def mark(self):
        self.file.flush()
        self.skip = len([r for r in open(self.file.name).read().splitlines() if r.strip()])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        self.file.flush()
        self.file.seek(0)
        rows = [r.split(",") for r in self.file.read().strip().splitlines() if r.strip()]
        rows = rows[getattr(self, "skip", 0):] or rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel (k_engine, one launch per step) from the committed ncu capture of
    the same workload (profiles/r01_ncu_engine.json), or None."""
    p = ROOT / "profiles" / "r01_ncu_engine.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


# --------------------------------------------------------------- CPU side

def cpu_reference_sample(w, slices, threads, repeats=1):
    """Reference CPU path (oracle/_ref = the unmodified reference library, or
    the C restatement when it was not built) on a bounded sample: the engine
    is brought to slice s0 untimed, then `slices` slices are processed with
    the reference's own WindowEngine (flush_pending with `threads` workers,
    run_detection, slide). Returns (Mpps samples, kind, description)."""
    from oracle import oracle as O
    from paper_1805_09246_b200 import synth

    kind = "reference" if O.available("ref") else "port"
    be = O.backend("ref" if kind == "reference" else "ora")
    n_slices = w.spec["n_slices"]
    # straddle the first report so the sample has the steady-state mix of
    # scan-only and scan+detect slices the full trace has
    s0 = max(0, min(w.k - 1 - slices // 2, n_slices - slices))
    tr = synth.trace(w)
    pairs, off = tr.generate(0, s0 + slices)
    wc = w.window_config(t0_us=0, workers=threads)
    eng = be.engine(w.sketch_params(), wc)
    eng.process_slices(pairs[: int(off[s0])], off[: s0 + 1], 0)
    eng.advance_to_slice(s0)
    sample = pairs[int(off[s0]): int(off[s0 + slices])]
    soff = off[s0: s0 + slices + 1] - off[s0]
    rates = []
    for _ in range(repeats):
        e = eng.clone() if kind == "reference" else None
        if e is None:  # the C port has no clone; rebuild (untimed)
            e = be.engine(w.sketch_params(), wc)
            e.process_slices(pairs[: int(off[s0])], off[: s0 + 1], 0)
            e.advance_to_slice(s0)
        t = time.perf_counter()
        e.process_slices(sample, soff, s0)
        e.advance_to_slice(s0 + slices)
        e.take_reports()
        dt = time.perf_counter() - t
        rates.append(len(sample) / dt / 1e6)
    desc = (f"slices {s0}..{s0 + slices - 1} of {w.name} ({len(sample)} packets, "
            f"{max(0, s0 + slices - (w.k - 1))} of them with per-slide detection), state "
            f"brought to slice {s0} untimed; WindowEngine with workers={threads}")
    return rates, kind, desc


# --------------------------------------------------------------- GPU side

def run_ours(args):
    import torch

    from paper_1805_09246_b200 import abi, native, synth

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = local
    w = workload(args, rank)
    tr = synth.trace(w)
    off = tr.offsets()
    total = int(off[-1])
    # pinned host trace (the e2e input) and its HBM copy (the `value` input)
    host = torch.empty(total * 8, dtype=torch.uint8, pin_memory=True)
    host_np = host.numpy().view(abi.PAIR_DTYPE)
    tr.generate(out=host_np)
    dtrace = host.to(f"cuda:{dev}", non_blocking=False)
    torch.cuda.synchronize()

    wc = w.window_config(t0_us=0)
    eng = native.WindowEngine.from_params(w.sketch_params(), wc, device=dev)
    stream = torch.cuda.ExternalStream(native.device_stream(dev), device=dev)
    comm = None
    if world > 1:
        # per-slide merge of every rank's stream onto rank 0 (NCCL max-reduce of
        # touched-cell maps inside the engine)
        import torch.distributed as dist

        uid = [native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = native.nccl_comm_create(world, uid[0], rank, dev)
        eng.set_merge(comm, rank, world, 0)

    def step(device_input=True):
        eng.reset()
        if device_input:
            eng.process_slices(offsets=off, device_ptr=dtrace.data_ptr())
        else:
            eng.process_slices_host_ptr(host.data_ptr(), off)
        eng.finish()
        return eng.take_reports()

    # profiling on from the first warm-up step: its first use allocates the
    # per-op timing buffers, which must not land in the timed region
    native.profile_enable(dev, True)
    # the clock sampler starts before the warm-up (NVML / nvidia-smi start-up
    # contends with the driver); only the samples from the timed region count
    clocks = clock_sampler(dev)
    clocks.__enter__()
    for _ in range(max(3, args.warmup)):
        blob = step()
    reports = abi.parse_blobs(blob)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # ---- timed region: HBM-resident input
    native.profile_read(dev)
    native.profile_read_engine(dev)
    eng.detect_latency()
    launches0 = native.kernel_launches()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark()
    ev0.record(stream)
    walls = []
    for _ in range(args.steps):
        tw = time.perf_counter()
        step()
        walls.append(round((time.perf_counter() - tw) * 1e3, 2))
    ev1.record(stream)
    ev1.synchronize()
    clocks.__exit__(None, None, None)
    print(f"timed step wall ms: {walls}", file=sys.stderr)
    torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    prof = native.profile_read(dev)
    eprof = native.profile_read_engine(dev)
    native.profile_enable(dev, False)
    launches = native.kernel_launches() - launches0
    det_us, det_windows = eng.detect_latency()
    ms_step = ms_total / args.steps
    value = total * world / (ms_step * 1e-3) / 1e6

    # ---- roofline of the dominant kernel
    rc = native.rsra_config(w.sketch_params())
    sc = native.slea_config(w.sketch_params())
    upd_per_pkt = sc.r + rc.r * 2.0 ** (-rc.tau)
    bytes_per_pkt = 8 + 4 * upd_per_pkt  # pair read + U stamp writes
    state_cells = eng.rsra().num_cells + eng.slea().num_cells
    row_len = eng.slea().row_length
    # one detection reads the whole state once (phase A) and writes / reads the
    # 1-bit SLEA bitmap; phase C reads r' x eta' bits per candidate
    bitmap_bytes = sc.r * ((row_len + 31) // 32 + 1) * 4
    entries = sum(len(r.entries) for r in reports)
    cands = sum(r.candidate_count for r in reports)
    det_bytes_step = len(reports) * (4 * state_cells + bitmap_bytes) + cands * sc.r * sc.eta / 8
    peak, peak_src = measured_peaks()
    if eprof["engine_launches"]:
        kname = "k_engine (persistent: K1 scan + per-slide detection, detect.cu)"
        k_ms, k_launches = eprof["engine_ms"], eprof["engine_launches"]
        k_bytes = (bytes_per_pkt * eprof["engine_pairs"] + det_bytes_step * args.steps)
    else:
        kname = "k_scan (K1) + k_detect per slice"
        k_ms = prof["scan_ms"] + prof["detect_ms"]
        k_launches = prof["scan_launches"] + prof["detect_windows"]
        k_bytes = bytes_per_pkt * prof["scan_pairs"] + det_bytes_step * args.steps
    achieved_gbs = k_bytes / (k_ms * 1e-3) / 1e9 if k_ms else 0.0

    # K1 alone, for the random-update roofline: one launch over the whole
    # resident trace (outside the timed region; its own CUDA events)
    scan_eng = native.WindowEngine.from_params(w.sketch_params(), wc, device=dev)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    native.update_pairs(scan_eng.rsra(), scan_eng.slea(), device_ptr=dtrace.data_ptr(), n=total)
    torch.cuda.synchronize()
    s0.record(stream)
    native.update_pairs(scan_eng.rsra(), scan_eng.slea(), device_ptr=dtrace.data_ptr(), n=total)
    s1.record(stream)
    s1.synchronize()
    scan_s = s0.elapsed_time(s1) * 1e-3
    del scan_eng
    r_rate = native.bench_random_updates(dev, state_cells, 1 << 28, mode=0, reps=3)
    r_rate_red = native.bench_random_updates(dev, state_cells, 1 << 28, mode=1, reps=3)
    scan_upd_rate = upd_per_pkt * total / scan_s if scan_s else 0.0
    traffic = ncu_traffic()
    roofline = {
        "bound": "hbm", "kernel": kname,
        "achieved": round(achieved_gbs, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved_gbs / peak, 4), "peak_source": peak_src,
        "traffic": traffic,
        "algorithmic_bytes_per_launch": round(k_bytes / max(1, k_launches)),
        "algorithmic_bytes": "28.16 B/packet (8 B pair + 5.039 x 4 B stamps) + per "
                             "detection 4 B/cell state read + 1 bit/cell SLEA bitmap",
        "avg_launch_us": round(k_ms * 1e3 / max(1, k_launches), 1),
        "launches_per_step": round(k_launches / args.steps, 2),
        "share_of_step": round(k_ms / ms_total, 4) if ms_total else None,
        "random_update_roofline": {
            "kernel": "k_scan (K1) alone over the resident trace, one launch",
            "achieved_updates_per_s": round(scan_upd_rate),
            "peak_updates_per_s_plain_store": round(r_rate),
            "peak_updates_per_s_red_max": round(r_rate_red),
            "frac": round(scan_upd_rate / r_rate, 4) if r_rate else None,
            "footprint_cells": state_cells,
            "note": "R = best-of-3 random u32 stores into a buffer of the sketch-state "
                    "footprint (srlg_bench_random_updates), SURVEY.md §8d",
        },
    }
    per_slide_us = det_us if det_windows else (
        prof["detect_ms"] * 1e3 / max(1, prof["detect_windows"]))
    scan_mpps = total / scan_s / 1e6 if scan_s else 0.0

    # ---- e2e: host pinned input through the C ABI, reports read back
    e2e = None
    if not args.no_e2e:
        for _ in range(2):  # untimed: first use allocates the host-input buffers
            step(device_input=False)
        native.io_bytes(dev)
        e_steps = max(2, min(args.steps, 5))
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        e_walls = []
        for _ in range(e_steps):
            tw = time.perf_counter()
            step(device_input=False)
            e_walls.append(round((time.perf_counter() - tw) * 1e3, 2))
        a1.record(stream)
        print(f"e2e step wall ms: {e_walls}", file=sys.stderr)
        a1.synchronize()
        wall = time.perf_counter() - t0
        h2d, d2h = native.io_bytes(dev)
        e_ms = max_over_ranks(max(a0.elapsed_time(a1), wall * 1e3)) / e_steps
        e2e = {"value": round(total * world / (e_ms * 1e-3) / 1e6, 1), "unit": "Mpps",
               "ms_per_step": round(e_ms, 3), "h2d_bytes_per_step": h2d // e_steps,
               "d2h_bytes_per_step": d2h // e_steps,
               "path": "srlg_engine_process_slices(host pinned pairs) + finish + "
                       "take_reports (C ABI)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rates, kind, desc = cpu_reference_sample(w, args.ref_slices, threads)
        cpu = {"value": round(statistics.median(rates), 3), "unit": "Mpps", "cores": threads,
               "kind": kind, "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "Mpps", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (deterministic Zipf edge-router trace, csrc/synth.c)",
            "config": config_json(w, total, world),
            "per_slide_estimate_us": round(per_slide_us, 2),
            "scan_only_mpps": round(scan_mpps, 1),
            "reports_per_step": len(reports),
            "entries_per_step": sum(len(r.entries) for r in reports),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks.summary(),
        }
        if world > 1:
            ms = eng.merge_stats()
            line["merge"] = {
                "kind": "per-slide NCCL max-reduce of u8 touched-cell maps onto rank 0 "
                        "(srlg_engine_set_merge)",
                "slice_merges_per_step": ms["slice_merges"],
                "bytes_per_rank_per_merge": ms["bytes_exchanged"] // max(1, ms["slice_merges"]),
            }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        del eng
        native.nccl_comm_destroy(comm)
        dist.destroy_process_group()


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    w = workload(args, 0)
    threads = os.cpu_count() or 1
    rates, kind, desc = cpu_reference_sample(w, args.ref_slices, threads,
                                             repeats=max(3, args.warmup) + args.steps)
    timed = rates[max(3, args.warmup):]
    value = statistics.median(timed)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "Mpps",
        "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u16", "data": "synthetic (same generator and seeds as the GPU arm)",
        "config": config_json(w, int(w.spec["packets"]), world),
        "cpu_baseline": {"value": round(value, 3), "unit": "Mpps", "cores": threads,
                         "kind": kind, "sample": desc},
        "e2e": {"value": round(value, 3), "unit": "Mpps", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
