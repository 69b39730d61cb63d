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

--gpus N > 1: one process per GPU (torchrun; bench.py launches it itself
when WORLD_SIZE is unset), one edge-router stream per rank (weak scaling),
merged onto rank 0 every slice inside the persistent engines (peer-memory
inbox, srlg_engine_merge_*); `--virtual N` runs N ranks as execution lanes
of one GPU instead (a functional / cost probe of the merge, not a scaling
number).
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
                    help="slices of the cpu_baseline per-slide sample (and of the N>1 "
                         "reference-arm sample)")
    ap.add_argument("--merge", choices=["inbox", "nccl"], default="inbox",
                    help="N>1: in-engine peer-memory merge (default) or per-slice NCCL reduce")
    ap.add_argument("--virtual", type=int, default=0,
                    help="run this many ranks as execution lanes of one GPU")
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
        "l2": l2_note(w),
        "parallelism": f"dp{world} (one edge-router stream per GPU)",
    }


def state_cells(w):
    """RSRA r x 2^q x eta cells + SLEA r' x row_len, row_len = 2^q' delta' +
    eta' - delta' (rsra.hpp:65-67, slea.hpp:33-35)"""
    p = w.params
    row_len = (1 << p["q_prime"]) * p["delta_prime"] + p["eta_prime"] - p["delta_prime"]
    return (p["r"] << p["q"]) * p["eta"] + p["r_prime"] * row_len


L2_BYTES = 126 * 1024 * 1024  # B200 (cudaDevAttrL2CacheSize is read at run time when a GPU is up)


def needs_flush(w):
    return 8 * int(w.spec["packets"]) < 2 * L2_BYTES


def l2_note(w):
    state = 4 * state_cells(w)
    fits = state < L2_BYTES
    trace = (f"inputs larger than L2 ({8 * int(w.spec['packets']) / 1e6:.0f} MB trace per step "
             ">> L2, no flush needed)" if not needs_flush(w) else
             f"trace ({8 * int(w.spec['packets']) / 1e6:.1f} MB) smaller than L2: L2 flushed "
             "(256 MB write) between timed steps, outside each step's CUDA-event span")
    return (trace + f"; sketch state {state / 1e6:.1f} MB "
            + ("kept L2-resident (evict_last policy)" if fits else
               "exceeds L2: per-slide state passes stream from HBM"))


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


def ncu_traffic(workload_name):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel (k_engine, one launch per step) from the committed ncu capture of
    the same workload (profiles/ncu_dram_<workload>.json, written by
    tools/ncu_dram.py), or None when that workload has no capture."""
    p = ROOT / "profiles" / f"ncu_dram_{workload_name}.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --------------------------------------------------------------- CPU side
# The reference CPU path (oracle/_ref = the unmodified reference library
# built from its sources; the C restatement when it is absent) on the GPU
# box's host cores. Only bench's cpu_baseline and --impl reference use it.

def _ref_backend():
    from oracle import oracle as O

    kind = "reference" if O.available("ref") else "port"
    return O.backend("ref" if kind == "reference" else "ora"), kind


def cpu_full_step(w, pairs, off, threads, steps):
    """the reference's own WindowEngine over the whole workload (process the
    pre-sliced trace, finish, take the reports), `steps` times: seconds each"""
    be, kind = _ref_backend()
    wc = w.window_config(t0_us=0, workers=threads)
    times = []
    for _ in range(steps):
        eng = be.engine(w.sketch_params(), wc)
        t = time.perf_counter()
        eng.process_slices(pairs, off, 0)
        eng.finish()
        eng.take_reports()
        times.append(time.perf_counter() - t)
        del eng
    return times, kind


def cpu_per_slide(w, pairs, off, slices, threads_list):
    """run_detection's pieces timed separately on the reference's own objects
    (window.cpp:89-111): per slice the flush_pending update
    (parallel_chunks over the slice's pairs, window.cpp:89-98), then
    run_detection (window.cpp:36-78) for the slices from k-1 on, then
    Rsra/Slea::slide (sliding_counters.cpp:18-22). The sketches are brought
    to the slice before the sample untimed; the sample straddles the first
    report."""
    be, kind = _ref_backend()
    n_slices = len(off) - 1
    s0 = max(0, min(w.k - 1 - slices // 2, n_slices - slices))
    slices = min(slices, n_slices - s0)  # workloads shorter than the sample (C1: one slice)
    wc = w.window_config(t0_us=0)
    base = be.sketch(w.sketch_params())
    for j in range(s0):  # untimed: the state at slice s0
        base.update(pairs[int(off[j]):int(off[j + 1])], max(threads_list))
        if w.reinit:
            base.reinit()
        else:
            base.slide()
    out = {}
    for threads in threads_list:
        sk = base.clone()
        t_up = t_det = t_sl = 0.0
        n_det = 0
        npk = 0
        for j in range(s0, s0 + slices):
            p = pairs[int(off[j]):int(off[j + 1])]
            t = time.perf_counter()
            sk.update(p, threads)
            t_up += time.perf_counter() - t
            npk += len(p)
            if j + 1 >= w.k:
                t = time.perf_counter()
                sk.detect(wc, j, False)
                t_det += time.perf_counter() - t
                n_det += 1
            t = time.perf_counter()
            if w.reinit:
                sk.reinit()
            else:
                sk.slide()
            t_sl += time.perf_counter() - t
        total = t_up + t_det + t_sl
        out[f"W={threads}"] = {
            "mpps": round(npk / total / 1e6, 3),
            "update_mpps": round(npk / t_up / 1e6, 3),
            "run_detection_ms_per_slide": round(t_det * 1e3 / max(1, n_det), 3),
            "slide_ms_per_slide": round(t_sl * 1e3 / slices, 3),
        }
    desc = (f"slices {s0}..{s0 + slices - 1} of {w.name} ({npk} packets, {n_det} with "
            f"run_detection), sketches brought to slice {s0} untimed")
    return out, kind, desc


def cpu_distributed_sample(streams, w, slices, threads):
    """run_distributed (distributed.cpp:35-117) over N edge-router streams on
    the reference's own objects, one slice at a time: every node's slice
    update (flush, :59-70), the transient global = copy of node 0 merged with
    every other node (merge_min, :72-85), run_detection on it, then every node
    slides (:87-99). Nodes are brought to the sample's first slice untimed.
    Returns (Mpps over all nodes' packets, description)."""
    be, kind = _ref_backend()
    n_slices = len(streams[0][1]) - 1
    s0 = max(0, min(w.k - 1 - slices // 2, n_slices - slices))
    slices = min(slices, n_slices - s0)
    wc = w.window_config(t0_us=0)
    nodes = [be.sketch(w.sketch_params()) for _ in streams]
    for j in range(s0):
        for sk, (p, o) in zip(nodes, streams):
            sk.update(p[int(o[j]):int(o[j + 1])], threads)
            sk.reinit() if w.reinit else sk.slide()
    npk = 0
    t = time.perf_counter()
    for j in range(s0, s0 + slices):
        for sk, (p, o) in zip(nodes, streams):
            part = p[int(o[j]):int(o[j + 1])]
            sk.update(part, threads)
            npk += len(part)
        if j + 1 >= w.k:
            g = nodes[0].clone()
            for sk in nodes[1:]:
                g.merge_min(sk)
            g.detect(wc, j, False)
            del g
        for sk in nodes:
            sk.reinit() if w.reinit else sk.slide()
    dt = time.perf_counter() - t
    desc = (f"run_distributed loop over {len(streams)} nodes, slices {s0}..{s0 + slices - 1} "
            f"({npk} packets), nodes brought to slice {s0} untimed, {threads} threads")
    return npk / dt / 1e6, kind, desc


# --------------------------------------------------------------- GPU side

def merged_setup(eng, rank, world, off, max_local_pairs):
    """in-engine merge group across the torchrun ranks: rank 0's engine owns
    the inbox, the others map it through its CUDA IPC handle"""
    import torch
    import torch.distributed as dist

    t = torch.tensor([max_local_pairs], dtype=torch.int64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_pairs = int(t.item())
    handle = [eng.merge_create(world, max_pairs) if rank == 0 else None]
    dist.broadcast_object_list(handle, src=0)
    if rank != 0:
        eng.merge_join(rank, handle[0])
    dist.barrier()


def engine_roofline(w, eng_prof, steps, upd_per_pkt, r_uniform, r_trace, k1_rate, hbm_peak,
                    peak_src, state_bytes, world, merged_entries):
    """The dominant kernel (k_engine, one launch per step) against the
    random-update rate R of SURVEY.md §8(d): achieved = U x packets per
    launch (U = r' + r 2^-tau updates per packet; plus, on a merge root, the
    other ranks' list entries it applies) / the launch's CUDA-event time."""
    k_ms, k_launches, k_pairs = (eng_prof["engine_ms"], eng_prof["engine_launches"],
                                 eng_prof["engine_pairs"])
    per_launch_s = k_ms * 1e-3 / max(1, k_launches)
    upd_per_launch = upd_per_pkt * k_pairs / max(1, k_launches) + merged_entries
    achieved = upd_per_launch / per_launch_s if per_launch_s else 0.0
    fits = state_bytes < L2_BYTES
    # beyond L2 the update rate depends on the trace's reuse (Zipf-hot cells
    # stay in L2): the bound is the same updates without any detection — K1
    # alone over the same trace — or the replayed index stream, whichever is
    # faster (the replay streams 4 B of index per update from HBM besides)
    peak = r_uniform if fits else max(r_trace, k1_rate)
    traffic = ncu_traffic(w.name)
    return {
        "bound": "l2_random_update" if fits else "hbm_random_update",
        "kernel": "k_engine (persistent: K1 scan + per-slide detection, detect.cu)",
        "achieved": round(achieved / 1e9, 3), "peak": round(peak / 1e9, 3),
        "unit": "Gupdates/s", "frac": round(achieved / peak, 4) if peak else None,
        "peak_source": ("R measured here: best-of-3 red.max to uniform random cells of the "
                        "state's footprint (srlg_bench_random_updates)" if fits else
                        "R measured here on the trace's own address distribution: max of K1 "
                        "alone over the same trace (no detection) and the trace's cell-index "
                        "stream replayed as red.max (srlg_bench_trace_updates)"),
        "r_uniform_gups": round(r_uniform / 1e9, 3),
        "r_trace_gups": round(r_trace / 1e9, 3),
        "traffic": traffic,
        "traffic_source": (f"profiles/ncu_dram_{w.name}.json (dram__bytes_read.sum + "
                           "dram__bytes_write.sum of one k_engine launch)" if traffic else None),
        "updates_per_launch": round(upd_per_launch),
        "algorithmic_updates": f"{upd_per_pkt:.7g} per packet (r' + r 2^-tau, SURVEY.md §8d)"
                               + (" + the merged ranks' list entries" if merged_entries else ""),
        "avg_launch_us": round(per_launch_s * 1e6, 1),
        "launches_per_step": round(k_launches / steps, 2),
        "trace_stream": {
            "achieved_gbs": round(8 * k_pairs / max(1, k_launches) / per_launch_s / 1e9, 1)
            if per_launch_s else None,
            "peak_gbs": hbm_peak, "peak_source": peak_src,
            "frac": round(8 * k_pairs / max(1, k_launches) / per_launch_s / 1e9 / hbm_peak, 4)
            if per_launch_s else None,
            "note": "8 B per packet read once from HBM by the scan",
        },
    }


def run_ours(args):
    import torch

    from paper_1805_09246_b200 import abi, native, synth

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = local
    virtual = args.virtual if world == 1 and args.virtual > 1 else 0
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
    comm = None
    peers = []  # virtual ranks: (engine, device trace, offsets)
    max_local = int(np.diff(off.astype(np.int64)).max())
    if virtual:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        per = max(4, min(16, sms // (2 * virtual)))
        root_lane = native.lane_create(dev, sms - per * (virtual - 1))
        eng = native.WindowEngine.from_params(w.sketch_params(), wc, device=root_lane)
        streams = []
        for r in range(1, virtual):
            wr = workload(args, r)
            trr = synth.trace(wr)
            pr, orr = trr.generate()
            streams.append((pr, orr))
            max_local = max(max_local, int(np.diff(orr.astype(np.int64)).max()))
        eng.merge_create(virtual, max_local)
        for r, (pr, orr) in enumerate(streams, start=1):
            e = native.WindowEngine.from_params(w.sketch_params(), wc,
                                                device=native.lane_create(dev, per))
            e.merge_attach(r, eng)
            peers.append((e, torch.from_numpy(pr.view(np.uint8)).cuda(), orr))
        total_all = total + sum(len(p) for p, _ in streams)
        torch.cuda.synchronize()
    else:
        eng = native.WindowEngine.from_params(w.sketch_params(), wc, device=dev)
        total_all = total * world
        if world > 1:
            if args.merge == "inbox":
                merged_setup(eng, rank, world, off, max_local)
            else:
                import torch.distributed as dist

                uid = [native.nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                comm = native.nccl_comm_create(world, uid[0], rank, dev)
                eng.set_merge(comm, rank, world, 0)
    eng_dev = root_lane if virtual else dev  # the root engine's execution context
    stream = torch.cuda.ExternalStream(native.device_stream(eng_dev), device=dev)

    def step(device_input=True):
        for e, _, _ in peers:
            e.reset()
        eng.reset()
        for e, t, o in peers:  # virtual ranks: launched first, they run concurrently
            e.process_slices(offsets=o, device_ptr=t.data_ptr())
        if device_input:
            eng.process_slices(offsets=off, device_ptr=dtrace.data_ptr())
        else:
            eng.process_slices_host_ptr(host.data_ptr(), off)
        eng.finish()
        for e, _, _ in peers:
            e.finish()
            e.take_reports()
        return eng.take_reports()

    # profiling on from the first warm-up step: its first use allocates the
    # per-op timing buffers, which must not land in the timed region
    native.profile_enable(eng_dev, True)
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
    native.profile_read(eng_dev)
    native.profile_read_engine(eng_dev)
    eng.detect_latency()
    if world > 1 or virtual:
        eng.merge_stats()
    launches0 = native.kernel_launches()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}") \
        if needs_flush(w) else None
    clocks.mark()
    ev0.record(stream)
    walls = []
    merged_bytes = 0
    spans = []
    for _ in range(args.steps):
        if flush is not None:  # trace smaller than L2: evict it between steps
            with torch.cuda.stream(stream):
                flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        tw = time.perf_counter()
        step()
        b.record(stream)
        spans.append((a, b))
        walls.append(round((time.perf_counter() - tw) * 1e3, 2))
        if (world > 1 or virtual) and rank == 0:
            merged_bytes += eng.merge_stats()["bytes_exchanged"]
    ev1.record(stream)
    ev1.synchronize()
    clocks.__exit__(None, None, None)
    print(f"timed step wall ms: {walls}", file=sys.stderr)
    torch.cuda.synchronize()
    barrier()
    # the K steps' device time (sum of the per-step spans: an L2 flush, when
    # one runs, falls between them); max over ranks
    ms_total = max_over_ranks(sum(a.elapsed_time(b) for a, b in spans))
    eprof = native.profile_read_engine(eng_dev)
    prof = native.profile_read(eng_dev)
    native.profile_enable(eng_dev, False)
    launches = native.kernel_launches() - launches0
    det_us, det_windows = eng.detect_latency()
    ms_step = ms_total / args.steps
    value = total_all / (ms_step * 1e-3) / 1e6

    # ---- roofline of the dominant kernel (k_engine) against R
    rc = native.rsra_config(w.sketch_params())
    sc = native.slea_config(w.sketch_params())
    upd_per_pkt = sc.r + rc.r * 2.0 ** (-rc.tau)
    cells = eng.rsra().num_cells + eng.slea().num_cells
    r_uniform = native.bench_random_updates(dev, cells, 1 << 28, mode=1, reps=3)
    r_sample = min(total, 1 << 27)
    r_trace, _ = native.bench_trace_updates(eng.rsra(), eng.slea(), dtrace.data_ptr(), r_sample)
    peak, peak_src = measured_peaks()
    merged_entries = merged_bytes / 4 / max(1, args.steps)
    # K1 alone over the resident trace (one launch, outside the timed region)
    scan_eng = native.WindowEngine.from_params(w.sketch_params(), wc, device=dev)
    k1_stream = torch.cuda.ExternalStream(native.device_stream(dev), device=dev)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    native.update_pairs(scan_eng.rsra(), scan_eng.slea(), device_ptr=dtrace.data_ptr(), n=total)
    torch.cuda.synchronize()
    s0.record(k1_stream)
    native.update_pairs(scan_eng.rsra(), scan_eng.slea(), device_ptr=dtrace.data_ptr(), n=total)
    s1.record(k1_stream)
    s1.synchronize()
    scan_s = s0.elapsed_time(s1) * 1e-3
    del scan_eng
    k1_rate = upd_per_pkt * total / scan_s if scan_s else 0.0
    roofline = engine_roofline(w, eprof, args.steps, upd_per_pkt, r_uniform, r_trace, k1_rate,
                               peak, peak_src, 4 * cells, world, merged_entries)
    roofline["share_of_step"] = round(eprof["engine_ms"] / ms_total, 4) if ms_total else None
    roofline["k1_scan_alone"] = {
        "kernel": "k_scan (K1) alone over the resident trace, one launch",
        "achieved_gups": round(upd_per_pkt * total / scan_s / 1e9, 3) if scan_s else None,
        "frac": round(upd_per_pkt * total / scan_s / roofline["peak"] / 1e9, 4) if scan_s else None,
    }
    per_slide_us = det_us if det_windows else (
        prof["detect_ms"] * 1e3 / max(1, prof["detect_windows"]))

    # ---- e2e: host pinned input through the C ABI, reports read back
    e2e = None
    if not args.no_e2e and not virtual:
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
    if rank == 0 and world == 1 and not virtual and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        pairs_np, off_np = host_np[:total], off
        per_slide, kind, desc = cpu_per_slide(w, pairs_np, off_np, args.ref_slices,
                                              sorted({1, threads}))
        best = per_slide[f"W={threads}"]
        cpu = {"value": best["mpps"], "unit": "Mpps", "cores": threads, "kind": kind,
               "sample": desc, "cpu_model": cpu_model(), "per_slide": per_slide,
               "note": "value = W=nproc packets / (update + run_detection + slide) time over "
                       "the sample; the reference's full C2 step is timed by --impl reference"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "Mpps",
            "n_gpus": 1 if virtual else world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (deterministic Zipf edge-router trace, csrc/synth.c)",
            "config": config_json(w, total, world),
            "per_slide_estimate_us": round(per_slide_us, 2),
            "scan_only_mpps": round(total / scan_s / 1e6, 1) if scan_s else None,
            "reports_per_step": len(reports),
            "entries_per_step": sum(len(r.entries) for r in reports),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks.summary(),
        }
        if world > 1 or virtual:
            n = virtual or world
            line["merge"] = {
                "kind": ("in-engine peer-memory inbox: ranks publish their slices' moved "
                         "cells, rank 0's persistent engine applies them before each "
                         "detection (srlg_engine_merge_*)" if args.merge == "inbox" or virtual
                         else "per-slide NCCL max-reduce of u8 touched-cell maps onto rank 0 "
                              "(srlg_engine_set_merge)"),
                "ranks": n,
                "slices_merged_per_step": len(off) - 1,
                "bytes_applied_per_step": round(merged_bytes / max(1, args.steps)),
            }
            if virtual:
                line["config"]["parallelism"] = (f"{virtual} virtual ranks on one GPU "
                                                 "(execution lanes; not a scaling number)")
                line["scaling"] = "weak (virtual ranks share one GPU)"
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        barrier()
        del eng
        if comm:
            native.nccl_comm_destroy(comm)
        dist.destroy_process_group()


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref, built from the unmodified sources) on the box's host cores,
    on this arm's metric and workload. N = 1: one step = the reference
    WindowEngine over the whole C2 trace (process, finish, reports) with all
    host threads. N > 1: rank 0 alone times the run_distributed loop over the
    N ranks' edge-router streams on a bounded sample (the full N x 100M-packet
    job would take minutes per step); the other ranks exit."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_1805_09246_b200 import abi, synth

    threads = os.cpu_count() or 1
    w = workload(args, 0)
    pairs, off = synth.trace(w).generate()
    warm = max(3, args.warmup)
    if world == 1:
        times, kind = cpu_full_step(w, pairs, off, threads, warm + args.steps)
        timed = times[warm:]
        sec = statistics.median(timed)
        value = len(pairs) / sec / 1e6
        ms = sec * 1e3
        desc = (f"the whole {w.name} step ({len(pairs)} packets, {len(off) - 1} slices, "
                f"{max(0, len(off) - w.k)} + 1 reports) through the reference WindowEngine "
                f"(process_slices + finish + reports), workers={threads}")
    else:
        streams = [(pairs, off)]
        for r in range(1, world):
            pr, orr = synth.trace(workload(args, r)).generate()
            streams.append((pr, orr))
        rates = []
        for _ in range(warm + args.steps):
            v, kind, desc = cpu_distributed_sample(streams, w, args.ref_slices, threads)
            rates.append(v)
        value = statistics.median(rates[warm:])
        ms = None
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "Mpps",
        "n_gpus": world, "steps": args.steps, "warmup": warm,
        "ms_per_step": round(ms, 1) if ms else None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u16",
        "data": "synthetic (same generator and seeds as the GPU arm)",
        "config": config_json(w, int(w.spec["packets"]), world),
        "cpu_baseline": {"value": round(value, 3), "unit": "Mpps", "cores": threads,
                         "kind": kind, "sample": desc, "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 3), "unit": "Mpps", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args):
    """--gpus N without torchrun: launch N ranks (one per GPU) through
    torch.distributed.run on this node and return its exit code"""
    import socket

    import torch

    n = torch.cuda.device_count() if args.impl == "ours" else args.gpus
    if n < args.gpus:
        print(f"bench.py --gpus {args.gpus}: this node has {n} GPU(s); use --virtual "
              f"{args.gpus} for virtual ranks on one GPU", file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.virtual:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
