#!/usr/bin/env python
"""Benchmark of the length-bucketed word sort on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

Workload: BASELINE.json config 4 by default (16M words, lengths Zipfian over
1-32 with 40% at L=5; seeded synthetic text, see paper_1407_6603_b200/synth.py)
-- the largest single-GPU configuration; BASELINE.json quotes its metric on
no single config, and configs 0-3 are parity cases (tests/).

One JSON line on rank 0:
  value      words/s with the text already resident in HBM: ingest (tokenize,
             length histogram, stable scatter into packed keys) + per-bucket
             sort + emit of the payload into HBM, CUDA events on the library's
             stream, L2 flushed (256 MiB memset) between timed steps.
  e2e        words/s through the C ABI with pinned HOST buffers, H2D of the text
             + all kernels + D2H of the payload in every step: a batch of K
             corpora through ws_sort_texts (3 in flight, wall clock around the
             call); e2e.single = one ws_sort_text call per step (CUDA events).
  roofline   dominant kernel: algorithmic bytes per launch / its CUDA-event
             duration inside the timed steps, against MEASURED_PEAKS.json.
  cpu_baseline  the reference algorithm (oracle/ C port of _bubble_rows etc.)
             on the host cores, on a bounded prefix sample of the same text.
`--impl reference` times that CPU path alone (rank 0; other ranks exit 0).
Multi-GPU: independent replicas (one corpus per rank, no collective in the
data path), weak scaling, max-over-ranks timing.
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

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sorted words/sec on 1 B200 (end-to-end) and % of HBM/int-pipe roofline; bit-exact"
UNIT = "words/s"
CPU_SAMPLE_WORDS = 120_000
FLUSH_BYTES = 256 << 20
INFLIGHT = 3  # corpora in flight in the serving (batch) e2e leg


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample-words", type=int, default=CPU_SAMPLE_WORDS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the oracle payload check")
    ap.add_argument("--profile-json", default=None, help="also write per-phase timings here")
    return ap.parse_args()


def rank_info():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def reduce_over_ranks(x: float, world: int, device, op: str = "max") -> float:
    """Whole-job figure of a per-rank value: the slowest rank's time ("max")
    or the job's total work ("sum"); identity on one rank."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def workload_name(cfg: int) -> str:
    from paper_1407_6603_b200 import synth

    return f"config{cfg}-{synth.CONFIGS[cfg].name}"


def corpus(cfg: int, rank: int) -> bytes:
    from paper_1407_6603_b200 import synth

    seed = synth.BASE_SEED + cfg + 7919 * rank  # rank 0 = the canonical seeded config
    return synth.generate(cfg, seed=seed)


# ---------------------------------------------------------------------------
# CPU baseline (oracle = C restatement of the reference algorithm)

def cpu_sample(text: bytes, words: int) -> bytes:
    from paper_1407_6603_b200 import synth

    return synth.prefix(text, words)


def extrapolate(full_hist: dict, sample_info: dict, timings: dict, threads: int) -> float | None:
    """Full-workload seconds of the bubble sort from per-bucket sample times
    (cost of bucket L ~ n_L(n_L - 1)/2 comparisons), LPT over `threads`."""
    jobs = []
    for L, n_full in full_hist.items():
        if L not in sample_info or L not in timings:
            return None
        n_s = sample_info[L][0]
        if n_s < 2 or timings[L] <= 0:
            if n_full >= 2:
                return None
            continue
        jobs.append(timings[L] * (n_full * (n_full - 1)) / (n_s * (n_s - 1)))
    loads = [0.0] * max(threads, 1)
    for j in sorted(jobs, reverse=True):
        i = loads.index(min(loads))
        loads[i] += j
    return max(loads) if loads else None


def run_cpu(text: bytes, sample_words: int, threads: int, full_hist: dict | None):
    from oracle import oracle

    sample = cpu_sample(text, sample_words)
    timings: dict = {}
    t0 = time.perf_counter()
    payload, info = oracle.sort_text(sample, mode="bubble", threads=threads, timings=timings)
    dt = time.perf_counter() - t0
    n_words = sum(v[0] for v in info.values())
    res = {
        "value": n_words / dt,
        "unit": UNIT,
        "cores": threads,
        "kind": "port",
        "sample": (f"first {n_words} words ({len(sample)} bytes) of the same seeded text; "
                   "tokenize + group-by-length + per-bucket bubble sort (engine.py:89-114 "
                   f"restated in C, one task per bucket on {threads} threads) + payload"),
        "seconds": dt,
    }
    if full_hist:
        ex = extrapolate(full_hist, info, timings, threads)
        if ex:
            res["extrapolated_full_seconds"] = ex
            res["extrapolated_full_words_per_s"] = sum(full_hist.values()) / ex
    return res, dt, n_words


# ---------------------------------------------------------------------------
# clocks during the timed region

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ingest_algorithmic_bytes(n_text: int, hist: dict) -> float:
    """Text bytes read + key bytes written (6-bit text keys: <= 5 characters in
    4 B, else 8 B per started 64 bits) + 8 B per long word (L > 32)."""
    out = float(n_text)
    for L, c in hist.items():
        if L > 32:
            out += 8.0 * c
        else:
            out += (4 if L <= 5 else 8 * ((6 * L + 63) // 64)) * c
    return out


def ncu_traffic(workload: str, kernel: str):
    """Per-launch DRAM bytes of `kernel` from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(p.read_text())
        return d[workload][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


# ---------------------------------------------------------------------------

def bench_reference(args) -> None:
    rank, world, _ = rank_info()
    if rank != 0:
        return
    text = corpus(args.config, 0)
    threads = os.cpu_count() or 1
    times = []
    n_words = 0
    for i in range(args.warmup + args.steps):
        _, dt, n_words = run_cpu(text, args.cpu_sample_words, threads, None)
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    value = n_words / t
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": workload_name(args.config),
                   "sample_words": n_words, "l2_flush": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": (f"first {n_words} words of the seeded config-{args.config} "
                                    "text per step (reference bubble sort restated in C, "
                                    "oracle/wsort_oracle.c)")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_ours(args) -> None:
    import torch

    from paper_1407_6603_b200._native import Handle
    from paper_1407_6603_b200.pipeline import BatchSorter, TextSorter

    rank, world, local = rank_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        return reduce_over_ranks(x, world, dev, "max")

    text = corpus(args.config, rank)
    n = len(text)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)

    # ---- device-resident leg --------------------------------------------
    h = Handle(local)
    h.ingest_text(text)  # places the text in HBM (untimed)
    lengths, counts, words = h.buckets()
    hist = dict(zip(lengths, counts))
    stream = torch.cuda.ExternalStream(h.stream(), device=dev)
    written = 0
    for _ in range(args.warmup):
        written = h.sort_resident(n)
    sampler = ClockSampler(local)
    dev_ms = []
    with sampler:
        h.profile(reset=True)
        h.set_profiling(True)
        launches0 = h.launch_count()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            barrier()
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            written = h.sort_resident(n)
            b.record(stream)
            torch.cuda.synchronize(dev)
            dev_ms.append(a.elapsed_time(b))
        launches = h.launch_count() - launches0
        h.set_profiling(False)
        phases = h.profile(reset=True)

        # ---- end-to-end leg through the C ABI with host buffers -------------
        ts = TextSorter(n, device=local)
        ts.load(text)
        estream = torch.cuda.ExternalStream(ts.handle.stream(), device=dev)
        for _ in range(args.warmup):
            e2e_written = ts.run()
        e2e_ms = []
        e2e_launches0 = ts.handle.launch_count()
        for _ in range(args.steps):
            with torch.cuda.stream(estream):
                flush.zero_()
            barrier()
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(estream)
            e2e_written = ts.run()
            b.record(estream)
            torch.cuda.synchronize(dev)
            e2e_ms.append(a.elapsed_time(b))
        e2e_launches = ts.handle.launch_count() - e2e_launches0

        # ---- serving leg: the same corpus as a batch of K jobs through
        # ws_sort_texts, INFLIGHT in flight (H2D of one overlaps the sort and
        # D2H of the previous ones); every job's H2D and D2H is in the region
        bs = BatchSorter(n, inflight=INFLIGHT, device=local)
        bs.load(text)
        bs.run(max(args.warmup, INFLIGHT))
        batch_launches0 = bs.handle.launch_count()
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        batch_sizes = bs.run(args.steps)
        torch.cuda.synchronize(dev)
        batch_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        batch_launches = bs.handle.launch_count() - batch_launches0

        # ---- stats leg: the reference's full SortStats semantics on the
        # device (order-preserving ingest, merge sort with inversion / K
        # counts, per-bucket stats read back), text already in HBM
        dtext = torch.frombuffer(bytearray(text), dtype=torch.uint8).to(dev)
        hsx = Handle(local)
        sstream = torch.cuda.ExternalStream(hsx.stream(), device=dev)
        for _ in range(args.warmup):
            hsx.ingest_text(None, device_ptr=dtext.data_ptr(), n=n)
            hsx.sort(True)
            hsx.bucket_stats(True)
        stats_ms = []
        for _ in range(args.steps):
            with torch.cuda.stream(sstream):
                flush.zero_()
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(sstream)
            hsx.ingest_text(None, device_ptr=dtext.data_ptr(), n=n)
            hsx.sort(True)
            hsx.bucket_stats(True)
            b.record(sstream)
            torch.cuda.synchronize(dev)
            stats_ms.append(a.elapsed_time(b))
    clocks = sampler.summary()
    # one extra (untimed) e2e step with per-phase events, for the timeline
    ts.handle.profile(reset=True)
    ts.handle.set_profiling(True)
    torch.cuda.synchronize(dev)
    ts.run()
    ts.handle.set_profiling(False)
    e2e_phases = ts.handle.profile(reset=True)

    t_dev = max_over_ranks(statistics.mean(dev_ms))
    t_e2e = max_over_ranks(statistics.mean(e2e_ms))
    t_batch = max_over_ranks(batch_ms)
    t_stats = max_over_ranks(statistics.mean(stats_ms))
    value = world * words / (t_dev * 1e-3)
    e2e_value = world * words / (t_e2e * 1e-3)
    batch_value = world * words / (t_batch * 1e-3)

    # per-phase aggregation (CUDA events on the library stream, timed steps)
    agg: dict = {}
    for p in phases:
        a_ = agg.setdefault(p["name"], {"ms": 0.0, "bytes": 0.0, "launches": 0, "kind": p["kind"]})
        a_["ms"] += p["ms"]
        a_["bytes"] += p["bytes"]
        a_["launches"] += max(p["launches"], 1)
    kern = {k: v for k, v in agg.items() if v["kind"] == 0}
    step_ms = sum(dev_ms)
    # The roofline kernel is the ingest: the largest single kernel of the step
    # in the serialised ncu launch list (profiles/), and the only one that runs
    # alone (before the per-class streams fork), so its events time it cleanly.
    # Its algorithmic bytes are exact: the text read once + every packed key
    # written once + 8 B per long-word (start, len) entry.
    if "ingest" in kern:
        dom = "ingest"
        kern["ingest"]["bytes"] = args.steps * ingest_algorithmic_bytes(n, hist)
    else:
        dom = max(kern, key=lambda k: kern[k]["ms"]) if kern else None
    peak, peak_src = measured_peak()
    roofline = None
    if dom:
        d = kern[dom]
        per_launch_bytes = d["bytes"] / d["launches"]
        per_launch_ms = d["ms"] / d["launches"]
        achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
        roofline = {
            "bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
            "traffic": ncu_traffic(workload_name(args.config), dom),
            "algorithmic_bytes_per_launch": per_launch_bytes,
            "ms_per_launch": per_launch_ms, "share_of_step": d["ms"] / step_ms,
        }

    parity = None
    cpu = None
    if rank == 0:
        if not args.no_check:
            from oracle import oracle

            want, _ = oracle.sort_text(text, mode="fast")
            parity = bool(ts.payload(e2e_written) == want)
            parity = parity and all(sz == len(want) for sz in batch_sizes)
            parity = parity and all(bs.payload(k, batch_sizes[0]) == want
                                    for k in range(min(INFLIGHT, args.steps)))
            dptr, dsize = h.output_device()
            parity = parity and (dsize == len(want))
        if world == 1 and not args.no_cpu_baseline:
            cpu, _, _ = run_cpu(text, args.cpu_sample_words, os.cpu_count() or 1, hist)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_dev, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": workload_name(args.config), "words": words,
                       "text_bytes": n, "payload_bytes": written, "buckets": len(lengths),
                       "l2_flush": "256 MiB memset on the timed stream between steps",
                       "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"},
            "e2e": {"value": batch_value, "unit": UNIT, "h2d_bytes_per_step": n,
                    "d2h_bytes_per_step": batch_sizes[0] if batch_sizes else 0,
                    "ms_per_step": t_batch, "gpu_launches": batch_launches,
                    "api": f"ws_sort_texts, batch of {args.steps} corpora, {INFLIGHT} in flight, "
                           "pinned host buffers, wall clock around the call",
                    "single": {"value": e2e_value, "ms_per_step": t_e2e,
                               "gpu_launches": e2e_launches,
                               "api": "ws_sort_text, one corpus per call, CUDA events"}},
            "stats_mode": {"value": world * words / (t_stats * 1e-3), "unit": UNIT,
                           "ms_per_step": t_stats,
                           "api": "ws_ingest_text(DEVICE_PTR) + ws_sort(h, 1) + ws_bucket_stats: "
                                  "corpus-order buckets, merge sort counting inversions and K, "
                                  "the reference's SortStats per bucket"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
            "parity_vs_oracle": parity,
            "phases_ms_per_step": {k: v["ms"] / args.steps for k, v in agg.items()},
        }
        line["e2e_timeline_ms"] = [[p["name"], round(p["start_ms"], 3), round(p["ms"], 3),
                                    int(p["bytes"])] for p in e2e_phases]
        if args.profile_json:
            Path(args.profile_json).write_text(json.dumps({"phases": agg, "steps": args.steps,
                                                           "dev_ms": dev_ms, "e2e_ms": e2e_ms,
                                                           "e2e_phases": e2e_phases},
                                                          indent=1))
        print(json.dumps(line), flush=True)
    ts.close()
    bs.close()
    hsx.close()
    h.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse_args()
    rank, world, _ = rank_info()
    if args.gpus > 1 and world == 1 and "RANK" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               "--master-port=29533", __file__] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
