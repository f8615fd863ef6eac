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
  roofline   the kernel family with the largest serialised share of the step:
             algorithmic bytes per launch / its CUDA-event duration (events
             around every launch in K profiled steps run after the timed
             ones), against MEASURED_PEAKS.json; roofline_rows lists every
             family (ingest; counting path: aggregate, distinct sort, run
             prefix, expand; sort paths: one-sweep radix, radix histogram,
             sample split, partition, slot sort; stats mode: ingest, tile
             sort, merge).
  cpu_baseline  the unmodified reference (baseline/_ref, numba _bubble_rows on
             a worker pool; tools/vendor_reference.sh) on the host cores, on a
             bounded prefix of the same text, with the oracle's C port of the
             same algorithm beside it ("port").
`--impl reference` times the reference's CPU path alone (rank 0; other ranks
exit 0). Every leg's output is byte-compared with the oracle after its loop.
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
REF_SAMPLE_WORDS = 60_000  # reference arm: per-step sample (~3 s of numba work on 16 threads)
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
    ap.add_argument("--ref-sample-words", type=int, default=REF_SAMPLE_WORDS,
                    help="--impl reference: words of the per-step sample")
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


def physical_cores() -> int | None:
    try:
        import psutil

        return psutil.cpu_count(logical=False)
    except Exception:
        return None


def run_cpu(text: bytes, sample_words: int, threads: int, full_hist: dict | None):
    """The oracle's C restatement of the reference pipeline (kind "port")."""
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
        "physical_cores": physical_cores(),
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
    return res, dt, n_words, payload


REF_DIR = ROOT / "baseline" / "_ref"


def reference_module():
    """The UNMODIFIED reference package installed by tools/vendor_reference.sh
    (git-ignored, shipped to the GPU box), or None when it is absent."""
    if not (REF_DIR / "wordsort" / "__init__.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_wordsort")
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import wordsort  # noqa: F401
        from wordsort import cli, engine, ingest, store
    except Exception:
        return None
    return {"ingest": ingest, "store": store, "engine": engine, "cli": cli}


def run_reference(text: bytes, sample_words: int, threads: int):
    """The reference's own pipeline through its public API, as `wordsort sort`
    runs it with the CLI defaults (cli.py:83-103: flat layout, NAIVE, STATIC,
    os.cpu_count() threads): tokenize -> build_store -> sort_all_parallel (the
    numba _bubble_rows, engine.py:89-114) -> emit_sorted -> payload join.
    Returns (seconds, words, payload) or None when the reference is absent."""
    ref = reference_module()
    if ref is None:
        return None
    sample = cpu_sample(text, sample_words)
    eng, st, ing = ref["engine"], ref["store"], ref["ingest"]
    cfg = eng.SortConfig(layout=st.LayoutKind.FLAT, variant=eng.SortVariant.NAIVE,
                         threads=threads, schedule=eng.SchedulePolicy.STATIC_BLOCK)
    t0 = time.perf_counter()
    words = ing.tokenize(sample)
    store = st.build_store(words, cfg.layout)
    if threads == 1:
        eng.sort_all_sequential(store, cfg.variant)
    else:
        eng.sort_all_parallel(store, cfg)
    payload = b"".join(w + b"\n" for w in st.emit_sorted(store))
    dt = time.perf_counter() - t0
    return dt, len(words), payload


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
    """--impl reference: the reference's own CPU path (baseline/_ref, the
    unmodified wordsort package: numba _bubble_rows on a worker pool) on the
    host cores, a bounded prefix of the same workload per step; the oracle's
    C port when the reference is not installed. Rank 0 only."""
    rank, world, _ = rank_info()
    if rank != 0:
        return
    text = corpus(args.config, 0)
    threads = os.cpu_count() or 1
    have_ref = reference_module() is not None
    times = []
    n_words = 0
    payload = b""
    for i in range(args.warmup + args.steps):
        if have_ref:
            dt, n_words, payload = run_reference(text, args.ref_sample_words, threads)
        else:
            _, dt, n_words, payload = run_cpu(text, args.ref_sample_words, threads, None)
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    value = n_words / t
    kind = "reference" if have_ref else "port"
    what = ("the unmodified reference (baseline/_ref wordsort: tokenize, build_store flat, "
            "sort_all_parallel NAIVE/STATIC with the numba _bubble_rows, emit_sorted, payload join)"
            if have_ref else "the reference bubble sort restated in C (oracle/wsort_oracle.c)")
    parity = None
    if not args.no_check:
        from oracle import oracle

        want, _ = oracle.sort_text(cpu_sample(text, args.ref_sample_words), mode="fast")
        parity = payload == want
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": workload_name(args.config),
                   "sample_words": n_words, "l2_flush": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "physical_cores": physical_cores(), "kind": kind,
                         "sample": (f"first {n_words} words of the seeded config-{args.config} "
                                    f"text per step through {what}")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity_vs_oracle": parity,
    }
    print(json.dumps(line), flush=True)


# Kernel families of the step and the profiling records (ws_profile names) that
# time them; each record carries its launch's algorithmic bytes.
FAMILIES = {
    "ingest": ("ingest",),
    "radix_onesweep": ("radix_l0",),
    "radix_hist": ("radix_hist_l0",),
    "sample_split": ("split_l1", "split_l2", "split_l3", "split_l4"),
    "partition": ("part_count_l1", "part_count_l2", "part_count_l3", "part_count_l4",
                  "part_scatter_l1", "part_scatter_l2", "part_scatter_l3", "part_scatter_l4"),
    "slot_sort": ("subsort_l1", "subsort_l2", "subsort_l3", "subsort_l4"),
    "tiny_sort": ("tiny",),  # small corpora (<= 512 KiB): one CTA per bucket after the ingest
    # distinct-word counting (texts that repeat their vocabulary): every key read once
    # and counted; distinct keys sorted (tiles + rank merge); run prefixes; payload records
    # (two kernels, as in the ncu launch list: the uint32-key launch and the wider keys' launch)
    "count_aggregate": ("dd_aggregate",),
    "count_aggregate_wide": ("dd_aggregate_hi",),
    "count_sort_distinct": ("dd_tiles", "dd_tiles_hi", "dd_rank", "dd_rank_hi"),
    "count_run_prefix": ("dd_prefix", "dd_prefix_hi"),
    "count_expand": ("dd_expand", "dd_expand_hi"),
}
STATS_FAMILIES = {
    "stats_ingest": ("ingest", "reorder"),
    "stats_tile_sort": ("tile_l0", "tile_l1", "tile_l2", "tile_l3", "tile_l4"),
    # merge kernels alone, and the merge-path partition launches of the same levels
    "stats_merge": ("mergek_l0", "mergek_l1", "mergek_l2", "mergek_l3", "mergek_l4"),
    "stats_merge_partition": ("msplit_l0", "msplit_l1", "msplit_l2", "msplit_l3", "msplit_l4"),
}


def family_rows(phases: list, families: dict, steps: int, peak: float, workload: str,
                override_bytes: dict | None = None) -> dict:
    """Per kernel family: algorithmic bytes and CUDA-event time of its launches
    (profiled steps), achieved GB/s and the fraction of the measured peak."""
    rows = {}
    for fam, names in families.items():
        recs = [p for p in phases if p["name"] in names and p["launches"] > 0]
        ms = sum(p["ms"] for p in recs)
        nbytes = sum(p["bytes"] for p in recs)
        launches = sum(p["launches"] for p in recs)
        if override_bytes and fam in override_bytes:
            nbytes = override_bytes[fam]
        if ms <= 0 or launches == 0:
            continue
        ach = nbytes / (ms * 1e-3) / 1e9
        rows[fam] = {"ms_per_step": ms / steps, "launches_per_step": launches / steps,
                     "algorithmic_bytes_per_launch": nbytes / launches,
                     "ms_per_launch": ms / launches, "achieved": ach, "unit": "GB/s",
                     "frac": ach / peak, "traffic": ncu_traffic(workload, fam)}
    return rows


def bench_ours(args) -> None:
    import torch

    from paper_1407_6603_b200._native import Handle, device_bytes
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
    want = None
    if not args.no_check:
        from oracle import oracle

        want, _ = oracle.sort_text(text, mode="fast")  # checker only, outside every timed region

    # ---- device-resident leg --------------------------------------------
    h = Handle(local)
    h.ingest_text(text)  # places the text in HBM (untimed)
    lengths, counts, words = h.buckets()
    hist = dict(zip(lengths, counts))
    stream = torch.cuda.ExternalStream(h.stream(), device=dev)
    written = 0
    for _ in range(args.warmup):
        written = h.sort_resident(n)

    def profiled(step, hh, s) -> list:
        """K more steps with per-kernel CUDA events, kernels serialised on one
        stream so each event pair times one launch alone (not the timed steps)."""
        hh.profile(reset=True)
        hh.set_profiling(2)
        for _ in range(args.steps):
            with torch.cuda.stream(s):
                flush.zero_()
            torch.cuda.synchronize(dev)
            step()
        torch.cuda.synchronize(dev)
        hh.set_profiling(False)
        return hh.profile(reset=True)

    sampler = ClockSampler(local)
    dev_ms = []
    with sampler:
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
        counted = h.counted_classes()
        # the timed path's own output, byte-compared after the loop
        resident_ok = None
        if want is not None:
            resident_ok = device_bytes(*h.output_device()) == want
        phases = profiled(lambda: h.sort_resident(n), h, stream)

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
        single_ok = None if want is None else ts.payload(e2e_written) == want

        # ---- serving leg: the same corpus as a batch of K jobs through
        # ws_sort_texts, INFLIGHT in flight (H2D of one overlaps the sort and
        # D2H of the previous ones); every job's H2D and D2H is in the region,
        # every job writes its own pinned output buffer (all K checked)
        bs = BatchSorter(n, inflight=INFLIGHT, device=local, outputs=max(args.steps, INFLIGHT))
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
        batch_ok = None
        if want is not None:
            batch_ok = all(bs.payload(k, sz) == want for k, sz in enumerate(batch_sizes))

        # ---- stats leg: the reference's full SortStats semantics on the
        # device (order-preserving ingest, merge sort with inversion / K
        # counts, per-bucket stats read back), text already in HBM
        dtext = torch.frombuffer(bytearray(text), dtype=torch.uint8).to(dev)
        hsx = Handle(local)
        sstream = torch.cuda.ExternalStream(hsx.stream(), device=dev)

        def stats_step():
            hsx.ingest_text(None, device_ptr=dtext.data_ptr(), n=n)
            hsx.sort(True)
            return hsx.bucket_stats(True)

        for _ in range(args.warmup):
            stats_step()
        stats_ms = []
        for _ in range(args.steps):
            with torch.cuda.stream(sstream):
                flush.zero_()
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(sstream)
            st_rows = stats_step()
            b.record(sstream)
            torch.cuda.synchronize(dev)
            stats_ms.append(a.elapsed_time(b))
        stats_phases = profiled(stats_step, hsx, sstream)
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

    # ---- rooflines: every kernel family of the step (CUDA events per launch
    # in K profiled steps after the timed ones), against the measured peak.
    # The ingest's bytes are exact: text read once + every packed key written
    # once + 8 B per long-word entry; the others come from the library's
    # per-launch accounting (keys read + keys or payload records written).
    peak, peak_src = measured_peak()
    wl = workload_name(args.config)
    rows = family_rows(phases, FAMILIES, args.steps, peak, wl,
                       {"ingest": args.steps * ingest_algorithmic_bytes(n, hist)})
    stats_rows = family_rows(stats_phases, STATS_FAMILIES, args.steps, peak, wl)
    serial_ms = sum(r["ms_per_step"] for r in rows.values())
    roofline = None
    if rows:
        dom = max(rows, key=lambda k: rows[k]["ms_per_step"])  # largest serialised share
        d = rows[dom]
        roofline = {"bound": "hbm", "kernel": dom, "achieved": d["achieved"], "peak": peak,
                    "unit": "GB/s", "frac": d["frac"],
                    "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                    "traffic": d["traffic"],
                    "algorithmic_bytes_per_launch": d["algorithmic_bytes_per_launch"],
                    "ms_per_launch": d["ms_per_launch"],
                    "share_of_step": d["ms_per_step"] / serial_ms if serial_ms else None,
                    "timing": "CUDA events per launch over K profiled steps after the timed ones, "
                              "kernels serialised on one stream"}
        for r in rows.values():
            r["share_of_step"] = r["ms_per_step"] / serial_ms if serial_ms else None

    parity = None
    cpu = None
    if rank == 0:
        if want is not None:
            parity = bool(resident_ok and single_ok and batch_ok)
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            port, _, _, port_payload = run_cpu(text, args.cpu_sample_words, threads, hist)
            ref = run_reference(text, args.cpu_sample_words, threads)
            if ref is not None:  # the reference's own numba path, beside the port
                dt, nw, ref_payload = ref
                cpu = {"value": nw / dt, "unit": UNIT, "cores": threads,
                       "physical_cores": physical_cores(), "kind": "reference",
                       "sample": (f"first {nw} words of the same seeded text through the "
                                  "unmodified reference (baseline/_ref wordsort: tokenize, "
                                  "build_store flat, sort_all_parallel NAIVE/STATIC with the "
                                  "numba _bubble_rows on a thread pool, emit_sorted, payload join)"),
                       "seconds": dt, "payload_equals_port": ref_payload == port_payload,
                       "port": port}
            else:
                cpu = port

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_dev, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": wl, "words": words,
                       "text_bytes": n, "payload_bytes": written, "buckets": len(lengths),
                       "l2_flush": "256 MiB memset on the timed stream between steps",
                       "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                       # lane classes (bit c: words of 1-5 / 6-10 / 11-21 / 22-32 characters) whose
                       # payload came from counting distinct words, not from sorting every occurrence
                       "counted_classes": counted},
            "e2e": {"value": batch_value, "unit": UNIT, "h2d_bytes_per_step": n,
                    "d2h_bytes_per_step": batch_sizes[0] if batch_sizes else 0,
                    "ms_per_step": t_batch, "gpu_launches": batch_launches,
                    "api": f"ws_sort_texts, batch of {args.steps} corpora, {INFLIGHT} in flight, "
                           "pinned host buffers (one output buffer per corpus), wall clock "
                           "around the call",
                    "single": {"value": e2e_value, "ms_per_step": t_e2e,
                               "gpu_launches": e2e_launches,
                               "api": "ws_sort_text, one corpus per call, CUDA events"}},
            "stats_mode": {"value": world * words / (t_stats * 1e-3), "unit": UNIT,
                           "ms_per_step": t_stats, "roofline_rows": stats_rows,
                           "api": "ws_ingest_text(DEVICE_PTR) + ws_sort(h, 1) + ws_bucket_stats: "
                                  "corpus-order buckets, merge sort counting inversions and K, "
                                  "the reference's SortStats per bucket"},
            "roofline": roofline,
            "roofline_rows": rows,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
            "parity_vs_oracle": parity,
            "parity_detail": {"resident_output": resident_ok, "single_call": single_ok,
                              "batch_all_outputs": batch_ok,
                              "batch_outputs_checked": len(batch_sizes)},
        }
        line["e2e_timeline_ms"] = [[p["name"], round(p["start_ms"], 3), round(p["ms"], 3),
                                    int(p["bytes"])] for p in e2e_phases]
        if args.profile_json:
            Path(args.profile_json).write_text(json.dumps({"phases": phases, "steps": args.steps,
                                                           "stats_phases": stats_phases,
                                                           "dev_ms": dev_ms, "e2e_ms": e2e_ms,
                                                           "e2e_phases": e2e_phases},
                                                          indent=1))
        print(json.dumps(line), flush=True)
    if world == 1:
        # The line is out: leave without tearing down the handles, the CUDA
        # context or the reference's numba pool (a teardown after the line
        # crashed twice on fresh boxes; faulthandler reports where if it recurs
        # on the multi-rank path below).
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    ts.close()
    bs.close()
    hsx.close()
    h.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    import faulthandler
    faulthandler.enable()
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
    # The JSON line is out. Skip interpreter teardown: with the reference's
    # numba thread pool and the CUDA context both alive, teardown crashed once
    # (SIGSEGV after the line was printed) on a fresh box.
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
