"""Host-side logic that runs without a GPU: generators, API types, bench
plumbing, and the multi-process (gloo) replica harness."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1407_6603_b200 import synth
from paper_1407_6603_b200.engine import SchedulePolicy, SortConfig, SortStats, SortVariant, compare_words
from paper_1407_6603_b200.store import FlatBucketMatrix, LayoutKind, build_buckets, emit_sorted

ROOT = Path(__file__).resolve().parent.parent


def test_generators_are_frozen(golden_configs):
    from conftest import config_text

    for key, rec in golden_configs.items():
        assert __import__("hashlib").sha256(config_text(rec)).hexdigest() == rec["text_sha"], key


def test_config_shapes():
    import re

    word = re.compile(rb"[A-Za-z0-9]+")
    t0 = synth.generate(0)
    w0 = word.findall(t0)
    assert 170_000 < len(t0) < 210_000 and len(w0) == 35_000
    lens = np.array([len(w) for w in w0])
    assert 3.9 < lens.mean() < 4.5 and 0.06 < (lens >= 8).mean() < 0.10 and lens.max() <= 14
    pmf = synth.config4_length_pmf()
    assert abs(pmf[5] - 0.4) < 1e-12 and abs(pmf.sum() - 1) < 1e-12
    t4 = synth.generate(4, words=50_000)
    assert len(word.findall(t4)) == 50_000


def test_prefix_cut():
    t = synth.generate(4, words=1000)
    p = synth.prefix(t, 10)
    assert p.count(b" ") + p.count(b"\n") == 10 and t.startswith(p)


def test_sort_types_mirror_reference():
    with pytest.raises(ValueError):
        SortConfig(LayoutKind.RAGGED, SortVariant.NAIVE, threads=0)
    c = SortConfig(LayoutKind.FLAT)
    assert c.variant is SortVariant.NAIVE and c.threads == 1 and c.schedule is SchedulePolicy.STATIC_BLOCK
    assert SortStats(1, 2, 3) + SortStats(4, 5, 6) == SortStats(5, 7, 9)
    assert compare_words(b"Zoo", b"abc") == -1 and compare_words(b"dog", b"dog") == 0
    with pytest.raises(AssertionError):
        compare_words(b"a", b"ab")
    assert SortVariant("early-exit") is SortVariant.EARLY_EXIT


def test_ragged_store_and_emit_are_host_containers():
    s = build_buckets([b"a", b"abc", b"b"])
    assert s.buckets == {1: [b"a", b"b"], 3: [b"abc"]} and s.lmax == 3 and s.word_count == 3
    assert emit_sorted(s) == [b"a", b"b", b"abc"]
    m = FlatBucketMatrix({2: np.frombuffer(b"abcd", np.uint8).reshape(2, 2)})
    assert m.words_for_length(2) == [b"ab", b"cd"] and m.count_for_length(3) == 0


def test_bench_extrapolation_helper():
    sys.path.insert(0, str(ROOT))
    import bench

    # bucket of 1000 words took 1 s on the sample; full bucket 2000 words
    sec = bench.extrapolate({5: 2000}, {5: (1000,)}, {5: 1.0}, threads=4)
    assert abs(sec - 1.0 * 2000 * 1999 / (1000 * 999)) < 1e-9
    # LPT makespan over 2 threads
    sec = bench.extrapolate({1: 10, 2: 10, 3: 10}, {1: (10,), 2: (10,), 3: (10,)},
                            {1: 3.0, 2: 2.0, 3: 2.0}, threads=2)
    assert abs(sec - 4.0) < 1e-9


WORKER = r"""
import os, sys, json
sys.path.insert(0, sys.argv[1])
import torch, torch.distributed as dist
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
import bench
from paper_1407_6603_b200 import synth
# every rank builds its own replica corpus (bench.corpus seeds by rank; a
# small word count stands in for config 4), no data exchange, weak scaling
text = synth.generate(0, seed=synth.BASE_SEED + 7919 * rank, words=2000)
ms = 10.0 + rank  # per-rank step time: the job's time is the slowest rank's
t_job = bench.reduce_over_ranks(ms, world, torch.device("cpu"), "max")
words = bench.reduce_over_ranks(2000.0, world, torch.device("cpu"), "sum")
lens = [None] * world
dist.all_gather_object(lens, len(text))
if rank == 0:
    print(json.dumps({"t_job": t_job, "words": words, "lens": lens}))
dist.barrier()
dist.destroy_process_group()
"""


def test_replica_harness_gloo_world2(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, str(script), str(ROOT)], env=e,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    res = json.loads(outs[0][0].strip().splitlines()[-1])
    assert res["t_job"] == 11.0 and res["words"] == 4000.0
    assert res["lens"][0] != res["lens"][1]  # distinct replica corpora


def test_counting_layout_fits_its_allocation_bounds(tmp_path):
    """csrc/plan.cuh: for any split of a text into words of 1..32 characters the
    counting path's tables, distinct-key lists and per-distinct-word arrays
    (dd_layout) fit what the host allocates and zeroes before the counts are
    known (dd_max_*); the same header is compiled into the kernels."""
    import subprocess

    root = Path(__file__).resolve().parent.parent
    exe = tmp_path / "dd_plan_bounds"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{root / 'paper_1407_6603_b200' / 'csrc'}",
                    str(root / "tests" / "cpp" / "dd_plan_bounds.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
