"""Timing-matrix harness (mirror of the reference's wordsort.bench): report
schema, derived columns and round trips on CPU; the device-timed matrix and
the CLI `bench` command on the GPU."""

import json

import pytest

from paper_1407_6603_b200 import harness
from paper_1407_6603_b200.engine import SortConfig, SortVariant
from paper_1407_6603_b200.harness import (BenchError, BenchReport, TimingRow, compute_efficiency,
                                          compute_speedup, derive, emit_report, parse_csv,
                                          render_csv, render_json, render_plot_data)
from paper_1407_6603_b200.store import LayoutKind
from paper_1407_6603_b200 import synth

TIMES = {1: (8.0, 120.0), 2: (5.0, 70.0), 4: (4.0, 40.0), 8: (3.2, 30.0)}


def _report():
    rows = []
    for t, (a, b) in TIMES.items():
        rows.append(TimingRow("ds1", LayoutKind.FLAT, SortVariant.NAIVE, t, [a, a]))
        rows.append(TimingRow("ds2", LayoutKind.RAGGED, SortVariant.EARLY_EXIT, t, [b]))
    return derive(BenchReport(rows=rows, meta={"reps": 2}))


def test_speedup_and_efficiency():
    assert compute_speedup(8.0, 3.2) == pytest.approx(2.5)
    assert compute_efficiency(2.5, 8) == pytest.approx(0.3125)
    assert compute_speedup(1.5, 1.5) == 1.0
    for bad in ((0.0, 1.0), (1.0, 0.0), (-1.0, 2.0)):
        with pytest.raises(ValueError):
            compute_speedup(*bad)
    with pytest.raises(ValueError):
        compute_efficiency(1.0, 0)
    with pytest.raises(ValueError):
        compute_efficiency(0.0, 2)


def test_derive_against_group_baseline():
    rep = _report()
    for r in rep.rows:
        base = TIMES[1][0] if r.dataset == "ds1" else TIMES[1][1]
        assert r.speedup * r.mean_seconds == pytest.approx(base)
        assert r.efficiency * r.threads == pytest.approx(r.speedup)
    orphan = derive(BenchReport(rows=[TimingRow("x", LayoutKind.FLAT, SortVariant.NAIVE, 4, [1.0])]))
    assert orphan.rows[0].speedup is None and orphan.rows[0].efficiency is None


def test_csv_round_trip_and_ragged_runs():
    rep = _report()
    text = render_csv(rep)
    head = text.splitlines()[0].split(",")
    assert head[:7] == ["dataset", "layout", "variant", "threads", "mean_seconds", "speedup",
                        "efficiency"]
    assert head[7:] == ["run_1", "run_2"]
    back = parse_csv(text)
    assert [(r.dataset, r.layout, r.variant, r.threads, r.runs, r.speedup, r.efficiency)
            for r in back.rows] == [(r.dataset, r.layout, r.variant, r.threads, r.runs,
                                     r.speedup, r.efficiency) for r in rep.rows]
    assert parse_csv("").rows == []


def test_json_and_plot_files():
    rep = _report()
    d = json.loads(render_json(rep))
    assert d["meta"] == {"reps": 2} and len(d["rows"]) == len(rep.rows)
    assert set(d["rows"][0]) == {"dataset", "layout", "variant", "threads", "runs",
                                 "mean_seconds", "speedup", "efficiency"}
    files = render_plot_data(rep)
    assert set(files) == {"speedup_ds1_flat_naive.dat", "time_ds1_flat_naive.dat",
                          "speedup_ds2_ragged_early-exit.dat", "time_ds2_ragged_early-exit.dat"}
    lines = files["time_ds1_flat_naive.dat"].splitlines()
    assert [int(l.split()[0]) for l in lines] == sorted(TIMES)
    assert emit_report(rep, "csv") == render_csv(rep).encode()
    assert emit_report(rep, "json") == render_json(rep).encode()
    assert set(emit_report(rep, "plot")) == set(files)
    with pytest.raises(ValueError):
        emit_report(rep, "xml")


def test_time_sort_rejects_zero_reps():
    with pytest.raises(ValueError):
        harness.time_sort([], SortConfig(LayoutKind.FLAT), reps=0)


def test_run_matrix_unreadable_dataset(tmp_path):
    with pytest.raises(BenchError, match="ghost"):
        harness.run_matrix([("ghost", tmp_path / "missing.txt")], [LayoutKind.FLAT],
                           [SortVariant.NAIVE], [1])


@pytest.mark.gpu
def test_time_sort_and_matrix_on_device(tmp_path):
    words = synth.random_words(7, 3000, max_len=12)
    row = harness.time_sort(words, SortConfig(LayoutKind.FLAT), reps=3, warmups=1)
    assert len(row.runs) == 3 and all(t > 0 for t in row.runs)
    assert len(harness.time_sort([], SortConfig(LayoutKind.RAGGED), reps=2, warmups=0).runs) == 2
    corpus = tmp_path / "tiny.txt"
    corpus.write_bytes(b" ".join(words))
    rep = harness.run_matrix([("tiny", corpus)], [LayoutKind.FLAT, LayoutKind.RAGGED],
                             [SortVariant.NAIVE], [2, 4], reps=2, warmups=0)
    assert [(r.layout.value, r.threads) for r in rep.rows] == [
        ("flat", 1), ("flat", 2), ("flat", 4), ("ragged", 1), ("ragged", 2), ("ragged", 4)]
    assert rep.meta["backend"] == "b200" and rep.meta["threads"] == [1, 2, 4]
    for r in rep.rows:
        assert r.speedup is not None and r.efficiency * r.threads == pytest.approx(r.speedup)


@pytest.mark.gpu
def test_cli_bench_formats(tmp_path, capsys):
    from paper_1407_6603_b200.cli import main

    corpus = tmp_path / "c.txt"
    corpus.write_bytes(b" ".join(synth.random_words(3, 2000, max_len=9)))
    out = tmp_path / "r.csv"
    assert main(["bench", str(corpus), "--layout", "flat", "--threads", "1,2", "--reps", "1",
                 "--warmups", "0", "--output", str(out)]) == 0
    rep = parse_csv(out.read_text())
    assert [r.threads for r in rep.rows] == [1, 2]
    assert main(["bench", str(corpus), "--layout", "flat", "--threads", "1", "--reps", "1",
                 "--warmups", "0", "--format", "plot", "--output", str(tmp_path / "p")]) == 0
    assert sorted(p.name for p in (tmp_path / "p").iterdir()) == ["speedup_c_flat_naive.dat",
                                                                  "time_c_flat_naive.dat"]
    assert main(["bench", str(tmp_path / "nope.txt")]) == 1
