"""The verify / bench harness on the B200 (reference: gridwave/verify.py,
gridwave/bench.py; cases mirror pkg/tests/test_cli.py verify / bench)."""

import json

import pytest

from paper_1209_3314_b200.cli import main
from paper_1209_3314_b200.experiments import CSV_COLUMNS, run_experiment, to_csv, to_json
from paper_1209_3314_b200.verify import run_suites

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _dev():
    import torch
    torch.cuda.set_device(0)


def test_verify_suites_pass_and_exit_0(capsys):
    assert main(["verify", "--suite", "all", "--cases", "4", "--size", "32x32", "--seed", "5"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines == ["recon: 4/4 pass", "edt: 4/4 pass", "queue: 4/4 pass", "tiling: 4/4 pass"]


def test_verify_larger_instances(capsys):
    assert main(["verify", "--suite", "all", "--cases", "6", "--size", "300x257", "--seed", "1"]) == 0


def test_verify_is_deterministic():
    a = run_suites("recon", 6, 9, (32, 32))
    b = run_suites("recon", 6, 9, (32, 32))
    assert [(r.passed, r.failed) for r in a] == [(r.passed, r.failed) for r in b]


def test_verify_single_suite(capsys):
    assert main(["verify", "--suite", "queue", "--cases", "10"]) == 0
    assert capsys.readouterr().out.strip() == "queue: 10/10 pass"


def test_bench_queue_counters_agree(tmp_path, capsys):
    out_json = tmp_path / "r.json"
    assert main(["bench", "--experiment", "queue", "--size", "96x96", "--json", str(out_json)]) == 0
    rows = json.loads(out_json.read_text())
    assert [r["queue_strategy"] for r in rows] == ["naive", "prefix_sum", "per_worker"]
    assert len({r["queued_total"] for r in rows}) == 1
    assert len({r["rounds"] for r in rows}) == 1
    assert capsys.readouterr().out.splitlines()[0] == ",".join(CSV_COLUMNS)


def test_bench_coverage_zero_queues_nothing():
    rows = run_experiment("coverage", size=(64, 64), seed=3, workers=2)
    by_pct = {r.coverage_pct: r for r in rows}
    assert by_pct[0].queued_total == 0
    assert by_pct[50].queued_total > 0


def test_bench_scaling_reports_speedup_column():
    rows = run_experiment("scaling", size=(1024, 1024), seed=1, workers=4)
    assert [r.workers for r in rows] == [1, 2, 4]
    assert rows[0].speedup_vs_1worker == 1.0
    assert all(r.speedup_vs_1worker is not None for r in rows)


def test_bench_overflow_reports_overflows():
    rows = run_experiment("overflow", size=(96, 96), seed=2, workers=2)
    assert rows[0].overflow_count == 0
    assert rows[1].overflow_count >= 2


def test_bench_csv_and_json_mirror_each_other():
    rows = run_experiment("tilesize", size=(256, 256), seed=4, workers=2)
    csv_lines = to_csv(rows).strip().splitlines()
    parsed = json.loads(to_json(rows))
    assert len(csv_lines) == len(parsed) + 1 == 5
    assert csv_lines[0] == ",".join(CSV_COLUMNS)
    for line, obj in zip(csv_lines[1:], parsed):
        assert set(obj) == set(CSV_COLUMNS)
        cells = line.split(",")
        assert cells[0] == obj["experiment"]
        assert cells[3] == obj["tile_dims"]
        assert int(cells[2]) == obj["workers"]
