"""Host-side parts of the harness (no GPU): the BenchReport CSV/JSON forms
(reference gridwave/bench.py:24-66), the verify report line and suite list
(gridwave/verify.py), and the CLI parser (gridwave/cli.py)."""

import json

import pytest

from paper_1209_3314_b200.cli import build_parser, dims as _parse_dims
from paper_1209_3314_b200.errors import ContractViolation
from paper_1209_3314_b200.experiments import CSV_COLUMNS, EXPERIMENTS, BenchReport, to_csv, to_json
from paper_1209_3314_b200.verify import SUITES, SuiteResult


def test_csv_columns_match_the_reference_order():
    assert CSV_COLUMNS == ("experiment", "variant", "workers", "tile_dims", "queue_strategy",
                           "coverage_pct", "wall_time_ms", "rounds", "bp_waves", "queued_total",
                           "overflow_count", "speedup_vs_1worker")
    assert set(EXPERIMENTS) == {"queue", "tilesize", "coverage", "overflow", "scaling"}


def test_csv_and_json_mirror_each_other():
    rows = [BenchReport("queue", "edt_parallel", 1, queue_strategy="naive", wall_time_ms=1.23456,
                        rounds=3, queued_total=10),
            BenchReport("scaling", "recon", 4, tile_dims="32x32", speedup_vs_1worker=None)]
    lines = to_csv(rows).strip().splitlines()
    objs = json.loads(to_json(rows))
    assert lines[0] == ",".join(CSV_COLUMNS)
    assert lines[1].split(",")[6] == "1.235"  # floats to 3 places
    assert lines[2].split(",")[-1] == ""  # None -> empty cell
    assert [set(o) for o in objs] == [set(CSV_COLUMNS)] * 2


def test_suite_line_and_names():
    assert SUITES == ("recon", "edt", "queue", "tiling")
    assert SuiteResult("recon", 4, 0).line() == "recon: 4/4 pass"
    assert not SuiteResult("edt", 3, 1).ok


def test_parser_subcommands_and_defaults():
    ap = build_parser()
    a = ap.parse_args(["recon", "--mask", "m.pgm", "--auto-marker", "40", "--out", "o.pgm"])
    assert (a.algo, a.conn, a.tile, a.queue, a.gbq_capacity) == ("fh", 8, "64x64", "perworker", "auto")
    a = ap.parse_args(["edt", "--input", "i.pgm", "--out", "d.f32", "--mode", "tiled"])
    assert a.mode == "tiled"
    a = ap.parse_args(["verify"])
    assert (a.suite, a.cases, a.size) == ("all", 25, "64x64")
    a = ap.parse_args(["bench", "--experiment", "queue"])
    assert (a.size, a.workers) == ("512x512", 4)
    with pytest.raises(SystemExit):
        ap.parse_args(["recon", "--mask", "m.pgm", "--out", "o.pgm"])  # marker source required


def test_parse_dims():
    assert _parse_dims("16x32") == (16, 32)
    for bad in ("16by16", "0x4", "x"):
        with pytest.raises(ContractViolation):
            _parse_dims(bad)
