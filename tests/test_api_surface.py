"""The drop-in surface without a GPU: every name the reference exports
(gridwave/__init__.py:51-92) is exported here, the rule types state the
reference rules on the host, and the pipeline's config contract holds."""

import numpy as np
import pytest

import paper_1209_3314_b200 as gw

# gridwave/__init__.py:51-92 (__all__), verbatim names
REFERENCE_ALL = [
    "BG", "FG", "Coord", "Image2D", "StructuringElement", "axis_half_neighbors",
    "half_neighbors", "neighbors", "ContractViolation", "EngineError", "GridwaveError",
    "NoBackgroundError", "PgmFormatError", "EngineConfig", "PropagationRule", "RunStats",
    "QueueConfig", "QueueStrategy", "ReconInput", "recon_fh", "recon_parallel", "recon_qb",
    "recon_sr", "recon_tiled", "regional_maxima", "VoronoiMap", "edt", "edt_exact_bruteforce",
    "edt_init", "edt_tiled", "finalize_distance_map", "MicroConfig", "PipelineConfig",
    "TileGrid", "partition", "run_pipeline", "BenchReport", "run_experiment", "to_csv",
    "to_json", "SuiteResult", "run_suites",
]


def test_reference_export_list_is_covered():
    missing = [n for n in REFERENCE_ALL if not hasattr(gw, n)]
    assert not missing
    assert set(REFERENCE_ALL) <= set(gw.__all__)


def test_module_level_reference_names():
    # recon.py / edt.py module names callers import directly
    import importlib
    recon = importlib.import_module("paper_1209_3314_b200.recon")
    edt = importlib.import_module("paper_1209_3314_b200.edt")
    tiles = importlib.import_module("paper_1209_3314_b200.tiles")
    for n in ("ReconRule", "raster_pass", "antiraster_pass", "parallel_sweeps"):
        assert hasattr(recon, n), n
    for n in ("DistanceRule", "init_packed", "edt_propagate"):
        assert hasattr(edt, n), n
    assert hasattr(tiles, "EventRecord")


def test_recon_rule_hooks_state_the_reference_rule():
    J = np.array([[5, 0], [0, 9]], np.uint8)
    I = np.array([[5, 3], [7, 9]], np.uint8)
    r = gw.ReconRule(J, I, gw.SE8)
    assert r.condition(0, 1) and r.propose(0, 1) == 3       # raised to its mask
    assert not r.condition(1, 0)                               # 0 < 5: no raise
    assert r.condition(3, 2) and r.propose(3, 2) == 7
    assert r.improves(1, 0, 3) and not r.improves(1, 3, 3)
    assert list(r.iter_neighbors(0)) == [1, 2, 3]


def test_distance_rule_total_order():
    vr = np.full((3, 4), -1, np.int64)
    r = gw.DistanceRule(vr, gw.SE8)
    # q = (1,1): sources (0,0) [packed 0] and (2,2) [packed 10] are both at d2 = 2
    q = 1 * 4 + 1
    assert r.closer(q, 0, 10) and not r.closer(q, 10, 0)   # tie: smaller index wins
    assert r.closer(q, 0, -1) and not r.closer(q, -1, 0)   # anything beats unset
    assert r.sqdist(q, -1) == 1 << 62


def test_pipeline_rejects_foreign_rules_and_bad_tiles():
    img = gw.Image2D(4, 4, "u8", np.zeros((4, 4), np.uint8))

    class Custom(gw.PropagationRule):
        pass

    with pytest.raises(gw.ContractViolation):
        gw.run_pipeline(img, Custom(4, 4, gw.SE8), lambda: [], (2, 2))
    rule = gw.ReconRule(img.data, img.data, gw.SE8)
    with pytest.raises(gw.ContractViolation):
        gw.run_pipeline(img, rule, lambda: [], (0, 2))
    with pytest.raises(gw.ContractViolation):
        gw.run_pipeline(img, rule, lambda: [], (2, 2), gw.PipelineConfig(max_waves=0))


def test_event_record_line():
    from paper_1209_3314_b200.tiles import EventRecord
    import json
    e = EventRecord(3, "TP", 1, -1, 0, 1.0, 2.0)
    assert json.loads(e.to_line()) == {"task": 3, "kind": "TP", "wave": 1, "tile": -1,
                                       "worker": 0, "start": 1.0, "end": 2.0}
