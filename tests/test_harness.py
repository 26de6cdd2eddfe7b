"""CPU: the harness's host pieces against the reference (tests/golden/harness.json,
made by tests/golden/make_harness_golden.py): the RMAT / planted-partition
samplers draw for draw, RunConfig validation and its report `config` object,
and the JSON / CSV report writers (test_bench.py:31-47, :156-176)."""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2305_17408_b200 import generators as G
from paper_2305_17408_b200.harness import emit_report, parse_report
from paper_2305_17408_b200.pipeline import RunConfig

H = json.loads((GOLDEN / "harness.json").read_text())


def _digest(keys):
    return hashlib.sha256(np.ascontiguousarray(keys, dtype=np.int64).tobytes()).hexdigest()


@pytest.mark.parametrize("case", H["rmat"], ids=lambda c: f"V{c['V']}E{c['E']}")
def test_rmat_matches_reference(case):
    keys = G.rmat_keys(case["V"], case["E"], tuple(case["probs"]), case["seed"])
    assert keys.size == case["E"]
    assert keys[:16].tolist() == case["head"]
    assert _digest(keys) == case["sha256"]


@pytest.mark.parametrize("case", H["planted"], ids=lambda c: f"g{c['groups']}s{c['size']}")
def test_planted_matches_reference(case):
    d, s, labels = G.planted_edges(case["groups"], case["size"], case["p_in"], case["p_out"],
                                   case["seed"], case["shuffle"])
    n = case["groups"] * case["size"]
    keys = np.unique(d.astype(np.int64) * n + s)
    assert keys.size == case["num_edges"]
    assert _digest(keys) == case["sha256"]
    assert labels.tolist() == case["labels"]


def test_generator_argument_errors():
    with pytest.raises(ValueError, match="num_vertices must be positive"):
        G.rmat_keys(0, 0)
    with pytest.raises(ValueError, match="sum to 1"):
        G.rmat_keys(8, 4, (0.5, 0.5, 0.5, 0.0))
    with pytest.raises(ValueError, match="cannot place"):
        G.rmat_keys(4, 17)
    with pytest.raises(ValueError, match=">= 1"):
        G.planted_edges(0, 4, 0.5, 0.1)
    assert G.rmat_keys(4, 16).tolist() == list(range(16))  # complete graph


def test_run_config_validation_and_dict():
    with pytest.raises(ValueError):
        RunConfig(mode="O4")
    with pytest.raises(ValueError):
        RunConfig(rmat=(16, 32), planted=(2, 4, 0.5, 0.1))
    for case in H["pipeline"]:
        kw = {k: tuple(v) if isinstance(v, list) else v for k, v in case["kwargs"].items()}
        assert RunConfig(**kw).as_dict() == case["report"]["config"]
    assert list(RunConfig().as_dict()) == list(H["density"][0]["report"]["config"])


def test_json_round_trip(tmp_path):
    report = {"a": 1, "b": [1, 2], "c": {"d": None}}
    path = emit_report(report, "json", tmp_path / "r.json")
    assert parse_report(path, "json") == report


def test_csv_round_trip_and_empty(tmp_path):
    rows = [{"x": 1, "y": "a"}, {"x": 2, "y": "b"}]
    path = emit_report(rows, "csv", tmp_path / "r.csv")
    assert parse_report(path, "csv") == [{"x": "1", "y": "a"}, {"x": "2", "y": "b"}]
    emit_report([], "csv", tmp_path / "e.csv")
    assert (tmp_path / "e.csv").read_text().strip() == "empty"


def test_bad_format(tmp_path):
    with pytest.raises(ValueError):
        emit_report({}, "xml", tmp_path / "r.xml")
    with pytest.raises(ValueError, match="list of row dicts"):
        emit_report({"a": 1}, "csv", tmp_path / "r.csv")
    with pytest.raises(ValueError):
        parse_report(tmp_path / "r.xml", "xml")


def test_threaded_candidates_equal_single_call():
    """oracle/synth.py's chunked thread-pool candidate draw (used to build the
    C5 graph for the host baseline) equals one vectorised call."""
    from oracle import synth as osynth
    n = (1 << 20) + 12345
    args = (100_000, 16, 0.4, 0.05, 16, 1, 3)
    d1, s1 = osynth.candidates(*args, 0, n)
    d2, s2 = osynth._candidates_threaded(*args, n, threads=5)
    assert np.array_equal(d1, d2) and np.array_equal(s1, s2)
