"""CPU: selector state machine (reference selector.py:46-154), pure host logic.

Timings are injected synthetically like the reference's `drive` helper
(test_selector.py:22-33); no kernels run.
"""
import statistics

import numpy as np
import pytest

from paper_2305_17408_b200.kernels import AggregateOp, KernelKind
from paper_2305_17408_b200.selector import (
    INTER,
    INTRA,
    ChoiceCache,
    Phase,
    SelectorError,
    SelectorState,
    plan_iteration,
    record_timing,
)

KEYS = ((INTRA, KernelKind.CSR_INTRA_BLOCKED), (INTRA, KernelKind.DENSE_BLOCK),
        (INTER, KernelKind.CSR_INTER), (INTER, KernelKind.COO_ATOMIC))


def drive(s, table):
    feed = {k: list(v) for k, v in table.items()}
    i = 0
    while s.phase is Phase.PROFILING:
        plan = plan_iteration(s, i)
        s = record_timing(s, INTRA, plan.kernel_intra, feed[(INTRA, plan.kernel_intra)].pop(0))
        if s.phase is Phase.PROFILING:
            s = record_timing(s, INTER, plan.kernel_inter, feed[(INTER, plan.kernel_inter)].pop(0))
        i += 1
    return s, i


def test_defaults():
    s = SelectorState.fresh(AggregateOp.SUM)
    assert s.candidates_intra == (KernelKind.CSR_INTRA_BLOCKED, KernelKind.DENSE_BLOCK)
    assert s.candidates_inter == (KernelKind.CSR_INTER, KernelKind.COO_ATOMIC)
    assert s.total_profiling_iters == 6


def test_max_drops_dense_block():
    s = SelectorState.fresh(AggregateOp.MAX)
    assert KernelKind.DENSE_BLOCK not in s.candidates_intra


def test_bad_profile_iters():
    with pytest.raises(ValueError):
        SelectorState.fresh(AggregateOp.SUM, profile_iters_per_candidate=0)


def test_round_robin_then_lock():
    s = SelectorState.fresh(AggregateOp.SUM)
    plans = [plan_iteration(s, i) for i in range(4)]
    assert [p.kernel_intra for p in plans] == [KernelKind.CSR_INTRA_BLOCKED,
                                               KernelKind.DENSE_BLOCK] * 2
    table = {k: [10.0, 10.0, 10.0] for k in KEYS}
    table[(INTRA, KernelKind.DENSE_BLOCK)] = [1.0, 2.0, 3.0]
    s, iters = drive(s, table)
    assert iters == 6
    assert s.choice_intra is KernelKind.DENSE_BLOCK
    assert s.choice_inter is KernelKind.CSR_INTER  # tie -> list order
    assert not plan_iteration(s, 99).is_profiling


def test_record_after_lock_and_unknown_candidate():
    s = SelectorState.fresh(AggregateOp.SUM)
    with pytest.raises(SelectorError):
        record_timing(s, INTRA, KernelKind.COO_ATOMIC, 1.0)
    s, _ = drive(s, {k: [1.0] * 3 for k in KEYS})
    with pytest.raises(SelectorError):
        record_timing(s, INTRA, KernelKind.DENSE_BLOCK, 1.0)


def test_functional_state():
    s = SelectorState.fresh(AggregateOp.SUM)
    s2 = record_timing(s, INTRA, KernelKind.CSR_INTRA_BLOCKED, 5.0)
    assert s.timings == {} and s2.timings != {}


def test_argmin_median_matches_bruteforce():
    rng = np.random.default_rng(505)
    for _ in range(300):
        s = SelectorState.fresh(AggregateOp.SUM)
        table = {k: rng.uniform(1.0, 1000.0, size=3).tolist() for k in KEYS}
        s, _ = drive(s, table)
        for role, cands, got in ((INTRA, s.candidates_intra, s.choice_intra),
                                 (INTER, s.candidates_inter, s.choice_inter)):
            meds = [statistics.median(table[(role, k)]) for k in cands]
            assert got is cands[int(np.argmin(meds))]


def test_unequal_candidate_counts_lock():
    s = SelectorState.fresh(AggregateOp.MAX)  # 1 intra vs 2 inter candidates
    s, iters = drive(s, {k: [1.0, 2.0, 3.0] * 2 for k in KEYS})
    assert s.phase is Phase.LOCKED and iters == 6


def test_choice_cache_roundtrip(tmp_path):
    s, _ = drive(SelectorState.fresh(AggregateOp.SUM), {k: [1.0] * 3 for k in KEYS})
    c = ChoiceCache(tmp_path / "choices.json")
    key = ChoiceCache.key("g0", AggregateOp.SUM, 64)
    c.put(key, s)
    s2 = ChoiceCache(tmp_path / "choices.json").get(key)
    assert s2.phase is Phase.LOCKED and s2.total_profiling_iters == 0
    assert (s2.choice_intra, s2.choice_inter) == (s.choice_intra, s.choice_inter)
    with pytest.raises(SelectorError):
        c.put(key, SelectorState.fresh(AggregateOp.SUM))


def test_choice_cache_run_pair_and_counts(tmp_path):
    s, _ = drive(SelectorState.fresh(AggregateOp.SUM), {k: [1.0] * 3 for k in KEYS})
    c = ChoiceCache(tmp_path / "sub" / "choices.json")
    key = ChoiceCache.key("g1", AggregateOp.SUM, 48, "bwd")
    assert key.endswith("|bwd") and c.get(key) is None and c.misses == 1
    run = (KernelKind.DENSE_BLOCK, KernelKind.COO_ATOMIC)
    c.put(key, s, run=run)
    c2 = ChoiceCache(tmp_path / "sub" / "choices.json")
    assert c2.get_run(key) == run and c2.get(key) is not None and c2.hits == 1
    assert c2.get_run(ChoiceCache.key("g1", AggregateOp.SUM, 48, "fwd")) is None
