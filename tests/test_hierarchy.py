"""The GRINNDER tier session (hierarchy.py) reproduces the reference's byte
ledger event for event (golden ledgers from grinder.simulate.simulate_epoch,
tests/golden/ledger_cases.npz)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2605_11517_b200 as g2
from paper_2605_11517_b200.hierarchy import (CacheState, HierarchyConfig, PolicySpec, TierSession,
                                             ledger_summary, schedule_partitions, simulate_epoch)

CASES = ["layer_lru", "partition_lru", "vertex", "no_bypass", "tight"]


@pytest.fixture(scope="module")
def ledger_golden():
    z = np.load(GOLDEN / "ledger_cases.npz")
    return {k: z[k] for k in z.files}


def _plan(gold):
    g = g2.generate_kronecker(7, 6, seed=3)
    plan = g2.build_partition_plan(g, gold["labels"], 4)
    return plan


@pytest.mark.parametrize("name", CASES)
def test_simulated_ledger_matches_reference(ledger_golden, name):
    plan = _plan(ledger_golden)
    cfg = HierarchyConfig(**json.loads(str(ledger_golden[f"{name}/config"])))
    pol = PolicySpec("GRINNDER", bypass_enabled=name != "no_bypass")
    led = simulate_epoch(plan, [6, 5, 5, 3], pol, cfg, epochs=2)
    want = json.loads(str(ledger_golden[f"{name}/events"]))
    assert [list(e) for e in led.events] == want
    assert json.loads(json.dumps(ledger_summary(led), sort_keys=True)) == \
        json.loads(str(ledger_golden[f"{name}/summary"]))
    assert json.loads(json.dumps(led.stage_table(1), sort_keys=True)) == \
        json.loads(str(ledger_golden[f"{name}/stage_table"]))
    assert led.audit_issues == []


def test_cache_state_lru_and_reserve():
    c = CacheState(100)
    assert c.lookup_admit("a", 40) == (False, [])
    assert c.lookup_admit("b", 40) == (False, [])
    assert c.lookup_admit("a", 40) == (True, [])          # a is now most recent
    assert c.lookup_admit("c", 40) == (False, ["b"])      # LRU eviction
    assert c.set_reserved(50) == ["a"]
    assert c.lookup_admit("big", 60) == (False, [])       # streams through uncached
    assert c.refresh("c") and not c.refresh("zzz")


def test_schedule_matches_reference_orders(ledger_golden):
    # orders recorded from grinder.hierarchy.schedule_partitions on this plan
    plan = _plan(ledger_golden)
    assert schedule_partitions(plan, set()) == [0, 3, 1, 2]
    assert schedule_partitions(plan, {3}) == [3, 1, 2, 0]
    assert schedule_partitions(plan, {1, 2}, 8) == [2, 3, 1, 0]


def test_policy_and_config_validation():
    with pytest.raises(ValueError):
        HierarchyConfig(page_size=1000)
    with pytest.raises(ValueError):
        PolicySpec("NOPE")
    plan = g2.build_partition_plan(g2.build_csr([(0, 1), (1, 0)], 2), np.zeros(2, np.int32), 1)
    with pytest.raises(NotImplementedError):
        TierSession(plan, [2, 2], "NAIVE", HierarchyConfig())
    with pytest.raises(ValueError):
        TierSession(plan, [2], "GRINNDER", HierarchyConfig())
