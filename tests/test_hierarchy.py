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


@pytest.mark.parametrize("seed", range(6))
def test_manager_dry_run_equals_oracle_byte_model(seed):
    """The manager's non-executing run and the oracle's restatement of the
    reference byte model (oracle/ledger.py) agree on random plans, widths,
    host capacities, page sizes and bypass settings."""
    from oracle import ledger as oled
    rng = np.random.default_rng(seed)
    g = g2.generate_kronecker(int(rng.integers(6, 9)), int(rng.integers(3, 9)), seed=seed)
    P = int(rng.integers(1, 6))
    plan = g2.build_partition_plan(g, g2.random_partition(g.num_vertices, P, seed), P)
    dims = [int(x) for x in rng.integers(1, 9, size=int(rng.integers(2, 5)))]
    n = g.num_vertices
    kw = dict(host_capacity=int(rng.choice([0, 64, n * 4, n * 4 * max(dims) * 3])),
              bytes_per_value=int(rng.choice([4, 8])), page_size=int(rng.choice([16, 64, 4096])))
    bypass = bool(rng.integers(0, 2))
    ours = simulate_epoch(plan, dims, PolicySpec("GRINNDER", bypass_enabled=bypass),
                          HierarchyConfig(**kw), epochs=2)
    ref = oled.simulate_epoch(plan, dims, oled.PolicySpec("GRINNDER", bypass_enabled=bypass),
                              oled.HierarchyConfig(**kw), epochs=2)
    assert ours.events == ref.events
    assert ledger_summary(ours) == oled.ledger_summary(ref)
    assert ours.stage_table(2) == ref.stage_table(2)


def test_storage_tier_row_runs_round_trip(tmp_path):
    """grd_mem_runs on a mapped tier file: packed row runs written at record
    offsets read back bit for bit (untouched regions of the file read as
    zeros); a deleted object leaves the residency (its file is kept for the
    next incarnation)."""
    import torch
    from paper_2605_11517_b200.hierarchy import StorageTier
    levels = []
    st = StorageTier(1 << 30, str(tmp_path), levels.append)
    st.sizes[("act", 1)] = 15 * 5 * 4
    st.activate()
    rows = torch.arange(7 * 5, dtype=torch.float32).reshape(7, 5)
    first, count = np.array([2, 10, 11 + 1]), np.array([3, 1, 3])
    st.io(("act", 1), True, 5 * 4, first, count, rows, create=True)
    st.grow(("act", 1), rows.numel() * 4)
    back = torch.empty_like(rows)
    st.io(("act", 1), False, 5 * 4, first, count, back)
    assert torch.equal(back, rows)
    whole = torch.empty((15, 5), dtype=torch.float32)
    st.io(("act", 1), False, 5 * 4 * 15, [0], [1], whole)
    assert torch.equal(whole[2:5], rows[:3]) and torch.equal(whole[10], rows[3])
    assert not whole[5:10].any()
    assert levels[-1] == rows.numel() * 4
    st.delete(("act", 1))
    assert st.level == 0 and not st.exists(("act", 1))
    st.close()
