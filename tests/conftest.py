"""Shared fixtures: golden vectors from the reference, GPU gating."""

from __future__ import annotations

import os
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: takes more than a few seconds")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def small_golden():
    z = np.load(GOLDEN / "small_cases.npz")
    cases = {}
    for key in z.files:
        name, field = key.split("/", 1)
        cases.setdefault(name, {})[field] = z[key]
    return cases


@pytest.fixture(scope="session")
def config1_golden():
    return dict(np.load(GOLDEN / "config1.npz"))


def rel_l2(x, ref) -> float:
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-30))


def small_case_inputs(case):
    """Rebuild a golden small case's inputs with the product's host code
    (generator / dataset / model are bit-exact with the reference)."""
    from paper_2605_11517_b200 import generate_kronecker, make_random_dataset, create_model
    scale, deg, F, C, P, L, H, rn, epochs = [int(x) for x in case["spec"]]
    g = generate_kronecker(scale, deg, seed=scale)
    ds = make_random_dataset(g, feature_dim=F, num_classes=C, seed=scale + 1)
    model = create_model(F, C, num_layers=L, hidden_dim=H, seed=scale + 3,
                         aggregation_mode=str(case["mode"]), row_normalize=bool(rn),
                         dropout_rate=float(case["dropout"]))
    return SimpleNamespace(graph=g, dataset=ds, model=model, labels=case["labels"], P=P, L=L,
                           epochs=epochs, mode=str(case["mode"]), rownorm=bool(rn),
                           dropout=float(case["dropout"]))
