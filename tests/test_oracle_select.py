"""Pins for Delta_kv, HKVD selection and the gradual-filtering schedule (§3.3)."""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import cacheblend_oracle as O
from tests.conftest import GOLDEN


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def test_deviation_golden():
    for c in _load("deviation.json")["cases"]:
        rng = np.random.default_rng(0)
        k = rng.standard_normal((c["n_tok"], c["n_kv"], c["hd"]))
        v = rng.standard_normal((c["n_tok"], c["n_kv"], c["hd"]))
        k2, v2 = k.copy(), v.copy()
        p = c["perturb"]
        if p:
            (k2 if p["which"] == "k" else v2)[p["tok"], p["head"], p["dim"]] += p["delta"]
        np.testing.assert_allclose(O.kv_deviation(k2, v2, k, v), c["expect"], atol=1e-15)


def test_deviation_modes_and_rotation_invariance():
    rng = np.random.default_rng(1)
    k, v = rng.standard_normal((6, 2, 8)), rng.standard_normal((6, 2, 8))
    k2, v2 = k + 0.1 * rng.standard_normal(k.shape), v + 0.2 * rng.standard_normal(v.shape)
    dkv, dk, dv = (O.kv_deviation(k2, v2, k, v, m) for m in ("kv", "k", "v"))
    np.testing.assert_allclose(dkv, dk + dv, rtol=1e-14)
    # R1: comparing rotated keys equals comparing unrotated keys (R orthogonal)
    pos = rng.integers(0, 5000, 6)
    rk, rk2 = O.rope_rotate(k, pos[:, None], 1e4), O.rope_rotate(k2, pos[:, None], 1e4)
    np.testing.assert_allclose(O.kv_deviation(rk2, v2, rk, v), dkv, rtol=1e-10)


def test_select_golden():
    for c in _load("select_hkvd.json")["cases"]:
        out = O.select_hkvd(np.array(c["dev"]), np.array(c["cand"]), c["k"])
        assert out.tolist() == c["expect"], c


def test_select_brute_force():
    """Brute force by counting: token j is selected iff fewer than k candidates beat it, where a beats
    b when dev_a > dev_b or (dev_a == dev_b and tok_a < tok_b)."""
    rng = np.random.default_rng(2)
    for trial in range(300):
        n = int(rng.integers(1, 12))
        cand = np.sort(rng.choice(100, n, replace=False))
        dev = rng.integers(0, 4, n).astype(float) * 0.5     # many ties
        k = int(rng.integers(0, n + 1))
        expect = [cand[j] for j in range(n)
                  if sum((dev[a] > dev[j]) or (dev[a] == dev[j] and cand[a] < cand[j]) for a in range(n)) < k]
        assert O.select_hkvd(dev, cand, k).tolist() == expect


def test_schedule_golden():
    g = _load("schedule.json")
    for c in g["ratio_cases"]:
        np.testing.assert_allclose(O.schedule_ratios(c["r"], c["L"]), c["ratios_layers_1_to_L_minus_1"],
                                   atol=1e-12)
    for c in g["count_cases"]:
        ks = O.schedule(c["r"], c["N"], c["L"])
        assert ks[0] == c["N"] and ks[1] == c["k_first"] and ks[-1] == c["k_last"], (c, ks[:2], ks[-1])


@pytest.mark.parametrize("r", [0.0, 0.05, 0.15, 0.3, 0.5, 0.85, 1.0])
@pytest.mark.parametrize("L", [2, 3, 5, 32, 80])
def test_schedule_properties(r, L):
    ratios = O.schedule_ratios(r, L)
    assert len(ratios) == L - 1
    assert abs(np.mean(ratios) - r) < 1e-12                       # mean exactly r (R4)
    assert all(a >= b - 1e-15 for a, b in zip(ratios, ratios[1:]))  # r1 >= r2 >= ...
    assert all(0.0 <= x <= 1.0 for x in ratios)
    ks = O.schedule(r, 1000, L)
    assert all(a >= b for a, b in zip(ks[1:], ks[2:]))
    assert all(k == min(1000, math.ceil(x * 1000 - 1e-9)) for k, x in zip(ks[1:], ratios))
