"""Loading controller (§6): the oracle pinned to the paper's worked examples
(tests/golden/controller.json), and the library's host implementation (cb_controller_*,
no GPU needed) checked against the oracle."""
import json
import os

import numpy as np
import pytest

from oracle import cacheblend_oracle as O
from tests.conftest import GOLDEN

G = json.load(open(os.path.join(GOLDEN, "controller.json")))


def test_paper_examples():
    r_star = G["r_star"]
    llama7, llama70 = G["examples"]
    # Llama-7B: 15 % costs 3 ms/layer -> Prefill = 20 ms/layer (T_recompute = r x Prefill); NVMe load 16 ms
    pre7 = llama7["recompute_ms_at_15pct"] / 0.15
    assert O.t_recompute(0.15, pre7) == pytest.approx(3.0)
    assert (O.t_recompute(0.15, pre7) <= llama7["load_ms"]) == llama7["hidden_at_15pct"]
    r = O.controller_ratio(pre7, llama7["load_ms"], r_star)
    assert r == pytest.approx(0.8)  # recompute up to the 16 ms the load takes anyway
    assert O.t_recompute(r, pre7) == pytest.approx(llama7["max_free_recompute_ms"])
    # Llama-70B: 15 % costs 7 ms, load 4 ms: not hidden; the controller stays at r* = 15 %
    pre70 = llama70["recompute_ms_at_15pct"] / 0.15
    assert (O.t_recompute(0.15, pre70) <= llama70["load_ms"]) == llama70["hidden_at_15pct"]
    assert O.controller_ratio(pre70, llama70["load_ms"], r_star) == pytest.approx(r_star)


def test_load_estimator_and_bounds():
    # Llama-7B per-token per-layer KV: K and V, 4096 values each, 2 B -> 16 KiB; 4K tokens over 4 GiB/s
    kv = 2 * 4096 * 2
    bpm = 4 * 2**30 / 1e3
    assert O.t_load(kv, 4096, bpm) == pytest.approx(4096 * kv / bpm)
    assert O.t_load(kv, 8192, bpm) == pytest.approx(2 * O.t_load(kv, 4096, bpm))       # linear in L
    assert O.t_load(kv, 4096, 2 * bpm) == pytest.approx(O.t_load(kv, 4096, bpm) / 2)   # inverse in speed
    for load in (0.0, 1.0, 5.0, 50.0, 500.0):
        r = O.controller_ratio(20.0, load)
        assert 0.15 <= r <= 1.0
    assert O.controller_ratio(20.0, 500.0) == 1.0


def test_pick_device_paper_rule():
    # Llama-7B (Prefill 20 ms/layer, 15 % -> 3 ms): NVMe 16 ms (cost 1), CPU RAM 0.5 ms (cost 10),
    # cloud 40 ms (cost 0.1), a second RAM tier 2 ms (cost 10): only the RAM tiers hide under 3 ms
    load, cost = [16.0, 0.5, 40.0, 2.0], [1.0, 10.0, 0.1, 10.0]
    assert O.controller_pick_device(20.0, load, cost) == 1  # cheapest qualifying, tie -> earlier
    assert O.controller_pick_device(200.0, load, cost) == 0  # 30 ms recompute hides NVMe (cheaper than RAM)
    assert O.controller_pick_device(1.0, load, cost) == -1


def test_library_controller_matches_oracle():
    from paper_2405_16444_b200 import api
    from paper_2405_16444_b200.build import build
    build()
    rng = np.random.default_rng(0)
    for _ in range(200):
        pre, kv, n, bpm = rng.uniform(0.1, 100), rng.uniform(1e3, 1e6), int(rng.integers(0, 20000)), rng.uniform(1e3, 1e8)
        rmin = rng.uniform(0, 1)
        r, ld = api.controller_ratio(pre, kv, n, bpm, rmin)
        assert ld == pytest.approx(O.t_load(kv, n, bpm), rel=1e-12)
        assert r == pytest.approx(O.controller_ratio(pre, ld, rmin), rel=1e-12)
        nd = int(rng.integers(0, 6))
        load, cost = rng.uniform(0, 50, nd).tolist(), rng.integers(0, 4, nd).astype(float).tolist()
        assert api.controller_pick_device(pre, load, cost) == O.controller_pick_device(pre, load, cost)
    with pytest.raises(api.CacheBlendError):
        api.controller_ratio(0.0, 1.0, 1, 1.0)
    with pytest.raises(api.CacheBlendError):
        api.controller_ratio(1.0, 1.0, 1, 1.0, r_min=1.5)


def test_library_controller_schedule():
    """cb_controller_schedule = cb_schedule(cb_controller_ratio(...)): the controller's ratio drives the
    blend's per-layer counts."""
    from paper_2405_16444_b200 import api
    from paper_2405_16444_b200.build import build
    build()
    rng = np.random.default_rng(1)
    for _ in range(100):
        pre, kv, bpm = rng.uniform(0.05, 50), rng.uniform(1e3, 1e6), rng.uniform(1e3, 1e8)
        n, L = int(rng.integers(1, 20000)), int(rng.integers(2, 81))
        ks, r, ld = api.controller_schedule(pre, kv, bpm, n, L, 0.15)
        r2, ld2 = api.controller_ratio(pre, kv, n, bpm, 0.15)
        assert r == r2 and ld == ld2
        assert ks == O.schedule(r, n, L)
