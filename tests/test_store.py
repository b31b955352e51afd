"""Chunk KV store (§6 "KV cache store") on CPU: hashing of chunk token ids,
and LRU eviction checked step by step against a plain OrderedDict model of the paper's rule ("when the
storage devices are full, we evict the least recently used KV cache"). Host bookkeeping only
(malloc-backed store); the GPU request path through the store is in test_gpu_parity.py."""
import collections

import numpy as np
import pytest
import torch

from paper_2405_16444_b200.build import build


@pytest.fixture(scope="module")
def api():
    build()
    from paper_2405_16444_b200 import api
    return api


def test_chunk_hash(api):
    a = np.arange(100, dtype=np.int32)
    assert api.chunk_hash(a) == api.chunk_hash(a.copy())          # deterministic
    b = a.copy(); b[57] += 1
    assert api.chunk_hash(a) != api.chunk_hash(b)                  # one token differs
    assert api.chunk_hash(a[:99]) != api.chunk_hash(a)             # prefix differs
    assert api.chunk_hash(a[::-1].copy()) != api.chunk_hash(a)     # order matters
    hs = {api.chunk_hash(np.random.default_rng(i).integers(0, 32000, 512)) for i in range(2000)}
    assert len(hs) == 2000


def test_lru_matches_model(api):
    rng = np.random.default_rng(1)
    cap = 10_000
    st = api.Store(cap, pinned=False)
    model = collections.OrderedDict()  # key -> bytes of the entry (K + V), most recent last
    evictions = hits = misses = 0
    for step in range(3000):
        key = int(rng.integers(0, 40))
        if rng.random() < 0.5:
            nbytes = int(rng.integers(1, 1200)) * 4
            k = torch.full((1, nbytes // 4), float(step)); v = -k
            st.put(key, k.view(1, nbytes // 4, 1, 1), v.view(1, nbytes // 4, 1, 1))
            model.pop(key, None)
            while model and sum(model.values()) + 2 * nbytes > cap:
                model.popitem(last=False)
                evictions += 1
            model[key] = 2 * nbytes
        else:
            n = st.lookup(key)
            if key in model:
                hits += 1
                model.move_to_end(key)
                assert n > 0
            else:
                misses += 1
                assert n == -1
        assert st.keys() == list(reversed(model.keys()))
    s = st.stats()
    assert s["used"] == sum(model.values()) <= cap
    assert (s["hits"], s["misses"], s["evictions"], s["entries"]) == (hits, misses, evictions, len(model))


def test_put_errors(api):
    st = api.Store(100, pinned=False)
    with pytest.raises(api.CacheBlendError):
        st.put(1, torch.zeros(1, 20, 1, 1), torch.zeros(1, 20, 1, 1))  # 160 B > 100 B
    assert st.lookup(1, touch=False) == -1
