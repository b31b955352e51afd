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


def _sha_ref(model_id: bytes, tokens) -> bytes:
    import hashlib
    import struct
    a = np.asarray(tokens, dtype="<i4")
    return hashlib.sha256(struct.pack("<I", len(model_id)) + model_id + a.tobytes()).digest()


def test_chunk_digest_is_sha256(api):
    """The store key is SHA-256 (FIPS 180-4, here hashlib as the reference) of (u32 LE len(model_id) ||
    model_id || LE int32 token ids), across the 55/56/64-byte padding boundaries and long inputs."""
    rng = np.random.default_rng(0)
    for n in [0, 1, 11, 12, 13, 14, 15, 16, 100, 512, 1024]:
        for mid in [b"", b"m", b"mistral-7b|bf16|seed1", bytes(range(200))]:
            tok = rng.integers(-(2 ** 31), 2 ** 31 - 1, n, dtype=np.int64).astype(np.int32)
            assert api.chunk_digest(mid, tok) == _sha_ref(mid, tok), (n, mid)


def test_chunk_digest_binds_model(api):
    a = np.arange(100, dtype=np.int32)
    m1 = api.model_identity(_Shape(), "bf16", "seed1")
    m2 = api.model_identity(_Shape(d_model=64), "bf16", "seed1")
    assert api.chunk_digest(m1, a) == api.chunk_digest(m1, a.copy())   # deterministic
    assert api.chunk_digest(m1, a) != api.chunk_digest(m2, a)          # another model, same tokens
    b = a.copy(); b[57] += 1
    assert api.chunk_digest(m1, a) != api.chunk_digest(m1, b)          # one token differs
    assert api.chunk_digest(m1, a[:99]) != api.chunk_digest(m1, a)     # prefix differs
    st = api.Store(1 << 20, pinned=False)
    st.put(api.chunk_digest(m1, a), torch.ones(1, 4, 1, 1), torch.ones(1, 4, 1, 1))
    assert st.lookup(api.chunk_digest(m1, a)) == 4
    assert st.lookup(api.chunk_digest(m2, a)) == -1                    # model 2 never sees model 1's KV
    with pytest.raises(ValueError):
        st.lookup(b"short")


class _Shape:
    def __init__(self, **kw):
        self.n_layers, self.d_model, self.n_q_heads, self.n_kv_heads, self.head_dim = 2, 32, 4, 2, 8
        self.d_ff, self.vocab, self.rope_theta, self.rms_eps = 64, 100, 10000.0, 1e-5
        self.__dict__.update(kw)


def _k(i: int) -> bytes:
    return int(i).to_bytes(4, "little") * 8


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
            st.put(_k(key), k.view(1, nbytes // 4, 1, 1), v.view(1, nbytes // 4, 1, 1))
            model.pop(key, None)
            while model and sum(model.values()) + 2 * nbytes > cap:
                model.popitem(last=False)
                evictions += 1
            model[key] = 2 * nbytes
        else:
            n = st.lookup(_k(key))
            if key in model:
                hits += 1
                model.move_to_end(key)
                assert n > 0
            else:
                misses += 1
                assert n == -1
        assert st.keys() == [_k(x) for x in reversed(model.keys())]
    s = st.stats()
    assert s["used"] == sum(model.values()) <= cap
    assert (s["hits"], s["misses"], s["evictions"], s["entries"]) == (hits, misses, evictions, len(model))


def test_put_errors(api):
    st = api.Store(100, pinned=False)
    with pytest.raises(api.CacheBlendError):
        st.put(_k(1), torch.zeros(1, 20, 1, 1), torch.zeros(1, 20, 1, 1))  # 160 B > 100 B
    assert st.lookup(_k(1), touch=False) == -1


def test_two_level_lru_matches_model(api, tmp_path):
    """RAM + disk levels (the store spans storage devices, LRU-evicting when full): RAM
    evictions spill to disk files (the disk level evicting its own least recently used files), a touching
    lookup reads a disk entry back into RAM; checked step by step against a two-OrderedDict model, with every
    entry's bytes verified after it comes back from disk."""
    rng = np.random.default_rng(2)
    cap_r, cap_d = 12_000, 30_000
    st = api.Store(cap_r, pinned=False)
    st.set_disk(str(tmp_path), cap_d)
    ram, disk = collections.OrderedDict(), collections.OrderedDict()  # key -> entry bytes (K + V); LRU first
    content = {}
    c = dict(hits=0, misses=0, evictions=0, dhits=0, spills=0, devict=0)

    def spill(key, nb):
        if nb > cap_d:
            return
        while disk and sum(disk.values()) + nb > cap_d:
            disk.popitem(last=False)
            c["devict"] += 1
        disk[key] = nb
        c["spills"] += 1

    def make_room(nb):
        while ram and sum(ram.values()) + nb > cap_r:
            key, vb = ram.popitem(last=False)
            spill(key, vb)
            c["evictions"] += 1

    for step in range(2500):
        key = int(rng.integers(0, 30))
        if rng.random() < 0.45:
            n = int(rng.integers(1, 1000))
            k = torch.arange(n, dtype=torch.float32) + step
            st.put(_k(key), k.view(1, n, 1, 1), (-k).view(1, n, 1, 1))
            ram.pop(key, None)
            disk.pop(key, None)
            make_room(8 * n)
            ram[key] = 8 * n
            content[key] = k
        else:
            got = st.get(_k(key), (1, -1, 1, 1), torch.float32) if key in content else None
            if key in ram:
                c["hits"] += 1
                ram.move_to_end(key)
            elif key in disk:
                nb = disk.pop(key)
                make_room(nb)
                ram[key] = nb
                c["hits"] += 1
                c["dhits"] += 1
            else:
                if key in content:
                    assert got is None
                else:
                    assert st.lookup(_k(key)) == -1
                c["misses"] += 1
                continue
            kk, vv = got
            assert torch.equal(kk.flatten(), content[key]) and torch.equal(vv.flatten(), -content[key])
        assert st.keys() == [_k(x) for x in reversed(ram.keys())]
    s, d = st.stats(), st.disk_stats()
    assert s["used"] == sum(ram.values()) and d["used"] == sum(disk.values()) <= cap_d
    assert (s["hits"], s["misses"], s["evictions"]) == (c["hits"], c["misses"], c["evictions"])
    assert (d["entries"], d["hits"], d["spills"], d["evictions"]) == (len(disk), c["dhits"], c["spills"], c["devict"])
    assert len(list(tmp_path.glob("*.cbkv"))) == len(disk)
    st.close()
    assert not list(tmp_path.glob("*.cbkv"))  # the store deletes its files


def test_disk_level_errors(api, tmp_path):
    st = api.Store(1000, pinned=False)
    with pytest.raises(api.CacheBlendError):
        st.set_disk(str(tmp_path / "missing"), 10_000)
    st.set_disk(str(tmp_path), 10_000)
    st.put(_k(1), torch.ones(1, 100, 1, 1), torch.ones(1, 100, 1, 1))  # 800 B
    st.put(_k(2), torch.ones(1, 100, 1, 1), torch.ones(1, 100, 1, 1))  # evicts 1 to disk
    assert st.lookup(_k(1), touch=False) == 100 and st.disk_stats()["entries"] == 1
    st.set_disk(str(tmp_path), 0)  # disabling drops the level and its files
    assert st.lookup(_k(1), touch=False) == -1 and not list(tmp_path.glob("*.cbkv"))
