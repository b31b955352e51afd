"""Paged hand-off: the oracle's page layout pinned by a hand-written example and
by its inverse (gathering pages back through the block table recovers every token)."""
import numpy as np

from oracle import cacheblend_oracle as O


def test_hand_example():
    # 1 layer, 5 tokens (values 10..14), 1 kv head, head_dim 1, block_size 2, pages 3, 0, 2 of a 4-page pool
    kv = np.arange(10, 15, dtype=np.float32).reshape(1, 5, 1, 1)
    p = O.kv_to_paged(kv, [3, 0, 2], 2, 4)
    assert p.shape == (1, 4, 2, 1, 1)
    want = {(3, 0): 10, (3, 1): 11, (0, 0): 12, (0, 1): 13, (2, 0): 14}
    for (pg, sl), val in want.items():
        assert p[0, pg, sl, 0, 0] == val
    assert np.isnan(p[0, 1]).all() and np.isnan(p[0, 2, 1]).all()  # unused page, tail slot


def test_inverse_gather():
    rng = np.random.default_rng(0)
    for T, bs in ((1, 16), (33, 16), (64, 16), (100, 7)):
        kv = rng.standard_normal((3, T, 2, 4)).astype(np.float32)
        n_blocks = -(-T // bs)
        table = rng.permutation(n_blocks + 3)[:n_blocks]
        p = O.kv_to_paged(kv, table, bs, n_blocks + 3)
        back = np.stack([p[:, table[t // bs], t % bs] for t in range(T)], axis=1)
        np.testing.assert_array_equal(back, kv)
