"""Request-parallel host logic (SURVEY §8(e) partitioning 2) on CPU: the longest-first assignment and the
max-over-ranks / sum-over-ranks reductions bench.py quotes, exercised with a world_size-2 gloo group."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2405_16444_b200.dist import assign_requests
from synth import workload as W


def test_assign_requests_longest_first():
    sizes = [5, 9, 9, 1, 7, 3, 3]
    parts = assign_requests(sizes, 3)
    assert sorted(i for p in parts for i in p) == list(range(len(sizes)))       # each request exactly once
    assert parts == assign_requests(sizes, 3)                                   # deterministic
    # LPT trace: 9(1)->r0, 9(2)->r1, 7(4)->r2, 5(0)->r2 (7<9), 3(5)->r0, 3(6)->r1, 1(3)->r0
    assert parts == [[1, 3, 5], [2, 6], [0, 4]]
    loads = [sum(sizes[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(sizes)                                 # LPT bound


def test_assign_batched_config_balance():
    reqs = W.config_requests("batched", 1)
    sizes = [r.n_ctx for r in reqs]
    assert len(sizes) == 64 and min(sizes) >= 4 * 256 and max(sizes) <= 8 * 1024
    for world in (1, 2, 4, 8):
        parts = assign_requests(sizes, world)
        loads = [sum(sizes[i] for i in p) for p in parts]
        assert sum(loads) == sum(sizes)
        assert max(loads) <= sum(sizes) / world + max(sizes)
    with pytest.raises(ValueError):
        assign_requests(sizes, 0)


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    from paper_2405_16444_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, _ = D.world_info()
    tokens, ms = 1000 * (r + 1), 10.0 + 5.0 * r           # rank 1 is the slow one
    value, ms_max, tok = D.job_throughput(tokens, ms)
    parts = D.assign_requests([r_.n_ctx for r_ in W.config_requests("batched", 1)], w)
    np.save(os.path.join(out_dir, f"r{r}.npy"), np.array([value, ms_max, tok, len(parts[r])], dtype=np.float64))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_reductions():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, port, d), nprocs=2, join=True)
        res = [np.load(os.path.join(d, f"r{r}.npy")) for r in range(2)]
    for v in res:  # every rank sees the same job numbers: 3000 tokens over the slowest rank's 15 ms
        assert v[1] == 15.0 and v[2] == 3000.0
        assert abs(v[0] - 3000.0 / 0.015) < 1e-6
    assert res[0][3] + res[1][3] == 64
