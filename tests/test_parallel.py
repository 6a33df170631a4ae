"""Host logic of the multi-GPU path on CPU: shard bounds, and the gloo world_size-2 gather
reassembling a sharded query in the original order (the per-shard function here is a stand-in that
only tags pairs; the GPU query itself is covered by the gpu tests)."""
import os
import socket

import numpy as np
import pytest

from paper_2304_09439_b200.parallel import query_sharded, shard_bounds


@pytest.mark.parametrize("N,world", [(0, 2), (1, 2), (7, 2), (8, 4), (1000, 8), (5, 8)])
def test_shard_bounds_cover_exactly(N, world):
    seen = []
    for r in range(world):
        lo, hi = shard_bounds(N, world, r)
        assert 0 <= lo <= hi <= N
        seen.extend(range(lo, hi))
    assert seen == list(range(N))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    pairs = rng.integers(0, 100, size=(N, 2)).astype(np.int32)
    poses = rng.standard_normal((N, 2, 7)).astype(np.float32)

    def fake_query(p, po):  # stand-in: a deterministic tag of each pair
        return (p[:, 0] * 1000 + p[:, 1]).astype(np.float32), (p[:, 0] % 2).astype(np.uint8)

    probs, labels = query_sharded(fake_query, pairs, poses, rank, world)
    want_p, want_l = fake_query(pairs, poses)
    q.put((rank, bool(np.array_equal(probs, want_p) and np.array_equal(labels, want_l))))
    dist.destroy_process_group()


@pytest.mark.parametrize("N", [9, 64])
def test_gloo_world2_gather(N):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}
