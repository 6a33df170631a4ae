"""Host logic of the multi-GPU path on CPU: shard bounds, and the gloo world_size-2 gather
reassembling a sharded query in the original order.  The per-shard function is a REAL query — the CPU
oracle's (test infrastructure may call it) — so the test proves that sharding the pairs and gathering
the shards gives bitwise the unsharded answer; the GPU query's own sharded
equality is covered by tests/test_multi_gpu.py and test_parity_gpu.py."""
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

    import locc_synth as ls
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = ls.make_workload("C1", N=N, K=300, S=8)
    flat = ls.weight_set("spread_bias")

    def query(p, po):  # the oracle's collision query of one shard (single-threaded, deterministic)
        r = oracle.query(flat, wl.points, p, po, n_threads=1)
        return r["probs"].astype(np.float32), r["labels"].astype(np.uint8)

    probs, labels = query_sharded(query, wl.pairs, wl.poses, rank, world)
    want_p, want_l = query(wl.pairs, wl.poses)
    q.put((rank, bool(np.array_equal(probs, want_p) and np.array_equal(labels, want_l)
                      and (want_l == 1).any() and (want_l == 0).any())))
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
