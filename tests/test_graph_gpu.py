"""The query CUDA graph (include/locc.h locc_query: an asynchronous device-buffer query of one
sub-batch is captured on its second call and replayed after that).

A replay must equal the direct path (LOCC_NO_GRAPH=1) bitwise when the buffers' contents change
between calls, after a weight reload (the context's generation) and after a larger query regrew the
scratch buffers the graph points into (the allocation epoch); and stats() must say it replayed.
"""
import os

import numpy as np
import pytest

import locc_synth as ls

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def locc_mod():
    from paper_2304_09439_b200 import build as b
    b.build()
    from paper_2304_09439_b200 import locc
    return locc


def _call(ctx, mode, bufs, s):
    p, q, pr, lb, lg, gr = bufs
    if mode == "query":
        ctx.query_into(p, q, pr, labels=lb, logits=lg, stream=s.cuda_stream)
    elif mode == "grad":
        ctx.query_grad_into(p, q, pr, gr, labels=lb, logits=lg, stream=s.cuda_stream)
    else:
        ctx.query_cells_into(p, q, pr, labels=lb, logits=lg, stream=s.cuda_stream)


@pytest.mark.parametrize("mode", ["query", "grad", "cells"])
@pytest.mark.parametrize("precision", [0, 1])
def test_query_graph_replay_equals_direct(locc_mod, mode, precision):
    import torch
    pts, _ = ls.make_shapes(12, 800, seed=61)
    n = 700
    inputs = [ls.make_pairs_poses(pts, n, s=0.5, seed=62 + k) for k in range(3)]
    big = ls.make_pairs_poses(pts, 3000, s=0.5, seed=66)
    w0, w1 = ls.weight_set("spread_bias"), ls.weight_set("spread")
    unet = ls.flatten_unet(ls.make_unet_weights("he")) if mode == "cells" else None
    results = {}
    for no_graph in (True, False):
        if no_graph:
            os.environ["LOCC_NO_GRAPH"] = "1"
        try:
            ctx = locc_mod.Locc(M=6, H=256, F=64, precision=precision, device=0)
            ctx.load_weights_mem(w0)
            ctx.set_shapes(pts)
            if unet is not None:
                ctx.load_unet_weights_mem(unet)
                ctx.encode_shapes()
            s = torch.cuda.Stream()
            p = torch.empty(n, 2, dtype=torch.int32, device="cuda")
            q = torch.empty(n, 2, 7, dtype=torch.float32, device="cuda")
            bufs = (p, q, torch.empty(n, device="cuda"), torch.empty(n, dtype=torch.uint8, device="cuda"),
                    torch.empty(n, device="cuda"), torch.empty(n, 14, device="cuda"))
            outs, replays = [], []
            # calls: 0 direct, 1 captured, 2.. replays; new contents every call; weights reloaded before
            # call 4; a larger query_debug (scratch regrowth, the graph's key untouched) before call 6
            for k in range(8):
                if k == 4:
                    ctx.load_weights_mem(w1)
                    if unet is not None:  # new weights drop the cached grids
                        ctx.encode_shapes()
                if k == 6:  # not a graphed call: only the allocation epoch tells the graph
                    ctx.query_debug(*big)
                a, b = inputs[k % 3]
                with torch.cuda.stream(s):
                    p.copy_(torch.from_numpy(a), non_blocking=False)
                    q.copy_(torch.from_numpy(b), non_blocking=False)
                _call(ctx, mode, bufs, s)
                s.synchronize()
                outs.append([t.cpu().numpy().copy() for t in bufs[2:] if mode == "grad" or t is not bufs[5]])
                st = ctx.stats()
                assert st["pairs"] == n
                replays.append(st["graph_replay"])
            ctx.close()
        finally:
            os.environ.pop("LOCC_NO_GRAPH", None)
        results[no_graph] = (outs, replays)
    direct, graphed = results[True], results[False]
    assert direct[1] == [0] * 8
    # the first call with a key runs directly, the second is captured (and launched as the graph)
    assert graphed[1] == [0, 1, 1, 1, 0, 1, 0, 1], graphed[1]
    for k in range(8):
        for x, y in zip(direct[0][k], graphed[0][k]):
            assert np.array_equal(x, y, equal_nan=True), f"call {k} differs from the direct path"
