"""Small-batch latency: device time (CUDA events around one call) and host wall time (call +
synchronize) of locc_query at N = 64 .. 16384 (bf16), with the query CUDA graph and without
(LOCC_NO_GRAPH=1), and the library's per-stage timing (crop, encoder, predictor)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import locc_synth as ls  # noqa: E402
from paper_2304_09439_b200 import locc  # noqa: E402

wl = ls.make_workload("C2")
for graph in (True, False):
    if not graph:
        os.environ["LOCC_NO_GRAPH"] = "1"
    with locc.Locc(precision=locc.LOCC_PREC_BF16, device=0) as ctx:
        ctx.load_weights_mem(ls.weight_set("spread"))
        ctx.set_shapes(wl.points)
        s = torch.cuda.Stream()
        for n in (64, 1024, 4096, 16384):
            p = torch.from_numpy(wl.pairs[:n]).cuda()
            q = torch.from_numpy(wl.poses[:n]).cuda()
            pr = torch.empty(n, device="cuda")
            for _ in range(5):
                ctx.query_into(p, q, pr, stream=s.cuda_stream)
            s.synchronize()
            dev, wall = [], []
            for _ in range(20):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter()
                e0.record(s)
                ctx.query_into(p, q, pr, stream=s.cuda_stream)
                e1.record(s)
                s.synchronize()
                wall.append((time.perf_counter() - t0) * 1e3)
                dev.append(e0.elapsed_time(e1))
            replay = ctx.stats()["graph_replay"]
            ctx.set_timing(True)
            ctx.query_into(p, q, pr, stream=s.cuda_stream)
            s.synchronize()
            st = ctx.stats()
            ctx.set_timing(False)
            dev.sort()
            wall.sort()
            print(f"graph={int(graph)} (replayed {replay}) N={n}: device {dev[10]:.3f} ms (min {dev[0]:.3f}), "
                  f"host wall {wall[10]:.3f} ms; stages: crop {st['crop_ms']:.3f} encoder {st['encoder_ms']:.3f} "
                  f"head {st['head_ms']:.3f} total {st['total_ms']:.3f} ms; {st['kernel_launches']} launches",
                  flush=True)
