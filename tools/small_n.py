"""Small-batch latency breakdown: device time of locc_query at N = 64 .. 16384 (bf16), with the
library's per-stage timing (crop, encoder, predictor)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import locc_synth as ls  # noqa: E402
from paper_2304_09439_b200 import locc  # noqa: E402

wl = ls.make_workload("C2")
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
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
        for _ in range(20):
            ctx.query_into(p, q, pr, stream=s.cuda_stream)
        with torch.cuda.stream(s):
            e1.record(s)
        s.synchronize()
        ctx.set_timing(True)
        ctx.query_into(p, q, pr, stream=s.cuda_stream)
        s.synchronize()
        st = ctx.stats()
        ctx.set_timing(False)
        print(f"N={n}: {e0.elapsed_time(e1) / 20:.3f} ms/query; stages: crop {st['crop_ms']:.3f} encoder "
              f"{st['encoder_ms']:.3f} head {st['head_ms']:.3f} total {st['total_ms']:.3f} ms; "
              f"{st['kernel_launches']} launches")
