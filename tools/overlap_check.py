"""C3 step with the crop of sub-batch s+1 overlapped with the encoder of s (default) and serialised
(LOCC_NO_OVERLAP=1): step time, and the per-stage device times of a timed step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import locc_synth as ls  # noqa: E402
from paper_2304_09439_b200 import locc  # noqa: E402

wl = ls.make_workload("C3")
dp, dq = torch.from_numpy(wl.pairs).cuda(), torch.from_numpy(wl.poses).cuda()
pr = torch.empty(len(wl.pairs), device="cuda")
s = torch.cuda.Stream()
with locc.Locc(precision=locc.LOCC_PREC_BF16, device=0) as ctx:
    ctx.load_weights_mem(ls.weight_set("spread"))
    ctx.set_shapes(wl.points)
    for rep in range(2):
        for mode in ("overlap", "serial"):
            if mode == "serial":
                os.environ["LOCC_NO_OVERLAP"] = "1"
            else:
                os.environ.pop("LOCC_NO_OVERLAP", None)
            for _ in range(2):
                ctx.query_into(dp, dq, pr, stream=s.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(3):
                ctx.query_into(dp, dq, pr, stream=s.cuda_stream)
            e1.record(s)
            s.synchronize()
            ms = e0.elapsed_time(e1) / 3
            ctx.set_timing(True)
            os.environ["LOCC_TIMELINE"] = "1"
            ctx.query_into(dp, dq, pr, stream=s.cuda_stream)
            s.synchronize()
            st = ctx.stats()
            os.environ.pop("LOCC_TIMELINE", None)
            ctx.set_timing(False)
            print(f"{mode}: {ms:.1f} ms/step ({len(wl.pairs) / ms / 1e3:.3f} M/s); timed step: encoder {st['encoder_ms']:.1f} "
                  f"crop {st['crop_ms']:.1f} head {st['head_ms']:.1f} total {st['total_ms']:.1f} ms", flush=True)
