"""A/B of library builds in deterministic mode (locc_set_deterministic) on the C3 step.
usage: python tools/ab_det.py a.so b.so ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import locc_synth as ls  # noqa: E402
from paper_2304_09439_b200 import locc  # noqa: E402

wl = ls.make_workload("C3")
flat = ls.weight_set("spread")
dp, dq = torch.from_numpy(wl.pairs).cuda(), torch.from_numpy(wl.poses).cuda()
pr = torch.empty(len(wl.pairs), device="cuda")
s = torch.cuda.Stream()
for path in sys.argv[1:]:
    locc._lib = None
    locc.LIB_PATH = os.path.abspath(path)
    with locc.Locc(precision=locc.LOCC_PREC_BF16, device=0) as ctx:
        ctx.set_deterministic(True)
        ctx.load_weights_mem(flat)
        ctx.set_shapes(wl.points)
        for _ in range(2):
            ctx.query_into(dp, dq, pr, stream=s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            ctx.query_into(dp, dq, pr, stream=s.cuda_stream)
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{os.path.basename(path)} deterministic: {ms:.2f} ms/step = {len(wl.pairs) / ms / 1e3:.3f} M checks/s", flush=True)
