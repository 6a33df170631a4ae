"""Run each NEXT mode once at a bench-sized workload (for ncu captures): encode-once (grid encode,
U-Net, cell selection, predictor), pose gradient, closed loop.  Usage: python tools/next_modes.py [pairs]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import locc_synth as ls  # noqa: E402
from paper_2304_09439_b200 import locc  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    wl = ls.make_workload("C3", N=N)
    ctx = locc.Locc(precision=locc.LOCC_PREC_BF16, device=0)
    ctx.load_weights_mem(ls.flatten_weights(ls.make_weights("spread", calib=ls.load_calibration())))
    ctx.set_shapes(wl.points)
    ctx.load_unet_weights_mem(ls.flatten_unet(ls.make_unet_weights()))
    ctx.encode_shapes()
    dp, dq = torch.from_numpy(wl.pairs).cuda(), torch.from_numpy(wl.poses).cuda()
    probs = torch.empty(N, device="cuda")
    grad = torch.empty(N, 14, device="cuda")
    ctx.query_cells_into(dp, dq, probs)
    ctx.query_grad_into(dp, dq, probs, grad)
    ids, body, st = ls.make_sim_scene(wl.points, 30000)
    d_ids, d_body, d_st = torch.from_numpy(ids).cuda(), torch.from_numpy(body).cuda(), torch.from_numpy(st).cuda()
    ctx.sim_run(dict(ls.SIM_DEFAULTS, detector="cells"), d_ids, d_body, d_st)
    torch.cuda.synchronize()
    print("ok", float(probs.mean()), float(grad.abs().mean()), bool(torch.isfinite(d_st).all()))
    ctx.close()


if __name__ == "__main__":
    main()
