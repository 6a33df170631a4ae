"""A small run of every tensor-core kernel for compute-sanitizer (memcheck / racecheck / synccheck).

C1-like pairs through locc_query in a bf16 context (segment_xf, crop, scan, crop_emit, encoder_tc,
head_tc), the deterministic walk, the pose gradient (head_tc<., true>), and the encode-once path
(grid encode + conv_tc U-Net + cells_select + head_tc) on a few shapes.

usage: compute-sanitizer --tool <tool> python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import locc_synth as ls  # noqa: E402
from paper_2304_09439_b200 import locc  # noqa: E402


def main():
    pts, _ = ls.make_shapes(6, 300, seed=90)
    pairs, poses = ls.make_pairs_poses(pts, 40, s=0.5, seed=91)
    flat = ls.weight_set("spread_bias")
    with locc.Locc(precision=locc.LOCC_PREC_BF16, device=0, max_batch=16) as ctx:
        ctx.load_weights_mem(flat)
        ctx.set_shapes(pts)
        p, l, g = ctx.query(pairs, poses)
        ctx.set_deterministic(True)
        p2, _, _ = ctx.query(pairs, poses)
        ctx.set_deterministic(False)
        _, _, _, grad = ctx.query_grad(pairs, poses)
        ctx.load_unet_weights_mem(ls.flatten_unet(ls.make_unet_weights("he")))
        ctx.encode_shapes()
        c = ctx.query_cells(pairs, poses)
    assert np.isfinite(p).all() and np.isfinite(grad).all() and np.isfinite(c["probs"]).all()
    print("sanitize run ok:", len(pairs), "pairs; max |p - p_det|", float(np.abs(p - p2).max()))


if __name__ == "__main__":
    main()
