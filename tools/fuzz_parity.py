"""Randomised parity sweep: the CUDA path (through the C ABI) against the CPU oracle on random configs.

Each case draws K (1..3000), M (1..8), S shapes, N pairs, the pose density s, a weight set and a
precision, then checks the bars of tests/test_parity_gpu.py: kept counts, crop masks and occupied-cell
counts bit-exact; probabilities within 1e-5 (fp32) / 5e-4 of the bf16-emulating oracle (bf16), labels
equal away from the 0.5 band; plus self-pairs, coincident poses and pairs repeated inside the batch.

usage: python tools/fuzz_parity.py [cases] [seed]      (on the GPU box; prints one line per case)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import locc_synth as ls  # noqa: E402
import oracle  # noqa: E402
from paper_2304_09439_b200 import locc  # noqa: E402

P_TOL = {0: 1e-5, 1: 5e-4}


def case(rng, i):
    K = int(rng.choice([1, 2, 31, 32, 33, 100, 511, 777, 1500, 2048, 2049, 3000]))
    M = int(rng.integers(1, 9))
    S = int(rng.integers(1, 40))
    N = int(rng.integers(1, 260))
    s = float(rng.choice([0.05, 0.2, 0.5, 0.8, 1.0]))
    kind = str(rng.choice(ls.WEIGHT_SETS))
    prec = int(rng.integers(0, 2))
    pts, _ = ls.make_shapes(S, K, seed=1000 + i)
    pairs, poses = ls.make_pairs_poses(pts, N, s=s, seed=2000 + i)
    if N >= 3:
        pairs[0, 1] = pairs[0, 0]          # a self pair
        poses[1, 1] = poses[1, 0]          # coincident poses
        pairs[2], poses[2] = pairs[0], poses[0]  # a repeated pair
    flat = ls.weight_set(kind)
    ref = oracle.query(flat, pts, pairs, poses, M=M, bf16_emul=prec == 1)
    with locc.Locc(M=M, precision=prec, device=0, max_batch=int(rng.choice([0, 7, 64]))) as ctx:
        ctx.load_weights_mem(flat)
        ctx.set_shapes(pts)
        got = ctx.query_debug(pairs, poses)
    ok = (np.array_equal(got["kept"], ref["kept"]) and np.array_equal(got["masks"], ref["masks"])
          and np.array_equal(got["occ"], ref["occ"]))
    dp = float(np.abs(got["probs"].astype(np.float64) - ref["probs"]).max(initial=0.0))
    band = np.abs(ref["probs"] - 0.5) <= 1e-3
    lab = np.array_equal(got["labels"][~band], ref["labels"][~band])
    ok = ok and dp <= P_TOL[prec] and lab
    if N >= 3:  # the repeated pair: bitwise (both precisions; bf16's default walk is deterministic, Q24)
        ok = ok and got["probs"][2] == got["probs"][0]
    desc = f"K={K} M={M} S={S} N={N} s={s} {kind} {'bf16' if prec else 'fp32'}"
    return ok, desc, dp, int(got["kept"].sum())


def main(n=60, seed=1):
    rng = np.random.default_rng(seed)
    bad = 0
    t0 = time.time()
    for i in range(n):
        ok, desc, dp, kept = case(rng, i)
        bad += not ok
        print(f"case {i:3d} {'ok  ' if ok else 'FAIL'} {desc}: kept rows {kept}, max|dp| {dp:.2e}", flush=True)
    print(f"{n - bad}/{n} cases within the parity bars ({time.time() - t0:.0f} s)")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:3]))
