"""Write tests/golden/spread_calibration.json — the two scalars of the `spread` weight set.

Reading Q16: with SPEC init the logits of random weights are all positive, so
label parity would be vacuous.  `spread` = seeded draws with enc.l1.W bound x10 and zero
biases; then out.W is scaled by c and out.b set to b so that the fp64 ORACLE's logits on a
fixed calibration batch (the first 1024 pairs of config C2) have std 2 and median 0.
`python tools/calibrate_spread.py spread_bias` does the same for the `spread_bias` set (the
spread weights with non-zero hidden biases) and writes tests/golden/spread_bias_calibration.json.
This script calls only oracle/ and locc_synth (never the CUDA path).
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import locc_synth as ls  # noqa: E402
import oracle  # noqa: E402


def main(kind="spread"):
    wl = ls.make_workload("C2")
    n = 1024
    w = ls.make_weights(kind, calib=None)
    w["out.b"][:] = 0.0  # the raw logits are taken with a zero output bias, which the calibration then sets
    r = oracle.query(ls.flatten_weights(w), wl.points, wl.pairs[:n], wl.poses[:n])
    ev = np.isfinite(r["logits"])
    lg = r["logits"][ev]
    c = 2.0 / float(np.std(lg))
    b = -c * float(np.median(lg))
    out = {"scale": c, "bias": b, "calibration_batch": "C2 pairs[0:1024] (K=1500, s=0.5, seeds 1/2/3)",
           "evaluated_pairs": int(ev.sum()), "raw_logit_std": float(np.std(lg)),
           "raw_logit_median": float(np.median(lg)), "written_by": f"tools/calibrate_spread.py {kind} (oracle only)"}
    path = ls.default_calibration_path(kind)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    w2 = ls.make_weights(kind, calib=out)
    r2 = oracle.query(ls.flatten_weights(w2), wl.points, wl.pairs[:n], wl.poses[:n])
    lg2 = r2["logits"][ev]
    print(json.dumps(out), "check std", np.std(lg2), "median", np.median(lg2),
          "label1 frac", r2["labels"][ev].mean())


if __name__ == "__main__":
    main(*sys.argv[1:2])
