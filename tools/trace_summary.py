"""Summarise the encoder's per-tile trace (tools/trace_run.py output; rank-0 CTA of cluster 0).

Events (kernels_encoder_tc.cu trace_ev): 0 MMA sees h1 block 0, 1 MMA tile start, 2 MMA L2b start,
3 MMA L3 start, 4 MMA tile issue end, 5 MMA p1, 6 L1 tile start, 7 L1 tile end, 8 E2 sees D2a,
9 E2 sees h2 free, 10 E2 tile end, 11 E2 sees D2b, 12 E3 sees D3 part 0, 13 E3 part 0 done,
14 E3 sees D3 part 1, 15 E3 part 1 done.  Prints the per-tile period and, per role, the mean busy
time and the mean time it waited on its input (cycles).
usage: python tools/trace_summary.py gpurun_out/r2_trace.txt
"""
import sys

import numpy as np


def main(path):
    T = []
    for ln in open(path):
        if ln.startswith("trace r0 "):
            v = [int(x) for x in ln.split()[3:]]
            if min(v) > 0:
                T.append(v)
    T = np.array(T[2:-2], dtype=np.float64)  # drop warm-up / tail tiles
    per = np.diff(T[:, 1])
    print(f"tiles {len(T)}; MMA tile period mean {per.mean():.0f} cycles (median {np.median(per):.0f})")
    e3_wait0 = T[1:, 12] - T[:-1, 15]
    e3_busy0 = T[:, 13] - T[:, 12]
    e3_wait1 = T[:, 14] - T[:, 13]
    e3_busy1 = T[:, 15] - T[:, 14]
    print(f"E3: part0 busy {e3_busy0.mean():.0f}, part1 busy {e3_busy1.mean():.0f}, "
          f"wait for part0 {e3_wait0.mean():.0f}, wait for part1 {e3_wait1.mean():.0f}; "
          f"E3 busy fraction {(e3_busy0.mean() + e3_busy1.mean()) / per.mean():.2f}")
    e2_busy = T[:, 10] - T[:, 8]
    print(f"E2: D2a seen -> tile end {e2_busy.mean():.0f}; D2a->D2b {np.mean(T[:, 11] - T[:, 8]):.0f}")
    l1 = T[:, 7] - T[:, 6]
    print(f"L1: tile {l1.mean():.0f} (start->end), gap to next start {np.mean(T[1:, 6] - T[:-1, 7]):.0f}")
    print(f"MMA: start->h1 seen {np.mean(T[:, 0] - T[:, 1]):.0f}, ->L2b {np.mean(T[:, 2] - T[:, 1]):.0f}, "
          f"->L3 {np.mean(T[:, 3] - T[:, 1]):.0f}, ->issue end {np.mean(T[:, 4] - T[:, 1]):.0f}")
    print(f"MMA L2b waited on E3 part0 release: next tile L2b start - E3 part0 done = "
          f"{np.mean(T[1:, 2] - T[:-1, 13]):.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
