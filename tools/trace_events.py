"""Median event times of the encoder trace relative to each tile's MMA start (tools/trace_run.py output),
with the tensor-core probe completions of rank 2 (rank-1 clock).  usage: python tools/trace_events.py trace.txt"""
import sys

import numpy as np

NAMES = {0: "MMA h1 block 0 seen", 1: "MMA tile start", 2: "MMA L2b issue (D3E0 ok)", 3: "MMA L3 start",
         4: "MMA issue end", 5: "MMA p1", 6: "L1 start", 7: "L1 end", 8: "E2 sees D2a", 9: "E2 h2 free",
         10: "E2 tile end", 11: "E2 sees D2b", 12: "E3 sees D3 p0", 13: "E3 p0 done", 14: "E3 sees D3 p1",
         15: "E3 p1 done", 16: "MMA h2 chunk 4 seen", 17: "MMA chunk 5", 18: "MMA chunk 6", 19: "MMA chunk 7",
         20: "MMA L2a issued", 21: "MMA L2b issued", 22: "MMA L3p0 K-half 0 issued", 23: "MMA L3p1 K-half 0 issued"}
for e in range(24, 32):
    NAMES[e] = f"E3 warp {(e - 24) % 4} part {(e - 24) // 4} done"


def main(path):
    T = []
    for ln in open(path):
        if ln.startswith("trace r0 "):
            v = [int(x) for x in ln.split()[3:]]
            if min(v) > 0:
                T.append(v)
    T = np.array(T[2:-2], dtype=np.float64)
    R = T - T[:, 1:2]
    print(f"tiles {len(T)}, period median {np.median(np.diff(T[:, 1])):.0f}")
    for e in sorted(range(T.shape[1]), key=lambda e: np.median(R[:, e])):
        print(f"{e:2d} {NAMES.get(e, '?'):28s} {np.median(R[:, e]):7.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
