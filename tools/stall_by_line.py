"""Aggregate ncu source-page warp-stall samples of the encoder by CUDA source line.

usage: python tools/stall_by_line.py <source.csv from ncu --page source --csv> <nvdisasm -g -c output of the same kernel>
The SASS offsets of the ncu page (relative to the kernel's first instruction) are matched with the
line table of nvdisasm so that samples can be attributed to kernels_encoder_tc.cu lines.
"""
import csv
import re
import sys
from collections import Counter, defaultdict


def main(src_csv, nvd):
    rows = list(csv.reader(open(src_csv)))
    hdr = rows[1]
    ia, isrc, iall, inot, iex = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                       "Warp Stall Sampling (Not-issued Samples)", "Instructions Executed"))
    data = [r for r in rows[2:] if len(r) > iex and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    lines = {}
    cur = None
    for l in open(nvd):
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            lines[int(m.group(1), 16)] = cur
    by = Counter()
    ex = Counter()
    tot = 0
    for r in data:
        off = int(r[ia], 16) - base
        k = lines.get(off, ("?", 0))
        s = int(r[iall] or 0)
        by[k] += s
        ex[k] += int(r[iex] or 0)
        tot += s
    print(f"total samples {tot}")
    for k, v in by.most_common(45):
        print(f"{v:8d} {100.0 * v / tot:5.1f}%  exec {ex[k]:10d}  {k[0]}:{k[1]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
