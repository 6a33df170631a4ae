"""Executed-instruction mix of one warp role (ncu source page + nvdisasm line table).

usage: python tools/role_mix.py <source.csv> <nvdisasm -g -c output> <kernel .cu> <role name prefix>
"""
import csv
import re
import sys
from collections import Counter

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from stall_by_role import role_ranges  # noqa: E402


def main(src_csv, nvd, cu, role):
    rows = list(csv.reader(open(src_csv)))
    hdr = rows[1]
    ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    data = [r for r in rows[2:] if len(r) > iex and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    cu_name = cu.split("/")[-1]
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
    lo = hi = None
    for a, b, name in role_ranges(cu):
        if name.startswith(role):
            offs = [o for o, (f, ln) in lines.items() if f == cu_name and a <= ln < b]
            lo, hi = min(offs), max(offs)
    mix = Counter()
    tot = 0
    for r in data:
        o = int(r[ia], 16) - base
        if lo <= o <= hi:
            src = r[isrc].strip()
            op = src.split()[1] if src.startswith("@") else src.split()[0]
            n = int(r[iex] or 0)
            mix[op.split(".")[0]] += n
            tot += n
    print(f"{role}: {tot} warp-instructions")
    for op, n in mix.most_common(30):
        print(f"  {op:12s} {n:12d} {100.0 * n / tot:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:5])
