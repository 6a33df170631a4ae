"""Warp-stall samples of the encoder per warp role and stall reason (ncu source page + nvdisasm).

usage: python tools/stall_by_role.py <source.csv> <nvdisasm -g -c output> <kernel .cu>
Roles are found from the '// ============ <role>' markers of the kernel source; every SASS
instruction between the first and last instruction of a role's own lines (inlined helpers
included) is attributed to that role.
"""
import csv
import re
import sys
from collections import Counter, defaultdict


def role_ranges(cu):
    marks = []
    for i, l in enumerate(open(cu), 1):
        m = re.search(r"// ============ ([^:(]+)", l)
        if m:
            marks.append((i, m.group(1).strip()))
        if "---- teardown" in l:
            marks.append((i, None))
    out = []
    for (a, name), (b, _) in zip(marks, marks[1:]):
        if name:
            out.append((a, b, name))
    return out


def main(src_csv, nvd, cu):
    rows = list(csv.reader(open(src_csv)))
    hdr = rows[1]
    ia = hdr.index("Address")
    iall = hdr.index("Warp Stall Sampling (All Samples)")
    iex = hdr.index("Instructions Executed")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    ir = [hdr.index(h) for h in reasons]
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
    rr = role_ranges(cu)
    spans = {}
    for off, (f, ln) in lines.items():
        if f != cu_name:
            continue
        for a, b, name in rr:
            if a <= ln < b:
                lo, hi = spans.get(name, (off, off))
                spans[name] = (min(lo, off), max(hi, off))
    tot = Counter()
    per = defaultdict(Counter)
    ex = Counter()
    for r in data:
        off = int(r[ia], 16) - base
        role = "other"
        for name, (lo, hi) in spans.items():
            if lo <= off <= hi:
                role = name
        tot[role] += int(r[iall] or 0)
        ex[role] += int(r[iex] or 0)
        for h, i in zip(reasons, ir):
            per[role][h] += int(r[i] or 0)
    T = sum(tot.values())
    for role, v in tot.most_common():
        top = ", ".join(f"{k[6:]} {100.0 * c / max(v, 1):.0f}%" for k, c in per[role].most_common(6) if c)
        print(f"{role:28s} {100.0 * v / T:5.1f}% of samples, {ex[role]:12d} warp-instr  | {top}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
