"""Summarise a round's ncu captures (gpurun_out/) into profiles/<tag>_summary.md + JSON.

Reads the launch list (gpu__time_duration of one step) and the --set full raw pages of the hot
kernels; writes the per-kernel share of the step, DRAM traffic per launch and the headline metrics.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "launch__registers_per_thread": "registers",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "Ghz": 1e9}


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            out[KEYS[h]] = x * SCALE.get(u, 1.0)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    res = []
    for r in rows[hi + 1:]:
        name = r[ik].split("(")[0].replace("locc::<unnamed>::", "")
        res.append((name, float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1e-9)))
    return res


def main(tag="r1"):
    L = launches(os.path.join(OUT, f"launches_{tag}.csv"))
    # one sub-batch = the launches up to and including the first predictor
    nsub = next((i + 1 for i, (name, _) in enumerate(L) if "head" in name), 8)
    step, per = {}, {}
    for name, t in L[:nsub]:
        step[name] = step.get(name, 0.0) + t
    tot = sum(step.values())
    kern = {}
    for k in ("encoder_tc", "crop_compact", "crop_count", "crop_emit", "head_tc", "head_tile"):
        p = os.path.join(OUT, f"raw_{tag}_{k}.csv")
        if os.path.exists(p):
            kern[k] = raw(p)
    lines = [f"# ncu summary, {tag}", "",
             "Workload: `python bench.py --pairs 262144 --steps 1 --warmup 1` (C3 recipe, one 262,144-pair sub-batch; "
             "the 1,048,576-pair step is four of these).  ncu 2025, `--clock-control none`, 1 x B200.", "",
             "## Launch list of one sub-batch (gpu__time_duration, serialised, cold cache)", "",
             "| kernel | ms | share |", "|---|---|---|"]
    for name, t in L[:nsub]:
        lines.append(f"| {name} | {t * 1e3:.3f} | {100 * t / tot:.1f}% |")
    lines += ["", f"Total {tot * 1e3:.2f} ms.", "", "## `--set full` per kernel (one launch)", "",
              "| kernel | ms | DRAM read GB | DRAM write GB | tensor pipe active | SM throughput | regs | SM clock GHz |",
              "|---|---|---|---|---|---|---|---|"]
    for k, d in kern.items():
        lines.append(f"| {k} | {1e3 * d.get('duration', 0):.3f} | {d.get('dram_read', 0) / 1e9:.3f} | "
                     f"{d.get('dram_write', 0) / 1e9:.3f} | {d.get('tensor_active_pct', 0):.1f}% | "
                     f"{d.get('sm_throughput_pct', 0):.1f}% | {d.get('registers', 0):.0f} | {d.get('sm_clock', 0) / 1e9:.2f} |")
    md = "\n".join(lines) + "\n"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write(md)
    js = {"tag": tag, "launches_one_subbatch": [{"kernel": n, "ms": t * 1e3} for n, t in L[:nsub]], "kernels": kern}
    json.dump(js, open(os.path.join(ROOT, "profiles", f"{tag}_summary.json"), "w"), indent=1)
    if "encoder_tc" in kern:
        e = kern["encoder_tc"]
        traffic = {"bf16": e.get("dram_read", 0) + e.get("dram_write", 0),
                   "source": f"profiles/{tag}_summary.json (ncu --set full, one 262,144-pair launch)",
                   "pairs_per_launch": 262144}
        cr = [kern[k] for k in ("crop_compact", "crop_count", "crop_emit") if k in kern]
        if cr:  # the crop's measured DRAM bytes and warp instructions per pair (one sub-batch)
            traffic["crop_bytes_per_pair"] = sum(k.get("dram_read", 0) + k.get("dram_write", 0) for k in cr) / 262144
            traffic["crop_warp_instructions_per_pair"] = sum(k.get("inst_executed", 0) for k in cr) / 262144
            traffic["crop_kernels"] = [k for k in ("crop_compact", "crop_count", "crop_emit") if k in kern]
        json.dump(traffic, open(os.path.join(ROOT, "profiles", "encoder_traffic.json"), "w"), indent=1)
    print(md)


if __name__ == "__main__":
    main(*sys.argv[1:])
