"""Summarise the NEXT-mode ncu captures (tools/profile_next.sh) into profiles/<tag>_summary.md + JSON."""
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
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "Ghz": 1e9,
         "Mhz": 1e6}
CAPS = [("grid_gemm", "grid encode layers 1+2 (one 128-column half, 699 shapes x 1500 points) on tcgen05 "
                      "(3xTF32, conv_tc_kernel pts mode: layer 1 computed in the producers)"),
        ("grid_cellmax", "grid encode: cell-wise max of layer 3 over the chunk's sorted points"),
        ("conv_c1", "U-Net c1 on tcgen05 (3xTF32): valid 3^3 conv 256 -> 128 (once per shape table)"),
        ("conv_d1", "U-Net d1 on tcgen05: transposed valid conv [d2; c1] -> 128 (once per shape table)"),
        ("cells_select", "encode-once query: cell selection + pooled embedding"),
        ("head_cells", "head_tc_kernel<0,0>: tensor-core predictor on pooled cell embeddings"),
        ("head_grad", "head_tc_kernel<1,1>: tensor-core predictor + pose gradient (crop path)"),
        ("sim_integrate", "closed loop: penalty + semi-implicit Euler")]


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                out[KEYS[h]] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
            except ValueError:
                pass
    return out


def main(tag="r1next"):
    res = {}
    lines = [f"# ncu summary, NEXT modes ({tag})", "",
             "Workload: `python tools/next_modes.py` (262,144 C3-recipe pairs over 1030 shapes; grids encoded "
             "once; closed loop at 30,000 environments).  `ncu --set full --clock-control none`, one launch "
             "per kernel, 1 x B200.  Captured by `tools/profile_next.sh`.", "",
             "| kernel | what | ms | DRAM R/W GB | L2 read GB | issue active | FMA pipe | tensor pipe | occupancy | regs |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for k, what in CAPS:
        p = os.path.join(OUT, f"next_raw_{tag}_{k}.csv")
        if not os.path.exists(p):
            continue
        d = raw(p)
        res[k] = d
        lines.append(f"| {k} | {what} | {1e3 * d.get('duration', 0):.3f} | {d.get('dram_read', 0) / 1e9:.3f} / "
                     f"{d.get('dram_write', 0) / 1e9:.3f} | {32 * d.get('l2_read_sectors', 0) / 1e9:.2f} | "
                     f"{d.get('issue_active_pct', 0):.0f}% | {d.get('fma_pipe_pct', 0):.0f}% | "
                     f"{d.get('tensor_pct', 0):.0f}% | "
                     f"{d.get('occupancy_pct', 0):.0f}% | {d.get('registers', 0):.0f} |")
    json.dump(res, open(os.path.join(ROOT, "profiles", f"{tag}_summary.json"), "w"), indent=1)
    open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
