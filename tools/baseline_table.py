"""Print BASELINE.md §4's results table from a bench line (default profiles/r2_bench_line.json)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path=os.path.join(ROOT, "profiles", "r2_bench_line.json")):
    d = json.load(open(path))
    sw = d["sweep"]
    o1 = sw["oracle_1_thread"]["value"]
    oc = d["cpu_baseline"]
    c1, c2 = sw["C1"], sw["C2"]
    pct = lambda r: f"{100 * r.get('encoder_roofline_frac', 0):.0f} %"
    print("| Config | GPUs | Precision | Σ kept rows / pair | checks/s | % TC roofline | Oracle checks/s (1 core / all n cores) |")
    print("|---|---|---|---|---|---|---|")
    print(f"| C1 64 pairs | 1 | fp32 / bf16 | {c1['bf16']['kept_rows_per_pair']:.0f} | {c1['fp32']['checks_per_s']:,.0f} / "
          f"{c1['bf16']['checks_per_s']:,.0f} ({c1['bf16']['ms']:.2f} ms per query) | — / {pct(c1['bf16'])} | "
          f"{o1:.1f} / {oc['value']:.0f} ({oc['cores']} cores) |")
    print(f"| C2 16K pairs | 1 | fp32 / bf16 | {c2['bf16']['kept_rows_per_pair']:.0f} | {c2['fp32']['checks_per_s']:,.0f} / "
          f"{c2['bf16']['checks_per_s']:,.0f} | — / {pct(c2['bf16'])} | same |")
    print(f"| C3 1M pairs | 1 | bf16 | {sw['C5']['K=1500']['1048576']['kept_rows_per_pair']:.0f} | **{d['value']:,.0f}** (e2e from "
          f"host buffers {d['e2e']['value']:,.0f}; " + (f"opt-in fast walk {d['fast_walk']['value']:,.0f}" if 'fast_walk' in d else f"deterministic mode {d['deterministic']['value']:,.0f}") + ") | "
          f"**{100 * d['roofline']['frac']:.0f} %** (encoder kernel) | same ({oc['sample'].split(' pairs')[0].replace('first ', '')}-pair sample) |")
    c4 = "; ".join(f"{int(e):,}: {v['ms_per_dt_encode_once']:.2f} / {v['ms_per_dt_crop_bf16']:.1f}" for e, v in sw["C4"].items())
    print(f"| C4 sim step, E envs × 3 pairs, 4 substeps per Δt | 1 | bf16 | — | ms per Δt (encode-once / crop detector): {c4} | — | — |")
    for K, rows in sw["C5"].items():
        if not isinstance(rows, dict):
            continue
        kr = list(rows.values())[-1]["kept_rows_per_pair"]
        cells = "; ".join(f"{int(n):,}: {v['checks_per_s'] / 1e6:.2f} M ({pct(v)})" for n, v in rows.items())
        print(f"| C5 K = {K[2:]}, N = 1K … 4M | 1 | bf16 | {kr:.0f} | {cells} | in parentheses | — |")
    print("| C3 / C4 / C5 at 2, 4, 8 GPUs | 2/4/8 | bf16 | — | the driver's scaling run (`SCALE_rNN.json`); this sandbox has one GPU | — | — |")
    c = d["clocks"]
    print(f"\nclock {c['sm_mhz']} MHz, power median {c.get('power_w_median')} W, reasons {c['reasons']}")


if __name__ == "__main__":
    main(*sys.argv[1:])
