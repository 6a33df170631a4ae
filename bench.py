"""Benchmark of the LOCC batched collision query on B200 (BASELINE.json metric: collision checks/sec).

Default: N=1 GPU, workload C3 = 1,048,576 pairs over 1030 synthetic shapes, K=1500, M=6, H=256,
F=64, pose density s=0.5, bf16 tensor-core encoder.  A "step" = one locc_query over the whole
batch (every stage of the hot path: transforms, crop + compaction, encoder, pooling, predictor).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision bf16|fp32] [--pairs N]
  python bench.py --impl reference ...   # the CPU oracle (this tier's reference arm)

Multi-GPU (one process per GPU; `--gpus N` re-launches itself under torch.distributed.run when
WORLD_SIZE is unset): the global batch is N x 1,048,576 pairs, each rank computes its own contiguous
shard and the library gathers every rank's probabilities and labels on every rank with NCCL
(locc_query_allgather, the path's only collective) inside the timed step (weak scaling); time = max
over ranks; value = all pairs / that time.

The N = 1 line also carries the BASELINE.json config table (`sweep`: C1/C2 in fp32 and bf16, C5's
K x N grid with its roofline fractions, C4's closed-loop times, the oracle at 1 and all host threads)
and the opt-in fast bf16 walk's throughput (`fast_walk`; the headline is the default deterministic walk).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "collision checks/sec (LOCC inference)"
UNIT = "checks/s"
FLOP_PER_ROW = 2 * (3 * 256 + 2 * 256 * 256)  # encoder layers 1-3 per kept row
HEAD_FLOP = 2 * (2 * (71 * 128 + 2 * 128 * 128) + 3 * 128 * 128 + 128)  # predictor per evaluated pair
PROJ_FLOP = 2 * 2 * 256 * 64  # the two projections to F per evaluated pair (crop path)


def fp32_peak_tflops(mhz):
    """FP32 FFMA peak: 148 SMs x 128 lanes x 2 flop x clock (B200_PROFILING.md unit counts)."""
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="locc", choices=["locc", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--pairs", type=int, default=1 << 20)
    ap.add_argument("--K", type=int, default=1500)
    ap.add_argument("--s", type=float, default=0.5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-grad", action="store_true", help="skip the NEXT-2 pose-gradient measurement")
    ap.add_argument("--no-cells", action="store_true", help="skip the NEXT-1 encode-once measurement")
    ap.add_argument("--no-sim", action="store_true", help="skip the NEXT-3 closed-loop measurement")
    ap.add_argument("--sim-envs", type=int, default=30000)
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-table sweep (C1/C2/C4/C5)")
    ap.add_argument("--allgather", action="store_true",
                    help="time the library NCCL gather (locc_query_allgather) even in a world of one rank")
    return ap.parse_args()


def relaunch_distributed(a):
    """`--gpus N` without a torchrun environment: start N ranks of this script under
    torch.distributed.run (rendezvous on 127.0.0.1) and return their exit code; rank 0 prints the line."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < a.gpus:
        raise SystemExit(f"bench.py --gpus {a.gpus}: only {have} CUDA device(s) visible")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def workload_name(a):
    return (f"C3: {a.pairs} pairs/GPU over 1030 synthetic non-convex shapes, K={a.K}, M=6, H=256, F=64, "
            f"pose density s={a.s}, spread weights (seeded random init)")


def make_inputs(a, rank):
    import locc_synth as ls
    pts, _ = ls.make_shapes(1030, a.K, seed=1)
    pairs, poses = ls.make_pairs_poses(pts, a.pairs, s=a.s, seed=2 + rank)
    flat = ls.flatten_weights(ls.make_weights("spread", calib=ls.load_calibration()))
    return pts, pairs, poses, flat


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.limit")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons, pw, lim, capped = [], [], set(), [], [], 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
                lim.append(float(f[9]))
            except (ValueError, IndexError):
                pass
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
            capped += f[8].lower() == "active"
        # the power trace: draw against the enforced limit while the encoder runs (the sw_power_cap
        # samples are the ones where the driver lowered the SM clock to stay under the limit)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None, "power_w_max": max(pw) if pw else None,
                "power_limit_w": statistics.median(lim) if lim else None, "sw_power_cap_samples": capped}


def cpu_baseline(pts, pairs, poses, flat, target_s=15.0):
    """The oracle as it stands (fp64 network, bf16-emulating to match the GPU arithmetic), timed on
    this host's cores on a bounded prefix of the same workload."""
    import oracle
    cores = os.cpu_count() or 1
    n = max(4 * cores, 64)
    oracle.query(flat, pts, pairs[:cores], poses[:cores], bf16_emul=True, n_threads=cores)  # warm-up
    t = time.perf_counter()
    oracle.query(flat, pts, pairs[:n], poses[:n], bf16_emul=True, n_threads=cores)
    dt = time.perf_counter() - t
    n2 = int(min(len(pairs), max(n, n * target_s / max(dt, 1e-3))))
    t = time.perf_counter()
    oracle.query(flat, pts, pairs[:n2], poses[:n2], bf16_emul=True, n_threads=cores)
    dt2 = time.perf_counter() - t
    return {"value": n2 / dt2, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {n2} pairs of the workload ({dt2:.1f} s, {cores} threads, bf16-emulating fp64 oracle)"}


def run_reference(a):
    """--impl reference: the CPU oracle on the host cores, same config/metric, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pts, pairs, poses, flat = make_inputs(a, 0)
    import oracle
    cores = os.cpu_count() or 1
    # size the per-step sample to ~8 s of host work (a warm probe first), so K + W steps take minutes
    oracle.query(flat, pts, pairs[:cores], poses[:cores], bf16_emul=True, n_threads=cores)
    n0 = max(4 * cores, 64)
    t = time.perf_counter()
    oracle.query(flat, pts, pairs[:n0], poses[:n0], bf16_emul=True, n_threads=cores)
    dt = time.perf_counter() - t
    n = int(max(n0, min(len(pairs) // (a.steps + 2), n0 * 8.0 / max(dt, 1e-3))))
    for i in range(a.warmup):
        oracle.query(flat, pts, pairs[:n], poses[:n], bf16_emul=True, n_threads=cores)
    times = []
    for i in range(a.steps):
        sl = slice(n * (i + 1), n * (i + 2))
        t = time.perf_counter()
        oracle.query(flat, pts, pairs[sl], poses[sl], bf16_emul=True, n_threads=cores)
        times.append(time.perf_counter() - t)
    ms = 1e3 * statistics.mean(times)
    v = n / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(a), "sample_pairs_per_step": n},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{n} consecutive pairs of the workload per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def time_query(ctx, torch, stream, pairs, poses, probs, labels, reps=3, warm=2, flush=None):
    """Mean device time (ms) of one locc_query over device-resident inputs (CUDA events on the
    query's stream; the L2 flushed before each timed call when the batch is large)."""
    for _ in range(warm):
        ctx.query_into(pairs, poses, probs, labels, stream=stream.cuda_stream)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            if flush is not None:
                flush.zero_()
            e0.record(stream)
        ctx.query_into(pairs, poses, probs, labels, stream=stream.cuda_stream)
        with torch.cuda.stream(stream):
            e1.record(stream)
        stream.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts)


def run_sweep(a, locc, torch, stream, flush, peaks):
    """BASELINE.json configs as a table: C1 and C2 in fp32 and bf16; C5 = K x N with
    the encoder's tensor-core roofline fraction per cell; C4 = the closed-loop step at 4K-65K
    environments with both detectors; the oracle at 1 host thread (its all-threads rate is cpu_baseline)."""
    import locc_synth as ls
    import oracle
    out = {}
    flat = ls.weight_set("spread")
    peak_s = peaks.get("bf16_tflops_sustained", 1400.0)
    peak_b = peaks.get("bf16_tflops", 1640.0)

    def one(points, pairs, poses, prec):
        ctx = locc.Locc(precision=prec, device=torch.cuda.current_device())
        ctx.load_weights_mem(flat)
        ctx.set_shapes(points)
        n = len(pairs)
        dp, dq = torch.from_numpy(pairs).cuda(), torch.from_numpy(poses).cuda()
        pr, lb = torch.empty(n, device="cuda"), torch.empty(n, dtype=torch.uint8, device="cuda")
        ms = time_query(ctx, torch, stream, dp, dq, pr, lb, flush=flush if n >= 65536 else None)
        ctx.set_timing(True)
        ctx.query_into(dp, dq, pr, lb, stream=stream.cuda_stream)
        stream.synchronize()
        st = ctx.stats()
        ctx.close()
        r = {"pairs": n, "ms": ms, "checks_per_s": n / (ms / 1e3), "kept_rows_per_pair": st["kept_rows"] / n}
        if prec == locc.LOCC_PREC_BF16 and st["encoder_ms"] > 0:
            # the burst peak for a query shorter than 50 ms (the board reaches its power cap later), the
            # sustained one for longer ones (MEASURED_PEAKS.json; B200_PROFILING.md)
            peak, kind = (peak_b, "burst") if ms < 50.0 else (peak_s, "sustained")
            tf = FLOP_PER_ROW * st["kept_rows"] / (st["encoder_ms"] / 1e3) / 1e12
            r["encoder_tflops"] = tf
            r["encoder_roofline_frac"] = tf / peak
            r["step_roofline_frac"] = FLOP_PER_ROW * st["kept_rows"] / (ms / 1e3) / 1e12 / peak
            r["peak_tflops"], r["peak_kind"] = peak, kind
        return r

    # C1 (64 pairs over 16 shapes) and C2 (16,384 pairs over 1030 shapes), both precisions
    for name in ("C1", "C2"):
        wl = ls.make_workload(name)
        out[name] = {p: one(wl.points, wl.pairs, wl.poses, getattr(locc, f"LOCC_PREC_{p.upper()}"))
                     for p in ("fp32", "bf16")}
    # C5: K x N (bf16); 4M pairs per query at the largest N
    out["C5"] = {"note": "bf16, s = 0.5; K sets the kept rows per pair, so the encoder FLOPs scale with K "
                         "(this path crops then encodes; the paper's K-independence is the encode-once mode's)"}
    for K in (512, 1500, 4096):
        pts, _ = ls.make_shapes(1030, K, seed=1)
        pairs, poses = ls.make_pairs_poses(pts, 1 << 22, s=0.5, seed=2)
        row = {}
        for n in (1024, 16384, 262144, 1 << 20, 1 << 22):
            row[str(n)] = one(pts, pairs[:n], poses[:n], locc.LOCC_PREC_BF16)
        out["C5"][f"K={K}"] = row
    # C4: closed-loop step (dt = 0.01/4 s in 4 substeps), both detectors, bf16 context
    pts, _ = ls.make_shapes(1030, 1500, seed=1)
    ctx = locc.Locc(precision=locc.LOCC_PREC_BF16, device=torch.cuda.current_device())
    ctx.load_weights_mem(flat)
    ctx.set_shapes(pts)
    ctx.load_unet_weights_mem(ls.flatten_unet(ls.make_unet_weights()))
    ctx.encode_shapes()
    c4 = {}
    for E in (4096, 8192, 16384, 32768, 65536):
        ids, body, st0 = ls.make_sim_scene(pts, E, seed=6)
        di, db = torch.from_numpy(ids).cuda(), torch.from_numpy(body).cuda()
        row = {}
        for det in ("cells", "crop"):
            sim = dict(ls.SIM_DEFAULTS, detector=det)
            ds = torch.from_numpy(st0).cuda()
            for _ in range(2):
                ctx.sim_run(sim, di, db, ds, stream=stream.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
            for k in range(3):
                ctx.sim_run(sim, di, db, ds, t0=k * sim["h"] * sim["substeps"], stream=stream.cuda_stream)
            with torch.cuda.stream(stream):
                e1.record(stream)
            stream.synchronize()
            row[det] = e0.elapsed_time(e1) / 3
        c4[str(E)] = {"pairs_per_substep": 3 * E, "ms_per_dt_encode_once": row["cells"],
                      "ms_per_dt_crop_bf16": row["crop"]}
    ctx.close()
    out["C4"] = c4
    # the oracle at one host thread (bounded sample)
    wl = ls.make_workload("C2")
    oracle.query(flat, wl.points, wl.pairs[:2], wl.poses[:2], bf16_emul=True, n_threads=1)
    t = time.perf_counter()
    n1 = 0
    while time.perf_counter() - t < 5.0:
        oracle.query(flat, wl.points, wl.pairs[n1:n1 + 4], wl.poses[n1:n1 + 4], bf16_emul=True, n_threads=1)
        n1 += 4
    out["oracle_1_thread"] = {"value": n1 / (time.perf_counter() - t), "unit": UNIT, "cores": 1,
                              "sample": f"first {n1} pairs of C2, bf16-emulating fp64 oracle"}
    return out


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(relaunch_distributed(a))
    import torch
    import torch.distributed as dist

    from paper_2304_09439_b200 import build as b
    b.build()
    from paper_2304_09439_b200 import locc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"bench.py --gpus {a.gpus} launched with WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prec = locc.LOCC_PREC_BF16 if a.precision == "bf16" else locc.LOCC_PREC_FP32

    pts, pairs, poses, flat = make_inputs(a, rank)
    N = len(pairs)
    ctx = locc.Locc(precision=prec, device=local)
    ctx.load_weights_mem(flat)
    ctx.set_shapes(pts)
    d_pairs = torch.from_numpy(pairs).cuda()
    d_poses = torch.from_numpy(poses).cuda()
    d_probs = torch.empty(N, device="cuda")
    d_labels = torch.empty(N, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step():
        ctx.query_into(d_pairs, d_poses, d_probs, d_labels, stream=stream.cuda_stream)

    if world > 1 or a.allgather:
        # the global batch: this rank's pairs at its shard [rank N, (rank + 1) N) (the only slice the
        # library reads); every rank ends each step with all world x N results (NCCL, in the library)
        uid = [locc.comm_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(world, rank, uid[0])
        g_pairs = torch.zeros(world * N, 2, dtype=torch.int32, device="cuda")
        g_poses = torch.zeros(world * N, 2, 7, device="cuda")
        g_pairs[rank * N:(rank + 1) * N] = d_pairs
        g_poses[rank * N:(rank + 1) * N] = d_poses
        g_probs = torch.empty(world * N, device="cuda")
        g_labels = torch.empty(world * N, dtype=torch.uint8, device="cuda")

        def step():  # noqa: F811
            ctx.query_allgather_into(g_pairs, g_poses, g_probs, g_labels, stream=stream.cuda_stream)

    for _ in range(a.warmup):
        step()
    stream.synchronize()
    ctx.set_timing(True)
    # one step with the crop pipeline serialised (LOCC_NO_OVERLAP): kept rows, launches and the per-stage
    # device times (crop, predictor) for the rooflines — in the timed steps the crop of sub-batch s + 1
    # overlaps the encoder of sub-batch s, so its elapsed time there is not its cost
    os.environ["LOCC_NO_OVERLAP"] = "1"
    try:
        step()
        stream.synchronize()
        st = ctx.stats()
    finally:
        del os.environ["LOCC_NO_OVERLAP"]
    ctx.set_timing(False)

    clocks = Clocks(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    enc_ms = []
    for i in range(a.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
        ctx.set_timing(True)
        step()
        with torch.cuda.stream(stream):
            ev[i][1].record(stream)
        stream.synchronize()
        tst = ctx.stats()  # the timed step's own launch counts
        enc_ms.append(tst["encoder_ms"])
        ctx.set_timing(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # roofline of the dominant kernel (the encoder), algorithmic FLOPs of the kept rows only
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    kept = st["kept_rows"]
    launches_per_step = tst["kernel_launches"]
    subs = max(1, tst["sub_batches"])
    enc_s = statistics.mean(enc_ms) / 1e3
    achieved = FLOP_PER_ROW * kept / enc_s / 1e12 if enc_s > 0 else None
    if prec == locc.LOCC_PREC_BF16:
        peak = peaks.get("bf16_tflops_sustained", 1400.0)
        roof = {"bound": "tensor", "unit": "TFLOP/s",
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained" if peaks else "fallback 1.4 PF sustained"}
    else:
        mhz = clk.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
        roof = {"bound": "alu", "unit": "TFLOP/s",
                "peak_source": f"148 SM x 128 FP32 FMA/clk x 2 x {mhz:.0f} MHz (median SM clock under load)"}
    traffic, crop_ncu, tj = None, None, {}
    tp = os.path.join(ROOT, "profiles", "encoder_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic, crop_ncu = tj.get(a.precision), tj.get("crop_bytes_per_pair")
        except Exception:
            traffic = None
    roof.update({"achieved": achieved, "peak": peak, "frac": (achieved / peak) if achieved else None,
                 "traffic": traffic, "kernel": "encoder_tc_kernel" if prec else "encoder_f32_kernel",
                 "launches_per_step": subs, "flop_per_launch": FLOP_PER_ROW * kept / subs,
                 "avg_launch_ms": 1e3 * enc_s / subs, "encoder_share_of_step": (1e3 * enc_s) / ms})
    mhz_load = clk.get("sm_mhz") or 1965.0
    if st.get("head_ms"):
        hf = (HEAD_FLOP + PROJ_FLOP) * st["evaluated_pairs"]
        if prec == locc.LOCC_PREC_BF16 and not os.environ.get("LOCC_HEAD_FFMA"):
            hk = {"kernel": "head_tc_kernel", "bound": "tensor",
                  "peak": peaks.get("bf16_tflops_sustained", 1374.0) * 1.1 / 2.25 / 3,
                  "peak_source": "MEASURED_PEAKS bf16 sustained x 1.1/2.25 (tf32) / 3 (3xTF32 split)"}
        else:
            hk = {"kernel": "head_tile_kernel", "bound": "alu", "peak": fp32_peak_tflops(mhz_load),
                  "peak_source": "148 SM x 128 FP32 FMA/clk x 2 x median SM clock"}
        hk.update({"ms_per_step": st["head_ms"], "achieved": hf / (st["head_ms"] / 1e3) / 1e12, "unit": "TFLOP/s",
                   "flop_per_evaluated_pair": HEAD_FLOP + PROJ_FLOP})
        hk["frac"] = hk["achieved"] / hk["peak"]
        roof["predictor"] = hk
    if st.get("crop_ms"):
        # The crop (segment_xf + crop_compact) is issue-bound (ncu: DRAM ~12 %, L2 ~32 % of peak; the shape
        # table is L2-resident): its roofline is warp-instruction issue, 4 per SM per cycle x 148 SMs at the
        # median SM clock under load, with the ncu-counted warp instructions per pair of the round's
        # capture.  north_star's HBM view (algorithmic point bytes 2 K 12 B + 69 B per pair per crop time)
        # and the measured DRAM bytes per pair ride along.
        hbm = peaks.get("hbm_gbs", 6546.6)
        cb = (2 * a.K * 12 + 69) * N
        crop_s = st["crop_ms"] / 1e3
        ci = tj.get("crop_warp_instructions_per_pair")
        issue_peak = 148 * 4 * mhz_load * 1e6 / 1e9  # G warp-instructions / s
        roof["crop"] = {"bound": "alu", "kernels": "segment_xf + crop_compact (one launch: crop, look-back, rows)",
                        "note": "timed with the crop serialised (LOCC_NO_OVERLAP); its blocks cannot run beside the "
                                "encoder's CTAs, so in the measured steps its time is exposed",
                        "ms_per_step": st["crop_ms"], "unit": "G warp-instructions/s",
                        "achieved": (ci * N / crop_s / 1e9) if ci else None, "peak": issue_peak,
                        "peak_source": f"148 SM x 4 schedulers x 1 warp-instruction/clk x {mhz_load:.0f} MHz",
                        "frac": (ci * N / crop_s / 1e9 / issue_peak) if ci else None,
                        "warp_instructions_per_pair_ncu": ci,
                        "point_bytes_rate_gbs": cb / crop_s / 1e9, "point_bytes_frac_of_hbm": cb / crop_s / 1e9 / hbm,
                        "algorithmic_bytes_per_pair": 2 * a.K * 12 + 69,
                        "dram_bytes_per_pair_ncu": crop_ncu,
                        "ncu_source": "profiles/encoder_traffic.json (from the round's ncu capture)"}

    line = {"metric": METRIC, "value": world * N / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": a.precision, "data": "synthetic",
            "config": {"workload": workload_name(a), "pairs_per_gpu": N, "global_pairs": world * N,
                       "kept_rows_per_step": kept, "kept_rows_per_pair": kept / N,
                       "evaluated_pairs": st["evaluated_pairs"], "sub_batches": subs,
                       "l2": "L2 flushed (256 MB write) before every timed step; working set (GBs of rows) >> L2",
                       "parallelism": f"pair-batch shards, 1 process/GPU x {world}"
                                      + (", library NCCL gather of all results on every rank (locc_query_allgather)"
                                         if world > 1 or a.allgather else "")},
            "gpu_launches": launches_per_step * a.steps, "clocks": clk, "roofline": roof}

    # NEXT-2: the same step with the pose gradient (locc_query_grad), device-timed the same way
    if not a.no_grad:
        d_grad = torch.empty(N, 14, device="cuda")

        def gstep():
            ctx.query_grad_into(d_pairs, d_poses, d_probs, d_grad, d_labels, stream=stream.cuda_stream)

        for _ in range(a.warmup):
            gstep()
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(a.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                gev[i][0].record(stream)
            gstep()
            with torch.cuda.stream(stream):
                gev[i][1].record(stream)
        torch.cuda.synchronize()
        gms = statistics.mean([s.elapsed_time(e) for s, e in gev])
        if world > 1:
            t = torch.tensor([gms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gms = float(t.item())
        line["pose_grad"] = {"metric": "collision checks with d logit / d pose per second", "value": world * N / (gms / 1e3),
                             "unit": UNIT, "ms_per_step": gms, "overhead_vs_forward": gms / ms - 1.0,
                             "api": "locc_query_grad (grad [N][14] fp32)"}

    # small-batch latency (SURVEY §8(d) C5's small-N floor): device time of one locc_query call
    lat = {}
    for n_small in (1024, 16384):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            ctx.query_into(d_pairs[:n_small], d_poses[:n_small], d_probs[:n_small], d_labels[:n_small],
                           stream=stream.cuda_stream)
        with torch.cuda.stream(stream):
            e0.record(stream)
        for _ in range(10):
            ctx.query_into(d_pairs[:n_small], d_poses[:n_small], d_probs[:n_small], d_labels[:n_small],
                           stream=stream.cuda_stream)
        with torch.cuda.stream(stream):
            e1.record(stream)
        torch.cuda.synchronize()
        lat[str(n_small)] = e0.elapsed_time(e1) / 10
    line["latency_ms_per_query"] = lat

    # NEXT-1: the paper's encode-once inference on the same pairs (grids cached once per shape table)
    if not a.no_cells:
        import locc_synth as ls
        ctx.load_unet_weights_mem(ls.flatten_unet(ls.make_unet_weights()))
        ctx.encode_shapes()
        enc_ms_first = ctx.encode_ms()  # includes the kernels' first-launch (module load) costs
        ctx.encode_shapes()
        enc_ms = ctx.encode_ms()

        def cstep():
            ctx.query_cells_into(d_pairs, d_poses, d_probs, d_labels, stream=stream.cuda_stream)

        for _ in range(a.warmup):
            cstep()
        cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(a.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                cev[i][0].record(stream)
            cstep()
            with torch.cuda.stream(stream):
                cev[i][1].record(stream)
        torch.cuda.synchronize()
        cms = statistics.mean([s.elapsed_time(e) for s, e in cev])
        if world > 1:
            t = torch.tensor([cms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            cms = float(t.item())
        ctx.set_timing(True)
        cstep()
        stream.synchronize()
        cst = ctx.stats()
        ctx.set_timing(False)
        hf = HEAD_FLOP * cst["evaluated_pairs"]
        mhz_load = clk.get("sm_mhz") or 1965.0
        if os.environ.get("LOCC_HEAD_FFMA"):
            hroof = {"kernel": "head_tile_kernel", "bound": "alu", "peak": fp32_peak_tflops(mhz_load),
                     "peak_source": "148 SM x 128 FP32 FMA/clk x 2 x median SM clock"}
        else:
            # 3xTF32 on tcgen05: the fp32-accurate contraction costs three tf32 products, so its peak is
            # the tf32 peak / 3; tf32 peak = measured sustained bf16 x the guide's nominal 1.1 / 2.25
            tf32 = peaks.get("bf16_tflops_sustained", 1374.0) * 1.1 / 2.25
            hroof = {"kernel": "head_tc_kernel", "bound": "tensor", "peak": tf32 / 3,
                     "peak_source": "MEASURED_PEAKS bf16 sustained x 1.1/2.25 (tf32) / 3 (3xTF32 split)"}
        hroof.update({"unit": "TFLOP/s", "achieved": hf / (cst["head_ms"] / 1e3) / 1e12,
                      "frac": hf / (cst["head_ms"] / 1e3) / 1e12 / hroof["peak"],
                      "flop_per_evaluated_pair": HEAD_FLOP})
        line["encode_once"] = {"metric": "collision checks/sec, encode-once mode (locc_query_cells)",
                               "kernels": {"cells_select_ms": cst["encoder_ms"], "head_ms": cst["head_ms"],
                                           "head_roofline": hroof},
                               "value": world * N / (cms / 1e3), "unit": UNIT, "ms_per_step": cms,
                               "encode_ms_per_shape_table": enc_ms, "encode_ms_first_call": enc_ms_first,
                               "shapes": int(len(pts)),
                               "note": "grids encoded once per shape table (not in the timed step); grid layers "
                                       "2-3 and U-Net on tcgen05 (3xTF32) in bf16 contexts, fp32 FFMA in fp32 ones"}

    # NEXT-3: closed-loop substeps (30,000 environments, dt = 0.01/4 s in 4 substeps)
    if not a.no_sim and not a.no_cells:
        import locc_synth as ls
        E = a.sim_envs
        ids, body, st0 = ls.make_sim_scene(pts, E, seed=5 + rank)
        d_ids = torch.from_numpy(ids).cuda()
        d_body = torch.from_numpy(body).cuda()
        d_con = torch.zeros(E, 3, dtype=torch.int32, device="cuda")
        res = {}
        for det in ("cells", "crop"):
            sim = dict(ls.SIM_DEFAULTS, detector=det)
            d_st = torch.from_numpy(st0).cuda()
            t = 0.0
            for _ in range(a.warmup):
                ctx.sim_run(sim, d_ids, d_body, d_st, t0=t, contacts=d_con, stream=stream.cuda_stream)
                t += sim["h"] * sim["substeps"]
            sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
            torch.cuda.synchronize()
            ncon = 0
            for i in range(a.steps):
                with torch.cuda.stream(stream):
                    sev[i][0].record(stream)
                ctx.sim_run(sim, d_ids, d_body, d_st, t0=t, contacts=d_con, stream=stream.cuda_stream)
                with torch.cuda.stream(stream):
                    sev[i][1].record(stream)
                t += sim["h"] * sim["substeps"]
            torch.cuda.synchronize()
            ncon = int(d_con.sum().item())
            sms = statistics.mean([s_.elapsed_time(e_) for s_, e_ in sev])
            if world > 1:
                tt = torch.tensor([sms], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                sms = float(tt.item())
            res[det] = {"ms_per_dt": sms, "contact_pair_substeps_last_dt": ncon,
                        "finite_state": bool(torch.isfinite(d_st).all().item())}
        # Fig. 3c's axis: time per dt against the number of environments (encode-once detector)
        sweep = {}
        for Es in (4096, 16384, 65536):
            ids_s, body_s, st_s = ls.make_sim_scene(pts, Es, seed=6 + rank)
            di, db, ds = (torch.from_numpy(x).cuda() for x in (ids_s, body_s, st_s))
            sim = dict(ls.SIM_DEFAULTS, detector="cells")
            for _ in range(2):
                ctx.sim_run(sim, di, db, ds, stream=stream.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
            for k in range(5):
                ctx.sim_run(sim, di, db, ds, t0=k * sim["h"] * sim["substeps"], stream=stream.cuda_stream)
            with torch.cuda.stream(stream):
                e1.record(stream)
            torch.cuda.synchronize()
            sweep[str(Es)] = e0.elapsed_time(e1) / 5
        line["closed_loop"] = {"metric": "device time per simulated dt (4 substeps), locc_sim_run",
                               "ms_per_dt_vs_envs_encode_once": sweep,
                               "envs_per_gpu": E, "pairs_per_substep": 3 * E, "unit": "ms",
                               "detector_encode_once": res["cells"], "detector_crop_" + a.precision: res["crop"],
                               "note": "PAPER.md:91/:100 scene: bowl shaken + 2 dropped objects per env; "
                                       "query + pose gradient + penalty + semi-implicit Euler on the GPU"}

    # e2e: same metric through the public API with HOST buffers (pinned), copies in the timed region
    if not a.no_e2e:
        h_pairs = torch.from_numpy(pairs).pin_memory()
        h_poses = torch.from_numpy(poses).pin_memory()
        h_probs = torch.empty(N).pin_memory()
        h_labels = torch.empty(N, dtype=torch.uint8).pin_memory()
        ctx.query_into(h_pairs, h_poses, h_probs, h_labels)
        ts = []
        for _ in range(max(2, min(a.steps, 3))):
            t = time.perf_counter()
            ctx.query_into(h_pairs, h_poses, h_probs, h_labels)
            ts.append(time.perf_counter() - t)
        e2e_s = statistics.mean(ts)
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        line["e2e"] = {"value": world * N / e2e_s, "unit": UNIT, "h2d_bytes_per_step": N * (8 + 56),
                       "d2h_bytes_per_step": N * (4 + 1), "timer": "host perf_counter around the synchronous call"}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(pts, pairs, poses, flat)
    if world == 1:
        # the headline is the default (deterministic) bf16 walk; the opt-in fast walk (locc_set_
        # deterministic(ctx, 0): ~5 % faster, batch composition moves probabilities by <= 1e-5)
        if prec == locc.LOCC_PREC_BF16:
            ctx.set_deterministic(False)
            fms = time_query(ctx, torch, stream, d_pairs, d_poses, d_probs, d_labels, reps=a.steps,
                             warm=1, flush=flush)
            ctx.set_deterministic(True)
            line["fast_walk"] = {"value": N / (fms / 1e3), "unit": UNIT, "ms_per_step": fms,
                                 "api": "locc_set_deterministic(ctx, 0)",
                                 "note": "not bitwise invariant to batch composition (<= 1e-5 in probability)"}
        if not a.no_sweep:
            line["sweep"] = run_sweep(a, locc, torch, stream, flush, peaks)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
