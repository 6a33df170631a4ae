"""Checked build run: this pool's substitute for compute-sanitizer (closed here; profiles/r2_sanitize_memcheck.txt).

1. Builds /tmp/liblocc_checked.so with -DLOCC_CHECKED=1: device-side bounds checks (LOCC_CHECK,
   csrc/internal.h) on the global-memory indices of the crop, both encoders, both predictors and the
   cell selection; a failed check prints the condition and traps.
2. Self-test: a child process shrinks the rows capacity the checks see (LOCC_CHECK_SELFTEST) and must
   fail with LOCC_E_CUDA and a "LOCC_CHECK failed" line, so the checks are known to be live.
3. Race probe (racecheck/synccheck stand-in): the tensor-core kernels' results on the same batch do not
   depend on timing, so repeated queries (both walk modes, the pose gradient, the encode-once path) must
   be bitwise equal run to run; a race on the cross-CTA mbarrier/TMEM protocol would show up as a
   difference (or as the watchdog's trap).
4. The -m gpu parity suite against the checked library (LOCC_LIB).

usage: python tools/checked_run.py [pytest args...]      (on the GPU box)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = "/tmp/liblocc_checked.so"


def selftest_child():
    import locc_synth as ls
    from paper_2304_09439_b200 import locc
    pts, _ = ls.make_shapes(4, 300, seed=90)
    pairs, poses = ls.make_pairs_poses(pts, 16, s=0.5, seed=91)
    with locc.Locc(precision=locc.LOCC_PREC_BF16, device=0) as ctx:
        ctx.load_weights_mem(ls.weight_set("spread_bias"))
        ctx.set_shapes(pts)
        try:
            ctx.query(pairs, poses)
        except locc.LoccError as e:
            print("selftest: query failed as expected:", e)
            sys.exit(3)
    print("selftest: query succeeded (the check did not fire)")
    sys.exit(0)


def race_probe(reps=5):
    import numpy as np

    import locc_synth as ls
    from paper_2304_09439_b200 import locc
    pts, _ = ls.make_shapes(40, 1500, seed=92)
    pairs, poses = ls.make_pairs_poses(pts, 20000, s=0.5, seed=93)
    with locc.Locc(precision=locc.LOCC_PREC_BF16, device=0) as ctx:
        ctx.load_weights_mem(ls.weight_set("spread_bias"))
        ctx.set_shapes(pts)
        ctx.load_unet_weights_mem(ls.flatten_unet(ls.make_unet_weights("he")))
        ctx.encode_shapes()
        for det in (False, True):
            ctx.set_deterministic(det)
            ref = ctx.query(pairs, poses)
            refg = ctx.query_grad(pairs, poses)
            for _ in range(reps):
                got = ctx.query(pairs, poses)
                gg = ctx.query_grad(pairs, poses)
                assert all(np.array_equal(a, b) for a, b in zip(got, ref)), f"query differs run to run (det={det})"
                assert all(np.array_equal(a, b) for a, b in zip(gg, refg)), f"grad differs run to run (det={det})"
        ctx.set_deterministic(False)
        refc = ctx.query_cells(pairs, poses)
        for _ in range(reps):
            c = ctx.query_cells(pairs, poses)
            assert all(np.array_equal(c[k], refc[k]) for k in refc), "encode-once query differs run to run"
    print(f"race probe: {len(pairs)} pairs x {reps} repeats, both walk modes, grad and encode-once: bitwise equal")


def main():
    from paper_2304_09439_b200 import build
    build.build(out=LIB, flags=("-DLOCC_CHECKED=1",))
    env = dict(os.environ, LOCC_LIB=LIB)
    r = subprocess.run([sys.executable, __file__, "--selftest-child"], env=dict(env, LOCC_CHECK_SELFTEST="1"),
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    fired = r.returncode == 3 and "LOCC_CHECK failed" in out
    print("selftest:", "check fired" if fired else "CHECK DID NOT FIRE", f"(rc {r.returncode})")
    print("\n".join(ln for ln in out.splitlines() if "LOCC_CHECK" in ln or "selftest" in ln)[:2000])
    if not fired:
        sys.exit(1)
    r = subprocess.run([sys.executable, __file__, "--race-probe"], env=env, timeout=1200)
    if r.returncode:
        sys.exit(r.returncode)
    args = sys.argv[1:] or ["-x", "-q"]
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests"), "-m", "gpu"] + args,
                       env=env, cwd=ROOT)
    sys.exit(r.returncode)


if __name__ == "__main__":
    if "--selftest-child" in sys.argv:
        selftest_child()
    elif "--race-probe" in sys.argv:
        race_probe()
    else:
        main()
