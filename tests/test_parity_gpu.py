"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star):
  * crop masks, kept counts n_s, occupied-cell counts C_s: bit-exact;
  * fp32 path: |p - p_oracle| <= 1e-5; labels identical except where |p_oracle - 0.5| <= 1e-3;
  * bf16 path: |p - p_oracle_bf16emul| <= 5e-4 with identical labels outside the 1e-3 band, and
    |p - p_oracle_fp64| <= 2e-2 (reading Q18).
"""
import json
import os

import numpy as np
import pytest

import locc_synth as ls
from conftest import cube26, pose

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
P_TOL = {0: 1e-5, 1: 5e-4}


@pytest.fixture(scope="module")
def locc_mod():
    from paper_2304_09439_b200 import build as b
    b.build()
    from paper_2304_09439_b200 import locc
    return locc


@pytest.fixture(scope="module", params=ls.WEIGHT_SETS)
def wflat(request):
    """Every parity suite runs over both calibrated sets: `spread` (zero hidden biases) and
    `spread_bias` (every bias non-zero: b1, the bf16 b2 bias MMA, the b3 fold, the projection and
    predictor biases)."""
    return ls.weight_set(request.param)


@pytest.fixture(scope="module")
def c1():
    return ls.make_workload("C1")


@pytest.fixture(scope="module")
def c1_oracle(oracle_mod, c1, wflat):
    return {emul: oracle_mod.query(wflat, c1.points, c1.pairs, c1.poses, bf16_emul=emul) for emul in (False, True)}


def make_ctx(locc_mod, flat, points, precision, M=6, H=256, F=64, max_batch=0):
    ctx = locc_mod.Locc(M=M, H=H, F=F, precision=precision, device=0, max_batch=max_batch)
    ctx.load_weights_mem(flat)
    ctx.set_shapes(points)
    return ctx


def assert_parity(got, ref, precision, ref64=None):
    assert np.array_equal(got["kept"], ref["kept"]), "kept counts differ"
    assert np.array_equal(got["masks"], ref["masks"]), "crop masks differ"
    assert np.array_equal(got["occ"], ref["occ"]), "occupied-cell counts differ"
    short = ref["kept"].sum(1) == 0
    assert np.all(got["probs"][short] == 0) and np.all(got["labels"][short] == 0)
    assert np.all(np.isneginf(got["logits"][short]))
    dp = np.abs(got["probs"].astype(np.float64) - ref["probs"])
    assert dp.max() <= P_TOL[precision], f"max |dp| = {dp.max():.3g}"
    band = np.abs(ref["probs"] - 0.5) <= 1e-3
    assert np.array_equal(got["labels"][~band], ref["labels"][~band])
    if ref64 is not None:
        assert np.abs(got["probs"].astype(np.float64) - ref64["probs"]).max() <= 2e-2
    return dp.max()


# ----------------------------------------------------------------------------- C1 parity
@pytest.mark.parametrize("precision", [0, 1])
def test_c1_parity(locc_mod, c1, c1_oracle, wflat, precision):
    with make_ctx(locc_mod, wflat, c1.points, precision) as ctx:
        got = ctx.query_debug(c1.pairs, c1.poses)
    ref = c1_oracle[precision == 1]
    assert_parity(got, ref, precision, ref64=c1_oracle[False])
    ne = ref["kept"] > 0
    tol = 2e-4 if precision == 0 else 2e-2
    np.testing.assert_allclose(got["emb"][ne], ref["emb"][ne], atol=tol, rtol=tol)
    assert np.all(got["emb"][~ne] == 0)


@pytest.mark.parametrize("precision", [0, 1])
def test_c1_parity_with_ragged_subbatches_and_device_buffers(locc_mod, c1, c1_oracle, wflat, precision):
    import torch
    ref = c1_oracle[precision == 1]
    with make_ctx(locc_mod, wflat, c1.points, precision, max_batch=7) as ctx:
        got = ctx.query_debug(c1.pairs, c1.poses)
        assert_parity(got, ref, precision)
        # device-resident inputs/outputs on a caller stream: same bits as the host path
        pairs = torch.from_numpy(c1.pairs).cuda()
        poses = torch.from_numpy(c1.poses).cuda()
        probs = torch.empty(len(c1.pairs), device="cuda")
        labels = torch.empty(len(c1.pairs), dtype=torch.uint8, device="cuda")
        s = torch.cuda.Stream()
        ctx.query_into(pairs, poses, probs, labels, stream=s.cuda_stream)
        s.synchronize()
        assert np.array_equal(probs.cpu().numpy(), got["probs"])
        assert np.array_equal(labels.cpu().numpy(), got["labels"])


# ----------------------------------------------------------------------------- worked example
@pytest.mark.parametrize("precision", [0, 1])
def test_w1_worked_example_gpu(locc_mod, precision):
    g = json.load(open(os.path.join(GOLD, "w1_boxes.json")))
    c = cube26()
    zero = ls.flatten_weights(ls.make_weights("zero"))
    with make_ctx(locc_mod, zero, np.stack([c, c]), precision) as ctx:
        pairs = np.array([[0, 1]] * len(g["rows"]), np.int32)
        poses = np.stack([np.stack([pose(), pose(r["qB"], r["tB"])]) for r in g["rows"]])
        got = ctx.query_debug(pairs, poses)
    for i, row in enumerate(g["rows"]):
        assert tuple(got["kept"][i]) == (row["nA"], row["nB"])
        assert tuple(got["occ"][i]) == (row["CA"], row["CB"])
        if row["short"]:
            assert got["probs"][i] == 0 and np.isneginf(got["logits"][i])
        else:
            assert got["probs"][i] == 0.5 and got["labels"][i] == 0 and got["logits"][i] == 0


def test_identity_probe_gpu(locc_mod):
    """Closed form (W1 row 2): e_A[0:6] = (1/2, 1/6, 1/6, 0, 1/6, 1/6) through both encoders; with
    dyadic operands the bf16 tensor-core path is exact up to the final /C."""
    from test_oracle_network import perms, probe_weights
    g = json.load(open(os.path.join(GOLD, "w1_boxes.json")))
    row = g["rows"][g["identity_probe_row"]]
    c = cube26()
    s, t = perms()
    w = ls.flatten_weights(probe_weights(s, t))
    for precision in (0, 1):
        with make_ctx(locc_mod, w, np.stack([c, c]), precision) as ctx:
            got = ctx.query_debug(np.array([[0, 1]], np.int32), np.stack([pose(), pose(row["qB"], row["tB"])])[None])
        np.testing.assert_allclose(got["emb"][0, 0, :6], g["identity_probe_eA_first6"], atol=1e-7)
        assert np.all(got["emb"][0, 0, 6:] == 0)


# ----------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("K,M,s", [(1, 6, 0.5), (77, 6, 0.3), (300, 1, 0.5), (300, 7, 0.25), (2000, 5, 0.1)])
def test_edge_shapes(locc_mod, oracle_mod, wflat, precision, K, M, s):
    pts, _ = ls.make_shapes(5, K, seed=40 + K)
    pairs, poses = ls.make_pairs_poses(pts, 24, s=s, seed=41)
    pairs[0] = [2, 2]  # self pair
    poses[1, 1] = poses[1, 0]  # coincident poses: everything kept
    ref = oracle_mod.query(wflat, pts, pairs, poses, M=M, bf16_emul=precision == 1)
    with make_ctx(locc_mod, wflat, pts, precision, M=M) as ctx:
        got = ctx.query_debug(pairs, poses)
    assert_parity(got, ref, precision)


@pytest.mark.parametrize("precision", [0, 1])
def test_all_short_circuit_and_empty(locc_mod, wflat, precision):
    pts, _ = ls.make_shapes(3, 200, seed=50)
    with make_ctx(locc_mod, wflat, pts, precision) as ctx:
        poses = np.stack([np.stack([pose(), pose(t=(5.0 + i, 0, 0))]) for i in range(10)])
        pr, lb, lg = ctx.query(np.zeros((10, 2), np.int32), poses)
        assert np.all(pr == 0) and np.all(lb == 0) and np.all(np.isneginf(lg))
        pr, lb, lg = ctx.query(np.zeros((0, 2), np.int32), np.zeros((0, 2, 7), np.float32))
        assert pr.size == 0


def test_invalid_inputs_fail_loudly(locc_mod, wflat):
    pts, _ = ls.make_shapes(3, 100, seed=51)
    with make_ctx(locc_mod, wflat, pts, 0) as ctx:
        ok = np.stack([pose(), pose()])[None]
        with pytest.raises(locc_mod.LoccError):
            ctx.query(np.array([[0, 3]], np.int32), ok)
        bad = ok.copy()
        bad[0, 1, :4] = 0
        with pytest.raises(locc_mod.LoccError):
            ctx.query(np.array([[0, 1]], np.int32), bad)
        bad = ok.copy()
        bad[0, 0, 5] = np.nan
        with pytest.raises(locc_mod.LoccError):
            ctx.query(np.array([[0, 1]], np.int32), bad)
    with pytest.raises(locc_mod.LoccError):
        locc_mod.Locc(M=0)
    ctx = locc_mod.Locc(precision=0, device=0)
    with pytest.raises(locc_mod.LoccError):  # no weights / shapes yet
        ctx.query(np.array([[0, 0]], np.int32), ok)
    with pytest.raises(locc_mod.LoccError):
        ctx.load_weights_mem(wflat[:-1])
    with pytest.raises(locc_mod.LoccError):
        ctx.set_shapes(np.full((2, 10, 3), np.nan, np.float32))
    ctx.close()


def test_weight_file_path(locc_mod, c1, wflat, tmp_path):
    kind = "spread_bias" if np.array_equal(wflat, ls.weight_set("spread_bias")) else "spread"
    w = ls.make_weights(kind, calib=ls.load_calibration(kind=kind))
    path = ls.write_weights(str(tmp_path / "w.txt"), w)
    with make_ctx(locc_mod, wflat, c1.points, 0) as a, locc_mod.Locc(precision=0, device=0) as b:
        b.load_weights(path)
        b.set_shapes(c1.points)
        assert np.array_equal(a.query(c1.pairs, c1.poses)[0], b.query(c1.pairs, c1.poses)[0])


# ----------------------------------------------------------------------------- invariants
def assert_invariant(a, b, precision, keys=("probs", "logits", "labels"), det=False):
    """fp32, and bf16 in its default deterministic walk: bitwise.  bf16 with the opt-in fast walk
    (locc_set_deterministic(ctx, 0)): the tensor-core layer-3 walk splits each 128-row part between two
    walkers, so the fp32 summation order of a segment's cell values depends on where the segment falls
    in its tile (reading Q24): the pooled mean moves by a few fp32 ulps (<= 1e-5 relative for
    <= 216 cells) and probabilities by <= 1e-5; labels agree away from 0.5."""
    if precision == 0 or det:
        for k in keys:
            assert np.array_equal(a[k], b[k]), k
        return
    if "probs" in keys:
        assert np.abs(a["probs"].astype(np.float64) - b["probs"]).max(initial=0) <= 1e-5
    if "logits" in keys:
        la, lb = a["logits"].astype(np.float64), b["logits"].astype(np.float64)
        fin = np.isfinite(la)
        assert np.array_equal(fin, np.isfinite(lb))
        assert np.all(np.abs(la[fin] - lb[fin]) <= 1e-4 * np.maximum(1.0, np.abs(la[fin])))
    if "labels" in keys:
        away = np.abs(a["probs"].astype(np.float64) - 0.5) > 1e-5
        assert np.array_equal(a["labels"][away], b["labels"][away])
    if "emb" in keys:
        np.testing.assert_allclose(a["emb"], b["emb"], rtol=1e-5, atol=1e-6)
    for k in ("kept", "occ", "masks"):
        if k in keys:
            assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("precision,det", [(0, False), (1, False), (1, True)])
def test_invariances(locc_mod, c1, wflat, precision, det):
    """Point order, object swap, q -> -q and batch composition leave every output unchanged: bitwise
    in fp32 and in deterministic bf16 contexts, within the walk's summation-order bound otherwise."""
    with make_ctx(locc_mod, wflat, c1.points, precision) as ctx:
        ctx.set_deterministic(det)
        base = ctx.query_debug(c1.pairs, c1.poses)
        sw = ctx.query_debug(c1.pairs[:, ::-1].copy(), c1.poses[:, ::-1].copy())
        neg = c1.poses.copy()
        neg[:, :, :4] *= -1
        ng = ctx.query_debug(c1.pairs, neg)
        one = ctx.query_debug(c1.pairs[5:6], c1.poses[5:6])
        perm = np.random.default_rng(3).permutation(len(c1.pairs))
        pm = ctx.query_debug(c1.pairs[perm], c1.poses[perm])
    assert_invariant(base, sw, precision, det=det)
    assert_invariant(base, ng, precision, det=det)
    assert_invariant({k: v[5:6] for k, v in base.items()}, one, precision, det=det)
    assert_invariant({k: v[perm] for k, v in base.items()}, pm, precision, det=det)
    assert_invariant({"emb": base["emb"]}, {"emb": sw["emb"][:, ::-1]}, precision, keys=("emb",), det=det)
    rng = np.random.default_rng(4)
    pts2 = np.stack([p[rng.permutation(p.shape[0])] for p in c1.points])
    with make_ctx(locc_mod, wflat, pts2, precision) as ctx:
        ctx.set_deterministic(det)
        pp = ctx.query_debug(c1.pairs, c1.poses)
    assert_invariant(base, pp, precision, keys=("probs", "logits", "kept", "occ", "emb"), det=det)


def test_batch_composition_bitwise_bf16(locc_mod, wflat):
    """A default bf16 context (deterministic walk) at C2 scale: every pair's outputs are bitwise the same
    alone, in a shuffled batch, in a batch tail, in ragged sub-batches (both crop buffer sets) — its
    segments land at different tile positions in each."""
    wl = ls.make_workload("C2", N=3000)
    idx = (0, 7, 1500, 2999)
    with make_ctx(locc_mod, wflat, wl.points, 1) as ctx:
        base = ctx.query(wl.pairs, wl.poses)
        perm = np.random.default_rng(5).permutation(len(wl.pairs))
        pm = ctx.query(wl.pairs[perm], wl.poses[perm])
        tail = ctx.query(wl.pairs[1234:], wl.poses[1234:])
        singles = [ctx.query(wl.pairs[i:i + 1], wl.poses[i:i + 1]) for i in idx]
    with make_ctx(locc_mod, wflat, wl.points, 1, max_batch=701) as ctx:
        sub = ctx.query(wl.pairs, wl.poses)
        assert ctx.stats()["sub_batches"] == 5
    for a, b in zip(base, sub):
        assert np.array_equal(a, b)
    for a, b in zip(base, pm):
        assert np.array_equal(a[perm], b)
    for a, b in zip(base, tail):
        assert np.array_equal(a[1234:], b)
    for i, s in zip(idx, singles):
        for a, b in zip(base, s):
            assert np.array_equal(a[i:i + 1], b)


@pytest.mark.parametrize("H,F", [(96, 64), (160, 32)])
def test_fp32_other_widths(locc_mod, oracle_mod, H, F):
    """The fp32 crop path at point-MLP widths other than 256 (the register-tiled GEMM's partial feature
    groups, point_mlp.cuh) and another F (the generic predictor) against the oracle."""
    w = ls.flatten_weights(ls.make_weights("spread", H, F, calib=ls.load_calibration()), H, F)
    wl = ls.make_workload("C1", N=40, S=8)
    ref = oracle_mod.query(w, wl.points, wl.pairs, wl.poses, H=H, F=F)
    with locc_mod.Locc(M=6, H=H, F=F, precision=0, device=0) as ctx:
        ctx.load_weights_mem(w)
        ctx.set_shapes(wl.points)
        got = ctx.query_debug(wl.pairs, wl.poses)
    assert_parity(got, ref, 0)


# ----------------------------------------------------------------------------- full sizes
@pytest.mark.parametrize("precision", [0, 1])
def test_c2_sampled_parity(locc_mod, oracle_mod, wflat, precision):
    wl = ls.make_workload("C2")
    with make_ctx(locc_mod, wflat, wl.points, precision) as ctx:
        pr, lb, lg = ctx.query(wl.pairs, wl.poses)
        st = ctx.stats()
    assert st["pairs"] == len(wl.pairs) and st["kept_rows"] > 0
    idx = np.random.default_rng(9).choice(len(wl.pairs), 96, replace=False)
    ref = oracle_mod.query(wflat, wl.points, wl.pairs[idx], wl.poses[idx], bf16_emul=precision == 1)
    assert np.abs(pr[idx] - ref["probs"]).max() <= P_TOL[precision]
    band = np.abs(ref["probs"] - 0.5) <= 1e-3
    assert np.array_equal(lb[idx][~band], ref["labels"][~band])
    ev = np.isfinite(lg)
    assert np.all((pr[ev] > 0) & (pr[ev] < 1)) and st["evaluated_pairs"] == ev.sum()


def test_c3_full_size_bf16(locc_mod, oracle_mod, wflat):
    """BASELINE config C3 (1,048,576 pairs, bf16, the bench launch configuration): sampled outputs
    against the oracle, kept = popcount(mask) everywhere, bitwise swap invariance on the whole batch and
    bitwise batch-composition invariance of the sampled pairs (the default walk is the deterministic
    one, reading Q24)."""
    import torch
    wl = ls.make_workload("C3")
    N = len(wl.pairs)
    with make_ctx(locc_mod, wflat, wl.points, 1) as ctx:
        pairs = torch.from_numpy(wl.pairs).cuda()
        poses = torch.from_numpy(wl.poses).cuda()
        probs = torch.empty(N, device="cuda")
        labels = torch.empty(N, dtype=torch.uint8, device="cuda")
        ctx.query_into(pairs, poses, probs, labels)
        probs2 = torch.empty(N, device="cuda")
        ctx.query_into(pairs.flip(1).contiguous(), poses.flip(1).contiguous(), probs2)
        assert torch.equal(probs, probs2)
        pr = probs.cpu().numpy()
        lb = labels.cpu().numpy()
        sub = np.random.default_rng(10).choice(N, 2048, replace=False)
        dbg = ctx.query_debug(wl.pairs[sub], wl.poses[sub])
    pc = np.array([[sum(bin(int(w)).count("1") for w in dbg["masks"][i, s]) for s in range(2)] for i in range(len(sub))])
    assert np.array_equal(pc, dbg["kept"])
    assert np.array_equal(dbg["probs"], pr[sub])  # batch composition
    idx = sub[:512]  # 512 pairs sampled over the whole batch (every sub-batch and encoder cluster range)
    ref = oracle_mod.query(wflat, wl.points, wl.pairs[idx], wl.poses[idx], bf16_emul=True)
    assert np.abs(pr[idx] - ref["probs"]).max() <= 5e-4
    band = np.abs(ref["probs"] - 0.5) <= 1e-3
    assert np.array_equal(lb[idx][~band], ref["labels"][~band])
    assert np.array_equal(dbg["kept"][:512], ref["kept"])


def test_tensor_core_predictor_vs_fp32_predictor(locc_mod, wflat):
    """Crop path in a bf16 context: the 3xTF32 tensor-core predictor (Q32) against the CUDA-core fp32
    predictor on the same embeddings (LOCC_HEAD_FFMA switches the kernel): |dp| <= 2e-5, labels equal
    outside the 1e-4 band, the same short-circuits."""
    wl = ls.make_workload("C1", N=2000, S=64)
    with make_ctx(locc_mod, wflat, wl.points, 1) as ctx:
        p_tc, l_tc, g_tc = ctx.query(wl.pairs, wl.poses)
        os.environ["LOCC_HEAD_FFMA"] = "1"
        try:
            p_ff, l_ff, g_ff = ctx.query(wl.pairs, wl.poses)
        finally:
            del os.environ["LOCC_HEAD_FFMA"]
    assert np.array_equal(np.isneginf(g_tc), np.isneginf(g_ff))
    assert np.abs(p_tc.astype(np.float64) - p_ff).max() <= 2e-5
    band = np.abs(p_ff - 0.5) <= 1e-4
    assert np.array_equal(l_tc[~band], l_ff[~band])


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("K", [512, 4096])
def test_k_sweep_parity(locc_mod, oracle_mod, wflat, precision, K):
    """BASELINE.json config 5's K values (512 / 4096 points per object): C1-sized batches against the
    oracle at the same bars as C1 (the full-size sweep is a bench setting, `bench.py --K`)."""
    wl = ls.make_workload("C1", N=48, K=K, S=12)
    ref = oracle_mod.query(wflat, wl.points, wl.pairs, wl.poses, bf16_emul=precision == 1)
    with make_ctx(locc_mod, wflat, wl.points, precision) as ctx:
        got = ctx.query_debug(wl.pairs, wl.poses)
    assert_parity(got, ref, precision)
    assert (ref["kept"].sum(1) > 0).mean() > 0.8


@pytest.mark.parametrize("K", [2048, 2049, 10000])
def test_large_k_parity(locc_mod, oracle_mod, wflat, K):
    """The fused crop at its largest K (kFusedMaxK = 2048: the shared-memory row lists of eight warps
    are 64 KB) and the two-pass crop (crop_count -> scan -> crop_emit) that serves K above it."""
    wl = ls.make_workload("C1", N=16, K=K, S=6)
    ref = oracle_mod.query(wflat, wl.points, wl.pairs, wl.poses, bf16_emul=True)
    with make_ctx(locc_mod, wflat, wl.points, 1) as ctx:
        got = ctx.query_debug(wl.pairs, wl.poses)
    assert_parity(got, ref, 1)


@pytest.mark.parametrize("precision", [0, 1])
def test_fused_crop_equals_two_pass(locc_mod, wflat, precision, monkeypatch):
    """crop_compact (one kernel: crop, look-back offsets, rows) against crop_count -> scan -> crop_emit
    (LOCC_CROP_2PASS, read at context creation): every output bitwise equal, over ragged sub-batches
    (the overlapped crop pipeline's two buffer sets) and with the debug outputs (masks, C_s)."""
    wl = ls.make_workload("C2", N=6000)
    outs = []
    for two_pass in (False, True):
        if two_pass:
            monkeypatch.setenv("LOCC_CROP_2PASS", "1")
        with make_ctx(locc_mod, wflat, wl.points, precision, max_batch=1500) as ctx:
            q = ctx.query(wl.pairs, wl.poses)
            assert ctx.stats()["sub_batches"] == 4
            d = ctx.query_debug(wl.pairs[:700], wl.poses[:700])
        outs.append((q, d))
        monkeypatch.delenv("LOCC_CROP_2PASS", raising=False)
    (q0, d0), (q1, d1) = outs
    for a, b in zip(q0, q1):
        assert np.array_equal(a, b)
    for k in d0:
        assert np.array_equal(d0[k], d1[k]), k


def test_c3_sharded_equals_unsharded_bf16(locc_mod, wflat):
    """pairs are independent, so the C3 batch split into 8 contiguous shards of
    ceil(N/8) pairs (each a separate query, as the 8 ranks of a multi-GPU run compute them) gives
    BITWISE the probabilities, labels and logits of the single 1,048,576-pair query — in a
    deterministic context (locc_set_deterministic), the bf16 path's bitwise mode; swapping the objects
    of every pair is bitwise invariant there too."""
    import torch
    from paper_2304_09439_b200.parallel import shard_bounds
    wl = ls.make_workload("C3")
    N = len(wl.pairs)
    with make_ctx(locc_mod, wflat, wl.points, 1) as ctx:
        ctx.set_deterministic(True)
        pairs = torch.from_numpy(wl.pairs).cuda()
        poses = torch.from_numpy(wl.poses).cuda()
        out = [torch.empty(N, device="cuda"), torch.empty(N, dtype=torch.uint8, device="cuda"),
               torch.empty(N, device="cuda")]
        ctx.query_into(pairs, poses, *out)
        sh = [torch.full((N,), 7.0, device="cuda"), torch.full((N,), 7, dtype=torch.uint8, device="cuda"),
              torch.full((N,), 7.0, device="cuda")]
        for r in range(8):
            lo, hi = shard_bounds(N, 8, r)
            ctx.query_into(pairs[lo:hi], poses[lo:hi], *(t[lo:hi] for t in sh))
        for a, b in zip(out, sh):
            assert torch.equal(a, b)
        swapped = torch.empty(N, device="cuda")
        ctx.query_into(pairs.flip(1).contiguous(), poses.flip(1).contiguous(), swapped)
        assert torch.equal(out[0], swapped)
