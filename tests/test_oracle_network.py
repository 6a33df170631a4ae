"""Pins of the oracle's network (O6-O9) against closed forms, textbook reductions and
exact invariants — never against a retyped copy of its own formulas."""
import json
import os

import numpy as np
from scipy.special import expit

import locc_synth as ls
from conftest import cube26, pose

GOLD = os.path.join(os.path.dirname(__file__), "golden")
H, F = 256, 64


def probe_weights(sigma, tau, b1=0.0, bF=None):
    """Identity-probe with permutations: W1 = [I3; -I3; 0], W2 = P_sigma, W3 = P_tau,
    W_F row j selects feature tau(sigma(j)).  Then e[j] = mean over occupied cells of the
    per-cell max of (x+, y+, z+, x-, y-, z-)[j] (+ b1) + bF[j] for j < 6, else bF[j]."""
    w = ls.make_weights("zero", H, F)
    for i in range(3):
        w["enc.l1.W"][i, i] = 1.0
        w["enc.l1.W"][3 + i, i] = -1.0
    w["enc.l1.b"][:6] = b1
    w["enc.l2.W"][sigma, np.arange(H)] = 1.0  # h2[sigma(i)] = h1[i]
    w["enc.l3.W"][tau, np.arange(H)] = 1.0    # h3[tau(k)] = h2[k]
    for j in range(6):
        w["enc.proj.W"][j, tau[sigma[j]]] = 1.0
    if bF is not None:
        w["enc.proj.b"][:] = bF
    return w


def perms(seed=0):
    rng = np.random.default_rng(seed)
    s, t = rng.permutation(H), rng.permutation(H)
    assert not np.array_equal(s[s], np.arange(H))  # not an involution: a transpose would show
    return s, t


def test_identity_probe_worked_example(oracle_mod):
    g = json.load(open(os.path.join(GOLD, "w1_boxes.json")))
    row = g["rows"][g["identity_probe_row"]]
    c = cube26()
    s, t = perms()
    bF = np.arange(F) * 0.25
    # b1 = 1: the 9 kept points have x = 1/2 and y, z in {-1/2, 0, 1/2} (three each), so
    # (x+1, y+1, z+1, 1-x, 1-y, 1-z) averages to (3/2, 1, 1, 1/2, 1, 1) over the 9 cells.
    for b1, want in ((0.0, np.array(g["identity_probe_eA_first6"])), (1.0, np.array([1.5, 1, 1, 0.5, 1, 1]))):
        w = ls.flatten_weights(probe_weights(s, t, b1=b1, bF=bF))
        r = oracle_mod.query(w, np.stack([c, c]), np.array([[0, 1]], np.int32),
                             np.stack([pose(), pose(row["qB"], row["tB"])])[None], n_threads=1)
        np.testing.assert_array_equal(r["emb"][0, 0, :6], want + bF[:6])
        np.testing.assert_array_equal(r["emb"][0, 0, 6:], bF[6:])


def test_identity_probe_groupby(oracle_mod):
    """e[0:6] == textbook group-by (np.maximum.at per cell, then mean over occupied cells)."""
    pts, _ = ls.make_shapes(10, 400, seed=21)
    pairs, poses = ls.make_pairs_poses(pts, 40, s=0.5, seed=22)
    s, t = perms(1)
    w = ls.flatten_weights(probe_weights(s, t))
    r = oracle_mod.query(w, pts, pairs, poses)
    K = pts.shape[1]
    checked = 0
    for i in range(len(pairs)):
        for side in range(2):
            shp = pairs[i, side]
            keep = np.array([(r["masks"][i, side, k // 32] >> (k % 32)) & 1 for k in range(K)], bool)
            if r["kept"][i].sum() == 0:
                continue
            if not keep.any():
                assert np.all(r["emb"][i, side] == 0) and r["occ"][i, side] == 0
                continue
            _, _, _, cell = oracle_mod.shape_prep(pts[shp])
            p = pts[shp][keep].astype(np.float64)
            feats = np.concatenate([np.maximum(p, 0), np.maximum(-p, 0)], 1)
            g = np.full((216, 6), -np.inf)
            np.maximum.at(g, cell[keep], feats)
            occ = np.isfinite(g[:, 0])
            assert r["occ"][i, side] == occ.sum()
            np.testing.assert_allclose(r["emb"][i, side, :6], g[occ].mean(0), rtol=0, atol=1e-15)
            checked += 1
    assert checked > 20


def head_weights():
    """Encoder = identity probe; obj.l1 unit0 = tx+10, unit1 = e0+10, unit2 = qhat_x+10;
    obj.l2/l3 and pair.l1-3 identity; out = u0 + 2 u1 + 3 u2 - 60.  Closed form:
    logit = max(tx_A, tx_B) + 2 max(e0_A, e0_B) + 3 max(qcx_A, qcx_B)."""
    s, t = perms(2)
    w = probe_weights(s, t)
    W = w["obj.l1.W"]
    W[0, F + 4] = 1.0
    W[1, 0] = 1.0
    W[2, F + 1] = 1.0
    w["obj.l1.b"][:3] = 10.0
    for name in ("obj.l2", "obj.l3", "pair.l1", "pair.l2", "pair.l3"):
        w[name + ".W"][:] = np.eye(128, dtype=np.float32)
    w["out.W"][0, :3] = [1.0, 2.0, 3.0]
    w["out.b"][0] = -60.0
    return ls.flatten_weights(w)


def canon(q):
    q = q.astype(np.float64) / np.linalg.norm(q.astype(np.float64))
    nz = q[np.nonzero(q)[0][0]]
    return q * np.sign(nz)


def test_head_closed_form(oracle_mod):
    pts, _ = ls.make_shapes(8, 400, seed=23)
    pairs, poses = ls.make_pairs_poses(pts, 60, s=0.4, seed=24)
    r = oracle_mod.query(head_weights(), pts, pairs, poses)
    ev = 0
    for i in range(len(pairs)):
        if r["kept"][i].sum() == 0:
            assert r["logits"][i] == -np.inf and r["probs"][i] == 0
            continue
        tx = max(poses[i, 0, 4], poses[i, 1, 4])
        e0 = max(r["emb"][i, 0, 0], r["emb"][i, 1, 0])
        qx = max(canon(poses[i, 0, :4])[1], canon(poses[i, 1, :4])[1])
        want = float(tx) + 2 * e0 + 3 * qx
        assert abs(r["logits"][i] - want) < 1e-12
        assert abs(r["probs"][i] - expit(want)) < 1e-12
        assert 0 < r["probs"][i] < 1 and r["labels"][i] == (r["probs"][i] > 0.5)
        ev += 1
    assert ev > 30


def test_quaternion_canonical_sign_w_zero(oracle_mod):
    """w = 0: the first non-zero component decides the sign, so q and -q agree exactly."""
    c = cube26()
    pts = np.stack([c, c])
    w = head_weights()
    for q in [(0, -1, 0, 0), (0, 0, -1, 0), (0, 0, 0, -1), (0, -0.6, 0.8, 0)]:
        pa = pose(q, (0.5, 0, 0))
        pb = pose(t=(0, 0, 0))
        r1 = oracle_mod.query(w, pts, np.array([[0, 1]], np.int32), np.stack([pa, pb])[None], n_threads=1)
        pa2 = pa.copy()
        pa2[:4] = -pa2[:4]
        r2 = oracle_mod.query(w, pts, np.array([[0, 1]], np.int32), np.stack([pa2, pb])[None], n_threads=1)
        assert r1["logits"][0] == r2["logits"][0]


def spread():
    return ls.flatten_weights(ls.make_weights("spread", H, F, calib=ls.load_calibration()))


def test_point_order_invariance(oracle_mod):
    """permuting a cloud's points leaves e, C, n and the output bitwise unchanged."""
    pts, _ = ls.make_shapes(6, 300, seed=25)
    pairs, poses = ls.make_pairs_poses(pts, 12, s=0.5, seed=26)
    w = spread()
    r0 = oracle_mod.query(w, pts, pairs, poses)
    rng = np.random.default_rng(27)
    perm = np.stack([rng.permutation(300) for _ in range(6)])
    pts2 = np.take_along_axis(pts, perm[:, :, None], 1)
    r1 = oracle_mod.query(w, pts2, pairs, poses)
    for k in ("probs", "logits", "kept", "occ", "emb", "labels"):
        assert np.array_equal(r0[k], r1[k]), k


def test_swap_and_sign_invariance(oracle_mod):
    """swapping the two objects changes nothing (max across the pair is symmetric);
    q -> -q on any pose changes nothing (the crop uses R(q) = R(-q); the head canonicalises)."""
    pts, _ = ls.make_shapes(6, 300, seed=28)
    pairs, poses = ls.make_pairs_poses(pts, 16, s=0.5, seed=29)
    w = spread()
    r0 = oracle_mod.query(w, pts, pairs, poses)
    r1 = oracle_mod.query(w, pts, pairs[:, ::-1].copy(), poses[:, ::-1].copy())
    assert np.array_equal(r0["logits"], r1["logits"]) and np.array_equal(r0["probs"], r1["probs"])
    assert np.array_equal(r0["kept"], r1["kept"][:, ::-1]) and np.array_equal(r0["emb"], r1["emb"][:, ::-1])
    neg = poses.copy()
    neg[:, :, :4] *= -1
    r2 = oracle_mod.query(w, pts, pairs, neg)
    for k in ("logits", "kept", "occ", "emb", "masks"):
        assert np.array_equal(r0[k], r2[k]), k


def test_batch_composition_invariance(oracle_mod):
    pts, _ = ls.make_shapes(6, 300, seed=30)
    pairs, poses = ls.make_pairs_poses(pts, 20, s=0.5, seed=31)
    w = spread()
    r = oracle_mod.query(w, pts, pairs, poses, n_threads=3)
    for i in (0, 7, 19):
        ri = oracle_mod.query(w, pts, pairs[i:i + 1], poses[i:i + 1], n_threads=1)
        assert ri["logits"][0] == r["logits"][i] or (np.isinf(ri["logits"][0]) and np.isinf(r["logits"][i]))
        assert np.array_equal(ri["emb"][0], r["emb"][i])


def test_bf16_emulation_exact_on_dyadic_net(oracle_mod):
    """Dyadic weights (k/4, |k| <= 8) and dyadic coordinates (k/8): every operand of layers 2-3
    is already a bf16 value, so bf16 emulation must change nothing (bitwise)."""
    rng = np.random.default_rng(32)
    c = cube26()
    w = ls.make_weights("zero", H, F)
    for name in ("enc.l1.W", "enc.l2.W", "enc.l3.W"):
        sh = w[name].shape
        w[name] = (rng.integers(-8, 9, sh) / 4 * (rng.random(sh) < (0.5 if name == "enc.l1.W" else 0.02))).astype(np.float32)
    w["enc.l2.W"] /= 4
    w["enc.l3.W"] /= 4
    w["enc.proj.W"] = (rng.integers(-4, 5, w["enc.proj.W"].shape) / 8).astype(np.float32)
    flat = ls.flatten_weights(w)
    P = np.stack([pose(), pose(t=(1, 0, 0)), pose(t=(0.5, 0.5, 0)), pose()])
    pts = np.stack([c, c * 0.5])
    pairs = np.array([[0, 0], [0, 1]], np.int32)
    poses = np.stack([P[:2], P[2:]])
    r0 = oracle_mod.query(flat, pts, pairs, poses, bf16_emul=False)
    r1 = oracle_mod.query(flat, pts, pairs, poses, bf16_emul=True)
    assert np.any(r0["emb"] != 0)
    assert np.array_equal(r0["emb"], r1["emb"]) and np.array_equal(r0["logits"], r1["logits"])


def test_bf16_emulation_is_close_not_equal(oracle_mod):
    pts, _ = ls.make_shapes(6, 400, seed=33)
    pairs, poses = ls.make_pairs_poses(pts, 16, s=0.5, seed=34)
    w = spread()
    r0 = oracle_mod.query(w, pts, pairs, poses)
    r1 = oracle_mod.query(w, pts, pairs, poses, bf16_emul=True)
    d = np.abs(r0["probs"] - r1["probs"])
    assert d.max() > 0 and d.max() < 2e-2
    assert np.array_equal(r0["kept"], r1["kept"])


def test_weight_file_roundtrip(oracle_mod, tmp_path):
    w = ls.make_weights("he")
    path = ls.write_weights(str(tmp_path / "w.txt"), w)
    flat, (M, Hh, Ff) = oracle_mod.load_weights(path)
    assert (M, Hh, Ff) == (6, H, F)
    assert np.array_equal(flat, ls.flatten_weights(w)) and flat.size == oracle_mod.n_params(H, F) == 240961
    txt = open(path).read().replace("enc.l2.W", "enc.l9.W")
    open(path, "w").write(txt)
    try:
        oracle_mod.load_weights(path)
        raise AssertionError("bad manifest accepted")
    except ValueError:
        pass
