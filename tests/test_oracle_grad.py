"""Pins of the oracle's pose gradient (NEXT-2): d logit / d [q_A, t_A, q_B, t_B]
at fixed crops.  Pinned against central finite differences of the forward logit (which is itself
pinned to the query's logit), a closed form on a hand-built head, and exact invariances — never
against a retyped backward."""
import numpy as np

import locc_synth as ls
from test_oracle_network import canon, head_weights, spread

H, F = 256, 64


def rand_case(seed):
    rng = np.random.default_rng(seed)
    eA, eB = rng.normal(0, 1, F), rng.normal(0, 1, F)
    pa = np.concatenate([rng.normal(0, 1, 4), rng.normal(0, 0.5, 3)])
    pb = np.concatenate([rng.normal(0, 1, 4), rng.normal(0, 0.5, 3)])
    return eA, eB, pa, pb


def fd_grad(oracle_mod, w, eA, eB, pa, pb, h=1e-6):
    g = np.zeros(14)
    for j in range(14):
        for sgn in (1, -1):
            a, b = pa.copy(), pb.copy()
            (a if j < 7 else b)[j % 7] += sgn * h
            g[j] += sgn * oracle_mod.head_grad(w, eA, eB, a, b)[0]
    return g / (2 * h)


def test_head_logit_matches_query(oracle_mod):
    """The gradient's forward is the query's predictor: same logit from the query's embeddings."""
    pts, _ = ls.make_shapes(6, 300, seed=40)
    pairs, poses = ls.make_pairs_poses(pts, 24, s=0.5, seed=41)
    w = spread()
    r = oracle_mod.query(w, pts, pairs, poses)
    lg, _, _ = oracle_mod.query_grad(w, pts, pairs, poses)
    n = 0
    for i in range(len(pairs)):
        if r["kept"][i].sum() == 0:
            continue
        l1, _ = oracle_mod.head_grad(w, r["emb"][i, 0], r["emb"][i, 1], poses[i, 0].astype(np.float64),
                                     poses[i, 1].astype(np.float64))
        assert abs(l1 - r["logits"][i]) <= 1e-12 * max(1.0, abs(l1))
        assert lg[i] == r["logits"][i]
        n += 1
    assert n > 10


def test_grad_matches_finite_differences(oracle_mod):
    """Central differences (h = 1e-6) on the fp64 forward; the network is piecewise linear in z, so
    away from ReLU kinks the only truncation error is the quaternion normalisation's (O(h^2))."""
    w = spread()
    for seed in range(8):
        eA, eB, pa, pb = rand_case(100 + seed)
        _, g = oracle_mod.head_grad(w, eA, eB, pa, pb)
        fd = fd_grad(oracle_mod, w, eA, eB, pa, pb)
        scale = max(1e-3, np.abs(g).max())
        assert np.abs(g - fd).max() <= 1e-6 * scale, (seed, g, fd)
        assert np.abs(g).max() > 0


def test_grad_closed_form(oracle_mod):
    """head_weights(): logit = max(tx_A, tx_B) + 2 max(e0_A, e0_B) + 3 max(qcx_A, qcx_B), so
    d/dt_x of the larger-tx side is 1 (other side 0, y/z 0), and d/dq of the larger-qcx side is
    3 d(qc_x)/dq = 3 s (e_x - qc qc_x) / |q| with s the canonical sign."""
    w = head_weights()
    rng = np.random.default_rng(42)
    for _ in range(10):
        eA, eB = rng.normal(0, 0.3, F), rng.normal(0, 0.3, F)
        pa = np.concatenate([rng.normal(0, 1, 4), rng.normal(0, 0.5, 3)])
        pb = np.concatenate([rng.normal(0, 1, 4), rng.normal(0, 0.5, 3)])
        # the probe encoder's e is ignored here: head_weights' obj.l1 reads e0 from z directly
        _, g = oracle_mod.head_grad(w, eA, eB, pa, pb)
        want = np.zeros(14)
        want[4 if pa[4] > pb[4] else 11] = 1.0
        ca, cb = canon(pa[:4]), canon(pb[:4])
        side, q, c = (0, pa[:4], ca) if ca[1] > cb[1] else (7, pb[:4], cb)
        s = np.sign(q[np.nonzero(q)[0][0]])
        ex = np.array([0.0, 1.0, 0.0, 0.0])
        want[side:side + 4] = 3 * s * (ex - c * c[1]) / np.linalg.norm(q)
        np.testing.assert_allclose(g, want, rtol=0, atol=1e-12)


def test_grad_invariances(oracle_mod):
    """Exact symmetries of the logit: scale invariance in q (q . dq = 0), q -> -q (dq -> -dq,
    dt unchanged), and swapping the objects (gradient halves swap)."""
    w = spread()
    for seed in range(6):
        eA, eB, pa, pb = rand_case(200 + seed)
        _, g = oracle_mod.head_grad(w, eA, eB, pa, pb)
        for side, p in ((0, pa), (7, pb)):
            assert abs(np.dot(p[:4], g[side:side + 4])) <= 1e-12 * max(1.0, np.abs(g).max())
        na = pa.copy()
        na[:4] *= -1
        _, gn = oracle_mod.head_grad(w, eA, eB, na, pb)
        np.testing.assert_allclose(gn[:4], -g[:4], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(gn[4:], g[4:], rtol=1e-12, atol=1e-15)
        _, gs = oracle_mod.head_grad(w, eB, eA, pb, pa)
        np.testing.assert_allclose(gs, np.concatenate([g[7:], g[:7]]), rtol=1e-12, atol=1e-15)


def test_query_grad_short_circuit_and_per_pair(oracle_mod):
    pts, _ = ls.make_shapes(6, 300, seed=43)
    pairs, poses = ls.make_pairs_poses(pts, 30, s=0.6, seed=44)
    w = spread()
    r = oracle_mod.query(w, pts, pairs, poses)
    lg, g, mg = oracle_mod.query_grad(w, pts, pairs, poses)
    sc = r["kept"].sum(1) == 0
    assert sc.any() and (~sc).any()
    assert np.all(g[sc] == 0) and np.all(np.isneginf(lg[sc])) and np.all(np.isinf(mg[sc]))
    assert np.all(mg[~sc] >= 0) and np.all(np.isfinite(mg[~sc]))
    for i in np.nonzero(~sc)[0]:
        _, gi = oracle_mod.head_grad(w, r["emb"][i, 0], r["emb"][i, 1], poses[i, 0].astype(np.float64),
                                     poses[i, 1].astype(np.float64))
        assert np.array_equal(gi, g[i])
