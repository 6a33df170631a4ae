"""Exact-arithmetic pins of the whole network (SURVEY.md §8(c) "Dyadic exact nets", the bias probe).

* Dyadic exact net: every weight and bias a small dyadic number (k/2, k/4, ...), rows with a few
  non-zeros, coordinates k/2 (the W1 cube, PAPER-independent worked example W1), crops chosen so
  every occupied-cell count C_s is 1, 2 or 4 (the mean's 1/C is exact).  Then every intermediate of
  O6-O9 is exactly representable in bf16 (h1, h2, W2, W3), tf32 (predictor operands) and fp32, so the
  fp64 oracle, the bf16-emulating oracle, the fp32 GPU path and the bf16 tensor-core GPU path (with
  its 3xTF32 predictor) must agree BITWISE on e and on the logit; p = sigmoid(logit) within 2 ulp
  (the GPU's fp32 exp against fp64).
* Bias probe (tests/test_oracle_pins.py encoder_bias_probe): W2 = 0, W3 = a permutation, dyadic b2,
  b3, W_F, b_F: e = W_F ReLU(ReLU(b2) + b3) + b_F bitwise on every non-empty side, through the bf16
  path's 3-term b2 bias MMA and its b3 handling and through the fp32 path.
* Full-precision b2: b2 with a full 24-bit mantissa; the bf16 path rounds h2 = ReLU(b2) to bf16, so
  e is bitwise the bf16-emulating oracle's (the 3-term split must reproduce b2 exactly); the fp32
  path adds b3 and sums the cells in fp32, so e is within a few ulps of the fp64 oracle.
"""
import itertools

import numpy as np
import pytest

import locc_synth as ls
from conftest import cube26, pose
from test_oracle_pins import encoder_bias_probe

H, F, P = 256, 64, 128


def _sparse(rng, o, i, nnz, vals):
    W = np.zeros((o, i), np.float32)
    for r in range(o):
        cols = rng.choice(i, size=nnz, replace=False)
        W[r, cols] = rng.choice(vals, size=nnz)
    return W


def dyadic_net(seed=90):
    """Small dyadic weights: W1 entries k/2 (|k| <= 4), hidden rows with 2-3 non-zeros in
    {+-1/2, +-1}, biases multiples of 1/8 in [-1/2, 1/2], out.W entries +-1/16.  With coordinates in
    {0, +-1/2} every h1 is a multiple of 1/4 below 4 in magnitude and every h2 a multiple of 1/8 below
    16: bf16-exact (8 significant bits)."""
    rng = np.random.default_rng(seed)
    w = ls.make_weights("zero", H, F)
    w["enc.l1.W"] = (rng.integers(-4, 5, (H, 3)) / 2).astype(np.float32)
    bias = lambda n: (rng.integers(-4, 5, n) / 8).astype(np.float32)
    w["enc.l1.b"] = bias(H)
    w["enc.l2.W"] = _sparse(rng, H, H, 2, [-0.5, 0.5, -1.0, 1.0])
    w["enc.l2.b"] = bias(H)
    w["enc.l3.W"] = _sparse(rng, H, H, 3, [-0.5, 0.5, -1.0, 1.0])
    w["enc.l3.b"] = bias(H)
    w["enc.proj.W"] = _sparse(rng, F, H, 3, [-0.5, 0.5, 1.0])
    w["enc.proj.b"] = bias(F)
    w["obj.l1.W"] = _sparse(rng, P, F + 7, 3, [-0.5, 0.5, 1.0])
    w["obj.l1.b"] = bias(P)
    for name in ("obj.l2", "obj.l3", "pair.l1", "pair.l2", "pair.l3"):
        w[name + ".W"] = _sparse(rng, P, P, 2, [-0.5, 0.5, 1.0])
        w[name + ".b"] = bias(P)
    w["out.W"] = (rng.choice([-1.0, 1.0], (1, P)) / 16).astype(np.float32)
    w["out.b"] = np.array([-45 / 64], np.float32)  # centres the logits of dyadic_cases() on 0
    return w


def dyadic_cases():
    """cube26 against itself under identity / 180-degree / 120-degree rotations and dyadic offsets,
    every case with C_A, C_B in {1, 2, 4} (found by enumeration; the test re-checks the counts)."""
    vals = [0.375, 0.625, 0.75, 1.0, 1.125]
    qs = [(1, 0, 0, 0), (0, 0, 0, 1), (0, 1, 0, 0), (0.5, 0.5, 0.5, 0.5)]
    P_ = [np.stack([pose(), pose(q, t)]) for q in qs for t in itertools.product(vals, vals, vals)]
    # the W1 "separated" row too: both crops empty -> short-circuit
    P_.append(np.stack([pose(), pose(t=(2.0, 0.0, 0.0))]))
    poses = np.array(P_, np.float32)
    return np.stack([cube26()] * 2), np.tile(np.array([[0, 1]], np.int32), (len(poses), 1)), poses


@pytest.fixture(scope="module")
def dyadic(oracle_mod):
    pts, pairs, poses = dyadic_cases()
    flat = ls.flatten_weights(dyadic_net())
    ref = oracle_mod.query(flat, pts, pairs, poses)
    keep = np.isin(ref["occ"], [1, 2, 4]).all(1) | (ref["kept"].sum(1) == 0)
    pairs, poses = pairs[keep], poses[keep]
    ref = oracle_mod.query(flat, pts, pairs, poses)
    return flat, pts, pairs, poses, ref


def test_dyadic_net_is_exact_in_the_oracle(oracle_mod, dyadic):
    """The pin's premise: bf16 emulation changes nothing on this net (bitwise), the ReLUs and the
    pair max are exercised (mixed signs before every ReLU), and the logits are not saturated."""
    flat, pts, pairs, poses, ref = dyadic
    r1 = oracle_mod.query(flat, pts, pairs, poses, bf16_emul=True)
    assert np.array_equal(ref["emb"], r1["emb"]) and np.array_equal(ref["logits"], r1["logits"])
    ev = np.isfinite(ref["logits"])
    assert ev.sum() >= 300 and (~ev).sum() >= 1
    lg = ref["logits"][ev]
    assert np.unique(lg).size > 20 and np.abs(lg).max() < 8
    assert 0.1 < (ref["labels"][ev] == 1).mean() < 0.9
    e = ref["emb"][ev]
    assert (e > 0).any() and (e < 0).any()


@pytest.fixture(scope="module")
def locc_mod():
    from paper_2304_09439_b200 import build as b
    b.build()
    from paper_2304_09439_b200 import locc
    return locc


def _ctx(locc_mod, flat, pts, precision):
    ctx = locc_mod.Locc(M=6, H=H, F=F, precision=precision, device=0)
    ctx.load_weights_mem(flat)
    ctx.set_shapes(pts)
    return ctx


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [0, 1])
def test_dyadic_net_bitwise_gpu(locc_mod, dyadic, precision):
    flat, pts, pairs, poses, ref = dyadic
    with _ctx(locc_mod, flat, pts, precision) as ctx:
        got = ctx.query_debug(pairs, poses)
    assert np.array_equal(got["kept"], ref["kept"]) and np.array_equal(got["occ"], ref["occ"])
    assert np.array_equal(got["emb"].astype(np.float64), ref["emb"]), "e differs from the exact value"
    ev = np.isfinite(ref["logits"])
    assert np.array_equal(got["logits"][ev].astype(np.float64), ref["logits"][ev]), "logit differs"
    assert np.all(np.isneginf(got["logits"][~ev])) and np.all(got["probs"][~ev] == 0)
    p = got["probs"][ev].astype(np.float64)
    assert np.all(np.abs(p - ref["probs"][ev]) <= 2 * np.spacing(np.float32(1.0)) * np.maximum(p, 1e-30) + 1e-12)
    assert np.array_equal(got["labels"], ref["labels"])


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [0, 1])
def test_encoder_bias_probe_bitwise_gpu(locc_mod, oracle_mod, precision):
    """b2 (the bf16 path's bias MMA), b3 and b_F reach e exactly: e = W_F ReLU(ReLU(b2) + b3) + b_F."""
    w, forms = encoder_bias_probe()
    pts, _ = ls.make_shapes(6, 300, seed=74)
    pairs, poses = ls.make_pairs_poses(pts, 64, s=0.5, seed=75)
    flat = ls.flatten_weights(w)
    with _ctx(locc_mod, flat, pts, precision) as ctx:
        got = ctx.query_debug(pairs, poses)
    ne = got["kept"] > 0
    assert ne.sum() > 40 and (~ne).sum() > 0
    e = np.broadcast_to(forms["as defined"], got["emb"][ne].shape)
    assert np.array_equal(got["emb"][ne].astype(np.float64), e)
    assert np.all(got["emb"][~ne] == 0)
    ref = oracle_mod.query(flat, pts, pairs, poses, bf16_emul=precision == 1)
    assert np.abs(got["probs"].astype(np.float64) - ref["probs"]).max() <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [0, 1])
def test_full_precision_b2_gpu(locc_mod, oracle_mod, precision):
    """b2 with full 24-bit mantissas (the bf16 path splits it into three bf16 terms that must sum to
    b2 exactly, then rounds h2 to bf16 like the emulating oracle): bitwise in bf16; the fp32 path's
    fp32 b2 + b3 is within 1 ulp of the fp64 oracle."""
    rng = np.random.default_rng(77)
    w, _ = encoder_bias_probe()
    b2 = rng.uniform(0.01, 0.5, H) * rng.choice([-1.0, 1.0], H)
    w["enc.l2.b"] = b2.astype(np.float32)
    assert np.mean(w["enc.l2.b"] != w["enc.l2.b"].astype(np.float64).round(6)) > 0.9  # not short decimals
    w["enc.proj.W"][:] = 0
    w["enc.proj.W"][np.arange(F), rng.choice(H, F, replace=False)] = 1.0  # e[i] = m[sel(i)] + b_F[i]
    pts, _ = ls.make_shapes(6, 300, seed=74)
    pairs, poses = ls.make_pairs_poses(pts, 64, s=0.5, seed=75)
    flat = ls.flatten_weights(w)
    ref = oracle_mod.query(flat, pts, pairs, poses, bf16_emul=precision == 1)
    with _ctx(locc_mod, flat, pts, precision) as ctx:
        got = ctx.query_debug(pairs, poses)
    ne = got["kept"] > 0
    if precision == 1:
        assert np.array_equal(got["emb"][ne].astype(np.float64), ref["emb"][ne])
    else:  # fp32 b2 + b3, then the fp32 sum of C equal cell values and / C: a few ulps
        g = got["emb"][ne]
        assert np.all(np.abs(g.astype(np.float64) - ref["emb"][ne]) <= 1e-6 * np.maximum(1.0, np.abs(ref["emb"][ne])))
