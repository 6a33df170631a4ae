"""GPU parity of the encode-once mode (NEXT-1: locc_load_unet_weights_mem, locc_encode_shapes,
locc_query_cells) against the oracle (oracle_query_cells / oracle_encode_grid).

Bars (Q27-Q30): selected-cell bits and counts bit-exact (both sides take the decision with
the same fp32 arithmetic on the same fp32 cell centres); embedding grids within 2e-5 of max|E| (fp32
sums of up to 6912 terms against fp64); pooled e within 2e-5; |p - p_oracle| <= 1e-5 and labels
identical outside |p_oracle - 0.5| <= 1e-3; short-circuit exactly where neither side selects a cell.
"""
import numpy as np
import pytest

import locc_synth as ls
from test_oracle_cells import identity_encoder, unet_probe

pytestmark = pytest.mark.gpu
E_TOL = 2e-5


@pytest.fixture(scope="module")
def locc_mod():
    from paper_2304_09439_b200 import build as b
    b.build()
    from paper_2304_09439_b200 import locc
    return locc


@pytest.fixture(scope="module", params=[("spread", "spread"), ("spread_bias", "he")], ids=["spread", "bias"])
def weights(request):
    """(predictor weights, U-Net weights): zero biases, or every bias non-zero (the `spread_bias`
    set and the U-Net's `he` biases: conv/deconv biases, the projection bias)."""
    kind, ukind = request.param
    w = ls.weight_set(kind)
    u = ls.flatten_unet(ls.make_unet_weights(ukind))
    return w, u


@pytest.fixture(scope="module")
def wl():
    """300 pairs over 12 shapes (K = 1500, s = 0.5): ragged against max_batch 128."""
    w = ls.make_workload("C1", N=300, S=12)
    return w.points, w.pairs, w.poses


@pytest.fixture(scope="module")
def wl_oracle(oracle_mod, wl, weights):
    pts, pairs, poses = wl
    return oracle_mod.query_cells(weights[0], weights[1], pts, pairs, poses)


def make_ctx(locc_mod, w, u, points, max_batch=0, M=6):
    ctx = locc_mod.Locc(M=M, H=256, F=64, precision=0, device=0, max_batch=max_batch)
    ctx.load_weights_mem(w)
    ctx.load_unet_weights_mem(u)
    ctx.set_shapes(points)
    ctx.encode_shapes()
    return ctx


def assert_cells_parity(got, ref, E_gpu=None, pairs=None):
    assert np.array_equal(got["nsel"], ref["nsel"]), "selected-cell counts differ"
    assert np.array_equal(got["cells"], ref["cells"]), "selected-cell bits differ"
    if E_gpu is not None:
        used = np.unique(pairs)
        scale = np.abs(ref["grids"][used]).max()
        err = np.abs(E_gpu[used].astype(np.float64) - ref["grids"][used]).max()
        assert err <= E_TOL * scale, f"grid max err {err:.3g} (scale {scale:.3g})"
    assert np.abs(got["emb"].astype(np.float64) - ref["emb"]).max() <= E_TOL * max(1.0, np.abs(ref["emb"]).max())
    short = ref["nsel"].sum(1) == 0
    assert np.all(got["probs"][short] == 0) and np.all(np.isneginf(got["logits"][short]))
    dp = np.abs(got["probs"].astype(np.float64) - ref["probs"]).max()
    assert dp <= 1e-5, f"max |dp| = {dp:.3g}"
    band = np.abs(ref["probs"] - 0.5) <= 1e-3
    assert np.array_equal(got["labels"][~band], ref["labels"][~band])
    return dp


def test_cells_parity(locc_mod, wl, wl_oracle, weights):
    pts, pairs, poses = wl
    with make_ctx(locc_mod, *weights, pts, max_batch=128) as ctx:
        E, ms = ctx.cell_embeddings()
        got = ctx.query_cells(pairs, poses, debug=True)
    assert ms > 0
    assert (wl_oracle["nsel"].sum(1) == 0).any() and (wl_oracle["nsel"].sum(1) > 0).mean() > 0.8
    assert_cells_parity(got, wl_oracle, E, pairs)


def test_cells_parity_bf16_context(locc_mod, wl, wl_oracle, weights):
    """bf16 contexts run the U-Net and the predictor on the tensor cores (3xTF32, Q32): the
    selection is bit-exact; the grids within 5e-4 of max|E| (the tensor core's fp32 accumulation over
    K = 27 x 256 truncates: measured ~1e-4), probabilities within 5e-4 of the fp64 oracle with identical
    labels outside the 1e-3 band — the bf16 bar against an exact reference."""
    pts, pairs, poses = wl
    ctx = locc_mod.Locc(M=6, H=256, F=64, precision=1, device=0, max_batch=128)
    ctx.load_weights_mem(weights[0])
    ctx.load_unet_weights_mem(weights[1])
    ctx.set_shapes(pts)
    ctx.encode_shapes()
    E, _ = ctx.cell_embeddings()
    got = ctx.query_cells(pairs, poses, debug=True)
    ctx.close()
    ref = wl_oracle
    assert np.array_equal(got["cells"], ref["cells"]) and np.array_equal(got["nsel"], ref["nsel"])
    used = np.unique(pairs)
    assert np.abs(E[used] - ref["grids"][used]).max() <= 5e-4 * np.abs(ref["grids"][used]).max()
    short = ref["nsel"].sum(1) == 0
    assert np.all(got["probs"][short] == 0) and np.all(np.isneginf(got["logits"][short]))
    dp = np.abs(got["probs"].astype(np.float64) - ref["probs"]).max()
    assert dp <= 5e-4, f"max |dp| = {dp:.3g}"
    band = np.abs(ref["probs"] - 0.5) <= 1e-3
    assert np.array_equal(got["labels"][~band], ref["labels"][~band])


@pytest.mark.parametrize("chunk", [None, "1000", "4000"])
def test_cells_grid_encode_tensor_cores(locc_mod, wl, wl_oracle, weights, monkeypatch, chunk):
    """bf16 contexts encode the grid's layers 2-3 on the tensor cores (3xTF32, K = 256) in chunks of
    whole shapes.  With the U-Net forced onto CUDA cores (LOCC_CONV_FFMA), E must meet the fp32 bar
    (E_TOL of the fp64 oracle) for any chunking: one shape per chunk (1500 rows, a ragged last tile),
    two shapes per chunk, and all 12 in one; and the fp32 grid path (LOCC_GRID_FFMA) must agree."""
    pts, pairs, poses = wl
    monkeypatch.setenv("LOCC_CONV_FFMA", "1")
    if chunk:
        monkeypatch.setenv("LOCC_GRID_CHUNK", chunk)
    ctx = locc_mod.Locc(M=6, H=256, F=64, precision=1, device=0, max_batch=128)
    ctx.load_weights_mem(weights[0])
    ctx.load_unet_weights_mem(weights[1])
    ctx.set_shapes(pts)
    ctx.encode_shapes()
    E_tc, _ = ctx.cell_embeddings()
    monkeypatch.setenv("LOCC_GRID_FFMA", "1")
    ctx.encode_shapes()
    E_ff, _ = ctx.cell_embeddings()
    ctx.close()
    ref = wl_oracle["grids"]
    used = np.unique(pairs)
    scale = np.abs(ref[used]).max()
    err_tc = np.abs(E_tc[used].astype(np.float64) - ref[used]).max()
    err_ff = np.abs(E_ff[used].astype(np.float64) - ref[used]).max()
    assert err_tc <= E_TOL * scale, f"tensor-core grid: E err {err_tc:.3g} (scale {scale:.3g}, fp32 path {err_ff:.3g})"
    assert np.abs(E_tc - E_ff).max() <= E_TOL * scale


def test_cells_probe_weights_gpu(locc_mod, oracle_mod, wl):
    """The identity-encoder / delta-kernel U-Net probe (closed form pinned in test_oracle_cells):
    the device grids reproduce the oracle's exactly up to fp32 rounding of the copied values."""
    pts, pairs, poses = wl
    w, u = identity_encoder(), unet_probe()
    ref = oracle_mod.query_cells(w, u, pts, pairs[:40], poses[:40])
    with make_ctx(locc_mod, w, u, pts) as ctx:
        E, _ = ctx.cell_embeddings()
        got = ctx.query_cells(pairs[:40], poses[:40], debug=True)
    used = np.unique(pairs[:40])
    np.testing.assert_allclose(E[used], ref["grids"][used], rtol=1e-6, atol=1e-7)
    assert np.array_equal(got["cells"], ref["cells"])


def test_cells_device_buffers_and_symmetries(locc_mod, wl, weights):
    import torch
    pts, pairs, poses = wl
    with make_ctx(locc_mod, *weights, pts) as ctx:
        h = ctx.query_cells(pairs, poses)
        N = len(pairs)
        dp, dq = torch.from_numpy(pairs).cuda(), torch.from_numpy(poses).cuda()
        probs = torch.empty(N, device="cuda")
        labels = torch.empty(N, dtype=torch.uint8, device="cuda")
        s = torch.cuda.Stream()
        ctx.query_cells_into(dp, dq, probs, labels, stream=s.cuda_stream)
        s.synchronize()
        assert np.array_equal(probs.cpu().numpy(), h["probs"]) and np.array_equal(labels.cpu().numpy(), h["labels"])
        sw = ctx.query_cells(pairs[:, ::-1].copy(), poses[:, ::-1].copy())
        neg = poses.copy()
        neg[:, :, :4] *= -1
        ng = ctx.query_cells(pairs, neg)
    assert np.array_equal(sw["probs"], h["probs"]) and np.array_equal(ng["probs"], h["probs"])


def test_cells_state_errors(locc_mod, wl, weights):
    pts, pairs, poses = wl
    ctx = locc_mod.Locc(M=6, H=256, F=64, precision=0, device=0)
    ctx.load_weights_mem(weights[0])
    ctx.set_shapes(pts)
    with pytest.raises(locc_mod.LoccError):
        ctx.encode_shapes()          # no U-Net weights
    ctx.load_unet_weights_mem(weights[1])
    with pytest.raises(locc_mod.LoccError):
        ctx.query_cells(pairs, poses)  # not encoded
    ctx.encode_shapes()
    ctx.query_cells(pairs[:4], poses[:4])
    ctx.set_shapes(pts[:4])           # new shape table invalidates the grids
    with pytest.raises(locc_mod.LoccError):
        ctx.query_cells(pairs[:1] % 4, poses[:1])
    ctx.close()


@pytest.mark.parametrize("M", [3, 5, 8])
def test_cells_parity_other_grid_sizes(locc_mod, oracle_mod, weights, M):
    """The selection kernel's generic-M path (M = 6 is specialised) and the U-Net at other grid edges
    (M = 3: a single 1^3 interior after the valid conv; M = 8: 512 cells, 16 selection words)."""
    w = ls.make_workload("C1", N=40, S=6)
    ref = oracle_mod.query_cells(weights[0], weights[1], w.points, w.pairs, w.poses, M=M)
    with make_ctx(locc_mod, weights[0], weights[1], w.points, M=M) as ctx:
        E, _ = ctx.cell_embeddings()
        got = ctx.query_cells(w.pairs, w.poses, debug=True)
    assert_cells_parity(got, ref, E, w.pairs)


@pytest.mark.parametrize("M", [3, 8])
def test_cells_grid_encode_tensor_cores_other_grid_sizes(locc_mod, oracle_mod, weights, monkeypatch, M):
    """The tensor-core grid encode (bf16 context, U-Net on CUDA cores) at other grid edges: cell ids
    0..M^3-1 (up to 511) in the cell-max kernel; E to the fp32 bar of the fp64 oracle."""
    monkeypatch.setenv("LOCC_CONV_FFMA", "1")
    w = ls.make_workload("C1", N=40, S=6)
    ref = oracle_mod.query_cells(weights[0], weights[1], w.points, w.pairs, w.poses, M=M)
    ctx = locc_mod.Locc(M=M, H=256, F=64, precision=1, device=0)
    ctx.load_weights_mem(weights[0])
    ctx.load_unet_weights_mem(weights[1])
    ctx.set_shapes(w.points)
    ctx.encode_shapes()
    E, _ = ctx.cell_embeddings()
    ctx.close()
    scale = np.abs(ref["grids"]).max()
    assert np.abs(E.astype(np.float64) - ref["grids"]).max() <= E_TOL * scale


def test_cells_empty_and_disjoint_batches(locc_mod, weights, wl):
    pts, pairs, poses = wl
    with make_ctx(locc_mod, *weights, pts) as ctx:
        out = ctx.query_cells(pairs[:0], poses[:0], debug=True)
        assert out["probs"].shape == (0,)
        far = poses[:16].copy()
        far[:, 1, 4] += 10.0  # B far from A: no cell on either side, short-circuit
        got = ctx.query_cells(pairs[:16], far, debug=True)
    assert np.all(got["nsel"] == 0) and np.all(got["probs"] == 0) and np.all(got["labels"] == 0)
    assert np.all(np.isneginf(got["logits"])) and np.all(got["emb"] == 0) and np.all(got["cells"] == 0)


def test_cells_parity_global_max(locc_mod, oracle_mod, weights):
    """The appendix's global max pooling (locc_set_unet_global_pool(1)) against the oracle's."""
    w = ls.make_workload("C1", N=60, S=6)
    ref = oracle_mod.query_cells(weights[0], weights[1], w.points, w.pairs, w.poses, global_max=True)
    ctx = locc_mod.Locc(M=6, H=256, F=64, precision=0, device=0)
    ctx.load_weights_mem(weights[0])
    ctx.load_unet_weights_mem(weights[1])
    ctx.set_shapes(w.points)
    ctx.set_unet_global_pool(1)
    ctx.encode_shapes()
    E, _ = ctx.cell_embeddings()
    got = ctx.query_cells(w.pairs, w.poses, debug=True)
    ctx.close()
    assert_cells_parity(got, ref, E, w.pairs)


@pytest.mark.parametrize("H,F", [(256, 16), (128, 32)])
def test_cells_parity_other_widths(locc_mod, oracle_mod, H, F):
    """Encode-once at the appendix's F = 16 and a narrower point MLP: the generic selection and
    predictor paths against the oracle."""
    w = ls.flatten_weights(ls.make_weights("spread", H, F, calib=ls.load_calibration()), H, F)
    u = ls.flatten_unet(ls.make_unet_weights("spread", H, F), H, F)
    wl = ls.make_workload("C1", N=60, S=6)
    ref = oracle_mod.query_cells(w, u, wl.points, wl.pairs, wl.poses, H=H, F=F)
    ctx = locc_mod.Locc(M=6, H=H, F=F, precision=0, device=0)
    ctx.load_weights_mem(w)
    ctx.load_unet_weights_mem(u)
    ctx.set_shapes(wl.points)
    ctx.encode_shapes()
    E, _ = ctx.cell_embeddings()
    got = ctx.query_cells(wl.pairs, wl.poses, debug=True)
    ctx.close()
    assert_cells_parity(got, ref, E, wl.pairs)
