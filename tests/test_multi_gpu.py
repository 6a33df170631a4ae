"""Multi-GPU forms of the library on the one GPU this harness has.

* A multi-device context (locc_config.n_devices > 1) with device_ids = [0, 0]: two sub-contexts on the
  same GPU, each with its own stream and scratch, exercise the sharding, the fan-out of every call and
  the gather into the caller's buffers (host and device-resident, synchronous and on a caller stream).
  Pairs are independent, so the sharded answer must equal the single-context answer BITWISE (fp32, and
  bf16 with locc_set_deterministic).  (Two ranks whose kernels wait on one another are never run on one
  GPU; these sub-contexts do not wait on one another.)
* The library-owned NCCL gather (locc_comm_init + locc_query_allgather) in a world of one rank: the
  collective runs and leaves the unsharded answer.
"""
import numpy as np
import pytest

import locc_synth as ls

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def locc_mod():
    from paper_2304_09439_b200 import build as b
    b.build()
    from paper_2304_09439_b200 import locc
    return locc


@pytest.fixture(scope="module")
def wl():
    return ls.make_workload("C1", N=3001, S=40)


def _ctx(locc_mod, precision, devices=None, max_batch=0, det=True, unet=False, wl=None):
    ctx = locc_mod.Locc(precision=precision, device=0, devices=devices, max_batch=max_batch)
    ctx.set_deterministic(det)
    ctx.load_weights_mem(ls.weight_set("spread_bias"))
    ctx.set_shapes(wl.points)
    if unet:
        ctx.load_unet_weights_mem(ls.flatten_unet(ls.make_unet_weights("he")))
        ctx.encode_shapes()
    return ctx


@pytest.mark.parametrize("precision", [0, 1])
def test_group_query_equals_single_context(locc_mod, wl, precision):
    import torch
    with _ctx(locc_mod, precision, wl=wl) as one, _ctx(locc_mod, precision, devices=[0, 0], max_batch=700,
                                                        wl=wl) as grp:
        a = one.query_debug(wl.pairs, wl.poses)
        b = grp.query_debug(wl.pairs, wl.poses)
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        # device buffers on a caller stream, and the pose gradient
        pairs, poses = torch.from_numpy(wl.pairs).cuda(), torch.from_numpy(wl.poses).cuda()
        N = len(wl.pairs)
        p1, p2 = torch.empty(N, device="cuda"), torch.empty(N, device="cuda")
        g1, g2 = torch.empty(N, 14, device="cuda"), torch.empty(N, 14, device="cuda")
        s = torch.cuda.Stream()
        one.query_grad_into(pairs, poses, p1, g1, stream=s.cuda_stream)
        grp.query_grad_into(pairs, poses, p2, g2, stream=s.cuda_stream)
        s.synchronize()
        assert torch.equal(p1, p2) and torch.equal(g1, g2)
        st = grp.stats()
        assert st["pairs"] == N
    with pytest.raises(locc_mod.LoccError):  # an invalid id on any shard is reported
        with _ctx(locc_mod, precision, devices=[0, 0], wl=wl) as grp:
            bad = wl.pairs.copy()
            bad[-1, 0] = len(wl.points)
            grp.query(bad, wl.poses)


def test_group_encode_once_and_sim(locc_mod, wl):
    import torch
    with _ctx(locc_mod, 0, unet=True, wl=wl) as one, _ctx(locc_mod, 0, devices=[0, 0], unet=True, wl=wl) as grp:
        a = one.query_cells(wl.pairs, wl.poses, debug=True)
        b = grp.query_cells(wl.pairs, wl.poses, debug=True)
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        E1, _ = one.cell_embeddings()
        E2, _ = grp.cell_embeddings()
        assert np.array_equal(E1, E2)
        ids, body, state = ls.make_sim_scene(wl.points, 257, seed=81)
        outs = []
        for ctx in (one, grp):
            d_st = torch.from_numpy(state.copy()).cuda()
            d_con = torch.zeros(257, 3, dtype=torch.int32, device="cuda")
            for k in range(3):
                ctx.sim_run(dict(ls.SIM_DEFAULTS, substeps=2), torch.from_numpy(ids).cuda(),
                            torch.from_numpy(body).cuda(), d_st, t0=0.01 * k, contacts=d_con)
            outs.append((d_st.cpu().numpy(), d_con.cpu().numpy()))
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("precision", [0, 1])
def test_allgather_world_of_one(locc_mod, wl, precision):
    import torch
    with _ctx(locc_mod, precision, wl=wl) as ctx:
        ctx.comm_init(1, 0, locc_mod.comm_unique_id())
        pr, lb, lg = ctx.query(wl.pairs, wl.poses)
        N = len(wl.pairs)
        hp, hl, hg = np.zeros(N, np.float32), np.zeros(N, np.uint8), np.zeros(N, np.float32)
        ctx.query_allgather_into(wl.pairs, wl.poses, hp, hl, hg)
        assert np.array_equal(hp, pr) and np.array_equal(hl, lb) and np.array_equal(hg, lg)
        pairs, poses = torch.from_numpy(wl.pairs).cuda(), torch.from_numpy(wl.poses).cuda()
        dp = torch.empty(N, device="cuda")
        ctx.query_allgather_into(pairs, poses, dp)
        assert np.array_equal(dp.cpu().numpy(), pr)
