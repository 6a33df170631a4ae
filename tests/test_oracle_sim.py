"""Pins of the oracle's closed-loop substep (NEXT-3, Q31): the semi-implicit Euler integrator
against its discrete closed forms (free fall, constant spin via a matrix power), the kinematic bowl's
trajectory, the broad phase, the penalty force descending the collision score (checked by re-querying
the oracle's own network at the new poses), and the body-swap symmetry."""
import numpy as np

import locc_synth as ls
from test_oracle_network import spread

SIM = dict(ls.SIM_DEFAULTS)


def scene(E=16, seed=70):
    pts, _ = ls.make_shapes(10, 600, seed=seed)
    ids, body, st = ls.make_sim_scene(pts, E, seed=seed + 1)
    return pts, ids, body, st.astype(np.float64)


def test_free_fall_and_spin_closed_forms(oracle_mod):
    pts, ids, body, st = scene()
    st[:, 1, 4:7] += np.array([5.0, 0, 0])   # far from the bowl and from each other: all culled
    st[:, 2, 4:7] += np.array([-5.0, 0, 0])
    rng = np.random.default_rng(71)
    st[:, 1:, 7:10] = rng.normal(0, 0.1, (len(st), 2, 3))
    st[:, 1:, 10:13] = rng.normal(0, 3.0, (len(st), 2, 3))
    sim = dict(SIM, substeps=7)
    out, con, mg = oracle_mod.sim_run(spread(), pts, sim, ids, body, st, t0=0.3)
    assert con.sum() == 0 and np.all(mg[:, 2] > 1.0)
    h, n, g = sim["h"], 7, np.array(sim["gravity"])
    # semi-implicit Euler: v_n = v_0 + n h g, t_n = t_0 + n h v_0 + h^2 g n (n + 1) / 2
    np.testing.assert_allclose(out[:, 1:, 7:10], st[:, 1:, 7:10] + n * h * g, rtol=0, atol=1e-13)
    np.testing.assert_allclose(out[:, 1:, 4:7], st[:, 1:, 4:7] + n * h * st[:, 1:, 7:10] + h * h * g * n * (n + 1) / 2,
                               rtol=0, atol=1e-13)
    # constant spin: q_n = normalise((I + h/2 Omega(w))^n q_0), Omega(w) q = (0, w) (x) q
    for e in range(len(st)):
        for b in (1, 2):
            w = st[e, b, 10:13]
            Om = np.array([[0, -w[0], -w[1], -w[2]], [w[0], 0, -w[2], w[1]], [w[1], w[2], 0, -w[0]],
                           [w[2], -w[1], w[0], 0]])
            q = np.linalg.matrix_power(np.eye(4) + 0.5 * h * Om, n) @ st[e, b, :4]
            np.testing.assert_allclose(out[e, b, :4], q / np.linalg.norm(q), rtol=0, atol=1e-13)
            np.testing.assert_array_equal(out[e, b, 10:13], w)
    # the kinematic bowl at the end time t0 + n h
    tau = 0.3 + n * h
    a, f = np.array(sim["amp"]), sim["freq"]
    np.testing.assert_allclose(out[:, 0, 4:7], np.tile(a * np.sin(2 * np.pi * f * tau), (len(st), 1)), atol=1e-15)
    np.testing.assert_allclose(out[:, 0, 7:10], np.tile(a * 2 * np.pi * f * np.cos(2 * np.pi * f * tau), (len(st), 1)),
                               atol=1e-15)


def test_penalty_descends_the_score(oracle_mod):
    """One substep with contact forces only (no gravity, bodies at rest): for each contact pair of
    dynamic bodies the first-order change of the logit is -lambda h^2 (sum |g_t|^2 / m + ...) / n < 0,
    so re-querying at the new poses must show a smaller logit (up to ReLU-region changes)."""
    pts, ids, body, st = scene(E=48, seed=72)
    st[:, 1:, 4] += 5.0  # both dynamic bodies away from the bowl (its pairs culled), relative pose kept
    sim = dict(SIM, substeps=1, gravity=(0.0, 0.0, 0.0), amp=(0.0, 0.0, 0.0), ks=50.0, kd=0.0)
    w = spread()
    out, con, _ = oracle_mod.sim_run(w, pts, sim, ids, body, st)
    pairs = [(0, 1), (0, 2), (1, 2)]
    dec = tot = 0
    for e in np.nonzero(con[:, 2] > 0)[0]:  # the pair of the two dynamic bodies
        a, b = pairs[2]
        pr = np.array([[ids[e, a], ids[e, b]]], np.int32)
        before = np.stack([st[e, a, :7], st[e, b, :7]])[None].astype(np.float32)
        after = np.stack([out[e, a, :7], out[e, b, :7]])[None].astype(np.float32)
        l0, _, _ = oracle_mod.query_grad(w, pts, pr, before)
        l1, _, _ = oracle_mod.query_grad(w, pts, pr, after)
        tot += 1
        dec += l1[0] < l0[0]
    assert tot >= 5 and dec >= 0.9 * tot, (dec, tot)


def test_body_swap_symmetry(oracle_mod):
    pts, ids, body, st = scene(E=12, seed=73)
    w = spread()
    out, con, _ = oracle_mod.sim_run(w, pts, SIM, ids, body, st)
    sw = [0, 2, 1]
    out2, con2, _ = oracle_mod.sim_run(w, pts, SIM, ids[:, sw], body[:, sw], st[:, sw])
    np.testing.assert_allclose(out2[:, sw], out, rtol=1e-9, atol=1e-12)
    assert np.array_equal(con2[:, [1, 0, 2]], con)
    assert con.sum() > 0


def test_cells_detector_runs_and_contacts(oracle_mod):
    pts, ids, body, st = scene(E=8, seed=74)
    u = ls.flatten_unet(ls.make_unet_weights())
    out, con, mg = oracle_mod.sim_run(spread(), pts, dict(SIM, detector="cells"), ids, body, st, unet_flat=u)
    assert np.all(np.isfinite(out)) and con.sum() > 0
    np.testing.assert_allclose(np.linalg.norm(out[:, :, :4], axis=-1), 1.0, atol=1e-12)
