"""Pin the CPU oracle (oracle/smes_oracle.py) against the reference.

Two sources: (1) the reference's own known-answer tests, restated with their
file:line; (2) golden fixtures generated from the reference itself by
tests/golden/make_golden.py.  CPU only.
"""
import math
import os

import numpy as np
import pytest

from oracle import smes_oracle as O


# ---------------------------------------------------------------- known answers

def test_two_term_weights():
    # test_routing.py:113-120
    r = O.route_batch(np.array([[[2.0, 1.0, 0.0, -1.0]]]), 0, 2)
    assert abs(r.weights[0, 0, 0] - math.exp(2) / (math.exp(2) + math.exp(1))) < 1e-12
    assert abs(r.weights[0, 0, 1] - 0.268941) < 1e-6
    assert r.weights[0, 0, 2] == 0.0 and r.weights[0, 0, 3] == 0.0


def test_hand_traced_two_stage():
    # test_routing.py:147-160
    probs = np.array([[0.4, 0.3, 0.2, 0.1], [0.1, 0.5, 0.3, 0.1]])
    z = np.array([[4.0, 3.0, 2.0, 1.0], [1.0, 5.0, 3.0, 1.0]])
    r = O.route_batch(z[:, None, :], 1, 1, full_probs=probs[:, None, :])
    assert r.shared[0].tolist() == [1]
    assert r.adaptive[0, 0].tolist() == [0] and r.adaptive[1, 0].tolist() == [2]
    assert r.unions[0].tolist() == [0, 1, 2]


def test_identical_logits_union():
    # test_routing.py:106-111 (naive = K_s 0)
    z = np.tile(np.array([3.0, 1.0, 2.0, 0.0]), (3, 1))[:, None, :]
    r = O.route_batch(z, 0, 2)
    assert r.unions[0].tolist() == [0, 2]


def test_tie_lowest_index():
    # linalg.py:86-101, test_linalg.py:106-107
    assert O.top_k_rows(np.array([[1.0, 3.0, 3.0, 0.0, 3.0]]), 2).tolist() == [[1, 2]]


def test_plan_hand_example():
    # test_execution.py:27-37
    p = O.build_execution_plan([np.array([0, 2]), np.array([2, 3])], 4)
    assert p.loads.tolist() == [1, 0, 2, 1]
    assert list(zip(p.gather_instances.tolist(), p.gather_experts.tolist())) == [(0, 0), (0, 2), (1, 2), (1, 3)]
    assert p.segment_offsets.tolist() == [0, 1, 1, 3, 4]


def _routing(active, weights):
    active = np.asarray(active)
    weights = np.asarray(weights, dtype=np.float64)
    return O.Routing(np.zeros((active.shape[1], 0), np.int64), active, active,
                     [np.unique(active[:, i, :]) for i in range(active.shape[1])], weights, weights)


def test_lb_known_values():
    # test_balance.py:42-69
    assert O.compute_load_stats(_routing([[[0, 1], [2, 3]]], [[[.5, .5, 0, 0], [0, 0, .5, .5]]])).value == 1.0
    w = np.zeros((2, 3, 5)); w[:, :, 0] = 1.0
    assert O.compute_load_stats(_routing([[[0], [0], [0]], [[0], [0], [0]]], w)).value == 5.0
    s = O.compute_load_stats(_routing([[[0, 1]], [[1, 2]]], [[[.6, .4, 0, 0]], [[0, .7, .3, 0]]]))
    assert abs(s.value - 1.55) < 1e-12
    assert np.allclose(s.frequency, [0.5, 1.0, 0.5, 0.0]) and np.allclose(s.mass, [0.3, 0.55, 0.15, 0.0])


def test_lb_gradient_vs_finite_difference():
    # test_balance.py:128-161: gradient w.r.t. logits with frequency frozen
    rng = np.random.default_rng(5)
    z = rng.normal(size=(3, 6, 7))
    for dense in (False, True):
        r = O.route_batch(z, 1, 2)
        st = O.compute_load_stats(r, dense)
        g = O.lb_loss_gradient(st, r)
        eps = 1e-6
        for (t, b, e) in [(0, 0, 0), (1, 3, 4), (2, 5, 6), (0, 2, 3)]:
            zp, zm = z.copy(), z.copy()
            zp[t, b, e] += eps; zm[t, b, e] -= eps
            def val(zz):
                rr = O.frozen_routing(zz, r.shared, r.adaptive, r.active)
                probs = rr.full_probs if dense else rr.weights
                return (z.shape[2] / r.k_total) * np.dot(st.frequency, probs.sum(axis=(0, 1)) / (6 * 3))
            fd = (val(zp) - val(zm)) / (2 * eps)
            assert abs(fd - g[t, b, e]) < 1e-5


def test_budget_errors():
    with pytest.raises(O.OracleError, match="candidates"):
        O.route_batch(np.zeros((2, 1, 4)), 3, 2)
    with pytest.raises(O.OracleError):
        O.route_batch(np.zeros((2, 1, 4)), 0, 0)


# ---------------------------------------------------------------- golden fixtures

def test_routing_golden(golden_dir):
    g = np.load(os.path.join(golden_dir, "routing_golden.npz"))
    for i in range(int(g["n"])):
        c = lambda k: g[f"c{i}_{k}"]
        tw = c("task_weights") if f"c{i}_task_weights" in g.files else None
        r = O.route_batch(c("z"), int(c("k_shared")), int(c("k_adaptive")), tw)
        assert np.array_equal(r.shared, c("shared"))
        assert np.array_equal(r.adaptive, c("adaptive"))
        assert np.array_equal(r.active, c("active"))
        assert np.array_equal(np.array([u.size for u in r.unions]), c("union_sizes"))
        assert np.array_equal(np.concatenate(r.unions), c("union_flat"))
        assert np.abs(r.weights - c("weights")).max() < 1e-15
        if f"c{i}_loads" in g.files:
            p = O.build_execution_plan(r.unions, c("z").shape[2])
            for k in ("loads", "segment_offsets", "gather_instances", "gather_experts", "row_keys"):
                assert np.array_equal(getattr(p, k), c(k)), k


def _params(g):
    return O.LayerParams(g["router_w"], g["router_b"],
                         [(g["expert_w"], g["expert_b"], str(g["act"]))],
                         g["head_w"], g["head_b"], g["task_weights"])


@pytest.mark.parametrize("i", range(5))
def test_layer_golden(golden_dir, i):
    g = np.load(os.path.join(golden_dir, f"layer_golden_{i}.npz"))
    p = _params(g)
    f = O.forward_sparse(g["h"], p, int(g["k_shared"]), int(g["k_adaptive"]))
    rel = lambda a, b: np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
    assert rel(f.router_logits, g["router_logits"]) < 1e-13
    assert np.array_equal(f.routing.active, g["active"])
    assert np.array_equal(f.plan.gather_instances, g["gather_instances"])
    assert rel(f.layer_outs[-1], g["packed_out"]) < 1e-12
    assert rel(f.task_reps, g["task_reps"]) < 1e-12
    assert rel(f.predictions, g["predictions"]) < 1e-12
    bw = O.backward(f, p, g["labels"], g["lam"], float(g["beta"]), bool(int(g["dense"])))
    assert abs(bw.task_value - float(g["task_value"])) < 1e-12
    assert abs(bw.lb_value - float(g["lb_value"])) < 1e-12
    assert np.array_equal(bw.stats.counts, g["stats_counts"])
    assert rel(bw.layers[0][0], g["g_expert_w"]) < 1e-10
    assert rel(bw.layers[0][1], g["g_expert_b"]) < 1e-10
    assert rel(bw.router_w, g["g_router_w"]) < 1e-10
    assert rel(bw.router_b, g["g_router_b"]) < 1e-10
    assert rel(bw.head_w, g["g_head_w"]) < 1e-10
    assert rel(bw.head_b, g["g_head_b"]) < 1e-10
    assert rel(bw.d_hidden, g["d_hidden"]) < 1e-10


def test_two_layer_expert_grads_vs_finite_difference():
    """The 2-layer expert stack (not in the reference) is validated by central
    differences with frozen selections, the reference's grad_check recipe
    (training.py:537-596)."""
    rng = np.random.default_rng(11)
    b, t, e, d, dff = 12, 3, 6, 6, 10
    p = O.init_layer_params(rng, d, d, e, t, d_ff=dff, router_scale=1.0)
    p.layers = [(w, rng.normal(size=bb.shape) * 0.1, a) for (w, bb, a) in p.layers]
    h = rng.normal(size=(b, d))
    y = (rng.uniform(size=(t, b)) < 0.4).astype(float)
    beta = 0.05
    f = O.forward_sparse(h, p, 1, 2)
    bw = O.backward(f, p, y, None, beta)

    def loss(pp, hh):
        ff = O.forward_sparse(hh, pp, 1, 2, frozen=f.routing, frozen_plan=f.plan)
        st = O.LoadStats(bw.stats.frequency, None, None, None, b, t, 3, False)
        mass = ff.routing.weights.sum(axis=(0, 1)) / (b * t)
        lb = (e / 3) * np.dot(st.frequency, mass)
        return O.weighted_bce(ff.predictions, y, np.ones(t)) + beta * lb

    eps = 1e-6
    checks = [("layers", 0, 0, (1, 2, 3)), ("layers", 1, 0, (2, 1, 4)), ("layers", 0, 1, (3, 5)),
              ("layers", 1, 1, (0, 2)), ("router_w", None, None, (1, 2, 3)), ("head_w", None, None, (2, 1)),
              ("h", None, None, (4, 2))]
    for name, li, wi, idx in checks:
        def perturbed(delta):
            import copy
            pp = copy.deepcopy(p)
            hh = h.copy()
            if name == "layers":
                arrs = [list(x) for x in pp.layers]
                arrs[li][wi] = np.array(arrs[li][wi], dtype=float)
                arrs[li][wi][idx] += delta
                pp.layers = [tuple(x) for x in arrs]
            elif name == "h":
                hh[idx] += delta
            else:
                getattr(pp, name)[idx] += delta
            return loss(pp, hh)
        fd = (perturbed(eps) - perturbed(-eps)) / (2 * eps)
        if name == "layers":
            an = bw.layers[li][wi][idx]
        elif name == "h":
            an = bw.d_hidden[idx]
        else:
            an = getattr(bw, name)[idx]
        assert abs(fd - an) <= 1e-6 + 1e-4 * abs(an), (name, li, wi, idx, fd, an)
