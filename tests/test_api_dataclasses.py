"""Host-side checks of the drop-in dataclasses (no GPU): the reference's fields and constructors
(experts.py:26-60, routing.py:64-99, model.py:36-111, linalg.py:116-141), the views that tie the
reference's per-map ``Affine`` lists to the stacked tensors the kernels read, and the reference's
validation errors."""
import pytest
import torch

import paper_2602_09386_b200 as smes


def _aff(d_out, d_in, seed):
    g = torch.Generator().manual_seed(seed)
    return smes.Affine(torch.randn(d_out, d_in, generator=g), torch.randn(d_out, generator=g))


def test_expert_pool_reference_form_and_views():
    layers = [_aff(6, 5, e) for e in range(4)]
    pool = smes.ExpertPool(layers, "relu")
    assert pool.num_experts == 4 and pool.d_in == 5 and pool.d_out == 6
    assert pool.weight.shape == (4, 6, 5) and pool.bias.shape == (4, 6)
    # layers are views of the stacked storage: in-place updates go both ways
    pool.layers[2].weight.add_(1.0)
    assert torch.equal(pool.weight[2], pool.layers[2].weight)
    pool.weight.mul_(2.0)
    assert torch.equal(pool.layers[1].weight, pool.weight[1])
    # rebinding a layer's weight re-stacks on the next access
    pool.layers[0].weight = torch.zeros(6, 5)
    assert float(pool.weight[0].abs().sum()) == 0.0
    # assigning the stacked weight rebinds every layer
    pool.weight = torch.ones(4, 6, 5)
    assert float(pool.layers[3].weight.sum()) == 30.0
    s = smes.ExpertPool.stacked(torch.zeros(3, 2, 4), torch.zeros(3, 2), "identity")
    assert s.num_experts == 3 and len(s.layers) == 3 and s.layers[0].d_in == 4


def test_expert_pool_validation():
    with pytest.raises(smes.ConfigError):
        smes.ExpertPool([], "relu")
    with pytest.raises(smes.ConfigError):
        smes.ExpertPool([_aff(2, 3, 0)], "gelu")
    with pytest.raises(smes.ShapeError, match="expert 1 maps 3->4, expected 3->2"):
        smes.ExpertPool([_aff(2, 3, 0), _aff(4, 3, 1)])
    with pytest.raises(smes.ShapeError):
        smes.Affine(torch.zeros(2, 3), torch.zeros(3))


def test_router_bank_reference_form():
    maps = [_aff(8, 5, t) for t in range(3)]
    rb = smes.RouterBank(maps, [1.0, 2.0, 0.5])
    assert rb.num_tasks == 3 and rb.num_experts == 8 and rb.d_in == 5
    assert rb.weight.shape == (3, 8, 5) and rb.bias.shape == (3, 8)
    assert torch.equal(rb.maps[1].weight, rb.weight[1])
    assert rb.task_weights.dtype == torch.float64
    with pytest.raises(smes.ConfigError):
        smes.RouterBank([])
    with pytest.raises(smes.ShapeError, match="router 1 has shape"):
        smes.RouterBank([_aff(8, 5, 0), _aff(7, 5, 1)])
    with pytest.raises(smes.ShapeError):
        smes.RouterBank(maps, [1.0, 2.0])
    with pytest.raises(smes.ConfigError):
        smes.RouterBank(maps, [1.0, -2.0, 0.5])


def _model(T=3, E=8, d=5, d_out=6):
    enc1, enc2 = _aff(7, 4, 90), _aff(d, 7, 91)
    pool = smes.ExpertPool([_aff(d_out, d, e) for e in range(E)], "relu")
    rb = smes.RouterBank([_aff(E, d, 10 + t) for t in range(T)])
    heads = [_aff(1, d_out, 20 + t) for t in range(T)]
    return smes.MoeModel(enc1, enc2, pool, rb, heads, [1.0] * T, 0.01, smes.RoutingBudget(2, 1))


def test_moe_model_fields_and_blocks():
    m = _model()
    assert len(m.heads) == 3 and m.head_w.shape == (3, 6) and m.head_b.shape == (3,)
    assert (m.num_features, m.d_hidden, m.d_in, m.d_out, m.num_experts, m.num_tasks) == (4, 7, 5, 6, 8, 3)
    names = list(m.parameter_blocks())
    # reference checkpoint order (model.py:94-111)
    assert names[:4] == ["encoder1.weight", "encoder1.bias", "encoder2.weight", "encoder2.bias"]
    assert names[4:6] == ["expert_0.weight", "expert_0.bias"]
    assert names[4 + 16:4 + 18] == ["router_0.weight", "router_0.bias"]
    assert names[-2:] == ["head_2.weight", "head_2.bias"]
    assert m.parameter_blocks()["head_1.weight"].shape == (1, 6)
    assert m.num_parameters() == sum(v.numel() for v in m.parameter_blocks().values())
    # heads are views of the stacked head weights the kernels read
    m.heads[1].weight.add_(1.0)
    assert torch.equal(m.head_w[1], m.heads[1].weight[0])


def test_moe_model_validation():
    m = _model()
    with pytest.raises(smes.ConfigError, match="2 heads for 3 routers"):
        smes.MoeModel(m.encoder1, m.encoder2, m.experts, m.routers, m.heads[:2], [1.0] * 3, 0.0,
                      smes.RoutingBudget(2, 1))
    with pytest.raises(smes.ConfigError):
        smes.MoeModel(m.encoder1, m.encoder2, m.experts, m.routers, m.heads, [1.0] * 3, -0.1,
                      smes.RoutingBudget(2, 1))
    with pytest.raises(smes.ConfigError, match="head 0 must map d_out -> 1"):
        smes.MoeModel(m.encoder1, m.encoder2, m.experts, m.routers, [_aff(2, 6, 0)] * 3, [1.0] * 3, 0.0,
                      smes.RoutingBudget(2, 1))
    with pytest.raises(smes.ConfigError):
        smes.MoeModel(m.encoder1, m.encoder2, m.experts, m.routers, m.heads, [1.0] * 3, 0.0,
                      smes.RoutingBudget(5, 4))
    with pytest.raises(smes.ConfigError, match="encoder output width"):
        smes.MoeModel(m.encoder1, _aff(4, 7, 0), m.experts, m.routers, m.heads, [1.0] * 3, 0.0,
                      smes.RoutingBudget(2, 1))


def test_init_model_structure():
    g = torch.Generator().manual_seed(0)
    m = smes.init_model(g, 12, 16, 8, 8, 6, 3, smes.RoutingBudget(2, 1), expert_nonlinearity="relu", device="cpu")
    assert isinstance(m.experts, smes.ExpertPool) and len(m.experts.layers) == 6
    assert len(m.routers.maps) == 3 and len(m.heads) == 3
    assert float(m.routers.weight.abs().max()) <= 1e-3 / 8 ** 0.5 + 1e-12      # near-zero routers (model.py:32)
    assert torch.all(m.encoder1.bias == 0.01)


def test_device_helpers_need_cuda():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(smes.CudaError):
        smes.softmax(torch.zeros(2, 3))
