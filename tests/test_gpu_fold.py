"""Head-folding kernels (csrc/fold.cu) vs a plain PyTorch fp32 reference of the same algebra."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_09386_b200._lib import call, ptr


@pytest.mark.parametrize("E,T,d_out,d_in", [(32, 8, 256, 512), (16, 4, 128, 128), (8, 13, 96, 64), (4, 32, 64, 256)])
def test_fold_and_unfold(E, T, d_out, d_in):
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(E + T + d_in)
    ldg = (T + 7) // 8 * 8
    hw = torch.randn(T, d_out, generator=g, device=dev)
    W = (torch.randn(E, d_out, d_in, generator=g, device=dev) / d_in ** 0.5).to(torch.bfloat16)
    b = torch.randn(E, d_out, generator=g, device=dev)
    G = torch.full((E, ldg, d_in), 7.0, device=dev).to(torch.bfloat16)
    c = torch.full((E, ldg), 7.0, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    work = torch.zeros(call("smes_fold_work_floats", E, T, d_out, d_in), device=dev)
    call("smes_fold_heads", E, T, ldg, d_out, d_in, ptr(hw), ptr(W), ptr(b), ptr(G), ptr(c), ptr(work), st)
    Wf = W.float()
    refG = torch.einsum("tj,ejk->etk", hw, Wf)
    torch.cuda.synchronize()
    assert (G[:, :T].float() - refG).abs().max().item() <= 1e-2 * refG.abs().max().item()
    assert torch.all(G[:, T:] == 0) and torch.all(c[:, T:] == 0)
    assert torch.allclose(c[:, :T], torch.einsum("tj,ej->et", hw, b), rtol=1e-4, atol=1e-4)

    Qt = torch.zeros(E, d_in + 1, ldg, device=dev)
    Qt[:, :, :T] = torch.randn(E, d_in + 1, T, generator=g, device=dev)
    dW = torch.full((E, d_out, d_in), float("nan"), device=dev)
    db = torch.full((E, d_out), float("nan"), device=dev)
    dhw = torch.full((T, d_out), float("nan"), device=dev)
    csum = Qt[:, d_in, :]                         # the ones-column row of Qt
    call("smes_unfold_grads", E, T, ldg, d_out, d_in, ptr(Qt), (d_in + 1) * ldg, ptr(csum), (d_in + 1) * ldg,
         ptr(hw), ptr(W), ptr(b), ptr(dW), ptr(db), ptr(work), ptr(dhw), st)
    torch.cuda.synchronize()
    Q = Qt[:, :d_in, :T]                          # (E, d_in, T)
    cs = csum[:, :T]
    ref_dW = torch.einsum("tj,ekt->ejk", hw, Q)
    ref_db = torch.einsum("tj,et->ej", hw, cs)
    ref_dhw = torch.einsum("ekt,ejk->tj", Q, Wf) + torch.einsum("et,ej->tj", cs, b)
    for got, ref in ((dW, ref_dW), (db, ref_db), (dhw, ref_dhw)):
        assert (got - ref).abs().max().item() <= 1e-5 * ref.abs().max().item() + 1e-6
