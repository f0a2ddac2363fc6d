"""Head-folding kernels (csrc/fold.cu) vs a plain PyTorch fp32 reference of the same algebra."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_09386_b200._lib import call, ptr


@pytest.mark.parametrize("E,T,d_out,d_in", [(32, 8, 256, 512), (16, 4, 128, 128), (8, 13, 96, 64), (4, 32, 64, 256),
                                            (16, 8, 1024, 1024), (32, 32, 512, 1024), (8, 13, 2048, 1024)])
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

    Qf = torch.zeros(E, ldg, d_in, device=dev)
    Qf[:, :T] = torch.randn(E, T, d_in, generator=g, device=dev)
    cs_full = torch.zeros(E, ldg, device=dev)
    cs_full[:, :T] = torch.randn(E, T, generator=g, device=dev)
    dW = torch.full((E, d_out, d_in), float("nan"), device=dev)
    db = torch.full((E, d_out), float("nan"), device=dev)
    dhw = torch.full((T, d_out), float("nan"), device=dev)
    call("smes_unfold_grads", E, T, ldg, d_out, d_in, ptr(Qf), ldg * d_in, d_in, 1, ptr(cs_full), ldg,
         ptr(hw), ptr(W), ptr(b), ptr(dW), ptr(db), ptr(work), ptr(dhw), st)
    torch.cuda.synchronize()
    Q = Qf[:, :T].transpose(1, 2)                 # (E, d_in, T)
    cs = cs_full[:, :T]
    ref_dW = torch.einsum("tj,ekt->ejk", hw, Q)
    ref_db = torch.einsum("tj,et->ej", hw, cs)
    ref_dhw = torch.einsum("ekt,ejk->tj", Q, Wf) + torch.einsum("et,ej->tj", cs, b)
    # split-K CUDA-core path: fp32 throughout; tensor-core path (E*d_out*d_in >= 2^24): bf16 hi + lo
    # operand pairs with fp32 accumulation
    tol = 1e-5 if E * d_out * d_in < (1 << 24) else 1e-4
    for got, ref in ((dW, ref_dW), (db, ref_db), (dhw, ref_dhw)):
        assert (got - ref).abs().max().item() <= tol * ref.abs().max().item() + 1e-6


@pytest.mark.parametrize("E,T,d_out,d_in", [(32, 8, 256, 512), (8, 13, 96, 64), (16, 8, 1024, 1024)])
def test_unfold_k_major_layout(E, T, d_out, d_in):
    """Q in (E, d_in, ldg) layout (the small-bank wgrad orientation) gives the same grads."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(7 * E + T)
    ldg = (T + 7) // 8 * 8
    hw = torch.randn(T, d_out, generator=g, device=dev)
    W = (torch.randn(E, d_out, d_in, generator=g, device=dev) / d_in ** 0.5).to(torch.bfloat16)
    b = torch.randn(E, d_out, generator=g, device=dev)
    Qf = torch.zeros(E, ldg, d_in, device=dev)
    Qf[:, :T] = torch.randn(E, T, d_in, generator=g, device=dev)
    Qk = Qf.transpose(1, 2).contiguous()          # (E, d_in, ldg)
    cs = torch.zeros(E, ldg, device=dev)
    cs[:, :T] = torch.randn(E, T, generator=g, device=dev)
    work = torch.zeros(call("smes_fold_work_floats", E, T, d_out, d_in), device=dev)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for Q, strides in ((Qf, (ldg * d_in, d_in, 1)), (Qk, (d_in * ldg, 1, ldg))):
        dW = torch.zeros(E, d_out, d_in, device=dev)
        db = torch.zeros(E, d_out, device=dev)
        dhw = torch.zeros(T, d_out, device=dev)
        call("smes_unfold_grads", E, T, ldg, d_out, d_in, ptr(Q), *strides, ptr(cs), ldg, ptr(hw), ptr(W), ptr(b),
             ptr(dW), ptr(db), ptr(work), ptr(dhw), st)
        torch.cuda.synchronize()
        outs.append((dW.clone(), db.clone(), dhw.clone()))
    for a, c in zip(outs[0], outs[1]):
        assert torch.allclose(a, c, rtol=1e-5, atol=1e-6)
