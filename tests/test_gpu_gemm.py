"""tcgen05 grouped GEMM (csrc/gemm.cu) vs a plain PyTorch fp32 reference of the same op."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2602_09386_b200 import _lib
from paper_2602_09386_b200._lib import call, ptr


def _segments(loads, align=128):
    seg = [0]
    for n in loads:
        seg.append(seg[-1] + (n + align - 1) // align * align)
    return seg


def _packed(loads, d, gen, dev):
    seg = _segments(loads)
    x = torch.zeros(seg[-1] + 128, d, device=dev)
    for g, n in enumerate(loads):
        x[seg[g]:seg[g] + n] = torch.randn(n, d, generator=gen, device=dev)
    return seg, x


@pytest.mark.parametrize("N,K", [(256, 128), (128, 256), (512, 256), (96, 64), (64, 512)])
@pytest.mark.parametrize("act", [0, 1])
def test_ragged_m_forward(N, K, act):
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(N * 7 + K + act)
    loads = [300, 0, 129, 1, 128, 517]
    E = len(loads)
    seg, x = _packed(loads, K, g, dev)
    R = x.shape[0]
    xb = x.to(torch.bfloat16).contiguous()
    w = (torch.randn(E, N, K, generator=g, device=dev) / K ** 0.5).to(torch.bfloat16).contiguous()
    b = torch.randn(E, N, generator=g, device=dev).contiguous()
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    out = torch.full((R, N), float("nan"), device=dev).to(torch.bfloat16)
    bits = torch.zeros((N + 31) // 32, R, dtype=torch.int32, device=dev) if N % 32 == 0 and act else None
    call("smes_gemm_ragged_m", ptr(xb), K, R, ptr(w), E, N, K, 0, ptr(seg_t), ptr(b), act, ptr(bits), None, R,
         ptr(out), N, 0, R, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, n = seg[e], loads[e]
        if n == 0:
            continue
        ref = xb[lo:lo + n].float() @ w[e].float().T + b[e]
        if act:
            ref = ref.clamp_min(0)
        got = out[lo:lo + n].float()
        err = (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
        assert err < 1e-2, (e, err)
        if bits is not None:
            word = bits[:, lo:lo + n].T.contiguous()   # (n, N/32)
            expect = (ref.to(torch.bfloat16).float() > 0)
            for j in range(N // 32):
                m = ((word[:, j:j + 1].long() >> torch.arange(32, device=dev)) & 1).bool()
                assert torch.equal(m, expect[:, 32 * j:32 * j + 32])


def test_ragged_m_fp32_out_unaligned_rows():
    """Plain GEMM (router logits): 1 group, M not a multiple of 128, fp32 out, clipped store."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(3)
    M, N, K = 1000, 256, 256
    a = torch.randn(M, K, generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn(1, N, K, generator=g, device=dev) * 1e-3).to(torch.bfloat16)
    b = torch.randn(1, N, generator=g, device=dev)
    seg = torch.tensor([0, 1024], dtype=torch.int32, device=dev)
    out = torch.full((M + 24, N), 7.0, device=dev)
    call("smes_gemm_ragged_m", ptr(a), K, M, ptr(w), 1, N, K, 0, ptr(seg), ptr(b), 0, None, None, 0, ptr(out), N, 1,
         M, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = a.float() @ w[0].float().T + b[0]
    assert (out[:M] - ref).abs().max().item() <= 1e-5 * ref.abs().max().item() + 1e-6
    assert torch.all(out[M:] == 7.0)   # rows >= m_limit untouched


@pytest.mark.parametrize("N,K", [(256, 512), (128, 256)])
def test_ragged_m_dgrad_masked(N, K):
    """dgrad: C[m, n] = mask(sum_k A[m, k] W_g[k, n]) with W stored (G, K, N)."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(11 + N)
    loads = [200, 77, 0, 384]
    E = len(loads)
    seg, a = _packed(loads, K, g, dev)
    R = a.shape[0]
    ab = a.to(torch.bfloat16)
    w = (torch.randn(E, K, N, generator=g, device=dev) / K ** 0.5).to(torch.bfloat16)
    bits = torch.randint(-2 ** 31, 2 ** 31 - 1, (N // 32, R), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    out = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
    call("smes_gemm_ragged_m", ptr(ab), K, R, ptr(w), E, N, K, 1, ptr(seg_t), None, 0, None, ptr(bits), R, ptr(out),
         N, 0, R, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, n = seg[e], loads[e]
        if n == 0:
            continue
        ref = ab[lo:lo + n].float() @ w[e].float()
        word = bits[:, lo:lo + n].T.long()
        mask = torch.cat([((word[:, j:j + 1] >> torch.arange(32, device=dev)) & 1) for j in range(N // 32)], 1).bool()
        ref = torch.where(mask, ref, torch.zeros_like(ref))
        got = out[lo:lo + n].float()
        assert (got - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


@pytest.mark.parametrize("I,J", [(256, 512), (512, 256), (128, 128), (64, 256)])
def test_ragged_k_wgrad(I, J):
    """wgrad: C_g[i, j] = sum_{m in g} P[m, i] Q[m, j] (fp32), empty groups -> exact zeros."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(I + 3 * J)
    loads = [300, 0, 129, 640]
    E = len(loads)
    seg, pm = _packed(loads, I, g, dev)
    _, qm = _packed(loads, J, g, dev)
    R = pm.shape[0]
    pb, qb = pm.to(torch.bfloat16), qm.to(torch.bfloat16)
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    out = torch.full((E, I, J), float("nan"), device=dev)
    call("smes_gemm_ragged_k", ptr(pb), I, ptr(qb), J, R, E, I, J, ptr(seg_t), ptr(out), None,
         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, hi = seg[e], seg[e + 1]
        ref = pb[lo:hi].float().T @ qb[lo:hi].float()
        if loads[e] == 0:
            assert torch.all(out[e] == 0)
            continue
        err = (out[e] - ref).abs().max().item() / ref.abs().max().item()
        assert err < 1e-5, (e, err)


@pytest.mark.parametrize("I,J", [(256, 512), (512, 256), (128, 128)])
def test_ragged_k_wgrad_with_fused_bias(I, J):
    """db_g[i] = sum_m P[m, i] via the in-tile ones-tile MMA (Q's extra columns are ignored)."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(7 * I + J)
    loads = [200, 0, 77, 640]
    E = len(loads)
    seg, pm = _packed(loads, I, g, dev)
    _, qm = _packed(loads, J, g, dev)
    R = pm.shape[0]
    pb = pm.to(torch.bfloat16)
    qb = torch.zeros(R, J + 64, dtype=torch.bfloat16, device=dev)
    qb[:, :J] = qm.to(torch.bfloat16)
    qb[:, J] = 1.0
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    out = torch.full((E, I, J), float("nan"), device=dev)
    db = torch.full((E, I), float("nan"), device=dev)
    call("smes_gemm_ragged_k", ptr(pb), I, ptr(qb), J + 64, R, E, I, J, ptr(seg_t), ptr(out), ptr(db),
         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, hi = seg[e], seg[e + 1]
        ref = pb[lo:hi].float().T @ qb[lo:hi, :J].float()
        refb = pb[lo:hi].float().sum(0)
        if loads[e] == 0:
            assert torch.all(out[e] == 0) and torch.all(db[e] == 0)
            continue
        assert (out[e] - ref).abs().max().item() / ref.abs().max().item() < 1e-5
        assert (db[e] - refb).abs().max().item() / refb.abs().max().item() < 1e-5


@pytest.mark.parametrize("N,K", [(8, 512), (16, 256), (32, 128)])
def test_ragged_m_narrow_fp32(N, K):
    """N <= 32 fp32-out tile (folded head projections P = H G_e^T + c_e)."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(5 * N + K)
    loads = [300, 0, 129, 1, 517]
    E = len(loads)
    seg, x = _packed(loads, K, g, dev)
    R = x.shape[0]
    xb = x.to(torch.bfloat16).contiguous()
    w = (torch.randn(E, N, K, generator=g, device=dev) / K ** 0.5).to(torch.bfloat16).contiguous()
    b = torch.randn(E, N, generator=g, device=dev).contiguous()
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    out = torch.full((R, N), float("nan"), device=dev)
    call("smes_gemm_ragged_m", ptr(xb), K, R, ptr(w), E, N, K, 0, ptr(seg_t), ptr(b), 0, None, None, 0,
         ptr(out), N, 1, R, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, n = seg[e], loads[e]
        if n == 0:
            continue
        ref = xb[lo:lo + n].float() @ w[e].float().T + b[e]
        err = (out[lo:lo + n] - ref).abs().max().item() / ref.abs().max().item()
        assert err < 1e-5, (e, err)


@pytest.mark.parametrize("K,N", [(8, 512), (16, 256), (8, 128)])
def test_ragged_m_dgrad_small_k_masked(K, N):
    """K = T dgrad of the folded heads: C[m, n] = mask(sum_t A[m, t] G_g[t, n]), A with a wider ld."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(K + N)
    loads = [200, 0, 77, 384]
    E = len(loads)
    lda = 16
    seg, a = _packed(loads, lda, g, dev)
    a[:, K:] = 0
    R = a.shape[0]
    ab = a.to(torch.bfloat16).contiguous()
    w = (torch.randn(E, K, N, generator=g, device=dev)).to(torch.bfloat16).contiguous()
    bits = torch.randint(-2 ** 31, 2 ** 31 - 1, (N // 32, R), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    out = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
    call("smes_gemm_ragged_m", ptr(ab), lda, R, ptr(w), E, N, K, 1, ptr(seg_t), None, 0, None, ptr(bits), R,
         ptr(out), N, 0, R, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, n = seg[e], loads[e]
        if n == 0:
            continue
        ref = ab[lo:lo + n, :K].float() @ w[e].float()
        word = bits[:, lo:lo + n].T.long()
        mask = torch.cat([((word[:, j:j + 1] >> torch.arange(32, device=dev)) & 1) for j in range(N // 32)], 1).bool()
        ref = torch.where(mask, ref, torch.zeros_like(ref))
        assert (out[lo:lo + n].float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


@pytest.mark.parametrize("I,J", [(512, 8), (256, 16), (513, 8)])
def test_ragged_k_wgrad_narrow(I, J):
    """Folded wgrad Qt_g[i, t] = sum_{m in g} H[m, i] C[m, t] with J = T <= 16 (BN = 16 tile);
    I = d + 1 reads the ones column of H (per-expert sums of C)."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(I + J)
    loads = [300, 0, 129, 640]
    E = len(loads)
    ldp = (I + 63) // 64 * 64
    seg, pm = _packed(loads, ldp, g, dev)
    _, qm = _packed(loads, 16, g, dev)
    qm[:, J:] = 0
    R = pm.shape[0]
    pb, qb = pm.to(torch.bfloat16).contiguous(), qm.to(torch.bfloat16).contiguous()
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    out = torch.full((E, I, J), float("nan"), device=dev)
    call("smes_gemm_ragged_k", ptr(pb), ldp, ptr(qb), 16, R, E, I, J, ptr(seg_t), ptr(out), None,
         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, hi = seg[e], seg[e + 1]
        ref = pb[lo:hi, :I].float().T @ qb[lo:hi, :J].float()
        if loads[e] == 0:
            assert torch.all(out[e] == 0)
            continue
        assert (out[e] - ref).abs().max().item() / ref.abs().max().item() < 1e-5


@pytest.mark.parametrize("N,K,b_mn,act,f32", [(1024, 512, 0, 1, 0), (512, 1024, 1, 0, 0), (256, 256, 0, 0, 1),
                                              (768, 256, 1, 0, 1)])
def test_ragged_m_cta_pairs(N, K, b_mn, act, f32):
    """The CTA-pair kernel (cta_group::2, taken for N % 256 == 0, K >= 256 and >= 64 K rows): odd
    and even tile counts per group (a pair's second tile empty), empty groups, bias + relu + mask
    (forward), the relu mask applied to the output (dgrad, MN-major B), bf16 and fp32 outputs."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(N + K + b_mn)
    loads = [20000, 0, 129, 17000, 128, 30517, 1]          # 157, 0, 2, 133, 1, 239, 1 tiles
    E = len(loads)
    seg, x = _packed(loads, K, g, dev)
    R = x.shape[0]
    assert R >= 64 * 1024
    xb = x.to(torch.bfloat16).contiguous()
    if b_mn:
        w = (torch.randn(E, K, N, generator=g, device=dev) / K ** 0.5).to(torch.bfloat16).contiguous()
        weff = w.float()                                      # (E, K, N): out = x w
    else:
        w = (torch.randn(E, N, K, generator=g, device=dev) / K ** 0.5).to(torch.bfloat16).contiguous()
        weff = w.float().transpose(1, 2)
    b = torch.randn(E, N, generator=g, device=dev).contiguous() if not b_mn else None
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    odt = torch.float32 if f32 else torch.bfloat16
    out = torch.full((R, N), float("nan"), device=dev).to(odt)
    bits_out = torch.zeros(N // 32, R, dtype=torch.int32, device=dev) if act else None
    mask_in = torch.randint(0, 2 ** 31, (N // 32, R), generator=g, device=dev, dtype=torch.int32) if b_mn else None
    call("smes_gemm_ragged_m", ptr(xb), K, R, ptr(w), E, N, K, b_mn, ptr(seg_t), ptr(b), act, ptr(bits_out),
         ptr(mask_in), R, ptr(out), N, int(f32), R, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, n = seg[e], loads[e]
        if n == 0:
            continue
        ref = xb[lo:lo + n].float() @ weff[e]
        if b is not None:
            ref = ref + b[e]
        if act:
            ref = ref.clamp_min(0)
        if mask_in is not None:
            m = ((mask_in[:, lo:lo + n].T.long().unsqueeze(2) >> torch.arange(32, device=dev)) & 1).reshape(n, N)
            ref = ref * m
        got = out[lo:lo + n].float()
        err = (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
        assert err < 1e-2, (e, err)
        if bits_out is not None:
            word = bits_out[:, lo:lo + n].T.contiguous()
            expect = got > 0
            for j in range(N // 32):
                mm = ((word[:, j:j + 1].long() >> torch.arange(32, device=dev)) & 1).bool()
                assert torch.equal(mm, expect[:, 32 * j:32 * j + 32])


@pytest.mark.parametrize("I,J,bias", [(1024, 576, True), (384, 320, True), (512, 256, False)])
def test_ragged_k_wgrad_cta_pairs(I, J, bias, monkeypatch):
    """The CTA-pair wgrad (SMES_GEMM_PAIR_K=1; I >= 256, J >= 256 and >= 64 K rows): i-tile pairs with an empty
    second tile (I = 384), partial j tiles (J = 576, 320), empty groups, the fused bias column."""
    monkeypatch.setenv("SMES_GEMM_PAIR_K", "1")
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(11 * I + J)
    loads = [30000, 0, 77, 36000, 128, 1]
    E = len(loads)
    seg, pm = _packed(loads, I, g, dev)
    _, qm = _packed(loads, J, g, dev)
    R = pm.shape[0]
    assert R >= 64 * 1024
    pb = pm.to(torch.bfloat16)
    qb = torch.zeros(R, J + 64, dtype=torch.bfloat16, device=dev)
    qb[:, :J] = qm.to(torch.bfloat16)
    qb[:, J] = 1.0
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    out = torch.full((E, I, J), float("nan"), device=dev)
    db = torch.full((E, I), float("nan"), device=dev) if bias else None
    call("smes_gemm_ragged_k", ptr(pb), I, ptr(qb), J + 64, R, E, I, J, ptr(seg_t), ptr(out), ptr(db),
         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for e in range(E):
        lo, hi = seg[e], seg[e + 1]
        ref = pb[lo:hi].float().T @ qb[lo:hi, :J].float()
        if loads[e] == 0:
            assert torch.all(out[e] == 0)
            if bias:
                assert torch.all(db[e] == 0)
            continue
        # fp32 accumulation over up to 36 K rows: ~1e-4 of the largest entry (the single-CTA kernel
        # gives the same error on these operands)
        assert (out[e] - ref).abs().max().item() / ref.abs().max().item() < 3e-4, e
        if bias:
            refb = pb[lo:hi].float().sum(0)
            assert (db[e] - refb).abs().max().item() / refb.abs().max().item() < 3e-4, e


@pytest.mark.parametrize("nparts,n", [(1, 4096), (2, 8 * 1024 * 1024), (3, 1028), (8, 4096), (9, 4096),
                                      (64, 65536), (2, 1001)])
def test_part_reduce_split_k_partials(nparts, n):
    """smes_part_reduce (the split-K partial sum of the router / head weight gradients): the
    few-partials float4 path (nparts <= 8, n % 4 == 0) and the column-block path, against torch."""
    g = torch.Generator(device="cuda").manual_seed(nparts * 31 + n)
    part = torch.randn(nparts, n, generator=g, device="cuda")
    out = torch.full((n,), float("nan"), device="cuda")
    call("smes_part_reduce", ptr(part), nparts, n, ptr(out), torch.cuda.current_stream().cuda_stream)
    ref = part.double().sum(0)
    assert torch.allclose(out.double(), ref, rtol=1e-5, atol=1e-5 * nparts)
    if nparts == 1:
        assert torch.equal(out, part[0])


@pytest.mark.parametrize("J,I", [(256, 512), (128, 256), (64, 64)])
def test_ragged_k_gather_matches_packed(J, I):
    """smes_gemm_ragged_k_gather (Q rows by TMA gather4 from their source rows, -1 = zero row)
    equals the packed ragged-K GEMM bit for bit, bias sums included."""
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(J + I)
    loads = [300, 0, 129, 1, 700, 64]
    G = len(loads)
    seg, Pm = _packed(loads, I, g, dev)
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    R = Pm.shape[0]
    Pb = Pm.to(torch.bfloat16)
    n = sum(loads)
    cg = torch.Generator(device="cpu").manual_seed(I)
    perm = torch.randperm(n + 5, generator=cg)[:n]
    src = torch.randn(n + 5, J + 64, generator=cg).to(torch.bfloat16).to(dev)
    gather = torch.full((R,), -1, dtype=torch.int32)
    k = 0
    for e, m in enumerate(loads):
        for i in range(m):
            gather[seg[e] + i] = int(perm[k])
            k += 1
    gather = gather.to(dev)
    Q = torch.zeros(R, J + 64, dtype=torch.bfloat16, device=dev)
    real = gather >= 0
    Q[real] = src[gather[real].long()]
    st = torch.cuda.current_stream().cuda_stream
    C0 = torch.full((G, I, J), float("nan"), device=dev)
    C1 = torch.full((G, I, J), float("nan"), device=dev)
    d0 = torch.full((G, I), float("nan"), device=dev)
    d1 = torch.full((G, I), float("nan"), device=dev)
    call("smes_gemm_ragged_k", ptr(Pb), I, ptr(Q), J + 64, R, G, I, J, ptr(seg_t), ptr(C0), ptr(d0), st)
    call("smes_gemm_ragged_k_gather", ptr(Pb), I, ptr(src), J + 64, src.shape[0], ptr(gather), R, G, I, J,
         ptr(seg_t), ptr(C1), ptr(d1), st)
    torch.cuda.synchronize()
    assert torch.equal(C0, C1)
    assert torch.equal(d0, d1)
    ref = torch.stack([Pb[seg[e]:seg[e + 1]].float().T @ Q[seg[e]:seg[e + 1], :J].float() for e in range(G)])
    assert torch.allclose(C1, ref, rtol=1e-3, atol=1e-3)
