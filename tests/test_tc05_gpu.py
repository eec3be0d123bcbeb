"""tcgen05 prefill GEMM (csrc/gemm_tc05.cu) vs float64.

Bar: |C - C64| <= 2e-6 * (|A| @ |W|) elementwise (f32-level: the split keeps
22 significand bits per operand), ragged M / N / K, all epilogues, a
multi-tile persistent schedule; the split's hi + lo reconstructs x within
2^-22 relative."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2406_19707_b200 import _lib
    _lib.load()


def test_split_roundtrip():
    import torch
    from paper_2406_19707_b200 import tcgemm
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    X = torch.randn(37, 100, device="cuda", generator=g) * torch.logspace(-6, 6, 100, device="cuda")
    X[5] = 0
    A = tcgemm.split_rows(X)
    hi = A.hl[:, :100].double()
    lo = A.hl[:, A.Kp:A.Kp + 100].double()
    rec = (hi + lo) * A.inv_scale.double()[:, None]
    amax = X.abs().amax(dim=1, keepdim=True).double()
    assert ((rec - X.double()).abs() <= amax * 2.0 ** -22 + 1e-30).all()
    assert (A.hl[:, 100:A.Kp] == 0).all() and (A.hl[:, A.Kp + 100:] == 0).all()
    W = torch.randn(100, 70, device="cuda", generator=g)
    B = tcgemm.split_weight(W)
    rec = (B.hl[:, :100].double() + B.hl[:, B.Kp:B.Kp + 100].double()) * B.inv_scale.double()[:, None]
    torch.testing.assert_close(rec, W.t().double(), rtol=2.0 ** -21, atol=0)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (200, 300, 100), (1024, 1536, 768),
                                   (513, 2304, 5120), (4096, 640, 5120), (96, 20480, 512),
                                   (256, 512, 20480)])
@pytest.mark.parametrize("epilogue", [0, 1, 2])
def test_gemm_tc05_vs_float64(M, N, K, epilogue):
    """f32-level error vs float64: max over elements of |err| / (|A| @ |W|)
    below 3e-6 (~50 f32 ulps; IEEE-f32 cuBLAS on the same operands: 0.05-1.4e-6,
    printed).  What is left is the tensor core's truncating accumulation of
    the hi.hi term (K / 16 steps)."""
    import torch
    from paper_2406_19707_b200 import tcgemm
    g = torch.Generator(device="cuda")
    g.manual_seed(M + 7 * N + 13 * K + epilogue)
    X = torch.randn(M, K, device="cuda", generator=g)
    X[:, :3] *= 40.0                                   # outlier channels
    W = torch.randn(K, N, device="cuda", generator=g) / K ** 0.5
    R = torch.randn(M, N, device="cuda", generator=g)
    out = tcgemm.matmul(X, W, epilogue=epilogue, R=R if epilogue == 2 else None)
    ref = X.double() @ W.double()
    mag = X.double().abs() @ W.double().abs()
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    f32 = X @ W
    torch.backends.cuda.matmul.allow_tf32 = old
    f32_rel = float(((f32.double() - ref).abs() / mag).max())
    if epilogue == 1:
        ref = ref.clamp_min(0)
    elif epilogue == 2:
        ref = ref + R.double()
        mag = mag + R.double().abs()
    rel = float(((out.double() - ref).abs() / mag).max())
    print(f"M{M} N{N} K{K} e{epilogue}: tc05 {rel:.3g}  cublas-f32 {f32_rel:.3g}")
    assert torch.isfinite(out).all()
    assert rel < 3e-6, (rel, f32_rel)
    again = tcgemm.matmul(X, W, epilogue=epilogue, R=R if epilogue == 2 else None)
    assert torch.equal(out, again)                     # deterministic


def test_gemm_tc05_few_ctas():
    """More tiles than CTAs: every CTA loops over several tiles (accumulator
    double buffering, ring phases across tiles)."""
    import torch
    from paper_2406_19707_b200 import tcgemm
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    X = torch.randn(1000, 640, device="cuda", generator=g)
    W = torch.randn(640, 1100, device="cuda", generator=g)
    A, B = tcgemm.split_rows(X), tcgemm.split_weight(W)
    ref = X.double() @ W.double()
    mag = X.double().abs() @ W.double().abs()
    first = tcgemm.gemm(A, B)
    assert float(((first.double() - ref).abs() / mag).max()) < 3e-6
    for ctas in (1, 3, 7):
        assert torch.equal(tcgemm.gemm(A, B, max_ctas=ctas), first), ctas


def _prefill_attention(qkv, nb, N, Hg, d):
    import ctypes
    import torch
    from paper_2406_19707_b200 import _lib
    sz = ctypes.c_size_t()
    _lib.call("ig_prefill_attention_scratch", nb, N, Hg, d, ctypes.byref(sz), kernels=0)
    work = torch.empty(sz.value, dtype=torch.uint8, device="cuda")
    out = torch.full((nb * N, Hg * d), float("nan"), device="cuda")
    _lib.call("ig_prefill_attention", qkv.data_ptr(), qkv.stride(0), nb, N, Hg, d, work.data_ptr(), out.data_ptr(),
              out.stride(0), _lib.stream_handle())
    return out


@pytest.mark.parametrize("nb,N,Hg,d", [(2, 200, 2, 128), (1, 1, 1, 128), (3, 129, 3, 64), (1, 700, 2, 64),
                                       (2, 1000, 1, 128)])
def test_prefill_attention_tc05_vs_float64(nb, N, Hg, d):
    """ig_prefill_attention (csrc/prefill_attn.cu: two-pass causal attention on
    tcgen05 with exact f16 hi/lo splits) vs float64 causal softmax attention
    (model.py:156-180, causal): ragged query / key tiles, a single token, d 64
    and 128, several sequences and heads; deterministic."""
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(nb * 1000 + N + Hg + d)
    qkv = torch.randn(nb * N, 3 * Hg * d, device="cuda", generator=g) * 2
    out = _prefill_attention(qkv, nb, N, Hg, d)
    again = _prefill_attention(qkv, nb, N, Hg, d)
    assert torch.equal(out, again)
    x = qkv.double().view(nb, N, 3, Hg, d)
    q, k, v = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))          # nb, Hg, N, d
    s = q @ k.transpose(-1, -2) / float(torch.tensor(d, dtype=torch.float32).sqrt())
    mask = torch.ones(N, N, dtype=torch.bool, device="cuda").tril()
    s = s.masked_fill(~mask, float("-inf"))
    ref = torch.softmax(s, dim=-1) @ v                                      # nb, Hg, N, d
    ref = ref.permute(0, 2, 1, 3).reshape(nb * N, Hg * d)
    err = float((out.double() - ref).abs().max())
    # IEEE-f32 attention on the same inputs (torch math path) as the yardstick
    xf = qkv.view(nb, N, 3, Hg, d)
    qf, kf, vf = (xf[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    sf = (qf @ kf.transpose(-1, -2)) / torch.tensor(d, dtype=torch.float32).sqrt()
    sf = sf.masked_fill(~mask, float("-inf"))
    f32 = (torch.softmax(sf, dim=-1) @ vf).permute(0, 2, 1, 3).reshape(nb * N, Hg * d)
    f32_err = float((f32.double() - ref).abs().max())
    print(f"prefill attention nb{nb} N{N} Hg{Hg} d{d}: tc05 {err:.3g}  f32 {f32_err:.3g}")
    assert torch.isfinite(out).all()
    assert err < max(4 * f32_err, 1e-6), (err, f32_err)
