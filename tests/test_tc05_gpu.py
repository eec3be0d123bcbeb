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
