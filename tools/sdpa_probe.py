import torch, time
import torch.nn.functional as F
from torch.nn.attention import sdpa_kernel, SDPBackend
H, N, d = 40, 4096, 128
q, k, v = (torch.randn(H, N, d, device="cuda") for _ in range(3))
def run(backends, blocked):
    with sdpa_kernel(backends):
        if not blocked:
            return F.scaled_dot_product_attention(q, k, v, is_causal=True)
        out = torch.empty_like(q)
        for r0 in range(0, N, 2048):
            r1 = min(N, r0 + 2048)
            mask = torch.ones(r1 - r0, r1, dtype=torch.bool, device=q.device).tril(r0)
            out[..., r0:r1, :] = F.scaled_dot_product_attention(q[..., r0:r1, :], k[..., :r1, :], v[..., :r1, :], attn_mask=mask)
        return out
ref = run([SDPBackend.MATH], True).double()
exact = None
for name, be, blocked in (("math_blocked", [SDPBackend.MATH], True), ("efficient_causal", [SDPBackend.EFFICIENT_ATTENTION], False),
                          ("efficient_blocked", [SDPBackend.EFFICIENT_ATTENTION], True), ("cudnn_causal", [SDPBackend.CUDNN_ATTENTION], False)):
    try:
        o = run(be, blocked); torch.cuda.synchronize()
        t = time.time()
        for _ in range(3): o = run(be, blocked)
        torch.cuda.synchronize()
        ms = (time.time() - t) / 3 * 1e3
        err = float((o.double() - ref).abs().max())
        print(name, round(ms, 1), "ms", "maxerr vs math", err, flush=True)
    except Exception as e:
        print(name, "failed", repr(e)[:200], flush=True)
