"""Model description the decode path consumes, plus GPU-side fixture builders.

The engine accepts any object shaped like the reference ``Model``
(reference model.py:33-105): ``.spec`` with layers / model_dim / heads /
ffn_dim / ln_eps, ``.layers`` of objects with the ten LayerWeights fields
(model.py:63-79, x @ W convention, float32), and ``.skewed``.  So a model
built, skewed and saved by the reference (or loaded with ``load_model``
below from its manifest format) drops straight in.

``generate_synthetic_gpu`` / ``skew_model_gpu`` rebuild the reference recipes
(model.py:108-153, skewing.py:30-104) on the GPU for shapes whose CPU build
would take hours (OPT-13B: 12.6 G weights).  They use torch's RNG, so the
weights are distributed like the reference's, not bit-identical to them;
bench.py says so in its "data" field.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

import numpy as np

LAYER_FIELDS = ("w_q", "w_k", "w_v", "w_o", "ffn_in", "ffn_out",
                "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")
OUTLIER_FEEDBACK = 1.5  # reference model.py:22


@dataclass(frozen=True)
class ModelSpec:
    """Reference ModelSpec (model.py:33-60)."""
    layers: int
    model_dim: int
    heads: int
    ffn_dim: int
    ln_eps: float = 1e-5
    outlier_channels: int = 0
    outlier_scale: float = 1.0
    seed: int = 0

    @property
    def head_dim(self) -> int:
        return self.model_dim // self.heads

    def validate(self) -> None:
        if self.layers < 1:
            raise ValueError("layers must be >= 1")
        if self.heads < 1 or self.model_dim % self.heads != 0:
            raise ValueError("model_dim must be a positive multiple of heads")
        if self.ffn_dim < 1:
            raise ValueError("ffn_dim must be >= 1")
        if self.ln_eps <= 0:
            raise ValueError("ln_eps must be positive")


class LayerWeights:
    """Ten-field layer (model.py:63-79); arrays may be numpy or torch."""

    def __init__(self, **kw):
        for f in LAYER_FIELDS:
            setattr(self, f, kw[f])


class Model:
    def __init__(self, spec: ModelSpec, layers: list, skewed: bool = False,
                 outlier_indices=None):
        self.spec = spec
        self.layers = layers
        self.skewed = skewed
        self.outlier_indices = outlier_indices


# shapes of the BASELINE.json configs
SHAPES = {
    "opt-125m": dict(layers=12, model_dim=768, heads=12, ffn_dim=3072),
    "opt-6.7b": dict(layers=32, model_dim=4096, heads=32, ffn_dim=16384),
    "opt-13b": dict(layers=40, model_dim=5120, heads=40, ffn_dim=20480),
    "llama-2-7b": dict(layers=32, model_dim=4096, heads=32, ffn_dim=11008),
    "opt-30b": dict(layers=48, model_dim=7168, heads=56, ffn_dim=28672),
}


def load_model(path: str) -> Model:
    """Read the reference's manifest + raw <f4 payload format (model.py:284-409)."""
    with open(path, "r", encoding="utf-8") as f:
        man = json.load(f)
    sp = man["spec"]
    spec = ModelSpec(int(sp["layers"]), int(sp["model_dim"]), int(sp["heads"]),
                     int(sp["ffn_dim"]), float(sp["ln_eps"]), int(sp["outlier_channels"]),
                     float(sp["outlier_scale"]), int(sp["seed"]))
    spec.validate()
    blob = np.fromfile(os.path.join(os.path.dirname(path) or ".", man["payload"]), dtype=np.uint8)
    table = {}
    for e in man["tensors"]:
        off, nb = int(e["offset"]), int(e["nbytes"])
        shape = tuple(int(s) for s in e["shape"])
        if off + nb > blob.size:
            raise ValueError(f"payload truncated at tensor {e['name']!r}")
        table[e["name"]] = blob[off:off + nb].view("<f4").reshape(shape).astype(np.float32)
    layers = [LayerWeights(**{f: table[f"layer.{i}.{f}"] for f in LAYER_FIELDS})
              for i in range(spec.layers)]
    return Model(spec, layers, bool(man.get("skewed", False)),
                 table.get("outlier_indices", np.zeros(0, np.float32)).astype(np.int64))


def generate_synthetic_gpu(spec: ModelSpec, device="cuda", seed: int | None = None) -> Model:
    """The reference recipe (model.py:108-153) on the GPU with torch's RNG:
    iid N(0,1)/sqrt(fan_in) projections, LN gains 1+0.02N, biases 0.02N,
    outlier channels' LN gains x outlier_scale, and the rectified FFN
    write-back of 1.5*(scale-1) through hidden unit (j mod ffn_dim)."""
    import torch
    spec.validate()
    g = torch.Generator(device=device)
    g.manual_seed(spec.seed if seed is None else seed)
    D, F = spec.model_dim, spec.ffn_dim
    perm = torch.randperm(D, generator=g, device=device)[: spec.outlier_channels]
    picks = torch.sort(perm).values
    fb = OUTLIER_FEEDBACK * (spec.outlier_scale - 1.0)

    def dense(r, c, fan):
        w = torch.empty(r, c, device=device, dtype=torch.float32)
        w.normal_(generator=g)
        return w.mul_(1.0 / math.sqrt(fan))

    def vec(base):
        v = torch.empty(D, device=device, dtype=torch.float32).normal_(generator=g)
        return v.mul_(0.02).add_(base)

    layers = []
    for _ in range(spec.layers):
        wq, wk, wv, wo = (dense(D, D, D) for _ in range(4))
        fi, fo = dense(D, F, D), dense(F, D, F)
        g1, b1, g2, b2 = vec(1.0), vec(0.0), vec(1.0), vec(0.0)
        g1[picks] *= spec.outlier_scale
        g2[picks] *= spec.outlier_scale
        if fb > 0:
            hid = picks % F
            fi[picks, hid] += fb
            fo[hid, picks] += fb
        layers.append(LayerWeights(w_q=wq, w_k=wk, w_v=wv, w_o=wo, ffn_in=fi, ffn_out=fo,
                                   ln1_gain=g1, ln1_bias=b1, ln2_gain=g2, ln2_bias=b2))
    return Model(spec, layers, False, picks.cpu().numpy())


def skew_model_gpu(model: Model, calib_tokens: int | None = None, seed: int = 0,
                   calib_input=None, forward_dtype=None) -> Model:
    """Offline skew (skewing.py:30-104) on the GPU, in place: forward a
    seeded 4*d-row calibration prompt, SVD each head's Q (f64), take A = V with
    the max-|entry|-positive sign rule (skewing.py:59-66), fold A into the
    W_Q / W_K head slices.  The blocks are kept as model.skew_matrices
    ([L][H] d x d, f64 numpy) with their singular values (model.skew_sigmas),
    like the reference's SkewSet (skewing.py:14-27).  forward_dtype=float64
    runs the calibration forward in f64 (the oracle's q are f32 NumPy)."""
    import torch
    from . import prefill as _pf
    spec = model.spec
    d = spec.head_dim
    n = calib_tokens if calib_tokens is not None else 4 * d
    dev = model.layers[0].w_q.device
    if calib_input is not None:        # e.g. the reference's random_prompt(4d, D, seed)
        x = calib_input.to(device=dev, dtype=torch.float32)
    else:
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        x = torch.empty(max(n, 2), spec.model_dim, device=dev).normal_(generator=g)
    mats, sigmas = [], []
    for lw in model.layers:
        if forward_dtype is not None and forward_dtype != torch.float32:
            lw64 = type(lw)(**{f: getattr(lw, f).to(forward_dtype) for f in LAYER_FIELDS})
            out, q = _pf.dense_block_forward(x.to(forward_dtype), lw64, spec)
            out = out.float()
        else:
            out, q = _pf.dense_block_forward(x, lw, spec)
        qh = q.view(q.shape[0], spec.heads, d).permute(1, 0, 2).double()  # H x n x d
        _, sv, vh = torch.linalg.svd(qh, full_matrices=False)
        a = vh.transpose(1, 2)                                           # H x d x d (= V)
        piv = a.abs().argmax(dim=1, keepdim=True)
        sign = torch.sign(torch.gather(a, 1, piv))
        sign[sign == 0] = 1
        a = a * sign
        mats.append(a.cpu().numpy())
        sigmas.append(sv.cpu().numpy())
        a = a.float()
        for which in ("w_q", "w_k"):
            w = getattr(lw, which).view(spec.model_dim, spec.heads, d)
            w.copy_(torch.einsum("Dhi,hij->Dhj", w, a))
        x = out
    model.skewed = True
    model.skew_matrices = mats
    model.skew_sigmas = sigmas
    return model
