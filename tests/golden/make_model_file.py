"""Write a tiny skewed model with the REAL reference's save_model (manifest +
raw <f4 payload, model.py:284-332) for the load_model parity test.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_model_file.py
"""
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from speckv import model, skewing  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
spec = model.ModelSpec(layers=2, model_dim=32, heads=2, ffn_dim=64, outlier_channels=4,
                       outlier_scale=2.0, seed=5)
sk, _ = skewing.skew_model(model.generate_synthetic(spec), calib_seed=1)
model.save_model(sk, os.path.join(OUT, "tiny_skewed.json"))
print("wrote", os.path.join(OUT, "tiny_skewed.json"))
