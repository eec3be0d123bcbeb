"""The fixture configurations of tests/golden/make_golden.py, in oracle terms."""

from oracle import speckv_port as O

MODELS = {
    "m64": O.ModelSpec(layers=3, model_dim=64, heads=4, ffn_dim=256, outlier_channels=8,
                       outlier_scale=2.0, seed=0),
    "m256": O.ModelSpec(layers=3, model_dim=256, heads=2, ffn_dim=1024, outlier_channels=8,
                        outlier_scale=2.0, seed=3),
}

RUNS = {
    "spec": dict(scheme="speculative", prompt_len=48, gen_len=6, batch=2),
    "spec_counter": dict(scheme="speculative", prompt_len=40, gen_len=12, batch=1,
                         pool_limit=int(0.8 * 52), pool_policy=O.Policy.COUNTER),
    "spec_lru": dict(scheme="speculative", prompt_len=40, gen_len=12, batch=1, pool_limit=36,
                     pool_policy=O.Policy.LRU),
    "spec_fifo": dict(scheme="speculative", prompt_len=40, gen_len=12, batch=1, pool_limit=36,
                      pool_policy=O.Policy.FIFO),
    "spec_alpha2_cap05": dict(scheme="speculative", prompt_len=64, gen_len=5, batch=1,
                              speculation=O.SpeculationConfig(0.3, 2.0, 0.5, 1)),
    "spec_identity": dict(scheme="speculative", prompt_len=32, gen_len=4, batch=1,
                          speculation=O.SpeculationConfig(0.3, 1e9, 1.0, 1)),
    "full": dict(scheme="full", prompt_len=32, gen_len=4, batch=1),
}

_cache = {}


def models(name):
    """(plain, skewed) oracle models, cached per session."""
    if name not in _cache:
        plain = O.generate_synthetic(MODELS[name])
        _cache[name] = (plain, O.skew_model(plain, calib_seed=0))
    return _cache[name]


def run_config(rname, **extra):
    kw = dict(RUNS[rname])
    kw.update(extra)
    return O.RunConfig(**kw)
