"""Drive every path kernel once at a small size, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_path.py
    compute-sanitizer --tool racecheck python tools/sanitize_path.py
    compute-sanitizer --tool synccheck python tools/sanitize_path.py

Engine decode on a 3-layer D=256 / d=128 model (the 512-B-row tensor-core
attention, both GEMMs, rehearse/select/plan/fetch/append) in resident and
refetch modes with f16 and f32 pools, plus a pool-limit run (eviction)."""
import copy
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    from oracle import speckv_port as O
    import paper_2406_19707_b200 as G
    spec = O.ModelSpec(layers=3, model_dim=256, heads=2, ffn_dim=1024, outlier_channels=8,
                       outlier_scale=2.0, seed=3)
    sk = O.skew_model(O.generate_synthetic(spec), calib_seed=0)
    for limit in (None, 44):
        ocfg = O.RunConfig(scheme="speculative", prompt_len=40, gen_len=4, batch=2, pool_limit=limit)
        sessions = [O.Session(sk, ocfg, O.random_prompt(40, 256, b)) for b in range(2)]
        for pool in ("f16", "f32"):
            for resident in (True, False):
                for dense in ("tc", "ig"):
                    cfg = G.RunConfig(scheme="speculative", prompt_len=40, gen_len=4, batch=2,
                                      pool_limit=limit)
                    eng = G.DecodeEngine.from_sessions(sk, cfg, copy.deepcopy(sessions), pool_dtype=pool,
                                                       resident=resident, dense=dense)
                    try:
                        for _ in range(4):
                            out = eng.decode_step()
                        assert np.all(np.isfinite(out.cpu().numpy()))
                    finally:
                        eng.close()
    print("sanitize_path: all configurations ran")


if __name__ == "__main__":
    main()
