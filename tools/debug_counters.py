import copy, sys
import numpy as np
sys.path.insert(0, '.')
from oracle import speckv_port as O
from tests.golden_cfg import models, run_config
from tests.test_engine_gpu import engine_cfg, oracle_sessions
from paper_2406_19707_b200 import DecodeEngine
plain, sk = models("m64")
for rname, model in (("full", plain), ("spec", sk)):
    ocfg = run_config(rname, record_selection=True, batch=1)
    sessions = oracle_sessions(model, ocfg)
    eng = DecodeEngine.from_sessions(model, engine_cfg(ocfg), copy.deepcopy(sessions), pool_dtype="f32")
    print(rname, "init", eng.counter[0, 0, 0, :6].cpu().numpy(), eng.counter[1, 0, 0, :6].cpu().numpy())
    for t in range(3):
        eng.decode_step()
        for s in sessions: s.decode_step()
        print(rname, t, "L0", eng.counter[0, 0, 0, :6].cpu().numpy(), sessions[0].pools[0][0].fetch_counter[:6],
              "L1", eng.counter[1, 0, 0, :6].cpu().numpy(), sessions[0].pools[1][0].fetch_counter[:6],
              "lf", eng.lastf[0, 0, 0, :3].cpu().numpy(), sessions[0].pools[0][0].last_fetch_seq[:3])
