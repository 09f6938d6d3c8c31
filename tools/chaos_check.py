"""Strict teacher-forced check of one config on the fp32 engine (band64) and the
fp64 engine (reference operation order): worst error / tolerance among envs
with |theta_in| <= 1.4, and the count outside."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2410_14117_b200 as uuv  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from tests import parity as P  # noqa: E402
from tests.test_gpu_parity import CONFIGS, _cfg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "station_20sub_target"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
for prec in ("fp32", "fp64"):
    kw = dict(CONFIGS[name]); kw["n"] = n
    cfg = _cfg(precision=prec, **kw)
    gpu = uuv.B200EnvBatch(cfg)
    ref = orc.OracleBatch(cfg, threads=0)
    act = orc.bench_actions(cfg["seed"], n, ref.action_dim)
    for _ in range(300):
        gpu.step_ex(act); ref.step(act)
    worst, nout = 0.0, 0
    for t in range(24):
        s = P.f32(ref.states())
        ref.set_states(s); gpu.set_states(s); gpu.set_step_counts(ref.step_counts())
        gpu.step_ex(act); _, rr, dr, _ = ref.step(act, with_reason=True)
        sr, sg = ref.states(), gpu.states()
        live = (np.abs(s[:, 4]) <= 1.4) & ~dr & (np.abs(-rr - 10.0) >= 1e-4)
        sc = P.abs_err(sg[live], sr[live], P.STATE_ANGLES) / (P.ABS_TOL + P.REL_TOL * np.abs(sr[live]))
        if sc.size:
            worst = max(worst, float(sc.max())); nout += int((sc > 1).any(axis=1).sum())
        print(t, int(live.sum()), flush=True) if not sc.size else None
    print(name, prec, "worst err/tol", round(worst, 3), "env-steps outside", nout, flush=True)
