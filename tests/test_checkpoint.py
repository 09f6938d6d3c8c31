"""UUVSIMP1 policy checkpoints: round trip, error cases, and interchange with the
reference's own numpy Policy (pkg/src/uuvsim/checkpoint.py, nets.py) when the
reference is importable (build container only; skipped elsewhere)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2410_14117_b200 import checkpoint as C
from paper_2410_14117_b200 import rollout as R

REF = Path("/root/reference/pkg/src")


def _policy():
    pol = R.ActorCritic(36, 8, seed=4)
    with torch.no_grad():
        for p in pol.parameters():
            p.add_(0.05 * torch.randn_like(p))
    norm = R.RunningNorm(36, "cpu")
    norm.update(torch.randn(100, 36) * 3 + 1)
    return pol, norm


def test_round_trip(tmp_path):
    pol, norm = _policy()
    path = tmp_path / "p.bin"
    C.save_checkpoint(path, pol, norm)
    pol2, norm2 = C.load_checkpoint(path)
    for a, b in zip(pol.parameters(), pol2.parameters()):
        torch.testing.assert_close(a, b, rtol=0, atol=0)
    for a, b in ((norm.mean, norm2.mean), (norm.var, norm2.var), (norm.count, norm2.count)):
        torch.testing.assert_close(a, b, rtol=0, atol=0)


def test_errors(tmp_path):
    pol, norm = _policy()
    path = tmp_path / "p.bin"
    C.save_checkpoint(path, pol, norm)
    blob = path.read_bytes()
    for bad, msg in ((b"NOTUUVS1" + blob[8:], "not a uuvsim policy checkpoint"),
                     (blob[:8] + (2).to_bytes(4, "little") + blob[12:], "unsupported checkpoint version"),
                     (blob[:30], "truncated in normalizer block"),
                     (blob[:-8], "parameters, expected")):
        path.write_bytes(bad)
        with pytest.raises(C.CheckpointError, match=msg):
            C.load_checkpoint(path)


@pytest.mark.skipif(not REF.is_dir(), reason="reference package not mounted")
def test_interchange_with_reference_policy(tmp_path):
    sys.path.insert(0, str(REF))
    try:
        from uuvsim import checkpoint as RC
    finally:
        sys.path.remove(str(REF))
    pol, norm = _policy()
    path = tmp_path / "ours.bin"
    C.save_checkpoint(path, pol, norm)
    rpol, rnorm = RC.load_checkpoint(str(path))               # ours -> reference
    obs = np.random.default_rng(0).normal(size=(16, 36)) * 3
    rmean, rval, _ = rpol.forward(rnorm.normalize(obs))       # reference numpy, fp64
    with torch.no_grad():
        z = (torch.from_numpy(obs) - norm.mean) / torch.sqrt(norm.var + 1e-8)
        mean, val = pol.double()(z.clamp(-10, 10))
    np.testing.assert_allclose(mean.numpy(), rmean, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(val.numpy(), rval, rtol=1e-12, atol=1e-12)
    path2 = tmp_path / "ref.bin"
    RC.save_checkpoint(str(path2), rpol, rnorm)               # reference -> ours
    assert path2.read_bytes() == path.read_bytes()
