"""GPU parity of NEXT row f3 — the rejection-sampling comparator (
DESIGN.md O15, reading R23) — against the oracle: probe pixels, per-candidate
scores, mean and the kept / filled VPL set must all be bitwise equal."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2203_11484_b200 as V
import scenegen
from gpu_helpers import GpuScene, assert_vpls_bitwise, vpls_to_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,pilot,budget", [(1, 1024, 256), (1, 1024, 1024), (2, 4096, 1024), (3, 2048, 512)])
def test_rejection_bitwise(cfg, pilot, budget):
    s = scenegen.make_scene(cfg)
    gs, os_ = GpuScene(s), oracle.OracleScene(s)
    lab = np.zeros(s.n_tris, np.uint8)
    pv, info = gs.generate(labels=lab, M=pilot, K_near=0)
    out, ri = V.generate_rejection(gs.scene, gs.bvh, pv, budget, seed=s.seed)
    opv = vpls_to_oracle(V.decode_vpls(pv))
    oo, oi = os_.rejection(opv, budget, seed=s.seed)
    assert np.array_equal(ri["probes"].cpu().numpy(), oi["probes"])
    sc = ri["scores"].cpu().numpy()
    assert np.array_equal(sc.view(np.uint32), oi["scores"].view(np.uint32))
    assert ri["mean"] == oi["mean"] and ri["accepted"] == oi["accepted"] and ri["n_scanned"] == oi["n_scanned"]
    assert_vpls_bitwise(V.decode_vpls(out), oo)
    assert (sc > 0).any()


def test_rejection_budget_above_pilot_and_bad_args():
    s = scenegen.make_scene(1)
    gs = GpuScene(s)
    pv, _ = gs.generate(labels=np.zeros(s.n_tris, np.uint8), M=64, K_near=0)
    out, ri = V.generate_rejection(gs.scene, gs.bvh, pv, 100, seed=1)
    assert out.shape[0] == ri["accepted"] <= 64 and ri["n_scanned"] == 64   # budget above the pilot: all scanned
    with pytest.raises(V.VplError):
        V.generate_rejection(gs.scene, gs.bvh, pv, 0, seed=1)


@pytest.mark.parametrize("cfg,pilot,chains,per_chain", [(1, 1024, 16, 16), (2, 4096, 64, 16), (3, 2048, 32, 8)])
def test_metropolis_bitwise(cfg, pilot, chains, per_chain):
    """NEXT f4 (O16, reading R24): scores, pool order, accepted count and the
    emitted VPL set bitwise against the oracle."""
    s = scenegen.make_scene(cfg)
    gs, os_ = GpuScene(s), oracle.OracleScene(s)
    lab = np.zeros(s.n_tris, np.uint8)
    pv, _ = gs.generate(labels=lab, M=pilot, K_near=0)
    out, gi = V.generate_metropolis(gs.scene, gs.bvh, pv, chains, per_chain, burn=32, radius=16, seed=s.seed)
    oo, oi = os_.metropolis(vpls_to_oracle(V.decode_vpls(pv)), chains, per_chain, burn=32, radius=16, seed=s.seed)
    assert np.array_equal(gi["scores"].cpu().numpy().view(np.uint32), oi["scores"].view(np.uint32))
    assert np.array_equal(gi["pool"].cpu().numpy(), oi["pool"])
    assert gi["accepted"] == oi["accepted"]
    assert_vpls_bitwise(V.decode_vpls(out), oo)


def test_metropolis_rejects_bad_arguments():
    s = scenegen.make_scene(1)
    gs = GpuScene(s)
    pv, _ = gs.generate(labels=np.zeros(s.n_tris, np.uint8), M=64, K_near=0)
    for kw in (dict(chains=0, per_chain=4), dict(chains=4, per_chain=0), dict(chains=4, per_chain=4, radius=0)):
        with pytest.raises(V.VplError):
            V.generate_metropolis(gs.scene, gs.bvh, pv, seed=1, **kw)
