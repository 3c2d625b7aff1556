"""GPU checks of NEXT row f1 (the equal-sample comparison harness):
the error-sum kernel against float64 numpy, the IR comparator's VPL set
(all patches FAR, budget rule) bitwise against the oracle, and the harness
end to end on C1."""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import oracle
import paper_2203_11484_b200 as V
import scenegen
from gpu_helpers import GpuScene, assert_vpls_bitwise

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [0, 1, 1000, 3 * 1920 * 1080 + 7])
def test_image_error_matches_float64(n):
    g = torch.Generator().manual_seed(n)
    a = torch.rand(n, generator=g, dtype=torch.float32)
    r = torch.rand(n, generator=g, dtype=torch.float32)
    e = V.image_error(a.cuda(), r.cuda())
    d = a.double() - r.double()
    ref = [float((d * d).sum()), float((r.double() ** 2).sum()), float(d.abs().sum()), float(r.double().abs().sum())]
    for x, y in zip(e["sums"], ref):
        assert abs(x - y) <= 1e-12 * max(abs(y), 1.0), (x, y)
    if n:
        assert math.isclose(e["rmse"], math.sqrt(ref[0] / n), rel_tol=1e-12)
    e2 = V.image_error(a.cuda(), r.cuda())
    assert e2["sums"] == e["sums"]                                    # deterministic order


def test_image_error_zero_for_identical_images():
    a = torch.rand(12345, device="cuda")
    e = V.image_error(a, a.clone())
    assert e["rmse"] == 0.0 and e["mae"] == 0.0


def test_ir_comparator_vpls_bitwise():
    """IR comparator = the walk of O10 with every patch FAR in budget mode:
    K = 0, M_far = M, the first M deposits — bitwise the oracle's."""
    s = scenegen.make_scene(2)
    gs, os_ = GpuScene(s), oracle.OracleScene(s)
    lab = np.zeros(s.n_tris, np.uint8)
    v, info = gs.generate(labels=lab, K_near=0)
    ov, oinfo = os_.generate_vpls(lab, K_near=0)
    assert info == oinfo and info["K"] == 0 and info["M_far"] == s.M
    assert_vpls_bitwise(V.decode_vpls(v), ov)


def test_compare_estimators_c1():
    from paper_2203_11484_b200.compare import compare_estimators
    s = scenegen.make_scene(1)
    out, imgs = compare_estimators(s, M_list=(256,), ref_M=8192, return_images=True)
    run = out["runs"][0]
    assert run["hybrid"]["K"] > 0 and run["ir"]["K"] == 0 and run["ir"]["M_far"] == 256
    for k in ("hybrid", "ir"):
        assert 0 < run[k]["rel_rmse"] < 10 and math.isfinite(run[k]["rmse"])
    # the harness's hybrid image at M = s.M is the frame's image (same calls, same seed)
    img = V.Renderer(s).frame()
    assert torch.equal(imgs[256][0], img)
    e = V.image_error(imgs[256][1], imgs["ref"])
    assert e["sums"] == run["ir"]["sums"]
