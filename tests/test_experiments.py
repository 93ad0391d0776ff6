"""The section 5 experiment harness (tools/experiments.py): sizing rules
pinned to the values the paper prints, and a reduced GPU run of the robustness and
applicability studies (no breakdown, no bound exceeded: tab:success1-5)."""
import importlib.util
import os

import pytest

from conftest import ROOT

spec = importlib.util.spec_from_file_location("experiments", os.path.join(ROOT, "tools", "experiments.py"))


@pytest.fixture(scope="module")
def ex():
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_sketch_sizes_match_the_paper(ex):
    # s1 = (50^2 + 50) / (0.6 * 0.5^2) = 17000
    assert ex.s_count(50, 0.5, 0.6) == 17000
    # p1 = 0.3 .. 0.6 -> s1 = 5600, 4200, 3360, 2800 (n = 20)
    assert [ex.s_count(20, 0.5, p) for p in (0.3, 0.4, 0.5, 0.6)] == [5600, 4200, 3360, 2800]
    # "s(2) varies from 28 to 20" for p(2) = 0.1 .. 0.4 (eta = 1, R#12)
    assert ex.s_gauss(20, 0.5, 0.1) == 28 and ex.s_gauss(20, 0.5, 0.4) == 20


def test_bounds_shape(ex):
    # eq:ortho2ss is 6 (mn u + n(n+1) u); Phi reduces to Theta when eps_s = eps_b
    m, n = 20000, 50
    assert ex.ortho_bound(m, n) == pytest.approx(6 * (m * n + n * (n + 1)) * 2.0 ** -53, rel=1e-15)
    assert ex.resid_bound(m, n, 0.5, 0.5, 1.0) < ex.resid_bound(m, n, 0.75, 1.25, 1.0)
    assert ex.resid_bound(m, n, 0.5, 0.5, 2.0) == pytest.approx(2 * ex.resid_bound(m, n, 0.5, 0.5, 1.0))


@pytest.mark.gpu
def test_robustness_reduced(ex):
    import torch
    recs = ex.robustness(ex.Runner(torch.device("cuda", 0)), 10, lambda r: None)
    for r in recs:
        assert r["breakdowns"] == 0 and r["exceed"] == 0, r


@pytest.mark.gpu
def test_applicability_reduced(ex):
    import torch
    recs = ex.applicability(ex.Runner(torch.device("cuda", 0)), 2, lambda r: None)
    ours = [r for r in recs if r["method"] in ("slhc3", "sslhc3") and r["family"] != "arrowhead"]
    for r in ours:
        assert r["breakdowns"] == 0 and r["exceed"] == 0, r
