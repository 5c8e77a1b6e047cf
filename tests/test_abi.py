"""CPU checks of the C ABI: the library loads without a GPU, exports every
symbol include/genalpha.h declares, and its host-only entry points
(ga_params, ga_query) agree with the oracle / reject bad input."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import params as oparams

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "genalpha.h")).read()
    return sorted(set(re.findall(r"^\s*(?:ga_status|void|int|const char\*)\s+(ga_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def ga():
    from paper_2102_11536_b200 import build
    build.build()
    import paper_2102_11536_b200.genalpha as g
    return g


def test_exports_every_declared_symbol(ga):
    declared = _header_functions()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(ga.lib, name), name
    assert sorted(ga.EXPORTED) == declared


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("rho", [0.0, 0.3, 0.5, 1.0])
def test_params_match_oracle(ga, k, rho):
    al, be, gm, af, th = ga.ga_params(k, rho)
    oal, obe, ogm, oaf = oparams.scheme_params(k, rho, 0)
    np.testing.assert_allclose(al, oal, rtol=1e-14)
    np.testing.assert_allclose(be, obe, rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(gm, ogm, rtol=1e-14)
    np.testing.assert_array_equal(af, oaf)
    assert abs(th - oparams.theta_max_closed_form(rho)) < 1e-13


def test_params_printed_set_and_errors(ga):
    al, be, gm, af, th = ga.ga_params(2, 0.5, param_set=1)
    oal, obe, ogm, _ = oparams.scheme_params(2, 0.5, 1)
    np.testing.assert_allclose(al, oal, rtol=1e-14)
    np.testing.assert_allclose(be, obe, rtol=1e-14)
    assert abs(th - 1.1764705882352942) < 1e-12  # block-1 lambda=-1 crossing of the printed set
    with pytest.raises(ga.GAError):
        ga.ga_params(2, 1.0, param_set=1)       # printed set undefined at rho = 1
    with pytest.raises(ga.GAError):
        ga.ga_params(2, 0.3, 0.5)                # rho_s > rho_b
    with pytest.raises(ga.GAError):
        ga.ga_params(2, -0.1)
    with pytest.raises(ga.GAError):
        ga.ga_params(5, 0.5)


def test_query_sizes(ga):
    cfg = synth.config("c2", n=16)
    prob = synth.make_problem(cfg)
    d = ga.make_desc(prob["patches"], 3, 16, 2, k=2, rho=0.0, dt=1e-3)
    nf, ws, sc, smin = ga.ga_query(d)
    assert nf == (16 + 3 - 2) ** 2
    assert ws >= 2 * 49 * nf * 8
    assert sc >= smin > 0


def test_query_lshape_and_elastic(ga):
    p, n = 3, 8
    m = n + p
    d = ga.make_desc(synth.lshape_patches(p, n, 0.1, 5), p, n, 2, k=2, rho=0.3, dt=1e-3)
    nf, *_ = ga.ga_query(d)
    assert nf == 3 * m * m - 10 * m + 8
    ctrl = synth.control_net(3, 2, 4, 0.15, 4)
    d = ga.make_desc([((0, 0, 0), ctrl)], 2, 4, 3, ncomp=3, k=2, rho=0.5, dt=1e-3)
    nf, *_ = ga.ga_query(d)
    assert nf == 3 * 4 ** 3


def test_query_rejects_bad_desc(ga):
    ctrl = synth.control_net(2, 2, 4)
    for kw, code in [(dict(k=0), ga.GA_ERR_ARG), (dict(rho=1.5), ga.GA_ERR_PARAM), (dict(dt=0.0), ga.GA_ERR_ARG),
                     (dict(ncomp=3), ga.GA_ERR_ARG), (dict(pcg_maxit=0), ga.GA_ERR_ARG)]:
        d = ga.make_desc([((0, 0), ctrl)], 2, 4, 2, **kw)
        with pytest.raises(ga.GAError) as ei:
            ga.ga_query(d)
        assert ei.value.code == code, kw
    d = ga.make_desc([((0, 0), ctrl), ((0, 0), ctrl)], 2, 4, 2)
    with pytest.raises(ga.GAError):
        ga.ga_query(d)  # two patches in one cell
