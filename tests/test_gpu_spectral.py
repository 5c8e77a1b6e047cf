"""GPU spectral tooling: ga_spectral_scan (rho(G(Theta)) by the closed-form
cubics of the 3x3 diagonal blocks Lambda_j) against the oracle's eigenvalues of the
full amplification matrix built by stepping unit vectors (oracle/spectral.py), and the
stability limit from a GPU scan against the closed form of reading R9 (G3)."""
import numpy as np
import pytest

from oracle import params, spectral

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("rho", [0.0, 0.3, 0.5, 1.0])
def test_spectral_scan_matches_oracle(k, rho):
    import torch

    from paper_2102_11536_b200 import spectral_scan
    th = np.concatenate([np.linspace(1e-4, 4.5, 397), [params.theta_max_closed_form(rho)]])
    got = spectral_scan(torch.tensor(th, device="cuda"), k, rho).cpu().numpy()
    ref = np.array([spectral.spectral_radius(t, k, rho) for t in th])
    # multiple roots (e.g. the triple root at the bifurcation) make both sides accurate to ~eps^(1/3)
    assert np.abs(got - ref).max() < 2e-5, np.abs(got - ref).max()


@pytest.mark.parametrize("rho", [0.0, 0.3, 0.5, 0.9])
def test_spectral_scan_stability_limit(rho):
    import torch

    from paper_2102_11536_b200 import spectral_scan
    th = np.linspace(1e-3, 5.0, 200001)
    for k in (1, 2, 3):
        r = spectral_scan(torch.tensor(th, device="cuda"), k, rho).cpu().numpy()
        first = th[np.argmax(r > 1.0 + 1e-8)]
        assert abs(first - params.theta_max_closed_form(rho)) < 1e-3, (k, rho, first)  # k-independent
