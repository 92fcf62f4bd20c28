"""Spectral analysis helpers on the CPU (SPEC.md:450-466 trivial examples)."""
import numpy as np
import pytest

from paper_1901_01685_b200 import analysis
from paper_1901_01685_b200._native import Csr


def test_spectral_radius_trivial():
    assert analysis.spectral_radius(np.zeros((4, 4))).rho == 0.0
    R = np.array([[0.0, -0.5], [0.5, 0.0]])  # rotation-like: eigenvalues +-0.5i
    s = analysis.spectral_radius(R)
    assert s.rho == pytest.approx(0.5) and np.iscomplexobj(s.eigenvalues)
    with pytest.raises(ValueError):
        analysis.spectral_radius(np.zeros((2, 3)))


def test_condition_number_trivial():
    assert analysis.condition_number(np.eye(5)) == pytest.approx(1.0)
    assert analysis.condition_number(np.diag([1.0, 10.0])) == pytest.approx(10.0)
    A = Csr(2, 2, np.array([0, 1, 2], np.int32), np.array([0, 1], np.int32), np.array([1.0, 10.0]))
    assert analysis.condition_number(A) == pytest.approx(10.0)
