"""Host-side spectrum helpers (eigensolver.cpp:177-198)."""
import numpy as np
import pytest

from paper_1408_3839_b200.api import DimensionError, average_energy_per_cell, spectral_bands


def test_spectral_bands_regroups_kpoints():
    eig = np.array([[-1.0, 2.0], [-0.5, 3.0], [-0.8, 2.5]])
    bands, lo, hi = spectral_bands(eig)
    assert bands.shape == (2, 3)
    assert np.array_equal(bands[0], [-1.0, -0.5, -0.8]) and lo[0] == -1.0 and hi[1] == 3.0


def test_average_energy_per_cell():
    ev = np.sort(np.array([3.0, -1.0, 0.5, -2.0, 1.0, 4.0]))
    assert average_energy_per_cell(ev, 2, 2) == pytest.approx((-2.0 - 1.0 + 0.5 + 1.0) / 2)
    with pytest.raises(DimensionError):
        average_energy_per_cell(ev, 4, 2)
