"""The production sketch Omega (Alg. 2 step 1; one Omega for every level, R8):
the device Philox4x32-10 + Box-Muller generator of spdhss_build (reading R29),
checked element by element against oracle/omega.py (independent implementation of
the same counter-based generator, pinned by the Random123 known answers) and, on
its own output, for the N(0,1) moments, the Kolmogorov-Smirnov distance and column
independence on >= 4e6 samples."""
import numpy as np
import pytest
from scipy import stats

from gpu_util import host
from oracle.omega import philox_normal as oracle_philox

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


@pytest.mark.parametrize("n,w,seed", [(1000, 7, 1), (32768, 110, 3002), (3, 5, 2 ** 40 + 17)])
def test_device_omega_is_the_oracle_generator(spd, n, w, seed):
    z = host(spd.philox_normal(n, w, seed))
    zo = oracle_philox(n, w, seed)
    # same counters and uniforms; log / cos rounding differ by a few ulps
    assert np.abs(z - zo).max() <= 1e-14 * max(1.0, np.abs(zo).max())


def test_device_omega_distribution(spd):
    n, w = 1 << 20, 4
    z = host(spd.philox_normal(n, w, 1234))
    x = z.ravel()
    N = x.size
    assert abs(x.mean()) < 5 / np.sqrt(N)
    assert abs(x.var() - 1.0) < 5 * np.sqrt(2.0 / N)
    assert abs(stats.skew(x)) < 5 * np.sqrt(6.0 / N)
    assert abs(stats.kurtosis(x)) < 5 * np.sqrt(24.0 / N)
    assert stats.kstest(x, "norm").statistic < 1.63 / np.sqrt(N)
    C = np.corrcoef(z.T)
    assert np.abs(C[~np.eye(w, dtype=bool)]).max() < 5 / np.sqrt(n)
