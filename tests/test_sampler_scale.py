"""P7 at the survey's scale (Alg. 1's θ̂_b ~ N(μ̂_b, σ̂_b²)).

* 10^8 contract normals (NC-3: Philox4x32-10, (a+1)·2^-32 / b·2^-32 uniforms, Box-Muller with the
  contract log and sin/cos): mean, variance, skewness and excess kurtosis within 5 standard
  errors; chi-square over 1000 equiprobable bins; a KS statistic on a 2^16-edge grid (a lower
  bound of the exact KS statistic, so the bound tests deviations down to 1/2^16 of the range);
  correlations within a pair, across the two pairs of one Philox block and across trials.
* The contract log and sin/cos(πx) on 10^7 points each against an 80-bit long-double reference
  (64-bit mantissa, so the reference is good to ~2^-11 ulp of a double): zlog <= 2 ulp,
  zsincospi <= 1.1 ulp (NC-3).  At 10^7 points the sin/cos polynomials reach 1.06 ulp
  on ~1.6e-5 of the points, all at |f| > 0.2 of the reduced argument (where the result sits just
  above 0.5 and the ulp halves); the 1500-point check of test_oracle_pins.py never saw one.
  This is sampler quality, not parity: both sides compute the same bits.
"""
import math
import os

import numpy as np
import pytest

THREADS = max(1, min(16, os.cpu_count() or 1))


def _phi(x):
    from scipy.special import ndtr

    return ndtr(x)


def test_1e8_normals_moments_chi2_ks(oracle):
    from scipy import stats

    n_chunks, pairs = 10, 5_000_000
    n = 2 * n_chunks * pairs
    edges_ks = np.linspace(-7.0, 7.0, 2 ** 16 + 1)
    q_edges = stats.norm.ppf(np.linspace(0, 1, 1001)[1:-1])
    h_ks = np.zeros(len(edges_ks) + 1, np.int64)
    h_chi = np.zeros(1000, np.int64)
    s1 = s2 = s3 = s4 = 0.0
    c_pair = c_block = c_trial = 0.0
    for c in range(n_chunks):
        # vary the whole key: trials, recurrence t and pair k (k even/odd use different words)
        z = oracle.normal_batch(2208 + c, c * pairs, pairs, t=37 * c, k=c % 4, threads=THREADS)
        zz = z.ravel()
        s1 += zz.sum(); s2 += (zz ** 2).sum(); s3 += (zz ** 3).sum(); s4 += (zz ** 4).sum()
        h_ks += np.bincount(np.searchsorted(edges_ks, zz), minlength=len(edges_ks) + 1)
        h_chi += np.bincount(np.searchsorted(q_edges, zz), minlength=1000)
        c_pair += float(np.dot(z[:, 0], z[:, 1]))
        c_trial += float(np.dot(z[:-1, 0], z[1:, 0]))
        if c == 0:                                   # the other pair of the same Philox blocks
            w = oracle.normal_batch(2208, 0, pairs, t=0, k=1, threads=THREADS)
            c_block = float(np.corrcoef(z[:, 0], w[:, 0])[0, 1])
    m1 = s1 / n
    var = s2 / n - m1 ** 2
    skew = (s3 / n) / var ** 1.5
    kurt = (s4 / n) / var ** 2 - 3.0
    assert abs(m1) < 5 * math.sqrt(1 / n)
    assert abs(var - 1) < 5 * math.sqrt(2 / n)
    assert abs(skew) < 5 * math.sqrt(6 / n)
    assert abs(kurt) < 5 * math.sqrt(24 / n)
    assert stats.chisquare(h_chi).pvalue > 1e-4
    cdf = np.cumsum(h_ks)[:-1] / n                  # empirical CDF at the grid edges
    d = float(np.max(np.abs(cdf - _phi(edges_ks))))
    assert math.sqrt(n) * d < 1.95, d               # KS critical value at p = 1e-3
    half = n_chunks * pairs
    assert abs(c_pair / half) < 5 / math.sqrt(half)
    assert abs(c_trial / half) < 5 / math.sqrt(half)
    assert abs(c_block) < 5 / math.sqrt(pairs)


def _ulp(ref_ld):
    return np.spacing(np.abs(ref_ld.astype(np.float64)))


def test_zlog_1e7_points_within_2_ulp(oracle):
    assert np.finfo(np.longdouble).nmant >= 63, "needs x87 long double for the reference"
    rng = np.random.default_rng(5)
    a = rng.integers(0, 2 ** 32, size=5_000_000, dtype=np.uint64)
    xs = np.concatenate([(a.astype(np.float64) + 1.0) * 2.0 ** -32,        # the sampler's domain
                         rng.random(2_500_000) + 2.0 ** -60,
                         rng.uniform(0.5, 2.0, 2_500_000)])
    got = oracle.zlog_batch(xs)
    ref = np.log(xs.astype(np.longdouble))
    nz = xs != 1.0
    err = np.abs(got[nz].astype(np.longdouble) - ref[nz]) / _ulp(ref[nz])
    assert float(err.max()) <= 2.0, float(err.max())
    assert np.all(got[xs <= 1.0] <= 0.0) and np.all(got[xs == 1.0] == 0.0)


def test_zsincospi_1e7_points_within_1p1_ulp(oracle):
    assert np.finfo(np.longdouble).nmant >= 63
    rng = np.random.default_rng(6)
    m = np.concatenate([rng.integers(0, 2 ** 52, size=5_000_000, dtype=np.uint64),
                        rng.integers(0, 2 ** 32, size=5_000_000, dtype=np.uint64) << np.uint64(20)])
    s, c = oracle.zsincospi_batch(m)
    # exact reduction in integers: x = m / 2^51 = n/2 + f, |f| <= 1/4
    n = (m + np.uint64(1 << 49)) >> np.uint64(50)
    j = m.astype(np.int64) - (n.astype(np.int64) << 50)
    f = j.astype(np.longdouble) / np.longdouble(2.0 ** 51)
    pi = np.longdouble("3.14159265358979323846264338327950288419716939937510582097494")
    sf, cf = np.sin(pi * f), np.cos(pi * f)
    q = (n & np.uint64(3)).astype(np.int64)
    rs = np.select([q == 0, q == 1, q == 2, q == 3], [sf, cf, -sf, -cf])
    rc = np.select([q == 0, q == 1, q == 2, q == 3], [cf, -sf, -cf, sf])
    for got, ref in ((s, rs), (c, rc)):
        zero = np.abs(ref) < np.longdouble(1e-300)
        assert np.all(got[zero] == 0.0)
        err = np.abs(got[~zero].astype(np.longdouble) - ref[~zero]) / _ulp(ref[~zero])
        assert float(err.max()) <= 1.1, float(err.max())
        assert float((err > 1.0).mean()) < 1e-4


def test_log_table_generator_within_1_ulp(oracle):
    """The 91 table entries logc_j = -zlog_fdlibm(1/c_j) (NC-3): fdlibm's log <= 1 ulp there."""
    cj = 1.0 + np.arange(-37, 54) / 128.0
    invc = 1.0 / cj
    got = -np.array([oracle.zlog_fdlibm(x) for x in invc])
    ref = -np.log(invc.astype(np.longdouble))
    nz = invc != 1.0
    err = np.abs(got[nz].astype(np.longdouble) - ref[nz]) / _ulp(ref[nz])
    assert float(err.max()) <= 1.0
