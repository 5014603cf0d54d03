"""The analytic half of the certified fp32 draw's proof, checked on the CPU.

The GPU half -- the measured radius and angle bounds over every 32-bit word, and the composed
per-arm bound on 2^28 seeded samples -- is tests/test_gpu_parity.py::test_certified_draw_bounds.
Here the constants compiled into paper_2208_06102_b200/csrc/certify.cuh are read back and the
inequalities of the derivation are checked in exact rational arithmetic, so a constant edited
below what its term needs fails, independently of the GPU.
"""
import math
import re
from fractions import Fraction as F

import numpy as np
import pytest

from tests.conftest import ROOT

SRC = open(f"{ROOT}/paper_2208_06102_b200/csrc/certify.cuh").read()
U = F(1, 2**24)          # fp32 unit roundoff
UD = F(1, 2**53)         # fp64 unit roundoff


def f32(x):
    return F(float(np.float32(x)))


def const(name, env):
    """Evaluates `constexpr float name = <expr>;` of certify.cuh with fp32 literal rounding."""
    m = re.search(rf"constexpr float {name} = ([^;]+);", SRC)
    assert m, name
    expr = re.sub(r"(\d[\d.]*(?:e-?\d+)?)f\b", r"f32(\1)", m.group(1))
    val = eval(expr, {"f32": f32, **env})                      # noqa: S307 -- the repo's own source
    return f32(float(val))                                       # the compiler rounds to fp32


@pytest.fixture(scope="module")
def C():
    env = {}
    for n in ("kAlpha", "kBeta", "kAng", "kRMax", "kZr", "kZb", "kSig", "kTheta", "kSigScale"):
        env[n] = const(n, env)
    return env


def test_radius_cap_covers_the_largest_radius(C):
    # u1 >= 2^-32: r = sqrt(-2 ln u1) <= sqrt(64 ln 2); the fp32 radius adds at most e_r there
    rmax = math.sqrt(64 * math.log(2))
    er = float(C["kAlpha"]) * rmax + float(C["kBeta"]) / rmax
    assert rmax + er < float(C["kRMax"])


def normal_constants_ok(C):
    """|z32 - z| <= e_r (1 + 2 kAng + 2u + 2ud) + r32 (kAng + u (1 + kAng) + ud), with e_r the
    checked radius bound evaluated with two upward roundings (x (1 + 2^-23)^2)."""
    a, b, ang = C["kAlpha"], C["kBeta"], C["kAng"]
    grow = (1 + 2 * U) ** 2 * (1 + 2 * ang + 2 * U + 2 * UD)
    return C["kZr"] >= a * grow + (ang + U * (1 + ang) + UD) * (1 + 4 * U) and C["kZb"] >= b * grow


def test_normal_error_constants(C):
    assert normal_constants_ok(C)


def test_normal_error_constants_negative_control(C):
    """The check has teeth: the angle term dropped from kZr, or kZb without its growth, fails."""
    assert not normal_constants_ok(dict(C, kZr=C["kAlpha"] * F(1000002, 1000000)))
    assert not normal_constants_ok(dict(C, kZb=C["kBeta"]))


def test_theta_error_constants(C):
    """theta32 = RN32(sigma32 z32 + mu32) against theta = RN64(sigma z + mu) (NC-4), mu32 =
    RN32(RN64(mu - ref)), sigma32 = RN32(sigma):
      |sigma32 - sigma| |z32|            <= u sigma32 rmax'     (sigma term)
      |mu32 - (mu - ref)|                <= u |mu32| + ud |mu - ref|, |mu32| <= |theta32|(1+2u) + sigma32 rmax'
      |theta32 - (sigma32 z32 + mu32)|   <= u |theta32| (1 + 2u)
      |theta - (sigma z + mu)|           <= ud (|theta32| + E + |ref|)
    so kSig must cover 2 u rmax' (+ the fp64 terms) and kTheta 2u + 2ud (+ their growth)."""
    rmaxp = C["kRMax"] * (1 + C["kAng"]) * (1 + U)
    sigma_terms = 2 * U * rmaxp * (1 + 2 * U) + 2 * UD * rmaxp
    assert C["kSig"] >= sigma_terms * (1 + 2**-20)
    theta_terms = (2 * U + 2 * UD) * (1 + 4 * U)
    assert C["kTheta"] >= theta_terms
    # sigma <= sigma32 (1 + 2^-23): the sigma-proportional terms use sigma32 x kSigScale
    assert C["kSigScale"] >= 1 + 2 * U


def test_key_packing_term():
    """Replacing the low `bits` mantissa bits of theta32 by the arm index moves it by less than
    2^bits ulp <= 2^(bits-23) |key|; the kernel adds 2^(bits-23) (1 + 1e-6) to kTheta."""
    rng = np.random.default_rng(5)
    for bits in (1, 3, 4, 5):
        x = (rng.standard_normal(200000) * 10.0 ** rng.uniform(-6, 6, 200000)).astype(np.float32)
        idx = rng.integers(0, 2**bits, x.size).astype(np.int32)
        keep = np.int32(~((1 << bits) - 1))
        key = ((x.view(np.int32) & keep) | idx).view(np.float32)
        d = np.abs(key.astype(np.float64) - x.astype(np.float64))
        assert np.all(d <= 2.0 ** (bits - 23) * np.abs(key.astype(np.float64)))


def test_certification_test_is_sound_on_a_worked_case(C):
    """The certification inequality, evaluated by hand for two arms: separating intervals pass,
    touching intervals fail (the exact path decides)."""
    kth = float(C["kTheta"]) + 2.0 ** (4 - 23) * 1.000001
    smax, ez, c = 2.0, 5e-6, 1e-12
    S = smax * float(C["kSigScale"]) * (ez + float(C["kSig"])) + c

    def certified(m1, m2):
        return (m2 - kth * abs(m2)) - (m1 + kth * abs(m1)) > 2 * S

    assert certified(0.0, 1e-3)
    assert not certified(0.0, 2 * S * 0.99)
