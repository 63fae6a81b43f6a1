"""Pins for the oracle's pair RNG (reading C-7)."""
import math

import numpy as np
import pytest

import oracle
from conftest import read_golden


@pytest.mark.parametrize("row", read_golden("philox4x32_10_kat.txt"))
def test_philox_known_answers(row):
    # Random123 published known answers (tests/golden/philox4x32_10_kat.txt)
    vals = [int(t, 16) for t in row]
    out = oracle.philox4x32_10(vals[0:4], vals[4:6])
    assert [int(o) for o in out] == vals[6:10]


@pytest.mark.parametrize("row", read_golden("philox2x32_10_kat.txt"))
def test_philox2x32_known_answers(row):
    vals = [int(t, 16) for t in row]
    out = oracle.philox2x32_10(vals[0:2], vals[2])
    assert [int(o) for o in out] == vals[3:5]


def test_pair_words_symmetric_and_keyed():
    # xi_ij = xi_ji: counter uses (min id, max id)
    for (a, b, s) in [(0, 1, 0), (5, 3, 7), (123456, 99, 2**33 + 5)]:
        assert oracle.pair_words(42, s, a, b) == oracle.pair_words(42, s, b, a)
    # different step / seed / pair give different words (independence in time)
    base = oracle.pair_words(42, 0, 0, 1)
    assert oracle.pair_words(42, 1, 0, 1) != base
    assert oracle.pair_words(43, 0, 0, 1) != base
    assert oracle.pair_words(42, 0, 0, 2) != base
    # layout (C-7): k_s = Philox2x32-10({s lo, s hi}, seed lo ^ seed hi)[0];
    # (w0, w1) = Philox2x32-10({min id, max id}, k_s) -- checked against the raw generator
    seed = (7 << 32) | 42
    s = 2**32 + 17
    ks = int(oracle.philox2x32_10([s & 0xFFFFFFFF, s >> 32], 42 ^ 7)[0])
    assert oracle.step_key(seed, s) == ks
    w = oracle.philox2x32_10([3, 9], ks)
    assert oracle.pair_words(seed, s, 9, 3) == (int(w[0]), int(w[1]))
    # consecutive steps use different keys
    assert len({oracle.step_key(42, t) for t in range(1000)}) == 1000


def test_box_muller_closed_forms():
    # u1 = (w0+1) 2^-32 = 1 exactly -> ln u1 = 0 -> xi = 0
    assert oracle.xi(0xFFFFFFFF, 12345) == 0.0
    # w1 = 0 -> cos(0) = 1 -> xi = sqrt(-2 ln u1), u1 = 2^-32 for w0 = 0
    assert oracle.xi(0, 0) == pytest.approx(math.sqrt(2 * 32 * math.log(2)), rel=1e-15)
    # w1 = 2^31 -> cos(pi) = -1 ; w0 = 2^31 - 1 -> u1 = 1/2
    assert oracle.xi(2**31 - 1, 2**31) == pytest.approx(-math.sqrt(2 * math.log(2)), rel=1e-15)
    # w1 = 2^30 -> cos(pi/2) = 0
    assert abs(oracle.xi(7, 2**30)) < 1e-15
    # maximum |xi| with 32-bit u1: 6.6604
    assert abs(oracle.xi(0, 0)) == pytest.approx(6.6604, abs=1e-4)


def test_xi_statistics_gaussian():
    # <xi> = 0, <xi^2> = 1, over many pairs of one step
    xs = np.array([oracle.xi(*oracle.pair_words(42, 3, i, i + 1 + (i % 7))) for i in range(40000)])
    n = xs.size
    assert abs(xs.mean()) < 5 / math.sqrt(n)
    assert abs(xs.var() - 1.0) < 5 * math.sqrt(2 / n)
    # fourth moment of a Gaussian is 3
    assert abs((xs**4).mean() - 3.0) < 0.15
    # independent across steps for the same pair: correlation ~ 0
    ys = np.array([oracle.xi(*oracle.pair_words(42, 4, i, i + 1 + (i % 7))) for i in range(40000)])
    assert abs(np.corrcoef(xs, ys)[0, 1]) < 5 / math.sqrt(n)
