"""The exactness argument of the FP64-pipe modular arithmetic (DESIGN R-FP64), checked on the host.

The product's fmulmod(b, w) (hy_arith.cuh) computes b*w mod q with six FP64 operations:
    h = fl(b w);  l = fma(b, w, -h) = b w - h;  c = rint(fl(h qinv + M) - M), M = 1.5 2^52;
    r = fma(-c, q, h) + l.
It is exact (r = b w - c q, an integer) when |h qinv| < 2^51, and then
    |r| <= q/2 + |b| q 2^-52        (lemma: c = round(h qinv) is off round(h/q) by <= |h/q| 2^-53, |l| <= |h| 2^-53).
The forward (Cooley-Tukey) passes run 8 stages with no reduction, a' = a + t, b' = a - t, t = fmulmod(b, w), so the
largest operand bound beta_s (in units of q) follows beta_{s+1} = beta_s + 1/2 + beta_s q 2^-52, and the pass output
(after 8 stages) is itself multiplied again (key-switch IP, ModDown epilogue).  These tests
  1. emulate fmulmod exactly with Python integers / correctly rounded floats and check the lemma on random and
     extreme operands for every prime of every parameter set;
  2. iterate the recurrence from a canonical ([0, q)) and a centred (|v| <= q/2 + 1) start and check that the
     largest operand ever handed to fmulmod stays below 2^51 for every prime (the kernels' precondition).
This is a check of the product's arithmetic design, not an oracle pin (the oracle uses __int128 %).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

M = 1.5 * 2.0**52


def fmulmod_emulated(b: int, w: int, q: int):
    """The six FP64 operations of hy_arith.cuh fmulmod, emulated exactly (IEEE binary64, round to nearest)."""
    bd, wd, qd = float(b), float(w), float(q)
    assert bd == b and wd == w and qd == q
    qinv = 1.0 / qd                                   # fl(1/q), as the context's PrimeConst.qinv
    h = bd * wd                                       # fl(b w)
    l_exact = b * w - int(h)                          # fma(b, w, -h): exact, representable
    assert float(l_exact) == l_exact
    x = Fraction(h) * Fraction(qinv) + Fraction(M)    # fma(h, qinv, M) before its single rounding
    assert abs(Fraction(h) * Fraction(qinv)) < 2**51, "magic-rounding precondition violated"
    c = round(x) - int(M)                             # round-half-even to an integer in [2^52, 2^53), minus M
    t = int(h) - c * q                                # fma(-c, q, h): exact when |t| < 2^53
    assert abs(t) < 2**53
    r = t + l_exact                                   # final add: exact when |r| < 2^53
    assert abs(r) < 2**53
    return r


def _primes():
    out = []
    for name, prm in synth.PARAMS.items():
        o = oracle.Oracle(**prm)
        out += [(name, int(q)) for q in o.moduli]
    return out


PRIMES = _primes()


def beta_after(stages: int, beta0: float, q: int) -> list:
    """operand bounds (units of q) at the input of stage 1..stages and after the last stage"""
    b = [beta0]
    for _ in range(stages):
        b.append(b[-1] + 0.5 + b[-1] * q * 2.0**-52)
    return b


@pytest.mark.parametrize("name,q", sorted(set(PRIMES), key=lambda x: x[1])[-6:] + sorted(set(PRIMES))[:2])
def test_fmulmod_lemma(name, q):
    g = np.random.default_rng(q % 1000003)
    bmax = int(6.7 * q)
    cases = [(bmax, q - 1), (-bmax, q - 1), (q - 1, q - 1), (0, q - 1), (bmax, 1), (-(q // 2), q - 1)]
    cases += [(int(g.integers(-bmax, bmax)), int(g.integers(0, q))) for _ in range(300)]
    for b, w in cases:
        r = fmulmod_emulated(b, w, q)
        assert (r - b * w) % q == 0
        assert abs(r) <= q / 2 + abs(b) * q * 2.0**-52 + 1


def test_forward_pass_growth_below_2_51():
    """every forward pass's largest fmulmod operand (8 stages from canonical input, then the IP / epilogue product
    of the pass output) stays below 2^51 / (w/q) for every prime in use (w < q)"""
    worst = 0.0
    for _, q in PRIMES:
        for beta0 in (1.0, 0.5 + 1.0 / q):          # canonical [0, q) (u2d loads) / fred format
            b = beta_after(8, beta0, q)
            # stage inputs b[0..7] and the pass output b[8] all meet a fmulmod; ModDown epilogue adds q/2 + 1
            worst = max(worst, (b[8] + 0.5) * q)
    assert worst < 2.0**51, worst
    # the documented figures (DESIGN R-FP64) for a 2^48 prime
    b = beta_after(8, 1.0, 2**48)
    assert abs(b[8] - 6.62) < 0.01
    assert abs(beta_after(8, 0.5, 2**48)[8] - 5.81) < 0.01


def test_inverse_pass_growth():
    """Gentleman-Sande: sums double per stage and are re-centred (fred) after every register round of <= 3 stages,
    so the largest fmulmod operand is a - b with |a|, |b| <= 4 q_max (canonical start): far below 2^51."""
    for _, q in PRIMES:
        assert 8 * q < 2.0**51
