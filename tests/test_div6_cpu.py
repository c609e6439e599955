"""The point-Jacobi update divides by the diagonal 6 (inner_solvers.py:88).  The kernel replaces the IEEE
division by q = RN(x z), e = fma(-6, q, x), q' = fma(e, z, q) with z = RN(1/6) (csrc/bs_engine.cu, div6):
this pins that sequence to the correctly rounded quotient with exact rational arithmetic (CPython's
int / int -> float conversion is correctly rounded), on random and adversarial operands inside the
exponent window the kernel uses it for; outside it the kernel calls the generic division."""

import math
import random
from fractions import Fraction as F

Z = float.fromhex("0x1.5555555555555p-3")


def div6(x: float) -> float:
    q = x * Z                         # RN(x z)
    e = float(F(x) - 6 * F(q))        # fma(-6, q, x): exact, so the conversion does not round
    assert F(e) == F(x) - 6 * F(q)
    return float(F(q) + F(e) * F(Z))  # fma(e, z, q): one rounding


def test_reciprocal_constant():
    assert Z == 1.0 / 6.0
    assert abs(F(Z) * 6 - 1) <= F(1, 2 ** 54)  # relative error 2^-54: q is within one ulp of x / 6


def test_three_operation_quotient_is_correctly_rounded():
    rng = random.Random(7)
    cases = []
    for _ in range(20000):  # random significands across the kernel's exponent window (biased 200..1800)
        m = rng.getrandbits(52)
        cases.append(math.ldexp(1.0 + m / 2.0 ** 52, rng.randint(-820, 776)) * rng.choice((-1, 1)))
    for _ in range(10000):  # neighbours of exact multiples of 6 and of rounding boundaries
        k = rng.getrandbits(53) | (1 << 52)
        for d in (-3, -2, -1, 0, 1, 2, 3):
            x = float(6 * k + d)
            cases.append(x)
            cases.append(math.ldexp(x, -70))
    for _ in range(5000):  # significands next to all ones / all zeros
        cases.append(math.ldexp(1.0 + ((1 << 52) - 1 - rng.getrandbits(10)) / 2.0 ** 52, rng.randint(-50, 50)))
        cases.append(math.ldexp(1.0 + rng.getrandbits(10) / 2.0 ** 52, rng.randint(-50, 50)))
    for x in cases:
        assert div6(x) == x / 6.0, x.hex()
