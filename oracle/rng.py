"""CPU restatement of the numpy Generator draws the environment consumes
(TEST INFRASTRUCTURE ONLY -- never imported by the product).

numpy 2.3.5 (numpy/random/src/distributions/distributions.c), PCG64 stream:
  next_double            (next_uint64 >> 11) * 2^-53
  standard_normal        random_standard_normal: 256-level ziggurat
  poisson                random_poisson: multiplication method (lam < 10),
                         PTRS transformed rejection (lam >= 10) with
                         random_loggam

The ziggurat tables are read from the generated device header
paper_2407_14783_b200/csrc/qb_ziggurat.h, so checking this restatement
against numpy draw for draw (tests/test_rng_restatement.py) pins the very
tables the CUDA sampler uses.
"""
import math
import os
import re

import numpy as np

_HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2407_14783_b200", "csrc",
                    "qb_ziggurat.h")


def _tables():
    src = open(_HDR).read()

    def arr(name):
        body = re.search(name + r"\[256\] = \{(.*?)\};", src, re.S).group(1)
        return [t.strip() for t in body.replace("\n", " ").split(",") if t.strip()]

    ki = np.array([int(t.rstrip("ULL"), 16) for t in arr("qb_zig_ki")], dtype=np.uint64)
    wi = np.array([float.fromhex(t) for t in arr("qb_zig_wi")])
    fi = np.array([float.fromhex(t) for t in arr("qb_zig_fi")])
    r = float.fromhex(re.search(r"#define QB_ZIG_R (\S+)", src).group(1))
    return ki, wi, fi, r


KI, WI, FI, ZIG_R = _tables()


class Stream:
    """A PCG64 word stream (the state of a numpy Generator's bit generator)."""

    def __init__(self, bit_generator):
        self.bg = bit_generator

    def next64(self):
        return int(self.bg.random_raw())

    def next_double(self):
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def standard_normal(s: Stream) -> float:
    """distributions.c random_standard_normal."""
    while True:
        r = s.next64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 0x1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * WI[idx]
        if sign:
            x = -x
        if rabs < KI[idx]:
            return x
        if idx == 0:
            while True:
                xx = -(1.0 / ZIG_R) * math.log1p(-s.next_double())
                yy = -math.log1p(-s.next_double())
                if yy + yy > xx * xx:
                    return -(ZIG_R + xx) if (rabs >> 8) & 0x1 else ZIG_R + xx
        elif (FI[idx - 1] - FI[idx]) * s.next_double() + FI[idx] < math.exp(-0.5 * x * x):
            return x


_LG = (8.333333333333333e-02, -2.777777777777778e-03, 7.936507936507937e-04, -5.952380952380952e-04,
       8.417508417508418e-04, -1.917526917526918e-03, 6.410256410256410e-03, -2.955065359477124e-02,
       1.796443723688307e-01, -1.39243221690590e+00)


def loggam(x: float) -> float:
    """distributions.c random_loggam (Stirling series, shifted below 7)."""
    if x == 1.0 or x == 2.0:
        return 0.0
    n = int(7 - x) if x < 7.0 else 0
    x0 = x + n
    x2 = (1.0 / x0) * (1.0 / x0)
    gl0 = _LG[9]
    for k in range(8, -1, -1):
        gl0 *= x2
        gl0 += _LG[k]
    gl = gl0 / x0 + 0.5 * 1.8378770664093453e+00 + (x0 - 0.5) * math.log(x0) - x0
    if x < 7.0:
        for _ in range(n):
            gl -= math.log(x0 - 1.0)
            x0 -= 1.0
    return gl


def poisson(s: Stream, lam: float) -> int:
    """distributions.c random_poisson (mult for lam < 10, PTRS otherwise)."""
    if lam >= 10:
        slam, loglam = math.sqrt(lam), math.log(lam)
        b = 0.931 + 2.53 * slam
        a = -0.059 + 0.02483 * b
        invalpha = 1.1239 + 1.1328 / (b - 3.4)
        vr = 0.9277 - 3.6224 / (b - 2)
        while True:
            U = s.next_double() - 0.5
            V = s.next_double()
            us = 0.5 - abs(U)
            k = int(math.floor((2 * a / us + b) * U + lam + 0.43))
            if us >= 0.07 and V <= vr:
                return k
            if k < 0 or (us < 0.013 and V > us):
                continue
            lv = math.log(V) if V > 0.0 else -math.inf
            if lv + math.log(invalpha) - math.log(a / (us * us) + b) <= -lam + k * loglam - loggam(k + 1):
                return k
    if lam == 0:
        return 0
    enlam = math.exp(-lam)
    x, prod = 0, 1.0
    while True:
        prod *= s.next_double()
        if prod > enlam:
            x += 1
        else:
            return x
