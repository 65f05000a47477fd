"""Exact emulation of paper_1203_1269_b200/csrc/fastmath.cuh (exp_neg, log_pos, pow_abs_fast)
against glibc (math.exp / math.log, what the reference calls): every product / sum rounded
as the device code rounds it (explicit fma = one rounding, via fractions). rcp.approx is
seeded from a float32 reciprocal; two Newton steps make the seed irrelevant.
Prints ulp histograms; used to choose the formulation (see fastmath.cuh header)."""
import math
import random
import struct
from fractions import Fraction as F

import numpy as np


def fma(a, b, c):
    return float(F(a) * F(b) + F(c))


def _bits(x):
    return struct.unpack('<Q', struct.pack('<d', x))[0]


def _mk(h, l):
    return struct.unpack('<d', struct.pack('<Q', ((h & 0xffffffff) << 32) | l))[0]


def ulps(a, b):
    ia = struct.unpack('<q', struct.pack('<d', a))[0]
    ib = struct.unpack('<q', struct.pack('<d', b))[0]
    return abs(ia - ib)


EXP_P = [1.0 / math.factorial(j) for j in range(2, 14)]
LN2_HI, LN2_LO = 6.93147180369123816490e-01, 1.90821492927058770002e-10
LG = [6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01,
      2.222219843214978396e-01, 1.818357216161805012e-01, 1.531383769920937332e-01,
      1.479819860511658591e-01]


def exp_neg(s):
    x = min(max(-s, -1000.0), 1000.0)
    kd = fma(x, 1.4426950408889634, 6755399441055744.0)
    kf = kd - 6755399441055744.0
    k = int(kf)
    rh = fma(kf, -LN2_HI, x)
    rl = kf * -LN2_LO
    r = rh + rl
    P = EXP_P[11]
    for j in range(10, -1, -1):
        P = fma(P, r, EXP_P[j])
    t = fma(r * r, P, rl)
    hi = 1.0 + rh
    lo = (1.0 - hi) + rh
    e = hi + (lo + t)
    k1 = k >> 1
    return (e * 2.0 ** k1) * 2.0 ** (k - k1)


def fast_two_sum(a, b):
    s = a + b
    return s, b - (s - a)


def log_pos(a):
    sub = a < 2.2250738585072014e-308
    a2 = a * 18014398509481984.0 if sub else a
    hx = _bits(a2) >> 32
    k = (hx >> 20) - 1023 - (54 if sub else 0)
    hx &= 0x000fffff
    i = (hx + 0x95f64) & 0x100000
    m = _mk(hx | (i ^ 0x3ff00000), _bits(a2) & 0xffffffff)
    k += i >> 20
    f = m - 1.0
    den = 2.0 + f
    r = float(np.float32(1.0) / np.float32(den))
    r = fma(r, fma(-den, r, 1.0), r)
    r = fma(r, fma(-den, r, 1.0), r)
    s = f * r
    hf = 0.5 * f
    hfsq = hf * f
    hfsq_lo = fma(hf, f, -hfsq)
    z = s * s
    w = z * z
    t1 = w * fma(w, fma(w, LG[5], LG[3]), LG[1])
    t2 = z * fma(w, fma(w, fma(w, LG[6], LG[4]), LG[2]), LG[0])
    c = fma(s, hfsq + (t2 + t1), -hfsq_lo)
    dh, dl = fast_two_sum(f, -hfsq)
    dk = float(k)
    rh, rl = fast_two_sum(dk * LN2_HI, dh)
    return rh + (rl + (dl + fma(dk, LN2_LO, c)))


def pow_abs(delta, p):
    a = abs(delta)
    return 0.0 if a == 0.0 else exp_neg(-(p * log_pos(a)))


def hist(pairs):
    h = {}
    for got, want in pairs:
        u = min(ulps(got, want), 9)
        h[u] = h.get(u, 0) + 1
    return sorted(h.items())


if __name__ == "__main__":
    random.seed(3)
    ss = [random.choice([random.random() * 1e-6, random.random(), random.random() * 40,
                         random.random() * 700, 708 + random.random() * 40]) for _ in range(20000)]
    print("exp_neg vs glibc exp(-s):", hist((exp_neg(s), math.exp(-s)) for s in ss))
    aa = [random.choice([random.random(), 10 ** random.uniform(-300, 0), 1 - random.random() * 1e-6,
                         1 + random.random() * 1e-12, random.random() * 1e-310]) for _ in range(20000)]
    aa = [a for a in aa if a > 0]
    print("log_pos vs glibc log:", hist((log_pos(a), math.log(a)) for a in aa))
    pp = [(random.random(), random.choice([1.0, 1.5, 1.9, 1.95, 2.0])) for _ in range(10000)]
    print("pow_abs vs glibc exp(p log a):", hist((pow_abs(a, p), math.exp(p * math.log(a))) for a, p in pp))
