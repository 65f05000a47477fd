"""Exact-FMA emulation (fractions) of fastmath.cuh exp_neg vs glibc exp: ulp histogram for
degree-12 and degree-13 Taylor, plus the subnormal / underflow range."""
import math, random, struct
from fractions import Fraction as F
def fma(a,b,c): return float(F(a)*F(b)+F(c))
LOG2E = 1.4426950408889634
LN2_HI = 0.6931471805599453   # double(ln2)
LN2_LO = 2.3190468138462996e-17
C = [1.0/math.factorial(k) for k in range(14)]
MAGIC = 6755399441055744.0
def ulps(a,b):
    ia = struct.unpack('<q', struct.pack('<d', a))[0]; ib = struct.unpack('<q', struct.pack('<d', b))[0]
    return abs(ia-ib)
def expneg(s, deg=13):
    x = max(-s, -1000.0)
    kd = fma(x, LOG2E, MAGIC)
    k = int(kd - MAGIC)
    kf = kd - MAGIC
    r = fma(kf, -LN2_HI, x); r = fma(kf, -LN2_LO, r)
    p = C[deg]
    for j in range(deg-1, -1, -1): p = fma(p, r, C[j])
    k1 = k >> 1; k2 = k - k1
    return (p * 2.0**k1) * 2.0**k2
random.seed(1)
for deg in (12, 13):
    worst = 0; hist = {}
    for i in range(20000):
        s = random.choice([random.random()*1e-6, random.random(), random.random()*50, random.random()*700])
        u = ulps(expneg(s, deg), math.exp(-s)); worst = max(worst, u); hist[u] = hist.get(u,0)+1
    print(deg, worst, hist)
print(ulps(expneg(720.3), math.exp(-720.3)), expneg(720.3), math.exp(-720.3), expneg(800.0))
