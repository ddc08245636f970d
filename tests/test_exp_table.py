"""K2a's table-driven double exp (stats.cu exp_nonpos), emulated on the CPU
with exactly rounded fma (fractions): within 1 ulp of glibc's exp (the
reference's std::exp, selection.hpp:155-157) and usually equal to it; and the
committed table equals tools/gen_exp_table.py's output."""
import math
import os
import random
import re
import struct
from decimal import Decimal, getcontext
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_2505_24179_b200", "csrc", "exp_table.h")


def _table():
    vals = re.findall(r"(-?0x[0-9a-fA-F.]+p[-+]\d+)", open(HDR).read())
    v = [float.fromhex(x) for x in vals]
    assert len(v) == 512
    return list(zip(v[0::2], v[1::2]))


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _bits(x):
    return struct.unpack("<q", struct.pack("<d", x))[0]


def exp_nonpos(x, tab):
    """Line-by-line restatement of stats.cu exp_nonpos."""
    tiny = x < -700.0
    x = -700.0 if tiny else x
    t = _fma(x, 369.32993046757463, 6755399441055744.0)
    k = _bits(t) & 0xFFFFFFFF
    k = k - (1 << 32) if k >= (1 << 31) else k
    kd = t - 6755399441055744.0
    r = _fma(kd, -2.7076061740622863e-03, x)
    r = _fma(kd, -9.058776616587108e-20, r)
    q = _fma(r, 8.3333333333333332e-03, 4.1666666666666664e-02)
    q = _fma(q, r, 1.6666666666666666e-01)
    q = _fma(q, r, 0.5)
    q = _fma(q, r, 1.0)
    q = q * r
    hi, lo = tab[k & 255]
    y = hi + _fma(hi, q, lo)
    v = struct.unpack("<d", struct.pack("<q", _bits(y) + ((k >> 8) << 52)))[0]
    return 0.0 if tiny else v


def test_table_matches_generator():
    getcontext().prec = 60
    for j, (hi, lo) in enumerate(_table()):
        d = Decimal(2) ** (Decimal(j) / 256)
        assert hi == float(d) and lo == float(d - Decimal(hi))


def test_exp_within_one_ulp_of_glibc():
    tab = _table()
    rng = random.Random(5)
    xs = [0.0, -1e-300, -0.5, -1.0, -700.0, -699.9999, -0.0027076061740622863]
    xs += [-rng.random() * s for s in (1.0, 8.0, 50.0, 300.0) for _ in range(600)]
    same = 0
    for x in xs:
        got, ref = exp_nonpos(x, tab), math.exp(x)
        assert abs(_bits(got) - _bits(ref)) <= 1, (x, got, ref)
        same += got == ref
    assert same >= 0.99 * len(xs)
    assert exp_nonpos(-800.0, tab) == 0.0 and exp_nonpos(-math.inf, tab) == 0.0
