"""A third, independent implementation of MagicPIG decoding for TINY inputs, in
exact rational arithmetic (fractions) plus 50-digit mpmath for the
transcendental steps.  Used only to pin the C oracle (pin P7 / golden G1).

It follows PAPER.md directly and the exactness contract of DESIGN.md
(c = fl32(fl64(sum/|D|)), x = bf16(fl32(k - c)), s = bf16(fl64(sqrt(r2 - n2))),
bit = [exact dot > 0]) but shares no code with oracle/ or the CUDA path.
The sampling probability is evaluated with the formula exactly as printed
(P:87), not the oracle's rearranged form, so agreement also pins reading R11.
"""
from __future__ import annotations

from fractions import Fraction
from typing import Dict, List

import mpmath as mp

mp.mp.dps = 50


def round_fraction(x: Fraction, p: int, emin: int) -> Fraction:
    """Round to nearest, ties to even, to a binary format with p significant
    bits and minimum normal exponent emin (gradual underflow)."""
    if x == 0:
        return Fraction(0)
    s = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, emin)
    ulp = Fraction(2) ** (e - p + 1)
    q = a / ulp
    fl = q.numerator // q.denominator
    rem = q - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return s * fl * ulp


def to_f64(x: Fraction) -> Fraction:
    return round_fraction(x, 53, -1022)


def to_f32(x: Fraction) -> Fraction:
    return round_fraction(x, 24, -126)


def to_bf16(x: Fraction) -> Fraction:
    return round_fraction(x, 8, -126)


def mpf_to_fraction(v) -> Fraction:
    man, exp = mp.mpf(v).man_exp
    return Fraction(int(man)) * (Fraction(2) ** int(exp)) if exp >= 0 else Fraction(int(man), 2 ** (-int(exp)))


def sqrt_f64(x: Fraction) -> Fraction:
    """Correctly rounded double sqrt of an exactly representable value."""
    if x <= 0:
        return Fraction(0)
    with mp.workdps(120):
        r = mp.sqrt(mp.mpf(x.numerator) / mp.mpf(x.denominator))
        return to_f64(mpf_to_fraction(r))


def decode(k: List[List[Fraction]], v: List[List[Fraction]], q: List[Fraction],
           W: List[List[Fraction]], K: int, L: int, center: int, mips: int,
           min_collisions: int, sink: int, local: int) -> Dict:
    """k, v: n x d; q: d; W: (d+mips) x KL (all exact rationals)."""
    n, d = len(k), len(q)
    static = [(i < sink or i >= n - local) for i in range(n)]
    Dset = [i for i in range(n) if not static[i]]
    # centering, exact fixed point in units of 2^-64 (reading R2b)
    def fixq(fr: Fraction) -> int:  # trunc(v * 2^64)
        v = fr * (2 ** 64)
        t = abs(v.numerator) // v.denominator
        return t if v >= 0 else -t

    if center and Dset:
        c = []
        for j in range(d):
            ks = sum(fixq(k[i][j]) for i in Dset)
            c.append(to_f32(to_f64(to_f64(Fraction(ks, 2 ** 64)) / len(Dset))))
    else:
        c = [Fraction(0)] * d
    x = [[to_bf16(to_f32(k[i][j] - c[j])) for j in range(d)] for i in range(n)]
    n2q = [sum(fixq(t * t) for t in row) for row in x]
    r2q = max((n2q[i] for i in Dset), default=0)
    r2 = Fraction(r2q, 2 ** 64)
    xbar = [list(row) for row in x]
    if mips:  # Eq. (data transform) P:49-55
        for i in range(n):
            diff = to_f64(Fraction(r2q - n2q[i], 2 ** 64)) if r2q > n2q[i] else Fraction(0)
            xbar[i].append(to_bf16(sqrt_f64(diff)))
    qbar = list(q) + ([Fraction(0)] if mips else [])
    dp = len(qbar)

    def code(vec):
        out = []
        for t in range(L):
            cw = 0
            for b in range(K):
                j = t * K + b
                dot = sum((vec[r] * W[r][j] for r in range(dp)), Fraction(0))
                if dot > 0:
                    cw |= 1 << b
            out.append(cw)
        return out

    codes = [code(xbar[i]) for i in range(n)]
    qcode = code(qbar)
    cnt = [sum(1 for t in range(L) if codes[i][t] == qcode[t]) for i in range(n)]
    S = [i for i in Dset if cnt[i] >= min_collisions]
    T = [i for i in range(n) if static[i]]
    # estimator (Eq. close form P:133-139) in 50-digit arithmetic
    qn2 = sum((t * t for t in q), Fraction(0))
    z = {}
    logu = {}
    for i in S + T:
        l = mp.mpf(sum((q[j] * k[i][j] for j in range(d)), Fraction(0)).numerator) / \
            mp.mpf(sum((q[j] * k[i][j] for j in range(d)), Fraction(0)).denominator) / mp.sqrt(d)
        if i in T:
            z[i] = l
            continue
        dot = sum((qbar[r] * xbar[i][r] for r in range(dp)), Fraction(0))
        xn2 = sum((t * t for t in xbar[i]), Fraction(0))
        den2 = qn2 * xn2
        if den2 == 0:
            cosv = mp.mpf(0)
        else:
            cosv = (mp.mpf(dot.numerator) / mp.mpf(dot.denominator)) / mp.sqrt(
                mp.mpf(den2.numerator) / mp.mpf(den2.denominator))
        cosv = max(mp.mpf(-1), min(mp.mpf(1), cosv))
        p = 1 - mp.acos(cosv) / mp.pi
        xk = p ** K
        if min_collisions == 2:
            u = 1 - (1 - xk) ** L - L * xk * (1 - xk) ** (L - 1)
        else:
            u = 1 - (1 - xk) ** L
        logu[i] = mp.log(u)
        z[i] = l - logu[i]
    out = [mp.mpf(0)] * d
    if z:
        m = max(z.values())
        den = mp.mpf(0)
        for i, zi in z.items():
            w = mp.exp(zi - m)
            den += w
            for j in range(d):
                out[j] += w * mp.mpf(v[i][j].numerator) / mp.mpf(v[i][j].denominator)
        out = [o / den for o in out]
    return {"c": c, "xbar": xbar, "r2": r2, "codes": codes, "qcode": qcode, "counts": cnt,
            "S": S, "out": [float(o) for o in out], "logu": {i: float(u) for i, u in logu.items()}}
