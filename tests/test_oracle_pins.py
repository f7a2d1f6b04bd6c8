"""Pins for the CPU oracle (-m "not gpu").  Each test checks the oracle against
something other than itself: a closed form from PAPER.md, a Monte-Carlo
frequency, a special case that reduces to textbook attention, an invariant, an
exact-rational brute force (tests/exact_ref.py) or the hand-derived worked
example G1 (tests/golden/).  Pin ids follow SURVEY.md 8(c) C-4."""
from __future__ import annotations

import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from tests import exact_ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "g1_worked_example.json")
bf = synth.bf16_bits_from_f32


def _g1():
    with open(GOLDEN) as f:
        return json.load(f)


def _g1_arrays(g, mips):
    k = bf(np.array(g["keys"], np.float32))
    v = bf(np.array(g["values"], np.float32))
    q = bf(np.array([g["q"]], np.float32))
    W = np.array(g["W_columns"], np.float32).T.copy()  # [d][KL]
    if mips:
        W = np.vstack([W, np.array(g["W_mips_row"], np.float32)[None, :]])
    return k, v, q, W


# --------------------------------------------------------------------------- G1
@pytest.mark.parametrize("mips", [0, 1])
def test_g1_golden_oracle(mips):
    g = _g1()
    k, v, q, W = _g1_arrays(g, mips)
    r = oracle.decode_unit(k, v, q, W, K=g["K"], L=g["L"], center=1, mips=mips, sink=0, local=0)
    assert r["status"] == 0
    exp = g["mips1" if mips else "mips0"]
    np.testing.assert_array_equal(r["counts"][0], exp["counts"])
    S = [i for i in range(4) if r["in_s"][0, i] == 1]
    assert S == exp["S"]
    np.testing.assert_allclose(r["out"][0], exp["out"], rtol=1e-12, atol=1e-15)
    if not mips:
        np.testing.assert_array_equal(r["c"], exp["c"])
        codes = [[(int(r["codes"][i, t])) for t in range(3)] for i in range(4)]
        assert codes == exp["codes"]
        assert list(r["qcodes"][0]) == exp["qcode"]
        for i, u in exp["u"].items():
            assert math.isclose(math.exp(r["logu"][0, int(i)]), u, rel_tol=1e-12)
        np.testing.assert_allclose(oracle.exact_attention(q[0], k, v), exp["exact_attention"], rtol=1e-12)
    else:
        assert r["r2"] == exp["r2"]


@pytest.mark.parametrize("mips", [0, 1])
def test_g1_golden_exact_ref(mips):
    """The independent exact-arithmetic implementation reproduces G1 too."""
    g = _g1()
    F = Fraction
    k = [[F(x) for x in row] for row in g["keys"]]
    v = [[F(x) for x in row] for row in g["values"]]
    q = [F(x) for x in g["q"]]
    W = [[F(col[r]) for col in g["W_columns"]] for r in range(2)]
    if mips:
        W.append([F(x) for x in g["W_mips_row"]])
    r = exact_ref.decode(k, v, q, W, 1, 3, 1, mips, 2, 0, 0)
    exp = g["mips1" if mips else "mips0"]
    assert r["counts"] == exp["counts"] and r["S"] == exp["S"]
    np.testing.assert_allclose(r["out"], exp["out"], rtol=1e-14)
    if mips:
        assert [float(x[2]) for x in r["xbar"]] == exp["s"]


# --------------------------------------------------------------------------- P7
def _fr_bf16(u16):
    return [[Fraction(float(x)) for x in row] for row in synth.bf16_bits_to_f32(u16).astype(np.float64)]


@pytest.mark.parametrize("seed", range(24))
def test_p7_bruteforce_tiny(seed):
    """Oracle == exact rational / 50-digit brute force on tiny cases."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 14))
    d = int(rng.integers(2, 7))
    K = int(rng.integers(1, 4))
    L = int(rng.integers(2, 5))
    mips = int(seed % 2)
    center = int((seed // 2) % 2) if seed < 20 else 1
    sink = int(rng.integers(0, 3))
    local = int(rng.integers(0, 3))
    minc = 1 if seed % 7 == 3 else 2
    case = synth.make_random_case(seed, n, d, 1, K, L, mips)
    # use small dyadic values so that exact zeros and ties happen
    kf = np.round(synth.bf16_bits_to_f32(case["k"]) * 2) / 2
    k = bf(kf.astype(np.float32))
    v, q, W = case["v"], case["q"][:1], case["W"]
    r = oracle.decode_unit(k, v, q, W, K, L, center, mips, minc, sink, local)
    assert r["status"] in (0, oracle.OR_EDEGENERATE)
    Wf = [[Fraction(float(x)) for x in row] for row in W.astype(np.float64)]
    e = exact_ref.decode(_fr_bf16(k), _fr_bf16(v), _fr_bf16(q)[0], Wf, K, L, center, mips, minc,
                         sink, local)
    assert [float(x) for x in e["c"]] == [float(x) for x in r["c"]]
    np.testing.assert_array_equal(np.array(e["codes"], np.uint16).reshape(n, L), r["codes"])
    assert e["qcode"] == [int(x) for x in r["qcodes"][0]]
    assert e["counts"] == [int(x) for x in r["counts"][0]]
    assert e["S"] == [i for i in range(n) if r["in_s"][0, i] == 1]
    for i, lu in e["logu"].items():
        assert math.isclose(r["logu"][0, i], lu, rel_tol=1e-12, abs_tol=1e-13)
    np.testing.assert_allclose(r["out"][0], e["out"], rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------------- P3
def _u_exact(p: Fraction, K: int, L: int) -> Fraction:
    x = p ** K
    return 1 - (1 - x) ** L - L * x * (1 - x) ** (L - 1)


def test_p3_special_values():
    assert oracle.sampling_prob(1.0, 10, 150) == 1.0
    assert oracle.sampling_prob(0.0, 10, 150) == 0.0
    assert oracle.sampling_prob(0.5, 1, 2) == pytest.approx(0.25, rel=1e-15)
    for p in [0.1, 0.37, 0.5, 0.8, 0.99]:
        for K in [1, 3, 8]:
            assert oracle.sampling_prob(p, K, 2) == pytest.approx(p ** (2 * K), rel=1e-12)
        assert oracle.sampling_prob(p, 1, 3) == pytest.approx(3 * p * p - 2 * p ** 3, rel=1e-12)
        # min_collisions = 1: classic LSH 1-(1-p^K)^L
        assert oracle.sampling_prob(p, 4, 7, 1) == pytest.approx(1 - (1 - p ** 4) ** 7, rel=1e-12)


@pytest.mark.parametrize("K,L,expected", [(10, 150, 0.0096836728), (8, 75, 0.0350831429),
                                          (11, 300, 0.0097100889)])
def test_p3_budget_exact_rationals(K, L, expected):
    """Eq. (budget) P:472-476 against exact rational arithmetic."""
    ex = float(_u_exact(Fraction(1, 2), K, L))
    assert abs(ex - expected) < 1e-10
    assert oracle.expected_budget(K, L) == pytest.approx(ex, rel=1e-12)


def test_p3_stable_form_matches_exact_rationals():
    """The rearranged u (reading R11) equals the printed formula in exact
    arithmetic over p in (0, 1], where the naive double form breaks down."""
    worst_naive = 0.0
    for K, L in [(10, 150), (8, 75), (11, 300), (7, 35), (9, 120)]:
        for i in range(1, 101):
            p = Fraction(i, 100)
            ex = _u_exact(p, K, L)
            got = oracle.sampling_prob(float(p), K, L)
            if ex > 0:
                assert abs(Fraction(got) - ex) / ex < Fraction(1, 10 ** 11), (K, L, i)
                naive = oracle.sampling_prob_naive(float(p), K, L)
                worst_naive = max(worst_naive, float(abs(Fraction(naive) - ex) / ex))
    assert worst_naive > 1e-3  # the printed form in double really is unusable at small p


# --------------------------------------------------------------------------- P11
def test_p11_monotonicity():
    ps = np.linspace(0.0, 1.0, 101)
    for K in range(1, 13):
        for L in [2, 5, 35, 75, 150, 300]:
            u = [oracle.sampling_prob(p, K, L) for p in ps]
            assert all(b >= a - 1e-15 for a, b in zip(u, u[1:]))
            for p in [0.3, 0.5, 0.7, 0.9]:
                assert oracle.sampling_prob(p, K, L + 1) >= oracle.sampling_prob(p, K, L) - 1e-15
                assert oracle.sampling_prob(p, K + 1, L) <= oracle.sampling_prob(p, K, L) + 1e-15


# --------------------------------------------------------------------------- P2
@pytest.mark.parametrize("theta", [math.pi / 6, math.pi / 3, math.pi / 2, 2 * math.pi / 3])
def test_p2_simhash_single_bit_law(theta):
    """Single-projection collision frequency = 1 - theta/pi."""
    d, T = 6, 100_000
    rng = np.random.default_rng(7)
    W = synth.bf16_bits_to_f32(bf(rng.standard_normal((d, T), dtype=np.float32)))
    x = np.zeros(d)
    y = np.zeros(d)
    x[0] = 1.0
    y[0], y[1] = math.cos(theta), math.sin(theta)
    xb = synth.bf16_bits_to_f32(bf(x.astype(np.float32))).astype(np.float64)
    yb = synth.bf16_bits_to_f32(bf(y.astype(np.float32))).astype(np.float64)
    cx = oracle.encode_vec(xb, W, 1, T)
    cy = oracle.encode_vec(yb, W, 1, T)
    freq = float(np.mean(cx == cy))
    th = math.acos(float(xb @ yb) / (np.linalg.norm(xb) * np.linalg.norm(yb)))
    p = 1 - th / math.pi
    assert oracle.collision_prob(math.cos(th)) == pytest.approx(p, rel=1e-12)
    sigma = math.sqrt(p * (1 - p) / T)
    assert abs(freq - p) < 3.5 * sigma


# --------------------------------------------------------------------------- P1
@pytest.mark.parametrize("p_target", [0.55, 0.6, 0.65, 0.7])
def test_p1_two_table_rule_monte_carlo(p_target):
    """Frequency of ">= 2 of L tables share the K-bit code" over freshly drawn
    Gaussian projections == u(p) of Eq. (LSH sampling probability),
    through the oracle's real encode path.  K=10, L=150, d=3, 2e4 trials."""
    K, L, d, T = 10, 150, 3, 20_000
    theta = (1 - p_target) * math.pi
    x = np.array([1.0, 0.0, 0.0])
    y = np.array([math.cos(theta), math.sin(theta), 0.0])
    xb = synth.bf16_bits_to_f32(bf(x.astype(np.float32))).astype(np.float64)
    yb = synth.bf16_bits_to_f32(bf(y.astype(np.float32))).astype(np.float64)
    cosv = float(xb @ yb) / (np.linalg.norm(xb) * np.linalg.norm(yb))
    u = oracle.sampling_prob(oracle.collision_prob(cosv), K, L)
    rng = np.random.default_rng(int(p_target * 1000))
    hits = 0
    for t0 in range(0, T, 1000):
        Wb = synth.bf16_bits_to_f32(bf(rng.standard_normal((1000, d, K * L), dtype=np.float32)))
        for t in range(1000):
            cx = oracle.encode_vec(xb, Wb[t], K, L)
            cy = oracle.encode_vec(yb, Wb[t], K, L)
            hits += int(np.count_nonzero(cx == cy) >= 2)
    freq = hits / T
    z = (freq - u) / math.sqrt(u * (1 - u) / T)
    assert abs(z) < 4.0, (freq, u, z)


# --------------------------------------------------------------------------- P4/P5/P9
@pytest.mark.parametrize("seed", range(20))
def test_p4_uniform_u_all_keys_is_exact_attention(seed):
    """With u == 1 and S = all keys the estimator is Softmax(qK^T/sqrt d)V."""
    rng = np.random.default_rng(seed)
    n, d = int(rng.integers(1, 300)), int(rng.choice([8, 64, 128]))
    c = synth.make_random_case(seed, n, d, 1, 2, 2, 0)
    sel = np.ones(n, np.uint8)
    est = oracle.estimate(c["q"][0], c["k"], c["v"], sel, np.zeros(n))
    ex = oracle.exact_attention(c["q"][0], c["k"], c["v"])
    np.testing.assert_allclose(est["out"], ex, rtol=1e-12, atol=1e-14)
    # same through the static path (sel=2, u implicitly 1)
    est2 = oracle.estimate(c["q"][0], c["k"], c["v"], 2 * sel, np.full(n, 123.0))
    np.testing.assert_allclose(est2["out"], ex, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("seed", range(6))
def test_p5_all_static_is_exact_attention(seed):
    """sink + local >= n: nothing is sampled, every key is static."""
    n, d = 40 + seed, 16
    c = synth.make_random_case(seed, n, d, 2, 3, 4, seed % 2)
    r = oracle.decode_unit(c["k"], c["v"], c["q"], c["W"], 3, 4, 1, seed % 2, 2, sink=10, local=n)
    for g in range(2):
        ex = oracle.exact_attention(c["q"][g], c["k"], c["v"])
        np.testing.assert_allclose(r["out"][g], ex, rtol=1e-12, atol=1e-14)
        assert r["s_count"][g] == 0


def test_p9_centering_translation_invariance():
    """Softmax is translation invariant: attention over k - c equals over k."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        n, d = 200, 32
        k = rng.standard_normal((n, d))
        v = rng.standard_normal((n, d))
        q = rng.standard_normal(d)
        c = rng.standard_normal(d) * 3
        a = oracle.exact_attention_f64(q, k, v)
        b = oracle.exact_attention_f64(q, k - c[None, :], v)
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)


# --------------------------------------------------------------------------- P6
@pytest.mark.parametrize("seed", range(4))
def test_p6_mips_transform_invariants(seed):
    """Eq. (data transform) P:49-55: |kbar_i| = r and qbar.kbar_i = q.k_i before
    the bf16 rounding of s_i; the stored s_i is that value rounded once."""
    n, d = 257, 128
    c = synth.make_random_case(seed, n, d, 1, 1, 2, 1)
    sink, local = 4, 16
    t = oracle.key_transform(c["k"], sink, local, center=1, mips=1)
    assert t["status"] == 0
    x = synth.bf16_bits_to_f32(t["xbar"][:, :d]).astype(np.float64)
    # n2 exact fixed point: sum_d trunc(x^2 2^64), by Python integers
    for i in [0, 5, 100, 256]:
        ex = sum((Fraction(float(a)) ** 2 * 2 ** 64).__floor__() for a in x[i])
        assert t["n2_q"][i] == ex
        assert t["n2"][i] == float(exact_ref.to_f64(Fraction(ex, 2 ** 64)))
    D = [i for i in range(n) if not oracle.is_static(i, n, sink, local)]
    assert t["r2_q"] == max(t["n2_q"][i] for i in D)
    # real-arithmetic invariants of Eq. (data transform), before rounding s_i:
    # |kbar_i|^2 = r^2 and qbar . kbar_i = q . x_i  (qbar = [q, 0])
    s_exact = np.array([math.sqrt(float(Fraction(t["r2_q"] - t["n2_q"][i], 2 ** 64))) for i in range(n)])
    for i in D[:50]:
        assert t["n2"][i] + s_exact[i] ** 2 == pytest.approx(t["r2"], rel=1e-12)
    qv = synth.bf16_bits_to_f32(c["q"][0]).astype(np.float64)
    qbar = np.append(qv, 0.0)
    kbar = np.hstack([x, s_exact[:, None]])
    np.testing.assert_allclose(kbar @ qbar, x @ qv, rtol=1e-12, atol=1e-12)
    # stored s_i = bf16_rn(sqrt_rn(fl64((r2q - n2q) 2^-64))), rounded through exact rationals
    stored = t["xbar"][:, d]
    expect = []
    for i in range(n):
        dq = t["r2_q"] - t["n2_q"][i]
        v = exact_ref.to_f64(Fraction(dq, 2 ** 64)) if dq > 0 else Fraction(0)
        expect.append(exact_bits(float(exact_ref.sqrt_f64(v))))
    np.testing.assert_array_equal(stored, np.array(expect, np.uint16))
    # centering vector: c = fl32(fl64(fl64(ksum 2^-64) / |D|))
    kf = synth.bf16_bits_to_f32(c["k"]).astype(np.float64)
    for j in [0, 17, 127]:
        ks = sum(int(Fraction(float(kf[i, j])) * 2 ** 64) for i in D)
        assert t["ksum_q"][j] == ks
        cj = exact_ref.to_f32(exact_ref.to_f64(exact_ref.to_f64(Fraction(ks, 2 ** 64)) / len(D)))
        assert float(t["c"][j]) == float(cj)


def exact_bits(s: float) -> int:
    """bf16 bits of RNE(s) computed through exact rationals."""
    r = exact_ref.to_bf16(Fraction(s))
    f = np.float32(float(r))
    return int(np.array([f]).view(np.uint32)[0] >> 16)


# --------------------------------------------------------------------------- P8
def test_p8_code_identities():
    rng = np.random.default_rng(11)
    d, K, L = 16, 8, 40
    W = synth.bf16_bits_to_f32(bf(rng.standard_normal((d, K * L), dtype=np.float32)))
    for _ in range(20):
        x = synth.bf16_bits_to_f32(bf(rng.standard_normal(d, dtype=np.float32))).astype(np.float64)
        cx = oracle.encode_vec(x, W, K, L)
        cn = oracle.encode_vec(-x, W, K, L)
        dots = x @ W.astype(np.float64)
        if np.all(dots != 0):
            np.testing.assert_array_equal(cn, (~cx) & ((1 << K) - 1))
    # a query equal to an indexed key collides in all L tables
    c = synth.make_random_case(5, 30, d, 1, K, L, 0)
    t = oracle.key_transform(c["k"], 0, 0, center=0, mips=0)
    codes = oracle.encode_keys(t["xbar"], c["W"], K, L)
    qc = oracle.encode_query(c["k"][7], c["W"], K, L, 0)
    assert oracle.collision_counts(codes, qc)[7] == L
    # x orthogonal to W_j -> bit 0 (sign(0) = 0, reading R6)
    W2 = np.zeros((2, 2), np.float32)
    W2[:, 0] = [1.0, 1.0]
    W2[:, 1] = [1.0, -1.0]
    assert list(oracle.encode_vec(np.array([1.0, -1.0]), W2, 2, 1)) == [0b10]
    assert list(oracle.encode_vec(np.array([1.0, 1.0]), W2, 2, 1)) == [0b01]


def test_exact_dot_sign_cancellation():
    """The sign is the sign of the exact value even when a double sum loses it."""
    a = np.array([2.0 ** 100, 1.0, -(2.0 ** 100)])
    b = np.ones(3)
    assert float(np.sum(a * b)) == 0.0  # the naive double sum loses the 1
    assert oracle.exact_dot_sign(a, b) == 1
    assert oracle.exact_dot_sign(a, -b) == -1
    assert oracle.exact_dot_sign(np.array([3.0, -3.0]), np.ones(2)) == 0
    rng = np.random.default_rng(0)
    for _ in range(300):
        m = int(rng.integers(1, 20))
        ex = rng.integers(-60, 60, size=m)
        a = np.ldexp(rng.integers(-255, 256, size=m).astype(np.float64), ex)
        b = np.ldexp(rng.integers(-255, 256, size=m).astype(np.float64), -ex)
        exact = sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b))
        assert oracle.exact_dot_sign(a, b) == (exact > 0) - (exact < 0)


def test_bf16_rounding_matches_exact():
    rng = np.random.default_rng(2)
    vals = np.concatenate([rng.standard_normal(2000) * 10.0 ** rng.integers(-40, 38, 2000),
                           [1 + 2.0 ** -8, 1 + 3 * 2.0 ** -8, 2.0 ** -133, 2.0 ** -134, 1e-45]])
    for v in vals:
        r = oracle.bf16_from_double(float(v))
        ex = exact_ref.to_bf16(Fraction(float(v)))
        assert oracle.bf16_to_double(r) == float(ex), v


# --------------------------------------------------------------------------- P10
@pytest.mark.parametrize("seed", range(25))
def test_p10_bucketed_tables_equal_bruteforce(seed):
    """Query through per-table buckets (the paper's HT) == direct
    recount of code matches."""
    rng = np.random.default_rng(seed)
    n, d, K, L = int(rng.integers(1, 400)), 8, int(rng.integers(1, 6)), int(rng.integers(2, 20))
    c = synth.make_random_case(seed, n, d, 1, K, L, 0)
    t = oracle.key_transform(c["k"], 0, 0, center=1, mips=0)
    codes = oracle.encode_keys(t["xbar"], c["W"], K, L)
    qc = oracle.encode_query(c["q"][0], c["W"], K, L, 0)
    np.testing.assert_array_equal(oracle.bucket_query(codes, qc, K), oracle.collision_counts(codes, qc))


# --------------------------------------------------------------------------- merge (P12 host half)
@pytest.mark.parametrize("P", [1, 2, 3, 7])
def test_merge_of_split_estimates_equals_whole(P):
    """LSE merge of partial states (recursive attention) == one softmax."""
    n, d = 300, 32
    c = synth.make_random_case(P, n, d, 1, 2, 2, 0)
    rng = np.random.default_rng(P)
    sel = rng.integers(0, 3, n).astype(np.uint8)
    logu = np.log(rng.uniform(0.01, 1.0, n))
    whole = oracle.estimate(c["q"][0], c["k"], c["v"], sel, logu)
    cuts = np.linspace(0, n, P + 1).astype(int)
    parts = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        e = oracle.estimate(c["q"][0], c["k"][a:b], c["v"][a:b], sel[a:b], logu[a:b])
        parts.append(np.concatenate([[e["m"], e["s"]], e["a"]]))
    np.testing.assert_allclose(oracle.merge_partials(np.array(parts)), whole["out"], rtol=1e-12, atol=1e-14)


def test_degenerate_empty_everything():
    """S and T both empty -> OR_EDEGENERATE and a zero output row."""
    c = synth.make_random_case(1, 20, 8, 1, 16, 2, 0)
    r = oracle.decode_unit(c["k"], c["v"], c["q"], c["W"], 16, 2, 1, 0, 2, sink=0, local=0)
    if r["s_count"][0] == 0:
        assert r["status"] == oracle.OR_EDEGENERATE
        assert np.all(r["out"] == 0)


def test_w_must_be_bf16_representable():
    c = synth.make_random_case(1, 8, 4, 1, 2, 2, 0)
    W = c["W"].copy()
    W[0, 0] = np.float32(1.0 + 2.0 ** -20)
    r = oracle.decode_unit(c["k"], c["v"], c["q"], W, 2, 2, 1, 0, 2, 0, 0)
    assert r["status"] == oracle.OR_ENOTREPR


# --------------------------------------------------------------------------- x = bf16(fl32(k - c)), wide operands
def test_centered_key_rounding_when_k_minus_c_is_inexact_in_double():
    """x_i = bf16_rn(fl32(k_i - c)) (C-2 contract) when |k| / |c| > 2^29: k - c then spans more than
    53 bits, so the oracle's fp64 difference is inexact and its pair rounding (f32_round_pair, the TwoSum residue
    branch) decides fl32.  Checked against exact rational rounding (tests/exact_ref.py), with keys near fp32 and
    bf16 rounding boundaries and centering vectors of both signs."""
    d = 128
    rng = np.random.default_rng(29)
    for trial in range(6):
        n = 12
        kf = np.zeros((n, d), np.float32)
        # dynamic keys (positions 1 .. 10 with sink 1, local 1): tiny values, |D| = 10 -> c has a full mantissa
        kf[1:11, :] = (rng.integers(-7, 8, (10, d)) * 2.0 ** (-12 - trial)).astype(np.float32)
        # the static keys carry large values: 2^18 +- a few bf16 ulps, and values just off bf16 midpoints
        big = 2.0 ** (16 + trial) * (1.0 + rng.integers(0, 128, d) / 128.0)
        kf[0, :] = big.astype(np.float32) * np.where(rng.random(d) < 0.5, -1.0, 1.0)
        kf[11, :] = (big * (1.0 + 2.0 ** -8)).astype(np.float32)
        k = synth.bf16_bits_from_f32(kf)
        t = oracle.key_transform(k, 1, 1, center=1, mips=0)
        assert t["status"] == 0
        kx = synth.bf16_bits_to_f32(k).astype(np.float64)
        c = t["c"].astype(np.float64)
        assert np.max(np.abs(kx[[0, 11]]) / np.maximum(np.abs(c), 1e-300)) > 2.0 ** 29
        for i in (0, 11):
            for j in range(d):
                exact = exact_ref.to_bf16(exact_ref.to_f32(Fraction(float(kx[i, j])) - Fraction(float(c[j]))))
                got = float(synth.bf16_bits_to_f32(t["xbar"][i:i + 1, j:j + 1])[0, 0])
                assert got == float(exact), (trial, i, j, got, float(exact))
