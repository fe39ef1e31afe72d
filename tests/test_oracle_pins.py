"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Each test names the passage (PAPER.md line / equation) or DESIGN.md reading it
pins, and is chosen so that a plausible slip (dropped term, wrong sign or index,
transposed operand) in the oracle fails at least one of them.  None of these
tests touches the CUDA path.
"""
import heapq
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- Lorenzo (A4)
@pytest.mark.parametrize("nd", [1, 2, 3])
def test_lorenzo_exact_on_linear_fields(orc, nd):
    """Lorenzo (PAPER.md:151 footnote) annihilates linear fields: every interior
    residual (all indices >= 1) is exactly 0; face residuals equal the slopes."""
    shape = {1: (37,), 2: (9, 13), 3: (6, 7, 9)}[nd]
    slopes = [0.5, -2.0, 0.25][:nd]
    grids = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
    x = (3.0 + sum(s * g for s, g in zip(slopes, grids))).astype(np.float32)
    for idx in np.ndindex(*shape):
        d = float(orc.lorenzo(x, idx))
        nz = [a for a in range(nd) if idx[a] == 0]
        if not nz and nd > 1:
            assert d == 0.0, idx
        elif not nz:                      # 1D Lorenzo is exact on constants only
            assert d == slopes[0], idx
        elif len(nz) == nd - 1 and nd > 0:
            # on an axis line through the origin: 1D Lorenzo along the nonzero axis
            a = [a for a in range(nd) if idx[a] != 0][0]
            assert d == slopes[a], (idx, d)
    # interior codes are all zero through the whole estimate
    r = orc.estimate(x, 1e-3, mode="rel", debug=True)
    codes = r["debug"]["codes"]
    inner = codes[tuple(slice(1, None) for _ in range(nd))]
    assert np.all(inner == 32767) if nd > 1 else len(np.unique(inner)) == 1


def test_lorenzo_3d_matches_7_neighbour_formula(orc):
    """3D Lorenzo = x - (x100+x010+x001 - x110-x101-x011 + x111) (PAPER.md:151, 7
    neighbours); on small-integer data fp32 arithmetic is exact, so the nested
    order must agree with the inclusion-exclusion sum exactly."""
    rng = np.random.default_rng(1)
    x = rng.integers(-50, 50, size=(5, 6, 7)).astype(np.float32)
    xp = np.zeros((6, 7, 8))
    xp[1:, 1:, 1:] = x
    for (i, j, k) in [(0, 0, 1), (2, 3, 4), (4, 5, 6), (1, 0, 3), (3, 2, 0)]:
        I, J, K = i + 1, j + 1, k + 1
        pred = (xp[I - 1, J, K] + xp[I, J - 1, K] + xp[I, J, K - 1] - xp[I - 1, J - 1, K]
                - xp[I - 1, J, K - 1] - xp[I, J - 1, K - 1] + xp[I - 1, J - 1, K - 1])
        assert float(orc.lorenzo(x, (i, j, k))) == xp[I, J, K] - pred


def test_constant_field_zero_entropy(orc):
    """A constant field has zero entropy (BASELINE north_star); SZ BR = offset 0.5
    (SPEC 'all-zero errors -> 0.5')."""
    x = np.full((12, 8), 3.5, np.float32)
    r = orc.estimate(x, 1e-3, mode="abs")
    assert r["sz_entropy"] == 0.0
    assert r["sz_bits_per_value"] == 0.5
    with pytest.raises(orc.OracleError) as e:
        orc.estimate(x, 1e-3, mode="rel")        # VR = 0 with a relative bound
    assert e.value.status == -5


def test_hand_example_2d(orc):
    g = gold("hand_2d_4x4.json")
    x = np.fromfunction(lambda i, j: i + 2 * j, (4, 4)).astype(np.float32)
    r = orc.estimate(x, g["eb_abs"], mode="abs", debug=True)
    codes = r["debug"]["codes"].astype(np.int64)
    exp = np.array(g["codes"])
    assert np.array_equal(np.where(codes >= 0, codes - 32767, -1), exp)
    for k in ("sz_entropy", "sz_bits_per_value", "value_range", "sz_psnr"):
        assert r[k] == pytest.approx(g[k], rel=1e-12), k


def test_power_of_two_scale_invariance(orc):
    """x -> 2^k x leaves every code, coefficient and bit count unchanged in rel
    mode and shifts every block exponent by k; PSNR_zfp is unchanged (A4/A9/A14)."""
    import synth
    x = synth.c1_field((40, 44), seed=3)
    a = orc.estimate(x, 1e-4, mode="rel", debug=True)
    for k in (-7, 5):
        y = (x.astype(np.float64) * 2.0 ** k).astype(np.float32)
        b = orc.estimate(y, 1e-4, mode="rel", debug=True)
        da, db = a["debug"], b["debug"]
        assert np.array_equal(da["codes"], db["codes"])
        assert np.array_equal(da["coef"], db["coef"])
        assert np.array_equal(da["bits"], db["bits"])
        assert np.array_equal(da["emax"] + k, db["emax"])
        assert b["zfp_psnr"] == pytest.approx(a["zfp_psnr"], rel=1e-12)
        assert b["sz_bits_per_value"] == a["sz_bits_per_value"]


# ------------------------------------------------------------- quantiser (A5)
def test_quantizer_linear_spec_examples(orc):
    """SPEC linear_spec: eb=0.5 -> bin width 1, midpoints -1,0,1; 0.4 -> centre bin.
    Bin width 2*eb."""
    r_f = np.float32(1.0 / (2 * 0.5))
    assert orc.quantize(0.4, r_f) == 32767
    assert orc.quantize(-0.4, r_f) == 32767
    assert orc.quantize(1.0, r_f) == 32768
    assert orc.quantize(-1.0, r_f) == 32766
    assert orc.quantize(0.6, r_f) == 32768
    # half-even ties (reading R5)
    assert orc.quantize(0.5, r_f) == 32767
    assert orc.quantize(1.5, r_f) == 32769
    assert orc.quantize(2.5, r_f) == 32769
    assert orc.quantize(-2.5, r_f) == 32765
    # overflow slot for |d|/(2eb) >= 32767.5, NaN and inf (reading R5)
    assert orc.quantize(32767.0, r_f) == 32767 + 32767
    assert orc.quantize(-32767.0, r_f) == 0
    assert orc.quantize(32767.5, r_f) == 65535
    assert orc.quantize(float("inf"), r_f) == 65535
    assert orc.quantize(float("nan"), r_f) == 65535


def test_quantizer_half_bin_bound(orc):
    """|d - 2eb*code| <= eb for every in-range residual (SZ error-bound contract)."""
    rng = np.random.default_rng(7)
    eb = 0.013
    r_f = np.float32(1.0 / (2.0 * eb))
    for d in rng.normal(0, 50 * eb, 2000).astype(np.float32):
        s = orc.quantize(d, r_f)
        assert s != 65535
        code = s - 32767
        assert abs(float(d) - 2 * eb * code) <= eb * (1 + 1e-6)


# --------------------------------------------------------------- entropy (A6)
def test_entropy_examples(orc):
    for c in gold("entropy_examples.json")["cases"]:
        assert orc.entropy(c["counts"]) == pytest.approx(c["H"], rel=1e-12, abs=1e-15)


def test_bitrate_uniform_four_bins(orc):
    """SPEC: uniform over 4 bins -> 2 + 0.5 = 2.5 bits (Eq. bitrate-sz with the offset)."""
    eb = 0.5
    steps = np.array([0.0, 1.0, 2.0, 3.0] * 10, np.float64)  # residual codes 0..3 cyclic
    x = np.concatenate([[0.0], np.cumsum(steps)]).astype(np.float32)
    # first residual after the origin is x[1]-x[0]=0, ..., 40 residuals, 10 per code
    r = orc.estimate(x, eb, mode="abs")
    assert r["sz_entropy"] == pytest.approx(2.0, rel=1e-14)
    assert r["sz_bits_per_value"] == pytest.approx(2.5, rel=1e-14)


def _huffman_len(counts):
    counts = [c for c in counts if c > 0]
    if len(counts) == 1:
        return counts[0]  # one symbol still needs 1 bit per value
    h = [(c, i, {i: 0}) for i, c in enumerate(counts)]
    heapq.heapify(h)
    nxt = len(counts)
    while len(h) > 1:
        a, _, da = heapq.heappop(h)
        b, _, db = heapq.heappop(h)
        m = {k: v + 1 for k, v in {**da, **db}.items()}
        heapq.heappush(h, (a + b, nxt, m))
        nxt += 1
    depth = h[0][2]
    return sum(counts[i] * depth[i] for i in depth)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_entropy_vs_actual_huffman(orc, seed):
    """Shannon bound: H <= L_huffman/N < H + 1 on the actual
    codes of tiny fields (brute-force Huffman coding of the slot sequence)."""
    import synth
    x = synth.c1_field((24, 20), seed=seed)
    r = orc.estimate(x, 1e-3, mode="rel", debug=True)
    hist = r["debug"]["hist"]
    N = int(hist.sum())
    assert N == r["n_sz_points"] == x.size - 1
    L = _huffman_len([int(c) for c in hist if c])
    H = r["sz_entropy"]
    assert H * N <= L + 1e-9
    assert L < (H + 1) * N


# ------------------------------------------------------------- SZ PSNR (A7)
def test_psnr_sz_table(orc):
    g = gold("psnr_sz_table.json")
    x = np.array([[0.0, 1.0], [0.25, 0.5]], np.float32)  # VR = 1
    for e, p in zip(g["eb_rel"], g["psnr_db"]):
        r = orc.estimate(x, e, mode="rel")
        assert r["sz_psnr"] == pytest.approx(p, rel=1e-12)


# -------------------------------------------------------------- lift (A8)
A = np.array([[4, 4, 4, 4], [5, 1, -1, -5], [-4, 4, 4, -4], [-2, 6, -6, 2]], dtype=object)
AF = [[Fraction(int(v), 16) for v in row] for row in A]
AINV = [[Fraction(v, 4) for v in row] for row in
        [[4, 6, -4, -1], [4, 2, 4, 5], [4, -2, 4, -5], [4, -6, -4, 1]]]


def _apply_sep(M, blk, nd):
    """Exact rational separable application of 4x4 matrix M along every axis."""
    t = np.array([Fraction(int(v)) for v in blk.ravel()], dtype=object).reshape((4,) * nd)
    for a in range(nd):
        t = np.moveaxis(t, a, 0)
        out = np.empty_like(t)
        for r in range(4):
            acc = sum(M[r][c] * t[c] for c in range(4))
            out[r] = acc
        t = np.moveaxis(out, 0, a)
    return t.ravel()


def test_matrix_pair_is_inverse():
    prod = [[sum(AINV[i][k] * AF[k][j] for k in range(4)) for j in range(4)] for i in range(4)]
    assert prod == [[Fraction(int(i == j)) for j in range(4)] for i in range(4)]
    # A is not orthogonal (reading R8): A A^T is not diagonal
    aat = [[sum(AF[i][k] * AF[j][k] for k in range(4)) for j in range(4)] for i in range(4)]
    assert aat[1][3] == Fraction(-8, 256)


@pytest.mark.parametrize("nd", [1, 2, 3])
def test_lift_linear_part_equals_A(orc, nd):
    rng = np.random.default_rng(nd)
    unit = 2 ** (4 * nd)
    for _ in range(20):
        blk = rng.integers(-2 ** 26 // unit, 2 ** 26 // unit, size=4 ** nd) * unit
        got = orc.fwd_xform(blk, nd)
        exp = _apply_sep(AF, blk, nd)
        assert all(Fraction(int(g)) == e for g, e in zip(got, exp))
        back = orc.inv_xform(got, nd)
        assert np.array_equal(back, blk)


def test_lift_examples(orc):
    c = 12345 * 16
    assert list(orc.fwd_xform(np.full(4, c), 1)) == [c, 0, 0, 0]
    s = 16 * 77
    assert list(orc.fwd_xform(np.array([0, s, 2 * s, 3 * s]), 1)) == [3 * s // 2, -s, 0, 0]
    # constant block in 3D: exactly (DC, 0, ..., 0) for ANY integer DC (A15)
    for dc in (1, -7, 2 ** 29 - 3):
        out = orc.fwd_xform(np.full(64, dc), 3)
        assert out[0] == dc and not out[1:].any()


@pytest.mark.parametrize("nd,tol", [(1, 4), (2, 16), (3, 64)])
def test_lift_round_trip_tolerance(orc, nd, tol):
    """Forward then inverse lift is within 2^(2d) integer units (north_star
    'within a stated tolerance'); inputs span the full 30-bit range."""
    rng = np.random.default_rng(100 + nd)
    worst = 0
    for _ in range(400):
        blk = rng.integers(-2 ** 30 + 1, 2 ** 30, size=4 ** nd)
        back = orc.inv_xform(orc.fwd_xform(blk, nd), nd).astype(np.int64)
        worst = max(worst, int(np.abs(back - blk).max()))
    assert worst <= tol


def test_paper_bot_family_orthogonal():
    """Paper's parametric T(t) is orthogonal for the five named
    transforms (self-test; ZFP's lift above is deliberately not, reading R8)."""
    for t in (0.0, 0.25, 2 / math.pi * math.atan(1 / 3), 2 / math.pi * math.atan(1 / 2), 0.5):
        s = math.sqrt(2) * math.sin(math.pi / 2 * t)
        c = math.sqrt(2) * math.cos(math.pi / 2 * t)
        T = 0.5 * np.array([[1, 1, 1, 1], [c, s, -s, -c], [1, -1, -1, 1], [s, -c, c, -s]])
        assert np.abs(T @ T.T - np.eye(4)).max() < 1e-12


# ------------------------------------------------------- reorder (A10)
def test_sequency_perm(orc):
    for nd in (1, 2, 3):
        p = orc.sequency_perm(nd)
        assert sorted(p) == list(range(4 ** nd))
        keys = []
        for n in p:
            idx = [(n // 4 ** (nd - 1 - a)) % 4 for a in range(nd)]
            keys.append((sum(idx), sum(i * i for i in idx), n))
        assert keys == sorted(keys)
    assert list(orc.sequency_perm(1)) == [0, 1, 2, 3]
    # 2D starts (0,0),(0,1),(1,0),(1,1),(0,2),(2,0)
    assert list(orc.sequency_perm(2)[:6]) == [0, 1, 4, 5, 2, 8]


# ------------------------------------------------------ negabinary (A11)
def _negabinary_value(u):
    return sum(((u >> k) & 1) * (-2) ** k for k in range(32))


def test_negabinary(orc):
    assert [orc.negabinary(c) for c in (0, 1, -1, 2, -2, 3)] == [0, 1, 3, 6, 2, 7]
    rng = np.random.default_rng(5)
    for c in list(rng.integers(-2 ** 31, 2 ** 31, 3000)) + [-2 ** 30 - 5, 2 ** 30 + 5]:
        u = orc.negabinary(int(c))
        assert orc.negabinary_inv(u) == int(c)
        if abs(int(c)) <= 2 ** 31 // 3:
            assert _negabinary_value(u) == int(c)


# ------------------------------------------------------------ BFP (A9)
def test_bfp_pins(orc):
    for case in gold("bfp_pins.json")["cases"]:
        if "block" in case:
            blk = np.array(case["block"], np.float32)
        else:
            blk = np.array([int(h, 16) for h in case["block_bits_hex"]], np.uint32).view(np.float32)
        e = orc.block_emax(blk)
        assert e == case["emax"]
        if case["ints"] is not None:
            assert list(orc.block_bfp(blk, e)) == case["ints"]


def test_bfp_range(orc):
    rng = np.random.default_rng(9)
    for _ in range(200):
        blk = (rng.standard_normal(64) * 10.0 ** rng.uniform(-30, 30)).astype(np.float32)
        e = orc.block_emax(blk)
        ints = orc.block_bfp(blk, e)
        assert np.abs(ints.astype(np.int64)).max() < 2 ** 30
        assert np.abs(ints.astype(np.int64)).max() >= 2 ** 28  # max value aligned to the top


# ------------------------------------------------------ precision (A12)
def test_precision_rule(orc):
    assert orc.precision(1, -14, 3) == 1 + 14 + 8
    assert orc.precision(-20, 0, 2) == 0
    assert orc.precision(100, -100, 1) == 32


# ------------------------------------------------- EC bit count (A13)
def test_gt_hand_example(orc):
    g = gold("gt_hand_1d.json")
    assert orc.gt_count(g["u"], g["kmin"]) == g["gt_bits"]


def test_gt_all_zero(orc):
    assert orc.gt_count(np.zeros(64, np.uint32), 0) == 32
    assert orc.gt_count(np.zeros(16, np.uint32), 10) == 22


def _random_words(rng, size):
    kind = rng.integers(0, 4)
    if kind == 0:   # staircase-shaped magnitudes
        top = rng.integers(0, 32)
        tops = np.sort(rng.integers(-1, top + 1, size))[::-1]
        return np.array([0 if t < 0 else (1 << int(t)) | int(rng.integers(0, 1 << int(t)) if t > 0 else 0)
                         for t in tops], np.uint32)
    if kind == 1:
        return rng.integers(0, 2 ** 32, size, dtype=np.uint64).astype(np.uint32)
    if kind == 2:
        u = np.zeros(size, np.uint32)
        u[rng.integers(0, size, 3)] = rng.integers(0, 2 ** 32, 3, dtype=np.uint64).astype(np.uint32)
        return u
    return (rng.integers(0, 2 ** 12, size) * (rng.random(size) < 0.3)).astype(np.uint32)


@pytest.mark.parametrize("nd", [1, 2, 3])
def test_gt_count_equals_written_stream(orc, nd):
    """The simulated count equals the length of an actually written EC bitstream,
    and that stream decodes back to the words truncated at kmin (north_star:
    'ZFP bit counts compared with actually bit-plane-encoding the blocks')."""
    rng = np.random.default_rng(11 + nd)
    size = 4 ** nd
    for _ in range(300):
        u = _random_words(rng, size)
        kmin = int(rng.integers(0, 33))
        n = orc.gt_count(u, kmin)
        buf, nw = orc.gt_encode(u, kmin)
        assert nw == n
        dec, nr = orc.gt_decode(buf, nw, size, kmin)
        assert nr == nw
        mask = 0 if kmin >= 32 else (0xFFFFFFFF ^ ((1 << kmin) - 1))
        assert np.array_equal(dec, u & np.uint32(mask))


def test_gt_monotone_in_kmin(orc):
    rng = np.random.default_rng(3)
    for _ in range(100):
        u = _random_words(rng, 64)
        counts = [orc.gt_count(u, k) for k in range(33)]
        assert all(a >= b for a, b in zip(counts, counts[1:]))
        assert counts[32] == 0


def test_gt_constant_block_closed_form(orc):
    """Constant block -> words (DC', 0...0); bits = 34 + F - 2 kmin for the top
    set bit F >= kmin of DC' (SURVEY 8(c) A15 derivation)."""
    rng = np.random.default_rng(4)
    for _ in range(300):
        nd = int(rng.integers(1, 4))
        size = 4 ** nd
        u = np.zeros(size, np.uint32)
        u[0] = int(rng.integers(1, 2 ** 32))
        F = int(u[0]).bit_length() - 1
        kmin = int(rng.integers(0, F + 1))
        assert orc.gt_count(u, kmin) == 34 + F - 2 * kmin


# --------------------------------------------- per-block header (A13, whole field)
@pytest.mark.parametrize("shape,kmin", [((8,), 17), ((8, 8), 15), ((8, 8, 8), 13)])
def test_header_constant_field_through_estimate(orc, shape, kmin):
    """The ZFP per-block header through the whole-field estimate (orc_estimate, not the
    gt_count helper): a constant field x = 1.0 gives emax = 1, i = 2^29 and, after the
    lift, the words (DC', 0, ..., 0) with DC' = negabinary(2^29) = 2^30 + 2^29 (digits 30
    and 29: (-2)^30 + (-2)^29 = 2^29), so F = 30.  With eb_abs = 2^-10 (minexp -10) the
    precision is p = 1 + 10 + 2(d+1), kmin = 32 - p, and every block costs
    header 9 + (34 + F - 2 kmin) bits ((31-F) negative tests, 3 bits at
    plane F, 2 per plane below).  A wrong header constant or cut rule fails this."""
    nd = len(shape)
    assert kmin == 32 - (1 + 10 + 2 * (nd + 1))
    x = np.ones(shape, np.float32)
    r = orc.estimate(x, 2.0 ** -10, mode="abs")
    nblocks = int(np.prod([n // 4 for n in shape]))
    per_block = 9 + 34 + 30 - 2 * kmin
    assert r["zfp_total_bits"] == nblocks * per_block
    assert r["n_blocks"] == nblocks


@pytest.mark.parametrize("shape", [(8,), (8, 8), (8, 8, 8)])
def test_header_precision_zero_block_costs_one_bit(orc, shape):
    """p = 0 (eb far above the block's magnitude, P:436 'maximum bit-plane determined by
    the error bound'): the block is a single header bit and its whole content is the error.
    Constant 1.0 field, eb_abs = 2^40: bits = 1 per block; the DC coefficient 2^29 is
    dropped, E_b = w_0 (2^29)^2 2^(2(1-30)) = 4^d (the block's squared-error sum), so
    MSE = 1.0 exactly -- the error of reconstructing 1.0 as 0."""
    x = np.ones(shape, np.float32)
    r = orc.estimate(x, 2.0 ** 40, mode="abs")
    nblocks = int(np.prod([n // 4 for n in shape]))
    assert r["zfp_total_bits"] == nblocks
    assert r["zfp_mse"] == 1.0


def test_header_golden_hand_count(orc):
    """tests/golden/gt_hand_1d.json: 42 EC bits + the 9-bit header = 51."""
    g = gold("gt_hand_1d.json")
    assert orc.gt_count(g["u"], g["kmin"]) + 9 == g["block_bits_with_header"] == 51


# -------------------------------------------- threaded oracle (bit-identical)
@pytest.mark.parametrize("shape,stride", [((37, 45, 70), None), ((203, 517), (1, 10)),
                                          ((1001,), None), ((20, 24, 36), (2, 1, 3))])
def test_threaded_oracle_is_bit_identical(orc, shape, stride):
    """orc_estimate_mt (slabs of blocks per thread, exact merges, E_b summed in block
    order) returns the single-threaded result bit for bit, dumps included."""
    rng = np.random.default_rng(sum(shape))
    x = np.cumsum(rng.standard_normal(shape), axis=-1).astype(np.float32)
    a = orc.estimate(x, 1e-4, stride=stride, debug=True, threads=1)
    for t in (2, 3, 7):
        b = orc.estimate(x, 1e-4, stride=stride, debug=True, threads=t)
        for k in a:
            if k == "debug":
                for kk in a[k]:
                    assert np.array_equal(a[k][kk], b[k][kk]), (t, kk)
            else:
                assert a[k] == b[k] or (a[k] != a[k] and b[k] != b[k]), (t, k)
    assert a["hist_total"] == a["n_sz_points"] == int(a["debug"]["hist"].sum())
    assert a["hist_ovf"] == int(a["debug"]["hist"][65535])


# ---------------------------------------------------------- error (A14)
def test_gain_weights_are_inverse_column_norms(orc):
    cn = [sum(AINV[r][c] ** 2 for r in range(4)) for c in range(4)]
    assert cn == [4, 5, 4, Fraction(13, 4)]
    assert orc.gain(3, 0) == 64.0
    assert orc.gain(3, 1 + 4 * 3 + 16 * 1) == 5 * 3.25 * 5
    assert orc.gain(2, 4 * 3 + 3) == 3.25 * 3.25


def _decode_block(orc, blk, nd, minexp):
    """Actual reconstruction: truncate words at kmin, undo negabinary/reorder,
    inverse lift, dequantise; returns (weighted estimate E_b, true squared error)."""
    size = 4 ** nd
    e = orc.block_emax(blk)
    ints = orc.block_bfp(blk, e)
    coef = orc.fwd_xform(ints, nd)
    perm = orc.sequency_perm(nd)
    u = np.array([orc.negabinary(int(coef[perm[j]])) for j in range(size)], np.uint32)
    p = orc.precision(e, minexp, nd)
    kmin = 32 - p
    mask = 0 if kmin >= 32 else (0xFFFFFFFF ^ ((1 << kmin) - 1))
    ct = np.zeros(size, np.int32)
    for j in range(size):
        ct[perm[j]] = orc.negabinary_inv(int(u[j]) & mask)
    rec = orc.inv_xform(ct, nd).astype(np.float64) * 2.0 ** (e - 30)
    true = float(((rec - blk.astype(np.float64)) ** 2).sum())
    est = orc.block_err(coef, u, nd, kmin, e)
    unweighted = 0.0
    for j in range(size):
        d = int(coef[perm[j]]) - int(ct[perm[j]])
        unweighted += float(d) ** 2
    unweighted *= 2.0 ** (2 * (e - 30))
    return est, true, unweighted, kmin


@pytest.mark.parametrize("nd", [2, 3])
def test_error_estimate_vs_actual_decode(orc, nd):
    """Gain-weighted truncation error (reading R14) matches the MSE
    of an actual decode within +-15% on smooth blocks; unit weights (the literal
    Theorem thm:1 premise) would be off by ~4^d."""
    rng = np.random.default_rng(20 + nd)
    E = T = U = 0.0
    for _ in range(300):
        g = np.meshgrid(*[np.arange(4.0)] * nd, indexing="ij")
        blk = rng.normal() + sum(rng.normal() * gi for gi in g) + 0.1 * sum(rng.normal() * gi * gi for gi in g)
        blk = blk + 0.02 * rng.standard_normal(blk.shape)
        blk = blk.astype(np.float32).ravel()
        minexp = int(rng.integers(-16, -8))
        est, true, unw, kmin = _decode_block(orc, blk, nd, minexp)
        assert kmin > 0
        E += est
        T += true
        U += unw
    assert 0.85 < E / T < 1.15
    assert U / T < 0.5


def test_error_zero_when_all_planes_kept(orc):
    rng = np.random.default_rng(8)
    for nd in (1, 2, 3):
        blk = rng.standard_normal(4 ** nd).astype(np.float32)
        e = orc.block_emax(blk)
        coef = orc.fwd_xform(orc.block_bfp(blk, e), nd)
        perm = orc.sequency_perm(nd)
        u = np.array([orc.negabinary(int(coef[p])) for p in perm], np.uint32)
        assert orc.block_err(coef, u, nd, 0, e) == 0.0
        # kmin = 32 drops everything: E = sum w c^2 2^(2(e-30))
        full = sum(orc.gain(nd, n) * float(coef[n]) ** 2 for n in range(4 ** nd)) * 2.0 ** (2 * (e - 30))
        assert orc.block_err(coef, u, nd, 32, e) == pytest.approx(full, rel=1e-14)


# ------------------------------------------------------ ZFP rate (A15)
@pytest.mark.parametrize("shape", [(16,), (8, 12), (4, 8, 8)])
def test_all_zero_field_rate(orc, shape):
    """Empty blocks cost the 1-bit header only -> 1/4^d bits per value."""
    x = np.zeros(shape, np.float32)
    r = orc.estimate(x, 1e-3, mode="abs")
    assert r["zfp_bits_per_value"] == pytest.approx(1.0 / 4 ** len(shape), rel=1e-15)
    assert r["zfp_mse"] == 0.0 and r["zfp_psnr"] == math.inf


# ------------------------------------------------------ selection (A16)
def test_delta_inversion(orc):
    """Alg. 1 line 7: delta from PSNR_sz = PSNR_zfp (Eq. psnr-pdf-linear).
    VR = 1 at 84.77 dB -> delta = 2e-4 (SPEC example); round trip to 1e-12."""
    psnr = 80.0 + 10 * math.log10(3.0)
    ch, bm, ebm, m = orc.select(3.0, psnr, 5.0, psnr, 1.0, 1e-4, 1e-9)
    assert m == 1
    assert ebm * 2 == pytest.approx(2e-4, rel=1e-12)
    assert bm == pytest.approx(3.0, rel=1e-12)        # same PSNR -> same bin -> same rate
    assert ch == 0
    # ZFP 6.02 dB better -> SZ needs one more bit per value
    ch, bm, ebm, m = orc.select(3.0, psnr, 3.9, psnr + 20 * math.log10(2.0), 1.0, 1e-4, 1e-9)
    assert bm == pytest.approx(4.0, rel=1e-12) and ch == 1


def test_selection_ties_and_unmatched(orc):
    psnr = 60.0
    ch, bm, _, m = orc.select(4.0, psnr, 4.0, psnr, 2.0, 2e-3 / math.sqrt(3) * 1.0, 1.0)
    # construct an exact tie through the unmatched path: MSE = 0
    ch, bm, ebm, m = orc.select(4.0, psnr, 4.0, math.inf, 2.0, 1e-3, 0.0)
    assert m == 0 and ch == 1 and bm == 4.0 and ebm == 1e-3     # tie -> ZFP
    ch, *_ = orc.select(3.9, psnr, 4.0, math.inf, 2.0, 1e-3, 0.0)
    assert ch == 0
    ch, bm, ebm, m = orc.select(4.0, -math.inf, 1.0, -math.inf, 0.0, 1e-3, 0.5)  # VR = 0
    assert m == 0 and ch == 1


def test_fixed_error_bound_selector_differs_from_rate_distortion(orc):
    """the selector of Lu et al. takes the higher compression ratio at the
    user's eb; "ZFP may have a higher PSNR than does SZ, even if its compression ratio is
    lower", which is where the rate-distortion selection (Alg. 1) disagrees with it."""
    psnr_sz = 20 * math.log10(1.0 / 1e-4) + 10 * math.log10(3.0)
    # ZFP 12.04 dB better than SZ at eb: SZ needs 2 more bits/value to match
    ch, bm, _, m = orc.select(3.0, psnr_sz, 3.5, psnr_sz + 20 * math.log10(4.0), 1.0, 1e-4, 1e-9)
    assert m == 1 and bm == pytest.approx(5.0, rel=1e-12) and ch == 1          # Alg. 1: ZFP
    assert orc.select_eb(3.0, 3.5) == 0                                        # Lu et al.: SZ
    assert orc.select_eb(3.5, 3.5) == 1                                        # tie -> ZFP
    assert orc.select_eb(4.0, 3.5) == 1


def test_fixed_error_bound_selector_on_fields(orc):
    """choice_eb is the lower bit-rate at eb; where matching is impossible (MSE = 0) the
    Alg. 1 fallback compares at eb too, so both selectors agree there."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((37, 45)).astype(np.float32)
    r = orc.estimate(x, 1e-3)
    assert r["choice_eb"] == (0 if r["sz_bits_per_value"] < r["zfp_bits_per_value"] else 1)
    xi = rng.integers(-3, 4, (20, 24)).astype(np.float32)        # exact in fp32, MSE = 0 at kmin = 0
    r = orc.estimate(xi, 2.0 ** -20, mode="abs")
    assert r["matched"] == 0 and r["zfp_mse"] == 0.0
    assert r["choice"] == r["choice_eb"]


# ------------------------------------------------------ sampling (A3)
def test_processed_block_counts(orc):
    assert orc.processed_blocks((1800, 3600), (1, 10)) == 40500
    assert orc.processed_blocks((1800, 3600), (1, 1)) == 405000
    assert orc.processed_blocks((512, 512, 512), (4, 4, 4)) == 32768
    assert orc.processed_blocks((100, 500, 500), None) == 25 * 125 * 125


@pytest.mark.parametrize("shape,stride", [((21, 30), (2, 3)), ((9, 10, 13), (2, 1, 3)), ((50,), (4,))])
def test_sampled_codes_are_restriction_of_full(orc, shape, stride):
    """Prediction uses original real neighbours: the sampled codes
    equal the full-field codes restricted to the processed blocks."""
    import synth
    rng = np.random.default_rng(2)
    x = (synth.grf(shape, 2.5, rng) * 3).astype(np.float32)
    full = orc.estimate(x, 1e-3, mode="rel", debug=True)["debug"]["codes"]
    samp = orc.estimate(x, 1e-3, mode="rel", stride=stride, debug=True)
    sc = samp["debug"]["codes"]
    mask = np.ones(shape, bool)
    for a, s in enumerate(stride):
        idx = (np.arange(shape[a]) // 4) % s == 0
        sh = [1] * len(shape)
        sh[a] = shape[a]
        mask &= idx.reshape(sh)
    mask.flat[0] = False
    assert np.array_equal(sc[mask], full[mask])
    assert np.all(sc[~mask] == -1)
    assert samp["n_sz_points"] == int(mask.sum())


def test_partial_blocks_edge_replication(orc):
    """Dims not multiple of 4 (reading R17): N_P counts real values only, padded
    slots replicate the last real plane; one ragged block equals its padded copy."""
    rng = np.random.default_rng(6)
    x = rng.standard_normal((5, 6)).astype(np.float32)
    r = orc.estimate(x, 1e-2, mode="rel", debug=True)
    assert r["n_values"] == 30 and r["n_blocks"] == 4
    pad = np.pad(x, ((0, 3), (0, 2)), mode="edge")
    rp = orc.estimate(pad, r["eb_abs"], mode="abs", debug=True)
    assert np.array_equal(r["debug"]["coef"], rp["debug"]["coef"])
    assert np.array_equal(r["debug"]["bits"], rp["debug"]["bits"])


# ------------------------------------------------------ errors (A1/A2)
def test_error_statuses(orc):
    x = np.ones((4, 4), np.float32)
    x[1, 1] = np.nan
    with pytest.raises(orc.OracleError) as e:
        orc.estimate(x, 1e-3, mode="abs")
    assert e.value.status == -4
    y = np.arange(16, dtype=np.float32).reshape(4, 4)
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(orc.OracleError) as e:
            orc.estimate(y, bad, mode="abs")
        assert e.value.status == -1
    with pytest.raises(orc.OracleError) as e:
        orc.estimate(np.ones(1, np.float32), 1e-3, mode="abs")   # no SZ point at all
    assert e.value.status == -5


def test_full_estimate_sanity_c1(orc):
    """Order-of-magnitude context: smooth field -> SZ BR a few
    bits, ZFP BR a few more, ZFP over-preserves PSNR."""
    import synth
    x = synth.c1_field()
    r = orc.estimate(x, 1e-4, mode="rel")
    assert r["n_values"] == 65536 and r["n_sz_points"] == 65535
    assert 2.0 < r["sz_bits_per_value"] < 12.0
    assert 2.0 < r["zfp_bits_per_value"] < 16.0
    assert r["zfp_psnr"] > r["sz_psnr"]
    assert r["matched"] == 1
    assert r["sz_eb_matched"] < r["eb_abs"]


# ------------------------------------------------------ N2: paper-literal estimator
@pytest.mark.parametrize("nd,m", [(1, 3), (2, 9), (3, 16)])
def test_paper_sample_positions(orc, nd, m):
    """3 / 9 / 16 sampled points per 1D / 2D / 3D block; reading R19: evenly spaced
    over the sequency order, first and last coefficient included."""
    pos = orc.paper_positions(nd)
    L = 4 ** nd - 1
    assert len(pos) == m and pos[0] == 0 and pos[-1] == L
    assert np.all(np.diff(pos) > 0)
    # evenly spaced: every position within half a step of i L / (m - 1)
    assert np.all(np.abs(pos - np.arange(m) * L / (m - 1)) <= 0.5)


def _nsb(u, kmin):
    u = int(u)
    return max(0, u.bit_length() - 1 - kmin + 1) if u else 0


@pytest.mark.parametrize("nd", [1, 2, 3])
def test_paper_block_interpolation_and_error(orc, nd):
    """orc_block_paper against the definitions written independently: n_sb at the samples
    (leading one down to the cut, A13), numpy.interp of n_sb over every sequency position
    (P:448-449), and the sampled error = value of the dropped negabinary planes
    ((u & low) ^ M) - M (a different formula from the oracle's c - c~) times the block
    exponent offset, squared."""
    rng = np.random.default_rng(40 + nd)
    size = 4 ** nd
    pos = orc.paper_positions(nd)
    for _ in range(200):
        # a staircase-like sequency vector: magnitudes decaying with j, random signs
        mag = (2.0 ** (rng.uniform(0, 29, size) * np.exp(-np.arange(size) / rng.uniform(2, 30))))
        c = (mag * rng.choice([-1, 1], size)).astype(np.int64).clip(-(1 << 30) + 1, (1 << 30) - 1)
        u = np.array([orc.negabinary(int(v)) for v in c], np.uint32)
        kmin = int(rng.integers(0, 33))
        emax = int(rng.integers(-20, 20))
        n2, mse = orc.block_paper(u, nd, kmin, emax)
        ns = np.array([_nsb(u[p], kmin) for p in pos], np.float64)
        interp = np.interp(np.arange(size), pos, ns)
        assert abs(n2 - 2.0 * interp.sum()) < 1e-6, (n2, 2 * interp.sum())
        low = (1 << kmin) - 1
        M = 0xAAAAAAAA & low
        ref = 0.0
        for p in pos:
            e = ((int(u[p]) & low) ^ M) - M
            ref += float(e) * float(e) * 2.0 ** (2 * (emax - 30))
        assert math.isclose(mse, ref, rel_tol=1e-12, abs_tol=0.0) or (mse == 0.0 and ref == 0.0)
    # constant n_sb over the block -> 2 * size * n exactly
    u = np.full(size, 0b101 << 10, np.uint32)
    n2, _ = orc.block_paper(u, nd, 8, 0)
    assert n2 == 2 * size * (12 - 8 + 1)


def test_paper_estimate_properties(orc):
    """Alg. 1 lines 3-10 as printed: delta from PSNR_sp by Eq. psnr-pdf-linear,
    BR_zfp = average interpolated n_sb, choice by line 10."""
    import synth
    x = synth.c1_field()
    r = orc.estimate_paper(x, 1e-4)
    assert r["status"] == 0 and r["matched"] == 1
    assert r["n_samples"] == 9 * 4096 and r["n_values"] == 65536
    assert r["zfp_nsb_bits"] == r["nsb2_total"] / 2 / r["n_values"]
    # delta = VR sqrt(12) 10^(-PSNR_sp / 20)   (Eq. psnr-pdf-linear with PSNR_sz = PSNR_sp)
    d = r["value_range"] * math.sqrt(12.0) * 10.0 ** (-r["zfp_psnr_sp"] / 20.0)
    assert math.isclose(r["sz_delta"], d, rel_tol=1e-12)
    assert math.isclose(r["zfp_psnr_sp"], 20 * math.log10(r["value_range"]) - 10 * math.log10(r["zfp_mse_sp"]),
                        rel_tol=1e-14)
    assert r["hist_total"] == 65535
    assert r["choice"] == (0 if r["sz_bits"] < r["zfp_nsb_bits"] else 1)
    # the literal reading's unit weights make PSNR_sp optimistic vs the gain-weighted PSNR
    # (~4^d low MSE in 2D)
    g = orc.estimate(x, 1e-4)
    assert r["zfp_psnr_sp"] > g["zfp_psnr"] + 6.0


def test_paper_unmatched_equals_regular_sz(orc):
    """No truncation at any sample (a tiny absolute bound: p = 32, kmin = 0) -> MSE_sp = 0,
    no PSNR to match: SZ at the user's bound, delta = 2 eb_abs (R16 ii), and then the
    re-quantised SZ estimate IS the regular one (same bins), bit for bit."""
    rng = np.random.default_rng(5)
    x = (1.0 + 0.25 * rng.standard_normal((24, 40))).astype(np.float32)
    eb = 2.0 ** -40
    r = orc.estimate_paper(x, eb, mode="abs")
    g = orc.estimate(x, eb, mode="abs")
    assert r["zfp_mse_sp"] == 0.0 and math.isinf(r["zfp_psnr_sp"]) and r["matched"] == 0
    assert r["sz_delta"] == 2 * eb
    assert r["sz_bits"] == g["sz_bits_per_value"] and r["hist_total"] == g["hist_total"]


def test_paper_sampled_blocks(orc):
    """Alg. 1 line 3: with strides, only the processed blocks enter both the
    ZFP samples and the SZ residual histogram."""
    import synth
    x = synth.c2_field(1, shape=(80, 160))
    r = orc.estimate_paper(x, 1e-4, stride=(1, 10))
    nb = orc.processed_blocks(x.shape, (1, 10))
    assert r["n_samples"] == 9 * nb
    assert r["hist_total"] == 16 * nb - 1          # every real point but the origin


# ------------------------------------------------------ N3: the ZFP stream (Alg. 1 line 13)
def _stream_cases():
    import synth
    return [("c1", synth.c1_field(), 1e-4, None), ("c1-loose", synth.c1_field(), 1e-2, None),
            ("c3", synth.c3_field(0, shape=(37, 45, 70)), 1e-3, None),
            ("c3-zeros", synth.c3_field(5, shape=(37, 45, 70)), 1e-5, None),
            ("c5-noise", synth.c5_field(2, shape=(32, 48, 64)), 1e-6, None),
            ("c4", synth.c4_field(0, shape=(64, 64, 64)), 1e-4, None),
            ("c2-sampled", synth.c2_field(3, shape=(120, 400)), 1e-4, (1, 10)),
            ("1d-odd", np.cumsum(np.random.default_rng(1).standard_normal(10001)).astype(np.float32), 1e-3, None)]


@pytest.mark.parametrize("i", range(8))
def test_zfp_stream_length_and_accuracy(orc, i):
    """The stream ACTUALLY written for Alg. 1 line 13 (fixed accuracy at eb) has
    exactly the length the estimator counted (sum of per-block header + EC bits, A13/A15),
    decodes within the error bound (max |x - x^| <= eb_abs), and its real MSE is within
    +-10 % of the gain-weighted estimate (A14; the literal unit-weight reading is >4x off)."""
    name, x, eb, stride = _stream_cases()[i]
    r = orc.estimate(x, eb, stride=stride)
    buf, nbits = orc.zfp_stream(x, eb, stride=stride)
    assert nbits == r["zfp_total_bits"], name
    y = orc.zfp_stream_decode(buf, nbits, x.shape, eb, r["value_range"], stride=stride)
    if stride is None:
        err = np.abs(y.astype(np.float64) - x)
        assert err.max() <= r["eb_abs"], (name, err.max(), r["eb_abs"])
        mse = float((err ** 2).mean())
        if r["zfp_mse"] > 0:
            assert 0.9 <= mse / r["zfp_mse"] <= 1.1, (name, mse, r["zfp_mse"])
        else:
            assert mse == 0.0


def test_zfp_stream_empty_and_constant(orc):
    """All-zero field: one 0 bit per block.  Constant block: header + the A15 closed form."""
    z = np.zeros((8, 12), np.float32)
    buf, nbits = orc.zfp_stream(z, 1e-3, mode="abs")
    assert nbits == 6 and not buf.any()
    c = np.full((4, 4, 4), 3.0, np.float32)
    buf, nbits = orc.zfp_stream(c, 1e-3, mode="abs")
    r = orc.estimate(c, 1e-3, mode="abs")
    assert nbits == r["zfp_total_bits"]
    y = orc.zfp_stream_decode(buf, nbits, c.shape, 1e-3, r["value_range"], mode="abs")
    assert np.abs(y - c).max() <= 1e-3


# ---------------------------------------------------------------- N4: variant quantisers
def _hist_of(codes):
    h = np.zeros(65536, np.uint64)
    for q, c in codes.items():
        h[32767 + int(q)] = c
    return h


def test_variants_hand_example(orc):
    """SURVEY 8(f) N4, reading R21: the log-scale and equal-probability
     quantisers evaluated with Eq. bit-rate-pdf and MSE = (1/12)
    sum delta_i^2 P_i on a 4-cell PDF, against values worked by hand
    (tests/golden/variants_hand.json)."""
    g = gold("variants_hand.json")
    r = orc.variants_from_hist(_hist_of(g["hist"]), g["value_range"], g["eb_abs"], g["log_base"], g["eqp_n"])
    delta = 2 * g["eb_abs"]
    H = -sum(p * math.log2(p) for p in g["log_bins_P"])
    assert r["log_bits"] == pytest.approx(H, rel=1e-14) and r["log_bins"] == 2
    assert r["log_mse"] == pytest.approx(g["log_mse_times_12"] * delta ** 2 / 12, rel=1e-14)
    assert 12 * r["log_mse"] == pytest.approx(
        sum(p * (w * delta) ** 2 for p, w in zip(g["log_bins_P"], g["log_bin_widths_cells"])), rel=1e-14)
    e = g["eqp_edges_cells"]
    assert r["eqp_mse"] == pytest.approx(sum((b - a) ** 2 for a, b in zip(e, e[1:])) * delta ** 2 / 36, rel=1e-14)
    assert r["eqp_mse"] == pytest.approx(g["eqp_mse_times_36"] / 36, rel=1e-14)
    assert r["eqp_bits"] == g["eqp_bits"] and r["lin_bits"] == g["lin_bits"]
    assert r["eqp_width_sum"] == pytest.approx(4.0, rel=1e-14)
    for k in ("log", "eqp"):
        assert r[k + "_psnr"] == pytest.approx(20 * math.log10(g["value_range"]) - 10 * math.log10(r[k + "_mse"]), rel=1e-14)


def test_variants_closed_forms(orc):
    """Closed forms the equations fix: (i) a base above every |code| leaves one log bin:
    BR = 0 and MSE = ((2b-1) delta)^2 / 12; (ii) equal counts in 2n-1 adjacent cells: the
    equal-probability bins ARE the cells, so its MSE and PSNR are the linear quantiser's
    delta^2 / 12 and Eq. psnr-pdf-linear, and BR = 1 + log2 n; (iii) all the
    mass in one cell: 2n-1 equal slices of width delta / (2n-1); (iv) the linear BR is the
    Shannon entropy of the counts and its PSNR equals Eq. psnr-sz."""
    eb, vr = 0.25, 100.0
    delta = 2 * eb
    h = _hist_of({-5: 7, 0: 100, 3: 9, 11: 1})
    r = orc.variants_from_hist(h, vr, eb, 12, 3)
    assert r["log_bits"] == 0.0 and r["log_bins"] == 1
    assert r["log_mse"] == pytest.approx((23 * delta) ** 2 / 12, rel=1e-14)
    assert r["lin_bits"] == pytest.approx(-sum(c / 117 * math.log2(c / 117) for c in (7, 100, 9, 1)), rel=1e-14)
    assert r["lin_psnr"] == pytest.approx(-20 * math.log10(eb / vr) + 10 * math.log10(3), rel=1e-13)
    for n in (1, 2, 5, 64):
        m = n - 1
        u = _hist_of({q: 13 for q in range(-m, m + 1)})
        r = orc.variants_from_hist(u, vr, eb, 2, n)
        assert r["eqp_mse"] == pytest.approx(delta ** 2 / 12, rel=1e-13)
        assert r["eqp_psnr"] == pytest.approx(r["lin_psnr"], rel=1e-13)
        assert r["eqp_bits"] == pytest.approx(1 + math.log2(n), rel=1e-15)
        one = _hist_of({4: 1000})
        r = orc.variants_from_hist(one, vr, eb, 2, n)
        assert r["eqp_mse"] == pytest.approx((delta / (2 * n - 1)) ** 2 / 12, rel=1e-12)
        assert r["eqp_width_sum"] == pytest.approx(1.0, rel=1e-12)


def test_variants_brute_force_from_residuals(orc):
    """Brute force through the whole estimate: the log-scale bins by math.log per code and the
    equal-probability edges as quantiles of the sorted codes, from the field's own codes
    (independent of the oracle's histogram walk); merging cells can only lower the entropy
    and raise the MSE (BR_log <= BR_lin, MSE_log >= delta^2 / 12); the widths tile the
    occupied support."""
    rng = np.random.default_rng(7)
    g = np.cumsum(np.cumsum(rng.standard_normal((48, 60)), 0), 1).astype(np.float32)
    for eb, b, n in ((1e-3, 2, 16), (1e-4, 3, 128), (3e-3, 10, 7)):
        full = orc.estimate(g, eb, debug=True)
        codes = full["debug"]["codes"].ravel()
        q = codes[(codes >= 0) & (codes < 65535)].astype(np.int64) - 32767
        r = orc.estimate_variants(g, eb, log_base=b, eqp_n=n)
        assert r["n_in"] == q.size and r["hist_ovf"] == int((codes == 65535).sum())
        delta = 2 * full["eb_abs"]
        # log-scale: bin id per code
        ids = []
        for v in q:
            a = abs(int(v))
            if a < b:
                ids.append(0)
                continue
            i = int(math.floor(math.log(a, b) + 1e-12))
            while b ** i > a:
                i -= 1
            while b ** (i + 1) <= a:
                i += 1
            ids.append(i if v > 0 else -i)
        ids = np.array(ids)
        H = M = 0.0
        for i in np.unique(ids):
            p = float((ids == i).mean())
            w = (2 * b - 1) if i == 0 else (b ** (abs(i) + 1) - b ** abs(i))
            H -= p * math.log2(p)
            M += p * (w * delta) ** 2 / 12
        assert r["log_bits"] == pytest.approx(H, rel=1e-10)
        assert r["log_mse"] == pytest.approx(M, rel=1e-10)
        assert r["log_bits"] <= r["lin_bits"] + 1e-12 and r["log_mse"] >= delta ** 2 / 12 * (1 - 1e-12)
        # equal-probability: the quantiles from the SORTED codes (no histogram): the unit of
        # mass number floor(k N / K) sits in cell qs[floor(k N / K)], at the fraction of that
        # cell's samples below it
        qs = np.sort(q)
        N, K = qs.size, 2 * n - 1
        s = [qs[0] - 0.5]
        for k in range(1, K):
            m = Fraction(k * N, K)
            cell = int(qs[int(m)])
            below = int(np.searchsorted(qs, cell, side="left"))
            inside = int(np.searchsorted(qs, cell, side="right")) - below
            s.append(cell - 0.5 + float((m - below) / inside))
        s.append(qs[-1] + 0.5)
        mse = float(((np.diff(np.array(s, dtype=np.float64)) * delta) ** 2).sum() / (12 * K))
        assert r["eqp_width_sum"] == pytest.approx(float(qs[-1] - qs[0] + 1), rel=1e-12)
        assert r["eqp_mse"] == pytest.approx(mse, rel=1e-10)
        assert r["eqp_bits"] == 1 + math.log2(n)


def test_variants_invalid_arguments(orc):
    h = _hist_of({0: 1})
    for b, n in ((1, 4), (2, 0), (2, 40000)):
        with pytest.raises(Exception):
            orc.variants_from_hist(h, 1.0, 0.1, b, n)
    with pytest.raises(Exception):
        orc.variants_from_hist(np.zeros(65536, np.uint64), 1.0, 0.1, 2, 4)   # no mass
