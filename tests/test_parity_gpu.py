"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): bit-exact quantisation codes, histograms, block
exponents, lifted int32 coefficients, negabinary words and per-block bit counts;
entropy, bit-rates and PSNRs within 1e-6 relative; choices 100% equal.
Inputs are the seeded synthetic generators in synth/ (DESIGN.md section 4).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

REL = 1e-6
EXACT_KEYS = ("n_sz_points", "n_values", "n_blocks", "zfp_total_bits", "minexp", "r_f", "choice_eb",
              "choice", "matched", "value_range", "eb_abs", "hist_total", "hist_ovf")
CLOSE_KEYS = ("sz_entropy", "sz_bits_per_value", "sz_psnr", "zfp_bits_per_value", "zfp_psnr",
              "zfp_mse", "zfp_err_sum", "sz_bits_matched", "sz_eb_matched", "sz_overflow_frac")


@pytest.fixture(scope="module")
def sel():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_1806_08901_b200 import build
    build.build()
    import paper_1806_08901_b200 as sel
    return sel


def close(a, b, rel=REL, abs_=0.0):
    """|a - b| <= rel * max(|a|, |b|): relative only (0 == 0 passes; no absolute floor,
    so tiny MSEs of small-scale fields are compared at full relative precision)."""
    if isinstance(a, float) and (math.isinf(a) or math.isinf(b)):
        return a == b
    return abs(a - b) <= max(rel * max(abs(a), abs(b)), abs_)


NEAR_TIE = 1e-9


def tie_margin(r) -> float:
    """Relative margin of Alg. 1 line 10's comparison, |BR_sz* - BR_zfp| / BR_zfp (SURVEY
    8(c) A16(iv)): a flip between two implementations needs a margin near 1e-12."""
    a, b = float(r["sz_bits_matched"]), float(r["zfp_bits_per_value"])
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


def compare_scalars(g, o, tag=""):
    for k in EXACT_KEYS:
        assert g[k] == o[k], (tag, k, g[k], o[k])
    for k in CLOSE_KEYS:
        assert close(float(g[k]), float(o[k])), (tag, k, g[k], o[k])
    assert g["status"] == 0
    assert g["hist_total"] == g["n_sz_points"], tag       # no code lost or duplicated


def run_gpu(sel, x, eb, mode="rel", stride=None, debug=False, offset_elems=0):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    if offset_elems:
        buf = torch.empty(x.size + offset_elems, dtype=torch.float32, device="cuda")
        buf[offset_elems:] = t.reshape(-1)
        t = buf[offset_elems:].view(x.shape)
    with sel.Plan(x.shape, eb, mode, stride) as p:
        if debug:
            p.set_option("debug", 1)
        r = p.estimate(t)
        dbg = {k: p.debug_copy(k) for k in ("codes", "hist", "emax", "coef", "uword", "bits", "err")} \
            if debug else None
    return r, dbg


def check_case(sel, orc, x, eb, mode="rel", stride=None, offset_elems=0, tag=""):
    o = orc.estimate(x, eb, mode=mode, stride=stride, debug=True)
    g, gd = run_gpu(sel, x, eb, mode, stride, debug=True, offset_elems=offset_elems)
    compare_scalars(g, o, tag)
    od = o["debug"]
    for k in ("codes", "hist", "emax", "coef", "uword", "bits"):
        assert np.array_equal(gd[k].reshape(od[k].shape), od[k]), (tag, k)
    assert np.allclose(gd["err"], od["err"], rtol=1e-12, atol=0), tag
    # the non-debug instantiation (the one bench.py times) agrees with the oracle
    # and is deterministic run to run (fixed tile -> partial mapping)
    g2, _ = run_gpu(sel, x, eb, mode, stride, debug=False, offset_elems=offset_elems)
    g3, _ = run_gpu(sel, x, eb, mode, stride, debug=False, offset_elems=offset_elems)
    compare_scalars(g2, o, tag + "/nodebug")
    for k in g2:
        assert g2[k] == g3[k] or (isinstance(g2[k], float) and math.isnan(g2[k])), (tag, k)
    # host-side Alg. 1 recomputation agrees with the device's choice
    assert sel.choose(g) == g["choice"]
    return g, o


# ---------------------------------------------------------------- configs (small)
def test_config1_exact(sel, orc):
    import synth
    x = synth.c1_field()
    check_case(sel, orc, x, 1e-4, tag="C1")


@pytest.mark.parametrize("i", [0, 1, 3])
@pytest.mark.parametrize("stride", [None, (1, 10), (3, 2)])
def test_config2_recipe_ragged(sel, orc, i, stride):
    import synth
    x = synth.c2_field(i, shape=(203, 517))          # ragged: neither dim % 4 == 0
    check_case(sel, orc, x, 1e-4, stride=stride, tag=f"C2r{i}{stride}")


@pytest.mark.parametrize("i", [0, 2, 3, 5, 9])
@pytest.mark.parametrize("eb", [1e-3, 1e-4, 1e-5])
def test_config3_recipe_ragged(sel, orc, i, eb):
    import synth
    x = synth.c3_field(i, shape=(37, 45, 70))
    check_case(sel, orc, x, eb, tag=f"C3r{i}/{eb}")


@pytest.mark.parametrize("i", [0, 1, 4])
@pytest.mark.parametrize("stride", [None, (4, 4, 4), (1, 2, 3)])
def test_config4_recipe(sel, orc, i, stride):
    import synth
    x = synth.c4_field(i, shape=(64, 64, 64))
    check_case(sel, orc, x, 1e-4, stride=stride, tag=f"C4s{i}{stride}")


@pytest.mark.parametrize("mix", [0, 1, 2])
@pytest.mark.parametrize("eb", [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7])
def test_config5_recipe(sel, orc, mix, eb):
    import synth
    x = synth.c5_field(mix, shape=(32, 48, 64))
    g, o = check_case(sel, orc, x, eb, tag=f"C5s{mix}/{eb}")
    if mix == 2 and eb <= 1e-6:
        assert o["sz_overflow_frac"] > 0.5          # the histogram-width stress really is hit


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("shape", [(100003,), (5,), (2, 3), (1, 1, 5), (3, 1, 9), (1, 700), (9, 10, 1)])
def test_odd_shapes(sel, orc, shape):
    rng = np.random.default_rng(len(shape) * 100 + shape[-1])
    x = np.cumsum(rng.standard_normal(int(np.prod(shape)))).reshape(shape).astype(np.float32)
    check_case(sel, orc, x, 1e-3, tag=f"odd{shape}")
    check_case(sel, orc, x, 0.01, mode="abs", tag=f"odd{shape}abs")


def test_misaligned_pointer_scalar_path(sel, orc):
    import synth
    x = synth.c2_field(4, shape=(64, 96))
    check_case(sel, orc, x, 1e-4, offset_elems=1, tag="misaligned")


def test_constant_and_zero_fields(sel, orc):
    for x in (np.full((17, 23), 2.5, np.float32), np.zeros((8, 8, 8), np.float32),
              np.full((40,), -1e-41, np.float32)):
        g, o = check_case(sel, orc, x, 1e-3, mode="abs", tag=f"const{x.shape}")
        assert g["sz_entropy"] == 0.0
    with pytest.raises(sel.SelError) as e:
        run_gpu(sel, np.full((8, 8), 1.0, np.float32), 1e-3, "rel")
    assert e.value.status == sel.SEL_EDEGENERATE


def test_nonfinite_rejected(sel):
    for bad in (np.nan, np.inf, -np.inf):
        x = np.ones((13, 9), np.float32)
        x[7, 3] = bad
        with pytest.raises(sel.SelError) as e:
            run_gpu(sel, x, 1e-3)
        assert e.value.status == sel.SEL_ENONFINITE


def test_single_value_degenerate(sel):
    with pytest.raises(sel.SelError) as e:
        run_gpu(sel, np.ones((1,), np.float32), 1e-3, "abs")
    assert e.value.status == sel.SEL_EDEGENERATE


def test_extreme_values(sel, orc):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((24, 28, 32)).astype(np.float32)
    x[:4, :4, :4] *= np.float32(1e-39)                   # subnormal block (emax clamp)
    x[4:8, :4, :4] = np.float32(3.0e38) * np.sign(x[4:8, :4, :4])   # near FLT_MAX
    x[8:12, 4:8, :] = 0.0                                 # empty blocks
    x[12:, :, :] *= (rng.random((12, 28, 32)) < 0.7)      # 30% zeros
    check_case(sel, orc, x, 1e-3, mode="abs", tag="extreme-abs")
    check_case(sel, orc, x, 1e-6, mode="rel", tag="extreme-rel")
    y = (rng.standard_normal((16, 16)) * 1e-30).astype(np.float32)   # BFP two-step scale path
    check_case(sel, orc, y, 1e-3, tag="tiny")


def test_offset_option(sel, orc):
    import synth
    x = synth.c1_field((64, 64), seed=4)
    o = orc.estimate(x, 1e-4, sz_offset=0.0)
    t = torch.from_numpy(x).cuda()
    with sel.Plan(x.shape, 1e-4) as p:
        p.set_option("sz_offset_bits", 0.0)
        g = p.estimate(t)
    compare_scalars(g, o, "offset0")


# ---------------------------------------------------------------- batch APIs
def test_batch_and_host_batch(sel, orc):
    import synth
    shape = (60, 88)
    xs = [synth.c2_field(i, shape=shape) for i in range(5)]
    ts = [torch.from_numpy(x).cuda() for x in xs]
    hs = [torch.from_numpy(x).pin_memory() for x in xs]
    with sel.Plan(shape, 1e-4) as p:
        single = [p.estimate(t) for t in ts]
        batch = p.estimate_batch(ts)                 # persistent k_batch (1 launch)
        l0 = p.launch_count
        p.estimate_batch(ts)
        assert p.launch_count - l0 == 1
        p.set_option("batch_kernel", 0)
        piped = p.estimate_batch(ts)                 # 3-stream pipeline of per-field kernels
        p.set_option("pipeline", 0)
        seq = p.estimate_batch(ts)                   # plain sequential per-field kernels
        host = p.estimate_batch_host(hs)
        host_np = p.estimate_batch_host(xs)
    for i, x in enumerate(xs):
        o = orc.estimate(x, 1e-4)
        for r in (single[i], batch[i], piped[i], seq[i], host[i], host_np[i]):
            compare_scalars(r, o, f"batch{i}")
        for r in (piped[i], host[i]):
            for k in seq[i]:
                if isinstance(seq[i][k], float):
                    assert close(r[k], seq[i][k], rel=1e-12), (i, k)
                else:
                    assert r[k] == seq[i][k], (i, k)


@pytest.mark.parametrize("batch_kernel", [1, 0])
def test_batch_reports_per_field_status(sel, batch_kernel):
    bad = torch.ones(8, 8, device="cuda")
    nan = torch.arange(64, dtype=torch.float32, device="cuda").view(8, 8).clone()
    nan[3, 3] = float("nan")
    good = torch.arange(64, dtype=torch.float32, device="cuda").view(8, 8)
    with sel.Plan((8, 8), 1e-3) as p:
        p.set_option("batch_kernel", batch_kernel)
        out = p.estimate_batch([bad, good, nan, good])
    assert out[0]["status"] == sel.SEL_EDEGENERATE and out[1]["status"] == 0
    assert out[2]["status"] == sel.SEL_ENONFINITE and out[3]["status"] == 0
    assert out[1]["choice"] == out[3]["choice"]


@pytest.mark.parametrize("nf", [1, 2, 3, 4, 5, 7])
@pytest.mark.parametrize("shape", [(8, 12), (4, 4, 8), (3, 5, 4), (1, 4)])
def test_batch_kernel_tiny_stacks(sel, orc, nf, shape):
    """Stacks of tiny fields: most CTAs get no task, phases are empty or shorter than
    the stage ring -- the task dataflow must neither deadlock nor mix fields."""
    rng = np.random.default_rng(nf * 100 + sum(shape))
    xs = [(rng.standard_normal(shape) * (i + 1)).astype(np.float32) for i in range(nf)]
    xs[0] = np.cumsum(xs[0].ravel()).reshape(shape).astype(np.float32)
    ts = [torch.from_numpy(x).cuda() for x in xs]
    with sel.Plan(shape, 1e-3) as p:
        out = p.estimate_batch(ts)
    for i, x in enumerate(xs):
        compare_scalars(out[i], orc.estimate(x, 1e-3), f"tiny{nf}/{i}")


@pytest.mark.parametrize("cfg,nf,stride", [(2, 12, None), (3, 3, None), (4, 2, None),
                                            (2, 12, (1, 10)), (4, 2, (4, 4, 4)), (3, 2, (1, 2, 3))])
def test_batch_full_size_stack_vs_per_field(sel, cfg, nf, stride):
    """A stack of full-size fields through k_batch (auto CTA groups, several flushes per
    CTA, second-level table in use on C2; tiles, or sampled-block tasks for strides > 1)
    equals the per-field kernels field by field,
    and repeats bit-identically.  The per-field kernels are checked against the oracle
    by the tests above."""
    import synth
    fs = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
    eb = synth.CONFIGS[cfg]["eb_rel"][0]
    with sel.Plan(tuple(fs[0].shape), eb, "rel", stride) as p:
        p.set_option("batch_kernel", 0)
        ref = [p.estimate(f) for f in fs]
        p.set_option("batch_kernel", 1)
        out1 = p.estimate_batch(fs)
        out2 = p.estimate_batch(fs)
    assert out1 == out2
    for i, (a, b) in enumerate(zip(out1, ref)):
        for k in a:
            if isinstance(a[k], float):
                assert a[k] == pytest.approx(b[k], rel=1e-12, abs=0), (cfg, i, k)
            else:
                assert a[k] == b[k], (cfg, i, k)


@pytest.mark.parametrize("shape,stride", [((40, 300), (1, 10)), ((40, 300), (3, 2)),
                                          ((20, 24, 36), (2, 1, 3)), ((9, 14, 20), (1, 1, 2))])
def test_batch_sampled_vs_oracle(sel, orc, shape, stride):
    """Sampled-block tasks of k_batch (strides > 1) give the oracle's results."""
    rng = np.random.default_rng(sum(shape))
    xs = [np.cumsum(rng.standard_normal(shape), axis=-1).astype(np.float32) * (i + 1)
          for i in range(5)]
    ts = [torch.from_numpy(x).cuda() for x in xs]
    with sel.Plan(shape, 1e-3, "rel", stride) as p:
        l0 = p.launch_count
        out = p.estimate_batch(ts)
        assert p.launch_count - l0 == 1            # one k_batch launch
    for i, x in enumerate(xs):
        compare_scalars(out[i], orc.estimate(x, 1e-3, stride=stride), f"sampled/{i}")


@pytest.mark.parametrize("groups", [1, 2, 3, 5])
def test_batch_groups(sel, orc, groups):
    """CTA groups (each group runs every G-th field) give the oracle's results."""
    shape = (40, 300)
    rng = np.random.default_rng(groups)
    xs = [np.cumsum(rng.standard_normal(shape), axis=1).astype(np.float32) for _ in range(7)]
    ts = [torch.from_numpy(x).cuda() for x in xs]
    with sel.Plan(shape, 1e-3) as p:
        p.set_option("groups", groups)
        out = p.estimate_batch(ts)
    for i, x in enumerate(xs):
        compare_scalars(out[i], orc.estimate(x, 1e-3), f"G{groups}/{i}")


@pytest.mark.parametrize("lag", [1, 2, 4])
def test_batch_lag_and_task_table_cache(sel, orc, lag):
    """Range lead (lag) variants, and one plan reused for stacks of different sizes and
    group counts: the host-built task table (cached per key) is rebuilt whenever the
    sequence changes; every result equals the oracle's."""
    shape = (36, 260)
    rng = np.random.default_rng(100 + lag)
    xs = [np.cumsum(rng.standard_normal(shape), axis=0).astype(np.float32) for _ in range(7)]
    ts = [torch.from_numpy(x).cuda() for x in xs]
    ref = [orc.estimate(x, 1e-3) for x in xs]
    with sel.Plan(shape, 1e-3) as p:
        p.set_option("lag", lag)
        for n, g in ((7, 0), (3, 1), (7, 2), (5, 0), (7, 0)):
            p.set_option("groups", g)
            out = p.estimate_batch(ts[:n])
            for i in range(n):
                compare_scalars(out[i], ref[i], f"lag{lag}/n{n}/G{g}/{i}")


@pytest.mark.parametrize("where", ["pinned", "cuda"])
@pytest.mark.parametrize("batch_kernel", [1, 0])
def test_estimate_batch_async(sel, orc, where, batch_kernel):
    """Stream-ordered entry: several calls enqueued back to back on one stream, each
    into its own results buffer, read after one synchronise -- equal to the oracle."""
    shape = (72, 100)
    rng = np.random.default_rng(7)
    stacks = [[np.cumsum(rng.standard_normal(shape), axis=k % 2).astype(np.float32) * (k + 1)
               for k in range(3)] for _ in range(3)]
    dev = [[torch.from_numpy(x).cuda() for x in st] for st in stacks]
    with sel.Plan(shape, 1e-3) as p:
        p.set_option("batch_kernel", batch_kernel)
        bufs = [p.results_buffer(3, "pinned" if where == "pinned" else "cuda") for _ in stacks]
        for d, b in zip(dev, bufs):
            p.estimate_batch_async(d, b)
        torch.cuda.synchronize()
        for st, b in zip(stacks, bufs):
            out = p.decode_results(b, 3)
            for i, x in enumerate(st):
                compare_scalars(out[i], orc.estimate(x, 1e-3), f"async/{i}")
        p.set_option("kernel_timing", 1)
        with pytest.raises(sel.SelError):
            p.estimate_batch_async(dev[0], bufs[0])


@pytest.mark.parametrize("shape", [(96, 128), (20, 24, 36), (1, 1, 8)])
def test_batch_kernel_many_fields(sel, orc, shape):
    """k_batch over a longer stack (parity buffers reused, phases overlap) == oracle."""
    rng = np.random.default_rng(sum(shape))
    xs = [np.cumsum(rng.standard_normal(shape), axis=-1).astype(np.float32) * (i + 1) for i in range(9)]
    ts = [torch.from_numpy(x).cuda() for x in xs]
    with sel.Plan(shape, 1e-4) as p:
        out = p.estimate_batch(ts)
        again = p.estimate_batch(ts)
    for i, x in enumerate(xs):
        compare_scalars(out[i], orc.estimate(x, 1e-4), f"mf{i}")
        assert out[i] == again[i]


def test_kernel_timing_option(sel):
    t = torch.randn(256, 256, device="cuda")
    with sel.Plan(t.shape, 1e-4) as p:
        p.set_option("kernel_timing", 1)
        for _ in range(3):
            p.estimate(t)
        ms, n = p.kernel_times(reset=True)
        assert n[1] == 3 and ms[1] > 0              # k_batch counted as the fused pass
        p.set_option("batch_kernel", 0)
        for _ in range(3):
            p.estimate(t)
        ms, n = p.kernel_times(reset=True)
    assert n == [3, 3, 3] and all(m > 0 for m in ms)


# ---------------------------------------------------------------- k_batch element-exact
def _part_sums(vals, lay, grid_shape, stride_all_one):
    """Sum per-block values (processed-block row-major order) over k_batch's parts."""
    ppt, rpp, rpt = lay["parts_per_task"], lay["rows_per_part"], lay["rows_per_tile"]
    nT = lay["n_tasks"]
    if lay["sampled"]:
        v = np.zeros(nT * ppt * 32, vals.dtype)
        v[: vals.size] = vals
        return v.reshape(nT * ppt, 32).sum(axis=1)
    nb0, nb1, nb2 = grid_shape
    ntj, ntk = lay["ntj"], lay["ntk"]
    g = np.zeros((nb0, ntj * rpt, ntk * 32), vals.dtype)
    g[:, :nb1, :nb2] = vals.reshape(nb0, nb1, nb2)
    g = g.reshape(nb0, ntj, ppt, rpp, ntk, 32).sum(axis=(3, 5))      # (bi, btj, p, btk)
    return g.transpose(0, 1, 3, 2).reshape(-1)                      # task (bi, btj, btk), part p


def check_batch_exact(sel, orc, xs, eb, stride=None, tag="", threads=0):
    """The benched kernel (k_batch, one launch for the stack, bench launch configuration)
    against the oracle ELEMENT BY ELEMENT: every field's 65,536-bin histogram bin-exact,
    the device-counted histogram total / overflow exact, every per-(task, part) ZFP
    partial's bit count exact and error to 1e-12, and the scalars (1e-6 / exact)."""
    shape = xs[0].shape
    ts = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in xs]
    with sel.Plan(shape, eb, "rel", stride) as p:
        plain = p.estimate_batch(ts)                     # no dumps: what bench.py times
        l0 = p.launch_count
        p.set_option("batch_debug", 1)
        out = p.estimate_batch(ts)
        assert p.launch_count - l0 == 1, "k_batch did not run"
        hist = p.batch_debug_copy("hist", len(xs))
        part = p.batch_debug_copy("part", len(xs))
        lay = p.batch_layout()
    assert out == plain, tag                              # the dumps change nothing
    nd = len(shape)
    grid = [1] * (3 - nd) + [(n + 3) // 4 for n in shape]
    ties = 0
    res = []
    for i, x in enumerate(xs):
        o = orc.estimate(x, eb, mode="rel", stride=stride, debug=("hist", "bits", "err"),
                         threads=threads)
        t = f"{tag}/{i}"
        compare_scalars(out[i], o, t)
        od = o["debug"]
        assert np.array_equal(hist[i].astype(np.uint64), od["hist"]), (t, "histogram")
        pb = _part_sums(od["bits"].astype(np.uint64), lay, grid, stride is None)
        assert np.array_equal(part[i]["bits"], pb), (t, "part bits")
        pe = _part_sums(od["err"], lay, grid, stride is None)
        assert np.allclose(part[i]["err"], pe, rtol=1e-12, atol=0), (t, "part err")
        ties += tie_margin(out[i]) < NEAR_TIE
        res.append((out[i], o))
    assert ties == 0, (tag, "near ties", ties)
    return res


@pytest.mark.parametrize("shape,stride", [((64, 256), None), ((203, 516), None), ((40, 300), (1, 10)),
                                          ((16, 40, 132), None), ((37, 45, 68), None),
                                          ((20, 24, 36), (2, 1, 3))])
def test_batch_exact_small(sel, orc, shape, stride):
    """k_batch element-exact on small ragged stacks (several tiles, partial tiles)."""
    import synth
    if len(shape) == 2:
        xs = [synth.c2_field(i, shape=shape) for i in range(4)]
    else:
        xs = [synth.c3_field(i, shape=shape) for i in (0, 5, 9)]
    check_batch_exact(sel, orc, xs, 1e-4, stride, tag=f"bx{shape}{stride}")


@pytest.mark.parametrize("shape", [(64, 64), (16, 16, 64)])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_batch_kernel_nonfinite(sel, shape, bad):
    """NaN / +Inf / -Inf through k_batch (aligned, tile path): SEL_ENONFINITE for that field
    only, single-field and in a stack."""
    rng = np.random.default_rng(1)
    good = rng.standard_normal(shape).astype(np.float32)
    x = good.copy()
    x.flat[x.size // 3] = bad
    tg, tx = torch.from_numpy(good).cuda(), torch.from_numpy(x).cuda()
    with sel.Plan(shape, 1e-3) as p:
        l0 = p.launch_count
        with pytest.raises(sel.SelError) as e:
            p.estimate(tx)
        assert e.value.status == sel.SEL_ENONFINITE
        assert p.launch_count - l0 == 1                   # it was k_batch
        out = p.estimate_batch([tg, tx, tg])
    assert out[1]["status"] == sel.SEL_ENONFINITE and out[0]["status"] == 0 and out[2]["status"] == 0


# ---------------------------------------------------------------- full sizes
def _padded_block(x, b, nd):
    sl = []
    for a in range(nd):
        idx = np.minimum(np.arange(4 * b[a], 4 * b[a] + 4), x.shape[a] - 1)
        sl.append(idx)
    return x[np.ix_(*sl)].reshape(-1)


def _sampled_block_check(orc, x, g, dbg, stride, nblocks=400, seed=0):
    """Per-block parity on sampled processed blocks, computed one by one with
    the oracle's step functions (full-size fields, BASELINE 'sampled outputs')."""
    nd = x.ndim
    nb = [(n + 3) // 4 for n in x.shape]
    npb = [(nb[a] + stride[a] - 1) // stride[a] for a in range(nd)]
    rng = np.random.default_rng(seed)
    perm = orc.sequency_perm(nd)
    r_f = np.float32(g["r_f"])
    for _ in range(nblocks):
        t = int(rng.integers(0, int(np.prod(npb))))
        pc = np.unravel_index(t, npb)
        b = [int(pc[a]) * stride[a] for a in range(nd)]
        blk = _padded_block(x, b, nd)
        e = orc.block_emax(blk)
        assert dbg["emax"][t] == e
        if e == -127:
            assert dbg["bits"][t] == 1
            continue
        coef = orc.fwd_xform(orc.block_bfp(blk, e), nd)
        assert np.array_equal(dbg["coef"][t], coef)
        u = np.array([orc.negabinary(int(coef[p])) for p in perm], np.uint32)
        assert np.array_equal(dbg["uword"][t], u)
        p = orc.precision(e, g["minexp"], nd)
        bits = 1 if p == 0 else 9 + orc.gt_count(u, 32 - p)
        assert dbg["bits"][t] == bits
        assert close(float(dbg["err"][t]), orc.block_err(coef, u, nd, 32 - p, e), rel=1e-12, abs_=0.0)
        # SZ codes of the block's real points
        for n in range(4 ** nd):
            idx = tuple(4 * b[a] + (n // 4 ** (nd - 1 - a)) % 4 for a in range(nd))
            if any(idx[a] >= x.shape[a] for a in range(nd)):
                continue
            if not any(idx):
                assert dbg["codes"][idx] == -1
                continue
            assert dbg["codes"][idx] == orc.quantize(orc.lorenzo(x, idx), r_f), idx


def _per_field_debug_check(sel, orc, x, eb, stride=None, tag=""):
    """Intermediates (codes, emax, coefficients, words, bits, errors) of the per-field
    debug kernels on sampled blocks of a full-size field."""
    st = stride or (1,) * x.ndim
    t = torch.from_numpy(x).cuda()
    with sel.Plan(x.shape, eb, "rel", stride) as p:
        g = p.estimate(t)
        p.set_option("debug", 1)
        gd = p.estimate(t)
        dbg = {k: p.debug_copy(k) for k in ("codes", "hist", "emax", "coef", "uword", "bits", "err")}
    for k in g:
        if isinstance(g[k], float):
            assert close(g[k], gd[k], rel=1e-12), (tag, k)
        else:
            assert g[k] == gd[k], (tag, k)
    assert int(dbg["hist"].sum()) == g["n_sz_points"]
    assert int(dbg["bits"].astype(np.uint64).sum()) == g["zfp_total_bits"]
    _sampled_block_check(orc, x, g, dbg, st)


def test_full_config2_fields(sel, orc):
    """C2 at full size: 20 fields (both kinds: 0 and 10 are piecewise-constant), every
    block and every 10th block column, element-exact through k_batch."""
    import synth
    xs = [synth.c2_field(i) for i in range(20)]
    check_batch_exact(sel, orc, xs, 1e-4, tag="C2full")
    check_batch_exact(sel, orc, xs, 1e-4, stride=(1, 10), tag="C2s")
    _per_field_debug_check(sel, orc, xs[0], 1e-4, tag="C2dbg")


@pytest.mark.parametrize("eb", [1e-3, 1e-4, 1e-5])
def test_full_config3_fields(sel, orc, eb):
    """C3 at full size: all 13 fields at every eb, element-exact through k_batch."""
    import synth
    xs = [synth.c3_field(i) for i in range(13)]
    check_batch_exact(sel, orc, xs, eb, tag=f"C3full/{eb}")
    if eb == 1e-5:
        _per_field_debug_check(sel, orc, xs[5], eb, tag="C3dbg")


def test_full_config4_fields(sel, orc):
    """C4 at full size: all 6 fields, every block and 1/64 of the blocks."""
    import synth
    xs = [synth.c4_field(i) for i in range(6)]
    check_batch_exact(sel, orc, xs, 1e-4, tag="C4full")
    check_batch_exact(sel, orc, xs, 1e-4, stride=(4, 4, 4), tag="C4s")


@pytest.mark.parametrize("mix", [0, 1, 2])
def test_full_config5_fields(sel, orc, mix):
    """C5 at full size (1024^3, 4 GiB): every eb of the sweep, element-exact through
    k_batch against the (threaded, bit-identical) oracle."""
    import synth
    x = synth.c5_field(mix)
    for eb in synth.CONFIGS[5]["eb_rel"]:
        (g, o), = check_batch_exact(sel, orc, [x], eb, tag=f"C5full{mix}/{eb}")
        if mix == 2 and eb <= 1e-6:
            assert g["sz_overflow_frac"] > 0.5


# ---------------------------------------------------------------- N1: multi-eb in one read
@pytest.mark.parametrize("case", ["c3", "c5", "c2", "c2s", "c4s", "odd1d", "odd3d", "abs", "t3edge", "t2edge",
                                  "t3k8", "t3one"])
def test_multi_eb_vs_oracle(sel, orc, case):
    """sel_estimate_multi (one read, k ebs) equals the oracle's single-eb estimate at every
    eb: exact integer keys (histogram total / overflow, ZFP bits, minexp, choices), the
    rest within 1e-6."""
    import synth
    mode, stride = "rel", None
    if case == "c3":
        x, ebs = synth.c3_field(5, shape=(37, 45, 70)), [1e-3, 1e-4, 1e-5]
    elif case == "c5":
        x, ebs = synth.c5_field(2, shape=(32, 48, 64)), [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7]
    elif case == "c2":
        x, ebs = synth.c2_field(3, shape=(203, 517)), [1e-2, 1e-4, 1e-6]
    elif case == "c2s":
        x, ebs, stride = synth.c2_field(0, shape=(120, 400)), [1e-3, 1e-4], (1, 10)
    elif case == "c4s":
        x, ebs, stride = synth.c4_field(0, shape=(64, 64, 64)), [1e-2, 1e-3, 1e-4, 1e-5], (4, 4, 4)
    elif case == "odd1d":
        rng = np.random.default_rng(11)
        x, ebs = np.cumsum(rng.standard_normal(100003)).astype(np.float32), [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-3, 3e-4]
    elif case == "odd3d":
        rng = np.random.default_rng(12)
        x, ebs = np.cumsum(rng.standard_normal((9, 14, 21)), axis=2).astype(np.float32), [1e-2, 1e-5]
    elif case == "t3edge":       # tile pipeline (fastest extent % 4 == 0), ragged far edges, several tiles
        x, ebs = synth.c3_field(5, shape=(37, 45, 136)), [1e-3, 1e-4, 1e-5]
    elif case == "t2edge":
        x, ebs = synth.c2_field(3, shape=(203, 516)), [1e-2, 1e-4, 1e-6]
    elif case == "t3k8":         # 8 ebs: the smallest windows, equal ebs, an unsorted list
        x, ebs = synth.c5_field(1, shape=(24, 40, 260)), [1e-4, 1e-2, 1e-3, 1e-3, 1e-6, 1e-5, 3e-4, 1e-7]
    elif case == "t3one":
        x, ebs = synth.c4_field(0, shape=(32, 32, 128)), [1e-4]
    else:
        x, ebs, mode = synth.c1_field(), [0.5, 0.01, 1e-4], "abs"
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    with sel.Plan(x.shape, ebs[0], mode, stride) as p:
        l0 = p.launch_count
        out = p.estimate_multi(t, ebs)
        assert p.launch_count - l0 == 2 + len(ebs)        # K1, one fused pass, k finalizes
        again = p.estimate_multi(t, ebs)
        p.set_option("multi_tile", 0)                      # the one-thread-per-block pass
        plain = p.estimate_multi(t, ebs)
    assert out == again                                    # deterministic, state re-zeroed
    for e, r, q in zip(ebs, out, plain):
        o = orc.estimate(x, e, mode=mode, stride=stride)
        compare_scalars(r, o, f"multi/{case}/{e}")
        compare_scalars(q, o, f"multi-plain/{case}/{e}")
        assert sel.choose(r) == r["choice"]


def test_multi_eb_errors(sel):
    t = torch.ones(8, 8, device="cuda")
    with sel.Plan((8, 8), 1e-3) as p:
        with pytest.raises(sel.SelError):
            p.estimate_multi(t, [])
        with pytest.raises(sel.SelError):
            p.estimate_multi(t, [1e-3] * 9)
        with pytest.raises(sel.SelError):
            p.estimate_multi(t, [1e-3, -1.0])
        out = p.estimate_multi(t, [1e-3, 1e-4])            # constant field, relative bound
    assert all(r["status"] == sel.SEL_EDEGENERATE for r in out)
    bad = torch.arange(64, dtype=torch.float32, device="cuda").view(8, 8).clone()
    bad[2, 2] = float("inf")
    with sel.Plan((8, 8), 1e-3) as p:
        out = p.estimate_multi(bad, [1e-3, 1e-4])
    assert all(r["status"] == sel.SEL_ENONFINITE for r in out)


@pytest.mark.parametrize("cfg", [3, 5])
def test_multi_eb_full_size(sel, orc, cfg):
    """Full-size N1 runs: C3 field 5 at its 3 ebs, C5 (mix 1) at its 6 ebs, from one read
    each, against the (threaded) oracle."""
    import synth
    x = synth.make_field(cfg, 5 if cfg == 3 else 1)
    ebs = synth.CONFIGS[cfg]["eb_rel"]
    t = torch.from_numpy(x).cuda()
    with sel.Plan(x.shape, ebs[0], "rel") as p:
        out = p.estimate_multi(t, ebs)
    for e, r in zip(ebs, out):
        o = orc.estimate(x, e, mode="rel", threads=0)
        compare_scalars(r, o, f"multi-full/C{cfg}/{e}")


# ---------------------------------------------------------------- N2: paper-literal estimator
PAPER_EXACT = ("nsb2_total", "n_samples", "n_values", "hist_total", "hist_ovf", "r_star", "choice",
               "matched", "status")
PAPER_CLOSE = ("zfp_nsb_bits", "zfp_mse_sp", "zfp_psnr_sp", "sz_delta", "sz_bits", "sz_entropy",
               "sz_overflow_frac", "value_range", "eb_abs")


def compare_paper(g, o, tag=""):
    for k in PAPER_EXACT:
        assert g[k] == o[k], (tag, k, g[k], o[k])
    for k in PAPER_CLOSE:
        assert close(float(g[k]), float(o[k])), (tag, k, g[k], o[k])


@pytest.mark.parametrize("case", ["c1", "c2r", "c2s", "c3r", "c4s", "c5", "odd1d", "odd2d", "unmatched"])
def test_paper_estimator_vs_oracle(sel, orc, case):
    """sel_estimate_paper (Alg. 1 lines 3-10 as printed) equals the oracle:
    the interpolated n_sb total, sample count, histogram at delta and the choice exactly,
    the rest within 1e-6."""
    import synth
    mode, stride, eb = "rel", None, 1e-4
    if case == "c1":
        x = synth.c1_field()
    elif case == "c2r":
        x = synth.c2_field(0, shape=(203, 516))
    elif case == "c2s":
        x, stride = synth.c2_field(3, shape=(120, 400)), (1, 10)
    elif case == "c3r":
        x, eb = synth.c3_field(5, shape=(37, 45, 70)), 1e-5
    elif case == "c4s":
        x, stride = synth.c4_field(0, shape=(64, 64, 64)), (4, 4, 4)
    elif case == "c5":
        x, eb = synth.c5_field(1, shape=(32, 48, 64)), 1e-6
    elif case == "odd1d":
        x = np.cumsum(np.random.default_rng(3).standard_normal(10007)).astype(np.float32)
    elif case == "odd2d":
        x = np.cumsum(np.random.default_rng(4).standard_normal((13, 27)), axis=1).astype(np.float32)
    else:
        rng = np.random.default_rng(5)
        x, eb, mode = (1.0 + 0.25 * rng.standard_normal((24, 40))).astype(np.float32), 2.0 ** -40, "abs"
    o = orc.estimate_paper(x, eb, mode=mode, stride=stride)
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    with sel.Plan(x.shape, eb, mode, stride) as p:
        l0 = p.launch_count
        g = p.estimate_paper(t)
        assert p.launch_count - l0 == 6
        g2 = p.estimate_paper(t)
        e = p.estimate(t)                            # the exact estimate still works after it
    assert g == g2
    compare_paper(g, o, case)
    compare_scalars(e, orc.estimate(x, eb, mode=mode, stride=stride), case + "/exact-after")
    if case == "unmatched":
        assert g["matched"] == 0 and g["sz_bits"] == e["sz_bits_per_value"]


def test_paper_estimator_full_size(sel, orc):
    """C4 field 0 (512^3) at 1/64 block sampling and a full C2 field, against the oracle."""
    import synth
    for x, stride in ((synth.c4_field(0), (4, 4, 4)), (synth.c2_field(10), None)):
        o = orc.estimate_paper(x, 1e-4, stride=stride)
        with sel.Plan(x.shape, 1e-4, "rel", stride) as p:
            g = p.estimate_paper(torch.from_numpy(x).cuda())
        compare_paper(g, o, f"full{x.shape}")


def test_paper_estimator_errors(sel):
    with sel.Plan((8, 8), 1e-3) as p:
        with pytest.raises(sel.SelError) as e:
            p.estimate_paper(torch.ones(8, 8, device="cuda"))
        assert e.value.status == sel.SEL_EDEGENERATE
        bad = torch.arange(64, dtype=torch.float32, device="cuda").view(8, 8).clone()
        bad[1, 1] = float("nan")
        with pytest.raises(sel.SelError) as e:
            p.estimate_paper(bad)
        assert e.value.status == sel.SEL_ENONFINITE


# ---------------------------------------------------------------- N3: the ZFP stream
@pytest.mark.parametrize("case", ["c1", "c2r", "c2s", "c3r", "c3z", "c4", "c5", "odd1d", "odd3d", "zeros"])
def test_zfp_stream_vs_oracle(sel, orc, case):
    """sel_compress_zfp (Alg. 1 line 13) writes the oracle's stream BIT FOR BIT, its length
    is the estimate's zfp_total_bits, and the oracle decodes it within the error bound."""
    import synth
    mode, stride, eb = "rel", None, 1e-4
    if case == "c1":
        x = synth.c1_field()
    elif case == "c2r":
        x = synth.c2_field(0, shape=(203, 516))
    elif case == "c2s":
        x, stride = synth.c2_field(3, shape=(120, 400)), (1, 10)
    elif case == "c3r":
        x, eb = synth.c3_field(2, shape=(37, 45, 70)), 1e-3
    elif case == "c3z":
        x, eb = synth.c3_field(5, shape=(37, 45, 70)), 1e-5
    elif case == "c4":
        x = synth.c4_field(0, shape=(64, 64, 64))
    elif case == "c5":
        x, eb = synth.c5_field(2, shape=(32, 48, 64)), 1e-6
    elif case == "odd1d":
        x = np.cumsum(np.random.default_rng(3).standard_normal(10007)).astype(np.float32)
    elif case == "odd3d":
        x = np.cumsum(np.random.default_rng(4).standard_normal((9, 14, 21)), axis=2).astype(np.float32)
    else:
        x, eb, mode = np.zeros((16, 20), np.float32), 1e-3, "abs"
    ref, nref = orc.zfp_stream(x, eb, mode=mode, stride=stride)
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    with sel.Plan(x.shape, eb, mode, stride) as p:
        buf, nbits = p.compress_zfp(t)
        if case != "zeros":
            r = p.estimate(t)
            assert nbits == r["zfp_total_bits"]
    assert nbits == nref
    got = buf.cpu().numpy()
    nb = (nbits + 7) // 8
    assert np.array_equal(got[:nb], ref[:nb]), case
    if stride is None and case != "zeros":
        o = orc.estimate(x, eb, mode=mode)
        y = orc.zfp_stream_decode(got, nbits, x.shape, eb, o["value_range"], mode=mode)
        assert np.abs(y.astype(np.float64) - x).max() <= o["eb_abs"]


def test_zfp_stream_full_size(sel, orc):
    """C4 field 2 (512^3, 2.1 M blocks): the stream equals the oracle's bit for bit."""
    import synth
    x = synth.c4_field(2)
    ref, nref = orc.zfp_stream(x, 1e-4)
    with sel.Plan(x.shape, 1e-4) as p:
        buf, nbits = p.compress_zfp(torch.from_numpy(x).cuda())
    assert nbits == nref
    assert np.array_equal(buf.cpu().numpy()[: (nbits + 7) // 8], ref[: (nbits + 7) // 8])


def test_zfp_stream_errors(sel):
    with sel.Plan((8, 8), 1e-3) as p:
        with pytest.raises(sel.SelError) as e:
            p.compress_zfp(torch.ones(8, 8, device="cuda"))
        assert e.value.status == sel.SEL_EDEGENERATE


# ---------------------------------------------------------------- small single fields
@pytest.mark.parametrize("shape,stride", [((256, 256), None), ((203, 517), None), ((100003,), None),
                                          ((37, 45, 70), None), ((64, 64, 64), (4, 4, 4)), ((120, 400), (1, 10)),
                                          ((5,), None), ((1, 1, 8), None), ((1024, 1024), None)])
def test_small_kernel_vs_oracle_and_batch(sel, orc, shape, stride):
    """One small field through sel_estimate runs the single cooperative launch k_small
    (value range -> blocks -> entropy / result); it equals the oracle and the k_batch /
    per-field path (1e-12), repeats bit-identically, and is one launch."""
    rng = np.random.default_rng(sum(shape))
    x = np.cumsum(rng.standard_normal(shape), axis=-1).astype(np.float32)
    t = torch.from_numpy(x).cuda()
    with sel.Plan(shape, 1e-4, "rel", stride) as p:
        l0 = p.launch_count
        a = p.estimate(t)
        assert p.launch_count - l0 == 1
        b = p.estimate(t)
        p.set_option("small_kernel", 0)
        c = p.estimate(t)
    assert a == b
    compare_scalars(a, orc.estimate(x, 1e-4, stride=stride), f"small{shape}")
    for k in a:
        if isinstance(a[k], float):
            assert close(a[k], c[k], rel=1e-12), (k, a[k], c[k])
        else:
            assert a[k] == c[k], k


def test_small_kernel_status(sel):
    with sel.Plan((16, 16), 1e-3) as p:
        with pytest.raises(sel.SelError) as e:
            p.estimate(torch.ones(16, 16, device="cuda"))
        assert e.value.status == sel.SEL_EDEGENERATE
        for bad in (float("nan"), float("inf"), -float("inf")):
            y = torch.arange(256, dtype=torch.float32, device="cuda").view(16, 16).clone()
            y[5, 7] = bad
            with pytest.raises(sel.SelError) as e:
                p.estimate(y)
            assert e.value.status == sel.SEL_ENONFINITE
        ok = p.estimate(torch.arange(256, dtype=torch.float32, device="cuda").view(16, 16))   # state was reset
        assert ok["status"] == 0


# ---------------------------------------------------------------- N4: variant quantisers
VAR_EXACT = ("n_in", "hist_ovf", "log_base", "log_bins", "eqp_n", "status")
VAR_CLOSE = ("lin_bits", "lin_psnr", "log_bits", "log_psnr", "log_mse", "eqp_bits", "eqp_psnr", "eqp_mse",
             "eqp_width_sum", "value_range", "eb_abs")


def compare_variants(g, o, tag=""):
    for k in VAR_EXACT:
        assert g[k] == o[k], (tag, k, g[k], o[k])
    for k in VAR_CLOSE:
        assert close(float(g[k]), float(o[k])), (tag, k, g[k], o[k])


@pytest.mark.parametrize("case", ["c1", "c2r", "c2s", "c3r", "c4s", "c5", "c5wide", "odd1d", "odd3d", "abs"])
def test_variants_vs_oracle(sel, orc, case):
    """sel_estimate_variants equals the oracle: the PDF's mass, the
    overflow count and the occupied log-scale bins exactly, bit-rates / MSEs / PSNRs of the
    linear, log-scale and equal-probability quantisers within 1e-6, for several bases and
    bin counts, on shapes that take the tile, marching and generic fused kernels."""
    import synth
    mode, stride, eb = "rel", None, 1e-4
    if case == "c1":
        x = synth.c1_field()
    elif case == "c2r":
        x = synth.c2_field(0, shape=(203, 516))
    elif case == "c2s":
        x, stride = synth.c2_field(3, shape=(120, 400)), (1, 10)
    elif case == "c3r":
        x, eb = synth.c3_field(5, shape=(37, 45, 70)), 1e-5
    elif case == "c4s":
        x, stride = synth.c4_field(0, shape=(64, 64, 64)), (4, 4, 4)
    elif case == "c5":
        x, eb = synth.c5_field(1, shape=(32, 48, 64)), 1e-3
    elif case == "c5wide":                        # codes out to the overflow slot
        x, eb = synth.c5_field(2, shape=(32, 48, 64)), 1e-6
    elif case == "odd1d":
        x = np.cumsum(np.random.default_rng(3).standard_normal(10007)).astype(np.float32)
    elif case == "odd3d":
        x = np.cumsum(np.random.default_rng(4).standard_normal((5, 13, 27)), axis=2).astype(np.float32)
    else:
        rng = np.random.default_rng(5)
        x, eb, mode = (1.0 + 0.25 * rng.standard_normal((24, 40))).astype(np.float32), 1e-3, "abs"
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    with sel.Plan(x.shape, eb, mode, stride) as p:
        for b, n in ((2, 128), (3, 1), (10, 7), (40000, 32768), (2, 1000)):
            o = orc.estimate_variants(x, eb, mode=mode, stride=stride, log_base=b, eqp_n=n)
            l0 = p.launch_count
            g = p.estimate_variants(t, b, n)
            assert p.launch_count - l0 == 4
            compare_variants(g, o, f"{case}/b{b}/n{n}")
        e = p.estimate(t)                            # the plan's other entries still work after it
    oe = orc.estimate(x, eb, mode=mode, stride=stride)
    compare_scalars(e, oe, case + "/exact-after")
    # the linear quantiser by the general equations is the SZ estimate itself
    if oe["hist_ovf"] == 0:
        assert close(g["lin_bits"], e["sz_entropy"]) and close(g["lin_psnr"], e["sz_psnr"])


def test_variants_full_size_and_errors(sel, orc):
    """A full C3 field (100 x 500 x 500, the tile kernel) against the oracle; argument and
    status errors."""
    import synth
    x = synth.make_field(3, 5)
    o = orc.estimate_variants(x, 1e-4, log_base=2, eqp_n=128)
    t = torch.from_numpy(x).cuda()
    with sel.Plan(x.shape, 1e-4, "rel") as p:
        g = p.estimate_variants(t, 2, 128)
        compare_variants(g, o, "c3 full")
        for b, n in ((1, 4), (2, 0), (2, 32769)):
            with pytest.raises(sel.SelError) as ei:
                p.estimate_variants(t, b, n)
            assert ei.value.status == sel.SEL_EINVAL
        bad = t.clone()
        bad[3, 7, 9] = float("nan")
        with pytest.raises(sel.SelError) as ei:
            p.estimate_variants(bad, 2, 4)
        assert ei.value.status == sel.SEL_ENONFINITE
    c = torch.full((8, 12), 2.5, device="cuda")
    with sel.Plan((8, 12), 1e-3, "rel") as p:
        with pytest.raises(sel.SelError) as ei:
            p.estimate_variants(c, 2, 4)
        assert ei.value.status == sel.SEL_EDEGENERATE


def test_field_stack_equals_list(sel):
    """Plan.field_stack (pointers marshalled once) gives the same results as the list form,
    sync and async, and validates shapes like the list form."""
    import synth
    xs = [torch.from_numpy(synth.c1_field(seed=i)).cuda() for i in range(5)]
    with sel.Plan((256, 256), 1e-4) as p:
        ref = p.estimate_batch(xs)
        stk = p.field_stack(xs)
        assert len(stk) == 5
        assert p.estimate_batch(stk) == ref
        buf = p.results_buffer(5)
        p.estimate_batch_async(stk, buf)
        torch.cuda.synchronize()
        assert p.decode_results(buf, 5) == ref
        with pytest.raises(ValueError):
            p.field_stack([xs[0], torch.zeros(8, 8, device="cuda")])
