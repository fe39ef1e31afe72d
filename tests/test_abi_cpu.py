"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/sel.h declares, and the pure-host entry points behave."""
import math
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sel():
    from paper_1806_08901_b200 import build
    build.build()
    import paper_1806_08901_b200 as sel
    sel.lib()
    return sel


def header_functions():
    src = open(os.path.join(ROOT, "include", "sel.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sel_[a-z_]+)\s*\(", src)))


def test_header_and_binding_agree(sel):
    assert header_functions() == sorted(sel.EXPORTS)


def test_library_exports_every_header_symbol(sel):
    out = subprocess.check_output(["nm", "-D", "--defined-only", sel.LIB_PATH]).decode()
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for f in header_functions():
        assert f in syms, f


def test_library_is_sm100a(sel):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sel.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_result_struct_layout(sel, tmp_path):
    """The ctypes mirror has the C struct's size and every member's offset (gcc on
    include/sel.h)."""
    import ctypes
    names = [k for k, _ in sel.Result._fields_]
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"sel.h\"\nint main(void){\n"
    src += 'printf("%zu\\n", sizeof(sel_result));\n'
    for k in names:
        src += f'printf("%zu\\n", offsetof(sel_result, {k}));\n'
    src += "return 0;}\n"
    c = tmp_path / "layout.c"
    c.write_text(src)
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    vals = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert vals[0] == ctypes.sizeof(sel.Result)
    for k, off in zip(names, vals[1:]):
        assert getattr(sel.Result, k).offset == off, k


def test_strerror(sel):
    assert sel.strerror(0) == "ok"
    assert "NaN" in sel.strerror(sel.SEL_ENONFINITE)
    assert sel.strerror(12345) == "unknown status"


def test_plan_rejects_bad_arguments_without_gpu(sel):
    for kw in (dict(shape=(4, 4), eb=0.0), dict(shape=(4, 4), eb=-1.0), dict(shape=(4, 4), eb=math.nan),
               dict(shape=(4, 4, 4, 4), eb=1e-3), dict(shape=(0, 4), eb=1e-3),
               dict(shape=(8, 8), eb=1e-3, stride=(0, 1)), dict(shape=(8, 8), eb=1e-3, block=8),
               dict(shape=(8,), eb=1e-300, mode="abs")):
        with pytest.raises(sel.SelError) as e:
            sel.Plan(**kw)
        assert e.value.status == sel.SEL_EINVAL, kw


def test_choose_matches_oracle_selection(sel, orc):
    """sel_choose (host, Alg. 1 lines 7-10) agrees with the oracle's selection."""
    rng = np.random.default_rng(0)
    for _ in range(2000):
        vr = float(10 ** rng.uniform(-3, 3))
        eb = vr * float(10 ** rng.uniform(-7, -2))
        br_sz = float(rng.uniform(0.5, 20))
        br_zfp = float(rng.uniform(0.1, 25))
        mse = float((eb ** 2) * 10 ** rng.uniform(-3, 1)) if rng.random() > 0.05 else 0.0
        psnr_zfp = 20 * math.log10(vr) - 10 * math.log10(mse) if mse > 0 else math.inf
        psnr_sz = 20 * math.log10(vr / eb) + 10 * math.log10(3)
        ch, bm, ebm, m = orc.select(br_sz, psnr_sz, br_zfp, psnr_zfp, vr, eb, mse)
        r = dict(sz_bits_per_value=br_sz, zfp_bits_per_value=br_zfp, zfp_psnr=psnr_zfp,
                 zfp_mse=mse, value_range=vr, eb_abs=eb, sz_psnr=psnr_sz)
        assert sel.choose(r) == ch


def test_choose_eb_matches_oracle_selection(sel, orc):
    """sel_choose_eb (host, the fixed-error-bound selector of P:639-642) agrees with the
    oracle's, including ties (-> ZFP)."""
    rng = np.random.default_rng(1)
    for _ in range(2000):
        br_sz = float(rng.uniform(0.5, 20))
        br_zfp = br_sz if rng.random() < 0.1 else float(rng.uniform(0.1, 25))
        r = dict(sz_bits_per_value=br_sz, zfp_bits_per_value=br_zfp)
        assert sel.choose_eb(r) == orc.select_eb(br_sz, br_zfp)


def test_product_path_has_no_oracle_dependency():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_1806_08901_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f == "__init__.py" and \
                    "import oracle" not in txt, f
                assert "import oracle" not in txt and "orc.h" not in txt and "liborc" not in txt, f
