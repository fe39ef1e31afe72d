"""CPU ORACLE for the SZ-vs-ZFP rate-distortion estimator (arXiv 1806.08901).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_1806_08901_b200``);
neither imports the other.

The arithmetic lives in ``orc.c`` (plain sequential C, fp64 except the fp32
Lorenzo/quantise decision, R4/R5).  This module only marshals
arguments through ctypes and compiles ``orc.c`` with gcc on first use.

Parity status: every function is pinned by ``tests/test_oracle_pins.py``
(closed forms, brute force, invariants, hand examples under ``tests/golden``)
except the absolute agreement with the real SZ-1.4.11 / ZFP-0.5.0 codecs,
which is "parity unpinned" (the codecs are not in the container).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "orc.c")
_HDR = os.path.join(_HERE, "orc.h")
_LIB = os.path.join(_HERE, "liborc.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=gnu11", "-pthread", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
          "-Wall", "-Wextra"]

NSLOTS = 65536
OVF_SLOT = 65535
STATUS = {0: "OK", -1: "EINVAL", -4: "ENONFINITE", -5: "EDEGENERATE"}


class OracleError(RuntimeError):
    def __init__(self, status: int):
        super().__init__(f"oracle status {status} ({STATUS.get(status, '?')})")
        self.status = status


def build(force: bool = False) -> str:
    """Compile orc.c -> liborc.so (gcc, no fast-math, no FMA contraction)."""
    stale = (not os.path.exists(_LIB) or
             os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


class Result(C.Structure):
    _fields_ = [
        ("sz_bits_per_value", C.c_double), ("sz_psnr", C.c_double),
        ("zfp_bits_per_value", C.c_double), ("zfp_psnr", C.c_double),
        ("choice", C.c_int32), ("matched", C.c_int32),
        ("value_range", C.c_double), ("eb_abs", C.c_double), ("sz_entropy", C.c_double),
        ("sz_overflow_frac", C.c_double), ("sz_bits_matched", C.c_double),
        ("sz_eb_matched", C.c_double), ("zfp_mse", C.c_double),
        ("n_sz_points", C.c_uint64), ("n_values", C.c_uint64), ("n_blocks", C.c_uint64),
        ("zfp_total_bits", C.c_uint64), ("zfp_err_sum", C.c_double),
        ("minexp", C.c_int32), ("r_f", C.c_float), ("choice_eb", C.c_int32),
        ("pad_", C.c_int32), ("hist_total", C.c_uint64), ("hist_ovf", C.c_uint64),
    ]

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


class PaperResult(C.Structure):
    """Mirror of orc_paper_result (orc.h): the paper-literal estimator, SURVEY 8(f) N2."""
    _fields_ = [
        ("zfp_nsb_bits", C.c_double), ("zfp_mse_sp", C.c_double), ("zfp_psnr_sp", C.c_double),
        ("sz_delta", C.c_double), ("sz_bits", C.c_double), ("sz_entropy", C.c_double),
        ("sz_overflow_frac", C.c_double), ("value_range", C.c_double), ("eb_abs", C.c_double),
        ("nsb2_total", C.c_uint64), ("n_samples", C.c_uint64), ("n_values", C.c_uint64),
        ("hist_total", C.c_uint64), ("hist_ovf", C.c_uint64), ("r_star", C.c_float),
        ("choice", C.c_int32), ("matched", C.c_int32), ("status", C.c_int32),
    ]

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class VariantResult(C.Structure):
    """Mirror of orc_variant_result (orc.h): the variant quantisers, SURVEY 8(f) N4."""
    _fields_ = [
        ("lin_bits", C.c_double), ("lin_psnr", C.c_double),
        ("log_bits", C.c_double), ("log_psnr", C.c_double), ("log_mse", C.c_double),
        ("eqp_bits", C.c_double), ("eqp_psnr", C.c_double), ("eqp_mse", C.c_double),
        ("eqp_width_sum", C.c_double), ("value_range", C.c_double), ("eb_abs", C.c_double),
        ("n_in", C.c_uint64), ("hist_ovf", C.c_uint64),
        ("log_base", C.c_int32), ("log_bins", C.c_int32), ("eqp_n", C.c_int32), ("status", C.c_int32),
    ]

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class Debug(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("hist", C.c_void_p), ("emax", C.c_void_p),
                ("coef", C.c_void_p), ("uword", C.c_void_p), ("bits", C.c_void_p),
                ("err", C.c_void_p)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            P = C.c_void_p
            L.orc_estimate.argtypes = [P, C.c_int, P, C.c_int, C.c_double, P, C.c_double, P, P]
            L.orc_estimate.restype = C.c_int
            L.orc_estimate_mt.argtypes = [P, C.c_int, P, C.c_int, C.c_double, P, C.c_double, P, P,
                                          C.c_int]
            L.orc_estimate_mt.restype = C.c_int
            L.orc_estimate_paper.argtypes = [P, C.c_int, P, C.c_int, C.c_double, P, C.c_double, P]
            L.orc_estimate_paper.restype = C.c_int
            L.orc_variants_from_hist.argtypes = [P, C.c_double, C.c_double, C.c_int, C.c_int, P]
            L.orc_variants_from_hist.restype = C.c_int
            L.orc_estimate_variants.argtypes = [P, C.c_int, P, C.c_int, C.c_double, P, C.c_int, C.c_int, P]
            L.orc_estimate_variants.restype = C.c_int
            L.orc_paper_positions.argtypes = [C.c_int, P]
            L.orc_paper_positions.restype = C.c_int
            L.orc_block_paper.argtypes = [P, C.c_int, C.c_int, C.c_int32, P, P]
            L.orc_block_paper.restype = None
            L.orc_zfp_stream.argtypes = [P, C.c_int, P, C.c_int, C.c_double, P, P, C.c_uint64, P]
            L.orc_zfp_stream.restype = C.c_int
            L.orc_zfp_stream_decode.argtypes = [P, C.c_uint64, C.c_int, P, C.c_int, C.c_double, C.c_double,
                                                P, P]
            L.orc_zfp_stream_decode.restype = C.c_int
            L.orc_processed_blocks.argtypes = [C.c_int, P, P]
            L.orc_processed_blocks.restype = C.c_uint64
            L.orc_lorenzo.argtypes = [P, C.c_int, P, P]
            L.orc_lorenzo.restype = C.c_float
            L.orc_quantize.argtypes = [C.c_float, C.c_float]
            L.orc_quantize.restype = C.c_int32
            L.orc_entropy_counts.argtypes = [P, C.c_int64]
            L.orc_entropy_counts.restype = C.c_double
            for f in ("orc_fwd_lift4", "orc_inv_lift4"):
                getattr(L, f).argtypes = [P, C.c_int64]
                getattr(L, f).restype = None
            for f in ("orc_fwd_xform", "orc_inv_xform"):
                getattr(L, f).argtypes = [P, C.c_int]
                getattr(L, f).restype = None
            L.orc_sequency_perm.argtypes = [C.c_int, P]
            L.orc_sequency_perm.restype = None
            L.orc_negabinary.argtypes = [C.c_int32]
            L.orc_negabinary.restype = C.c_uint32
            L.orc_negabinary_inv.argtypes = [C.c_uint32]
            L.orc_negabinary_inv.restype = C.c_int32
            L.orc_block_emax.argtypes = [P, C.c_int]
            L.orc_block_emax.restype = C.c_int32
            L.orc_block_bfp.argtypes = [P, C.c_int, C.c_int32, P]
            L.orc_block_bfp.restype = None
            L.orc_precision.argtypes = [C.c_int32, C.c_int32, C.c_int]
            L.orc_precision.restype = C.c_int32
            L.orc_gt_count.argtypes = [P, C.c_int, C.c_int]
            L.orc_gt_count.restype = C.c_uint64
            L.orc_gt_encode.argtypes = [P, C.c_int, C.c_int, P, C.c_uint64]
            L.orc_gt_encode.restype = C.c_uint64
            L.orc_gt_decode.argtypes = [P, C.c_uint64, C.c_int, C.c_int, P]
            L.orc_gt_decode.restype = C.c_uint64
            L.orc_block_err.argtypes = [P, P, P, C.c_int, C.c_int, C.c_int32]
            L.orc_block_err.restype = C.c_double
            L.orc_gain.argtypes = [C.c_int, C.c_int]
            L.orc_gain.restype = C.c_double
            L.orc_select.argtypes = [C.c_double] * 7 + [P, P, P]
            L.orc_select.restype = C.c_int
            L.orc_select_eb.argtypes = [C.c_double, C.c_double]
            L.orc_select_eb.restype = C.c_int
            _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dims_stride(shape, stride):
    nd = len(shape)
    dims = np.ascontiguousarray(shape, dtype=np.int64)
    st = None if stride is None else np.ascontiguousarray(stride, dtype=np.int32)
    if st is not None and st.shape != (nd,):
        raise ValueError("stride must have one entry per dimension")
    return nd, dims, st


def processed_blocks(shape, stride=None) -> int:
    nd, dims, st = _dims_stride(shape, stride)
    return int(lib().orc_processed_blocks(nd, _ptr(dims), None if st is None else _ptr(st)))


def default_threads() -> int:
    """Host cores this process may run on (the affinity set)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def estimate_multi(x: np.ndarray, ebs, mode: str = "rel", stride=None, threads: int = 1) -> list:
    """SURVEY 8(f) N1 by its definition: the estimate of Alg. 1 lines 1-10 at every error
    bound of the rate-distortion sweep, one plain estimate per eb."""
    return [estimate(x, e, mode=mode, stride=stride, threads=threads) for e in ebs]


def estimate(x: np.ndarray, eb: float, mode: str = "rel", stride=None, sz_offset: float = 0.5,
             debug: bool = False, threads: int = 1) -> dict:
    """Alg. 1 lines 1-10 on a C-order float32 field.

    threads > 1 runs orc_estimate_mt: contiguous slabs of blocks per thread, exact merges,
    bit-identical to threads = 1 (0 = every core of the affinity set)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    nd, dims, st = _dims_stride(x.shape, stride)
    size = 4 ** nd
    res = Result()
    dbgs = None
    arrays = {}
    if debug:
        # debug=True: every dump; or an iterable of names ("codes", "hist", "emax",
        # "coef", "uword", "bits", "err") to keep memory bounded on full-size fields
        want = {k for k, _ in Debug._fields_} if debug is True else set(debug)
        npb = processed_blocks(x.shape, stride)
        spec = {
            "codes": (x.shape, np.int32), "hist": ((NSLOTS,), np.uint64),
            "emax": ((npb,), np.int32), "coef": ((npb, size), np.int32),
            "uword": ((npb, size), np.uint32), "bits": ((npb,), np.uint32),
            "err": ((npb,), np.float64),
        }
        arrays = {k: (np.zeros if k == "hist" else np.empty)(spec[k][0], spec[k][1]) for k in want}
        dbgs = Debug(*[_ptr(arrays[k]) if k in arrays else None for k, _ in Debug._fields_])
    nthr = default_threads() if threads == 0 else int(threads)
    st_ = lib().orc_estimate_mt(_ptr(x), nd, _ptr(dims), 1 if mode == "rel" else 0, float(eb),
                                None if st is None else _ptr(st), float(sz_offset), C.byref(res),
                                C.byref(dbgs) if dbgs is not None else None, nthr)
    if st_ != 0:
        raise OracleError(st_)
    out = res.to_dict()
    if debug:
        out["debug"] = arrays
    return out


def estimate_paper(x: np.ndarray, eb: float, mode: str = "rel", stride=None,
                   sz_offset: float = 0.5) -> dict:
    """SURVEY 8(f) N2, the paper-literal estimator (orc_estimate_paper): BR_zfp = the
    interpolated n_sb average of 3/9/16 sampled coefficients per block,
    PSNR_sp from the unit-weight MSE of those samples, SZ re-quantised at the
    delta that matches PSNR_sp (Alg. 1 lines 7-9), Alg. 1 line 10's choice."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    nd, dims, st = _dims_stride(x.shape, stride)
    res = PaperResult()
    st_ = lib().orc_estimate_paper(_ptr(x), nd, _ptr(dims), 1 if mode == "rel" else 0, float(eb),
                                   None if st is None else _ptr(st), float(sz_offset), C.byref(res))
    if st_ != 0:
        raise OracleError(st_)
    return res.to_dict()


def variants_from_hist(hist: np.ndarray, value_range: float, eb_abs: float, log_base: int = 2,
                       eqp_n: int = 128) -> dict:
    """SURVEY 8(f) N4 on a given 65,536-slot code histogram (orc_variants_from_hist)."""
    h = np.ascontiguousarray(hist, dtype=np.uint64)
    assert h.size == NSLOTS
    res = VariantResult()
    rc = lib().orc_variants_from_hist(_ptr(h), float(value_range), float(eb_abs), int(log_base), int(eqp_n),
                                      C.byref(res))
    if rc != 0:
        raise OracleError(rc)
    return res.to_dict()


def estimate_variants(x: np.ndarray, eb: float, mode: str = "rel", stride=None, log_base: int = 2,
                      eqp_n: int = 128) -> dict:
    """SURVEY 8(f) N4 (orc_estimate_variants): the log-scale and equal-probability
     quantisation estimates, with the linear one by the same general equations
    (P:396-403), on the field's code histogram (the stored PDF)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    nd, dims, st = _dims_stride(x.shape, stride)
    res = VariantResult()
    rc = lib().orc_estimate_variants(_ptr(x), nd, _ptr(dims), 1 if mode == "rel" else 0, float(eb),
                                     None if st is None else _ptr(st), int(log_base), int(eqp_n), C.byref(res))
    if rc != 0:
        raise OracleError(rc)
    return res.to_dict()


def zfp_stream(x: np.ndarray, eb: float, mode: str = "rel", stride=None):
    """SURVEY 8(f) N3 (Alg. 1 line 13): the fixed-accuracy ZFP stream of the processed
    blocks -> (bytes as uint8 array, length in bits)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    nd, dims, st = _dims_stride(x.shape, stride)
    nbits = C.c_uint64()
    m = 1 if mode == "rel" else 0
    sp = None if st is None else _ptr(st)
    rc = lib().orc_zfp_stream(_ptr(x), nd, _ptr(dims), m, float(eb), sp, None, 0, C.byref(nbits))
    if rc != 0:
        raise OracleError(rc)
    buf = np.zeros(((nbits.value + 31) // 32) * 4, np.uint8)
    rc = lib().orc_zfp_stream(_ptr(x), nd, _ptr(dims), m, float(eb), sp, _ptr(buf), buf.size, C.byref(nbits))
    if rc != 0:
        raise OracleError(rc)
    return buf, int(nbits.value)


def zfp_stream_decode(buf: np.ndarray, nbits: int, shape, eb: float, value_range: float, mode: str = "rel",
                      stride=None) -> np.ndarray:
    """Decode a zfp_stream back to float32 values (processed blocks; others 0)."""
    nd, dims, st = _dims_stride(tuple(shape), stride)
    out = np.zeros(shape, np.float32)
    b = np.ascontiguousarray(buf, dtype=np.uint8)
    rc = lib().orc_zfp_stream_decode(_ptr(b), int(nbits), nd, _ptr(dims), 1 if mode == "rel" else 0, float(eb),
                                     float(value_range), None if st is None else _ptr(st), _ptr(out))
    if rc != 0:
        raise OracleError(rc)
    return out


def paper_positions(nd: int) -> np.ndarray:
    pos = np.zeros(16, np.int32)
    m = lib().orc_paper_positions(nd, _ptr(pos))
    return pos[:m].copy()


def block_paper(u_seq, nd: int, kmin: int, emax: int):
    """(2 x sum of interpolated n_sb, sum of sampled squared errors) of one block."""
    u = np.ascontiguousarray(u_seq, dtype=np.uint32)
    n2 = C.c_uint64()
    mn = C.c_double()
    lib().orc_block_paper(_ptr(u), nd, int(kmin), int(emax), C.byref(n2), C.byref(mn))
    return int(n2.value), float(mn.value)


# ---- single steps (pin tests) ----
def lorenzo(x: np.ndarray, idx) -> np.float32:
    x = np.ascontiguousarray(x, dtype=np.float32)
    nd, dims, _ = _dims_stride(x.shape, None)
    i = np.ascontiguousarray(idx, dtype=np.int64)
    return np.float32(lib().orc_lorenzo(_ptr(x), nd, _ptr(dims), _ptr(i)))


def quantize(d: float, r_f: float) -> int:
    return int(lib().orc_quantize(float(np.float32(d)), float(np.float32(r_f))))


def entropy(counts) -> float:
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    return float(lib().orc_entropy_counts(_ptr(c), c.size))


def fwd_xform(blk: np.ndarray, nd: int) -> np.ndarray:
    b = np.ascontiguousarray(blk, dtype=np.int32).copy()
    assert b.size == 4 ** nd
    lib().orc_fwd_xform(_ptr(b), nd)
    return b


def inv_xform(blk: np.ndarray, nd: int) -> np.ndarray:
    b = np.ascontiguousarray(blk, dtype=np.int32).copy()
    assert b.size == 4 ** nd
    lib().orc_inv_xform(_ptr(b), nd)
    return b


def sequency_perm(nd: int) -> np.ndarray:
    p = np.empty(4 ** nd, np.int32)
    lib().orc_sequency_perm(nd, _ptr(p))
    return p


def negabinary(c: int) -> int:
    return int(lib().orc_negabinary(int(c)))


def negabinary_inv(u: int) -> int:
    return int(lib().orc_negabinary_inv(int(u) & 0xFFFFFFFF))


def block_emax(blk) -> int:
    b = np.ascontiguousarray(blk, dtype=np.float32)
    return int(lib().orc_block_emax(_ptr(b), b.size))


def block_bfp(blk, emax: int) -> np.ndarray:
    b = np.ascontiguousarray(blk, dtype=np.float32)
    o = np.empty(b.size, np.int32)
    lib().orc_block_bfp(_ptr(b), b.size, int(emax), _ptr(o))
    return o


def precision(emax: int, minexp: int, nd: int) -> int:
    return int(lib().orc_precision(int(emax), int(minexp), nd))


def gt_count(u, kmin: int) -> int:
    a = np.ascontiguousarray(u, dtype=np.uint32)
    return int(lib().orc_gt_count(_ptr(a), a.size, int(kmin)))


def gt_encode(u, kmin: int) -> tuple[bytes, int]:
    a = np.ascontiguousarray(u, dtype=np.uint32)
    cap = 64 * 33 + 64
    buf = np.zeros((cap + 7) // 8, np.uint8)
    n = int(lib().orc_gt_encode(_ptr(a), a.size, int(kmin), _ptr(buf), cap))
    return buf.tobytes(), n


def gt_decode(buf: bytes, nbits: int, size: int, kmin: int) -> tuple[np.ndarray, int]:
    b = np.frombuffer(buf, np.uint8).copy()
    u = np.zeros(size, np.uint32)
    n = int(lib().orc_gt_decode(_ptr(b), int(nbits), size, int(kmin), _ptr(u)))
    return u, n


def block_err(coef_nat, u_seq, nd: int, kmin: int, emax: int) -> float:
    c = np.ascontiguousarray(coef_nat, dtype=np.int32)
    u = np.ascontiguousarray(u_seq, dtype=np.uint32)
    p = sequency_perm(nd)
    return float(lib().orc_block_err(_ptr(c), _ptr(u), _ptr(p), nd, int(kmin), int(emax)))


def gain(nd: int, n: int) -> float:
    return float(lib().orc_gain(nd, n))


def select(br_sz, psnr_sz, br_zfp, psnr_zfp, vr, eb_abs, zfp_mse):
    bm = C.c_double()
    ebm = C.c_double()
    m = C.c_int32()
    ch = lib().orc_select(br_sz, psnr_sz, br_zfp, psnr_zfp, vr, eb_abs, zfp_mse,
                          C.byref(bm), C.byref(ebm), C.byref(m))
    return int(ch), bm.value, ebm.value, int(m.value)


def select_eb(br_sz, br_zfp):
    """Selection based on the error bound (Lu et al.)."""
    return int(lib().orc_select_eb(br_sz, br_zfp))
