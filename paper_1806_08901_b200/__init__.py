"""B200-native SZ-vs-ZFP rate-distortion estimator (arXiv 1806.08901, Alg. 1 lines 1-10).

Thin ctypes binding over the C ABI in ``include/sel.h`` (``libsel.so``, built in-tree by
``paper_1806_08901_b200.build``).  This module only marshals arguments: every step of
the estimate runs in the sm_100a kernels behind the ABI.  There is no CPU fallback --
if ``libsel.so`` is missing or CUDA is unavailable, calls raise.

PyTorch is used for device memory (``tensor.data_ptr()``) and streams
(``torch.cuda.current_stream().cuda_stream``) only.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsel.so")

SEL_OK, SEL_EINVAL, SEL_ENOMEM, SEL_ECUDA, SEL_ENONFINITE, SEL_EDEGENERATE, SEL_ENOTIMPL = (
    0, -1, -2, -3, -4, -5, -6)
EB_ABS, EB_REL = 0, 1

# every entry point declared in include/sel.h
EXPORTS = ("sel_plan", "sel_set_option", "sel_estimate", "sel_estimate_multi", "sel_estimate_paper",
           "sel_estimate_variants",
           "sel_compress_zfp",
           "sel_estimate_batch",
           "sel_estimate_batch_host", "sel_estimate_batch_async", "sel_choose", "sel_choose_eb",
           "sel_debug_copy", "sel_batch_layout", "sel_kernel_times",
           "sel_processed_blocks", "sel_processed_values", "sel_workspace_bytes",
           "sel_launch_count", "sel_plan_destroy", "sel_strerror")


class PaperResult(C.Structure):
    """Mirror of ``sel_paper_result`` (include/sel.h)."""
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
    """Mirror of ``sel_variant_result`` (include/sel.h)."""
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


class SelError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"sel status {status}: {msg}")
        self.status = status


class Result(C.Structure):
    """Mirror of ``sel_result`` (include/sel.h)."""
    _fields_ = [
        ("sz_bits_per_value", C.c_double), ("sz_psnr", C.c_double),
        ("zfp_bits_per_value", C.c_double), ("zfp_psnr", C.c_double),
        ("choice", C.c_int32), ("matched", C.c_int32),
        ("value_range", C.c_double), ("eb_abs", C.c_double), ("sz_entropy", C.c_double),
        ("sz_overflow_frac", C.c_double), ("sz_bits_matched", C.c_double),
        ("sz_eb_matched", C.c_double), ("zfp_mse", C.c_double),
        ("n_sz_points", C.c_uint64), ("n_values", C.c_uint64), ("n_blocks", C.c_uint64),
        ("zfp_total_bits", C.c_uint64), ("zfp_err_sum", C.c_double),
        ("minexp", C.c_int32), ("r_f", C.c_float), ("status", C.c_int32),
        ("choice_eb", C.c_int32), ("hist_total", C.c_uint64), ("hist_ovf", C.c_uint64),
    ]

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libsel.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1806_08901_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.sel_plan.argtypes = [C.POINTER(P), C.c_int, P, C.c_int, C.c_double, P, C.c_int32]
        L.sel_plan.restype = C.c_int
        L.sel_set_option.argtypes = [P, C.c_char_p, C.c_double]
        L.sel_set_option.restype = C.c_int
        L.sel_estimate.argtypes = [P, P, P, C.POINTER(Result)]
        L.sel_estimate.restype = C.c_int
        L.sel_compress_zfp.argtypes = [P, P, P, C.c_uint64, C.POINTER(C.c_uint64), P]
        L.sel_compress_zfp.restype = C.c_int
        L.sel_estimate_paper.argtypes = [P, P, P, C.POINTER(PaperResult)]
        L.sel_estimate_paper.restype = C.c_int
        L.sel_estimate_variants.argtypes = [P, P, C.c_int, C.c_int, P, C.POINTER(VariantResult)]
        L.sel_estimate_variants.restype = C.c_int
        L.sel_estimate_multi.argtypes = [P, P, C.c_int, P, P, P]
        L.sel_estimate_multi.restype = C.c_int
        L.sel_estimate_batch.argtypes = [P, P, C.c_int, P, P]
        L.sel_estimate_batch.restype = C.c_int
        L.sel_estimate_batch_async.argtypes = [P, P, C.c_int, P, P]
        L.sel_estimate_batch_async.restype = C.c_int
        L.sel_estimate_batch_host.argtypes = [P, P, C.c_int, P, P]
        L.sel_estimate_batch_host.restype = C.c_int
        L.sel_choose.argtypes = [C.POINTER(Result), C.POINTER(C.c_int32)]
        L.sel_choose.restype = C.c_int
        L.sel_choose_eb.argtypes = [C.POINTER(Result), C.POINTER(C.c_int32)]
        L.sel_choose_eb.restype = C.c_int
        L.sel_debug_copy.argtypes = [P, C.c_char_p, P, C.c_uint64]
        L.sel_debug_copy.restype = C.c_int
        L.sel_batch_layout.argtypes = [P, P]
        L.sel_batch_layout.restype = C.c_int
        L.sel_kernel_times.argtypes = [P, P, P, C.c_int]
        L.sel_kernel_times.restype = C.c_int
        for f in ("sel_processed_blocks", "sel_processed_values", "sel_launch_count"):
            getattr(L, f).argtypes = [P]
            getattr(L, f).restype = C.c_uint64
        L.sel_workspace_bytes.argtypes = [P]
        L.sel_workspace_bytes.restype = C.c_size_t
        L.sel_plan_destroy.argtypes = [P]
        L.sel_plan_destroy.restype = None
        L.sel_strerror.argtypes = [C.c_int]
        L.sel_strerror.restype = C.c_char_p
        _lib = L
    return _lib


def strerror(status: int) -> str:
    return lib().sel_strerror(status).decode()


def _check(status: int):
    if status != SEL_OK:
        raise SelError(status, strerror(status))


def _stream_ptr(stream):
    if stream is not None:
        return C.c_void_p(int(stream))
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _numel(shape) -> int:
    n = 1
    for s in shape:
        n *= int(s)
    return n


class FieldStack:
    """Marshalled pointers of a validated list of device fields (`Plan.field_stack`); holds
    references to the tensors so that the pointers stay valid."""
    __slots__ = ("ptrs", "n", "fields")

    def __init__(self, ptrs, n, fields):
        self.ptrs, self.n, self.fields = ptrs, n, fields

    def __len__(self):
        return self.n


def _device_ptr(t, shape=None, device=None) -> int:
    """Pointer of a contiguous float32 CUDA tensor holding prod(shape) values on the
    current device (the C ABI reads exactly prod(plan dims) floats from it)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor on a CUDA device")
    if not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError("field must be a contiguous float32 CUDA tensor")
    if shape is not None and t.numel() != _numel(shape):
        raise ValueError(f"field has {t.numel()} values, the plan's shape {tuple(shape)} needs "
                         f"{_numel(shape)}")
    dev = torch.cuda.current_device() if device is None else device
    if t.device.index != dev:
        raise ValueError(f"field is on {t.device}, the plan runs on cuda:{dev}")
    return t.data_ptr()


def _host_ptr(a, shape=None) -> int:
    n = None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous():
                raise ValueError("host field must be a contiguous float32 CPU tensor")
            n = a.numel()
            ptr = a.data_ptr()
    except ImportError:  # pragma: no cover
        pass
    if n is None:
        if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous):
            raise ValueError("host field must be a C-contiguous float32 array")
        n = a.size
        ptr = a.ctypes.data
    if shape is not None and n != _numel(shape):
        raise ValueError(f"host field has {n} values, the plan's shape {tuple(shape)} needs "
                         f"{_numel(shape)}")
    return ptr


class Plan:
    """An estimation plan for fields of one shape (owns the device workspace)."""

    def __init__(self, shape, eb: float, mode: str = "rel", stride=None, block: int = 4):
        shape = tuple(int(s) for s in shape)
        self.shape = shape
        self.ndims = len(shape)
        self.eb = float(eb)
        self.mode = mode
        self._dims = (C.c_int64 * max(self.ndims, 1))(*shape)
        self._stride = None if stride is None else (C.c_int32 * self.ndims)(*[int(s) for s in stride])
        self._h = C.c_void_p()
        self.device = None            # the CUDA device the plan's workspace lives on
        try:
            import torch
            if torch.cuda.is_available():
                self.device = torch.cuda.current_device()
        except ImportError:  # pragma: no cover
            pass
        m = EB_REL if mode == "rel" else EB_ABS
        if mode not in ("rel", "abs"):
            raise ValueError("mode must be 'rel' or 'abs'")
        _check(lib().sel_plan(C.byref(self._h), self.ndims, self._dims, m, self.eb,
                              self._stride, int(block)))

    # -- options / introspection
    def set_option(self, key: str, value: float):
        _check(lib().sel_set_option(self._h, key.encode(), float(value)))
        return self

    @property
    def processed_blocks(self) -> int:
        return int(lib().sel_processed_blocks(self._h))

    @property
    def processed_values(self) -> int:
        return int(lib().sel_processed_values(self._h))

    @property
    def workspace_bytes(self) -> int:
        return int(lib().sel_workspace_bytes(self._h))

    @property
    def launch_count(self) -> int:
        return int(lib().sel_launch_count(self._h))

    def kernel_times(self, reset: bool = False):
        ms = (C.c_double * 3)()
        n = (C.c_uint64 * 3)()
        _check(lib().sel_kernel_times(self._h, ms, n, int(reset)))
        return list(ms), list(n)

    # -- estimates
    def estimate(self, field, stream=None) -> dict:
        r = Result()
        _check(lib().sel_estimate(self._h, C.c_void_p(_device_ptr(field, self.shape, self.device)), _stream_ptr(stream),
                                  C.byref(r)))
        return r.to_dict()

    def compress_zfp(self, field, stream=None):
        """N3 (Alg. 1 line 13): the fixed-accuracy ZFP stream of `field` at the plan's eb
        (sel_compress_zfp) -> (uint8 CUDA tensor of the stream bytes, length in bits)."""
        import torch
        ptr = C.c_void_p(_device_ptr(field, self.shape, self.device))
        nbits = C.c_uint64()
        _check(lib().sel_compress_zfp(self._h, ptr, None, 0, C.byref(nbits), _stream_ptr(stream)))
        nbytes = (nbits.value + 31) // 32 * 4
        out = torch.empty(max(nbytes, 4), dtype=torch.uint8, device=field.device)
        _check(lib().sel_compress_zfp(self._h, ptr, C.c_void_p(out.data_ptr()), out.numel(), C.byref(nbits),
                                      _stream_ptr(stream)))
        return out[:nbytes], int(nbits.value)

    def estimate_paper(self, field, stream=None) -> dict:
        """N2: the paper-literal estimate (sel_estimate_paper): sampled-coefficient n_sb
        bit-rate, unit-weight PSNR_sp, SZ re-quantised at the matching delta."""
        r = PaperResult()
        _check(lib().sel_estimate_paper(self._h, C.c_void_p(_device_ptr(field, self.shape, self.device)),
                                        _stream_ptr(stream), C.byref(r)))
        return r.to_dict()

    def estimate_variants(self, field, log_base: int = 2, eqp_n: int = 128, stream=None) -> dict:
        """N4: the log-scale and equal-probability quantisation estimates on the field's
        code histogram (sel_estimate_variants)."""
        r = VariantResult()
        _check(lib().sel_estimate_variants(self._h, C.c_void_p(_device_ptr(field, self.shape, self.device)),
                                           int(log_base), int(eqp_n), _stream_ptr(stream), C.byref(r)))
        return r.to_dict()

    def estimate_multi(self, field, ebs, stream=None) -> list[dict]:
        """N1: the estimates at every error bound in `ebs` (1..8, the plan's mode) from one
        read of `field` (sel_estimate_multi); one result dict per eb."""
        k = len(ebs)
        arr = (C.c_double * k)(*[float(e) for e in ebs])
        out = (Result * k)()
        _check(lib().sel_estimate_multi(self._h, C.c_void_p(_device_ptr(field, self.shape, self.device)), k,
                                        arr, _stream_ptr(stream), out))
        return [o.to_dict() for o in out]

    def estimate_batch(self, fields, stream=None) -> list[dict]:
        if isinstance(fields, FieldStack):
            n, ptrs = fields.n, fields.ptrs
        else:
            n = len(fields)
            ptrs = (C.c_void_p * n)(*[_device_ptr(f, self.shape, self.device) for f in fields])
        out = (Result * n)()
        _check(lib().sel_estimate_batch(self._h, ptrs, n, _stream_ptr(stream), out))
        return [o.to_dict() for o in out]

    def field_stack(self, fields) -> "FieldStack":
        """Validate a list of device fields once and keep their pointers marshalled
        (argument marshalling only): pass the stack to `estimate_batch[_async]` instead of
        the list when the same resident fields are estimated repeatedly -- per call the list
        form costs ~1 us of Python per field, more than the kernel on small fields."""
        n = len(fields)
        ptrs = (C.c_void_p * n)(*[_device_ptr(f, self.shape, self.device) for f in fields])
        return FieldStack(ptrs, n, list(fields))

    def estimate_batch_async(self, fields, out, stream=None):
        """Enqueue the estimate of `fields` (a list of device tensors or a `field_stack`)
        and the copy of their results into `out` (a pinned-host or CUDA uint8 tensor from
        `results_buffer`) on `stream`; returns at once.  Decode with `decode_results(out)`
        after synchronising the stream."""
        if isinstance(fields, FieldStack):
            n, ptrs = fields.n, fields.ptrs
        else:
            n = len(fields)
            ptrs = (C.c_void_p * n)(*[_device_ptr(f, self.shape, self.device) for f in fields])
        if out.numel() < n * C.sizeof(Result):
            raise ValueError("results buffer too small")
        _check(lib().sel_estimate_batch_async(self._h, ptrs, n, _stream_ptr(stream),
                                              C.c_void_p(out.data_ptr())))

    @staticmethod
    def results_buffer(n: int, device="pinned"):
        """uint8 tensor for n results: page-locked host memory, or a CUDA device."""
        import torch
        nb = n * C.sizeof(Result)
        if device == "pinned":
            return torch.empty(nb, dtype=torch.uint8).pin_memory()
        return torch.empty(nb, dtype=torch.uint8, device=device)

    @staticmethod
    def decode_results(buf, n: int | None = None) -> list[dict]:
        raw = bytes(buf.cpu().numpy().tobytes()) if buf.is_cuda else bytes(buf.numpy().tobytes())
        n = len(raw) // C.sizeof(Result) if n is None else n
        arr = (Result * n).from_buffer_copy(raw[: n * C.sizeof(Result)])
        return [o.to_dict() for o in arr]

    def estimate_batch_host(self, fields, stream=None) -> list[dict]:
        n = len(fields)
        ptrs = (C.c_void_p * n)(*[_host_ptr(f, self.shape) for f in fields])
        out = (Result * n)()
        _check(lib().sel_estimate_batch_host(self._h, ptrs, n, _stream_ptr(stream), out))
        return [o.to_dict() for o in out]

    def debug_copy(self, what: str) -> np.ndarray:
        S = 4 ** self.ndims
        B = self.processed_blocks
        spec = {"codes": (np.int32, self.shape), "hist": (np.uint64, (65536,)),
                "emax": (np.int32, (B,)), "coef": (np.int32, (B, S)),
                "uword": (np.uint32, (B, S)), "bits": (np.uint32, (B,)),
                "err": (np.float64, (B,))}[what]
        a = np.empty(spec[1], spec[0])
        _check(lib().sel_debug_copy(self._h, what.encode(), a.ctypes.data_as(C.c_void_p), a.nbytes))
        return a

    def batch_layout(self) -> dict:
        o = (C.c_int64 * 8)()
        _check(lib().sel_batch_layout(self._h, o))
        keys = ("n_tasks", "parts_per_task", "rows_per_part", "rows_per_tile", "ntk", "ntj",
                "sampled", "groups")
        return dict(zip(keys, [int(v) for v in o]))

    def batch_debug_copy(self, what: str, nf: int) -> np.ndarray:
        """k_batch dumps of the last batch launch (option batch_debug=1): "hist" ->
        uint32[nf, 65536]; "part" -> structured [nf, n_tasks * parts_per_task] of
        (bits u64, err f64)."""
        lay = self.batch_layout()
        if what == "hist":
            a = np.empty((nf, 65536), np.uint32)
        elif what == "part":
            a = np.empty((nf, lay["n_tasks"] * lay["parts_per_task"]),
                         np.dtype([("bits", np.uint64), ("err", np.float64)]))
        else:
            raise ValueError(what)
        _check(lib().sel_debug_copy(self._h, ("batch_" + what).encode(),
                                    a.ctypes.data_as(C.c_void_p), a.nbytes))
        return a

    def close(self):
        if self._h:
            lib().sel_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def estimate(field, eb: float, mode: str = "rel", stride=None, stream=None) -> dict:
    """One-shot: SZ/ZFP rate-distortion estimate and Alg. 1 choice for a CUDA tensor."""
    with Plan(tuple(field.shape), eb, mode, stride) as p:
        return p.estimate(field, stream)


def choose(result: dict) -> int:
    """Host-side Alg. 1 lines 7-10 recomputed from a result dict."""
    r = Result()
    for k, _ in Result._fields_:
        if k in result:
            setattr(r, k, result[k])
    c = C.c_int32()
    _check(lib().sel_choose(C.byref(r), C.byref(c)))
    return int(c.value)


def choose_eb(result: dict) -> int:
    """Host-side fixed-error-bound selector (Lu et al.): the compressor
    with the lower bit-rate at the user's eb, ties to ZFP."""
    r = Result()
    for k, _ in Result._fields_:
        if k in result:
            setattr(r, k, result[k])
    c = C.c_int32()
    _check(lib().sel_choose_eb(C.byref(r), C.byref(c)))
    return int(c.value)
