"""paper_2203_01877_b200 -- B200-native hot path of TQP (arXiv 2203.01877).

Thin Python binding over libtqp.so (C ABI in include/tqp.h). This module only
marshals arguments: torch tensors in (device memory, streams), raw pointers and
sizes across the ABI, torch tensors out. Every step of the hot path runs in the
library's CUDA kernels; there is no CPU fallback. Importing the package without
a built libtqp.so raises ImportError.

Operators (same names as the C ABI, PAPER.md citations in include/tqp.h):
  sort, pkfk_join, pkfk_semi, smj_prepare / SmjPlan.expand, smj_join,
  filter_compact, groupby_agg
"""

import ctypes
import sys
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libtqp.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libtqp.so not built ({_LIB_PATH}); run `python -m paper_2203_01877_b200.build` "
                      "or __graft_entry__.build()")

_lib = ctypes.CDLL(_LIB_PATH)

TQP_OK, TQP_ERR_INVALID_ARGUMENT, TQP_ERR_DUPLICATE_BUILD_KEY, TQP_ERR_OUT_OF_MEMORY, TQP_ERR_CUDA, \
    TQP_ERR_OVERFLOW, TQP_ERR_CAPACITY = range(7)
TQP_U8, TQP_I32, TQP_I64, TQP_F64 = 1, 2, 3, 4
OPS = {"lt": 0, "le": 1, "gt": 2, "ge": 3, "eq": 4, "ne": 5, "<": 0, "<=": 1, ">": 2, ">=": 3, "==": 4, "!=": 5}
AGGS = {"sum": 0, "count": 1, "min": 2, "max": 3, "avg": 4}
MAX_PREDS, MAX_KEYS, MAX_AGGS = 16, 8, 16

EXPORTED = [
    "tqp_abi_version", "tqp_ctx_create", "tqp_ctx_destroy", "tqp_ctx_set_stream", "tqp_last_error",
    "tqp_ctx_launch_count", "tqp_ctx_guard_violations", "tqp_ctx_reset_counters", "tqp_ctx_set_profiling", "tqp_ctx_set_profiling_filter",
    "tqp_ctx_kernel_stats",
    "tqp_sort", "tqp_pkfk_join", "tqp_pkfk_semi", "tqp_pkfk_outer", "tqp_pkfk_join_payload", "tqp_pkfk_join_hash",
    "tqp_pkfk_join_i32", "tqp_pkfk_join_paper_order", "tqp_smj_prepare", "tqp_smj_expand", "tqp_smj_expand_i32", "tqp_smj_expand_checksum",
    "tqp_smj_release",
    "tqp_smj_join", "tqp_pack_keys", "tqp_filter_compact", "tqp_groupby_prepare", "tqp_groupby_fetch", "tqp_groupby_release",
    "tqp_groupby_agg", "tqp_groupby_merge", "tqp_smj_expand_payload", "tqp_partition", "tqp_minmax",
    "tqp_range_splitters", "tqp_gather", "tqp_pkfk_outer_build", "tqp_partition_plan_create", "tqp_partition_scatter",
    "tqp_partition_release", "tqp_ipc_alloc", "tqp_ipc_free", "tqp_ipc_open", "tqp_ipc_close", "tqp_jit_counters",
    "tqp_ctx_set_allocator", "tqp_ctx_trim", "tqp_ctx_cached_bytes",
]


class Col(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class Pred(ctypes.Structure):
    _fields_ = [("col", ctypes.c_int32), ("op", ctypes.c_int32), ("value", ctypes.c_int64)]


class Agg(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("n_factors", ctypes.c_int32), ("col", ctypes.c_int32 * 3),
                ("sign", ctypes.c_int32 * 3), ("add", ctypes.c_int64 * 3)]


_vp, _i64, _int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
_P = ctypes.POINTER
_sig = {
    "tqp_abi_version": ([], _int),
    "tqp_ctx_create": ([_int, _vp, _P(_vp)], _int),
    "tqp_ctx_destroy": ([_vp], None),
    "tqp_ctx_set_stream": ([_vp, _vp], _int),
    "tqp_last_error": ([_vp], ctypes.c_char_p),
    "tqp_ctx_launch_count": ([_vp], _i64),
    "tqp_ctx_guard_violations": ([_vp], _i64),
    "tqp_jit_counters": ([_vp, _vp, _vp], ctypes.c_int),
    "tqp_ctx_set_allocator": ([_vp, _vp, _vp, _vp], _int),
    "tqp_ctx_trim": ([_vp], _int),
    "tqp_ctx_cached_bytes": ([_vp], ctypes.c_size_t),
    "tqp_ctx_reset_counters": ([_vp], None),
    "tqp_ctx_set_profiling": ([_vp, _int], _int),
    "tqp_ctx_set_profiling_filter": ([_vp, ctypes.c_char_p], _int),
    "tqp_ctx_kernel_stats": ([_vp, ctypes.c_char_p, ctypes.c_size_t, _P(ctypes.c_double), _P(_i64),
                              _P(ctypes.c_double), _int, _P(_int)], _int),
    "tqp_sort": ([_vp, Col, _i64, _int, _vp, _vp], _int),
    "tqp_pkfk_join": ([_vp, Col, _i64, Col, _i64, _vp, _vp, _P(_i64)], _int),
    "tqp_pkfk_join_i32": ([_vp, Col, _i64, Col, _i64, _vp, _vp, _P(_i64)], _int),
    "tqp_pack_keys": ([_vp, _vp, _i64, _vp, _i64, _int, _vp, _vp, _P(_int)], _int),
    "tqp_pkfk_join_paper_order": ([_vp, Col, _i64, Col, _i64, _vp, _vp, _P(_i64)], _int),
    "tqp_pkfk_semi": ([_vp, Col, _i64, Col, _i64, _int, _vp, _vp, _P(_i64)], _int),
    "tqp_pkfk_outer": ([_vp, Col, _i64, Col, _i64, _vp, _vp, _P(_i64)], _int),
    "tqp_pkfk_join_hash": ([_vp, Col, _i64, Col, _i64, _vp, _vp, _P(_i64)], _int),
    "tqp_pkfk_join_payload": ([_vp, Col, _i64, Col, _i64, _P(Col), _int, _P(_vp), _P(Col), _int, _P(_vp), _vp, _vp,
                               _P(_i64)], _int),
    "tqp_smj_prepare": ([_vp, Col, _i64, Col, _i64, _P(_vp), _P(_i64)], _int),
    "tqp_smj_expand": ([_vp, _vp, _i64, _i64, _vp, _vp], _int),
    "tqp_smj_expand_i32": ([_vp, _vp, _i64, _i64, _vp, _vp], _int),
    "tqp_smj_expand_checksum": ([_vp, _vp, _i64, _i64, _P(ctypes.c_uint64)], _int),
    "tqp_smj_release": ([_vp, _vp], None),
    "tqp_smj_expand_payload": ([_vp, _vp, _i64, _i64, _P(Col), _int, _P(_vp), _P(Col), _int, _P(_vp), _vp, _vp], _int),
    "tqp_partition": ([_vp, Col, _i64, _vp, _int, _i64, _vp, _vp, _vp], _int),
    "tqp_minmax": ([_vp, Col, _i64, _vp], _int),
    "tqp_range_splitters": ([_vp, _vp, _int, _vp], _int),
    "tqp_gather": ([_vp, Col, _vp, _i64, _vp], _int),
    "tqp_pkfk_outer_build": ([_vp, Col, _i64, Col, _i64, _vp, _vp, _P(_i64)], _int),
    "tqp_partition_plan_create": ([_vp, Col, _i64, _vp, _int, _vp, _P(_vp)], _int),
    "tqp_partition_scatter": ([_vp, _vp, _i64, _P(_vp), _P(_vp), _P(_i64)], _int),
    "tqp_partition_release": ([_vp, _vp], None),
    "tqp_ipc_alloc": ([_vp, ctypes.c_size_t, _P(_vp), _vp], _int),
    "tqp_ipc_free": ([_vp, _vp], _int),
    "tqp_ipc_open": ([_vp, _vp, _P(_vp)], _int),
    "tqp_ipc_close": ([_vp, _vp], _int),
    "tqp_smj_join": ([_vp, Col, _i64, Col, _i64, _vp, _vp, _i64, _P(_i64)], _int),
    "tqp_filter_compact": ([_vp, _P(Col), _int, _i64, _P(Pred), _int, _vp, _vp, _P(_i64)], _int),
    "tqp_groupby_prepare": ([_vp, _P(Col), _int, _i64, _P(ctypes.c_int32), _int, _P(Pred), _int, _P(Agg), _int,
                             _P(_vp), _P(_i64)], _int),
    "tqp_groupby_fetch": ([_vp, _vp, _P(_vp), _P(_vp)], _int),
    "tqp_groupby_release": ([_vp, _vp], None),
    "tqp_groupby_agg": ([_vp, _P(Col), _int, _i64, _P(ctypes.c_int32), _int, _P(Pred), _int, _P(Agg), _int,
                         _P(_vp), _P(_vp), _i64, _P(_i64)], _int),
    "tqp_groupby_merge": ([_vp, _i64, _P(Col), _int, _P(Agg), _int, _P(_vp), _vp, _P(_vp), _P(_i64)], _int),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res


class TqpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libtqp status {status}: {msg}")
        self.status = status


def lib_path():
    return _LIB_PATH


def abi_version():
    return _lib.tqp_abi_version()


def jit_counters():
    """Plan-compiled dense group-by kernels (process-wide): {"available", "compiled",
    "failed", "launches"} -- include/tqp.h tqp_jit_counters."""
    c, f, l = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    ok = _lib.tqp_jit_counters(ctypes.byref(c), ctypes.byref(f), ctypes.byref(l))
    return {"available": bool(ok), "compiled": c.value, "failed": f.value, "launches": l.value}


_DT = {torch.uint8: TQP_U8, torch.bool: TQP_U8, torch.int32: TQP_I32, torch.int64: TQP_I64,
       torch.float64: TQP_F64}   # float64: group-by aggregate factor columns only


def _dev_tensor(t, device):
    """Marshal an input column: CUDA tensors pass through; host tensors are staged to the device."""
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    if t.dtype not in _DT:
        raise TypeError(f"unsupported column dtype {t.dtype}")
    if t.dim() != 1:
        t = t.reshape(-1)
    if t.device.type != "cuda":
        src = t if t.is_pinned() else t.contiguous()
        t = src.to(device, non_blocking=src.is_pinned())
    elif t.device != device:
        t = t.to(device)
    return t.contiguous()


def _col(t):
    return Col(t.data_ptr() if t.numel() else 0, _DT[t.dtype], 0)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() else None)


# libtqp's temporaries from torch's caching allocator (include/tqp.h tqp_ctx_set_allocator):
# one pool of HBM for both; called only when libtqp's own cache misses, and at trim/destroy
_ALLOC_T = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p)
_FREE_T = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)


@_ALLOC_T
def _torch_alloc(user, nbytes, device, stream):
    try:
        return torch.cuda.caching_allocator_alloc(int(nbytes), device, int(stream or 0))
    except Exception:   # out of memory: libtqp returns its cache and retries once, then reports it
        return None


@_FREE_T
def _torch_free(user, ptr, device, stream):
    try:
        torch.cuda.caching_allocator_delete(ptr)
    except Exception:
        pass


class Context:
    """A libtqp context bound to one CUDA device; work goes on torch's current stream.
    allocator="torch" (default): libtqp's temporaries come from torch's caching allocator
    (one HBM pool; ctx.trim() hands libtqp's cached blocks back to it); "cuda": cudaMalloc."""

    def __init__(self, device=None, allocator="torch"):
        if not torch.cuda.is_available():
            raise RuntimeError("libtqp needs a CUDA device (B200); no CPU fallback exists")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            s = torch.cuda.current_stream(self.device).cuda_stream
            self._check(_lib.tqp_ctx_create(self.device.index, ctypes.c_void_p(s), ctypes.byref(h)), None)
        self._h = h
        self._stream = s
        if allocator == "torch":
            self._check(_lib.tqp_ctx_set_allocator(self._h, ctypes.cast(_torch_alloc, ctypes.c_void_p),
                                                   ctypes.cast(_torch_free, ctypes.c_void_p), None))
        elif allocator != "cuda":
            raise ValueError("allocator must be 'torch' or 'cuda'")
        self.allocator = allocator

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and not sys.is_finalizing():   # at exit the process frees it all
            try:
                _lib.tqp_ctx_destroy(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------ plumbing
    def _check(self, st, h=-1):
        if st != TQP_OK:
            hh = self._h if h == -1 else h
            msg = _lib.tqp_last_error(hh).decode() if hh else "context creation failed"
            raise TqpError(st, msg)

    def _sync_stream(self):
        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            self._check(_lib.tqp_ctx_set_stream(self._h, ctypes.c_void_p(s)))
            self._stream = s

    def launch_count(self):
        return _lib.tqp_ctx_launch_count(self._h)

    def trim(self):
        """Return libtqp's cached temporary blocks to the allocator (synchronises)."""
        self._check(_lib.tqp_ctx_trim(self._h))

    def cached_bytes(self):
        return _lib.tqp_ctx_cached_bytes(self._h)

    def guard_violations(self):
        """Overwritten canaries after temporaries (checked mode, TQP_ALLOC_EXACT=1)."""
        return _lib.tqp_ctx_guard_violations(self._h)

    def reset_counters(self):
        _lib.tqp_ctx_reset_counters(self._h)

    def set_profiling(self, on=True, only=None):
        """Per-launch device timing; `only`: a kernel-name prefix to restrict it to."""
        self._check(_lib.tqp_ctx_set_profiling_filter(self._h, only.encode() if only else None))
        self._check(_lib.tqp_ctx_set_profiling(self._h, int(bool(on))))

    def kernel_stats(self):
        """{kernel name: (profiled device ms, profiled launches, algorithmic bytes)} since the
        last reset (synchronises)."""
        cap = 64
        names = ctypes.create_string_buffer(8192)
        ms = (ctypes.c_double * cap)()
        ln = (ctypes.c_int64 * cap)()
        by = (ctypes.c_double * cap)()
        k = ctypes.c_int(0)
        self._check(_lib.tqp_ctx_kernel_stats(self._h, names, 8192, ms, ln, by, cap, ctypes.byref(k)))
        nm = names.value.decode().split("\n")
        return {nm[i]: (ms[i], ln[i], by[i]) for i in range(k.value)}

    # ----------------------------------------------------------- operators
    def sort(self, keys, descending=False, return_keys=True):
        """Stable sort -> (sorted_keys | None, perm int64). PAPER.md:296-297, :352."""
        self._sync_stream()
        k = _dev_tensor(keys, self.device)
        n = k.numel()
        perm = torch.empty(n, dtype=torch.int64, device=self.device)
        out = torch.empty_like(k) if return_keys else None
        self._check(_lib.tqp_sort(self._h, _col(k), n, int(bool(descending)), _ptr(out), _ptr(perm)))
        return out, perm

    def pkfk_join(self, build_keys, probe_keys, index_dtype=torch.int64):
        """PK-FK join -> (left_idx, right_idx), ascending probe row. PAPER.md:55-100.
        index_dtype=torch.int32 selects tqp_pkfk_join_i32 (both sides < 2^31 rows)."""
        self._sync_stream()
        b = _dev_tensor(build_keys, self.device)
        p = _dev_tensor(probe_keys, self.device)
        if index_dtype not in (torch.int64, torch.int32):
            raise ValueError("index_dtype must be torch.int64 or torch.int32")
        lo = torch.empty(p.numel(), dtype=index_dtype, device=self.device)
        ro = torch.empty(p.numel(), dtype=index_dtype, device=self.device)
        m = ctypes.c_int64(0)
        fn = _lib.tqp_pkfk_join if index_dtype == torch.int64 else _lib.tqp_pkfk_join_i32
        self._check(fn(self._h, _col(b), b.numel(), _col(p), p.numel(), _ptr(lo), _ptr(ro), ctypes.byref(m)))
        return lo[:m.value], ro[:m.value]

    def pack_keys(self, a_cols, b_cols=None):
        """Composite keys (lists of columns, column 0 most significant) of one or two
        relations packed into int64 keys with a shared layout; returns
        (a_packed, b_packed or None, total_bits)."""
        self._sync_stream()
        a = [_dev_tensor(c, self.device) for c in a_cols]
        b = [_dev_tensor(c, self.device) for c in b_cols] if b_cols is not None else []
        if not a or (b and len(b) != len(a)):
            raise ValueError("pack_keys: one or two lists of the same number of key columns")
        na, nb = a[0].numel(), (b[0].numel() if b else 0)
        if any(c.numel() != na for c in a) or any(c.numel() != nb for c in b):
            raise ValueError("pack_keys: columns of one side must have equal length")
        ca = (Col * len(a))(*[_col(c) for c in a])
        cb = (Col * len(b))(*[_col(c) for c in b]) if b else None
        oa = torch.empty(na, dtype=torch.int64, device=self.device)
        ob = torch.empty(nb, dtype=torch.int64, device=self.device) if b else None
        bits = ctypes.c_int(0)
        self._check(_lib.tqp_pack_keys(self._h, ca, na, cb, nb, len(a), _ptr(oa), _ptr(ob), ctypes.byref(bits)))
        return oa, ob, bits.value

    def pkfk_join_paper_order(self, build_keys, probe_keys):
        """PK-FK join pairs in the paper's order: probe key descending, then probe row
        (reading R7)."""
        self._sync_stream()
        b = _dev_tensor(build_keys, self.device)
        p = _dev_tensor(probe_keys, self.device)
        lo = torch.empty(p.numel(), dtype=torch.int64, device=self.device)
        ro = torch.empty(p.numel(), dtype=torch.int64, device=self.device)
        m = ctypes.c_int64(0)
        self._check(_lib.tqp_pkfk_join_paper_order(self._h, _col(b), b.numel(), _col(p), p.numel(), _ptr(lo), _ptr(ro),
                                                   ctypes.byref(m)))
        return lo[:m.value], ro[:m.value]

    def pkfk_semi(self, build_keys, probe_keys, anti=False, return_mask=False):
        """Left-semi (anti=False) / left-anti selection of probe rows."""
        self._sync_stream()
        b = _dev_tensor(build_keys, self.device)
        p = _dev_tensor(probe_keys, self.device)
        sel = torch.empty(p.numel(), dtype=torch.int64, device=self.device)
        mask = torch.empty(p.numel(), dtype=torch.uint8, device=self.device) if return_mask else None
        m = ctypes.c_int64(0)
        self._check(_lib.tqp_pkfk_semi(self._h, _col(b), b.numel(), _col(p), p.numel(), int(bool(anti)),
                                       _ptr(mask), _ptr(sel), ctypes.byref(m)))
        return (sel[:m.value], mask) if return_mask else sel[:m.value]

    def pkfk_join_payload(self, build_keys, probe_keys, build_payload=(), probe_payload=(), indices=True):
        """PK-FK join with payload columns gathered into the output (GenerateOutput fused).
        Returns (build payload outputs, probe payload outputs, (left, right) or None)."""
        self._sync_stream()
        b = _dev_tensor(build_keys, self.device)
        p = _dev_tensor(probe_keys, self.device)
        bps = [_dev_tensor(c, self.device) for c in build_payload]
        pps = [_dev_tensor(c, self.device) for c in probe_payload]
        np_ = p.numel()
        bouts = [torch.empty(np_, dtype=c.dtype, device=self.device) for c in bps]
        pouts = [torch.empty(np_, dtype=c.dtype, device=self.device) for c in pps]
        lo = torch.empty(np_, dtype=torch.int64, device=self.device) if indices else None
        ro = torch.empty(np_, dtype=torch.int64, device=self.device) if indices else None
        ba = (Col * max(len(bps), 1))(*[_col(c) for c in bps])
        pa = (Col * max(len(pps), 1))(*[_col(c) for c in pps])
        bo = (_vp * max(len(bouts), 1))(*[t.data_ptr() for t in bouts])
        po = (_vp * max(len(pouts), 1))(*[t.data_ptr() for t in pouts])
        m = ctypes.c_int64(0)
        self._check(_lib.tqp_pkfk_join_payload(self._h, _col(b), b.numel(), _col(p), np_, ba, len(bps), bo, pa,
                                               len(pps), po, _ptr(lo), _ptr(ro), ctypes.byref(m)))
        n = m.value
        return ([t[:n] for t in bouts], [t[:n] for t in pouts], (lo[:n], ro[:n]) if indices else None)

    def pkfk_join_hash(self, build_keys, probe_keys):
        """Hash-join ablation of pkfk_join (same output; not the paper's method)."""
        self._sync_stream()
        b = _dev_tensor(build_keys, self.device)
        p = _dev_tensor(probe_keys, self.device)
        lo = torch.empty(p.numel(), dtype=torch.int64, device=self.device)
        ro = torch.empty(p.numel(), dtype=torch.int64, device=self.device)
        m = ctypes.c_int64(0)
        self._check(_lib.tqp_pkfk_join_hash(self._h, _col(b), b.numel(), _col(p), p.numel(), _ptr(lo), _ptr(ro),
                                            ctypes.byref(m)))
        return lo[:m.value], ro[:m.value]

    def pkfk_outer(self, build_keys, probe_keys, return_mask=False):
        """Probe-side outer join: build row per probe row (-1 = no match), probe rows in order."""
        self._sync_stream()
        b = _dev_tensor(build_keys, self.device)
        p = _dev_tensor(probe_keys, self.device)
        left = torch.empty(p.numel(), dtype=torch.int64, device=self.device)
        mask = torch.empty(p.numel(), dtype=torch.uint8, device=self.device) if return_mask else None
        m = ctypes.c_int64(0)
        self._check(_lib.tqp_pkfk_outer(self._h, _col(b), b.numel(), _col(p), p.numel(), _ptr(left), _ptr(mask),
                                        ctypes.byref(m)))
        return (left, mask) if return_mask else left

    def pkfk_outer_build(self, build_keys, probe_keys):
        """Outer join preserving the build side (Q13's customer LEFT OUTER JOIN orders):
        the inner pairs (ascending probe row), then (b, -1) for each unmatched build row."""
        self._sync_stream()
        b = _dev_tensor(build_keys, self.device)
        p = _dev_tensor(probe_keys, self.device)
        cap = b.numel() + p.numel()
        lo = torch.empty(cap, dtype=torch.int64, device=self.device)
        ro = torch.empty(cap, dtype=torch.int64, device=self.device)
        m = ctypes.c_int64(0)
        self._check(_lib.tqp_pkfk_outer_build(self._h, _col(b), b.numel(), _col(p), p.numel(), _ptr(lo), _ptr(ro),
                                              ctypes.byref(m)))
        return lo[:m.value], ro[:m.value]

    def smj_prepare(self, left, right):
        """Alg. 1 lines 1-9: sort, histograms, products, prefix sums -> SmjPlan (size known)."""
        self._sync_stream()
        l = _dev_tensor(left, self.device)
        r = _dev_tensor(right, self.device)
        plan = ctypes.c_void_p()
        size = ctypes.c_int64(0)
        self._check(_lib.tqp_smj_prepare(self._h, _col(l), l.numel(), _col(r), r.numel(), ctypes.byref(plan),
                                         ctypes.byref(size)))
        return SmjPlan(self, plan, size.value)

    def smj_join(self, left, right):
        """Generic m:n sort-merge join -> (left_idx, right_idx) in (key, l, r) order. PAPER.md:286-338."""
        plan = self.smj_prepare(left, right)
        try:
            return plan.expand(0, plan.size)
        finally:
            plan.release()

    def smj_join_payload(self, left, right, left_payload=(), right_payload=(), indices=False):
        """Alg. 1 with createOutput fused: the pairs' payload columns gathered
        in (key, l, r) order -> (left payload outputs, right payload outputs, (l, r) or None)."""
        plan = self.smj_prepare(left, right)
        try:
            return plan.expand_payload(0, plan.size, left_payload, right_payload, indices)
        finally:
            plan.release()

    # ------------------------------------------------ data-parallel exchange steps
    def partition(self, keys, splitters, row_base=0, rows=True):
        """Stable partition by key range (tqp_partition): dest = #splitters <= key. Returns
        (keys grouped by destination, their row_base + input row (int64) or None, device
        int64 counts per destination). No host sync."""
        self._sync_stream()
        k = _dev_tensor(keys, self.device)
        spl = _dev_tensor(torch.as_tensor(splitters, dtype=torch.int64) if not isinstance(splitters, torch.Tensor)
                          else splitters.to(torch.int64), self.device)
        parts = spl.numel() + 1
        ko = torch.empty_like(k)
        ro = torch.empty(k.numel(), dtype=torch.int64, device=self.device) if rows else None
        counts = torch.empty(parts, dtype=torch.int64, device=self.device)
        self._check(_lib.tqp_partition(self._h, _col(k), k.numel(), _ptr(spl), parts, int(row_base), _ptr(ko), _ptr(ro),
                                       _ptr(counts)))
        return ko, ro, counts

    def partition_plan(self, keys, splitters):
        """Fused-exchange partition, step 1 (tqp_partition_plan_create): -> (PartitionPlan,
        device int64 counts per destination). Keep `keys` and `splitters` alive."""
        self._sync_stream()
        k = _dev_tensor(keys, self.device)
        spl = _dev_tensor(splitters, self.device).to(torch.int64).contiguous()
        parts = spl.numel() + 1
        counts = torch.empty(parts, dtype=torch.int64, device=self.device)
        h = ctypes.c_void_p()
        self._check(_lib.tqp_partition_plan_create(self._h, _col(k), k.numel(), _ptr(spl), parts, _ptr(counts),
                                                   ctypes.byref(h)))
        return PartitionPlan(self, h, parts, (k, spl)), counts

    def ipc_alloc(self, nbytes):
        """A cudaMalloc'd buffer shareable with other processes -> (device pointer, 64-byte handle)."""
        p = ctypes.c_void_p()
        hb = ctypes.create_string_buffer(64)
        self._check(_lib.tqp_ipc_alloc(self._h, int(nbytes), ctypes.byref(p), hb))
        return p.value, hb.raw

    def ipc_free(self, ptr):
        self._check(_lib.tqp_ipc_free(self._h, ctypes.c_void_p(ptr)))

    def ipc_open(self, handle):
        """Map another process's buffer (64-byte handle) -> device pointer."""
        p = ctypes.c_void_p()
        self._check(_lib.tqp_ipc_open(self._h, ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(p)))
        return p.value

    def ipc_close(self, ptr):
        self._check(_lib.tqp_ipc_close(self._h, ctypes.c_void_p(ptr)))

    def minmax(self, keys):
        """Device int64 [min, max] of a key column ([INT64_MAX, INT64_MIN] when empty). No host sync."""
        self._sync_stream()
        k = _dev_tensor(keys, self.device)
        out = torch.empty(2, dtype=torch.int64, device=self.device)
        self._check(_lib.tqp_minmax(self._h, _col(k), k.numel(), _ptr(out)))
        return out

    def range_splitters(self, lohi, parts):
        """parts - 1 equal-width splitters over a device [lo, hi] (tqp_range_splitters)."""
        self._sync_stream()
        lh = _dev_tensor(lohi, self.device).to(torch.int64).contiguous()
        out = torch.empty(max(parts - 1, 0), dtype=torch.int64, device=self.device)
        self._check(_lib.tqp_range_splitters(self._h, _ptr(lh), int(parts), _ptr(out)))
        return out

    def gather(self, src, idx):
        """out[i] = src[idx[i]] (tqp_gather; idx int64 on the device)."""
        self._sync_stream()
        s = _dev_tensor(src, self.device)
        i = _dev_tensor(idx, self.device)
        if i.dtype != torch.int64:
            raise TypeError("gather: idx must be int64")
        out = torch.empty(i.numel(), dtype=s.dtype, device=self.device)
        self._check(_lib.tqp_gather(self._h, _col(s), _ptr(i), i.numel(), _ptr(out)))
        return out

    def filter_compact(self, cols, preds, mask=True, sel=True):
        """Listing 1 bitmap and/or Listing 2 selection vector -> (mask u8 | None, sel int64 | None)."""
        self._sync_stream()
        cs = [_dev_tensor(c, self.device) for c in cols]
        n = cs[0].numel() if cs else 0
        ca = (Col * max(len(cs), 1))(*[_col(c) for c in cs])
        pa = _preds(preds)
        mk = torch.empty(n, dtype=torch.uint8, device=self.device) if mask else None
        sv = torch.empty(n, dtype=torch.int64, device=self.device) if sel else None
        m = ctypes.c_int64(0)
        self._check(_lib.tqp_filter_compact(self._h, ca, len(cs), n, pa, len(preds), _ptr(mk), _ptr(sv),
                                            ctypes.byref(m)))
        return mk, (sv[:m.value] if sv is not None else None)

    def groupby_agg(self, cols, key_idx, aggs, preds=()):
        """Sort-based group-by (Alg. 2) with fused pre-filter.

        aggs: [(op, [(col, add, sign), ...])]. Returns dict(n_groups, keys=[tensor per key col],
        results=[SUM: int64 (G,2) = (lo, hi) of the int128 | COUNT/MIN/MAX: int64 | AVG: float64]);
        an aggregate with a float64 factor column is evaluated in fp64 and returns float64 (G,)."""
        self._sync_stream()
        cs = [_dev_tensor(c, self.device) for c in cols]
        n = cs[0].numel() if cs else 0
        ca = (Col * max(len(cs), 1))(*[_col(c) for c in cs])
        ki = (ctypes.c_int32 * max(len(key_idx), 1))(*key_idx)
        pa = _preds(preds)
        aa = _aggs(aggs)
        plan = ctypes.c_void_p()
        G = ctypes.c_int64(0)
        self._check(_lib.tqp_groupby_prepare(self._h, ca, len(cs), n, ki, len(key_idx), pa, len(preds), aa,
                                             len(aggs), ctypes.byref(plan), ctypes.byref(G)))
        try:
            g = G.value
            keys = [torch.empty(g, dtype=cs[k].dtype if cs[k].dtype != torch.bool else torch.uint8,
                                device=self.device) for k in key_idx]
            res = []
            for op, factors in aggs:
                o = AGGS[op] if isinstance(op, str) else int(op)
                if o != 1 and any(cs[c].dtype == torch.float64 for c, _, _ in factors):
                    res.append(torch.empty(g, dtype=torch.float64, device=self.device))
                elif o == 0:
                    res.append(torch.empty((g, 2), dtype=torch.int64, device=self.device))
                elif o == 4:
                    res.append(torch.empty(g, dtype=torch.float64, device=self.device))
                else:
                    res.append(torch.empty(g, dtype=torch.int64, device=self.device))
            kp = (ctypes.c_void_p * max(len(keys), 1))(*[t.data_ptr() if g else None for t in keys])
            rp = (ctypes.c_void_p * max(len(res), 1))(*[t.data_ptr() if g else None for t in res])
            self._check(_lib.tqp_groupby_fetch(self._h, plan, kp, rp))
        finally:
            _lib.tqp_groupby_release(self._h, plan)
        return {"n_groups": g, "keys": keys, "results": res}

    def _fetch(self, plan, G, key_dtypes, aggs):
        try:
            g = G
            keys = [torch.empty(g, dtype=dt, device=self.device) for dt in key_dtypes]
            res = []
            for op, _ in aggs:
                o = AGGS[op] if isinstance(op, str) else int(op)
                shape, dt = ((g, 2), torch.int64) if o == 0 else ((g,), torch.float64 if o == 4 else torch.int64)
                res.append(torch.empty(shape, dtype=dt, device=self.device))
            kp = (ctypes.c_void_p * max(len(keys), 1))(*[t.data_ptr() if g else None for t in keys])
            rp = (ctypes.c_void_p * max(len(res), 1))(*[t.data_ptr() if g else None for t in res])
            self._check(_lib.tqp_groupby_fetch(self._h, plan, kp, rp))
        finally:
            _lib.tqp_groupby_release(self._h, plan)
        return {"n_groups": g, "keys": keys, "results": res}

    def groupby_merge(self, key_cols, aggs, partials, counts):
        """Merge partial group-by rows (tqp_groupby_merge): key_cols = [tensor per key], partials[a] =
        int128 (m,2) SUM of aggregate a's expression (SUM/AVG) or int64 (MIN/MAX) or None (COUNT),
        counts = COUNT(*) per partial row. Returns the same dict as groupby_agg."""
        self._sync_stream()
        ks = [_dev_tensor(k, self.device) for k in key_cols]
        cnt = _dev_tensor(counts, self.device)
        m = cnt.numel()
        ca = (Col * max(len(ks), 1))(*[_col(k) for k in ks])
        aa = _aggs(aggs)
        ps = [None if p is None else p.to(self.device).contiguous() for p in partials]
        pp = (ctypes.c_void_p * max(len(ps), 1))(*[p.data_ptr() if p is not None and p.numel() else None
                                                     for p in ps])
        plan = ctypes.c_void_p()
        G = ctypes.c_int64(0)
        self._check(_lib.tqp_groupby_merge(self._h, m, ca, len(ks), aa, len(aggs), pp, _ptr(cnt),
                                           ctypes.byref(plan), ctypes.byref(G)))
        return self._fetch(plan, G.value, [k.dtype for k in ks], aggs)


class PartitionPlan:
    """Step 2 of the fused exchange: scatter(row_base, key_ptrs, row_ptrs, bases) writes
    destination d's rows at key_ptrs[d] + bases[d] (and row_ptrs[d] + bases[d]); the
    pointers may be peers' receive buffers (Context.ipc_open)."""

    def __init__(self, ctx, handle, parts, keep):
        self.ctx, self._h, self.parts, self._keep = ctx, handle, parts, keep

    def scatter(self, row_base, key_ptrs, row_ptrs, bases):
        c = self.ctx
        c._sync_stream()
        n = self.parts
        kp = (_vp * n)(*key_ptrs)
        rp = (_vp * n)(*row_ptrs) if row_ptrs is not None else None
        bp = (ctypes.c_int64 * n)(*bases)
        c._check(_lib.tqp_partition_scatter(c._h, self._h, int(row_base), kp, rp, bp))

    def release(self):
        if self._h:
            _lib.tqp_partition_release(self.ctx._h, self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def device_view(ptr, n, dtype, device):
    """A torch tensor over n elements of raw device memory at ptr (no copy, not owning)."""
    typestr = {torch.int64: "<i8", torch.int32: "<i4", torch.uint8: "|u1", torch.float64: "<f8"}[dtype]

    class _A:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr) if n else 0, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_A(), device=device) if n else torch.empty(0, dtype=dtype, device=device)


class SmjPlan:
    """Device-resident Alg. 1 state after line 9 (outSize known); expand() runs lines 10-14 on windows."""

    def __init__(self, ctx, handle, size):
        self.ctx, self._h, self.size = ctx, handle, size

    def expand(self, begin, end, out=None, index_dtype=torch.int64):
        """Pairs [begin, end) as (left_idx, right_idx); int32 outputs (index_dtype or
        the dtype of `out`) select tqp_smj_expand_i32."""
        self.ctx._sync_stream()
        k = end - begin
        if out is None:
            lo = torch.empty(k, dtype=index_dtype, device=self.ctx.device)
            ro = torch.empty(k, dtype=index_dtype, device=self.ctx.device)
        else:
            lo, ro = out
        if lo.dtype != ro.dtype or lo.dtype not in (torch.int64, torch.int32) or lo.numel() < k or ro.numel() < k:
            raise ValueError("expand: outputs must be two int64 or two int32 tensors of >= end-begin elements")
        fn = _lib.tqp_smj_expand if lo.dtype == torch.int64 else _lib.tqp_smj_expand_i32
        self.ctx._check(fn(self.ctx._h, self._h, begin, end, _ptr(lo), _ptr(ro)))
        return lo, ro

    def expand_payload(self, begin, end, left_payload=(), right_payload=(), indices=False):
        """Payload columns gathered by the pairs of [begin, end) (tqp_smj_expand_payload) ->
        (left outputs, right outputs, (l, r) or None)."""
        c = self.ctx
        c._sync_stream()
        lps = [_dev_tensor(t, c.device) for t in left_payload]
        rps = [_dev_tensor(t, c.device) for t in right_payload]
        m = end - begin
        louts = [torch.empty(m, dtype=t.dtype, device=c.device) for t in lps]
        routs = [torch.empty(m, dtype=t.dtype, device=c.device) for t in rps]
        lo = torch.empty(m, dtype=torch.int64, device=c.device) if indices else None
        ro = torch.empty(m, dtype=torch.int64, device=c.device) if indices else None
        la = (Col * max(len(lps), 1))(*[_col(t) for t in lps])
        ra = (Col * max(len(rps), 1))(*[_col(t) for t in rps])
        lo_p = (_vp * max(len(louts), 1))(*[t.data_ptr() for t in louts])
        ro_p = (_vp * max(len(routs), 1))(*[t.data_ptr() for t in routs])
        c._check(_lib.tqp_smj_expand_payload(c._h, self._h, begin, end, la, len(lps), lo_p, ra, len(rps), ro_p,
                                             _ptr(lo), _ptr(ro)))
        return louts, routs, ((lo, ro) if indices else None)

    def checksum(self, begin, end):
        """Fused consumer over pairs [begin, end) without materialising them:
        (sum_j mix64(mix64((l_j << 32) | r_j) ^ j), sum_j l_j, sum_j r_j), all mod 2^64."""
        self.ctx._sync_stream()
        out = (ctypes.c_uint64 * 3)()
        self.ctx._check(_lib.tqp_smj_expand_checksum(self.ctx._h, self._h, begin, end, out))
        return tuple(int(x) for x in out)

    def release(self):
        if self._h:
            _lib.tqp_smj_release(self.ctx._h, self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def _preds(preds):
    if len(preds) > MAX_PREDS:
        raise ValueError("too many predicates")
    arr = (Pred * max(len(preds), 1))()
    for i, (c, op, v) in enumerate(preds):
        arr[i].col, arr[i].op, arr[i].value = c, OPS[op] if isinstance(op, str) else int(op), int(v)
    return arr


def _aggs(aggs):
    if len(aggs) > MAX_AGGS:
        raise ValueError("too many aggregates")
    arr = (Agg * max(len(aggs), 1))()
    for i, (op, factors) in enumerate(aggs):
        arr[i].op = AGGS[op] if isinstance(op, str) else int(op)
        arr[i].n_factors = len(factors)
        for f, (c, add, sign) in enumerate(factors):
            arr[i].col[f], arr[i].add[f], arr[i].sign[f] = c, int(add), int(sign)
    return arr


def int128_to_ints(t):
    """(G, 2) int64 [lo, hi] tensor -> list of exact Python ints."""
    t = t.cpu()
    return [(int(lo) & ((1 << 64) - 1)) + (int(hi) << 64) for lo, hi in t.tolist()]


_default = {}


def context(device=None):
    """Process-wide default Context per device."""
    d = torch.cuda.current_device() if device is None else torch.device(device).index or 0
    if d not in _default:
        _default[d] = Context(d)
    return _default[d]


def sort(keys, descending=False, return_keys=True):
    return context().sort(keys, descending, return_keys)


def pkfk_join(build_keys, probe_keys, index_dtype=torch.int64):
    return context().pkfk_join(build_keys, probe_keys, index_dtype)


def pack_keys(a_cols, b_cols=None):
    return context().pack_keys(a_cols, b_cols)


def pkfk_join_paper_order(build_keys, probe_keys):
    return context().pkfk_join_paper_order(build_keys, probe_keys)


def pkfk_semi(build_keys, probe_keys, anti=False, return_mask=False):
    return context().pkfk_semi(build_keys, probe_keys, anti, return_mask)


def smj_prepare(left, right):
    return context().smj_prepare(left, right)


def smj_join(left, right):
    return context().smj_join(left, right)


def pkfk_join_payload(build_keys, probe_keys, build_payload=(), probe_payload=(), indices=True):
    return context().pkfk_join_payload(build_keys, probe_keys, build_payload, probe_payload, indices)


def pkfk_join_hash(build_keys, probe_keys):
    return context().pkfk_join_hash(build_keys, probe_keys)


def pkfk_outer(build_keys, probe_keys, return_mask=False):
    return context().pkfk_outer(build_keys, probe_keys, return_mask)


def smj_join_payload(left, right, left_payload=(), right_payload=(), indices=False):
    return context().smj_join_payload(left, right, left_payload, right_payload, indices)


def pkfk_outer_build(build_keys, probe_keys):
    return context().pkfk_outer_build(build_keys, probe_keys)


def partition(keys, splitters, row_base=0, rows=True):
    return context().partition(keys, splitters, row_base, rows)


def minmax(keys):
    return context().minmax(keys)


def range_splitters(lohi, parts):
    return context().range_splitters(lohi, parts)


def gather(src, idx):
    return context().gather(src, idx)


def filter_compact(cols, preds, mask=True, sel=True):
    return context().filter_compact(cols, preds, mask, sel)


def groupby_agg(cols, key_idx, aggs, preds=()):
    return context().groupby_agg(cols, key_idx, aggs, preds)
