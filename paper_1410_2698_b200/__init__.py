"""tds-b200: distance threshold search over 4-D trajectory segments on B200.

Thin ctypes binding of the C-ABI in ``include/tds.h`` (argument marshalling
only — every step of the search runs in the CUDA kernels of ``libtds.so``).
Paper: Gowanlock & Casanova, arXiv 1410.2698; see DESIGN.md.

    import torch, paper_1410_2698_b200 as tds
    idx = tds.Index(entries_cuda_f32_n_by_8, kinds=tds.ALL, m=1000, v=2, grid=(50, 50, 50))
    res = idx.search(queries, d=0.03, kind="spatiotemporal")
    qid, eid, t_in, t_out = res.fetch(sorted=True)

There is no CPU fallback: if ``libtds.so`` is missing or cannot be loaded the
import fails loudly.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TDS_LIB", os.path.join(_HERE, "libtds.so"))

TEMPORAL, SPATIAL, SPATIOTEMPORAL, ALL, AUTO = 1, 2, 4, 7, 8
KINDS = {"temporal": TEMPORAL, "spatial": SPATIAL, "spatiotemporal": SPATIOTEMPORAL, "auto": AUTO}
STATUS = {0: "TDS_OK", 1: "TDS_EINVAL", 2: "TDS_EDATA", 3: "TDS_ENOMEM", 4: "TDS_ECAPACITY", 5: "TDS_ECUDA"}

EXPORT = {"perm": 0, "bin_off": 1, "bin_hi": 2, "st_x": 3, "st_y": 4, "st_z": 5, "st_off_x": 6,
          "st_off_y": 7, "st_off_z": 8, "fsg_cell_off": 9, "fsg_A": 10, "extents": 11, "sorted_t0": 12,
          "wb_rec": 13, "wb_x": 14, "wb_y": 15, "wb_z": 16, "wb_fsg": 17}
_EXPORT_DT = {"bin_hi": np.float32, "extents": np.float32, "sorted_t0": np.float32, "wb_rec": np.float32,
              "wb_x": np.float32, "wb_y": np.float32, "wb_z": np.float32, "wb_fsg": np.float32}

# every symbol include/tds.h declares
ABI_SYMBOLS = ["tds_build_index", "tds_search", "tds_fetch_results", "tds_result_stats", "tds_result_count",
               "tds_result_free", "tds_index_free", "tds_last_error", "tds_index_export", "tds_index_info",
               "tds_version", "tds_kernel_launches", "tds_merge_trajectories", "tds_search_many",
               "tds_search_part", "tds_plan", "tds_time_partition", "tds_trim", "tds_test_inject_enomem",
               "tds_search_stream", "tds_result_host_block"]


class TdsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class _SearchReq(ctypes.Structure):
    """tds_search_req (include/tds.h)."""
    _fields_ = [("kind", ctypes.c_int), ("queries", ctypes.c_void_p), ("nq", ctypes.c_uint64),
                ("d", ctypes.c_double), ("t_start", ctypes.c_float), ("t_end", ctypes.c_float),
                ("capacity", ctypes.c_uint64), ("stream", ctypes.c_void_p)]


class _Params(ctypes.Structure):
    _fields_ = [("kinds", ctypes.c_uint32), ("m_bins", ctypes.c_int32), ("v_subbins", ctypes.c_int32),
                ("grid", ctypes.c_int32 * 3), ("flags", ctypes.c_uint32)]


TIME_ORDER = 1      # tds_index_params.flags: renumber D by t_start (the paper) instead of (bin, Morton)


class _Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("n_results", "n_queries", "pair_tests", "pairs_executed",
                                               "refined_pairs", "passes", "spilled", "fallback_queries")] + \
               [(k, ctypes.c_float) for k in ("ms_schedule", "ms_pairs", "ms_compact", "ms_total")] + \
               [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32), ("pair_tests_alt", ctypes.c_uint64),
                ("capacity", ctypes.c_uint64), ("refined32", ctypes.c_uint64), ("direct_records", ctypes.c_uint64)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libtds.so (raises if missing: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libtds.so not found at {path}: run `python -m paper_1410_2698_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    vp, u64, i32, f32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_float
    lib.tds_build_index.argtypes = [vp, u64, ctypes.POINTER(_Params), vp, ctypes.POINTER(vp)]
    lib.tds_search.argtypes = [vp, i32, vp, u64, ctypes.c_double, f32, f32, u64, vp, ctypes.POINTER(vp),
                               ctypes.POINTER(u64)]
    lib.tds_search_part.argtypes = [vp, i32, vp, u64, ctypes.c_double, f32, f32, u64, ctypes.c_uint32,
                                    ctypes.c_uint32, vp, ctypes.POINTER(vp), ctypes.POINTER(u64)]
    lib.tds_search_stream.argtypes = [vp, i32, vp, u64, ctypes.c_double, f32, f32, u64, ctypes.c_uint32,
                                      ctypes.c_uint32, vp, ctypes.POINTER(vp), ctypes.POINTER(u64)]
    lib.tds_result_host_block.argtypes = [vp, u64, ctypes.POINTER(vp), ctypes.POINTER(u64)]
    lib.tds_time_partition.argtypes = [vp, u64, ctypes.c_uint32, ctypes.c_uint32, vp, vp, ctypes.POINTER(u64)]
    lib.tds_plan.argtypes = [vp, i32, vp, u64, ctypes.c_double, f32, f32, vp, vp, vp, vp]
    lib.tds_fetch_results.argtypes = [vp, u64, u64, vp, vp, vp, vp, i32, i32, vp]
    lib.tds_merge_trajectories.argtypes = [vp, vp, u64, vp, u64, f32, vp, ctypes.POINTER(vp), ctypes.POINTER(u64)]
    lib.tds_result_stats.argtypes = [vp, ctypes.POINTER(_Stats)]
    lib.tds_result_count.argtypes = [vp]
    lib.tds_result_count.restype = u64
    lib.tds_result_free.argtypes = [vp]
    lib.tds_result_free.restype = None
    lib.tds_index_free.argtypes = [vp]
    lib.tds_index_free.restype = None
    lib.tds_last_error.restype = ctypes.c_char_p
    lib.tds_version.restype = ctypes.c_char_p
    lib.tds_kernel_launches.restype = ctypes.c_uint64
    lib.tds_trim.restype = None
    lib.tds_test_inject_enomem.argtypes = [i32, i32]
    lib.tds_test_inject_enomem.restype = ctypes.c_uint64
    lib.tds_index_export.argtypes = [vp, i32, vp, u64, ctypes.POINTER(u64)]
    lib.tds_search_many.argtypes = [vp, i32, ctypes.POINTER(_SearchReq), ctypes.POINTER(vp), ctypes.POINTER(u64)]
    lib.tds_index_info.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(ctypes.c_uint32)]
    for name in ("tds_build_index", "tds_search", "tds_fetch_results", "tds_result_stats",
                 "tds_index_export", "tds_index_info", "tds_merge_trajectories", "tds_search_many",
                 "tds_search_part", "tds_plan", "tds_time_partition", "tds_search_stream",
                 "tds_result_host_block"):
        getattr(lib, name).restype = i32
    _lib = lib
    return lib


def _check(code):
    if code != 0:
        raise TdsError(code, _lib.tds_last_error().decode())


def _stream_ptr(stream):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    try:
        import torch
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:
        pass
    return ctypes.c_void_p(0)


def _segments(x):
    """Return (pointer, n, keepalive) for an [n, 8] float32 array (torch cuda/cpu or numpy)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.dtype != torch.float32 or x.dim() != 2 or x.shape[1] != 8:
                raise ValueError("segments must be a float32 tensor of shape [n, 8]")
            x = x.contiguous()
            return ctypes.c_void_p(x.data_ptr()), x.shape[0], x
    except ImportError:
        pass
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32).reshape(-1, 8))
    if a.ctypes.data % 16:
        b = np.empty(a.shape[0] * 8 + 4, np.float32)
        off = (-b.ctypes.data % 16) // 4
        b = b[off:off + a.size].reshape(-1, 8)
        b[...] = a
        a = b
    return ctypes.c_void_p(a.ctypes.data), a.shape[0], a


def _u32(x):
    """(pointer, n, keepalive) for a 1-D uint32/int32 array (torch cuda/cpu or numpy)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.dtype not in (torch.int32,) or x.dim() != 1:
                x = x.to(torch.int32).reshape(-1)
            x = x.contiguous()
            return ctypes.c_void_p(x.data_ptr()), x.shape[0], x
    except ImportError:
        pass
    a = np.ascontiguousarray(np.asarray(x).astype(np.uint32).reshape(-1))
    return ctypes.c_void_p(a.ctypes.data), a.shape[0], a


class Index:
    """Resident index over the database D (tds_build_index, §4)."""

    def __init__(self, entries, kinds: int = ALL, m: int = 1000, v: int = 1, grid=(50, 50, 50), stream=None,
                 time_order: bool = False):
        lib = load_library()
        p = _Params(int(kinds), int(m), int(v), (ctypes.c_int32 * 3)(*[int(g) for g in grid]),
                    TIME_ORDER if time_order else 0)
        ptr, n, keep = _segments(entries)
        h = ctypes.c_void_p()
        _check(lib.tds_build_index(ptr, n, ctypes.byref(p), _stream_ptr(stream), ctypes.byref(h)))
        del keep
        self._h = h
        self.n = n
        self.m, self.v, self.grid, self.kinds = int(m), int(v), tuple(grid), int(kinds)

    def search(self, queries, d: float, window=(-math.inf, math.inf), kind="temporal", capacity: int = 0,
               stream=None, part: int = 0, nparts: int = 1) -> "Result":
        """tds_search, or with nparts > 1 part ``part`` of a work-balanced split
        (tds_search_part: disjoint parts whose union is the full result)."""
        lib = load_library()
        k = KINDS[kind] if isinstance(kind, str) else int(kind)
        ptr, nq, keep = _segments(queries)
        h = ctypes.c_void_p()
        n = ctypes.c_uint64()
        if nparts > 1:
            _check(lib.tds_search_part(self._h, k, ptr, nq, float(d), float(window[0]), float(window[1]),
                                       int(capacity), int(part), int(nparts), _stream_ptr(stream), ctypes.byref(h),
                                       ctypes.byref(n)))
        else:
            _check(lib.tds_search(self._h, k, ptr, nq, float(d), float(window[0]), float(window[1]), int(capacity),
                                  _stream_ptr(stream), ctypes.byref(h), ctypes.byref(n)))
        del keep
        return Result(h, n.value)

    def search_stream(self, queries, d: float, window=(-math.inf, math.inf), kind="temporal", chunk: int = 1 << 16,
                      stream=None, part: int = 0, nparts: int = 1) -> "Result":
        """tds_search_stream: ``queries`` in host memory (numpy or CPU tensor),
        searched ``chunk`` queries at a time with the copies overlapped; the
        result is host-resident."""
        lib = load_library()
        k = KINDS[kind] if isinstance(kind, str) else int(kind)
        ptr, nq, keep = _segments(queries)
        h = ctypes.c_void_p()
        n = ctypes.c_uint64()
        _check(lib.tds_search_stream(self._h, k, ptr, nq, float(d), float(window[0]), float(window[1]), int(chunk),
                                     int(part), int(nparts), _stream_ptr(stream), ctypes.byref(h), ctypes.byref(n)))
        del keep
        return Result(h, n.value)

    def plan(self, queries, d: float, window=(-math.inf, math.inf), kind="spatiotemporal", stream=None):
        """tds_plan: per query row (sel, lo, hi) of the schedule (numpy arrays)."""
        lib = load_library()
        k = KINDS[kind] if isinstance(kind, str) else int(kind)
        ptr, nq, keep = _segments(queries)
        sel = np.empty(nq, np.int32)
        lo = np.empty(nq, np.uint32)
        hi = np.empty(nq, np.uint32)
        _check(lib.tds_plan(self._h, k, ptr, nq, float(d), float(window[0]), float(window[1]), _stream_ptr(stream),
                            sel.ctypes.data_as(ctypes.c_void_p), lo.ctypes.data_as(ctypes.c_void_p),
                            hi.ctypes.data_as(ctypes.c_void_p)))
        del keep
        return sel, lo, hi

    def search_many(self, requests) -> list:
        """Independent searches of this index in one call (tds_search_many):
        ``requests`` is a list of dicts with the arguments of ``search`` (queries,
        d, and optionally window, kind, capacity, stream).  Requests on distinct
        streams run concurrently; returns one Result per request, in order."""
        lib = load_library()
        n = len(requests)
        reqs = (_SearchReq * max(n, 1))()
        keep = []
        for i, r in enumerate(requests):
            k = r.get("kind", "temporal")
            ptr, nq, kp = _segments(r["queries"])
            keep.append(kp)
            w = r.get("window", (-math.inf, math.inf))
            reqs[i] = _SearchReq(KINDS[k] if isinstance(k, str) else int(k), ptr, nq, float(r["d"]), float(w[0]),
                                 float(w[1]), int(r.get("capacity", 0)), _stream_ptr(r.get("stream")))
        hs = (ctypes.c_void_p * max(n, 1))()
        ns = (ctypes.c_uint64 * max(n, 1))()
        _check(lib.tds_search_many(self._h, n, reqs, hs, ns))
        del keep
        return [Result(ctypes.c_void_p(hs[i]), ns[i]) for i in range(n)]

    def export(self, what: str) -> np.ndarray:
        lib = load_library()
        nb = ctypes.c_uint64()
        _check(lib.tds_index_export(self._h, EXPORT[what], None, 0, ctypes.byref(nb)))
        out = np.empty(nb.value // 4, dtype=_EXPORT_DT.get(what, np.uint32))
        _check(lib.tds_index_export(self._h, EXPORT[what], out.ctypes.data_as(ctypes.c_void_p), nb.value,
                                    ctypes.byref(nb)))
        return out

    def export_nbytes(self, what: str) -> int:
        """Size in bytes of one exported index array (tds_index_export with no destination)."""
        nb = ctypes.c_uint64()
        _check(load_library().tds_index_export(self._h, EXPORT[what], None, 0, ctypes.byref(nb)))
        return int(nb.value)

    def close(self):
        if getattr(self, "_h", None):
            load_library().tds_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Result:
    """Result set of one search (tds_result)."""

    def __init__(self, h, n):
        self._h = h
        self.count = int(n)

    def stats(self) -> dict:
        st = _Stats()
        _check(load_library().tds_result_stats(self._h, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in _Stats._fields_}

    def fetch(self, sorted: bool = False, device: bool = True, first: int = 0, count=None, stream=None,
              out=None):
        """Return (query_id, entry_id, t_in, t_out).

        device=True -> torch CUDA tensors (int32 ids, float32 times);
        device=False -> numpy arrays.  ``out`` may supply preallocated buffers.
        """
        lib = load_library()
        cnt = self.count - first if count is None else int(count)
        if device:
            import torch
            if out is None:     # one allocation for the four columns
                buf = torch.empty((4, cnt), dtype=torch.int32, device="cuda")
                q, e, ti, to = buf[0], buf[1], buf[2].view(torch.float32), buf[3].view(torch.float32)
            else:
                q, e, ti, to = out
            ptrs = [ctypes.c_void_p(t.data_ptr()) for t in (q, e, ti, to)]
        else:
            if out is None:
                buf = np.empty((4, cnt), np.uint32)
                q, e, ti, to = buf[0], buf[1], buf[2].view(np.float32), buf[3].view(np.float32)
            else:
                q, e, ti, to = out
            ptrs = [ctypes.c_void_p(a.ctypes.data) for a in (q, e, ti, to)]
        _check(lib.tds_fetch_results(self._h, int(first), cnt, *ptrs, 1 if device else 0, 1 if sorted else 0,
                                     _stream_ptr(stream)))
        return q, e, ti, to

    REC_DTYPE = np.dtype([("qid", "<u4"), ("eid", "<u4"), ("t_in", "<f4"), ("t_out", "<f4")])

    def host_records(self) -> list:
        """Zero-copy numpy views (structured dtype REC_DTYPE) of the blocks of a
        host-resident result (tds_search_stream), valid until close()."""
        lib = load_library()
        out = []
        i = 0
        while True:
            p = ctypes.c_void_p()
            n = ctypes.c_uint64()
            _check(lib.tds_result_host_block(self._h, i, ctypes.byref(p), ctypes.byref(n)))
            if not n.value:
                return out
            buf = (ctypes.c_char * (16 * n.value)).from_address(p.value)
            out.append(np.frombuffer(buf, dtype=self.REC_DTYPE))
            i += 1

    def merge_trajectories(self, q_traj, e_traj, gap: float = 0.0, stream=None) -> "Result":
        """Trajectory-level answer (tds_merge_trajectories): records become
        (query trajectory, entry trajectory, t_in, t_out), maximal intervals."""
        lib = load_library()
        qp, nq, kq = _u32(q_traj)
        ep, ne, ke = _u32(e_traj)
        h = ctypes.c_void_p()
        n = ctypes.c_uint64()
        _check(lib.tds_merge_trajectories(self._h, qp, nq, ep, ne, float(gap), _stream_ptr(stream), ctypes.byref(h),
                                          ctypes.byref(n)))
        del kq, ke
        return Result(h, n.value)

    def close(self):
        if getattr(self, "_h", None):
            load_library().tds_result_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def time_partition(t_start, part: int, nparts: int, stream=None):
    """tds_time_partition: rows of D owned by ``part`` of ``nparts`` (contiguous
    t_start ranges of equal count, from the device sort of the t_start column);
    returns a CUDA int32 tensor in (t_start, row) order.  ``t_start`` is a 1-D
    float32 tensor (CUDA or CPU) or numpy array."""
    import torch
    lib = load_library()
    if isinstance(t_start, torch.Tensor):
        t = t_start.to(torch.float32).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(t_start, dtype=np.float32)))
    n = t.numel()
    rows = torch.empty(n // max(int(nparts), 1) + 1, dtype=torch.int32, device="cuda")
    cnt = ctypes.c_uint64()
    _check(lib.tds_time_partition(ctypes.c_void_p(t.data_ptr()), n, int(part), int(nparts), _stream_ptr(stream),
                                  ctypes.c_void_p(rows.data_ptr()), ctypes.byref(cnt)))
    return rows[:cnt.value]


def trim() -> None:
    """tds_trim: release the device memory the library's pools hold unused."""
    load_library().tds_trim()


def test_inject_enomem(k: int = -1, skip: int = 0) -> int:
    """TEST HOOK (tds_test_inject_enomem): after ``skip`` large allocations, fail
    the next k with TDS_ENOMEM (k >= 0); returns the failures injected so far."""
    return int(load_library().tds_test_inject_enomem(int(k), int(skip)))


def kernel_launches() -> int:
    """Kernels launched by the library in this process (monotone counter)."""
    return int(load_library().tds_kernel_launches())


def version() -> str:
    return load_library().tds_version().decode()
