"""ctypes binding of the sm_100a C-ABI library (include/rrs_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible every entry point raises.  PyTorch is used only for device tensors and
streams in the device-resident path.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RRS_B200_LIB: development override (kernel variants built under build/)
LIB_PATH = os.environ.get("RRS_B200_LIB") or os.path.join(_HERE, "_lib", "librrs_b200.so")

RRS_OK, RRS_ERR_INVALID, RRS_ERR_DIM, RRS_ERR_CUDA, RRS_ERR_NOMEM, RRS_ERR_STATE = range(6)
NOTION_CODES = {"halfspace": 0, "projection": 1, "asym_projection": 2}
POLE_UPDATE_CODES = {"per_refinement": 0, "per_direction": 1}

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_vp = ctypes.c_void_p


class RrsConfigC(ctypes.Structure):
    _fields_ = [
        ("total_directions", ctypes.c_int64),
        ("refinements", ctypes.c_int32),
        ("shrink", ctypes.c_double),
        ("notion", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("pole_update", ctypes.c_int32),
        ("early_exit", ctypes.c_int32),
    ]


class RrsStatsC(ctypes.Structure):
    _fields_ = [
        ("ms_generate", ctypes.c_double),
        ("ms_contract", ctypes.c_double),
        ("ms_univariate", ctypes.c_double),
        ("ms_update", ctypes.c_double),
        ("kernel_launches", ctypes.c_int64),
        ("contract_launches", ctypes.c_int64),
        ("ms_contract_total", ctypes.c_double),
        ("tensor_contract_launches", ctypes.c_int64),
        ("select_rows_fallback", ctypes.c_int64),
    ]


# (name, restype, argtypes) for every symbol declared in include/rrs_b200.h
SIGNATURES = [
    ("rrs_abi_version", ctypes.c_int, []),
    ("rrs_last_error", ctypes.c_char_p, []),
    ("rrs_device_count", ctypes.c_int, [ctypes.POINTER(ctypes.c_int32)]),
    ("rrs_engine_create", ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(_vp)]),
    ("rrs_engine_destroy", ctypes.c_int, [_vp]),
    ("rrs_engine_set_stream", ctypes.c_int, [_vp, _vp]),
    ("rrs_engine_synchronize", ctypes.c_int, [_vp]),
    ("rrs_engine_set_workspace_limit", ctypes.c_int, [_vp, ctypes.c_int64]),
    ("rrs_set_dataset_host", ctypes.c_int, [_vp, _dp, ctypes.c_int64, ctypes.c_int32]),
    ("rrs_set_dataset_device", ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int32]),
    ("rrs_depth_batch_host", ctypes.c_int,
     [_vp, _dp, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(RrsConfigC), _dp, _dp, _dp, _dp, _i64p]),
    ("rrs_depth_batch_device", ctypes.c_int,
     [_vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(RrsConfigC), _dp, _vp, _vp, _vp, _vp]),
    ("rrs_evaluate_directions_host", ctypes.c_int,
     [_vp, _dp, _dp, ctypes.c_int32, ctypes.c_int32, _dp, _i64p, _i64p]),
    ("rrs_cap_directions_host", ctypes.c_int,
     [_vp, _dp, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32,
      ctypes.c_uint32, _dp]),
    ("rrs_philox4x32_host", ctypes.c_int,
     [_vp, _u32p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint32, _u32p]),
    ("rrs_cap_directions_at_host", ctypes.c_int,
     [_vp, _dp, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32,
      ctypes.c_uint32, ctypes.c_uint32, _dp]),
    ("rrs_unit_rows_host", ctypes.c_int,
     [_vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
      ctypes.c_uint32, _dp]),
    ("rrs_stream_values_host", ctypes.c_int,
     [_vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int64,
      ctypes.c_int32, _dp]),
    ("rrs_project_host", ctypes.c_int, [_vp, _dp, ctypes.c_int64, ctypes.c_int32, _dp, ctypes.c_int32, _dp]),
    ("rrs_depth_of_projections_host", ctypes.c_int,
     [_vp, ctypes.c_int32, _dp, ctypes.c_int32, ctypes.c_int64, _dp, _dp]),
    ("rrs_engine_stats", ctypes.c_int, [_vp, ctypes.POINTER(RrsStatsC)]),
    ("rrs_engine_enable_timing", ctypes.c_int, [_vp, ctypes.c_int32]),
    ("rrs_engine_set_contract_path", ctypes.c_int, [_vp, ctypes.c_int32]),
    ("rrs_engine_set_select_path", ctypes.c_int, [_vp, ctypes.c_int32]),
    ("rrs_host_alloc", ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    ("rrs_host_free", ctypes.c_int, [ctypes.c_void_p]),
]

_lib = None
_lock = threading.Lock()


class LibraryNotBuilt(RuntimeError):
    pass


def load_library():
    """Load librrs_b200.so (raises if it was not built; no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryNotBuilt(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2506_08262_b200.build` "
                    "(the B200 path has no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            if L.rrs_abi_version() != 3:
                raise RuntimeError("librrs_b200.so ABI version mismatch")
            _lib = L
    return _lib


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _raise(rc):
    if rc == RRS_OK:
        return
    msg = load_library().rrs_last_error().decode()
    if rc == RRS_ERR_DIM:
        from .config import DimensionMismatch

        raise DimensionMismatch(msg)
    if rc == RRS_ERR_INVALID:
        raise ValueError(msg)
    if rc == RRS_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"librrs_b200: {msg}")


class _PinnedBlock:
    """Owner of one page-locked host allocation (rrs_host_alloc); freed when
    the last numpy view of it goes away."""

    def __init__(self, nbytes: int):
        ptr = ctypes.c_void_p()
        _raise(load_library().rrs_host_alloc(int(nbytes), ctypes.byref(ptr)))
        self.ptr = ptr.value
        self.nbytes = int(nbytes)

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.rrs_host_free(ctypes.c_void_p(self.ptr))
            self.ptr = None


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """Uninitialised numpy array in page-locked host memory (H2D by DMA)."""
    shape = tuple(int(s) for s in np.atleast_1d(shape))
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    block = _PinnedBlock(max(nbytes, 1))
    buf = (ctypes.c_char * max(nbytes, 1)).from_address(block.ptr)
    buf._owner = block  # the ctypes buffer keeps the block alive; numpy keeps the buffer
    return np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)


def device_count() -> int:
    c = ctypes.c_int32(0)
    load_library().rrs_device_count(ctypes.byref(c))
    return int(c.value)


def config_struct(cfg) -> RrsConfigC:
    return RrsConfigC(int(cfg.total_directions), int(cfg.refinements), float(cfg.shrink),
                      NOTION_CODES[cfg.notion], int(cfg.seed) % (1 << 64),
                      POLE_UPDATE_CODES[cfg.pole_update], 1 if getattr(cfg, "early_exit", False) else 0)


class Engine:
    """One rrs_engine (one CUDA device, one stream, resident dataset).

    The engine's dataset and workspace are shared state, and ctypes releases
    the GIL for every call, so a caller that sets the dataset and then runs on
    it must hold ``lock`` across both (solver.py does); the reference's
    functions are safe to call concurrently."""

    def __init__(self, device: int = 0):
        self.lock = threading.RLock()
        L = load_library()
        h = _vp()
        _raise(L.rrs_engine_create(int(device), ctypes.byref(h)))
        self._h = h
        self.device = int(device)
        self.dataset_key = None
        self.n = 0
        self.d = 0

    def close(self):
        if getattr(self, "_h", None):
            load_library().rrs_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- configuration
    def set_stream(self, stream_handle: int | None):
        _raise(load_library().rrs_engine_set_stream(self._h, stream_handle or None))

    def synchronize(self):
        _raise(load_library().rrs_engine_synchronize(self._h))

    def set_workspace_limit(self, nbytes: int):
        _raise(load_library().rrs_engine_set_workspace_limit(self._h, int(nbytes)))

    def set_contract_path(self, path: str):
        """'auto' | 'ffma' | 'tensor' | 'filter' | 'tensor3' | 'convert'
        (contraction kernel; tensor = the two-term FP16 split: contract_tc.cu
        for d <= 64, the pre-split contract_tcp.cu for 64 < d <= 256; convert =
        the same split with in-kernel converters above d = 64, contract_tcw.cu;
        filter = filter and refine, contract_tcf.cu, d <= 64; tensor3 = the
        three-term projection store, contract_tcs.cu)."""
        code = {"auto": 0, "ffma": 1, "tensor": 2, "filter": 4, "tensor3": 5, "convert": 6}[path]
        _raise(load_library().rrs_engine_set_contract_path(self._h, code))

    def set_select_path(self, path: str):
        """'auto' | 'radix' | 'wide' (order-statistic kernel of the projection
        notions: auto = the sample-bracket select v3 where it applies, radix =
        select v2 everywhere, wide = v3 with 1024-thread CTAs above n = 16k;
        bitwise equal depths)."""
        code = {"auto": 0, "radix": 2, "wide": 3}[path]
        _raise(load_library().rrs_engine_set_select_path(self._h, code))

    def enable_timing(self, on: bool = True):
        _raise(load_library().rrs_engine_enable_timing(self._h, 1 if on else 0))

    def stats(self) -> dict:
        s = RrsStatsC()
        _raise(load_library().rrs_engine_stats(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in RrsStatsC._fields_}

    # -- dataset
    def set_dataset(self, x: np.ndarray, key=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        _raise(load_library().rrs_set_dataset_host(self._h, _p(x), x.shape[0], x.shape[1]))
        self.dataset_key, self.n, self.d = key, x.shape[0], x.shape[1]

    def set_dataset_device(self, x_dev, key=None):
        """x_dev: CUDA float64 tensor (n, d), contiguous."""
        n, d = x_dev.shape
        _raise(load_library().rrs_set_dataset_device(self._h, x_dev.data_ptr(), n, d))
        self.dataset_key, self.n, self.d = key, n, d

    # -- RRS
    def depth_batch(self, Z: np.ndarray, cfg, q0: int = 0, trace: bool = False, eps=None):
        Z = np.ascontiguousarray(Z, dtype=np.float64).reshape(-1, self.d)
        Q = Z.shape[0]
        depth = np.empty(Q)
        argmin = np.empty((Q, self.d))
        counts = np.empty(Q, dtype=np.int64)
        tr = np.empty((Q, cfg.refinements, 2 + self.d)) if trace else None
        c = config_struct(cfg)
        e = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
        _raise(load_library().rrs_depth_batch_host(self._h, _p(Z), Q, int(q0), ctypes.byref(c), _p(e),
                                                   _p(depth), _p(argmin), _p(tr), _p(counts, _i64p)))
        return depth, argmin, tr, counts

    def depth_batch_device(self, Z_dev, cfg, q0, depth_dev, argmin_dev=None, trace_dev=None,
                           count_dev=None, eps=None):
        """All tensors CUDA, contiguous: Z float64 (Q,d); depth float64 (Q,);
        argmin float64 (Q,d); trace float64 (Q,r,2+d); count int64 (Q,)."""
        c = config_struct(cfg)
        e = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
        ptr = lambda t: None if t is None else t.data_ptr()
        _raise(load_library().rrs_depth_batch_device(
            self._h, Z_dev.data_ptr(), Z_dev.shape[0], int(q0), ctypes.byref(c), _p(e),
            depth_dev.data_ptr(), ptr(argmin_dev), ptr(trace_dev), ptr(count_dev)))

    def evaluate_directions(self, z, U, notion: str):
        z = np.ascontiguousarray(z, dtype=np.float64).reshape(-1)
        U = np.ascontiguousarray(U, dtype=np.float64)
        m = U.shape[0]
        out = np.empty(m)
        cle = np.zeros(m, dtype=np.int64)
        cge = np.zeros(m, dtype=np.int64)
        _raise(load_library().rrs_evaluate_directions_host(self._h, _p(z), _p(U), m, NOTION_CODES[notion],
                                                           _p(out), _p(cle, _i64p), _p(cge, _i64p)))
        return out, cle, cge

    def cap_directions(self, pole, eps, m, seed, refinement, query, index_base=0):
        pole = np.ascontiguousarray(pole, dtype=np.float64).reshape(-1)
        U = np.empty((m, pole.size))
        _raise(load_library().rrs_cap_directions_at_host(self._h, _p(pole), pole.size, float(eps), int(m),
                                                         int(seed) % (1 << 64), int(refinement) % (1 << 32),
                                                         int(query) % (1 << 32), int(index_base) % (1 << 32),
                                                         _p(U)))
        return U

    def unit_rows(self, seed, refinement, query, m, dim, v_base, index_base):
        U = np.empty((int(m), int(dim)))
        _raise(load_library().rrs_unit_rows_host(self._h, int(seed) % (1 << 64), int(refinement) % (1 << 32),
                                                 int(query) % (1 << 32), int(m), int(dim),
                                                 int(v_base) % (1 << 32), int(index_base) % (1 << 32), _p(U)))
        return U

    def stream_values(self, seed, refinement, query, index, offset, count, normal: bool):
        out = np.empty(int(count))
        _raise(load_library().rrs_stream_values_host(self._h, int(seed) % (1 << 64), int(refinement) % (1 << 32),
                                                     int(query) % (1 << 32), int(index) % (1 << 32),
                                                     int(offset) % (1 << 32), int(count), 1 if normal else 0,
                                                     _p(out)))
        return out

    def project(self, x, U):
        x = np.ascontiguousarray(x, dtype=np.float64)
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty((U.shape[0], x.shape[0]))
        _raise(load_library().rrs_project_host(self._h, _p(x), x.shape[0], x.shape[1], _p(U), U.shape[0],
                                               _p(out)))
        return out

    def depth_of_projections(self, notion: str, px, pz, out):
        _raise(load_library().rrs_depth_of_projections_host(self._h, NOTION_CODES[notion], _p(px), px.shape[0],
                                                            px.shape[1], _p(pz), _p(out)))
        return out

    def philox4x32(self, ctr, key0, key1):
        ctr = np.ascontiguousarray(ctr, dtype=np.uint32)
        out = np.empty_like(ctr)
        _raise(load_library().rrs_philox4x32_host(self._h, _p(ctr, _u32p), ctr.shape[1],
                                                  int(key0) & 0xFFFFFFFF, int(key1) & 0xFFFFFFFF,
                                                  _p(out, _u32p)))
        return out


_engines: dict[int, Engine] = {}


def engine(device: int | None = None) -> Engine:
    """Process-wide engine for `device` (default: torch's current device or 0)."""
    if device is None:
        device = _current_device()
    with _lock:
        e = _engines.get(device)
    if e is None:
        e = Engine(device)
        with _lock:
            _engines[device] = e
    return e


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0
