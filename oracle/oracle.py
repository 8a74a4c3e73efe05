"""ctypes wrapper for the CPU restatement in oracle/rrs_oracle.c.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs as the checker / the timed "port" baseline; the
product package (paper_2506_08262_b200) never imports it.

Every wrapper mirrors a reference function (paths relative to
/root/reference/pkg/src/depthforge):
  philox4x32          philox.py:27-65
  uniforms            philox.py:88-114
  ndtri               scipy.special.ndtri (Cephes), philox.py:117-125
  pairwise_sum        numpy add.reduce on a contiguous row
  cap_rows            directions.py:167-182 (generate_batch rows)
  project/_point      _kernels.pyx:171-199
  univariate          _kernels.pyx:270-351 (*_span kernels)
  evaluate_directions optimizer.py:98-142
  depth_batch         optimizer.py:254-279 (+ refined_random_search :145-226)
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "librrs_oracle.so")

NOTION_CODES = {"halfspace": 0, "projection": 1, "asym_projection": 2}

_dp = ctypes.POINTER(ctypes.c_double)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i64p = ctypes.POINTER(ctypes.c_int64)


class OrcCfg(ctypes.Structure):
    _fields_ = [
        ("total_directions", ctypes.c_int64),
        ("refinements", ctypes.c_int32),
        ("shrink", ctypes.c_double),
        ("notion", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("pole_update", ctypes.c_int32),
    ]


def build() -> str:
    """Compile the oracle (make -C oracle); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.orc_philox4x32.argtypes = [_u32p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint32, _u32p]
        L.orc_uniforms.argtypes = [ctypes.c_uint64, _u32p, _u32p, ctypes.c_int64,
                                   ctypes.c_uint32, ctypes.c_uint32, _dp]
        L.orc_ndtri.argtypes = [ctypes.c_double]
        L.orc_ndtri.restype = ctypes.c_double
        L.orc_ndtri_array.argtypes = [_dp, ctypes.c_int64, _dp]
        L.orc_pairwise_sum.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64]
        L.orc_pairwise_sum.restype = ctypes.c_double
        L.orc_cap_rows.argtypes = [_dp, ctypes.c_int32, ctypes.c_double, ctypes.c_int32,
                                   ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, _dp]
        L.orc_project.argtypes = [_dp, ctypes.c_int64, ctypes.c_int32, _dp, ctypes.c_int32, _dp]
        L.orc_project_point.argtypes = [_dp, ctypes.c_int32, _dp, ctypes.c_int32, _dp]
        L.orc_univariate.argtypes = [ctypes.c_int32, _dp, _dp, ctypes.c_int32, ctypes.c_int64,
                                     _dp, _i64p, _i64p]
        L.orc_evaluate_directions.argtypes = [_dp, ctypes.c_int64, ctypes.c_int32, _dp, _dp,
                                              ctypes.c_int32, ctypes.c_int32, _dp, _i64p, _i64p]
        L.orc_depth_batch.argtypes = [_dp, ctypes.c_int64, ctypes.c_int32, _dp, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.POINTER(OrcCfg), ctypes.c_int32,
                                      _dp, _dp, _dp]
        L.orc_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


def _check(rc):
    if rc:
        raise ValueError(lib().orc_last_error().decode())


def philox4x32(counter, key0, key1):
    c = np.ascontiguousarray(counter, dtype=np.uint32)
    out = np.empty_like(c)
    lib().orc_philox4x32(_p(c, _u32p), c.shape[1], key0 & 0xFFFFFFFF, key1 & 0xFFFFFFFF, _p(out, _u32p))
    return out


def uniforms(seed, v, j, l, q):
    v, j = np.broadcast_arrays(np.asarray(v, dtype=np.uint32), np.asarray(j, dtype=np.uint32))
    shape = v.shape
    v = np.ascontiguousarray(v.ravel())
    j = np.ascontiguousarray(j.ravel())
    out = np.empty(v.size)
    lib().orc_uniforms(seed % (1 << 64), _p(v, _u32p), _p(j, _u32p), v.size, l % (1 << 32),
                       q % (1 << 32), _p(out))
    return out.reshape(shape)


def ndtri(y):
    y = _f64(y)
    out = np.empty_like(y)
    lib().orc_ndtri_array(_p(y), y.size, _p(out))
    return out


def pairwise_sum(a):
    a = _f64(a)
    return lib().orc_pairwise_sum(_p(a), a.size, 1)


def cap_rows(pole, eps, m, seed, refinement, query):
    pole = _f64(pole).reshape(-1)
    d = pole.size
    out = np.empty((m, d))
    _check(lib().orc_cap_rows(_p(pole), d, float(eps), m, seed % (1 << 64),
                              refinement % (1 << 32), query % (1 << 32), _p(out)))
    return out


def project(x, u):
    x = _f64(x)
    u = _f64(u)
    out = np.empty((u.shape[0], x.shape[0]))
    lib().orc_project(_p(x), x.shape[0], x.shape[1], _p(u), u.shape[0], _p(out))
    return out


def project_point(z, u):
    z = _f64(z).reshape(-1)
    u = _f64(u)
    out = np.empty(u.shape[0])
    lib().orc_project_point(_p(z), z.size, _p(u), u.shape[0], _p(out))
    return out


def univariate(notion, px, pz, with_counts=False):
    px = _f64(px)
    pz = _f64(pz).reshape(-1)
    m, n = px.shape
    out = np.empty(m)
    cle = np.zeros(m, dtype=np.int64)
    cge = np.zeros(m, dtype=np.int64)
    _check(lib().orc_univariate(NOTION_CODES[notion], _p(px), _p(pz), m, n, _p(out),
                                _p(cle, _i64p), _p(cge, _i64p)))
    return (out, cle, cge) if with_counts else out


def evaluate_directions(z, x, U, notion, with_counts=False):
    x = _f64(x)
    z = _f64(z).reshape(-1)
    U = _f64(U)
    m = U.shape[0]
    out = np.empty(m)
    cle = np.zeros(m, dtype=np.int64)
    cge = np.zeros(m, dtype=np.int64)
    _check(lib().orc_evaluate_directions(_p(x), x.shape[0], x.shape[1], _p(z), _p(U), m,
                                         NOTION_CODES[notion], _p(out), _p(cle, _i64p),
                                         _p(cge, _i64p)))
    return (out, cle, cge) if with_counts else out


def depth_batch(queries, x, *, total_directions, refinements, shrink, notion, seed,
                pole_update="per_refinement", threads=0, q0=0, trace=False):
    """Returns (depth[Q], argmin[Q,d], trace[Q,r,2+d] or None)."""
    x = _f64(x)
    Z = _f64(queries).reshape(-1, x.shape[1])
    Q, d = Z.shape
    cfg = OrcCfg(total_directions, refinements, shrink, NOTION_CODES[notion], seed % (1 << 64),
                 0 if pole_update == "per_refinement" else 1)
    depth = np.empty(Q)
    argmin = np.empty((Q, d))
    tr = np.empty((Q, refinements, 2 + d)) if trace else None
    _check(lib().orc_depth_batch(_p(x), x.shape[0], d, _p(Z), Q, q0, ctypes.byref(cfg),
                                 threads, _p(depth), _p(argmin),
                                 _p(tr) if trace else ctypes.cast(None, _dp)))
    return depth, argmin, tr


def epsilons(refinements, shrink):
    """optimizer.py:175 schedule, evaluated exactly as the reference does."""
    return [(math.pi / 2.0) * shrink**l for l in range(refinements)]
