"""ctypes wrapper of oracle/c/liboracle.so — the C restatement of the reference
CPU path (checker and CPU baseline only; never used by the product)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "c", "liboracle.so")
_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "c")])
    lib = ctypes.CDLL(LIB)
    P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    lib.oc_msd_matrix.argtypes = [P, P, I, I, I, P, P, P, I]
    lib.oc_msd_matrix.restype = I
    lib.oc_path_cv_exact.argtypes = [P, P, I, I, I, D, P, P, P, P, P, P, P, I]
    lib.oc_path_cv_exact.restype = I
    lib.oc_max_threads.restype = I
    _lib = lib
    return lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _w(w, n):
    if w is None:
        return np.full(n, 1.0 / n)
    w = np.asarray(w, dtype=float)
    return w / w.sum()


def max_threads():
    return load().oc_max_threads()


def msd_matrix(frames, landmarks, w=None, w_align=None, nthreads=0):
    lib = load()
    fr = np.ascontiguousarray(frames, dtype=np.float64)
    lm = np.ascontiguousarray(landmarks, dtype=np.float64)
    T, n, _ = fr.shape
    L = lm.shape[0]
    D = np.empty((T, L))
    used = lib.oc_msd_matrix(_p(fr), _p(lm), T, L, n, _p(_w(w, n)), _p(_w(w_align, n)), _p(D), nthreads)
    return D, used


def path_cv_exact(frames, landmarks, lam, q=None, w=None, w_align=None, grad=True, nthreads=0):
    lib = load()
    fr = np.ascontiguousarray(frames, dtype=np.float64)
    lm = np.ascontiguousarray(landmarks, dtype=np.float64)
    T, n, _ = fr.shape
    L = lm.shape[0]
    q = np.arange(L, dtype=float) if q is None else np.ascontiguousarray(q, dtype=float)
    s, z = np.empty(T), np.empty(T)
    ds = np.empty((T, n, 3)) if grad else None
    dz = np.empty((T, n, 3)) if grad else None
    wv, wav = _w(w, n), _w(w_align, n)
    used = lib.oc_path_cv_exact(_p(fr), _p(lm), T, L, n, float(lam), _p(q), _p(wv), _p(wav), _p(s), _p(z),
                                _p(ds), _p(dz), nthreads)
    return {"s": s, "z": z, "ds": ds, "dz": dz, "threads": used}


def close_replay(frames, landmarks, lam, eps, q=None, w=None, w_align=None, grad=True, nthreads=0):
    lib = load()
    P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    lib.oc_close_replay.argtypes = [P, P, I, I, I, D, P, P, P, D, P, P, P, P, P, P, I]
    lib.oc_close_replay.restype = I
    fr = np.ascontiguousarray(frames, dtype=np.float64)
    lm = np.ascontiguousarray(landmarks, dtype=np.float64)
    T, n, _ = fr.shape
    L = lm.shape[0]
    q = np.arange(L, dtype=float) if q is None else np.ascontiguousarray(q, dtype=float)
    s, z = np.empty(T), np.empty(T)
    ds = np.empty((T, n, 3)) if grad else None
    dz = np.empty((T, n, 3)) if grad else None
    refresh = np.empty(T, dtype=np.uint8)
    dxy = np.empty(T)
    used = lib.oc_close_replay(_p(fr), _p(lm), T, L, n, float(lam), _p(q), _p(_w(w, n)), _p(_w(w_align, n)),
                               float(eps), _p(s), _p(z), _p(ds), _p(dz), _p(refresh), _p(dxy), nthreads)
    return {"s": s, "z": z, "ds": ds, "dz": dz, "refresh": refresh.astype(bool), "dxy": dxy, "threads": used}
