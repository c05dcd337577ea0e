"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the C restatement
(oracle/ffit_oracle.c -> oracle/_build/liboracle.so) and for the reference engine
compiled from its own sources (oracle/_ref/libffit_ref.so, see oracle/Makefile).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .model_text import parse

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libffit_ref.so")

_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)
_LL = ctypes.c_longlong


def build():
    """Build liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_unnorm.restype = _D
        L.orc_extended_term.restype = _D
        _lib = L
    return _lib


def ref_available(variant=None):
    return os.path.exists(ref_path(variant))


def ref_path(variant=None):
    """oracle/_ref builds: None = the reference's Release flags (baseline x86-64), "v3" /
    "v4" = the same sources with -march=x86-64-v3 / -v4 (oracle/Makefile)."""
    return REF_SO if not variant else os.path.join(HERE, "_ref", f"libffit_ref_{variant}.so")


_ref_variants = {}


def ref(variant=None):
    global _ref
    if not variant:
        if _ref is None:
            L = ctypes.CDLL(REF_SO)
            L.ref_last_error.restype = ctypes.c_char_p
            _ref = L
        return _ref
    if variant not in _ref_variants:
        L = ctypes.CDLL(ref_path(variant))
        L.ref_last_error.restype = ctypes.c_char_p
        _ref_variants[variant] = L
    return _ref_variants[variant]


def host_isa_levels():
    """The oracle/_ref ISA builds this host CPU can run (from /proc/cpuinfo flags)."""
    try:
        flags = set()
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    flags = set(line.split(":", 1)[1].split())
                    break
    except OSError:
        return []
    out = []
    if {"avx2", "fma", "bmi2", "movbe"} <= flags:
        out.append("v3")
        if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags:
            out.append("v4")
    return out


class RefColumn:
    """A reference DataSet (one column) inside one ISA build of oracle/_ref."""

    def __init__(self, variant, name, col):
        self.variant = variant
        self.L = ref(variant)
        self.col = np.ascontiguousarray(col, dtype=np.float64)
        self.h = ctypes.c_void_p()
        rc = self.L.ref_dataset_create(name.encode(), _dp(self.col), _LL(len(self.col)), ctypes.byref(self.h))
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_dataset_free(self.h)
            self.h = None

    def nll_points(self, text, names, points, threads, mode=1):
        """ref_nll_points_threaded: P points over `threads` host threads, each with its own
        reference Model over this DataSet."""
        points = np.ascontiguousarray(points, dtype=np.float64)
        P = points.shape[0]
        out = np.empty(P)
        arr = (ctypes.c_char_p * len(names))(*[n.encode() for n in names])
        rc = self.L.ref_nll_points_threaded(text.encode(), self.h, mode, arr, len(names), _dp(points), P, threads,
                                            _dp(out))
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())
        return out


def ref_nll_points_variant(variant, text, column, col, names, points, threads, mode=1):
    """ref_nll_points_threaded on one ISA build (a DataSet made for the call)."""
    return RefColumn(variant, column, col).nll_points(text, names, points, threads, mode)


def _dp(a):
    return a.ctypes.data_as(_DP)


def _cols_ptr(cols):
    arr = (_DP * max(1, len(cols)))()
    for i, c in enumerate(cols):
        arr[i] = _dp(c)
    return arr


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc:
        raise OracleError(rc, lib().orc_last_error().decode())


class OracleModel:
    """CPU restatement of one model-file text (test checker)."""

    def __init__(self, text: str):
        self.text = text
        self.pm = parse(text)
        self.nodes = self.pm.node_array()
        self.root = self.pm.root
        self.param_names = [p[0] for p in self.pm.params]
        self.theta = np.array(self.pm.theta(), dtype=np.float64)
        self.obs = self.pm.observables

    def set(self, name, value):
        self.theta[self.param_names.index(name)] = value

    def _theta(self, theta):
        t = self.theta if theta is None else np.ascontiguousarray(theta, dtype=np.float64)
        return t

    @staticmethod
    def _cols(cols):
        return [np.ascontiguousarray(c, dtype=np.float64) for c in cols]

    def nll(self, cols, theta=None):
        """(naive reference-order sum, Neumaier sum, first_invalid)."""
        cols = self._cols(cols)
        n = len(cols[0]) if cols else 0
        t = self._theta(theta)
        naive, comp, bad = _D(), _D(), _LL()
        _check(lib().orc_nll(self.nodes, self.root, _dp(t), _cols_ptr(cols), _LL(n),
                             ctypes.byref(naive), ctypes.byref(comp), ctypes.byref(bad)))
        return naive.value, comp.value, bad.value

    def probabilities(self, cols, theta=None):
        cols = self._cols(cols)
        n = len(cols[0])
        out = np.empty(n)
        _check(lib().orc_probabilities(self.nodes, self.root, _dp(self._theta(theta)),
                                       _cols_ptr(cols), _LL(n), _dp(out)))
        return out

    def eval_batch(self, node, cols, theta=None):
        cols = self._cols(cols)
        n = len(cols[0])
        out = np.empty(n)
        _check(lib().orc_eval_batch(self.nodes, node, _dp(self._theta(theta)),
                                    _cols_ptr(cols), _LL(n), _dp(out)))
        return out

    def normalization(self, theta=None, node=None):
        out = _D()
        _check(lib().orc_normalization(self.nodes, self.root if node is None else node,
                                       _dp(self._theta(theta)), ctypes.byref(out)))
        return out.value

    def simpson_norm(self, theta=None, node=None):
        out = _D()
        _check(lib().orc_simpson_norm(self.nodes, self.root if node is None else node,
                                      _dp(self._theta(theta)), ctypes.byref(out)))
        return out.value

    def extended_term(self, n, theta=None):
        return lib().orc_extended_term(self.nodes, self.root, _dp(self._theta(theta)), _LL(n))

    def nll_points(self, cols, thetas, threads=1):
        cols = self._cols(cols)
        thetas = np.ascontiguousarray(thetas, dtype=np.float64)
        P = thetas.shape[0]
        out = np.empty(P)
        _check(lib().orc_nll_points(self.nodes, self.root, _dp(thetas), thetas.shape[1], P,
                                    _cols_ptr(cols), _LL(len(cols[0])), threads, _dp(out)))
        return out

    def sample(self, n, seed, theta=None):
        cols = [np.zeros(n) for _ in self.obs]
        eff = _D()
        _check(lib().orc_sample(self.nodes, self.root, _dp(self._theta(theta)), _LL(n),
                                ctypes.c_ulonglong(seed), _cols_ptr(cols), ctypes.byref(eff)))
        return cols, eff.value


def rng_uniform(seed, n):
    out = np.empty(n)
    lib().orc_rng_uniform(ctypes.c_ulonglong(seed), _LL(n), _dp(out))
    return out


def rng_gauss(seed, n):
    out = np.empty(n)
    lib().orc_rng_gauss(ctypes.c_ulonglong(seed), _LL(n), _dp(out))
    return out


# --------------------------------------------------------------------------
# the reference engine itself (oracle/_ref), for pinning the restatement


def _rcheck(rc):
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())


class RefDataset:
    def __init__(self, name, col):
        self.col = np.ascontiguousarray(col, dtype=np.float64)
        self.h = ctypes.c_void_p()
        _rcheck(ref().ref_dataset_create(name.encode(), _dp(self.col), _LL(len(self.col)),
                                         ctypes.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_dataset_free(self.h)


class RefModel:
    """The unmodified reference engine (single observable, its own grammar)."""

    SCALAR, PRECISE, FAST = 0, 1, 2

    def __init__(self, text):
        self.text = text
        self.h = ctypes.c_void_p()
        _rcheck(ref().ref_model_parse(text.encode(), ctypes.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_model_free(self.h)

    def set(self, name, v):
        _rcheck(ref().ref_set_param(self.h, name.encode(), _D(v)))

    def get(self, name):
        v, e = _D(), _D()
        _rcheck(ref().ref_get_param(self.h, name.encode(), ctypes.byref(v), ctypes.byref(e)))
        return v.value, e.value

    def nll(self, ds, mode=1):
        v, ne, bad = _D(), ctypes.c_ulonglong(), _LL()
        _rcheck(ref().ref_nll(self.h, ds.h, mode, ctypes.byref(v), ctypes.byref(ne),
                              ctypes.byref(bad)))
        return v.value, ne.value, bad.value

    def nll_compensated(self, ds, mode=1):
        v, bad = _D(), _LL()
        _rcheck(ref().ref_nll_compensated(self.h, ds.h, mode, ctypes.byref(v), ctypes.byref(bad)))
        return v.value, bad.value

    def probabilities(self, ds, mode=1):
        out = np.empty(len(ds.col))
        _rcheck(ref().ref_probabilities(self.h, ds.h, mode, _dp(out)))
        return out

    def normalization(self):
        out = _D()
        _rcheck(ref().ref_normalization(self.h, ctypes.byref(out)))
        return out.value

    def eval_unnorm(self, xs):
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        out = np.empty(len(xs))
        _rcheck(ref().ref_eval_unnorm(self.h, _dp(xs), _LL(len(xs)), _dp(out)))
        return out

    def sample(self, n, seed):
        out = np.empty(n)
        eff = _D()
        _rcheck(ref().ref_sample(self.h, _LL(n), ctypes.c_ulonglong(seed), _dp(out),
                                 ctypes.byref(eff)))
        return out, eff.value

    def fit(self, ds, mode=1, tol=0.0, max_iter=0):
        conv, nll, calls, uv = ctypes.c_int(), _D(), ctypes.c_ulonglong(), ctypes.c_int()
        _rcheck(ref().ref_fit(self.h, ds.h, mode, _D(tol), ctypes.c_long(max_iter),
                              ctypes.byref(conv), ctypes.byref(nll), ctypes.byref(calls),
                              ctypes.byref(uv)))
        return dict(converged=bool(conv.value), nll=nll.value, calls=calls.value,
                    uncertainties_valid=bool(uv.value))


def ref_nll_points_threaded(text, ds, names, points, threads, mode=1):
    points = np.ascontiguousarray(points, dtype=np.float64)
    P = points.shape[0]
    out = np.empty(P)
    arr = (ctypes.c_char_p * len(names))(*[n.encode() for n in names])
    _rcheck(ref().ref_nll_points_threaded(text.encode(), ds.h, mode, arr, len(names),
                                          _dp(points), P, threads, _dp(out)))
    return out


def ref_rng_uniform(seed, n):
    out = np.empty(n)
    ref().ref_rng_uniform(ctypes.c_ulonglong(seed), _LL(n), _dp(out))
    return out


def ref_rng_gauss(seed, n):
    out = np.empty(n)
    ref().ref_rng_gauss(ctypes.c_ulonglong(seed), _LL(n), _dp(out))
    return out


def ref_expr_eval(text, variables, values):
    """The reference's compiled formula at rows of variable values (npts x nvars)."""
    vals = np.ascontiguousarray(np.atleast_2d(values), dtype=np.float64)
    arr = (ctypes.c_char_p * len(variables))(*[v.encode() for v in variables])
    out = np.empty(vals.shape[0])
    rc = ref().ref_expr_eval(text.encode(), arr, len(variables), _dp(vals), vals.shape[0], _dp(out))
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return out
