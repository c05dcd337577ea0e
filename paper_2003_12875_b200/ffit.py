"""Python mirror of the reference's likelihood interface, over the C ABI.

Names follow the reference (proj/include/ffit/eval.hpp:12-44, model.hpp, fit.hpp,
include/ffit.h): ``Model.from_string``, ``DataSet``, ``nll(model, ds, mode)`` ->
``NllValue``, ``probabilities``, ``normalization``, ``fit_to`` -> ``FitResult``,
with the GPU extensions (``nll_points``, ``eval_batch``, ``fit_gradient``,
device-resident datasets).  Errors raise ``FfitError`` carrying the reference's
status codes (1 usage, 2 data, 3 numeric; proj/include/ffit/errors.hpp:9-24).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import CP, DP, LL, ULL, VP, lib


class FfitError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(f"[{code}] {message}")
        self.code = code
        self.message = message


USAGE, DATA, NUMERIC = 1, 2, 3
NO_INVALID = 0xFFFFFFFFFFFFFFFF


class EvalMode(enum.IntEnum):
    Scalar = 0
    BatchPrecise = 1
    BatchFast = 2
    Gpu = 3


def _check(rc):
    if rc:
        raise FfitError(rc, lib().ffit_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(DP)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Model:
    """A parsed model (observables, parameters, PDF tree) with its GPU engine."""

    def __init__(self, handle, text=None):
        self._h = handle
        self.text = text

    @classmethod
    def from_string(cls, text: str) -> "Model":
        h = VP()
        _check(lib().ffit_model_parse(text.encode(), ctypes.byref(h)))
        return cls(h, text)

    @classmethod
    def from_file(cls, path: str) -> "Model":
        h = VP()
        _check(lib().ffit_model_load(path.encode(), ctypes.byref(h)))
        with open(path) as fh:
            return cls(h, fh.read())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib().ffit_model_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def param_names(self):
        L = lib()
        return [L.ffit_model_param_name(self._h, i).decode() for i in range(L.ffit_model_param_count(self._h))]

    @property
    def observables(self):
        L = lib()
        return [L.ffcu_model_observable_name(self._h, i).decode()
                for i in range(L.ffcu_model_observable_count(self._h))]

    @property
    def pdf_names(self):
        L = lib()
        return [L.ffcu_model_pdf_name(self._h, i).decode() for i in range(L.ffcu_model_pdf_count(self._h))]

    def observable_range(self):
        lo, hi = ctypes.c_double(), ctypes.c_double()
        _check(lib().ffit_model_observable_range(self._h, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def set(self, name, value):
        _check(lib().ffit_model_set_param(self._h, name.encode(), float(value)))

    def get(self, name):
        v, e = ctypes.c_double(), ctypes.c_double()
        _check(lib().ffit_model_get_param(self._h, name.encode(), ctypes.byref(v), ctypes.byref(e)))
        return v.value, e.value

    def is_constant(self, name):
        c = ctypes.c_int()
        _check(lib().ffit_model_param_is_constant(self._h, name.encode(), ctypes.byref(c)))
        return bool(c.value)

    def theta(self):
        return np.array([self.get(n)[0] for n in self.param_names])

    def plan(self):
        """The flattened evaluation plan: (terms, ncols, stride)."""
        L = lib()
        nt, nc, st = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(L.ffcu_plan_info(self._h, ctypes.byref(nt), ctypes.byref(nc), ctypes.byref(st)))
        terms = []
        for i in range(nt.value):
            vals = [ctypes.c_int() for _ in range(5)]
            _check(L.ffcu_plan_term(self._h, i, *[ctypes.byref(v) for v in vals]))
            terms.append(dict(zip(("kind", "col", "order", "flags", "coff"), [v.value for v in vals])))
        return terms, nc.value, st.value

    def point_constants(self, point=None):
        _, _, stride = self.plan()
        row = np.empty(stride)
        p = None if point is None else _f64(point)
        _check(lib().ffcu_point_constants(self._h, None if p is None else _dp(p), _dp(row)))
        return row

    def coef_derivatives(self, param, point=None):
        """d coef_c / d theta[param] for every plan term (host logic of the gradient pass)."""
        terms, _, _ = self.plan()
        out = np.empty(len(terms))
        p = None if point is None else _f64(point)
        j = self.param_names.index(param) if isinstance(param, str) else int(param)
        _check(lib().ffcu_coef_derivatives(self._h, None if p is None else _dp(p), j, _dp(out)))
        return out

    def extended_terms(self, points, n_events):
        pts = _f64(np.atleast_2d(points))
        out = np.empty(pts.shape[0])
        _check(lib().ffcu_extended_terms(self._h, _dp(pts), pts.shape[0], float(n_events), _dp(out)))
        return out


class DataSet:
    """SoA fp64 event columns resident in HBM (reference DataSet, dataset.hpp:20-51)."""

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep  # objects whose memory a view aliases

    @classmethod
    def from_columns(cls, columns: dict) -> "DataSet":
        names = list(columns)
        cols = [_f64(columns[n]) for n in names]
        n = len(cols[0]) if cols else 0
        if any(len(c) != n for c in cols):
            raise FfitError(USAGE, "columns have unequal lengths")
        cn = (CP * len(names))(*[s.encode() for s in names])
        cp = (DP * len(cols))(*[_dp(c) for c in cols])
        h = VP()
        _check(lib().ffcu_dataset_from_host(cn, cp, len(names), n, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, columns: dict, device: int | None = None) -> "DataSet":
        """Zero-copy view over device tensors (torch tensors: anything with data_ptr(),
        dtype, device, numel() and is_contiguous()).  Every column must be a contiguous
        float64 CUDA tensor of the same length, all on one device (the view's device;
        `device`, if given, must agree) -- the kernels read n doubles from each pointer."""
        names = list(columns)
        tensors = [columns[n] for n in names]
        if not tensors:
            raise FfitError(USAGE, "from_device needs at least one column")
        n = int(tensors[0].numel())
        devs = set()
        for name, t in zip(names, tensors):
            dt = str(getattr(t, "dtype", ""))
            if dt not in ("torch.float64", "float64"):
                raise FfitError(USAGE, f"column {name!r}: dtype {dt or type(t).__name__}, expected float64")
            dev = getattr(t, "device", None)
            if dev is None or getattr(dev, "type", None) != "cuda":
                raise FfitError(USAGE, f"column {name!r} is not on a CUDA device ({dev})")
            if not t.is_contiguous():
                raise FfitError(USAGE, f"column {name!r} is not contiguous (a strided view?)")
            if int(t.numel()) != n:
                raise FfitError(USAGE, f"column {name!r} has {int(t.numel())} rows, expected {n}")
            devs.add(dev.index if dev.index is not None else 0)
        if len(devs) != 1:
            raise FfitError(USAGE, f"columns span several devices: {sorted(devs)}")
        tdev = devs.pop()
        if device is not None and int(device) != tdev:
            raise FfitError(USAGE, f"device={device} but the columns live on cuda:{tdev}")
        cn = (CP * len(names))(*[s.encode() for s in names])
        cp = (VP * len(names))(*[t.data_ptr() for t in tensors])
        h = VP()
        _check(lib().ffcu_dataset_from_device(cn, cp, len(names), n, tdev, ctypes.byref(h)))
        return cls(h, keep=tensors)

    @classmethod
    def load_soa(cls, path: str):
        """HBM dataset from an .ffsoa file (pinned, chunked, overlapped upload).  Returns
        (dataset, seconds)."""
        h = VP()
        sec = ctypes.c_double()
        _check(lib().ffcu_dataset_load_soa(str(path).encode(), ctypes.byref(h), ctypes.byref(sec)))
        return cls(h), sec.value

    def save_soa(self, path: str):
        _check(lib().ffcu_dataset_save_soa(self._h, str(path).encode()))

    @classmethod
    def sample(cls, model: Model, n: int, seed: int):
        h = VP()
        eff = ctypes.c_double()
        _check(lib().ffit_sample(model.handle, n, seed, ctypes.byref(h), ctypes.byref(eff)))
        return cls(h), eff.value

    @classmethod
    def read_csv(cls, model: Model, path: str):
        h = VP()
        dropped = ctypes.c_long()
        _check(lib().ffit_dataset_read_csv(model.handle, path.encode(), ctypes.byref(h), ctypes.byref(dropped)))
        return cls(h), dropped.value

    def write_csv(self, path):
        _check(lib().ffit_dataset_write_csv(self._h, path.encode()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib().ffit_dataset_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n_rows(self):
        return int(lib().ffit_dataset_rows(self._h))

    def __len__(self):
        return self.n_rows

    @property
    def names(self):
        L = lib()
        return [L.ffcu_dataset_column_name(self._h, i).decode() for i in range(L.ffcu_dataset_ncols(self._h))]

    def column(self, name) -> np.ndarray:
        out = np.empty(self.n_rows)
        _check(lib().ffcu_dataset_download(self._h, self.names.index(name), _dp(out)))
        return out

    def copy_from_host(self, columns: dict):
        cols = [_f64(columns[n]) for n in self.names]
        cp = (DP * len(cols))(*[_dp(c) for c in cols])
        _check(lib().ffcu_dataset_copy_from_host(self._h, cp))

    def copy_from_host_async(self, columns: dict, stream_ptr):
        """Asynchronous refill on a CUDA stream (cudaStream_t as an int).  The columns must be
        C-contiguous float64 arrays (pinned for a real overlap) that stay alive until the copy
        has completed on that stream."""
        cols = [columns[n] for n in self.names]
        for c in cols:
            if not (isinstance(c, np.ndarray) and c.dtype == np.float64 and c.flags.c_contiguous):
                raise FfitError(1, "copy_from_host_async needs C-contiguous float64 columns")
        cp = (DP * len(cols))(*[_dp(c) for c in cols])
        _check(lib().ffcu_dataset_copy_from_host_async(self._h, cp, VP(stream_ptr)))

    def slice(self, begin, end) -> "DataSet":
        h = VP()
        _check(lib().ffcu_dataset_slice(self._h, begin, end, ctypes.byref(h)))
        return DataSet(h, keep=self)


@dataclass
class NllValue:
    """proj/include/ffit/eval.hpp:14-21"""
    value: float = 0.0
    n_entries: int = 0
    n_evaluations: int = 0
    first_invalid: int = -1


def nll(model: Model, ds: DataSet, mode: EvalMode = EvalMode.Gpu) -> NllValue:
    """Reference ffit::nll (proj/src/eval.cpp:165-172) on the GPU.

    Every mode runs the fused kernel (Scalar == BatchPrecise bitwise, as in the reference);
    first_invalid comes from the multi-point entry (same launch)."""
    if int(mode) not in tuple(EvalMode):
        raise FfitError(1, "unknown evaluation mode")
    vals, bad, launches = nll_points(model, ds, model.theta()[None, :])
    return NllValue(float(vals[0]), ds.n_rows, int(launches), int(bad[0]))


def nll_c(model: Model, ds: DataSet, mode: EvalMode = EvalMode.Gpu):
    """ffit_nll exactly as the reference C ABI exposes it: (value, n_evaluations)."""
    v = ctypes.c_double()
    ne = ctypes.c_ulonglong()
    _check(lib().ffit_nll(model.handle, ds.handle, int(mode), ctypes.byref(v), ctypes.byref(ne)))
    return v.value, ne.value


def nll_points(model: Model, ds: DataSet, points):
    """NLL at P parameter points (rows over model.param_names) in one launch.
    Returns (values[P], first_invalid[P], kernel launches)."""
    pts = _f64(np.atleast_2d(points))
    P = pts.shape[0]
    vals = np.empty(P)
    bad = np.empty(P, dtype=np.int64)
    ne = ctypes.c_ulonglong()
    _check(lib().ffcu_nll_points(model.handle, ds.handle, _dp(pts), P, _dp(vals),
                                 bad.ctypes.data_as(ctypes.POINTER(LL)), ctypes.byref(ne)))
    return vals, bad, ne.value


def nll_grad(model: Model, ds: DataSet, points=None):
    """NLL and dNLL/dtheta (all parameters, 0 for constant ones) at P points in one
    fused pass over the events.  points=None: the current values.  Returns
    (values[P], grads[P, npar], first_invalid[P], kernel launches)."""
    if points is None:
        points = model.theta()
    pts = _f64(np.atleast_2d(points))
    P = pts.shape[0]
    vals = np.empty(P)
    grads = np.empty((P, pts.shape[1]))
    bad = np.empty(P, dtype=np.int64)
    ne = ctypes.c_ulonglong()
    _check(lib().ffcu_nll_grad(model.handle, ds.handle, _dp(pts), P, _dp(vals), _dp(grads),
                               bad.ctypes.data_as(ctypes.POINTER(LL)), ctypes.byref(ne)))
    return vals, grads, bad, ne.value


def grad_slot_count(model: Model) -> int:
    n = ctypes.c_int()
    _check(lib().ffcu_grad_slot_count(model.handle, ctypes.byref(n)))
    return n.value


def nll_grad_partial(model: Model, ds: DataSet, points):
    """Uncombined per-slot Neumaier pairs (P x nslots x 2) of the gradient pass."""
    pts = _f64(np.atleast_2d(points))
    P = pts.shape[0]
    sc = np.empty((P, grad_slot_count(model), 2))
    bad = np.empty(P, dtype=np.int64)
    _check(lib().ffcu_nll_grad_partial(model.handle, ds.handle, _dp(pts), P, _dp(sc),
                                       bad.ctypes.data_as(ctypes.POINTER(LL)), None))
    return sc, bad


def nll_grad_finish(model: Model, points, slot_sums, n_events: float):
    """Host finish of the gradient from combined slot sums (P x nslots)."""
    pts = _f64(np.atleast_2d(points))
    sums = _f64(np.atleast_2d(slot_sums))
    P = pts.shape[0]
    vals = np.empty(P)
    grads = np.empty((P, pts.shape[1]))
    _check(lib().ffcu_nll_grad_finish(model.handle, _dp(pts), P, _dp(sums), float(n_events),
                                      _dp(vals), _dp(grads)))
    return vals, grads


def nll_points_partial(model: Model, ds: DataSet, points):
    """Uncombined Neumaier pairs (P x 2) of the event sum, for cross-rank combining."""
    pts = _f64(np.atleast_2d(points))
    P = pts.shape[0]
    sc = np.empty((P, 2))
    bad = np.empty(P, dtype=np.int64)
    _check(lib().ffcu_nll_points_partial(model.handle, ds.handle, _dp(pts), P, _dp(sc),
                                         bad.ctypes.data_as(ctypes.POINTER(LL)), None))
    return sc, bad


def nll_points_device(model: Model, ds: DataSet, points, d_sc_ptr, d_bad_ptr, stream_ptr=None,
                      upload_stream_ptr=None):
    """Async multi-point NLL into device buffers (2P doubles, P uint64) on a CUDA stream;
    upload_stream_ptr: copy the constant rows on that stream instead (a pipeline's copy stream)."""
    pts = _f64(np.atleast_2d(points))
    ne = ctypes.c_ulonglong()
    if upload_stream_ptr:
        _check(lib().ffcu_nll_points_device_upload(model.handle, ds.handle, _dp(pts), pts.shape[0],
                                                   VP(d_sc_ptr), VP(d_bad_ptr), VP(stream_ptr or 0),
                                                   VP(upload_stream_ptr), ctypes.byref(ne)))
    else:
        _check(lib().ffcu_nll_points_device(model.handle, ds.handle, _dp(pts), pts.shape[0],
                                            VP(d_sc_ptr), VP(d_bad_ptr), VP(stream_ptr or 0),
                                            ctypes.byref(ne)))
    return ne.value


def combine_shards_device(d_in_ptr, R, rows, P, d_offsets_ptr, d_out_ptr, d_bad_ptr, stream_ptr=None):
    """The sharded exchange's rank-order combine of R gathered [rows pairs | P indices] blocks."""
    _check(lib().ffcu_combine_shards_device(VP(d_in_ptr), R, rows, P, VP(d_offsets_ptr), VP(d_out_ptr),
                                            VP(d_bad_ptr), VP(stream_ptr or 0)))


def combine_pairs_device(d_in_ptr, R, P, d_out_ptr, stream_ptr=None):
    _check(lib().ffcu_combine_pairs_device(VP(d_in_ptr), R, P, VP(d_out_ptr), VP(stream_ptr or 0)))


def probabilities(model: Model, ds: DataSet, mode: EvalMode = EvalMode.Gpu, point=None) -> np.ndarray:
    """Reference ffit::probabilities (proj/src/eval.cpp:174-192) on the GPU."""
    out = np.empty(ds.n_rows)
    if point is None:
        _check(lib().ffit_probabilities(model.handle, ds.handle, int(mode), _dp(out)))
    else:
        p = _f64(point)
        _check(lib().ffcu_probabilities_at(model.handle, ds.handle, _dp(p), _dp(out)))
    return out


def eval_batch_device(model: Model, pdf: str | None, ds: DataSet, d_out_ptr, stream_ptr=None):
    """Unnormalised values of a named pdf into a device buffer (n doubles), asynchronous on
    a CUDA stream (None: the model's own stream)."""
    _check(lib().ffcu_eval_batch_device(model.handle, pdf.encode() if pdf else None, ds.handle, VP(d_out_ptr),
                                        VP(stream_ptr or 0)))


def eval_batch(model: Model, pdf: str, ds: DataSet) -> np.ndarray:
    """PdfSpec::eval_batch (proj/src/pdfs.cpp:212-269): unnormalised values of a named pdf."""
    out = np.empty(ds.n_rows)
    _check(lib().ffcu_eval_batch(model.handle, pdf.encode(), ds.handle, _dp(out)))
    return out


def normalization(model: Model, pdf: str | None = None, point=None) -> float:
    out = ctypes.c_double()
    p = None if point is None else _f64(point)
    _check(lib().ffcu_normalization(model.handle, None if pdf is None else pdf.encode(),
                                    None if p is None else _dp(p), ctypes.byref(out)))
    return out.value


def set_device_normalization(model: Model, on: bool = True) -> None:
    """Device-side numeric normalisation for this model's likelihood / probabilities /
    eval_batch calls (ffcu_model_set_device_normalization; off = the host's adaptive Simpson,
    bit-identical to the reference's)."""
    _check(lib().ffcu_model_set_device_normalization(model.handle, 1 if on else 0))


def device_normalization_enabled(model: Model) -> bool:
    return bool(lib().ffcu_model_device_normalization(model.handle))


def device_normalization(model: Model, pdf: str | None = None, points=None) -> np.ndarray:
    """The normalisation integral of a (sub-)pdf at P points by the device quadrature (the
    reference's adaptive Simpson, one warp per point); points = None: the current values."""
    if points is None:
        out = np.empty(1, dtype=np.float64)
        _check(lib().ffcu_device_normalization(model.handle, None if pdf is None else pdf.encode(), None, 1, _dp(out)))
        return out
    pts = _f64(np.atleast_2d(points))
    out = np.empty(pts.shape[0], dtype=np.float64)
    _check(lib().ffcu_device_normalization(model.handle, None if pdf is None else pdf.encode(), _dp(pts), pts.shape[0],
                                           _dp(out)))
    return out


def device_normalization_launches(model: Model) -> int:
    return int(lib().ffcu_device_normalization_launches(model.handle))


@dataclass
class FittedParameter:
    name: str
    value: float
    uncertainty: float


@dataclass
class FitResult:
    """proj/include/ffit/fit.hpp:25-33"""
    converged: bool
    nll_min: float
    parameters: list
    n_nll_calls: int
    wall_seconds: float
    uncertainties_valid: bool
    iterations: int = 0
    n_launches: int = 0
    trace: list = field(default_factory=list)
    analytic_gradient: bool = False
    edm: float = 0.0

    def value(self, name):
        return next(p.value for p in self.parameters if p.name == name)


def _result(h) -> FitResult:
    L = lib()
    try:
        params = [FittedParameter(L.ffit_result_param_name(h, i).decode(), L.ffit_result_param_value(h, i),
                                  L.ffit_result_param_uncertainty(h, i))
                  for i in range(L.ffit_result_param_count(h))]
        n = L.ffcu_result_trace(h, None, 0)
        tr = np.empty(max(n, 1))
        L.ffcu_result_trace(h, _dp(tr), n)
        return FitResult(bool(L.ffit_result_converged(h)), L.ffit_result_nll(h), params,
                         int(L.ffit_result_nll_calls(h)), L.ffit_result_wall_seconds(h),
                         bool(L.ffit_result_uncertainties_valid(h)), L.ffcu_result_iterations(h),
                         int(L.ffcu_result_launches(h)), list(tr[:n]),
                         bool(L.ffcu_result_analytic_gradient(h)), float(L.ffcu_result_edm(h)))
    finally:
        L.ffit_result_free(h)


def fit_to(model: Model, ds: DataSet, mode: EvalMode = EvalMode.Gpu, tolerance=0.0, max_iterations=0) -> FitResult:
    """Reference fit_to (proj/src/fit.cpp:86-251): Nelder-Mead, batched GPU points."""
    h = VP()
    _check(lib().ffit_fit(model.handle, ds.handle, int(mode), tolerance, max_iterations, ctypes.byref(h)))
    return _result(h)


def fit_gradient(model: Model, ds: DataSet, tolerance=0.0, max_iterations=0, analytic=None) -> FitResult:
    """Minuit-style BFGS.  analytic=True: gradients from the fused NLL + gradient pass
    (one point per iteration) when the model's layout fits it; False: central
    differences, 2d+1 points per launch; None: automatic (analytic, except for models
    with Expression pdfs whose formula-specialised builds make differences faster)."""
    h = VP()
    flag = -1 if analytic is None else (1 if analytic else 0)
    _check(lib().ffcu_fit_gradient_opts(model.handle, ds.handle, tolerance, max_iterations, flag,
                                        ctypes.byref(h)))
    return _result(h)


def last_launch(model: Model) -> dict:
    info = (ctypes.c_int * 6)()
    _check(lib().ffcu_last_launch(model.handle, info))
    return dict(zip(("threads", "events_per_thread", "tile", "ntiles", "nchunks", "grid"), list(info)))


def kernel_timer(enable: bool):
    _check(lib().ffcu_kernel_timer(1 if enable else 0))


def kernel_timer_read():
    """(summed ms, launches) of the fused NLL kernel since the last read."""
    ms = ctypes.c_double()
    cnt = ctypes.c_ulonglong()
    _check(lib().ffcu_kernel_timer_read(ctypes.byref(ms), ctypes.byref(cnt)))
    return ms.value, cnt.value


def kernel_launches() -> int:
    return int(lib().ffcu_kernel_launches())


def fp64_peak():
    """Measured FP64 FMA instructions/s on the current device (and the ms it took)."""
    v = ctypes.c_double()
    ms = ctypes.c_float()
    _check(lib().ffcu_fp64_peak(ctypes.byref(v), ctypes.byref(ms)))
    return v.value, ms.value


def fp64_issue_probe(others_per_8: int) -> float:
    """FP64 FMA instructions/s with `others_per_8` integer multiply-adds issued per eight DFMAs."""
    v = ctypes.c_double()
    _check(lib().ffcu_fp64_issue_probe(int(others_per_8), ctypes.byref(v)))
    return v.value


def math_probe(which: str, x) -> np.ndarray:
    """The fused kernel's device exp ("exp") or log ("log") over an array (test hook)."""
    x = _f64(x)
    out = np.empty_like(x)
    _check(lib().ffcu_math_probe({"exp": 0, "log": 1, "sqrt": 2, "rsqrt_seed": 3}[which], _dp(x), _dp(out), len(x)))
    return out


def sample_host(model: Model, n: int, seed: int):
    """Seeded generator into host arrays, one per observable (name -> array)."""
    names = model.observables
    cols = [np.empty(n) for _ in names]
    cp = (DP * len(cols))(*[_dp(c) for c in cols])
    eff = ctypes.c_double()
    _check(lib().ffcu_sample_host(model.handle, n, seed, cp, ctypes.byref(eff)))
    return dict(zip(names, cols)), eff.value


def expr_eval(text: str, variables, values) -> np.ndarray:
    """The Expression formula language on the host: compile `text` over `variables` and
    evaluate it at rows of values (npts x nvars) -- the per-event semantics the device
    interpreter follows (proj/docs/expression-grammar.md)."""
    vals = np.asarray(values, dtype=np.float64)
    if vals.ndim == 1:
        vals = vals[None, :]
    npts = vals.shape[0]
    buf = _f64(vals.reshape(-1)) if vals.size else np.zeros(1)
    arr = (CP * max(len(variables), 1))(*[v.encode() for v in variables])
    out = np.empty(max(npts, 1))
    _check(lib().ffcu_expr_eval(text.encode(), arr, len(variables), _dp(buf), npts, _dp(out)))
    return out[:npts]


def write_soa(path: str, columns: dict):
    """Write host columns (name -> 1-D float64 array) as an .ffsoa file."""
    names = list(columns)
    cols = [_f64(columns[n]) for n in names]
    n = len(cols[0]) if cols else 0
    if any(len(c) != n for c in cols):
        raise FfitError(USAGE, "columns have unequal lengths")
    cn = (CP * len(names))(*[s.encode() for s in names])
    cp = (DP * len(cols))(*[_dp(c) for c in cols])
    _check(lib().ffcu_soa_write(str(path).encode(), cn, cp, len(names), n))


def read_soa_host(path: str) -> dict:
    """Host columns of an .ffsoa file (checksums verified)."""
    nc, nr = ctypes.c_int(), LL()
    _check(lib().ffcu_soa_info(str(path).encode(), ctypes.byref(nc), ctypes.byref(nr)))
    names = []
    for i in range(nc.value):
        buf = ctypes.create_string_buffer(4096)
        _check(lib().ffcu_soa_column_name(str(path).encode(), i, buf, 4096))
        names.append(buf.value.decode())
    cols = [np.empty(nr.value) for _ in names]
    cp = (DP * len(cols))(*[_dp(c) if c.size else _dp(np.empty(1)) for c in cols])
    _check(lib().ffcu_soa_read_host(str(path).encode(), cp))
    return dict(zip(names, cols))


def expression_jit(enable=None) -> bool:
    """Formula-specialised (NVRTC) builds for Expression pdfs: query (None) or set; returns
    the previous setting."""
    return bool(lib().ffcu_expression_jit(-1 if enable is None else (1 if enable else 0)))


def expression_jit_status() -> str:
    return lib().ffcu_expression_jit_status().decode()


def expression_jit_source(model: Model, compile: bool = False, points=None) -> str:
    """The generated straight-line formula code of a model (compile=True also NVRTC-compiles
    the kernels around it; host only).  With `points` (P x n_params): the code of a launch
    over them, launch-constant formula subtrees cached per tile."""
    buf = ctypes.create_string_buffer(1 << 20)
    if points is None:
        _check(lib().ffcu_expression_jit_source(model.handle, 1 if compile else 0, buf, 1 << 20))
    else:
        pts = _f64(np.atleast_2d(points))
        _check(lib().ffcu_expression_jit_source_points(model.handle, _dp(pts), pts.shape[0], 1 if compile else 0,
                                                       buf, 1 << 20))
    return buf.value.decode()


def last_launch_jit(model: Model) -> int:
    """0: static kernels, 1: formula-specialised build, 2: plan-specialised build."""
    return int(lib().ffcu_last_launch_jit(model.handle))


def plan_spec_min_work(v: float = -2.0) -> float:
    """Event-point threshold of the plan-specialised builds (-1: off); returns the old one."""
    return float(lib().ffcu_plan_spec_min_work(float(v)))


def plan_spec_source(model: Model, points=None, compile: bool = False) -> str:
    """The plan-specialised likelihood source for a launch over `points` (compile: also
    NVRTC-compile it; no GPU needed)."""
    buf = ctypes.create_string_buffer(1 << 16)
    if points is None:
        _check(lib().ffcu_plan_spec_source(model.handle, None, 0, 1 if compile else 0, buf, len(buf)))
    else:
        pts = _f64(np.atleast_2d(points))
        _check(lib().ffcu_plan_spec_source(model.handle, _dp(pts), pts.shape[0], 1 if compile else 0, buf,
                                           len(buf)))
    return buf.value.decode()


def last_launch_cached(model: Model) -> int:
    """Terms of the last likelihood launch served by the launch-constant branch cache."""
    return int(lib().ffcu_last_launch_cached(model.handle))


def grad_spec_source(model: Model, compile_ks=None) -> str:
    """The plan-specialised gradient pass's generated spec (compile_ks = 0/1/2: also
    NVRTC-compile the kernel for that leaf-kind set; host only)."""
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib().ffcu_grad_spec_source(model.handle, -1 if compile_ks is None else int(compile_ks), buf, 1 << 16))
    return buf.value.decode()


def last_grad_jit(model: Model) -> bool:
    return bool(lib().ffcu_last_grad_jit(model.handle))


class ShardGroup:
    """The event-sharded likelihood of the C ABI (ffcu_shard_group_*, csrc/shard.hpp): one
    fused launch per rank and ONE NCCL all-gather per batch of points, combined in rank order
    on the device.  Two ways to build one:

    * ``ShardGroup.for_rank(model, shard, n_total, offset, world, rank, broadcast)`` -- one
      process per GPU; ``broadcast(obj)`` hands rank 0's NCCL id to every rank (e.g. via
      ``torch.distributed.broadcast_object_list``);
    * ``ShardGroup.local(model, columns, devices)`` -- one process, several devices.

    Every rank calls every method with the same points (collective); values are identical on
    every rank.  Import torch before the first group when both share a process (one NCCL)."""

    def __init__(self, handle, model, keep=None):
        self._h = handle
        self.model = model
        self._keep = keep

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().ffcu_nccl_unique_id(buf))
        return buf.raw

    @staticmethod
    def nccl_version() -> str:
        return lib().ffcu_nccl_version().decode()

    @classmethod
    def for_rank(cls, model: Model, shard: DataSet, n_total: int, offset: int, world: int, rank: int,
                 broadcast=None, nccl_id: bytes | None = None) -> "ShardGroup":
        if nccl_id is None:
            nid = cls.nccl_unique_id() if rank == 0 else None
            nccl_id = broadcast(nid) if broadcast is not None else nid
        if nccl_id is None or len(nccl_id) != 128:
            raise FfitError(USAGE, "a 128-byte NCCL id is required on every rank")
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        h = VP()
        _check(lib().ffcu_shard_group_create_rank(model.handle, shard.handle, int(n_total), int(offset), buf,
                                                  int(world), int(rank), ctypes.byref(h)))
        return cls(h, model, keep=shard)

    @classmethod
    def local(cls, model: Model, columns: dict, devices) -> "ShardGroup":
        names = model.observables
        cols = [_f64(columns[n]) for n in names]
        n = len(cols[0])
        if any(len(c) != n for c in cols):
            raise FfitError(USAGE, "columns have unequal lengths")
        cn = (CP * len(names))(*[s.encode() for s in names])
        cp = (DP * len(cols))(*[_dp(c) for c in cols])
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        h = VP()
        _check(lib().ffcu_shard_group_create_local(model.handle, cn, cp, len(names), n, devs, len(devices),
                                                   ctypes.byref(h)))
        return cls(h, model)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib().ffcu_shard_group_free(h)
            self._h = None

    def info(self) -> dict:
        w, nl = ctypes.c_int(), ctypes.c_int()
        nt, lr, lo = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_longlong()
        _check(lib().ffcu_shard_group_info(self._h, ctypes.byref(w), ctypes.byref(nl), ctypes.byref(nt),
                                           ctypes.byref(lr), ctypes.byref(lo)))
        return {"world": w.value, "local_devices": nl.value, "n_total": nt.value, "local_rows": lr.value,
                "local_offset": lo.value}

    def nll_points(self, points):
        """(values[P], first_invalid[P], launches) over all ranks' events."""
        pts = _f64(np.atleast_2d(points))
        P = pts.shape[0]
        vals = np.empty(P)
        bad = np.empty(P, dtype=np.int64)
        ne = ctypes.c_ulonglong()
        _check(lib().ffcu_shard_group_nll_points(self._h, _dp(pts), P, _dp(vals),
                                                 bad.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)),
                                                 ctypes.byref(ne)))
        return vals, bad, ne.value

    def nll_points_device(self, points, d_sc_ptr, d_bad_ptr, stream_ptr=None, upload_stream_ptr=None) -> int:
        """Async on a CUDA stream: combined pairs (2P doubles, no extended term) and global
        first-invalid indices (P uint64) into device buffers; upload_stream_ptr: copy the
        constant rows on that stream (a pipeline's copy stream)."""
        pts = _f64(np.atleast_2d(points))
        ne = ctypes.c_ulonglong()
        _check(lib().ffcu_shard_group_nll_points_device(self._h, _dp(pts), pts.shape[0], VP(d_sc_ptr),
                                                        VP(d_bad_ptr), VP(stream_ptr or 0),
                                                        VP(upload_stream_ptr or 0), ctypes.byref(ne)))
        return ne.value

    def nll_grad(self, points):
        """(values[P], grads[P, npar], first_invalid[P], launches) over all ranks' events."""
        pts = _f64(np.atleast_2d(points))
        P = pts.shape[0]
        npar = len(self.model.param_names)
        vals = np.empty(P)
        grads = np.empty((P, npar))
        bad = np.empty(P, dtype=np.int64)
        ne = ctypes.c_ulonglong()
        _check(lib().ffcu_shard_group_nll_grad(self._h, _dp(pts), P, _dp(vals), _dp(grads),
                                               bad.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)),
                                               ctypes.byref(ne)))
        return vals, grads, bad, ne.value

    def fit(self, tolerance=0.0, max_iterations=0) -> "FitResult":
        """The reference's Nelder-Mead on the sharded likelihood (fitted values -> model)."""
        h = VP()
        _check(lib().ffcu_shard_group_fit(self._h, tolerance, max_iterations, ctypes.byref(h)))
        return _result(h)

    def fit_gradient(self, tolerance=0.0, max_iterations=0, analytic=None) -> "FitResult":
        """Minuit-style BFGS on the sharded likelihood (as fit_gradient)."""
        h = VP()
        flag = -1 if analytic is None else (1 if analytic else 0)
        _check(lib().ffcu_shard_group_fit_gradient(self._h, tolerance, max_iterations, flag, ctypes.byref(h)))
        return _result(h)
