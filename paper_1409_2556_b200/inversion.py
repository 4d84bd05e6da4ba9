"""Python mirror of the reference's geostatistical inversion API (inversion.hpp:17-91) over the
C ABI (lt_gn_step / lt_gn_invert / lt_gn_objective): the Gauss-Newton consumer of J on the
device (csrc/gn.cu).

The prior is the reference's dense Q or `GridPrior`, a stationary exponential covariance per
parameter block on the FD grid (applied exactly by FFT on the device).  The forward handles
are Python callables: predict(s) -> h, and jacobian_and_predict(s) -> (J, h) with J a NumPy
array (copied to the device) or `tht_handles(model)`, whose Jacobian is written straight into
the device buffer by lt_jacobian_slice.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Union

import numpy as np

from . import capi
from .capi import check, dptr, lib
from .laptomo import Context, Grid, ThtForwardModel, default_context


@dataclass
class GridPrior:
    """Q = blockdiag_b variance[b] exp(-|(dx/l0, dy/l1[, dz/l2])|) over the cells of `grid`."""

    grid: Grid
    variances: Sequence[float]
    corr_lengths: Sequence[Sequence[float]]


@dataclass
class InversionProblem:
    """inversion.hpp:17-27."""

    y: np.ndarray
    r_diag: np.ndarray
    drift: np.ndarray                 # X, n_s x p
    prior: Union[np.ndarray, GridPrior]
    predict: Callable
    jacobian_and_predict: Callable    # s -> (J, h), or a DeviceJacobian


@dataclass
class GnOptions:
    max_gn: int = 15
    rtol: float = 1e-3
    damping: bool = True
    max_halvings: int = 5

    def c(self):
        return capi.LtGnOptions(int(self.max_gn), float(self.rtol), int(self.damping), int(self.max_halvings))


@dataclass
class GnIterate:
    s: np.ndarray
    beta: np.ndarray
    xi: np.ndarray
    objective: float
    misfit: float
    prior: float
    step_norm: float
    alpha: float
    saddle_residual: float
    drift_violation: float


@dataclass
class InversionResult:
    s_hat: np.ndarray
    beta_hat: np.ndarray
    history: List[dict]
    converged: bool
    stop_reason: str


class DeviceJacobian:
    """A jacobian_and_predict handle that writes J into the library's device buffer itself:
    fn(s, J_device_pointer) -> h."""

    def __init__(self, fn):
        self.fn = fn


_cudart = None


def _h2d(dst_ptr: int, src: np.ndarray):
    global _cudart
    if _cudart is None:
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                _cudart = C.CDLL(name)
                break
            except OSError:
                continue
    src = np.ascontiguousarray(src, dtype=np.float64)
    rc = _cudart.cudaMemcpy(C.c_void_p(dst_ptr), src.ctypes.data_as(C.c_void_p), C.c_size_t(src.nbytes), 1)
    if rc != 0:
        raise RuntimeError(f"cudaMemcpy H2D failed ({rc})")


class GaussNewtonSolver:
    """inversion.hpp:51-79 on the device."""

    def __init__(self, problem: InversionProblem, ctx: Optional[Context] = None):
        self.problem = problem
        self.ctx = ctx or default_context()
        pb = problem
        self._y = np.ascontiguousarray(np.asarray(pb.y, dtype=np.float64))
        self._r = np.ascontiguousarray(np.asarray(pb.r_diag, dtype=np.float64))
        X = np.asarray(pb.drift, dtype=np.float64)
        self.n_s, self.p = X.shape
        self._X = np.ascontiguousarray(X.T)  # column-major n_s x p
        self._err = None
        s = capi.LtGnProblem()
        s.n_y, s.n_s, s.p = self._y.size, self.n_s, self.p
        s.y, s.r_diag = dptr(self._y), dptr(self._r)
        s.drift = dptr(self._X) if self.p else None
        if isinstance(pb.prior, GridPrior):
            s.prior = None
            s.grid = pb.prior.grid.c()
            s.n_blocks = len(pb.prior.variances)
            for b, (v, l) in enumerate(zip(pb.prior.variances, pb.prior.corr_lengths)):
                s.variance[b] = float(v)
                for d in range(len(l)):
                    s.corr[b][d] = float(l[d])
        else:
            self._Q = np.ascontiguousarray(np.asarray(pb.prior, dtype=np.float64))
            s.prior = dptr(self._Q)

        def predict(user, sp, hp):
            try:
                h = np.asarray(pb.predict(np.ctypeslib.as_array(sp, (self.n_s,)).copy()), dtype=np.float64)
                np.ctypeslib.as_array(hp, (self._y.size,))[:] = h
                return 0
            except Exception as e:  # noqa: BLE001
                self._err = e
                return capi.LT_ERR_INTERNAL

        def jac(user, sp, jptr, hp):
            try:
                sv = np.ctypeslib.as_array(sp, (self.n_s,)).copy()
                if isinstance(pb.jacobian_and_predict, DeviceJacobian):
                    h = pb.jacobian_and_predict.fn(sv, int(jptr))
                else:
                    J, h = pb.jacobian_and_predict(sv)
                    _h2d(int(jptr), np.asarray(J))
                np.ctypeslib.as_array(hp, (self._y.size,))[:] = np.asarray(h, dtype=np.float64)
                return 0
            except Exception as e:  # noqa: BLE001
                self._err = e
                return capi.LT_ERR_INTERNAL

        self._pfn = capi.PREDICT_FN(predict)
        self._jfn = capi.JACOBIAN_FN(jac)
        s.predict, s.jacobian_and_predict = self._pfn, self._jfn
        self._c = s

    def _check(self, status):
        if status != capi.LT_OK and self._err is not None:
            e, self._err = self._err, None
            raise e
        check(status)

    def step(self, s, beta, options: GnOptions = GnOptions()) -> GnIterate:
        s = np.ascontiguousarray(np.asarray(s, dtype=np.float64))
        beta = np.ascontiguousarray(np.asarray(beta, dtype=np.float64))
        so, bo, xo = np.zeros(self.n_s), np.zeros(self.p), np.zeros(self._y.size)
        st = capi.LtGnStats()
        o = options.c()
        self._check(lib().lt_gn_step(self.ctx.handle, C.byref(self._c), dptr(s), dptr(beta) if self.p else None,
                                     C.byref(o), dptr(so), dptr(bo) if self.p else None, dptr(xo), C.byref(st)))
        return GnIterate(so, bo, xo, st.objective, st.misfit, st.prior, st.step_norm, st.alpha, st.saddle_residual,
                         st.drift_violation)

    def invert(self, s0, beta0, options: GnOptions = GnOptions()) -> InversionResult:
        s0 = np.ascontiguousarray(np.asarray(s0, dtype=np.float64))
        beta0 = np.ascontiguousarray(np.asarray(beta0, dtype=np.float64))
        sh, bh = np.zeros(self.n_s), np.zeros(self.p)
        hist = (capi.LtGnStats * max(options.max_gn, 1))()
        steps, conv = C.c_int(), C.c_int()
        reason = C.create_string_buffer(256)
        o = options.c()
        self._check(lib().lt_gn_invert(self.ctx.handle, C.byref(self._c), dptr(s0), dptr(beta0) if self.p else None,
                                       C.byref(o), dptr(sh), dptr(bh) if self.p else None, hist, C.byref(steps),
                                       C.byref(conv), reason, 256))
        h = [{f: getattr(hist[k], f) for f, _ in capi.LtGnStats._fields_} for k in range(steps.value)]
        return InversionResult(sh, bh, h, bool(conv.value), reason.value.decode())

    def objective(self, s, beta):
        s = np.ascontiguousarray(np.asarray(s, dtype=np.float64))
        beta = np.ascontiguousarray(np.asarray(beta, dtype=np.float64))
        o, m, p = C.c_double(), C.c_double(), C.c_double()
        self._check(lib().lt_gn_objective(self.ctx.handle, C.byref(self._c), dptr(s), dptr(beta) if self.p else None,
                                          C.byref(o), C.byref(m), C.byref(p)))
        return o.value, m.value, p.value


def tht_handles(model: ThtForwardModel):
    """predict / jacobian_and_predict of a ThtForwardModel over s = [ln kappa; ln S] (both blocks
    when the experiment includes storativity, else ln kappa with the model's ln S), rows in
    time-major order (t, s, r): the Jacobian slices go straight into the device buffer."""
    ex = model.experiment
    n = ex.grid.n_cells
    both = ex.include_storativity
    pairs = len(ex.sources) * len(ex.receivers)
    nt = len(ex.times)
    n_param = 2 * n if both else n

    def split(s):
        return (s[:n], s[n:]) if both else (s, model.log_storativity)

    def order(pred):  # (s r) t  ->  t (s r)
        return np.asarray(pred).reshape(pairs, nt).T.ravel()

    def predict(s):
        lk, ls = split(s)
        return order(model.predict_with(lk, ls))

    def jac(s, jptr):
        lk, ls = split(s)
        pencil = model.pencil(lk, ls)
        exc, keep = ex.c()
        h = np.zeros(nt * pairs)
        pred = np.zeros(pairs)
        for t in range(nt):
            check(lib().lt_jacobian_slice(pencil.handle, C.byref(exc), t, capi.LT_MEM_DEVICE,
                                          C.cast(jptr + 8 * t * pairs * n_param, capi.PD), dptr(pred)))
            h[t * pairs:(t + 1) * pairs] = pred
        pencil.close()
        return h

    return predict, DeviceJacobian(jac), order
