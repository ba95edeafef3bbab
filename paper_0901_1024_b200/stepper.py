"""Five-stage, fourth-order low-storage Runge-Kutta (Carpenter & Kennedy).

Coefficients and update order are the reference's (assemble.py:80-114):

    res = a_s * res + dt * rhs(t + c_s dt, y);   y = y + b_s * res

``rk4_step`` keeps the reference's generic signature and semantics (copies its
input, ValueError for dt <= 0) but works on torch tensors in place on the
device as well as on numpy arrays; the operator's fused path
(``B200MaxwellOperator.advance``) performs the same arithmetic inside the
stage kernel.
"""

from __future__ import annotations

import numpy as np

RK_A = (
    0.0,
    -567301805773.0 / 1357537059087.0,
    -2404267990393.0 / 2016746695238.0,
    -3550918686646.0 / 2091501179385.0,
    -1275806237668.0 / 842570457699.0,
)
RK_B = (
    1432997174477.0 / 9575080441755.0,
    5161836677717.0 / 13612068292357.0,
    1720146321549.0 / 2090206949498.0,
    3134564353537.0 / 4481467310338.0,
    2277821191437.0 / 14882151754819.0,
)
RK_C = (
    0.0,
    1432997174477.0 / 9575080441755.0,
    2526269341429.0 / 6820363962896.0,
    2006345519317.0 / 3224310063776.0,
    2802321613138.0 / 2924317926251.0,
)


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def rk4_step(state, t: float, dt: float, rhs_fn):
    """Advance one LSRK4 step; storage is the state plus one residual register.

    numpy input: float64 copy, as the reference (assemble.py:109).  torch
    input: a clone of the same dtype/device, so device states never leave HBM.
    """
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    if _is_torch(state):
        y = state.clone()
        res = None
        for a, b, c in zip(RK_A, RK_B, RK_C):
            k = rhs_fn(t + c * dt, y)
            res = dt * k if res is None else a * res + dt * k
            y = y + b * res
        return y
    y = np.array(state, dtype=np.float64, copy=True)
    res = np.zeros_like(y)
    tmp = np.empty_like(y)
    for a, b, c in zip(RK_A, RK_B, RK_C):
        k = np.asarray(rhs_fn(t + c * dt, y))
        if k.dtype != np.float64 or k.shape != y.shape:  # the reference's expressions, verbatim semantics
            res = a * res + dt * k
            y = y + b * res
            continue
        # the same roundings in place (fl(fl(a res) + fl(dt k)), fl(y + fl(b res))): no 6 K Np temporaries
        # per stage -- the state passed to rhs_fn is updated in place after it returns.  Large states go
        # through torch's CPU kernels on zero-copy views (all host cores; elementwise, so the same bits).
        if y.size >= _THREADED_MIN and _torch_cpu() is not None:
            th = _torch_cpu()
            ty, tr, tt, tk = th.from_numpy(y), th.from_numpy(res), th.from_numpy(tmp), th.from_numpy(np.ascontiguousarray(k))
            th.mul(tk, dt, out=tt)
            tr.mul_(a)
            tr.add_(tt)
            th.mul(tr, b, out=tt)
            ty.add_(tt)
            continue
        np.multiply(k, dt, out=tmp)
        np.multiply(res, a, out=res)
        res += tmp
        np.multiply(res, b, out=tmp)
        y += tmp
    return y


_THREADED_MIN = 1 << 22  # elements (32 MB of float64) from which the stage update runs multi-threaded


def _torch_cpu():
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    return torch
