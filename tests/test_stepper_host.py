"""The numpy branch of stepper.rk4_step (in-place stage updates) is bitwise the reference's
expressions (assemble.py:105-114: res = a res + dt rhs; y = y + b res), input untouched."""
import numpy as np

from paper_0901_1024_b200.stepper import RK_A, RK_B, RK_C, rk4_step


def _reference_form(state, t, dt, fn):
    y = np.array(state, dtype=np.float64, copy=True)
    res = np.zeros_like(y)
    for a, b, c in zip(RK_A, RK_B, RK_C):
        res = a * res + dt * np.asarray(fn(t + c * dt, y))
        y = y + b * res
    return y


def test_rk4_step_numpy_bitwise_reference_form():
    rng = np.random.default_rng(7)
    y0 = rng.normal(size=(6, 40, 20))
    keep = y0.copy()
    m = rng.normal(size=(20, 20))

    def fn(t, y):
        return 0.1 * (y @ m) + np.sin(t)

    got = rk4_step(y0, 0.25, 0.01, fn)
    assert np.array_equal(got, _reference_form(y0, 0.25, 0.01, fn))
    assert np.array_equal(y0, keep)


def test_rk4_step_float32_rhs_keeps_reference_promotion():
    rng = np.random.default_rng(8)
    y0 = rng.normal(size=(6, 8, 10))

    def fn(t, y):
        return (0.5 * y).astype(np.float32)

    assert np.array_equal(rk4_step(y0, 0.0, 0.02, fn), _reference_form(y0, 0.0, 0.02, fn))


def test_rk4_step_threaded_path_bitwise(monkeypatch):
    """Large states take torch's multi-threaded CPU kernels: still the reference's bits."""
    import paper_0901_1024_b200.stepper as st

    monkeypatch.setattr(st, "_THREADED_MIN", 1)
    rng = np.random.default_rng(9)
    y0 = rng.normal(size=(6, 300, 35))
    m = rng.normal(size=(35, 35))

    def fn(t, y):
        return 0.05 * (y @ m) - 0.3 * np.cos(t) * y

    assert np.array_equal(st.rk4_step(y0, 0.1, 0.003, fn), _reference_form(y0, 0.1, 0.003, fn))
