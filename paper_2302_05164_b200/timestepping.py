"""Time integration on the device-resident state.

Mirrors ``scantherm/timestepping.py``: ``run_scan_phase`` (:195-226),
``run_cooldown_phase`` (:310-370), ``InstabilityError`` (:21-32),
``PhaseStats``/``SimulationState`` (:157-183) and ``krylov_solve``
(:102-131), with the same step accounting (``n_steps = ceil(dur/dt -
1e-9)``, ``tau = (step - 1) dt``, last step clipped), the same stability
rule (|T| > 1e7 or non-finite), the same history order (update after
every accepted step) and the same Newton/PCG stopping rules.

The difference is where the loop runs: T and r_c are uploaded once, the
whole scan phase is one ``st_explicit_steps`` call (beam schedule
precomputed on the host, ``physics.flatten_schedule``), and each
backward-Euler step is one ``st_implicit_step`` call (Newton + Jacobi
PCG on the device).  When an ``on_step`` hook is given the phase falls
back to one device step per host iteration so the hook sees every state.
"""

import math
import time as _time
from dataclasses import dataclass, field

import numpy as np

from .physics import ScheduleError, flatten_schedule


class InstabilityError(RuntimeError):
    """Raised when the explicit integration diverges."""

    def __init__(self, step, t, dt, t_extreme):
        self.step = step
        self.t = t
        self.dt = dt
        self.t_extreme = t_extreme
        super().__init__(
            f"explicit step diverged at step {step} (t = {t:.6g} s, "
            f"dt = {dt:.3g} s): temperature reached {t_extreme:.3g} K; "
            f"dt exceeds the stability bound of the current mesh")


@dataclass
class PhaseStats:
    n_steps: int = 0
    dt: float = 0.0
    wall_time: float = 0.0
    t_max_seen: float = 0.0
    newton_iters: int = 0
    krylov_iters: int = 0
    dt_retries: int = 0


@dataclass
class SimulationState:
    forest: object
    dofmap: object
    op: object
    T: np.ndarray
    history: object
    time: float = 0.0
    phase_seconds: dict = field(default_factory=dict)

    def charge(self, phase, seconds):
        self.phase_seconds[phase] = self.phase_seconds.get(phase, 0.0) + seconds


_T_DIVERGED = 1.0e7


def _check_stable(T, step, t, dt):
    m = float(np.max(np.abs(T)))
    if not np.isfinite(m) or m > _T_DIVERGED:
        raise InstabilityError(step, t, dt, m)


def _scan_duration(layer_path):
    lps = layer_path if isinstance(layer_path, (list, tuple)) else [layer_path]
    return lps[0].scan_duration()


def run_scan_phase(state, layer_path, dt, on_step=None) -> PhaseStats:
    """Integrate one layer's scan with forward Euler (device-resident).

    ``layer_path`` may be a list of LayerPaths scanned concurrently."""
    op = state.op
    stats = PhaseStats(dt=dt)
    t0 = _time.perf_counter()
    duration = _scan_duration(layer_path)
    n_steps = max(0, math.ceil(duration / dt - 1e-9))
    if on_step is None and n_steps:
        dts, _ = flatten_schedule(layer_path, dt, 1)  # validates the schedule's start
        paths = layer_path if isinstance(layer_path, (list, tuple)) else [layer_path]
        for lp in paths:   # layer_beam_state raises past the layer (physics.py:150)
            if (n_steps - 1) * dt > lp.duration():
                raise ScheduleError(f"tau = {(n_steps - 1) * dt} beyond the layer duration "
                                    f"{lp.duration()}")
        dts = np.minimum(dt, duration - np.arange(n_steps, dtype=np.float64) * dt)
        op.set_state(state.T, state.history.r_c)
        # the whole layer on the device, beams evaluated there per step
        fail, ext, tmax = op.run_scan(layer_path, dt, n_steps)
        T, rc = op.get_state()
        state.T = T
        state.history.r_c[...] = rc.reshape(state.history.r_c.shape)
        if fail:
            tau = (fail - 1) * dt
            raise InstabilityError(fail, state.time + tau, float(dts[fail - 1]), ext)
        stats.t_max_seen = max(stats.t_max_seen, tmax)
    else:
        for step in range(1, n_steps + 1):
            tau = (step - 1) * dt
            dts, beams = flatten_schedule(layer_path, dt, 1, step0=step)
            state.T = op.explicit_fused_step(state.T, float(dts[0]), state.history.r_c,
                                             beams[0])
            _check_stable(state.T, step, state.time + tau, float(dts[0]))
            op.update_history(state.history, state.T)
            stats.t_max_seen = max(stats.t_max_seen, float(state.T.max()))
            if on_step is not None:
                on_step(state, step, min(step * dt, duration))
    state.time += duration
    stats.n_steps = n_steps
    stats.wall_time = _time.perf_counter() - t0
    state.charge("scan", stats.wall_time)
    return stats


def run_cooldown_phase(state, layer_path, dt_explicit, settings=None,
                       on_step=None) -> PhaseStats:
    """Explicit pre-phase, then backward Euler with the halving ladder."""
    op = state.op
    settings = settings or op.settings
    stats = PhaseStats(dt=settings.dt_implicit)
    t0 = _time.perf_counter()
    window = layer_path.cool_time
    step = 0
    op.set_state(state.T, state.history.r_c)

    n_exp = min(settings.explicit_cooldown_steps,
                max(0, math.ceil(window / dt_explicit - 1e-9)))
    if n_exp:
        dts = np.array([min(dt_explicit, window - i * dt_explicit) for i in range(n_exp)])
        if on_step is None:
            fail, ext, _ = op.run_explicit(dts, np.zeros((n_exp, 0)))
            if fail:
                T, rc = op.get_state()
                state.T = T
                state.history.r_c[...] = rc.reshape(state.history.r_c.shape)
                raise InstabilityError(fail, state.time, float(dts[fail - 1]), ext)
            step = n_exp
        else:
            for i in range(n_exp):
                fail, ext, _ = op.run_explicit(dts[i:i + 1], np.zeros((1, 0)))
                step += 1
                T, rc = op.get_state()
                state.T = T
                state.history.r_c[...] = rc.reshape(state.history.r_c.shape)
                if fail:
                    raise InstabilityError(step, state.time, float(dts[i]), ext)
                on_step(state, step, min((i + 1) * dt_explicit, window))

    elapsed = min(n_exp * dt_explicit, window)
    while window - elapsed > 1e-9 * max(settings.dt_implicit, dt_explicit):
        dt_step = min(settings.dt_implicit, window - elapsed)
        attempt = 0
        while True:
            out = op.implicit_step(dt_step, settings)
            if out is not None:
                break
            attempt += 1
            stats.dt_retries += 1
            if attempt > 3:
                raise RuntimeError(
                    f"implicit cool-down failed to converge at dt = "
                    f"{dt_step:.3g} s after 3 step halvings")
            dt_step /= 2.0
        n_newton, n_krylov = out
        op.finish_implicit_step()
        elapsed += dt_step
        step += 1
        stats.newton_iters += n_newton
        stats.krylov_iters += n_krylov
        if on_step is not None:
            T, rc = op.get_state()
            state.T = T
            state.history.r_c[...] = rc.reshape(state.history.r_c.shape)
            on_step(state, step, elapsed)

    T, rc = op.get_state()
    state.T = T
    state.history.r_c[...] = rc.reshape(state.history.r_c.shape)
    state.time += layer_path.cool_time
    stats.n_steps = step
    stats.wall_time = _time.perf_counter() - t0
    state.charge("cooldown", stats.wall_time)
    return stats


@dataclass
class StepCriteria:
    """Stability and accuracy step bounds (timestepping.py:35-46)."""
    dt_stability: float
    dt_accuracy: float
    safety: float

    @property
    def dt_used(self):
        return self.safety * min(self.dt_stability, self.dt_accuracy)


def estimate_spectral_radius(apply_fn, n, seed=0, tol=1e-9, max_iter=500):
    """Power iteration on a host callback (timestepping.py:49-67): start
    N(0,1) from default_rng(seed), normalised; stop when two Rayleigh
    quotients agree to tol; return the larger magnitude of the last two.
    ``compute_step_criteria`` runs the same iteration on the device."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    lam_prev = lam = 0.0
    for _ in range(max_iter):
        w = apply_fn(v)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0
        lam_prev, lam = lam, float(np.dot(v, w))
        v = w / nw
        if abs(lam - lam_prev) <= tol * abs(lam):
            break
    return max(abs(lam), abs(lam_prev))


def compute_step_criteria(op, settings=None, seed=0, tol=1e-9, max_iter=500) -> StepCriteria:
    """timestepping.py:70-99: rho(C~^-1 K) at the stiffest admissible state
    (k frozen to max(k_m, k_s)), dt_stability = 2 / rho, dt_accuracy = R / v.
    The whole power iteration runs on the device (st_spectral_radius); the
    host only draws the same start vector."""
    settings = settings or op.settings
    mat = op.params.material
    rho = op.spectral_radius(max(mat.k_m, mat.k_s), seed=seed, tol=tol, max_iter=max_iter)
    hs = op.params.laser
    return StepCriteria(dt_stability=2.0 / rho, dt_accuracy=hs.radius / hs.scan_velocity,
                        safety=settings.safety_factor)


class JacobianApply:
    """``apply_fn`` for krylov_solve that the device PCG recognises."""

    def __init__(self, op, T_lin, r_c, dt):
        self.op, self.T_lin, self.r_c, self.dt = op, T_lin, r_c, dt

    def __call__(self, v):
        return self.op.apply_jacobian(v, self.T_lin, self.r_c, self.dt)


def krylov_solve(apply_fn, b, diag_inv=None, tol=1e-10, max_iter=2000, x0=None):
    """Preconditioned CG for J x = b (timestepping.py:102-131).

    With a :class:`JacobianApply` the whole solve runs on the device, with
    the caller's ``diag_inv`` as the Jacobi preconditioner (or none); other
    callables run the reference loop around them."""
    if isinstance(apply_fn, JacobianApply) and x0 is None:
        return apply_fn.op.solve_jacobian(b, apply_fn.T_lin, apply_fn.r_c, apply_fn.dt,
                                          tol, max_iter, precondition=diag_inv is not None,
                                          diag_inv=diag_inv)
    n = len(b)
    x = np.zeros(n) if x0 is None else x0.copy()
    r = b - apply_fn(x) if x0 is not None else b.copy()
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), 0, True
    if np.linalg.norm(r) <= tol * bnorm:
        return x, 0, True
    z = r * diag_inv if diag_inv is not None else r.copy()
    p = z.copy()
    rz = float(np.dot(r, z))
    for it in range(1, max_iter + 1):
        Ap = apply_fn(p)
        alpha = rz / float(np.dot(p, Ap))
        x += alpha * p
        r -= alpha * Ap
        if np.linalg.norm(r) <= tol * bnorm:
            return x, it, True
        z = r * diag_inv if diag_inv is not None else r.copy()
        rz_new = float(np.dot(r, z))
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, max_iter, False
