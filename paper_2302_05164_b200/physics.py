"""Beam schedule on the host, flattened for the device step loop.

The scan-path types mirror ``scantherm/physics.py`` (Segment :32,
LayerPath :58, ScanPath :78, BeamState :96) and ``layer_beam_state``
reproduces :135-151 operation for operation, because parity of the
temperature field depends on the beam position rounding.  The new piece
is :func:`flatten_schedule`, which evaluates the whole layer's beam
states for a run of steps at once (``tau = (step - 1) * dt``,
``timestepping.py:211-214``) into a packed float64 table that the CUDA
step loop consumes without host round trips.

"""

from dataclasses import dataclass, field

import numpy as np


class ScheduleError(ValueError):
    """Query outside the build schedule."""


@dataclass
class Segment:
    x0: float
    y0: float
    x1: float
    y1: float
    v: float
    power: float

    @property
    def length(self) -> float:
        return float(np.hypot(self.x1 - self.x0, self.y1 - self.y0))

    @property
    def duration(self) -> float:
        return self.length / self.v

    def validate(self):
        if self.v <= 0.0:
            raise ValueError("scan speed must be positive")
        if self.power < 0.0:
            raise ValueError("power must be nonnegative")


@dataclass
class LayerPath:
    layer_index: int
    z: float
    segments: list = field(default_factory=list)
    cool_time: float = 0.0

    def scan_duration(self) -> float:
        return sum(s.duration for s in self.segments)

    def duration(self) -> float:
        return self.scan_duration() + self.cool_time


@dataclass
class ScanPath:
    layers: list = field(default_factory=list)

    def total_duration(self) -> float:
        return sum(lp.duration() for lp in self.layers)


@dataclass
class BeamState:
    position: np.ndarray
    z_top: float
    power: float
    active: bool

    @staticmethod
    def off(z_top=0.0):
        return BeamState(np.zeros(2), z_top, 0.0, False)


def layer_beam_state(lp, tau: float) -> BeamState:
    """Beam at time tau from the layer start (closed segment windows)."""
    if tau < 0.0:
        raise ScheduleError(f"tau = {tau} before the layer starts")
    t_seg = 0.0
    for seg in lp.segments:
        d = seg.duration
        if t_seg <= tau <= t_seg + d:
            s = (tau - t_seg) * seg.v
            frac = s / seg.length if seg.length > 0.0 else 0.0
            pos = np.array([seg.x0 + frac * (seg.x1 - seg.x0),
                            seg.y0 + frac * (seg.y1 - seg.y0)])
            return BeamState(pos, lp.z, seg.power, seg.power > 0.0)
        t_seg += d
    if tau <= lp.duration():
        return BeamState.off(lp.z)
    raise ScheduleError(f"tau = {tau} beyond the layer duration {lp.duration()}")


# packed beam record consumed by the C ABI (st_beam in include/scantherm_b200.h)
BEAM_DTYPE = np.dtype([("x", "f8"), ("y", "f8"), ("z_top", "f8"),
                       ("power", "f8"), ("active", "i4"), ("_pad", "i4")])


def pack_beams(beams):
    """List of BeamState (or None) -> contiguous BEAM_DTYPE array."""
    out = np.zeros(len(beams), dtype=BEAM_DTYPE)
    for i, b in enumerate(beams):
        if b is None:
            continue
        out[i]["x"] = float(b.position[0])
        out[i]["y"] = float(b.position[1])
        out[i]["z_top"] = float(b.z_top)
        out[i]["power"] = float(b.power)
        out[i]["active"] = int(bool(b.active) and float(b.power) > 0.0)
    return out


def _beam_track(lp, taus):
    """Vectorised layer_beam_state over an array of tau: the same closed
    segment windows (first match), the same float expressions in the same
    order; returns (x, y, z_top, power, active)."""
    n = len(taus)
    x = np.zeros(n)
    y = np.zeros(n)
    power = np.zeros(n)
    active = np.zeros(n, dtype=np.int32)
    if np.any(taus < 0.0):
        raise ScheduleError(f"tau = {float(taus.min())} before the layer starts")
    segs = lp.segments
    found = np.zeros(n, dtype=bool)
    t_seg = 0.0
    for seg in segs:
        d = seg.duration
        hit = (~found) & (t_seg <= taus) & (taus <= t_seg + d)
        if np.any(hit):
            s = (taus[hit] - t_seg) * seg.v
            frac = s / seg.length if seg.length > 0.0 else np.zeros_like(s)
            x[hit] = seg.x0 + frac * (seg.x1 - seg.x0)
            y[hit] = seg.y0 + frac * (seg.y1 - seg.y0)
            power[hit] = seg.power
            active[hit] = 1 if seg.power > 0.0 else 0
            found |= hit
        t_seg += d
    rest = ~found
    if np.any(rest & (taus > lp.duration())):
        raise ScheduleError(f"tau = {float(taus[rest].max())} beyond the layer duration "
                            f"{lp.duration()}")
    return x, y, np.full(n, float(lp.z)), power, active


def flatten_schedule(layer_paths, dt, n_steps, step0=1):
    """Beam records for steps step0 .. step0+n_steps-1 of a scan phase.

    ``layer_paths`` is one LayerPath or a list of concurrently scanned
    LayerPaths (multi-spot, BASELINE config 4: the source is linear in
    the beams).  Returns (dt_steps (n,), beams (n, n_beams) BEAM_DTYPE).
    Vectorised over the steps (a layer is tens of thousands of steps);
    identical to evaluating ``layer_beam_state`` at tau = (step - 1) dt
    for every step (tests/test_schedule.py).
    """
    if not isinstance(layer_paths, (list, tuple)):
        layer_paths = [layer_paths]
    duration = layer_paths[0].scan_duration()
    nb = len(layer_paths)
    steps = np.arange(step0, step0 + n_steps, dtype=np.int64)
    taus = (steps - 1).astype(np.float64) * dt
    dts = np.minimum(dt, duration - taus)
    beams = np.zeros((n_steps, nb), dtype=BEAM_DTYPE)
    for k, lp in enumerate(layer_paths):
        x, y, z, pw, act = _beam_track(lp, taus)
        beams["x"][:, k] = x
        beams["y"][:, k] = y
        beams["z_top"][:, k] = z
        beams["power"][:, k] = pw
        beams["active"][:, k] = act & (pw > 0.0)
    return dts, beams


def flatten_schedule_loop(layer_paths, dt, n_steps, step0=1):
    """Per-step reference form of flatten_schedule (tests)."""
    if not isinstance(layer_paths, (list, tuple)):
        layer_paths = [layer_paths]
    duration = layer_paths[0].scan_duration()
    nb = len(layer_paths)
    beams = np.zeros((n_steps, nb), dtype=BEAM_DTYPE)
    dts = np.empty(n_steps)
    for i in range(n_steps):
        step = step0 + i
        tau = (step - 1) * dt
        dts[i] = min(dt, duration - tau)
        beams[i] = pack_beams([layer_beam_state(lp, tau) for lp in layer_paths])
    return dts, beams


def segment_table(layer_paths):
    """Device beam schedule input (st_scan_layer / st_beam_schedule): per
    path the segment count, then every segment with the length, duration
    and start time the reference derives for it (Segment.length /
    .duration and layer_beam_state's running t_seg, physics.py:135-151),
    computed here in Python so the device sees the same doubles."""
    if not isinstance(layer_paths, (list, tuple)):
        layer_paths = [layer_paths]
    counts = np.array([len(lp.segments) for lp in layer_paths], dtype=np.int32)
    rows = []
    for lp in layer_paths:
        t_seg = 0.0
        for seg in lp.segments:
            d = seg.duration
            rows.append((seg.x0, seg.y0, seg.x1, seg.y1, seg.v, seg.power, seg.length, d, t_seg))
            t_seg += d
    segs = np.array(rows, dtype=np.float64).reshape(-1, 9)
    z = np.array([float(lp.z) for lp in layer_paths], dtype=np.float64)
    return counts, np.ascontiguousarray(segs), z
