"""Decoding schedules (host-side description; the GPU derives the same order
arithmetically, see csrc/lpic_sched.cuh).

Mirror of /root/reference/pkg/src/lpic/schedules.py: every schedule is
linear, pixel (i, j) is decoded in step a*i + j with a = W (sequential),
h+1 (wavefront) or 1 (diagonal); pixels inside a step go in raster order.
Diagonal mode redirects the taps (-1,1), (-1,2), (-2,2) to (i-2, j+1), or
to the first decoded in-bounds tap when that source is outside the image.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum

from .network import causal_taps


class ScheduleMode(IntEnum):
    SEQUENTIAL = 0
    WAVEFRONT = 1
    DIAGONAL = 2


_MODE_NAMES = {"seq": ScheduleMode.SEQUENTIAL, "sequential": ScheduleMode.SEQUENTIAL,
               "wave": ScheduleMode.WAVEFRONT, "wavefront": ScheduleMode.WAVEFRONT,
               "diag": ScheduleMode.DIAGONAL, "diagonal": ScheduleMode.DIAGONAL}


def parse_mode(name) -> ScheduleMode:
    if isinstance(name, ScheduleMode):
        return name
    key = str(name).lower()
    if key not in _MODE_NAMES:
        raise ValueError(f"unknown schedule mode {name!r}")
    return _MODE_NAMES[key]


DIAGONAL_UNAVAILABLE = ((-1, 1), (-1, 2), (-2, 2))
DIAGONAL_SOURCE = (-2, 1)


@dataclass
class Schedule:
    mode: ScheduleMode
    height: int
    width: int
    steps: list
    substitutions: dict = field(default_factory=dict)
    sub_offsets: tuple = ()

    @property
    def step_count(self) -> int:
        return len(self.steps)


def _dims(height: int, width: int) -> None:
    if height < 1 or width < 1:
        raise ValueError("image dimensions must be positive")


def _linear_steps(height: int, width: int, a: int, n_steps: int) -> list:
    steps = [[] for _ in range(n_steps)]
    for i in range(height):
        for j in range(width):
            steps[a * i + j].append((i, j))
    return steps


def sequential(height: int, width: int) -> Schedule:
    _dims(height, width)
    return Schedule(ScheduleMode.SEQUENTIAL, height, width,
                    [[(i, j)] for i in range(height) for j in range(width)])


def wavefront(height: int, width: int, kernel_half: int) -> Schedule:
    _dims(height, width)
    if kernel_half < 1:
        raise ValueError("kernel_half must be positive")
    a = kernel_half + 1
    return Schedule(ScheduleMode.WAVEFRONT, height, width,
                    _linear_steps(height, width, a, a * (height - 1) + width))


def diagonal_source(i: int, j: int, height: int, width: int, taps=None):
    """Substitute pixel for pixel (i, j)'s unavailable taps, or None."""
    si, sj = i + DIAGONAL_SOURCE[0], j + DIAGONAL_SOURCE[1]
    if 0 <= si < height and 0 <= sj < width:
        return (si, sj)
    taps = causal_taps(2) if taps is None else taps
    for di, dj in taps:
        ci, cj = i + int(di), j + int(dj)
        if 0 <= ci < height and 0 <= cj < width and ci + cj < i + j:
            return (ci, cj)
    return None


def diagonal(height: int, width: int, kernel_half: int) -> Schedule:
    _dims(height, width)
    if kernel_half != 2:
        raise ValueError("diagonal schedule is only defined for kernel_half=2")
    taps = causal_taps(2)
    subs = {}
    for i in range(height):
        for j in range(width):
            src = None
            resolved = False
            for di, dj in DIAGONAL_UNAVAILABLE:
                if not (0 <= i + di < height and 0 <= j + dj < width):
                    continue
                if not resolved:
                    src, resolved = diagonal_source(i, j, height, width, taps), True
                subs[(i, j, di, dj)] = src
    return Schedule(ScheduleMode.DIAGONAL, height, width,
                    _linear_steps(height, width, 1, height + width - 1), subs, DIAGONAL_UNAVAILABLE)


def build_schedule(mode, height: int, width: int, kernel_half: int) -> Schedule:
    mode = parse_mode(mode)
    if mode == ScheduleMode.SEQUENTIAL:
        return sequential(height, width)
    if mode == ScheduleMode.WAVEFRONT:
        return wavefront(height, width, kernel_half)
    return diagonal(height, width, kernel_half)


def schedule_slope(mode, width: int, kernel_half: int) -> int:
    """a in step(i, j) = a*i + j."""
    mode = parse_mode(mode)
    return width if mode == ScheduleMode.SEQUENTIAL else (kernel_half + 1 if mode == ScheduleMode.WAVEFRONT else 1)


def step_count(mode, height: int, width: int, kernel_half: int) -> int:
    return schedule_slope(mode, width, kernel_half) * (height - 1) + width


def nonempty_step_count(mode, height: int, width: int, kernel_half: int) -> int:
    """Network passes the decoder makes (empty wavefront steps are skipped)."""
    a = schedule_slope(mode, width, kernel_half)
    n = 0
    for t in range(step_count(mode, height, width, kernel_half)):
        lo = max(0, -(-(t - width + 1) // a))
        hi = min(height - 1, t // a)
        n += lo <= hi
    return n


def validate(schedule: Schedule, kernel_half: int) -> list[str]:
    """Check the schedule invariants exhaustively; returns the violations."""
    H, W = schedule.height, schedule.width
    out: list[str] = []
    step_of = {}
    for t, step in enumerate(schedule.steps):
        last = None
        for (i, j) in step:
            if not (0 <= i < H and 0 <= j < W):
                out.append(f"pixel ({i},{j}) out of bounds in step {t}")
                continue
            if (i, j) in step_of:
                out.append(f"pixel ({i},{j}) appears in steps {step_of[(i, j)]} and {t}")
            step_of[(i, j)] = t
            if last is not None and (i, j) <= last:
                out.append(f"step {t} is not in raster order at ({i},{j})")
            last = (i, j)
    if len(step_of) != H * W:
        out.append(f"{H * W - len(step_of)} pixels missing from the schedule")
    for (i, j), t in step_of.items():
        for di, dj in causal_taps(kernel_half):
            ti, tj = i + int(di), j + int(dj)
            if not (0 <= ti < H and 0 <= tj < W):
                continue
            if step_of.get((ti, tj), t) < t:
                continue
            key = (i, j, int(di), int(dj))
            if key not in schedule.substitutions:
                out.append(f"pixel ({i},{j}) needs tap ({ti},{tj}) before it is decoded")
                continue
            src = schedule.substitutions[key]
            if src is None:
                continue
            si, sj = src
            if not (0 <= si < H and 0 <= sj < W):
                out.append(f"substitution source ({si},{sj}) for ({i},{j}) out of bounds")
            elif step_of.get((si, sj), t) >= t:
                out.append(f"substitution source ({si},{sj}) for ({i},{j}) not decoded yet")
    return out
