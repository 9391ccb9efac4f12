"""Scaling grid for the exact engine -- the reference's ``binpaths.bench`` API
(pkg/src/binpaths/bench.py:1-135) with the GPU engine behind the runner.

Semantics kept from the reference (its tests pin them, tests/test_bench.py):

* every (N, M) cell is timed ``repetitions`` times, the median wall is kept
  and floored at 1e-12 s (bench.py:22-23, 80-82);
* within one N the smallest M is the baseline and is credited with speedup
  M0, so speedup(M) = M0 * wall(M0) / wall(M) and efficiency = speedup / M
  (bench.py:57-63, 83-97);
* the grid must list each N in one contiguous run with strictly ascending M
  (bench.py:36-53); an empty grid or a non-positive repetition count is
  ``InvalidInput``;
* CSV header ``N,M,wall_seconds,speedup,efficiency,baseline_M`` with repr
  floats (bench.py:19, 100-106) and three N-by-M text tables (:120-135).

For the GPU CLI the M axis is the number of GPU shards the canonical
super-blocks are split over (cli.py ``bench``); the harness itself is
engine-agnostic and times whatever ``runner(n, m)`` does.
"""
from __future__ import annotations

import statistics
import time
from dataclasses import dataclass
from typing import Callable, Iterable, List, Sequence, Tuple

from .errors import InvalidInput

BENCH_CSV_HEADER = "N,M,wall_seconds,speedup,efficiency,baseline_M"
_WALL_FLOOR = 1e-12  # clock-granularity guard (reference bench.py:22-23)
_TABLE_FIELDS = ("wall_seconds", "speedup", "efficiency")


@dataclass(frozen=True)
class BenchRecord:
    n: int
    m: int
    wall_seconds: float
    speedup: float
    efficiency: float
    baseline_m: int


def _runs_by_depth(cells: Sequence[Tuple[int, int]]) -> List[Tuple[int, List[int]]]:
    """Split the grid into contiguous runs of one N; validate the layout."""
    runs: List[Tuple[int, List[int]]] = []
    for n, m in cells:
        if runs and runs[-1][0] == n:
            runs[-1][1].append(m)
            continue
        if any(prev_n == n for prev_n, _ in runs):
            raise InvalidInput(f"grid lists N={n} in two separate runs; group them")
        runs.append((n, [m]))
    for n, ms in runs:
        if sorted(set(ms)) != ms:
            raise InvalidInput(f"worker counts for N={n} must be strictly ascending, got {ms}")
    return runs


def _median_wall(fn: Callable[[], None], repetitions: int) -> float:
    samples = []
    for _ in range(repetitions):
        start = time.perf_counter()
        fn()
        samples.append(time.perf_counter() - start)
    return max(statistics.median(samples), _WALL_FLOOR)


def run_bench(pairs: Iterable, runner: Callable, repetitions: int = 3) -> list:
    """Time ``runner(n, m)`` over the grid; return one ``BenchRecord`` per cell
    in grid order (reference bench.py:57-97)."""
    if isinstance(repetitions, bool) or not isinstance(repetitions, int) or repetitions < 1:
        raise InvalidInput(f"repetitions must be a positive integer, got {repetitions!r}")
    cells = [(int(n), int(m)) for n, m in pairs]
    if not cells:
        raise InvalidInput("empty benchmark grid")
    out = []
    for n, ms in _runs_by_depth(cells):
        walls = {m: _median_wall(lambda: runner(n, m), repetitions) for m in ms}
        m0 = ms[0]
        work = m0 * walls[m0]  # baseline "processor-seconds"
        for m in ms:
            speedup = work / walls[m]
            out.append(BenchRecord(n=n, m=m, wall_seconds=walls[m], speedup=speedup,
                                   efficiency=speedup / m, baseline_m=m0))
    return out


def records_to_csv(records: Sequence) -> str:
    rows = [BENCH_CSV_HEADER]
    rows += [f"{r.n},{r.m},{r.wall_seconds!r},{r.speedup!r},{r.efficiency!r},{r.baseline_m}" for r in records]
    return "\n".join(rows) + "\n"


def records_to_tables(records: Sequence) -> str:
    """wall / speedup / efficiency as right-aligned N-by-M tables, ``-`` for
    missing cells, 4 decimals (reference bench.py:120-135)."""
    ms = sorted({r.m for r in records})
    ns = sorted({r.n for r in records})
    cell = {(r.n, r.m): r for r in records}
    blocks = []
    for name in _TABLE_FIELDS:
        grid = [["N\\M", *map(str, ms)]]
        for n in ns:
            row = [str(n)]
            for m in ms:
                rec = cell.get((n, m))
                row.append("-" if rec is None else f"{getattr(rec, name):.4f}")
            grid.append(row)
        widths = [max(len(r[c]) for r in grid) for c in range(len(grid[0]))]
        lines = ["  ".join(v.rjust(w) for v, w in zip(r, widths)) for r in grid]
        blocks.append("\n".join([name, *lines, ""]))
    return "\n".join(blocks)
