"""Per-size policy ranking over MEASURED schedule costs.

The reference ranks policies with an analytic makespan model
(``gemmsched.costmodel``, costmodel.py:91-128) — explicitly not a hardware
measurement.  On the B200 the cost of a (size, policy) is the measured
device time of its schedule (``sweep.py``); what is kept from the reference
is the record shape and the ranking rule:

* ``CostEstimate`` fields ``makespan``/``utilization``/``atomic_writes``/
  ``full_stores``/``per_wg_cost`` (costmodel.py:61-73) — ``makespan`` is the
  median kernel time in microseconds and ``utilization`` the achieved
  fraction of the dense tensor-core peak;
* ``TuneRecord`` (costmodel.py:76-88) and the ranking of
  :func:`rank_costs` — ascending ``(makespan, Policy.sort_key())``, so
  equal times (identical schedules) credit the lowest canonical ordinal and
  data-parallel wins ties (costmodel.py:141-164);
* ``dp_utilization`` — the wave-quantisation efficiency T / (ceil(T/g)*g)
  (costmodel.py:131-138) that defines "wave-quantisation-bound" shapes.
"""

from __future__ import annotations

from dataclasses import dataclass

from .types import GridInfo, Policy, ProblemSize


@dataclass(frozen=True)
class CostEstimate:
    makespan: float
    utilization: float
    atomic_writes: int
    full_stores: int
    per_wg_cost: tuple[float, ...] = ()


@dataclass(frozen=True)
class TuneRecord:
    size: ProblemSize
    costs: tuple[tuple[Policy, CostEstimate], ...]
    winner: Policy
    runner_up: Policy
    gain: float


def rank_costs(size: ProblemSize, costs) -> TuneRecord:
    """Winner, runner-up and relative gain from (policy, estimate) pairs."""
    costs = tuple(costs)
    if not costs:
        raise ValueError("policies must be nonempty")
    order = sorted(costs, key=lambda pc: (pc[1].makespan, pc[0].sort_key()))
    best_p, best = order[0]
    second_p, second = order[1] if len(order) > 1 else order[0]
    gain = (second.makespan - best.makespan) / second.makespan if second.makespan > 0 else 0.0
    return TuneRecord(size=size, costs=costs, winner=best_p, runner_up=second_p, gain=gain)


def dp_utilization(grid: GridInfo, g: int) -> float:
    if grid.total_tiles < 1:
        raise ValueError("total_tiles must be >= 1")
    if g < 1:
        raise ValueError("g must be >= 1")
    waves = -(-grid.total_tiles // g)
    return grid.total_tiles / (waves * g)
