"""The paper's memory-traffic iteration cost model (proj/src/cost_model.cpp),
restated for the measurement side: bench.py reports the model's predicted per-iteration times at
the measured HBM bandwidth and the predicted / measured slowdown gamma of the accelerated solves
(compare_measured).  Pure host arithmetic on report fields -- no part of the solver path.
"""
from __future__ import annotations

from dataclasses import dataclass

from ._lib import InvalidArgument


@dataclass
class CostParams:
    """CostParams (cost_model.hpp:12-17): sizes and the sustained bandwidth (1.0 = normalised)."""
    n: float = 0.0
    nnz: float = 0.0
    m_tilde: float = 0.0
    bandwidth: float = 1.0


def _check(p: CostParams) -> None:  # cost_model.cpp:7-10
    if p.n < 0 or p.nnz < 0 or p.m_tilde < 0 or p.bandwidth <= 0:
        raise InvalidArgument("CostParams: sizes must be >= 0, bandwidth > 0")


def t_cg(p: CostParams) -> float:
    """(76 n + 12 nnz) / bandwidth (cost_model.cpp:14-17)."""
    _check(p)
    return (76.0 * p.n + 12.0 * p.nnz) / p.bandwidth


def t_iccg(p: CostParams) -> float:
    """(100 n + 24 nnz) / bandwidth (cost_model.cpp:19-22)."""
    _check(p)
    return (100.0 * p.n + 24.0 * p.nnz) / p.bandwidth


def t_sciccg(p: CostParams) -> float:
    """(116 n + 16 m~ n + 24 nnz) / bandwidth (cost_model.cpp:24-27)."""
    _check(p)
    return (116.0 * p.n + 16.0 * p.m_tilde * p.n + 24.0 * p.nnz) / p.bandwidth


def gamma_sciccg(m_tilde: float, nnz_av: float) -> float:
    """(116 + 16 m~ + 24 nnz_av) / (100 + 24 nnz_av) (cost_model.cpp:29-33)."""
    if m_tilde < 0 or nnz_av < 0:
        raise InvalidArgument("gamma_sciccg: arguments must be >= 0")
    return (116.0 + 16.0 * m_tilde + 24.0 * nnz_av) / (100.0 + 24.0 * nnz_av)


@dataclass
class CostComparison:
    predicted: float = 0.0
    measured: float = 0.0
    rel_error: float = 0.0


def compare_measured(base_iterations: int, base_wall: float, acc_iterations: int, acc_wall: float,
                     m_tilde: float, nnz_av: float) -> CostComparison:
    """compare_measured (cost_model.cpp:35-48) on the (iterations, wall_time) of two solve
    reports: measured gamma = accelerated per-iteration time / baseline per-iteration time."""
    if base_iterations <= 0 or acc_iterations <= 0:
        raise InvalidArgument("compare_measured: reports need at least one iteration")
    if base_wall <= 0.0:
        raise InvalidArgument("compare_measured: baseline wall time must be positive")
    c = CostComparison()
    c.predicted = gamma_sciccg(m_tilde, nnz_av)
    per_base = base_wall / base_iterations
    per_acc = acc_wall / acc_iterations
    c.measured = per_acc / per_base
    c.rel_error = (c.measured - c.predicted) / c.predicted
    return c
