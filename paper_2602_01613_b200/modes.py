"""Host-side mode/rank arithmetic of the TN layer (integer work, no compute).

Mirrors the reference's mode-shape and rank bookkeeping so that layer shapes,
cut bonds and stored-scalar counts agree exactly:
  balanced_split / default_mode_shape   tn_decompositions.py:45-63
  param_count_formula                   tn_decompositions.py:381-401
  maximal_ranks                         tn_decompositions.py:404-418
  tr_feasible / ranks_feasible          tn_decompositions.py:259-286,425-442
  RankSpec                              tn_decompositions.py:129-143
  select_ranks -> RankSpec              tn_decompositions.py:445-510
  FixedRank/RelativeError/ParamBudget   tensor_core.py:136-166 (truncation policies)
and adds the FLOP currency of the SPEC: 2 x product of all
involved mode sizes per pairwise step, canonical chain order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import InfeasibleBudgetError, RankError

FAMILIES = ("tucker", "tt", "tr")
DENSE = "dense"


def balanced_split(n: int) -> tuple[int, ...]:
    """Closest-to-square divisor pair of n; primes (and 1) stay whole."""
    if n <= 1:
        return (max(n, 1),)
    for a in range(math.isqrt(n), 1, -1):
        if n % a == 0:
            return (a, n // a)
    return (n,)


def default_mode_shape(rows: int, cols: int) -> tuple[tuple[int, ...], int]:
    """Row (output) modes first, then column (input) modes; returns (shape, rm)."""
    r, c = balanced_split(rows), balanced_split(cols)
    return r + c, len(r)


def param_count_formula(family: str, mode_shape, ranks) -> int:
    shape = tuple(int(s) for s in mode_shape)
    if family == DENSE:
        return math.prod(shape)
    ranks = tuple(int(r) for r in ranks)
    d = len(shape)
    if family == "tucker":
        if len(ranks) != d:
            raise RankError(f"need {d} tucker ranks")
        return math.prod(ranks) + sum(n * r for n, r in zip(shape, ranks))
    if family == "tt":
        if len(ranks) != d - 1:
            raise RankError(f"need {d - 1} tt bond ranks")
        b = (1,) + ranks + (1,)
        return sum(b[k] * shape[k] * b[k + 1] for k in range(d))
    if family == "tr":
        if len(ranks) != d:
            raise RankError(f"need {d} tr ranks")
        return sum(ranks[k] * shape[k] * ranks[(k + 1) % d] for k in range(d))
    raise RankError(f"unknown family {family!r}")


def maximal_ranks(family: str, mode_shape) -> tuple[int, ...]:
    """Smallest exact ranks; the TR closure is capped at 1 as in the reference."""
    shape = tuple(int(s) for s in mode_shape)
    d = len(shape)
    total = math.prod(shape)
    if family == "tucker":
        return tuple(min(n, total // n) for n in shape)
    tt = tuple(min(math.prod(shape[: k + 1]), math.prod(shape[k + 1 :])) for k in range(d - 1))
    if family == "tt":
        return tt
    if family == "tr":
        return (1,) + tt
    raise RankError(f"unknown family {family!r}")


def tr_feasible(mode_shape, ranks) -> tuple[int, ...]:
    """Ranks reachable by the sequential ring split (first split carries r0*r1)."""
    shape = tuple(int(s) for s in mode_shape)
    ranks = tuple(int(r) for r in ranks)
    d = len(shape)
    if len(ranks) != d:
        raise RankError(f"need {d} cyclic ranks, got {len(ranks)}")
    if any(r < 1 for r in ranks):
        raise RankError(f"ranks must be >= 1, got {ranks}")
    rest = math.prod(shape[1:])
    if ranks[0] * ranks[1 % d] > min(shape[0], rest):
        raise RankError(f"first split rank {ranks[0]}*{ranks[1 % d]} infeasible for {shape[0]}x{rest} unfolding")
    got = [ranks[0], ranks[1 % d]]
    prev, cols = ranks[1 % d], rest * ranks[0]
    for k in range(1, d - 1):
        cols //= shape[k]
        prev = min(ranks[k + 1], prev * shape[k], cols)
        got.append(prev)
    return tuple(got[:d])


def ranks_feasible(family: str, shape, ranks) -> bool:
    caps = maximal_ranks(family, shape)
    if family == "tucker":
        return all(r <= n for r, n in zip(ranks, shape))
    if family == "tt":
        if any(r > c for r, c in zip(ranks, caps)):
            return False
        left = 1
        for k, r in enumerate(ranks):
            if r > left * shape[k]:
                return False
            left = r
        return True
    try:
        return tuple(tr_feasible(shape, ranks)) == tuple(ranks)
    except RankError:
        return False


# --- truncation policies (tensor_core.py:136-166) ------------------------------


@dataclass(frozen=True)
class FixedRank:
    rank: int

    def __post_init__(self):
        if int(self.rank) < 1:
            raise RankError(f"fixed rank must be >= 1, got {self.rank}")
        object.__setattr__(self, "rank", int(self.rank))


@dataclass(frozen=True)
class RelativeError:
    epsilon: float

    def __post_init__(self):
        if not 0.0 < float(self.epsilon) <= 1.0:
            raise RankError(f"relative-error threshold must be in (0, 1], got {self.epsilon}")
        object.__setattr__(self, "epsilon", float(self.epsilon))


@dataclass(frozen=True)
class ParamBudget:
    budget: int

    def __post_init__(self):
        if int(self.budget) < 1:
            raise RankError(f"parameter budget must be >= 1, got {self.budget}")
        object.__setattr__(self, "budget", int(self.budget))


@dataclass(frozen=True)
class RankSpec:
    """Concrete ranks for a family, or a relative-error threshold to resolve them during
    decomposition (tn_decompositions.py:129-143: same fields, same RankError checks)."""

    family: str
    ranks: tuple | None = None
    rel_error: float | None = None

    def __post_init__(self):
        if self.family not in FAMILIES and self.family != DENSE:
            raise RankError(f"unknown family {self.family!r}")
        if self.ranks is not None:
            object.__setattr__(self, "ranks", tuple(int(r) for r in self.ranks))
            if any(r < 1 for r in self.ranks):
                raise RankError(f"ranks must be >= 1, got {self.ranks}")


def select_ranks(mode_shape, family: str, target) -> RankSpec:
    """Rank selection toward a truncation target (tn_decompositions.py:445-510).

    ParamBudget: budgets at or above the dense size give the maximal (exact) ranks, else the
    largest feasible uniform rank grown greedily position by position; FixedRank: the rank
    clipped to the caps, lowered at the first largest position until feasible; RelativeError:
    deferred to the decomposition (``RankSpec(rel_error=epsilon)``)."""
    shape = tuple(int(s) for s in mode_shape)
    if family == DENSE:
        return RankSpec(family=DENSE)
    if family not in FAMILIES:
        raise RankError(f"unknown family {family!r}")
    d = len(shape)
    npos = {"tucker": d, "tt": d - 1, "tr": d}[family]
    if isinstance(target, RelativeError):
        return RankSpec(family=family, ranks=None, rel_error=target.epsilon)
    caps = maximal_ranks(family, shape)
    if isinstance(target, FixedRank):
        ranks = [min(target.rank, c) for c in caps]
        while not ranks_feasible(family, shape, tuple(ranks)):
            i = max(range(len(ranks)), key=lambda t: (ranks[t], -t))
            ranks[i] = max(1, ranks[i] - 1)
        return RankSpec(family=family, ranks=tuple(ranks))
    if not isinstance(target, ParamBudget):
        raise TypeError(f"unsupported target {target!r}")
    budget = target.budget
    if budget >= math.prod(shape):
        return RankSpec(family=family, ranks=caps)
    floor_cost = param_count_formula(family, shape, (1,) * npos)
    if floor_cost > budget:
        raise InfeasibleBudgetError(
            f"budget {budget} below rank-1 configuration of {floor_cost} params", best_achievable=floor_cost
        )

    def fits(r) -> bool:
        return (
            all(a <= c for a, c in zip(r, caps))
            and ranks_feasible(family, shape, r)
            and param_count_formula(family, shape, r) <= budget
        )

    u = 1
    while fits((u + 1,) * npos):
        u += 1
    ranks = [u] * npos
    grew = True
    while grew:
        grew = False
        for i in range(npos):
            trial = ranks.copy()
            trial[i] += 1
            if fits(tuple(trial)):
                ranks, grew = trial, True
    return RankSpec(family=family, ranks=tuple(ranks))


# --- FLOP currency, canonical chain order ---


def chain_flops_per_token(family: str, mode_shape, row_mode_count: int, bonds_or_ranks) -> int:
    """TT/TR: pass the d+1 bonds (core k = (b[k], n_k, b[k+1])); Tucker: d ranks."""
    ms = tuple(mode_shape)
    rm = row_mode_count
    d = len(ms)
    if family == DENSE:
        return 2 * math.prod(ms)
    if family == "tucker":
        R = tuple(bonds_or_ranks)
        f = 0
        cur = list(ms[rm:])
        for k in range(d - 1, rm - 1, -1):
            f += 2 * math.prod(cur) * R[k]
            cur[k - rm] = R[k]
        f += 2 * math.prod(R[:rm]) * math.prod(R[rm:])
        cur = list(R[:rm])
        for k in range(rm):
            f += 2 * math.prod(cur) * ms[k]
            cur[k] = ms[k]
        return f
    b = tuple(bonds_or_ranks)
    r0 = b[0]
    f = 0
    for k in range(rm, d):
        mult = r0 if (k != d - 1 and r0 > 1) else 1
        f += 2 * math.prod(ms[rm:k]) * ms[k] * b[k + 1] * b[k] * mult
    for k in range(rm):
        mult = r0 if (k != 0 and r0 > 1) else 1
        f += 2 * math.prod(ms[k + 1 : rm]) * b[k + 1] * ms[k] * b[k] * mult
    return f


def cut_rank(family: str, mode_shape, row_mode_count: int, bonds_or_ranks) -> int:
    ms = tuple(mode_shape)
    rm = row_mode_count
    if family == "tucker":
        R = tuple(bonds_or_ranks)
        return min(math.prod(R[:rm]), math.prod(R[rm:]))
    if family in ("tt", "tr"):
        b = tuple(bonds_or_ranks)
        return b[0] * b[rm]
    rows = math.prod(ms[:rm])
    return min(rows, math.prod(ms) // rows)
