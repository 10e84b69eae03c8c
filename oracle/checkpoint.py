"""Activation checkpointing hyperparameter and memory model (§V-A) —
oracle (test infrastructure only; imported by tests/ alone).

* Eq. 1: M_activation ∝ G_inter · (N / (G_inter · ac)) + 1 + ac
  = N / ac + 1 + ac  (activation units per GPU).
* The rule: "set the value of ac to the factor of N / G_inter (the number
  of layers on each GPU) closest to √N"; ties go to the smaller factor (reading D-33).
  The rule is the paper's; Eq. 1's own argmin over the same factors differs for some
  (N, G_inter) — e.g. N = 14, G_inter = 2: the rule gives 1, Eq. 1 is minimised at 7
  (tests/test_oracle_checkpoint.py enumerates every case with N <= 256) — so both are kept.
* Checkpointing is numerically neutral: the recomputed forward is the same computation, so
  the gradients equal those of ac = 1 exactly.
"""
from fractions import Fraction
import math


def factors(n: int) -> list[int]:
    return [a for a in range(1, n + 1) if n % a == 0]


def select_checkpoint_interval(n_layers: int, g_inter: int) -> int:
    """The factor of N / G_inter closest to √N; ties -> smaller."""
    if g_inter <= 0 or n_layers % g_inter:
        raise ValueError("g_inter must divide the layer count")
    per = n_layers // g_inter
    root = math.sqrt(n_layers)
    return min(factors(per), key=lambda a: (abs(a - root), a))


def activation_units(n_layers: int, g_inter: int, ac: int) -> Fraction:
    """Eq. 1: G_inter · (N / (G_inter · ac)) + 1 + ac, exactly."""
    if g_inter <= 0 or n_layers % g_inter or (n_layers // g_inter) % ac:
        raise ValueError("BadCheckpointInterval: ac must divide N / G_inter")
    return g_inter * Fraction(n_layers, g_inter * ac) + 1 + ac


def eq1_argmin(n_layers: int, g_inter: int) -> list[int]:
    """Every factor of N / G_inter that minimises Eq. 1 (brute force)."""
    per = n_layers // g_inter
    vals = {a: activation_units(n_layers, g_inter, a) for a in factors(per)}
    best = min(vals.values())
    return [a for a, v in vals.items() if v == best]
