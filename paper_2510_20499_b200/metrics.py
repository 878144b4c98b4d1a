"""Algorithmic work and byte counts of a propagate trajectory.

The engine reports, per round r, the reference's dirty sets (bp_propagate_ex with
BP_FORCE_FRONTIER): R_r dirty rows with row-nnz sum A_r, V_r dirty vars with column-nnz sum B_r,
C_r changed vars. Full rounds have R = all rows, V = all vars.

  BP nnz visits      = Σ_r (A_r + B_r)
  algorithmic bytes  = Σ_r [ 12·A_r + 28·|R_r| + 16·min(n, A_r)          activity phase
                           + 12·B_r + 21·|V_r| + 40·min(m, B_r) + 16·|C_r| ] tightening phase

(12 B per CSR/CSC entry = int32 index + f64 value; 4 B row/col start + 24 B activity record written
per row; 16 B of bounds read once per touched var; 40 B activity+counts+row bounds per touched row;
17 B own bounds + integrality and 4 B col start per var; 16 B bounds written per changed var).
A full round is 24·N + 68·m + 37·n + 16·|C| ≈ 24·N + 105·n for m = n.
"""
from __future__ import annotations

import numpy as np

STAT_COLS = 12  # full, |R|, A (row nnz), |V|, B (col nnz), |C|, t_act, t_tight, t_xrow, t_xvar, t_gather (ns), spare


def trim(stats: np.ndarray, rounds: int) -> np.ndarray:
    return np.asarray(stats, dtype=np.int64).reshape(-1, STAT_COLS)[:rounds]


def nnz_visits(stats: np.ndarray) -> int:
    s = np.asarray(stats, dtype=np.int64).reshape(-1, STAT_COLS)
    return int(s[:, 2].sum() + s[:, 4].sum())


def algorithmic_bytes(stats: np.ndarray, n: int, m: int) -> int:
    s = np.asarray(stats, dtype=np.int64).reshape(-1, STAT_COLS)
    R, A, V, B, Cc = s[:, 1], s[:, 2], s[:, 3], s[:, 4], s[:, 5]
    act = 12 * A + 28 * R + 16 * np.minimum(n, A)
    tig = 12 * B + 21 * V + 40 * np.minimum(m, B) + 16 * Cc
    return int((act + tig).sum())
