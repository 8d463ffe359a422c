"""Parity helpers shared by the tests and bench.py's `parity` block (no oracle imports:
they compare device results with the reference-run fixtures in tests/golden/)."""

from __future__ import annotations

import numpy as np


def expand_unique(g, key):
    """Undo make_goldens.unique_rows: rows = uniq[inv]."""
    return g[f"{key}_uniq"][g[f"{key}_inv"]]


def sweep_indices(n, size):
    """The C5 fixture's candidates: n distinct indices from rng_from("sweep", 0), first
    occurrences kept (make_goldens.sweep_indices)."""
    from paper_2102_04199_b200.util import rng_from

    rng = rng_from("sweep", 0)
    out, seen = [], set()
    while len(out) < n:
        for v in rng.integers(0, size, n - len(out)):
            if int(v) not in seen:
                seen.add(int(v))
                out.append(int(v))
    return np.array(out, dtype=np.int64)


def rank_parity(got, ref_top, idx, z_ref, tol=1e-5) -> dict:
    """Ranking parity after tie-class canonicalisation.

    `got`: the device's top-k indices in order; `ref_top`: the reference's rank_history
    top-k over its fp64 scores; `idx`, `z_ref`: every candidate and its reference score.
    Both orders are total orders on (-score, index), so an exact-tie class (identical
    encoded features => bitwise-equal reference scores) is ordered by index in both, and
    any disagreement is a pair of candidates the two orders place differently.  Every
    such pair among the union of both lists is counted: a *tie flip* when the reference
    scores are equal (an exact-tie class left index order: a failure), a *near-tie flip*
    when they differ by at most tol * |z| (reported), a *hard flip* otherwise (a failure).
    """
    got = [int(v) for v in got]
    ref_top = [int(v) for v in ref_top]
    zmap = dict(zip(np.asarray(idx).tolist(), np.asarray(z_ref, dtype=np.float64).tolist()))
    union = list(dict.fromkeys(got + ref_top))
    k = len(got)
    gpos = {v: p for p, v in enumerate(got)}
    u = np.array(union, dtype=np.int64)
    z = np.array([zmap[v] for v in union])
    gp = np.array([gpos.get(v, k) for v in union])
    # reference order: a before b iff (-z_a, a) < (-z_b, b)
    ref_before = (z[:, None] > z[None, :]) | ((z[:, None] == z[None, :]) & (u[:, None] < u[None, :]))
    gpu_before = gp[:, None] < gp[None, :]
    both_out = (gp[:, None] == k) & (gp[None, :] == k)
    flip = gpu_before & ~ref_before & ~both_out
    np.fill_diagonal(flip, False)
    gap = np.abs(z[:, None] - z[None, :])
    near = gap <= tol * np.maximum(np.abs(z[:, None]), np.abs(z[None, :]))
    tie = gap == 0.0
    return {"exact": got == ref_top, "hard_flips": int((flip & ~near).sum()),
            "tie_flips": int((flip & tie).sum()), "near_flips": int((flip & near & ~tie).sum()),
            "max_flip_gap": float(gap[flip].max()) if flip.any() else 0.0}
