"""Synthetic WHFF operators with the reference's formulas (model.py:158-268)
and thermal loads (thermal.py:62-78) -- the input generator for tests and the
benchmark.  A, B, P and small C are built on the host exactly as the
reference does (same rng draw order, same numpy expressions, so small models
are identical); paper-scale C slits are generated slit by slit on the device
with the same expression in binary64 (model.py:258-268), then compressed on
the GPU, so the 60 GB dense operators never exist anywhere.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

AXES = ("x", "y", "z")
_NEIGHBOR_OFFSETS = [(-1, 0), (1, 0), (0, -1), (0, 1), (-1, -1), (1, 1), (-1, 1), (1, -1),
                     (-2, 0), (2, 0), (0, -2), (0, 2)]


@dataclass(frozen=True)
class Spec:
    grid_rows: int
    grid_cols: int
    S: int
    K: int
    M: int
    nnz_target: int = 5
    seed: int = 0
    n_fields: int | None = None
    c_scale: float = 1e-8
    c_kind: str = "smooth"

    @property
    def T(self):
        return self.grid_rows * self.grid_cols


def thermal_operator(spec, rng):
    """model.py:188-216."""
    import scipy.sparse as sp
    R, Cg = spec.grid_rows, spec.grid_cols
    T = R * Cg
    n_neigh = min(spec.nnz_target - 1, len(_NEIGHBOR_OFFSETS))
    offsets = _NEIGHBOR_OFFSETS[:n_neigh]
    alpha = (0.8 + 0.2 * rng.random(T)) * (0.5 / max(n_neigh, 1))
    leak = 0.002 + 0.008 * rng.random(T)
    rows, cols, vals = [], [], []
    r_idx, c_idx = np.divmod(np.arange(T), Cg)
    diag = np.ones(T)
    for dr, dc in offsets:
        rr, cc = r_idx + dr, c_idx + dc
        ok = (rr >= 0) & (rr < R) & (cc >= 0) & (cc < Cg)
        rows.append(np.arange(T)[ok])
        cols.append((rr * Cg + cc)[ok])
        vals.append(alpha[ok])
        diag -= alpha * ok
    diag -= leak
    rows.append(np.arange(T))
    cols.append(np.arange(T))
    vals.append(diag)
    A = sp.csr_matrix((np.concatenate(vals).astype(np.float32),
                       (np.concatenate(rows), np.concatenate(cols))), shape=(T, T))
    A.sort_indices()
    return A


def interpolation(spec):
    """model.py:219-249 (bilinear restriction, renormalised in float32)."""
    import scipy.sparse as sp
    R, Cg, S = spec.grid_rows, spec.grid_cols, spec.S
    sc = max(1, int(np.ceil(np.sqrt(S * Cg / R))))
    sr = int(np.ceil(S / sc))
    k = np.arange(S)
    fr = (k // sc) / max(sr - 1, 1) * (R - 1)
    fc = (k % sc) / max(sc - 1, 1) * (Cg - 1)
    fc = np.minimum(fc, Cg - 1)
    r0 = np.minimum(fr.astype(np.int64), R - 2) if R > 1 else np.zeros(S, np.int64)
    c0 = np.minimum(fc.astype(np.int64), Cg - 2) if Cg > 1 else np.zeros(S, np.int64)
    tr, tc = fr - r0, fc - c0
    rows = np.repeat(k, 4)
    cols = np.empty(4 * S, dtype=np.int64)
    vals = np.empty(4 * S, dtype=np.float64)
    r1, c1 = np.minimum(r0 + 1, R - 1), np.minimum(c0 + 1, Cg - 1)
    for i, (rr, cc, w) in enumerate([(r0, c0, (1 - tr) * (1 - tc)), (r0, c1, (1 - tr) * tc),
                                     (r1, c0, tr * (1 - tc)), (r1, c1, tr * tc)]):
        cols[i::4] = rr * Cg + cc
        vals[i::4] = w
    P = sp.csr_matrix((vals, (rows, cols)), shape=(S, spec.T))
    P.sum_duplicates()
    P = P.astype(np.float32)
    rs = np.asarray(P.sum(axis=1)).ravel()
    P = sp.diags(1.0 / rs).dot(P).astype(np.float32)
    P.sort_indices()
    return sp.csr_matrix(P)


@dataclass
class Operators:
    spec: Spec
    A: object
    B: np.ndarray
    P: object
    phases: dict          # axis -> phase of the smooth C (model.py:264)
    noise_rng_state: object = None

    def A64(self):
        return self.A.astype(np.float64)

    def P64(self):
        return self.P.astype(np.float64)


def generate(spec):
    """A, B, P and the per-axis C phases in the reference's rng order
    (model.py:175-180): A (alpha, leak), B, then one draw per axis."""
    rng = np.random.default_rng(np.random.SeedSequence(spec.seed))
    A = thermal_operator(spec, rng)
    B = (0.5 + rng.random(spec.T) * 1.0).astype(np.float32)
    P = interpolation(spec)
    phases = {}
    if spec.c_kind == "smooth":
        for axis in AXES:
            phases[axis] = rng.random() * 2 * np.pi
    return Operators(spec, A, B, P, phases)


def deformation_rows(spec, axis_index, phase, r0, r1, device=None, ncols=None):
    """Rows [r0, r1) of the smooth C of one axis (model.py:258-268).  On the
    host this is the reference's expression verbatim (optionally only the
    first `ncols` columns); on a CUDA device the same binary64 expression
    evaluated by torch (float32 result)."""
    K, S = spec.K, spec.S
    if device is None:
        j = np.arange(S if ncols is None else min(ncols, S), dtype=np.float64)
        k = np.arange(K, dtype=np.float64)[r0:r1]
        centers = (k / max(K - 1, 1)) * (S - 1)
        width = S * (0.08 + 0.04 * np.sin(2 * np.pi * k / max(K, 1) + axis_index))
        width = np.maximum(width, 2.0)
        amp = 1.0 + 0.3 * np.cos(2 * np.pi * k / max(K, 1) * (axis_index + 1))
        d = j[None, :] - centers[:, None]
        c = amp[:, None] * np.exp(-0.5 * (d / width[:, None]) ** 2)
        c += 0.05 * np.cos(2 * np.pi * j[None, :] / S * (2 + axis_index) + phase)
        return (spec.c_scale * c).astype(np.float32)
    import torch
    f64 = torch.float64
    j = torch.arange(S, dtype=f64, device=device)
    k = torch.arange(r0, r1, dtype=f64, device=device)
    centers = (k / max(K - 1, 1)) * (S - 1)
    width = S * (0.08 + 0.04 * torch.sin(2 * np.pi * k / max(K, 1) + axis_index))
    width = torch.clamp(width, min=2.0)
    amp = 1.0 + 0.3 * torch.cos(2 * np.pi * k / max(K, 1) * (axis_index + 1))
    d = j[None, :] - centers[:, None]
    c = amp[:, None] * torch.exp(-0.5 * (d / width[:, None]) ** 2)
    c += 0.05 * torch.cos(2 * np.pi * j[None, :] / S * (2 + axis_index) + phase)
    return (spec.c_scale * c).to(torch.float32)


def windows(spec):
    """model.py:271-284: field and slit row windows."""
    n_fields = spec.n_fields if spec.n_fields is not None else max(1, spec.K // (4 * spec.M))
    spf = (spec.K // n_fields) // spec.M
    width = spf * spec.M
    fields = [(f * width, (f + 1) * width) for f in range(n_fields)]
    slits = [[(f0 + s * spec.M, f0 + (s + 1) * spec.M) for s in range(spf)] for f0, _ in fields]
    return fields, slits


def heatload(spec, n_fields, n_slits, seed=0, dose_scale=1.0, cooling=1e-3):
    """thermal.py:62-78 synthetic_heatload -> (dark, {(f, s): footprint}, dose)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x48454154]))
    T = spec.T
    dark = (-cooling * (0.5 + 0.5 * rng.random(T))).astype(np.float32)
    pts = np.arange(T, dtype=np.float64)
    fps = {}
    for f in range(n_fields):
        for s in range(n_slits):
            center = ((f * n_slits + s + 0.5) / (n_fields * n_slits)) * T
            width = max(T * 0.02, 2.0)
            fp = np.exp(-0.5 * ((pts - center) / width) ** 2)
            fp *= 0.5 + 0.5 * rng.random()
            fps[(f, s)] = fp.astype(np.float32)
    return dark, fps, dose_scale
