"""Shared test helpers: run the CPU oracle on a Workload and compare."""
from __future__ import annotations

import dataclasses

import numpy as np

import oracle as O


def rel_rms(a, b) -> float:
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def truncate(w, B: int):
    """Same workload with only the first B symbols."""
    return dataclasses.replace(w, cp=list(w.cp[:B]))


def full_grids(w, packed: np.ndarray) -> list[np.ndarray]:
    """packed (B, A) active values -> per subband (B, L) full DFT-bin columns."""
    grids, off = [], 0
    for s, bins in zip(w.subbands, w.active_maps):
        g = np.zeros((w.B, s.L), np.complex128)
        g[:, bins] = packed[:, off:off + len(bins)]
        grids.append(g)
        off += len(bins)
    return grids


def oracle_tx(w, packed: np.ndarray, ref: bool = False):
    f = O.Ref.tx_discontinuous if ref else O.tx_discontinuous
    return f(full_grids(w, packed), [s.L for s in w.subbands], [s.c for s in w.subbands],
             [s.window for s in w.subbands], w.cp, w.N)


def oracle_rx(w, wave: np.ndarray, useful0: int, fused: bool, ref: bool = False):
    """Returns (packed (B, A), full (B, sum L)) like the GPU's two layouts."""
    f = O.Ref.rx_discontinuous if ref else O.rx_discontinuous
    packed, full = [], []
    for s, bins in zip(w.subbands, w.active_maps):
        cols = f(wave, useful0, w.cp, w.N, s.L, s.c, s.window, fused)
        full.append(cols)
        packed.append(cols[:, bins])
    return np.concatenate(packed, axis=1), np.concatenate(full, axis=1)
