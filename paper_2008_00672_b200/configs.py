"""The BASELINE.json workloads as plan specifications.

Synthetic stand-ins: there is no dataset; every config is seeded random QAM on
the allocation BASELINE.json describes.  Subband allocations are contiguous
and centred on DC; each subband's active bins are ``centered_active_map(L,
n_sc, skip_dc=False)`` around its centre bin, so subcarrier ``ls`` of subband
m lands on grid bin ``c_m + ls`` (fc_core.cpp:81-84), and its window is
``design_window(L, n_sc, n_tb)`` (fc_core.cpp:25-39).

Geometry backends.  Every builder takes ``geom``: an object with
``design_window(L, n_pass, n_tb)``, ``centered_active_map(L, n, skip_dc)``,
``cp(scs_khz, N, B)`` (the reference's cp_schedule), ``nr_cp(scs_khz, N, B)``
(5G-NR normal CP) and ``subband(**fields)``.  The default (``ApiGeometry``)
computes through this package's C ABI; bench.py's reference arm passes the
oracle's restatement instead, so that arm never loads the product library
(``tests/test_capi.py`` checks both backends give bit-identical geometry).
This module imports nothing from the product at import time.
"""
from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace
from typing import Any


class ApiGeometry:
    """Geometry through the product's C ABI (fcw_design_window, ...)."""

    def __init__(self):
        from . import api

        self.api = api

    def design_window(self, L, n_pass, n_tb):
        return self.api.design_window(L, n_pass, n_tb)

    def centered_active_map(self, L, n, skip_dc=True):
        return self.api.centered_active_map(L, n, skip_dc)

    def cp(self, scs_khz, N, B):
        return self.api.cp_schedule(self.api.make_numerology(scs_khz, N), B).per_symbol_high_rate

    def nr_cp(self, scs_khz, N, B):
        return self.api.nr_cp_schedule(self.api.make_numerology(scs_khz, N), B).per_symbol_high_rate

    def subband(self, **kw):
        return self.api.SubbandConfig(**kw)


def plain_subband(**kw):
    """A SubbandConfig-shaped record for geometry backends outside the product."""
    kw.setdefault("n_active", 0)
    kw.setdefault("n_tb", 0)
    kw.setdefault("l_ofdm", kw["L"])
    return SimpleNamespace(**kw)


def _geom(geom):
    return ApiGeometry() if geom is None else geom


@dataclass
class Workload:
    name: str
    N: int
    scs_khz: int
    cp: list[int]
    subbands: list[Any]
    active_maps: list[list[int]]
    bits_per_symbol: int
    units: int  # independent (antenna stream x frame) units of the full workload
    description: str

    @property
    def B(self) -> int:
        return len(self.cp)

    def plan(self):
        from . import api

        return api.Plan(self.N, self.cp, self.subbands, self.active_maps)


def _contiguous(geom, N: int, n_sc: list[int], Ls: list[int], n_tb: int) -> tuple[list[Any], list[list[int]]]:
    total = sum(n_sc)
    start = -(total // 2)
    subs, maps = [], []
    for n, L in zip(n_sc, Ls):
        c = (start + n // 2) % N
        subs.append(geom.subband(L=L, c=c, window=geom.design_window(L, n, n_tb), n_active=n, n_tb=n_tb, l_ofdm=L))
        maps.append(list(geom.centered_active_map(L, n, False)))
        start += n
    return subs, maps


def _pow2_at_least(v: int) -> int:
    p = 1
    while p < v:
        p *= 2
    return p


def config1(geom=None) -> Workload:
    """Mini-slot: 15 kHz, N=1024, 2 symbols, 1 PRB (12 sc), L=16, n_tb=2, QPSK.
    CP: the reference's cp_schedule preset [80, 72] (numerology.cpp:29-42,
    long CP on symbol 0); BASELINE.json's "normal CP of 72" is symbol 1's.
    bench.py states this in its config line."""
    geom = _geom(geom)
    N = 1024
    cp = list(geom.cp(15, N, 2))  # [80, 72]
    subs, maps = _contiguous(geom, N, [12], [16], 2)
    return Workload("c1_minislot_1prb_L16_N1024", N, 15, cp, subs, maps, 2, 65536,
                    "15 kHz, N=1024, B=2, 1x(L=16, 12 active, n_tb=2), QPSK; batch of 65536 instances; "
                    "CP [80, 72] = the reference's cp_schedule preset")


def config2(geom=None) -> Workload:
    """20 MHz full slot: 15 kHz, N=2048, 14 symbols, 106 PRB = 24/24/24/34 PRB, L=512, n_tb=4, 16-QAM."""
    geom = _geom(geom)
    N = 2048
    cp = list(geom.cp(15, N, 14))  # 160 at n%7==0, else 144
    n_sc = [24 * 12, 24 * 12, 24 * 12, 34 * 12]
    Ls = [_pow2_at_least(n + 8) for n in n_sc]
    subs, maps = _contiguous(geom, N, n_sc, Ls, 4)
    return Workload("c2_20mhz_slot_4sb_L512_N2048", N, 15, cp, subs, maps, 4, 1024,
                    "15 kHz, N=2048, B=14, 4x(L=512, 288/288/288/408 active, n_tb=4), 16-QAM")


def config4(streams: int = 4, geom=None) -> Workload:
    """100 MHz frame: 30 kHz, N=4096, 280 symbols, 273 x 1-PRB subbands, L=16, 256-QAM, 4 streams."""
    geom = _geom(geom)
    N = 4096
    cp = list(geom.nr_cp(30, N, 280))  # 352 every 14, else 288
    subs, maps = _contiguous(geom, N, [12] * 273, [16] * 273, 2)
    return Workload("c4_100mhz_frame_273sb_L16_N4096", N, 30, cp, subs, maps, 8, streams,
                    "30 kHz, N=4096, B=280, 273x(L=16, 12 active, n_tb=2), 256-QAM, 4 antenna streams")


def config5(streams: int = 64, frames: int = 8, geom=None) -> Workload:
    """Multi-antenna sweep: 30 kHz, N=4096, 280 symbols, 22x12 PRB + 1x9 PRB subbands, L=256, 256-QAM."""
    geom = _geom(geom)
    N = 4096
    cp = list(geom.nr_cp(30, N, 280))
    subs, maps = _contiguous(geom, N, [144] * 22 + [108], [256] * 23, 4)
    return Workload("c5_100mhz_64ant_x8frames_23sb_L256_N4096", N, 30, cp, subs, maps, 8, streams * frames,
                    "30 kHz, N=4096, B=280, 22x(L=256,144 active)+1x(L=256,108 active), n_tb=4, 256-QAM, "
                    "64 antenna streams x 8 frames")


@dataclass
class MixedWorkload:
    """Config 3: two numerologies on one 30.72 Msps carrier.
    Bank A: 15 kHz, N=2048, 48 PRB (576 sc), L=1024, CP 144, 14 symbols.
    Bank B: 30 kHz, N=1024, 24 PRB (288 sc), L=512, CP 72, 28 symbols.
    Guard: 2 PRB at 30 kHz (720 kHz) between them.  Both span 1 ms; B's
    waveform is offset by +184 samples so both symbol-0 CPs start together."""

    name: str
    banks: list[Workload]
    offsets: list[int]
    bits_per_symbol: int
    units: int
    description: str

    def plans(self) -> list:
        return [w.plan() for w in self.banks]

    def mixed(self, plans: list):
        from . import api

        return api.MixedNumerology(list(zip(plans, self.offsets)))


def config3(geom=None) -> MixedWorkload:
    geom = _geom(geom)
    fs_khz = 30720
    # bank A (15 kHz bins on N=2048): occupies [-9.00, -0.36) MHz
    NA, NB = 2048, 1024
    a_lo = -600  # in 15 kHz bins
    a_sc = 576
    cA = (a_lo + a_sc // 2) % NA
    subA = geom.subband(L=1024, c=cA, window=geom.design_window(1024, a_sc, 4), n_active=a_sc, n_tb=4, l_ofdm=1024)
    wA = Workload("c3_bankA_15khz", NA, 15, [144] * 14, [subA], [list(geom.centered_active_map(1024, a_sc, False))],
                  6, 1, "15 kHz, N=2048, 48 PRB, L=1024")
    # bank B (30 kHz bins on N=1024): occupies [+0.36, +9.00) MHz
    b_lo = 12  # in 30 kHz bins (guard [-0.36, +0.36) MHz = 2 PRB at 30 kHz)
    b_sc = 288
    cB = (b_lo + b_sc // 2) % NB
    subB = geom.subband(L=512, c=cB, window=geom.design_window(512, b_sc, 4), n_active=b_sc, n_tb=4, l_ofdm=512)
    wB = Workload("c3_bankB_30khz", NB, 30, [72] * 28, [subB], [list(geom.centered_active_map(512, b_sc, False))],
                  6, 1, "30 kHz, N=1024, 24 PRB, L=512")
    # align the symbol-0 CP starts: N_L,A - N_CP,A = 512 - 144 = 368; N_L,B - N_CP,B = 256 - 72 = 184
    off_b = (NA // 4 - 144) - (NB // 4 - 72)
    assert fs_khz == 15 * NA == 30 * NB
    return MixedWorkload("c3_mixed_numerology_20mhz", [wA, wB], [0, off_b], 6, 1024,
                         "15 kHz N=2048 48 PRB + 30 kHz N=1024 24 PRB, 2 PRB guard, 64-QAM, 1 ms units, fused RX")


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}


def get(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)


def algorithmic_bytes_per_unit(w: Workload, row_active: int, Q: int) -> dict:
    """TX reads the packed grid and writes Q samples; RX reads
    Q samples and writes the packed grid; complex fp32 = 8 B."""
    grid = 8 * w.B * row_active
    wave = 8 * Q
    return {"tx": grid + wave, "rx": grid + wave, "total": 2 * (grid + wave)}
