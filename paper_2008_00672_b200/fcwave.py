"""Drop-in for the reference's Python module ``_fcwave`` (proj/python/module.cpp:34-117),
hot-path subset: same function names, argument order, defaults and error
classes, backed by the sm_100a kernels.

    import paper_2008_00672_b200.fcwave as fc   # instead of: import _fcwave as fc
"""
from __future__ import annotations

import numpy as np

from . import api


def cp_schedule(scs_khz: int, n_fft: int, n_symbols: int) -> list[int]:  # module.cpp:50-52
    return api.cp_schedule(api.make_numerology(scs_khz, n_fft), n_symbols).per_symbol_high_rate


def derive_fc_params(N: int, L: int, overlap: float) -> api.FcParams:  # module.cpp:53
    return api.derive_fc_params(N, L, overlap)


def first_block_overlap(p: api.FcParams, l_cp: int) -> float:  # module.cpp:54
    return api.first_block_overlap(p, l_cp)


def cp_truncate(n_cp: int, I: int) -> tuple[int, int]:  # module.cpp:55-58
    return api.cp_truncate(n_cp, I)


def design_window(L: int, n_pass: int, n_tb: int) -> list[float]:  # module.cpp:59
    return api.design_window(L, n_pass, n_tb).tolist()


def _cfg(L: int, c: int, n_active: int, n_tb: int, n_pass: int) -> api.SubbandConfig:  # module.cpp:21-30
    return api.SubbandConfig(L=L, c=c, window=api.design_window(L, n_pass, n_tb), n_active=n_active, n_tb=n_tb,
                             l_ofdm=L)


def tx_discontinuous(grid_cols, L: int, N: int, c: int, n_active: int, n_tb: int, n_pass: int,
                     scs_khz: int = 15):  # module.cpp:77-92
    num = api.make_numerology(scs_khz, N)
    cols = [np.asarray(col, dtype=np.complex128) for col in grid_cols]
    cps = api.cp_schedule(num, len(cols))
    g = api.QamGrid(l_ofdm=L, active_map=[], symbols=cols)
    w = api.tx_discontinuous([g], [_cfg(L, c, n_active, n_tb, n_pass)], cps, N, 0.5, num.fs_hz())
    return w.samples, w.useful0


def rx_discontinuous(samples, useful0: int, n_symbols: int, L: int, N: int, c: int, n_active: int, n_tb: int,
                     n_pass: int, simplified: bool = False, scs_khz: int = 15):  # module.cpp:94-109
    num = api.make_numerology(scs_khz, N)
    w = api.Waveform(np.asarray(samples, dtype=np.complex128), num.fs_hz(), int(useful0))
    cps = api.cp_schedule(num, n_symbols)
    return api.rx_discontinuous(w, _cfg(L, c, n_active, n_tb, n_pass), cps, N, 0.5, simplified)
