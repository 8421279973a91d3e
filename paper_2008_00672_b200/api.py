"""Python host API of fcwave-b200, mirroring the reference's operator API.

Reference-shaped entry points (proj/include/fcwave/fc_sync.hpp,
numerology.hpp, fc_core.hpp, ofdm.hpp) take and return numpy complex128 like
the reference's std::complex<double> vectors; the work runs on the GPU through
the C ABI.  ``Plan`` is the batched, device-resident engine that bench.py and
production callers use: torch CUDA tensors (or raw device pointers) in and out,
S independent (antenna stream x frame) units per call.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import FCW_GRID_FULL, FCW_RX_FUSED, FCW_TX_ACCUMULATE, check, lib


# ------------------------------------------------------------------ geometry
@dataclass
class Numerology:  # numerology.hpp:14-20
    scs_khz: int = 15
    n_fft: int = 1024
    symbols_per_half_subframe: int = 7

    def fs_hz(self) -> float:
        return float(self.scs_khz) * 1000.0 * self.n_fft


@dataclass
class CpSchedule:  # numerology.hpp:23-31
    per_symbol_high_rate: list[int]

    def total(self) -> int:
        return int(sum(self.per_symbol_high_rate))


@dataclass
class FcParams:  # numerology.hpp:34-41
    L: int
    N: int
    overlap: float
    L_O: int
    L_S: int
    L_L: int
    L_T: int
    N_O: int
    N_S: int
    N_L: int
    N_T: int
    I: int

    def _c(self) -> _lib.FcParamsC:
        p = _lib.FcParamsC()
        for k in self.__dataclass_fields__:
            setattr(p, k, getattr(self, k))
        return p


@dataclass
class SubbandConfig:  # fc_core.hpp:20-27
    L: int
    c: int
    window: np.ndarray
    n_active: int = 0
    n_tb: int = 0
    l_ofdm: int = 0

    def __post_init__(self):
        self.window = np.ascontiguousarray(np.asarray(self.window, dtype=np.float64))
        if self.l_ofdm == 0:
            self.l_ofdm = self.L


@dataclass
class QamGrid:  # ofdm.hpp:27-33
    l_ofdm: int
    active_map: list[int] = field(default_factory=list)
    symbols: list = field(default_factory=list)  # B columns of l_ofdm complex

    def n_symbols(self) -> int:
        return len(self.symbols)


@dataclass
class Waveform:  # types.hpp:22-26
    samples: np.ndarray
    fs_hz: float = 0.0
    useful0: int = 0


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def make_numerology(scs_khz: int, n_fft: int) -> Numerology:
    """numerology.cpp:17-27: same checks and messages, in the host layer (the
    C ABI validates again in every call that takes a numerology)."""
    if n_fft < 16 or n_fft & (n_fft - 1):
        raise ValueError("n_fft must be a power of two >= 16")
    if scs_khz <= 0 or scs_khz % 15 or (scs_khz // 15) & (scs_khz // 15 - 1):
        raise ValueError("scs_khz must be 15*2^k")
    return Numerology(scs_khz, n_fft, 7)


def cp_schedule(num: Numerology, n_symbols: int) -> CpSchedule:
    out = np.zeros(max(n_symbols, 1), np.int32)
    check(lib().fcw_cp_schedule(num.scs_khz, num.n_fft, n_symbols, _i32p(out)))
    return CpSchedule(out.tolist())


def nr_cp_schedule(num: Numerology, n_symbols: int) -> CpSchedule:
    """5G-NR normal CP for any 15*2^mu kHz (288/352 at 30 kHz, N=4096)."""
    out = np.zeros(max(n_symbols, 1), np.int32)
    check(lib().fcw_nr_cp_schedule(num.scs_khz, num.n_fft, n_symbols, _i32p(out)))
    return CpSchedule(out.tolist())


def derive_fc_params(N: int, L: int, overlap: float = 0.5) -> FcParams:
    p = _lib.FcParamsC()
    check(lib().fcw_derive_fc_params(N, L, overlap, C.byref(p)))
    return FcParams(**{k: getattr(p, k) for k, _ in _lib.FcParamsC._fields_})


def first_block_overlap(p: FcParams, l_cp: int) -> float:
    v = C.c_double()
    pc = p._c()
    check(lib().fcw_first_block_overlap(C.byref(pc), l_cp, C.byref(v)))
    return v.value


def cp_truncate(n_cp_high: int, I: int) -> tuple[int, int]:
    a, b = C.c_int(), C.c_int()
    check(lib().fcw_cp_truncate(n_cp_high, I, C.byref(a), C.byref(b)))
    return a.value, b.value


def design_window(L: int, n_pass: int, n_tb: int) -> np.ndarray:
    w = np.zeros(max(L, 1), np.float64)
    check(lib().fcw_design_window(L, n_pass, n_tb, w.ctypes.data_as(C.POINTER(C.c_double))))
    return w[:L]


def centered_active_map(l_ofdm: int, n_active: int, skip_dc: bool = True) -> list[int]:
    b = np.zeros(max(n_active, 1), np.int32)
    check(lib().fcw_centered_active_map(l_ofdm, n_active, int(skip_dc), _i32p(b)))
    return b[:n_active].tolist()


def symbol_phase(n: int, c: int, cps: CpSchedule, N: int) -> complex:
    """symbol_phase (fc_sync.cpp:45-50), double precision."""
    cp = _i32(cps.per_symbol_high_rate)
    a, b = C.c_double(), C.c_double()
    check(lib().fcw_symbol_phase(n, c, _i32p(cp), len(cp), N, C.byref(a), C.byref(b)))
    return complex(a.value, b.value)


def block_phase(r: int, c: int, L_S: int, L: int) -> complex:
    """block_phase (fc_core.cpp:41-44), double precision."""
    a, b = C.c_double(), C.c_double()
    check(lib().fcw_block_phase(r, c, L_S, L, C.byref(a), C.byref(b)))
    return complex(a.value, b.value)


def symbol_sigma(n: int, cps: CpSchedule, N: int) -> int:
    cp = _i32(cps.per_symbol_high_rate)
    return int(lib().fcw_symbol_sigma(n, _i32p(cp), N))


def combined_length(n_symbols: int, cps: CpSchedule, p: FcParams) -> int:
    cp = _i32(cps.per_symbol_high_rate)
    pc = p._c()
    return int(lib().fcw_combined_length(n_symbols, _i32p(cp), C.byref(pc)))


# ------------------------------------------------------------------- engine
def _dev_ptr(x) -> int:
    """Raw device pointer of a torch CUDA tensor (or pass an int through)."""
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_cuda:
            raise ValueError("device entry point needs a CUDA tensor")
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    raise TypeError(f"unsupported buffer {type(x)}")


def _stream_ptr(stream) -> int | None:
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Plan:
    """Immutable device-resident FC-F-OFDM plan (fcw_plan_create).

    subbands: SubbandConfig list; active_maps: per subband the active DFT bins
    (packed grid order).  Defaults to the full L bins of each subband.
    """

    def __init__(self, N: int, cps: CpSchedule | Sequence[int], subbands: Sequence[SubbandConfig],
                 active_maps: Sequence[Sequence[int]] | None = None, overlap: float = 0.5):
        cp = cps.per_symbol_high_rate if isinstance(cps, CpSchedule) else list(cps)
        self.cp = _i32(cp)
        self.N, self.B, self.M = N, len(cp), len(subbands)
        self.subbands = list(subbands)
        if active_maps is None:
            active_maps = [list(range(s.L)) for s in subbands]
        if len(active_maps) != len(subbands):
            raise ValueError("one active map per subband required")
        self._bins = [_i32(a) for a in active_maps]
        arr = (_lib.SubbandC * max(1, self.M))()
        for m, s in enumerate(subbands):
            if len(s.window) != s.L:
                raise ValueError("window length must be L")
            arr[m].L, arr[m].l_ofdm, arr[m].c = s.L, s.l_ofdm, s.c
            arr[m].n_active, arr[m].n_tb = len(self._bins[m]), s.n_tb
            arr[m].active_bins = _i32p(self._bins[m])
            arr[m].window = s.window.ctypes.data_as(C.POINTER(C.c_double))
        h = C.c_void_p()
        check(lib().fcw_plan_create(C.byref(h), N, overlap, _i32p(self.cp), self.B, arr, self.M, 0))
        self._h = h
        info = _lib.PlanInfoC()
        check(lib().fcw_plan_get_info(self._h, C.byref(info)))
        self.Q = int(info.Q)
        self.useful0 = int(info.useful0)
        self.frame_samples = int(info.frame_samples)
        self.row_active = int(info.row_active)
        self.row_full = int(info.row_full)
        self.N_L, self.N_T = int(info.N_L), int(info.N_T)
        self.chunk = int(info.chunk)
        # informational: 0 general, 1 zero-bin (TMEM tables), 2 narrowband, 3 team-only kernels
        self.kernel_variant, self.tmem_rows = int(info.kernel_variant), int(info.tmem_rows)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().fcw_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- geometry queries (bit-exact checks against the oracle)
    def sigma(self) -> np.ndarray:
        out = np.zeros(self.B, np.int64)
        check(lib().fcw_plan_sigma(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def cp_split(self, m: int) -> tuple[np.ndarray, np.ndarray]:
        a, b = np.zeros(self.B, np.int32), np.zeros(self.B, np.int32)
        check(lib().fcw_plan_cp_split(self._h, m, _i32p(a), _i32p(b)))
        return a, b

    def bin_map(self, m: int) -> tuple[np.ndarray, np.ndarray]:
        L = self.subbands[m].L if 0 <= m < self.M else 1
        q, b = np.zeros(L, np.int32), np.zeros(L, np.int32)
        check(lib().fcw_plan_bin_map(self._h, m, _i32p(q), _i32p(b)))
        return q, b

    def rx_starts(self, useful0: int) -> np.ndarray:
        out = np.zeros(self.B, np.int64)
        check(lib().fcw_plan_rx_starts(self._h, useful0, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def fc_params(self, m: int) -> FcParams:
        p = _lib.FcParamsC()
        check(lib().fcw_plan_fc_params(self._h, m, C.byref(p)))
        return FcParams(**{k: getattr(p, k) for k, _ in _lib.FcParamsC._fields_})

    def row(self, full: bool = False) -> int:
        return self.row_full if full else self.row_active

    # -- device entry points
    def tx(self, grid, wave, S: int, full: bool = False, stream=None, grid_stride: int = 0,
           wave_stride: int = 0, accumulate: bool = False) -> None:
        flags = (FCW_GRID_FULL if full else 0) | (FCW_TX_ACCUMULATE if accumulate else 0)
        check(lib().fcw_tx(self._h, _dev_ptr(grid), grid_stride, _dev_ptr(wave), wave_stride, S, flags,
                           _stream_ptr(stream)))

    def rx(self, wave, wave_len: int, useful0: int, grid, S: int, fused: bool = True, full: bool = False,
           stream=None, wave_stride: int = 0, grid_stride: int = 0) -> None:
        flags = (FCW_RX_FUSED if fused else 0) | (FCW_GRID_FULL if full else 0)
        check(lib().fcw_rx(self._h, _dev_ptr(wave), wave_stride, wave_len, useful0, _dev_ptr(grid), grid_stride, S,
                           flags, _stream_ptr(stream)))

    def gen_qam(self, seed: int, unit0: int, S: int, bits_per_symbol: int, grid, stream=None) -> None:
        check(lib().fcw_gen_qam(self._h, seed, unit0, S, bits_per_symbol, _dev_ptr(grid), _stream_ptr(stream)))

    # -- reference-granularity per-symbol entry points (fc_sync.hpp:38-75),
    #    batched over S units of one (subband m, symbol n); device buffers
    def tx_symbol(self, m: int, n: int, sym, l_cp: int, out, S: int, stream=None, sym_stride: int = 0,
                  out_stride: int = 0) -> None:
        """tx_symbol (fc_sync.cpp:60-84): sym [S][L + l_cp] -> out [S][3N/2]."""
        check(lib().fcw_tx_symbol(self._h, m, n, _dev_ptr(sym), sym_stride, l_cp, _dev_ptr(out), out_stride, S,
                                  _stream_ptr(stream)))

    def combine_symbols(self, syms, wave, S: int, stream=None, sym_unit_stride: int = 0,
                        wave_stride: int = 0) -> None:
        """combine_symbols (fc_sync.cpp:96-112): syms [S][B][3N/2] -> wave [S][Q]."""
        check(lib().fcw_combine_symbols(self._h, _dev_ptr(syms), sym_unit_stride, _dev_ptr(wave), wave_stride, S,
                                        _stream_ptr(stream)))

    def rx_segment(self, wave, wave_len: int, useful0: int, n: int, y0, y1, S: int, stream=None,
                   wave_stride: int = 0, y_stride: int = 0) -> None:
        """rx_segment (fc_sync.cpp:145-156): the two N-sample blocks of symbol n."""
        check(lib().fcw_rx_segment(self._h, _dev_ptr(wave), wave_stride, wave_len, useful0, n, _dev_ptr(y0),
                                   _dev_ptr(y1), y_stride, S, _stream_ptr(stream)))

    def rx_block_freq(self, m: int, y, phase: complex, g, S: int, stream=None, y_stride: int = 0,
                      g_stride: int = 0) -> None:
        """rx_block_freq (fc_sync.cpp:178-193): y [S][N] -> g [S][L_m]."""
        check(lib().fcw_rx_block_freq(self._h, m, _dev_ptr(y), y_stride, float(phase.real), float(phase.imag),
                                      _dev_ptr(g), g_stride, S, _stream_ptr(stream)))

    def rx_symbol_simplified(self, m: int, g0, g1, out, S: int, stream=None, g_stride: int = 0,
                             out_stride: int = 0) -> None:
        """rx_symbol_simplified (fc_sync.cpp:195-243), Eq. (30): g0, g1 [S][L] -> out [S][L]."""
        check(lib().fcw_rx_symbol_simplified(self._h, m, _dev_ptr(g0), _dev_ptr(g1), g_stride, _dev_ptr(out),
                                             out_stride, S, _stream_ptr(stream)))

    def rx_symbol_direct(self, m: int, n: int, y0, y1, out, S: int, stream=None, y_stride: int = 0,
                         out_stride: int = 0) -> None:
        """rx_symbol_direct (fc_sync.cpp:158-176): y0, y1 [S][N] -> out [S][L]."""
        check(lib().fcw_rx_symbol_direct(self._h, m, n, _dev_ptr(y0), _dev_ptr(y1), y_stride, _dev_ptr(out),
                                         out_stride, S, _stream_ptr(stream)))

    # -- host entry points (numpy complex64, C-contiguous)
    # ---- link step around the path
    def link_stats(self, grid, S: int, seed: int, unit0: int, bits_per_symbol: int, stream=None,
                   grid_stride: int = 0) -> "LinkStats":
        """Per-unit EVM sums and hard-decision bit errors of a received packed
        device grid against the seeded transmit grid (scenario.cpp:469-494)."""
        out = (_lib.LinkStatC * max(S, 1))()
        check(lib().fcw_link_stats(self._h, _dev_ptr(grid), grid_stride, S, seed, unit0, bits_per_symbol, out,
                                   _stream_ptr(stream)))
        return LinkStats(np.array([o.evm_num for o in out[:S]]), np.array([o.evm_den for o in out[:S]]),
                         np.array([o.bit_errors for o in out[:S]], np.int64),
                         np.array([o.n_bits for o in out[:S]], np.int64))

    def awgn(self, wave, wave_len: int, S: int, sigma2: float, seed: int, unit0: int = 0, stream=None,
             wave_stride: int = 0) -> None:
        """awgn_with_variance (channel.cpp:136-141) in place on S device waveforms."""
        check(lib().fcw_awgn(self._h, _dev_ptr(wave), wave_stride, wave_len, S, sigma2, seed, unit0,
                             _stream_ptr(stream)))

    def wave_power(self, wave, wave_len: int, S: int, begin: int, end: int, stream=None,
                   wave_stride: int = 0) -> np.ndarray:
        """measure_power (channel.cpp:148-155) per unit."""
        out = (C.c_double * max(S, 1))()
        check(lib().fcw_wave_power(self._h, _dev_ptr(wave), wave_stride, wave_len, S, begin, end, out,
                                   _stream_ptr(stream)))
        return np.array(out[:S])

    def tx_host(self, grid: np.ndarray, S: int, full: bool = False, out: np.ndarray | None = None) -> np.ndarray:
        g = np.ascontiguousarray(grid, dtype=np.complex64)
        if g.size != S * self.B * self.row(full):
            raise ValueError("grid size does not match S*B*row")
        if out is None:
            out = np.empty((S, self.Q), np.complex64)
        check(lib().fcw_tx_host(self._h, g.ctypes.data, out.ctypes.data, S, FCW_GRID_FULL if full else 0))
        return out

    def _raw(self):
        return self._h

    def rx_host(self, wave: np.ndarray, wave_len: int, useful0: int, S: int, fused: bool = True, full: bool = False,
                out: np.ndarray | None = None) -> np.ndarray:
        w = np.ascontiguousarray(wave, dtype=np.complex64)
        if w.size != S * wave_len:
            raise ValueError("waveform size does not match S*wave_len")
        if out is None:
            out = np.empty((S, self.B, self.row(full)), np.complex64)
        flags = (FCW_RX_FUSED if fused else 0) | (FCW_GRID_FULL if full else 0)
        check(lib().fcw_rx_host(self._h, w.ctypes.data, wave_len, useful0, out.ctypes.data, S, flags))
        return out


class MixedNumerology:
    """Several single-numerology FC banks sharing one sample rate and one
    waveform (the paper's mixed-numerology use, Eq. (20b) with
    N_OFDM,m per bank).  The reference can only express one numerology per
    call (fc_sync.cpp:62-63,87); this composes banks on the device:

      TX: bank 0 stores its waveform, every further bank ADDS its own at a
          sample offset (FCW_TX_ACCUMULATE, the reference's `w += sub`,
          fc_sync.cpp:139).
      RX: each bank analyses the shared waveform with its own useful0
          (offset + its N_L).

    banks: list of (Plan, sample offset) with offsets >= 0.
    """

    def __init__(self, banks: Sequence[tuple[Plan, int]]):
        if not banks:
            raise ValueError("at least one bank required")
        self.banks = [(p, int(off)) for p, off in banks]
        for _, off in self.banks:
            if off < 0:
                raise ValueError("bank offsets must be >= 0")
        self.Q = max(off + p.Q for p, off in self.banks)
        self.frame_samples = max(p.frame_samples for p, _ in self.banks)

    def tx(self, grids, wave, S: int, stream=None) -> None:
        """grids[i]: device packed grid of bank i; wave: device complex64 [S][Q].
        Samples outside bank 0's span are zeroed first: later banks add onto them."""
        base = _dev_ptr(wave)
        p0, off0 = self.banks[0]
        check(lib().fcw_wave_zero(base, self.Q, S, 0, off0, _stream_ptr(stream)))
        check(lib().fcw_wave_zero(base, self.Q, S, off0 + p0.Q, self.Q, _stream_ptr(stream)))
        for i, ((p, off), g) in enumerate(zip(self.banks, grids)):
            p.tx(g, base + 8 * off, S, stream=stream, wave_stride=self.Q, accumulate=i > 0)

    def rx(self, wave, outs, S: int, fused: bool = True, stream=None) -> None:
        base = _dev_ptr(wave)
        for (p, off), o in zip(self.banks, outs):
            p.rx(base, self.Q, off + p.useful0, o, S, fused=fused, stream=stream, wave_stride=self.Q)


class PinnedBuffer:
    """Page-locked host buffer (fcw_host_alloc) exposed as ``.array`` (numpy)."""

    def __init__(self, shape, dtype=np.complex64):
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self._ptr = lib().fcw_host_alloc(max(n, 1))
        if not self._ptr:
            check(_lib.FCW_ENOMEM)
        raw = np.ctypeslib.as_array(C.cast(self._ptr, C.POINTER(C.c_uint8)), shape=(max(n, 1),))
        self.array = raw[:n].view(dtype).reshape(shape)

    def __del__(self):
        if getattr(self, "_ptr", None):
            lib().fcw_host_free(self._ptr)
            self._ptr = None


# ------------------------------------------------- reference-shaped functions
def _full_grid_rows(grids: Sequence[QamGrid], cfgs: Sequence[SubbandConfig], B: int) -> np.ndarray:
    cols = []
    for g, c in zip(grids, cfgs):
        a = np.asarray(g.symbols, dtype=np.complex128).reshape(B, -1)
        if a.shape[1] != c.L:
            raise ValueError("grid column size mismatch")
        cols.append(a)
    return np.concatenate(cols, axis=1).astype(np.complex64)


def tx_discontinuous(grids: Sequence[QamGrid], cfgs: Sequence[SubbandConfig], cps: CpSchedule, N: int,
                     overlap: float, fs_hz: float) -> Waveform:
    """fc_sync.hpp:52-54 — all subbands through ONE shared N-point transform per block."""
    if len(grids) != len(cfgs) or not grids:
        raise ValueError("one config per grid required")
    B = len(cps.per_symbol_high_rate)
    for g in grids:
        if g.n_symbols() != B:
            raise ValueError("grid symbol count must match CP schedule")
    plan = Plan(N, cps, cfgs, overlap=overlap)
    rows = _full_grid_rows(grids, cfgs, B)
    w = plan.tx_host(rows.reshape(-1), 1, full=True)[0]
    return Waveform(w.astype(np.complex128), fs_hz, plan.useful0)


def rx_discontinuous_all(w: Waveform, cfgs: Sequence[SubbandConfig], cps: CpSchedule, N: int, overlap: float,
                         simplified: bool = False) -> list[np.ndarray]:
    """All subbands in one pass; returns per subband a (B, L) complex128 array."""
    plan = Plan(N, cps, cfgs, overlap=overlap)
    if simplified:
        for c in cfgs:
            if derive_fc_params(N, c.L, overlap).L_S * 2 != c.L:
                raise ValueError("fused RX path requires 50 % overlap")
    samples = np.asarray(w.samples)
    out = plan.rx_host(samples.reshape(-1), len(samples), int(w.useful0), 1, fused=simplified, full=True)[0]
    res, off = [], 0
    for c in cfgs:
        res.append(out[:, off:off + c.L].astype(np.complex128))
        off += c.L
    return res


def rx_discontinuous(w: Waveform, cfg: SubbandConfig, cps: CpSchedule, N: int, overlap: float,
                     simplified: bool = False) -> list[np.ndarray]:
    """fc_sync.hpp:78-80 — returns B columns of L complex values."""
    return list(rx_discontinuous_all(w, [cfg], cps, N, overlap, simplified)[0])


# ------------------------------------------- continuous FC filterbank (f2)
@dataclass
class CpOfdmSignal:  # ofdm.hpp:52-56
    samples: np.ndarray
    cp_lengths: list[int] = field(default_factory=list)
    l_ofdm: int = 0


class ContPlan:
    """Device plan of the continuous FC filterbank (tx_continuous /
    rx_continuous, fc_core.hpp:64-77) for fixed subbands, per-subband TX stream
    lengths and RX waveform length; batched over S units like Plan."""

    def __init__(self, N: int, subbands: Sequence[SubbandConfig], stream_len: Sequence[int], rx_wave_len: int,
                 l_cp0: int = 0, overlap: float = 0.5):
        self.N, self.M = N, len(subbands)
        self.subbands = list(subbands)
        arr = (_lib.SubbandC * max(1, self.M))()
        for m, sb in enumerate(subbands):
            if len(sb.window) != sb.L:
                raise ValueError("window length must be L")
            arr[m].L, arr[m].l_ofdm, arr[m].c = sb.L, sb.L, sb.c
            arr[m].n_active, arr[m].n_tb = 0, sb.n_tb
            arr[m].active_bins = None
            arr[m].window = sb.window.ctypes.data_as(C.POINTER(C.c_double))
        lens = (C.c_int64 * max(1, self.M))(*[int(x) for x in stream_len])
        h = C.c_void_p()
        check(lib().fcw_cont_plan_create(C.byref(h), N, overlap, arr, self.M, lens, int(rx_wave_len), int(l_cp0)))
        self._h = h
        info = _lib.ContInfoC()
        lo = (C.c_int64 * max(1, self.M))()
        oo = (C.c_int64 * max(1, self.M))()
        check(lib().fcw_cont_plan_get_info(self._h, C.byref(info), lo, oo))
        self.tx_len, self.tx_stride, self.useful0 = int(info.tx_len), int(info.tx_stride), int(info.useful0)
        self.stream_total, self.rx_wave_len = int(info.stream_total), int(info.rx_wave_len)
        self.rx_out_total = int(info.rx_out_total)
        self.rx_out_len = [int(lo[m]) for m in range(self.M)]
        self.rx_out_off = [int(oo[m]) for m in range(self.M)]
        self.stream_len = [int(x) for x in stream_len]

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().fcw_cont_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tx(self, streams, wave, S: int, stream=None) -> None:
        """streams: device complex64 [S][stream_total]; wave: [S][tx_stride]."""
        check(lib().fcw_tx_continuous(self._h, _dev_ptr(streams), _dev_ptr(wave), S, _stream_ptr(stream)))

    def rx(self, wave, out, S: int, stream=None) -> None:
        """wave: device complex64 [S][rx_wave_len]; out: [S][rx_out_total]."""
        check(lib().fcw_rx_continuous(self._h, _dev_ptr(wave), _dev_ptr(out), S, _stream_ptr(stream)))


def tx_continuous(signals: Sequence[CpOfdmSignal], cfgs: Sequence[SubbandConfig], N: int, overlap: float,
                  fs_hz: float) -> Waveform:
    """fc_core.hpp:71-73 on the GPU (one unit, host arrays)."""
    import torch

    if len(signals) != len(cfgs) or not signals:
        raise ValueError("one config per subband signal required")  # fc_core.cpp:166
    lens = [len(sg.samples) for sg in signals]
    l_cp0 = signals[0].cp_lengths[0] if signals[0].cp_lengths else 0
    p = ContPlan(N, cfgs, lens, max(N, 1), l_cp0, overlap)
    flat = np.concatenate([np.asarray(sg.samples, np.complex64) for sg in signals])
    d_in = torch.from_numpy(flat).cuda()
    d_out = torch.empty(p.tx_stride, dtype=torch.complex64, device="cuda")
    p.tx(d_in, d_out, 1)
    torch.cuda.synchronize()
    return Waveform(d_out.cpu().numpy()[: p.tx_len].astype(np.complex128), fs_hz, p.useful0)


def rx_continuous(w: Waveform, cfg: SubbandConfig, p: FcParams) -> np.ndarray:
    """fc_core.hpp:77 on the GPU for one subband (p: derive_fc_params)."""
    import torch

    n = len(w.samples)
    if n < p.N:
        raise ValueError("waveform shorter than one FC block")  # fc_core.cpp:201
    cp = ContPlan(p.N, [cfg], [0], n, 0, p.overlap)
    d_w = torch.from_numpy(np.asarray(w.samples, np.complex64)).cuda()
    d_o = torch.empty(cp.rx_out_total, dtype=torch.complex64, device="cuda")
    cp.rx(d_w, d_o, 1)
    torch.cuda.synchronize()
    return d_o.cpu().numpy().astype(np.complex128)


# ------------------------------------------------------------ link metrics
@dataclass
class LinkStats:
    """Per-unit sums of the link step (scenario.cpp:481-491)."""
    evm_num: np.ndarray
    evm_den: np.ndarray
    bit_errors: np.ndarray
    n_bits: np.ndarray

    def evm_db(self) -> float:
        return evm_db_from_sums(float(np.sum(self.evm_num)), float(np.sum(self.evm_den)))

    def ber(self) -> float:
        return float(np.sum(self.bit_errors)) / float(np.sum(self.n_bits))


@dataclass
class ChannelRealization:  # channel.hpp:48-54
    delays_samples: np.ndarray
    gains: np.ndarray

    def frequency_response(self, n_fft: int) -> np.ndarray:
        """channel.cpp:91-98: DFT of the tap line on the n_fft grid."""
        h = np.zeros(n_fft, np.complex128)
        for d, g in zip(self.delays_samples, self.gains):
            h[int(d) % n_fft] += g
        return np.fft.fft(h)


def exponential_profile(rms_ds_ns: float, step_ns: float, n_taps: int) -> tuple[np.ndarray, np.ndarray]:
    """TdlProfile::exponential (channel.cpp:75-89): (delay_ns, power_lin)."""
    if rms_ds_ns <= 0.0 or step_ns <= 0.0 or n_taps < 1:
        raise ValueError("invalid exponential profile parameters")
    d = np.arange(n_taps) * step_ns
    p = np.exp(-d / rms_ds_ns)
    return d, p / p.sum()


def draw_tdl(delay_ns, power_lin, fs_hz: float, seed: int) -> ChannelRealization:
    """draw_tdl (channel.cpp:101-111) through the C ABI."""
    d = np.ascontiguousarray(delay_ns, np.float64)
    p = np.ascontiguousarray(power_lin, np.float64)
    dl = np.zeros(len(d), np.int32)
    g = np.zeros(2 * len(d), np.float64)
    check(lib().fcw_draw_tdl(d.ctypes.data, p.ctypes.data, len(d), fs_hz, seed, dl.ctypes.data, g.ctypes.data))
    return ChannelRealization(dl, g.view(np.complex128))


def apply_channel(wave_in, wave_out, wave_len: int, S: int, channels: Sequence[ChannelRealization], stream=None,
                  wave_stride: int = 0) -> None:
    """apply_channel (channel.cpp:113-124) on S device waveforms, one tap line per unit."""
    n = len(channels[0].gains) if channels else 0
    if any(len(c.gains) != n for c in channels) or len(channels) != S:
        raise ValueError("one channel realization per unit, equal tap counts")
    d = np.ascontiguousarray(np.concatenate([c.delays_samples for c in channels]) if S else np.zeros(0), np.int32)
    g = np.ascontiguousarray(np.concatenate([c.gains for c in channels]) if S else np.zeros(0), np.complex128)
    check(lib().fcw_apply_channel(_dev_ptr(wave_in), _dev_ptr(wave_out), wave_stride, wave_len, S, d.ctypes.data,
                                  g.ctypes.data, n, _stream_ptr(stream)))


def psd(wave, wave_len: int, S: int, seg_len: int, overlap_frac: float = 0.5, stream=None,
        wave_stride: int = 0) -> np.ndarray:
    """Welch PSD (metrics.cpp:128-155) of S device waveforms -> [S][seg_len]."""
    out = np.zeros((max(S, 1), seg_len), np.float64)
    check(lib().fcw_psd(_dev_ptr(wave), wave_stride, wave_len, S, seg_len, overlap_frac,
                        out.ctypes.data_as(C.POINTER(C.c_double)), _stream_ptr(stream)))
    return out[:S]


def evm_db_from_sums(num: float, den: float) -> float:
    """metrics.cpp:115-127 (evm_db) from accumulated sums: -10 log10(num/den),
    300 dB cap; zero reference power is an error."""
    if den <= 0.0:
        raise ValueError("zero reference power")
    if num <= 0.0:
        return 300.0
    return min(300.0, -10.0 * math.log10(num / den))


def awgn_noise_variance(power: float, snr_db: float, n_fft: int, n_active_total: int) -> float:
    """channel.cpp:120-127: Es per active subcarrier over an n_fft demodulation
    window divided by the linear SNR."""
    es = power * n_fft / n_active_total
    return es / 10.0 ** (snr_db / 10.0)
