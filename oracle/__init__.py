"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the FC-F-OFDM hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker.
The product package ``paper_2008_00672_b200`` never imports it.

Two back-ends, both built by ``make -C oracle`` (see oracle/Makefile):

* ``C``  — ``oracle/liboracle.so``: a plain-C double-precision restatement of
  the reference algorithm (oracle/fcw_oracle.c; each function cites the
  reference file:line it follows).
* ``Ref`` — ``oracle/_ref/libfcwave_ref.so``: the UNMODIFIED reference
  (/root/reference/proj/src/{numerology,ofdm,fc_core,fc_sync,fft}.cpp) compiled
  against the builder-written FFTW-API shim.  Built only where /root/reference
  exists; the .so then travels to the GPU box with the repo snapshot.

Complex arrays cross the boundary as numpy complex128.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(_HERE, "liboracle.so")
_REF_SO = os.path.join(_HERE, "_ref", "libfcwave_ref.so")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


class FcoParams(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("L", "N")] + [("overlap", C.c_double)] + [
        (n, C.c_int) for n in ("L_O", "L_S", "L_L", "L_T", "N_O", "N_S", "N_L", "N_T", "I")
    ]


def build(quiet: bool = True) -> None:
    import subprocess

    subprocess.run(["make", "-C", _HERE, "-s" if quiet else "-w"], check=True)


def _load(path):
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE_SO):
            build()
        _lib = C.CDLL(_ORACLE_SO)
        L = _lib
        L.fco_derive_params.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(FcoParams)]
        L.fco_cp_schedule.argtypes = [C.c_int, C.c_int, C.c_int, _i32p]
        L.fco_cp_truncate.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.fco_cp_truncate.restype = None
        L.fco_symbol_sigma.argtypes = [C.c_int, _i32p, C.c_int]
        L.fco_symbol_sigma.restype = C.c_int64
        L.fco_combined_length.argtypes = [C.c_int, _i32p, C.POINTER(FcoParams)]
        L.fco_combined_length.restype = C.c_int64
        L.fco_design_window.argtypes = [C.c_int, C.c_int, C.c_int, _f64p]
        L.fco_bin_map.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i32p]
        L.fco_bin_map.restype = None
        L.fco_rx_start.argtypes = [C.c_int64, C.c_int, C.c_int, _i32p, C.c_int]
        L.fco_rx_start.restype = C.c_int64
        L.fco_centered_active_map.argtypes = [C.c_int, C.c_int, C.c_int, _i32p]
        for f in (L.fco_block_phase,):
            f.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
            f.restype = None
        L.fco_symbol_phase.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.fco_symbol_phase.restype = None
        L.fco_zero_pad_symbol.argtypes = [_f64p, C.c_int, C.POINTER(FcoParams), C.c_int, _f64p]
        L.fco_first_block_window.argtypes = [C.POINTER(FcoParams), C.c_int, _f64p]
        L.fco_fft.argtypes = [_f64p, C.c_int, C.c_int]
        L.fco_fft.restype = None
        L.fco_tx_symbol.argtypes = [_f64p, C.c_int, C.c_int, C.c_int, _f64p, C.POINTER(FcoParams), _i32p, C.c_int, _f64p]
        L.fco_tx_discontinuous.argtypes = [
            C.c_int, C.c_double, _i32p, C.c_int, C.c_int, _i32p, _i32p, _f64p, _f64p, _f64p,
            C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.fco_rx_block_freq.argtypes = [_f64p, C.c_int, C.c_int, _f64p, C.POINTER(FcoParams), C.c_double, C.c_double, _f64p]
        L.fco_rx_symbol_direct.argtypes = [_f64p, _f64p, C.c_int, C.c_int, _f64p, C.POINTER(FcoParams), _i32p, C.c_int, _f64p]
        L.fco_rx_symbol_simplified.argtypes = [_f64p, _f64p, C.POINTER(FcoParams), _f64p]
        L.fco_rx_discontinuous.argtypes = [
            _f64p, C.c_int64, C.c_int64, C.c_int, C.c_double, _i32p, C.c_int, C.c_int, C.c_int,
            _f64p, C.c_int, _f64p]
        L.fco_splitmix64.argtypes = [C.POINTER(C.c_uint64)]
        L.fco_splitmix64.restype = C.c_uint64
        L.fco_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.fco_derive_seed.restype = C.c_uint64
        L.fco_qam_map.argtypes = [C.c_int, C.c_uint, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.fco_qam_map.restype = None
        L.fco_gen_grid.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, _f64p]
        L.fco_gen_grid.restype = None
        L.fco_qam_demap.argtypes = [C.c_int, C.c_double, C.c_double]
        L.fco_qam_demap.restype = C.c_uint
        _i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
        L.fco_link_stats.argtypes = [_f64p, C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, _f64p, _i64p]
        L.fco_link_stats.restype = None
        L.fco_awgn.argtypes = [_f64p, C.c_int64, C.c_double, C.c_uint64]
        L.fco_awgn.restype = None
        L.fco_measure_power.argtypes = [_f64p, C.c_int64, C.c_int64, C.c_int64]
        L.fco_measure_power.restype = C.c_double
        L.fco_draw_tdl.argtypes = [_f64p, _f64p, C.c_int, C.c_double, C.c_uint64, _i32p, _f64p]
        L.fco_draw_tdl.restype = None
        L.fco_apply_channel.argtypes = [_f64p, C.c_int64, _i32p, _f64p, C.c_int, _f64p]
        L.fco_apply_channel.restype = None
        L.fco_psd.argtypes = [_f64p, C.c_int64, C.c_int, C.c_double, _f64p]
        L.fco_tx_continuous.argtypes = [C.c_int, C.c_double, C.c_int, _i32p, _i32p, _f64p, _f64p, _i64p, C.c_int,
                                        _f64p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.fco_rx_continuous.argtypes = [_f64p, C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int, _f64p, _f64p,
                                        C.c_int64, C.POINTER(C.c_int64)]
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            raise OracleError("oracle/_ref not built (needs /root/reference at build time)")
        _ref = C.CDLL(_REF_SO)
        R = _ref
        R.fcwref_last_error.restype = C.c_char_p
        R.fcwref_tx.argtypes = [C.c_int, C.c_double, _i32p, C.c_int, C.c_int, _i32p, _i32p, _f64p, _f64p,
                                _f64p, C.c_longlong, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
        R.fcwref_rx.argtypes = [C.c_int, C.c_double, _i32p, C.c_int, C.c_int, C.c_int, _f64p, _f64p,
                                C.c_longlong, C.c_longlong, C.c_int, _f64p]
        R.fcwref_tx_symbol.argtypes = [_f64p, C.c_int, C.c_int, C.c_int, _f64p, C.c_int, C.c_double, _i32p,
                                       C.c_int, C.c_int, _f64p]
        R.fcwref_rx_symbol_direct.argtypes = [_f64p, _f64p, C.c_int, C.c_int, _f64p, C.c_int, C.c_double,
                                              _i32p, C.c_int, C.c_int, _f64p]
        R.fcwref_rx_block_freq.argtypes = [_f64p, C.c_int, C.c_int, _f64p, C.c_int, C.c_double, C.c_double,
                                           C.c_double, _f64p]
        R.fcwref_rx_symbol_simplified.argtypes = [_f64p, _f64p, C.c_int, C.c_int, _f64p, C.c_int, C.c_double, _f64p]
        R.fcwref_bench_txrx.argtypes = [C.c_int, C.c_double, _i32p, C.c_int, C.c_int, _i32p, _i32p, _f64p,
                                        _i32p, _i32p, _f32p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
        R.fcwref_bench_txrx.restype = C.c_double
        _u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
        _u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
        R.fcwref_qam_demap.argtypes = [C.c_int, _f64p, C.c_int, _u32p]
        R.fcwref_qam_map.argtypes = [C.c_int, _u32p, C.c_int, _f64p]
        R.fcwref_ber.argtypes = [_u8p, _u8p, C.c_longlong, C.POINTER(C.c_double)]
        R.fcwref_evm_db.argtypes = [_f64p, _f64p, C.c_longlong, C.POINTER(C.c_double)]
        R.fcwref_awgn_with_variance.argtypes = [_f64p, C.c_longlong, C.c_double, C.c_ulonglong]
        R.fcwref_measure_power.argtypes = [_f64p, C.c_longlong, C.c_longlong, C.c_longlong, C.POINTER(C.c_double)]
        _i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
        R.fcwref_draw_tdl.argtypes = [_f64p, _f64p, C.c_int, C.c_double, C.c_ulonglong, _i32p, _f64p]
        R.fcwref_apply_channel.argtypes = [_f64p, C.c_longlong, _i32p, _f64p, C.c_int]
        R.fcwref_psd.argtypes = [_f64p, C.c_longlong, C.c_int, C.c_double, _f64p]
        R.fcwref_tx_continuous.argtypes = [C.c_int, C.c_double, C.c_int, _i32p, _i32p, _f64p, _f64p, _i64p,
                                           C.c_int, _f64p, C.c_longlong, C.POINTER(C.c_longlong),
                                           C.POINTER(C.c_longlong)]
        R.fcwref_rx_continuous.argtypes = [_f64p, C.c_longlong, C.c_int, C.c_double, C.c_int, C.c_int, _f64p,
                                           _f64p, C.c_longlong, C.POINTER(C.c_longlong)]
        R.fcwref_awgn_noise_variance.argtypes = [_f64p, C.c_longlong, C.c_double, C.c_int, C.c_int,
                                                 C.POINTER(C.c_double)]
    return _ref


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _as_f64(a: np.ndarray) -> np.ndarray:
    return _c128(a).view(np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _check(rc: int, what: str, ref_lib=None):
    if rc == 0:
        return
    msg = ""
    if ref_lib is not None:
        msg = ref_lib.fcwref_last_error().decode()
    if rc == 2:
        raise IndexError(f"{what}: out of range {msg}")
    raise ValueError(f"{what}: invalid argument {msg}")


# ---------------------------------------------------------------- C oracle
@dataclass
class Params:
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

    def c(self) -> FcoParams:
        p = FcoParams()
        for k, v in self.__dict__.items():
            setattr(p, k, v)
        return p


def derive_params(N: int, L: int, overlap: float = 0.5) -> Params:
    p = FcoParams()
    _check(lib().fco_derive_params(N, L, overlap, C.byref(p)), "derive_params")
    return Params(**{k: getattr(p, k) for k, _ in FcoParams._fields_})


def cp_schedule(scs_khz: int, n_fft: int, n_symbols: int) -> list[int]:
    out = np.zeros(max(n_symbols, 1), np.int32)
    _check(lib().fco_cp_schedule(scs_khz, n_fft, n_symbols, out), "cp_schedule")
    return out.tolist()


def nr_cp_schedule(scs_khz: int, n_fft: int, n_symbols: int) -> list[int]:
    """5G-NR normal CP (3GPP TS 38.211 §5.3.1), restated independently of the
    product's fcw_nr_cp_schedule: N_CP = 144 kappa 2^-mu Tc, plus 16 kappa Tc on
    the first symbol of every 0.5 ms (l mod 7 * 2^mu == 0).  In samples at
    fs = n_fft * scs: 144 n_fft / 2048 and 16 * 2^mu * n_fft / 2048 (30 kHz,
    N = 4096: 288 / 352).  Same validation shape as the reference's
    cp_schedule (numerology.cpp:17-42)."""
    if n_fft < 16 or n_fft & (n_fft - 1):
        raise ValueError("n_fft must be a power of two >= 16")
    mu2 = scs_khz // 15
    if scs_khz <= 0 or scs_khz % 15 or mu2 & (mu2 - 1):
        raise ValueError("scs_khz must be 15*2^k")
    if n_symbols < 1:
        raise ValueError("n_symbols must be >= 1")
    if (144 * n_fft) % 2048 or (16 * mu2 * n_fft) % 2048:
        raise ValueError("n_fft does not scale the CP pattern to integers")
    short = 144 * n_fft // 2048
    extra = 16 * mu2 * n_fft // 2048
    return [short + (extra if n % (7 * mu2) == 0 else 0) for n in range(n_symbols)]


class Geometry:
    """Workload geometry backend for paper_2008_00672_b200.configs built from
    this oracle only (bench.py's reference arm: no product library loaded)."""

    design_window = staticmethod(lambda L, n, tb: design_window(L, n, tb))
    centered_active_map = staticmethod(lambda L, n, skip_dc=True: centered_active_map(L, n, skip_dc))
    cp = staticmethod(lambda scs, N, B: cp_schedule(scs, N, B))
    nr_cp = staticmethod(lambda scs, N, B: nr_cp_schedule(scs, N, B))

    @staticmethod
    def subband(**kw):
        from types import SimpleNamespace

        kw.setdefault("n_active", 0)
        kw.setdefault("n_tb", 0)
        kw.setdefault("l_ofdm", kw["L"])
        kw["window"] = np.ascontiguousarray(np.asarray(kw["window"], np.float64))
        return SimpleNamespace(**kw)


def cp_truncate(n_cp: int, I: int) -> tuple[int, int]:
    a, b = C.c_int(), C.c_int()
    lib().fco_cp_truncate(n_cp, I, C.byref(a), C.byref(b))
    return a.value, b.value


def symbol_sigma(n: int, cp, N: int) -> int:
    return int(lib().fco_symbol_sigma(n, _i32(cp), N))


def combined_length(B: int, cp, p: Params) -> int:
    pc = p.c()
    return int(lib().fco_combined_length(B, _i32(cp), C.byref(pc)))


def bin_map(L: int, c: int, N: int) -> tuple[np.ndarray, np.ndarray]:
    """(q, b) per shifted index p0 (fc_core.cpp:80-84): the map the oracle's
    synth / analysis use."""
    q, b = np.zeros(L, np.int32), np.zeros(L, np.int32)
    lib().fco_bin_map(L, c, N, q, b)
    return q, b


def rx_starts(useful0: int, cp, N: int, L: int) -> np.ndarray:
    """rx_segment window starts useful0 - N_L + sigma_n (fc_sync.cpp:148)."""
    p = derive_params(N, L)
    cpa = _i32(cp)
    return np.array([lib().fco_rx_start(useful0, p.N_L, n, cpa, N) for n in range(len(cp))], np.int64)


def design_window(L: int, n_pass: int, n_tb: int) -> np.ndarray:
    w = np.zeros(L, np.float64)
    _check(lib().fco_design_window(L, n_pass, n_tb, w), "design_window")
    return w


def centered_active_map(l_ofdm: int, n_active: int, skip_dc: bool = True) -> list[int]:
    out = np.zeros(max(n_active, 1), np.int32)
    _check(lib().fco_centered_active_map(l_ofdm, n_active, int(skip_dc), out), "centered_active_map")
    return out[:n_active].tolist()


def block_phase(r: int, c: int, L_S: int, L: int) -> complex:
    a, b = C.c_double(), C.c_double()
    lib().fco_block_phase(r, c, L_S, L, C.byref(a), C.byref(b))
    return complex(a.value, b.value)


def symbol_phase(n: int, c: int, cp, N: int) -> complex:
    a, b = C.c_double(), C.c_double()
    lib().fco_symbol_phase(n, c, _i32(cp), N, C.byref(a), C.byref(b))
    return complex(a.value, b.value)


def zero_pad_symbol(sym, p: Params, l_cp: int) -> np.ndarray:
    s = _as_f64(sym)
    out = np.zeros(2 * (3 * p.L // 2), np.float64)
    pc = p.c()
    _check(lib().fco_zero_pad_symbol(s, len(s) // 2, C.byref(pc), l_cp, out), "zero_pad_symbol")
    return out.view(np.complex128)


def first_block_window(p: Params, l_cp: int) -> np.ndarray:
    a = np.zeros(p.L, np.float64)
    pc = p.c()
    _check(lib().fco_first_block_window(C.byref(pc), l_cp, a), "first_block_window")
    return a


def fft(x, inverse: bool = False) -> np.ndarray:
    d = _as_f64(x).copy()
    lib().fco_fft(d, len(d) // 2, int(inverse))
    return d.view(np.complex128)


def tx_symbol(sym, L: int, c: int, window, p: Params, cp, n: int) -> np.ndarray:
    s = _as_f64(sym)
    out = np.zeros(2 * (3 * p.N // 2), np.float64)
    pc = p.c()
    _check(lib().fco_tx_symbol(s, len(s) // 2, L, c, np.asarray(window, np.float64), C.byref(pc), _i32(cp), n, out),
           "tx_symbol")
    return out.view(np.complex128)


def tx_discontinuous(grids, Ls, cs, windows, cp, N: int, overlap: float = 0.5):
    """grids: list over subbands of (B, L_m) complex arrays (full columns)."""
    B = len(cp)
    flat = np.concatenate([_c128(g).reshape(-1) for g in grids])
    wins = np.concatenate([np.asarray(w, np.float64) for w in windows])
    cap = 4 * N + B * (N + max(cp) + 1) + 16
    out = np.zeros(2 * cap, np.float64)
    Q, u0 = C.c_int64(), C.c_int64()
    _check(lib().fco_tx_discontinuous(N, overlap, _i32(cp), B, len(Ls), _i32(Ls), _i32(cs), wins,
                                      flat.view(np.float64), out, cap, C.byref(Q), C.byref(u0)), "tx_discontinuous")
    return out.view(np.complex128)[: Q.value].copy(), u0.value


def rx_block_freq(y, L: int, c: int, window, p: Params, phase: complex) -> np.ndarray:
    g = np.zeros(2 * L, np.float64)
    pc = p.c()
    lib().fco_rx_block_freq(_as_f64(y), L, c, np.asarray(window, np.float64), C.byref(pc), phase.real, phase.imag, g)
    return g.view(np.complex128)


def rx_symbol_direct(y0, y1, L: int, c: int, window, p: Params, cp, n: int) -> np.ndarray:
    out = np.zeros(2 * L, np.float64)
    pc = p.c()
    _check(lib().fco_rx_symbol_direct(_as_f64(y0), _as_f64(y1), L, c, np.asarray(window, np.float64), C.byref(pc),
                                      _i32(cp), n, out), "rx_symbol_direct")
    return out.view(np.complex128)


def rx_symbol_simplified(g0, g1, p: Params) -> np.ndarray:
    out = np.zeros(2 * p.L, np.float64)
    pc = p.c()
    _check(lib().fco_rx_symbol_simplified(_as_f64(g0), _as_f64(g1), C.byref(pc), out), "rx_symbol_simplified")
    return out.view(np.complex128)


def rx_discontinuous(wave, useful0: int, cp, N: int, L: int, c: int, window, simplified: bool = False,
                     overlap: float = 0.5) -> np.ndarray:
    B = len(cp)
    w = _as_f64(wave)
    out = np.zeros(2 * B * L, np.float64)
    _check(lib().fco_rx_discontinuous(w, len(w) // 2, useful0, N, overlap, _i32(cp), B, L, c,
                                      np.asarray(window, np.float64), int(simplified), out), "rx_discontinuous")
    return out.view(np.complex128).reshape(B, L)


def splitmix64_stream(seed: int, n: int) -> list[int]:
    st = C.c_uint64(seed)
    return [int(lib().fco_splitmix64(C.byref(st))) for _ in range(n)]


def derive_seed(seed: int, index: int) -> int:
    return int(lib().fco_derive_seed(seed, index))


def qam_map(bits_per_symbol: int, sym: int) -> complex:
    a, b = C.c_double(), C.c_double()
    lib().fco_qam_map(bits_per_symbol, sym, C.byref(a), C.byref(b))
    return complex(a.value, b.value)


def gen_grid(seed: int, unit0: int, units: int, B: int, A: int, bits_per_symbol: int) -> np.ndarray:
    out = np.zeros(2 * units * B * A, np.float64)
    lib().fco_gen_grid(seed, unit0, units, B, A, bits_per_symbol, out)
    return out.view(np.complex128).reshape(units, B, A)


# ------------------------------------------------------- link step (f1/f3)
def qam_demap(bits_per_symbol: int, y) -> np.ndarray:
    """ofdm.cpp:67-78 hard decision, per element (256-QAM extended)."""
    y = np.asarray(y, np.complex128).reshape(-1)
    L = lib()
    return np.array([L.fco_qam_demap(bits_per_symbol, float(v.real), float(v.imag)) for v in y], np.uint32)


def link_stats(rx, seed: int, unit0: int, bits_per_symbol: int):
    """Per-unit (evm_num, evm_den, bit_errors) of a packed rx grid [units][B][A]
    against the seeded transmit grid (scenario.cpp:469-494, metrics.cpp:105-127)."""
    rx = np.ascontiguousarray(rx, np.complex128)
    units, B, A = rx.shape
    out = np.zeros(2 * units, np.float64)
    errs = np.zeros(units, np.int64)
    lib().fco_link_stats(rx.view(np.float64).reshape(-1), seed, unit0, units, B, A, bits_per_symbol, out, errs)
    return out[0::2].copy(), out[1::2].copy(), errs


def awgn(wave, sigma2: float, seed: int) -> np.ndarray:
    """channel.cpp:136-141 awgn_with_variance (returns a new array)."""
    w = _c128(wave).copy()
    lib().fco_awgn(w.view(np.float64), len(w), sigma2, seed)
    return w


def measure_power(wave, begin: int, end: int) -> float:
    """channel.cpp:148-155."""
    w = _c128(wave)
    return float(lib().fco_measure_power(w.view(np.float64), len(w), begin, end))


def draw_tdl(delay_ns, power_lin, fs_hz: float, seed: int):
    """channel.cpp:101-111 -> (delays int32, gains complex128)."""
    d = np.ascontiguousarray(delay_ns, np.float64)
    p = np.ascontiguousarray(power_lin, np.float64)
    dl = np.zeros(len(d), np.int32)
    g = np.zeros(2 * len(d), np.float64)
    lib().fco_draw_tdl(d, p, len(d), fs_hz, seed, dl, g)
    return dl, g.view(np.complex128)


def apply_channel(wave, delays, gains) -> np.ndarray:
    """channel.cpp:113-124."""
    w = _as_f64(wave)
    out = np.zeros_like(w)
    lib().fco_apply_channel(w, len(w) // 2, _i32(delays), _as_f64(gains), len(delays), out)
    return out.view(np.complex128)


def psd(x, seg_len: int, overlap_frac: float = 0.5) -> np.ndarray:
    """metrics.cpp:128-155 Welch PSD."""
    w = _as_f64(x)
    out = np.zeros(seg_len, np.float64)
    _check(lib().fco_psd(w, len(w) // 2, seg_len, overlap_frac, out), "psd")
    return out


def _cont_cap(N, Ls, lens):
    return int(max((ln + L) // (L // 2) + 3 for L, ln in zip(Ls, lens)) * (N // 2) + 2 * N)


def tx_continuous(streams, Ls, cs, windows, N: int, overlap: float = 0.5, l_cp0: int = 0):
    """fc_core.cpp:163-198.  streams: one complex array per subband."""
    lens = np.array([len(x) for x in streams], np.int64)
    flat = np.concatenate([_c128(x) for x in streams]) if len(streams) else np.zeros(0, np.complex128)
    cap = _cont_cap(N, Ls, lens)
    out = np.zeros(2 * cap, np.float64)
    ol, u0 = C.c_int64(), C.c_int64()
    _check(lib().fco_tx_continuous(N, overlap, len(Ls), _i32(Ls), _i32(cs),
                                   np.concatenate([np.asarray(w, np.float64) for w in windows]),
                                   flat.view(np.float64), lens, l_cp0, out, cap, C.byref(ol), C.byref(u0)),
           "tx_continuous")
    return out.view(np.complex128)[: ol.value].copy(), u0.value


def rx_continuous(wave, N: int, L: int, c: int, window, overlap: float = 0.5) -> np.ndarray:
    """fc_core.cpp:200-223 for one subband."""
    w = _as_f64(wave)
    n = len(w) // 2
    cap = (n // max(1, N // L) + 2 * L) * 2 + 4 * L
    out = np.zeros(2 * cap, np.float64)
    no = C.c_int64()
    _check(lib().fco_rx_continuous(w, n, N, overlap, L, c, np.asarray(window, np.float64), out, cap, C.byref(no)),
           "rx_continuous")
    return out.view(np.complex128)[: no.value].copy()


def evm_db(num: float, den: float) -> float:
    """metrics.cpp:115-127 from the accumulated sums."""
    if den <= 0.0:
        raise ValueError("zero reference power")
    if num <= 0.0:
        return 300.0
    return min(300.0, -10.0 * float(np.log10(num / den)))


# ------------------------------------------------------- compiled reference
class Ref:
    """Thin wrappers over oracle/_ref/libfcwave_ref.so (the real reference)."""

    @staticmethod
    def tx_discontinuous(grids, Ls, cs, windows, cp, N: int, overlap: float = 0.5):
        R = ref()
        B = len(cp)
        flat = np.concatenate([_c128(g).reshape(-1) for g in grids])
        wins = np.concatenate([np.asarray(w, np.float64) for w in windows])
        cap = 4 * N + B * (N + max(cp) + 1) + 16
        out = np.zeros(2 * cap, np.float64)
        Q, u0 = C.c_longlong(), C.c_longlong()
        _check(R.fcwref_tx(N, overlap, _i32(cp), B, len(Ls), _i32(Ls), _i32(cs), wins, flat.view(np.float64), out,
                           cap, C.byref(Q), C.byref(u0)), "ref tx_discontinuous", R)
        return out.view(np.complex128)[: Q.value].copy(), u0.value

    @staticmethod
    def rx_discontinuous(wave, useful0: int, cp, N: int, L: int, c: int, window, simplified: bool = False,
                         overlap: float = 0.5):
        R = ref()
        B = len(cp)
        w = _as_f64(wave)
        out = np.zeros(2 * B * L, np.float64)
        _check(R.fcwref_rx(N, overlap, _i32(cp), B, L, c, np.asarray(window, np.float64), w, len(w) // 2, useful0,
                           int(simplified), out), "ref rx_discontinuous", R)
        return out.view(np.complex128).reshape(B, L)

    @staticmethod
    def tx_symbol(sym, L, c, window, N, cp, n, overlap=0.5):
        R = ref()
        s = _as_f64(sym)
        out = np.zeros(2 * (3 * N // 2), np.float64)
        _check(R.fcwref_tx_symbol(s, len(s) // 2, L, c, np.asarray(window, np.float64), N, overlap, _i32(cp),
                                  len(cp), n, out), "ref tx_symbol", R)
        return out.view(np.complex128)

    @staticmethod
    def rx_symbol_direct(y0, y1, L, c, window, N, cp, n, overlap=0.5):
        R = ref()
        out = np.zeros(2 * L, np.float64)
        _check(R.fcwref_rx_symbol_direct(_as_f64(y0), _as_f64(y1), L, c, np.asarray(window, np.float64), N,
                                         overlap, _i32(cp), len(cp), n, out), "ref rx_symbol_direct", R)
        return out.view(np.complex128)

    @staticmethod
    def bench_txrx(N, cp, Ls, cs, windows, n_active, active_bins, grids_packed_c64, units, threads,
                   simplified=True, overlap=0.5):
        R = ref()
        g = np.ascontiguousarray(grids_packed_c64, dtype=np.complex64).view(np.float32).reshape(-1)
        chk = C.c_double()
        t = R.fcwref_bench_txrx(N, overlap, _i32(cp), len(cp), len(Ls), _i32(Ls), _i32(cs),
                                np.concatenate([np.asarray(w, np.float64) for w in windows]), _i32(n_active),
                                _i32(np.concatenate([np.asarray(b) for b in active_bins])), g, units, threads,
                                int(simplified), C.byref(chk))
        if t < 0:
            raise OracleError(R.fcwref_last_error().decode())
        return t, chk.value

    # ---- link step (f1/f3) through the reference's own functions
    @staticmethod
    def qam_demap(bits_per_symbol: int, y) -> np.ndarray:
        y = _c128(np.asarray(y).reshape(-1))
        out = np.zeros(len(y), np.uint32)
        _check(ref().fcwref_qam_demap(bits_per_symbol, y.view(np.float64), len(y), out), "ref qam_demap", ref())
        return out

    @staticmethod
    def qam_map(bits_per_symbol: int, syms) -> np.ndarray:
        s = np.ascontiguousarray(syms, np.uint32)
        out = np.zeros(2 * len(s), np.float64)
        _check(ref().fcwref_qam_map(bits_per_symbol, s, len(s), out), "ref qam_map", ref())
        return out.view(np.complex128)

    @staticmethod
    def ber(a, b) -> float:
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        v = C.c_double()
        _check(ref().fcwref_ber(a, b, len(a), C.byref(v)), "ref ber", ref())
        return v.value

    @staticmethod
    def evm_db(ref_grid, rx) -> float:
        r = _c128(np.asarray(ref_grid).reshape(-1))
        x = _c128(np.asarray(rx).reshape(-1))
        v = C.c_double()
        _check(ref().fcwref_evm_db(r.view(np.float64), x.view(np.float64), len(r), C.byref(v)), "ref evm_db", ref())
        return v.value

    @staticmethod
    def awgn_with_variance(wave, sigma2: float, seed: int) -> np.ndarray:
        w = _c128(wave).copy()
        _check(ref().fcwref_awgn_with_variance(w.view(np.float64), len(w), sigma2, seed), "ref awgn", ref())
        return w

    @staticmethod
    def measure_power(wave, begin: int, end: int) -> float:
        w = _c128(wave)
        v = C.c_double()
        _check(ref().fcwref_measure_power(w.view(np.float64), len(w), begin, end, C.byref(v)), "ref power", ref())
        return v.value

    @staticmethod
    def awgn_noise_variance(wave, snr_db: float, n_fft: int, n_active: int) -> float:
        w = _c128(wave)
        v = C.c_double()
        _check(ref().fcwref_awgn_noise_variance(w.view(np.float64), len(w), snr_db, n_fft, n_active, C.byref(v)),
               "ref noise variance", ref())
        return v.value

    @staticmethod
    def tx_continuous(streams, Ls, cs, windows, N: int, overlap: float = 0.5, l_cp0: int = 0):
        lens = np.array([len(x) for x in streams], np.int64)
        flat = np.concatenate([_c128(x) for x in streams])
        cap = _cont_cap(N, Ls, lens)
        out = np.zeros(2 * cap, np.float64)
        ol, u0 = C.c_longlong(), C.c_longlong()
        _check(ref().fcwref_tx_continuous(N, overlap, len(Ls), _i32(Ls), _i32(cs),
                                          np.concatenate([np.asarray(w, np.float64) for w in windows]),
                                          flat.view(np.float64), lens, l_cp0, out, cap, C.byref(ol), C.byref(u0)),
               "ref tx_continuous", ref())
        return out.view(np.complex128)[: ol.value].copy(), u0.value

    @staticmethod
    def rx_continuous(wave, N: int, L: int, c: int, window, overlap: float = 0.5) -> np.ndarray:
        w = _as_f64(wave)
        n = len(w) // 2
        cap = (n // max(1, N // L) + 2 * L) * 2 + 4 * L
        out = np.zeros(2 * cap, np.float64)
        no = C.c_longlong()
        _check(ref().fcwref_rx_continuous(w, n, N, overlap, L, c, np.asarray(window, np.float64), out, cap,
                                          C.byref(no)), "ref rx_continuous", ref())
        return out.view(np.complex128)[: no.value].copy()

    @staticmethod
    def psd(x, seg_len: int, overlap_frac: float = 0.5) -> np.ndarray:
        w = _as_f64(x)
        out = np.zeros(seg_len, np.float64)
        _check(ref().fcwref_psd(w, len(w) // 2, seg_len, overlap_frac, out), "ref psd", ref())
        return out

    @staticmethod
    def draw_tdl(delay_ns, power_lin, fs_hz: float, seed: int):
        d = np.ascontiguousarray(delay_ns, np.float64)
        p = np.ascontiguousarray(power_lin, np.float64)
        dl = np.zeros(len(d), np.int32)
        g = np.zeros(2 * len(d), np.float64)
        _check(ref().fcwref_draw_tdl(d, p, len(d), fs_hz, seed, dl, g), "ref draw_tdl", ref())
        return dl, g.view(np.complex128)

    @staticmethod
    def apply_channel(wave, delays, gains) -> np.ndarray:
        w = _c128(wave).copy()
        _check(ref().fcwref_apply_channel(w.view(np.float64), len(w), _i32(delays), _as_f64(gains), len(delays)),
               "ref apply_channel", ref())
        return w
