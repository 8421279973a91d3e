"""ctypes binding of the C ABI declared in include/fcwave_b200.h.

The shared library is built in-tree (paper_2008_00672_b200/lib/) by
``paper_2008_00672_b200.build.build()``.  There is no fallback: if the library
is missing or a GPU call fails, the caller gets an exception.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libfcwave_b200.so")
# dev-only A/B knob: load a variant built by ``build.py --variant NAME``
if os.environ.get("FCW_LIB_VARIANT"):
    LIB_PATH = os.path.join(HERE, "lib", f"libfcwave_b200_{os.environ['FCW_LIB_VARIANT']}.so")

FCW_OK, FCW_EINVAL, FCW_ERANGE, FCW_ECUDA, FCW_ENOMEM, FCW_ENOTSUP = range(6)
FCW_GRID_FULL = 1
FCW_RX_FUSED = 2
FCW_TX_ACCUMULATE = 4

# Every symbol include/fcwave_b200.h declares (checked by tests/test_capi.py).
EXPORTS = [
    "fcw_plan_create", "fcw_plan_destroy", "fcw_plan_get_info", "fcw_plan_sigma", "fcw_plan_cp_split",
    "fcw_plan_bin_map", "fcw_plan_rx_starts", "fcw_plan_fc_params", "fcw_tx", "fcw_rx", "fcw_gen_qam",
    "fcw_tx_host", "fcw_rx_host", "fcw_host_alloc", "fcw_host_free", "fcw_derive_fc_params", "fcw_cp_schedule",
    "fcw_nr_cp_schedule", "fcw_cp_truncate", "fcw_first_block_overlap", "fcw_design_window",
    "fcw_centered_active_map", "fcw_symbol_sigma", "fcw_combined_length", "fcw_last_error", "fcw_version",
    "fcw_link_stats", "fcw_awgn", "fcw_wave_power", "fcw_psd", "fcw_draw_tdl", "fcw_apply_channel",
    "fcw_cont_plan_create", "fcw_cont_plan_destroy", "fcw_cont_plan_get_info", "fcw_tx_continuous",
    "fcw_rx_continuous", "fcw_wave_zero", "fcw_symbol_phase", "fcw_block_phase", "fcw_tx_symbol",
    "fcw_combine_symbols", "fcw_rx_segment", "fcw_rx_block_freq", "fcw_rx_symbol_simplified", "fcw_rx_symbol_direct",
]


class ContInfoC(C.Structure):
    _fields_ = [("N", C.c_int), ("M", C.c_int)] + [
        (n, C.c_int64) for n in ("tx_len", "tx_stride", "useful0", "stream_total", "rx_wave_len", "rx_out_total")
    ] + [("tx_pairs", C.c_int), ("rx_pairs", C.c_int)]


class LinkStatC(C.Structure):
    _fields_ = [("evm_num", C.c_double), ("evm_den", C.c_double), ("bit_errors", C.c_int64), ("n_bits", C.c_int64)]


class FcParamsC(C.Structure):
    _fields_ = [("L", C.c_int), ("N", C.c_int), ("overlap", C.c_double)] + [
        (n, C.c_int) for n in ("L_O", "L_S", "L_L", "L_T", "N_O", "N_S", "N_L", "N_T", "I")
    ]


class SubbandC(C.Structure):
    _fields_ = [("L", C.c_int), ("l_ofdm", C.c_int), ("c", C.c_int), ("n_active", C.c_int), ("n_tb", C.c_int),
                ("active_bins", C.POINTER(C.c_int)), ("window", C.POINTER(C.c_double))]


class PlanInfoC(C.Structure):
    _fields_ = [("N", C.c_int), ("B", C.c_int), ("M", C.c_int), ("overlap", C.c_double), ("Q", C.c_int64),
                ("useful0", C.c_int64), ("frame_samples", C.c_int64), ("row_active", C.c_int),
                ("row_full", C.c_int), ("N_L", C.c_int), ("N_T", C.c_int), ("chunk", C.c_int),
                ("kernel_variant", C.c_int), ("tmem_rows", C.c_int)]


_lib = None


class FcwError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[fcw {code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    """Raise the reference's exception class for a status code."""
    if rc == FCW_OK:
        return
    msg = lib().fcw_last_error().decode()
    if rc == FCW_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == FCW_ERANGE:
        raise IndexError(msg)  # std::out_of_range
    raise FcwError(rc, msg)


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"fcwave-b200 CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32p, f64p = C.c_void_p, C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_double)
    L.fcw_plan_create.argtypes = [C.POINTER(vp), C.c_int, C.c_double, i32p, C.c_int, C.POINTER(SubbandC), C.c_int,
                                  C.c_uint]
    L.fcw_plan_destroy.argtypes = [vp]
    L.fcw_plan_destroy.restype = None
    L.fcw_plan_get_info.argtypes = [vp, C.POINTER(PlanInfoC)]
    L.fcw_plan_sigma.argtypes = [vp, C.POINTER(C.c_int64)]
    L.fcw_plan_cp_split.argtypes = [vp, C.c_int, i32p, i32p]
    L.fcw_plan_bin_map.argtypes = [vp, C.c_int, i32p, i32p]
    L.fcw_plan_rx_starts.argtypes = [vp, i64, C.POINTER(C.c_int64)]
    L.fcw_plan_fc_params.argtypes = [vp, C.c_int, C.POINTER(FcParamsC)]
    L.fcw_tx.argtypes = [vp, vp, i64, vp, i64, C.c_int, C.c_uint, vp]
    L.fcw_rx.argtypes = [vp, vp, i64, i64, i64, vp, i64, C.c_int, C.c_uint, vp]
    L.fcw_gen_qam.argtypes = [vp, C.c_uint64, i64, C.c_int, C.c_int, vp, vp]
    L.fcw_link_stats.argtypes = [vp, vp, i64, C.c_int, C.c_uint64, i64, C.c_int, C.POINTER(LinkStatC), vp]
    L.fcw_awgn.argtypes = [vp, vp, i64, i64, C.c_int, C.c_double, C.c_uint64, i64, vp]
    L.fcw_wave_power.argtypes = [vp, vp, i64, i64, C.c_int, i64, i64, C.POINTER(C.c_double), vp]
    L.fcw_draw_tdl.argtypes = [vp, vp, C.c_int, C.c_double, C.c_uint64, vp, vp]
    L.fcw_apply_channel.argtypes = [vp, vp, i64, i64, C.c_int, vp, vp, C.c_int, vp]
    L.fcw_wave_zero.argtypes = [vp, i64, C.c_int, i64, i64, vp]
    dp = C.POINTER(C.c_double)
    L.fcw_symbol_phase.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, dp, dp]
    L.fcw_block_phase.argtypes = [i64, C.c_int, C.c_int, C.c_int, dp, dp]
    L.fcw_tx_symbol.argtypes = [vp, C.c_int, C.c_int, vp, i64, C.c_int, vp, i64, C.c_int, vp]
    L.fcw_combine_symbols.argtypes = [vp, vp, i64, vp, i64, C.c_int, vp]
    L.fcw_rx_segment.argtypes = [vp, vp, i64, i64, i64, C.c_int, vp, vp, i64, C.c_int, vp]
    L.fcw_rx_block_freq.argtypes = [vp, C.c_int, vp, i64, C.c_double, C.c_double, vp, i64, C.c_int, vp]
    L.fcw_rx_symbol_simplified.argtypes = [vp, C.c_int, vp, vp, i64, vp, i64, C.c_int, vp]
    L.fcw_rx_symbol_direct.argtypes = [vp, C.c_int, C.c_int, vp, vp, i64, vp, i64, C.c_int, vp]
    L.fcw_psd.argtypes = [vp, i64, i64, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_double), vp]
    L.fcw_cont_plan_create.argtypes = [C.POINTER(vp), C.c_int, C.c_double, vp, C.c_int, C.POINTER(C.c_int64), i64,
                                       C.c_int]
    L.fcw_cont_plan_destroy.argtypes = [vp]
    L.fcw_cont_plan_destroy.restype = None
    L.fcw_cont_plan_get_info.argtypes = [vp, C.POINTER(ContInfoC), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.fcw_tx_continuous.argtypes = [vp, vp, vp, C.c_int, vp]
    L.fcw_rx_continuous.argtypes = [vp, vp, vp, C.c_int, vp]
    L.fcw_tx_host.argtypes = [vp, vp, vp, C.c_int, C.c_uint]
    L.fcw_rx_host.argtypes = [vp, vp, i64, i64, vp, C.c_int, C.c_uint]
    L.fcw_host_alloc.argtypes = [C.c_size_t]
    L.fcw_host_alloc.restype = vp
    L.fcw_host_free.argtypes = [vp]
    L.fcw_host_free.restype = None
    L.fcw_derive_fc_params.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(FcParamsC)]
    L.fcw_cp_schedule.argtypes = [C.c_int, C.c_int, C.c_int, i32p]
    L.fcw_nr_cp_schedule.argtypes = [C.c_int, C.c_int, C.c_int, i32p]
    L.fcw_cp_truncate.argtypes = [C.c_int, C.c_int, i32p, i32p]
    L.fcw_first_block_overlap.argtypes = [C.POINTER(FcParamsC), C.c_int, f64p]
    L.fcw_design_window.argtypes = [C.c_int, C.c_int, C.c_int, f64p]
    L.fcw_centered_active_map.argtypes = [C.c_int, C.c_int, C.c_int, i32p]
    L.fcw_symbol_sigma.argtypes = [C.c_int, i32p, C.c_int]
    L.fcw_symbol_sigma.restype = C.c_int64
    L.fcw_combined_length.argtypes = [C.c_int, i32p, C.POINTER(FcParamsC)]
    L.fcw_combined_length.restype = C.c_int64
    L.fcw_last_error.restype = C.c_char_p
    L.fcw_version.restype = C.c_char_p
    _lib = L
    return L
