"""fcwave-b200: B200-native symbol-synchronized FC-F-OFDM TX synthesis and RX
analysis (arXiv 2008.00672), a drop-in for the reference ``fcwave`` hot path.

The compute path is hand-written sm_100a CUDA in ``csrc/`` behind the C ABI
``include/fcwave_b200.h``; this package is the Python host mirror of the
reference's operator API.  There is no CPU fallback.
"""
# The host API loads the CUDA library on first use; submodules that need no
# product code (``configs`` with an outside geometry backend) import without it.
_API = (
    "CpSchedule", "FcParams", "Numerology", "PinnedBuffer", "Plan", "QamGrid", "SubbandConfig", "Waveform",
    "centered_active_map", "combined_length", "cp_schedule", "cp_truncate", "derive_fc_params", "design_window",
    "first_block_overlap", "make_numerology", "nr_cp_schedule", "rx_discontinuous", "rx_discontinuous_all",
    "symbol_sigma", "tx_discontinuous", "symbol_phase", "block_phase",
)
__all__ = list(_API) + ["FcwError"]
__version__ = "0.1.0"


def __getattr__(name):
    if name in _API:
        from . import api

        return getattr(api, name)
    if name == "FcwError":
        from ._lib import FcwError

        return FcwError
    raise AttributeError(name)
