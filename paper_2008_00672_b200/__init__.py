"""fcwave-b200: B200-native symbol-synchronized FC-F-OFDM TX synthesis and RX
analysis (arXiv 2008.00672), a drop-in for the reference ``fcwave`` hot path.

The compute path is hand-written sm_100a CUDA in ``csrc/`` behind the C ABI
``include/fcwave_b200.h``; this package is the Python host mirror of the
reference's operator API.  There is no CPU fallback.
"""
from .api import (  # noqa: F401
    CpSchedule,
    FcParams,
    Numerology,
    PinnedBuffer,
    Plan,
    QamGrid,
    SubbandConfig,
    Waveform,
    centered_active_map,
    combined_length,
    cp_schedule,
    cp_truncate,
    derive_fc_params,
    design_window,
    first_block_overlap,
    make_numerology,
    nr_cp_schedule,
    rx_discontinuous,
    rx_discontinuous_all,
    symbol_sigma,
    tx_discontinuous,
)
from ._lib import FcwError  # noqa: F401

__version__ = "0.1.0"
