"""Continuous FC filterbank, CPU side: the C oracle's
tx_continuous / rx_continuous restatement pinned against the UNMODIFIED
reference (fc_core.cpp:155-223) compiled into oracle/_ref."""
import numpy as np
import pytest

import oracle as O

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

CASES = [
    (64, [16], [40], [7]),
    (256, [32, 64], [20, 100], [100, 71]),         # mixed L, different stream lengths (odd/even block counts)
    (1024, [16, 64, 256], [500, 200, 900], [230, 64, 513]),
    (2048, [512, 1024], [300, 1500], [1000, 2001]),
]


@needs_ref
@pytest.mark.parametrize("N,Ls,cs,lens", CASES)
def test_continuous_matches_reference(N, Ls, cs, lens):
    rng = np.random.default_rng(N + sum(lens))
    wins = [rng.uniform(0, 1, L) for L in Ls]
    streams = [rng.standard_normal(n) + 1j * rng.standard_normal(n) for n in lens]
    a, u = O.tx_continuous(streams, Ls, cs, wins, N, l_cp0=3)
    b, v = O.Ref.tx_continuous(streams, Ls, cs, wins, N, l_cp0=3)
    assert len(a) == len(b) and u == v
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))
    for L, c, w in zip(Ls, cs, wins):
        x = O.rx_continuous(a, N, L, c, w)
        y = O.Ref.rx_continuous(a, N, L, c, w)
        assert len(x) == len(y) and np.max(np.abs(x - y)) <= 1e-12 * np.max(np.abs(y))


@needs_ref
def test_continuous_block_counts():
    # continuous_block_count (fc_core.cpp:155-161) via the output lengths
    N, L = 128, 32
    for n in (0, 1, 15, 16, 17, 100):
        a, _ = O.Ref.tx_continuous([np.ones(max(n, 0), complex)], [L], [5], [np.ones(L)], N)
        p = O.derive_params(N, L)
        R = (n + p.L_O - p.L_L + p.L_S - 1) // p.L_S
        assert len(a) == (R - 1) * p.N_S + p.N


# Known answers of the reference's own continuous-FC tests
# (proj/tests/test_fc_core.cpp:209-316), restated on the C oracle.
def test_grid_samples_reproduce_padded_stream():  # test_fc_core.cpp:209-223
    rng = np.random.default_rng(17)
    L, N = 8, 32
    x = rng.standard_normal(24) + 1j * rng.standard_normal(24)
    w, _ = O.tx_continuous([x], [L], [N // 2], [np.ones(L)], N)
    p = O.derive_params(N, L)
    t = (p.L_O + np.arange(24)) * p.I
    assert np.max(np.abs(w[t] - x / np.sqrt(p.I))) < 1e-10


def test_zero_in_zero_out():  # test_fc_core.cpp:225-236
    w, _ = O.tx_continuous([np.zeros(16, complex)], [8], [11], [O.design_window(8, 6, 1)], 32)
    assert np.all(w == 0)
    assert np.all(O.rx_continuous(w, 32, 8, 11, O.design_window(8, 6, 1)) == 0)


def test_loopback_exact_when_L_equals_N():  # test_fc_core.cpp:238-253
    rng = np.random.default_rng(19)
    L = N = 16
    x = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    w, _ = O.tx_continuous([x], [L], [N // 2], [np.ones(L)], N, l_cp0=2)
    y = O.rx_continuous(w, N, L, N // 2, np.ones(L))
    p = O.derive_params(N, L)
    assert np.max(np.abs(y[p.L_O:p.L_O + 40] - x)) < 1e-10


def test_tone_phase_continuous_across_seams():  # test_fc_core.cpp:255-276
    L, N, c = 16, 64, 24
    w, _ = O.tx_continuous([np.ones(12 * L, complex)], [L], [c], [O.design_window(L, 12, 2)], N)
    amp = abs(w[6 * N])
    t = np.arange(4 * N, 8 * N)
    ideal = amp * np.exp(2j * np.pi * c * t / N)
    assert np.max(np.abs(np.angle(w[t] / ideal))) < 1e-9
