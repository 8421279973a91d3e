"""Link step around the path, CPU side: the C oracle's
demap / EVM / BER / AWGN / power restatements pinned against the UNMODIFIED
reference functions compiled into oracle/_ref (ofdm.cpp:67-78 qam_demap,
metrics.cpp:105-127 ber / evm_db, channel.cpp:37-42,120-155 GaussianRng,
awgn_with_variance, awgn_noise_variance, measure_power)."""
import numpy as np
import pytest

import oracle as O
from paper_2008_00672_b200 import api

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _grid_points(bits):
    return np.array([O.qam_map(bits, s) for s in range(1 << bits)])


@pytest.mark.parametrize("bits", [2, 4, 6, 8])
def test_demap_inverts_map(bits):
    pts = _grid_points(bits)
    assert np.array_equal(O.qam_demap(bits, pts), np.arange(1 << bits))
    # unit average power (ofdm.cpp:29-33)
    assert abs(np.mean(np.abs(pts) ** 2) - 1.0) < 1e-12


@needs_ref
@pytest.mark.parametrize("bits", [2, 4, 6])
def test_demap_matches_reference(bits):
    rng = np.random.default_rng(bits)
    y = (rng.standard_normal(20000) + 1j * rng.standard_normal(20000)) * 0.9
    pts = _grid_points(bits)
    # decision boundaries and ties: midpoints between levels, and far outliers (clamp)
    s = abs(pts[0].real - pts[1].real) if bits == 2 else np.min(np.abs(np.diff(np.unique(pts.real))))
    lv = np.unique(pts.real)
    mids = (lv[:-1] + lv[1:]) / 2
    edge = np.concatenate([mids + 1j * mids[::-1], lv * 7 + 1j * lv * -7, [0j, 1e9 - 1e9j]])
    for arr in (y, pts, edge):
        assert np.array_equal(O.qam_demap(bits, arr), O.Ref.qam_demap(bits, arr))
    assert s > 0
    syms = np.arange(1 << bits, dtype=np.uint32)
    assert np.array_equal(O.Ref.qam_map(bits, syms), pts)


@needs_ref
def test_awgn_power_noise_variance_match_reference():
    rng = np.random.default_rng(5)
    w = (rng.standard_normal(4096) + 1j * rng.standard_normal(4096)) * 0.3
    for seed in (0, 1, 0xDEADBEEF, O.derive_seed(7, 3)):
        assert np.array_equal(O.awgn(w, 0.25, seed), O.Ref.awgn_with_variance(w, 0.25, seed))
    assert O.measure_power(w, 100, 3000) == O.Ref.measure_power(w, 100, 3000)
    assert O.measure_power(w, -5, 10 ** 6) == O.Ref.measure_power(w, -5, 10 ** 6)  # clipped span
    p = O.measure_power(w, 0, len(w))
    assert api.awgn_noise_variance(p, 9.5, 1024, 600) == pytest.approx(
        O.Ref.awgn_noise_variance(w, 9.5, 1024, 600), rel=1e-15)


def test_gaussian_statistics():
    w = np.zeros(200000, np.complex128)
    n = O.awgn(w, 2.0, 11)
    assert abs(np.mean(np.abs(n) ** 2) - 2.0) < 0.03
    assert abs(np.mean(n.real ** 2) - 1.0) < 0.02 and abs(np.mean(n.real)) < 0.01


@needs_ref
@pytest.mark.parametrize("bits", [2, 4, 6])
def test_link_stats_match_reference_metrics(bits):
    units, B, A = 2, 3, 50
    tx = O.gen_grid(99, 4, units, B, A, bits)
    rng = np.random.default_rng(bits + 10)
    rx = tx + 0.25 * (rng.standard_normal(tx.shape) + 1j * rng.standard_normal(tx.shape))
    num, den, errs = O.link_stats(rx, 99, 4, bits)
    for u in range(units):
        assert api.evm_db_from_sums(num[u], den[u]) == pytest.approx(O.Ref.evm_db(tx[u], rx[u]), abs=1e-12)
        # bits as the reference draws them (scenario.cpp:120): one splitmix64 draw per bit, LSB first
        draws = O.splitmix64_stream(O.derive_seed(99, 4 + u), B * A * bits)
        tx_bits = np.array([d & 1 for d in draws], np.uint8)
        rx_sym = O.Ref.qam_demap(bits, rx[u].reshape(-1))
        rx_bits = np.array([(s >> b) & 1 for s in rx_sym for b in range(bits)], np.uint8)
        assert errs[u] == int(np.sum(tx_bits != rx_bits))
        assert errs[u] / (B * A * bits) == pytest.approx(O.Ref.ber(tx_bits, rx_bits), rel=1e-15)
    assert errs.sum() > 0  # noise large enough to make decisions fail


def test_evm_db_edges():
    assert api.evm_db_from_sums(0.0, 1.0) == 300.0
    assert api.evm_db_from_sums(1e-40, 1.0) == 300.0
    assert api.evm_db_from_sums(0.01, 1.0) == pytest.approx(20.0)
    with pytest.raises(ValueError):
        api.evm_db_from_sums(1.0, 0.0)


# ---------------------------------------------------------------- f4 Welch PSD
@needs_ref
@pytest.mark.parametrize("seg,ov", [(64, 0.5), (1024, 0.5), (256, 0.0), (128, 0.75), (4096, 0.5)])
def test_psd_matches_reference(seg, ov):
    rng = np.random.default_rng(seg)
    x = rng.standard_normal(3 * seg + 17) + 1j * rng.standard_normal(3 * seg + 17)
    assert np.array_equal(O.psd(x, seg, ov), O.Ref.psd(x, seg, ov))


def test_psd_known_answers():  # proj/tests/test_metrics.cpp:132-156
    seg = 64
    t = np.arange(seg * 40)
    p = O.psd(np.exp(2j * np.pi * 12 * t / seg), seg)
    assert int(np.argmax(p)) == 12 and p[12] / (p[20] + 1e-300) > 1e6
    n = O.awgn(np.zeros(seg * 150, complex), 1.0, 3)  # GaussianRng(3).next_complex() stream
    pn = O.psd(n, seg)
    assert np.all(np.abs(10 * np.log10(pn / pn.mean())) < 1.0)
    with pytest.raises(ValueError):  # std::invalid_argument
        O.psd(np.zeros(16, complex), 64)


# -------------------------------------------------------------- f3 TDL channel
@needs_ref
def test_tdl_matches_reference():
    from paper_2008_00672_b200 import api
    d, p = api.exponential_profile(100.0, 10.0, 12)
    for seed in (0, 5, O.derive_seed(9, 2)):
        a = O.draw_tdl(d, p, 122.88e6, seed)
        b = O.Ref.draw_tdl(d, p, 122.88e6, seed)
        c = api.draw_tdl(d, p, 122.88e6, seed)  # the C ABI's host draw
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert np.array_equal(c.delays_samples, b[0]) and np.array_equal(c.gains, b[1])
    rng = np.random.default_rng(1)
    x = rng.standard_normal(5000) + 1j * rng.standard_normal(5000)
    assert np.array_equal(O.apply_channel(x, a[0], a[1]), O.Ref.apply_channel(x, a[0], a[1]))
    # frequency response = DFT of the tap line (channel.cpp:91-98)
    h = api.ChannelRealization(a[0], a[1]).frequency_response(64)
    want = np.zeros(64, complex)
    for dd, g in zip(a[0], a[1]):
        want[dd % 64] += g
    assert np.allclose(h, np.fft.fft(want))
    assert abs(np.sum(p) - 1.0) < 1e-12
