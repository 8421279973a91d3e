"""GPU link step around the path: device AWGN, power
measurement, demap + BER / EVM sums, checked against the C oracle (itself
pinned to the reference's functions in tests/test_link.py) on identical
inputs."""
import numpy as np
import pytest

import oracle as O
from paper_2008_00672_b200 import api, configs

from helpers import rel_rms

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cfg", ["config1", "config2"])
def test_loopback_link_stats_exact(cfg):
    """Noise-free TX -> RX: no bit errors, EVM sums equal the oracle's over the
    same received grid (bit errors exact, sums to 1e-12)."""
    w = getattr(configs, cfg)()
    plan = w.plan()
    S, seed = 3, 21
    grid = torch.empty((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(seed, 5, S, w.bits_per_symbol, grid)
    wave = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, S)
    out = torch.empty_like(grid)
    plan.rx(wave, plan.Q, plan.useful0, out, S, fused=True)
    st = plan.link_stats(out, S, seed, 5, w.bits_per_symbol)
    torch.cuda.synchronize()
    num, den, errs = O.link_stats(out.cpu().numpy().astype(np.complex128), seed, 5, w.bits_per_symbol)
    assert np.array_equal(st.bit_errors, errs) and st.bit_errors.sum() == 0
    np.testing.assert_allclose(st.evm_num, num, rtol=1e-12)
    np.testing.assert_allclose(st.evm_den, den, rtol=1e-12)
    assert np.all(st.n_bits == w.B * plan.row_active * w.bits_per_symbol)
    # FC filtering is not perfect reconstruction: the loopback EVM is the
    # filter's own distortion (reference: 33.2 dB at C1, 38.8 dB at 52 PRB)
    assert st.evm_db() > 20.0


def test_awgn_matches_oracle():
    w = configs.config1()
    plan = w.plan()
    S, L = 2, 5000
    rng = np.random.default_rng(2)
    x = (rng.standard_normal((S, L)) + 1j * rng.standard_normal((S, L))).astype(np.complex64)
    d = _dev(x)
    plan.awgn(d, L, S, 0.37, 1234, 9)
    got = d.cpu().numpy()
    for u in range(S):
        want = O.awgn(x[u].astype(np.complex128), 0.37, O.derive_seed(1234, 9 + u))
        assert rel_rms(got[u] - x[u], want - x[u]) <= 1e-6
    # sigma2 = 0 leaves the waveform unchanged
    d2 = _dev(x)
    plan.awgn(d2, L, S, 0.0, 1, 0)
    assert np.array_equal(d2.cpu().numpy(), x)


def test_wave_power_matches_oracle():
    w = configs.config2()
    plan = w.plan()
    S, L = 3, 40000
    rng = np.random.default_rng(4)
    x = (rng.standard_normal((S, L)) + 1j * rng.standard_normal((S, L))).astype(np.complex64)
    p = plan.wave_power(_dev(x), L, S, 17, 39000)
    for u in range(S):
        assert p[u] == pytest.approx(O.measure_power(x[u].astype(np.complex128), 17, 39000), rel=1e-12)
    p2 = plan.wave_power(_dev(x), L, S, -100, 10 ** 9)  # clipped like measure_power
    assert p2[0] == pytest.approx(O.measure_power(x[0].astype(np.complex128), 0, L), rel=1e-12)
    with pytest.raises(ValueError):
        plan.wave_power(_dev(x), L, S, 500, 500)


@pytest.mark.parametrize("snr_db", [4.0, 10.0])
def test_noisy_link_ber_matches_oracle(snr_db):
    """The reference's link step (scenario.cpp:455-491): measure the core
    power, AWGN at the SNR, RX, demap, count.  GPU decisions equal the oracle's
    decisions on the same received grid, bit for bit."""
    w = configs.config2()
    plan = w.plan()
    S, seed = 2, 77
    grid = torch.empty((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(seed, 0, S, w.bits_per_symbol, grid)
    wave = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, S)
    pw = plan.wave_power(wave, plan.Q, S, plan.useful0, plan.useful0 + w.B * w.N + sum(w.cp))
    sigma2 = api.awgn_noise_variance(float(pw[0]), snr_db, w.N, plan.row_active)
    plan.awgn(wave, plan.Q, S, sigma2, seed + 1, 0)
    out = torch.empty_like(grid)
    plan.rx(wave, plan.Q, plan.useful0, out, S, fused=True)
    st = plan.link_stats(out, S, seed, 0, w.bits_per_symbol)
    rx = out.cpu().numpy().astype(np.complex128)
    num, den, errs = O.link_stats(rx, seed, 0, w.bits_per_symbol)
    assert np.array_equal(st.bit_errors, errs)
    np.testing.assert_allclose(st.evm_num, num, rtol=1e-12)
    assert st.bit_errors.sum() > 0 if snr_db < 8 else True
    # EVM tracks the SNR (flat AWGN): within a dB of it
    assert abs(st.evm_db() - snr_db) < 1.0


@pytest.mark.parametrize("seg", [64, 256, 1024, 4096])
def test_psd_matches_oracle(seg):
    """Welch PSD (metrics.cpp:128-155) of device waveforms vs the oracle."""
    w = configs.config5()
    plan = w.plan()
    S = 2
    grid = torch.empty((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(3, 0, S, w.bits_per_symbol, grid)
    wave = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, S)
    n = 40 * seg + 5
    got = api.psd(wave, n, S, seg, 0.5, wave_stride=plan.Q)
    x = wave.cpu().numpy()
    for u in range(S):
        want = O.psd(x[u, :n].astype(np.complex128), seg, 0.5)
        assert np.max(np.abs(got[u] - want)) <= 1e-5 * np.max(want)
        assert rel_rms(got[u], want) <= 1e-5


def test_psd_tone_and_errors():
    seg = 64
    t = np.arange(seg * 40)
    d = _dev(np.exp(2j * np.pi * 12 * t / seg).astype(np.complex64)[None])
    p = api.psd(d, len(t), 1, seg)[0]
    assert int(np.argmax(p)) == 12 and p[12] / p[20] > 1e6
    with pytest.raises(ValueError):
        api.psd(d, 16, 1, 64)  # waveform shorter than one segment (metrics.cpp:129-130)
    with pytest.raises(ValueError):
        api.psd(d, len(t), 1, 64, 1.0)


@pytest.mark.parametrize("S,n_taps", [(3, 16), (1, 5), (3, 7)])
def test_apply_channel_matches_oracle(S, n_taps):
    # odd S * n_taps: the gain table must stay 8-byte aligned in the scratch block
    L = 20000
    d, p = api.exponential_profile(300.0, 20.0, n_taps)
    chans = [api.draw_tdl(d, p, 122.88e6, O.derive_seed(4, u)) for u in range(S)]
    rng = np.random.default_rng(6)
    x = (rng.standard_normal((S, L)) + 1j * rng.standard_normal((S, L))).astype(np.complex64)
    din, dout = _dev(x), torch.empty((S, L), dtype=torch.complex64, device="cuda")
    api.apply_channel(din, dout, L, S, chans)
    got = dout.cpu().numpy()
    for u in range(S):
        want = O.apply_channel(x[u].astype(np.complex128), chans[u].delays_samples, chans[u].gains)
        assert rel_rms(got[u], want) <= 1e-6
    with pytest.raises(ValueError):
        api.apply_channel(din, din, L, S, chans)  # out of place only
