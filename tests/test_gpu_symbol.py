"""GPU parity of the reference-granularity per-symbol entry points
(fc_sync.hpp:38-75: tx_symbol, combine_symbols, rx_segment, rx_block_freq,
rx_symbol_simplified, rx_symbol_direct), called through the C ABI and
batched over units, against the CPU oracle's restatement of each function
(pinned to the reference in tests/test_oracle.py).  Tolerance: relative RMS
1e-5 (complex fp32 vs complex128); index work (rx_segment) bit-exact."""
import numpy as np
import pytest

import oracle as O
from paper_2008_00672_b200 import api

from helpers import rel_rms

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-5

# (N, [(L, c)], cp): config-1, config-5-like, mixed L, L == N, large L
CASES = [
    (1024, [(16, 512)], [80, 72, 72]),
    (4096, [(256, 2048 + 300), (256, 100)], [352, 288, 288, 288]),
    (256, [(32, 10), (64, 77), (16, 200)], [16, 12, 12, 12, 12]),
    (16, [(16, 8)], [2, 1, 1]),
    (2048, [(1024, 1500)], [160, 144, 144]),
]


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.complex64)).cuda()


def _rand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _plan(N, subs, cp, rng):
    wins = [rng.uniform(0.1, 1, L) for L, _ in subs]
    cfgs = [api.SubbandConfig(L=L, c=c, window=w) for (L, c), w in zip(subs, wins)]
    return api.Plan(N, cp, cfgs), wins


@pytest.mark.parametrize("N,subs,cp", CASES)
def test_tx_symbol_and_combine(N, subs, cp):
    rng = np.random.default_rng(N + len(subs))
    plan, wins = _plan(N, subs, cp, rng)
    S, B = 3, len(cp)
    for m, ((L, c), w) in enumerate(zip(subs, wins)):
        p = O.derive_params(N, L)
        syms = np.zeros((S, B, 3 * N // 2), np.complex64)
        for n in range(B):
            l_cp = O.cp_truncate(cp[n], N // L)[0]
            x = _rand(rng, S, L + l_cp)
            d_out = torch.empty((S, 3 * N // 2), dtype=torch.complex64, device="cuda")
            plan.tx_symbol(m, n, _dev(x), l_cp, d_out, S)
            torch.cuda.synchronize()
            got = d_out.cpu().numpy()
            for u in range(S):
                want = O.tx_symbol(x[u], L, c, w, p, cp, n)
                assert rel_rms(got[u], want) <= TOL, (m, n, u)
            syms[:, n] = got
        # combine_symbols (fc_sync.cpp:96-112): symbol n at sigma_n, in order
        d_w = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
        plan.combine_symbols(_dev(syms), d_w, S)
        torch.cuda.synchronize()
        want = np.zeros((S, plan.Q), np.complex128)
        for n in range(B):
            sg = O.symbol_sigma(n, cp, N)
            want[:, sg:sg + 3 * N // 2] += syms[:, n]
        assert rel_rms(d_w.cpu().numpy(), want) <= 1e-6


@pytest.mark.parametrize("N,subs,cp", CASES)
def test_rx_segment_block_freq_and_symbol_paths(N, subs, cp):
    rng = np.random.default_rng(7 * N + len(subs))
    plan, wins = _plan(N, subs, cp, rng)
    S, B = 2, len(cp)
    wave = _rand(rng, S, plan.Q + 37).astype(np.complex64)
    d_wave = _dev(wave)
    useful0 = plan.useful0 + 5
    for n in range(B):
        y0 = torch.empty((S, N), dtype=torch.complex64, device="cuda")
        y1 = torch.empty_like(y0)
        plan.rx_segment(d_wave, wave.shape[1], useful0, n, y0, y1, S)
        torch.cuda.synchronize()
        start = useful0 - O.derive_params(N, subs[0][0]).N_L + O.symbol_sigma(n, cp, N)
        assert np.array_equal(y0.cpu().numpy(), wave[:, start:start + N])  # bit-exact copy
        assert np.array_equal(y1.cpu().numpy(), wave[:, start + N // 2:start + 3 * N // 2])
        yy0 = y0.cpu().numpy().astype(np.complex128)
        yy1 = y1.cpu().numpy().astype(np.complex128)
        for m, ((L, c), w) in enumerate(zip(subs, wins)):
            p = O.derive_params(N, L)
            th = O.symbol_phase(n, c, cp, N)
            g = []
            for r, y in enumerate((y0, y1)):
                ph = O.block_phase(r, c, p.L_S, L) * th
                d_g = torch.empty((S, L), dtype=torch.complex64, device="cuda")
                plan.rx_block_freq(m, y, ph, d_g, S)
                torch.cuda.synchronize()
                got = d_g.cpu().numpy()
                for u in range(S):
                    want = O.rx_block_freq((yy0, yy1)[r][u], L, c, w, p, ph)
                    assert rel_rms(got[u], want) <= TOL, (n, m, r, u)
                g.append(d_g)
            d_s = torch.empty((S, L), dtype=torch.complex64, device="cuda")
            plan.rx_symbol_simplified(m, g[0], g[1], d_s, S)
            d_d = torch.empty_like(d_s)
            plan.rx_symbol_direct(m, n, y0, y1, d_d, S)
            torch.cuda.synchronize()
            gs, gd = d_s.cpu().numpy(), d_d.cpu().numpy()
            g0h, g1h = g[0].cpu().numpy().astype(np.complex128), g[1].cpu().numpy().astype(np.complex128)
            for u in range(S):
                assert rel_rms(gs[u], O.rx_symbol_simplified(g0h[u], g1h[u], p)) <= TOL, (n, m, u)
                assert rel_rms(gd[u], O.rx_symbol_direct(yy0[u], yy1[u], L, c, w, p, cp, n)) <= TOL, (n, m, u)
                # the fused path equals the direct path (fc_sync.hpp:66-68)
                assert rel_rms(gs[u], gd[u]) <= 2 * TOL


def test_per_symbol_chain_equals_rx_discontinuous():
    """tx_symbol -> combine_symbols -> rx_segment -> rx_block_freq x2 ->
    rx_symbol_simplified reproduces the whole-frame fcw_rx (fused)."""
    rng = np.random.default_rng(99)
    N, L, c, cp = 4096, 256, 2048 + 144, [352, 288, 288, 288, 288]
    plan, (w,) = _plan(N, [(L, c)], cp, rng)
    B, S = len(cp), 2
    p = O.derive_params(N, L)
    grid = _rand(rng, S, B, L)
    syms = np.zeros((S, B, 3 * N // 2), np.complex64)
    for n in range(B):
        l_cp = O.cp_truncate(cp[n], N // L)[0]
        x = np.fft.ifft(grid[:, n], axis=1) * np.sqrt(L)  # ofdm_modulate (ofdm.cpp:97-106)
        x = np.concatenate([x[:, L - l_cp:], x], axis=1)  # cp_insert (ofdm.cpp:108-116)
        d = torch.empty((S, 3 * N // 2), dtype=torch.complex64, device="cuda")
        plan.tx_symbol(0, n, _dev(x), l_cp, d, S)
        syms[:, n] = d.cpu().numpy()
    d_w = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.combine_symbols(_dev(syms), d_w, S)
    # the whole-frame TX of the same grid
    d_w2 = torch.empty_like(d_w)
    plan.tx(_dev(grid), d_w2, S, full=True)
    torch.cuda.synchronize()
    assert rel_rms(d_w.cpu().numpy(), d_w2.cpu().numpy()) <= 2 * TOL
    full = torch.empty((S, B, L), dtype=torch.complex64, device="cuda")
    plan.rx(d_w, plan.Q, plan.useful0, full, S, fused=True, full=True)
    torch.cuda.synchronize()
    for n in range(B):
        y0 = torch.empty((S, N), dtype=torch.complex64, device="cuda")
        y1 = torch.empty_like(y0)
        plan.rx_segment(d_w, plan.Q, plan.useful0, n, y0, y1, S)
        th = O.symbol_phase(n, c, cp, N)
        g = []
        for r, y in enumerate((y0, y1)):
            d_g = torch.empty((S, L), dtype=torch.complex64, device="cuda")
            plan.rx_block_freq(0, y, O.block_phase(r, c, p.L_S, L) * th, d_g, S)
            g.append(d_g)
        out = torch.empty((S, L), dtype=torch.complex64, device="cuda")
        plan.rx_symbol_simplified(0, g[0], g[1], out, S)
        torch.cuda.synchronize()
        assert rel_rms(out.cpu().numpy(), full[:, n].cpu().numpy()) <= 2 * TOL, n


def test_per_symbol_errors():
    rng = np.random.default_rng(1)
    plan, _ = _plan(1024, [(16, 512)], [80, 72], rng)
    y = torch.zeros((1, 1024), dtype=torch.complex64, device="cuda")
    wave = torch.zeros((1, plan.Q), dtype=torch.complex64, device="cuda")
    with pytest.raises(IndexError):  # rx_segment: symbol index outside CP schedule (fc_sync.cpp:146-147)
        plan.rx_segment(wave, plan.Q, plan.useful0, 2, y, y, 1)
    with pytest.raises(ValueError):  # waveform too short for symbol window (fc_sync.cpp:149-151)
        plan.rx_segment(wave, 100, plan.useful0, 1, y, y, 1)
    with pytest.raises(ValueError):  # CP exceeds leading overlap (fc_sync.cpp:35)
        plan.tx_symbol(0, 0, y, 9, y, 1)
    with pytest.raises(IndexError):
        plan.rx_block_freq(1, y, 1.0, y, 1)
