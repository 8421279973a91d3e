"""GPU continuous FC filterbank: ContPlan /
fcw_tx_continuous / fcw_rx_continuous against the C oracle's
tx_continuous / rx_continuous (pinned to the reference in tests/test_cont.py)
on identical inputs, batched over units, plus the reference's own known
answers (proj/tests/test_fc_core.cpp:209-276) on the GPU path."""
import numpy as np
import pytest

import oracle as O
from paper_2008_00672_b200 import api

from helpers import rel_rms

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-5

CASES = [
    (64, [16], [40], [7]),
    (256, [32, 64], [20, 100], [100, 71]),
    (1024, [16, 64, 256], [500, 200, 900], [230, 64, 513]),
    (2048, [512, 1024], [300, 1500], [1000, 2001]),
    (4096, [256] * 3, [3000, 3300, 3600], [2000, 2000, 1999]),
    (1024, [256, 256], [200, 700], [100, 257]),
    (2048, [512], [1024], [3000]),  # uniform L >= 512: team-wide short transforms
    (4096, [1024, 1024], [1000, 3000], [2500, 4100]),
    (1024, [16], [512], [300]),  # narrowband-eligible (config-1 geometry): nb kernels are not used for td I/O
    (4096, [256], [2048 + 700], [1500]),  # single uniform L = 256
]


@pytest.mark.parametrize("columns", [0, 1], ids=["time_domain_io", "column_passes"])
@pytest.mark.parametrize("N,Ls,cs,lens", CASES)
def test_continuous_tx_rx_match_oracle(N, Ls, cs, lens, columns, monkeypatch):
    # FCW_CONT_COLUMNS=1 forces the DFT_L / IDFT_L column passes around the
    # grid-I/O kernels; by default plans whose short paths support it run the
    # fused kernels with time-domain I/O (TX: uniform L = 256, RX: L <= 256)
    monkeypatch.setenv("FCW_CONT_COLUMNS", str(columns))
    rng = np.random.default_rng(N + len(Ls))
    wins = [rng.uniform(0, 1, L) for L in Ls]
    subs = [api.SubbandConfig(L=L, c=c, window=w) for L, c, w in zip(Ls, cs, wins)]
    S = 2
    streams = [[(rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64) for n in lens]
               for _ in range(S)]
    want = [O.tx_continuous([x.astype(np.complex128) for x in st], Ls, cs, wins, N, l_cp0=1) for st in streams]
    tx_len = len(want[0][0])
    plan = api.ContPlan(N, subs, lens, tx_len, l_cp0=1)
    assert plan.tx_len == tx_len and plan.useful0 == want[0][1]
    d_in = torch.from_numpy(np.stack([np.concatenate(st) for st in streams])).cuda()
    d_w = torch.empty((S, plan.tx_stride), dtype=torch.complex64, device="cuda")
    plan.tx(d_in, d_w, S)
    got = d_w.cpu().numpy()
    for u in range(S):
        assert rel_rms(got[u, :tx_len], want[u][0]) <= TOL, u
        # samples past the reference length carry only fp32 round-off of empty blocks
        assert np.max(np.abs(got[u, tx_len:]), initial=0.0) <= 1e-5 * np.max(np.abs(want[u][0]))
    # RX of the oracle's waveforms
    d_x = torch.from_numpy(np.stack([w[0] for w in want]).astype(np.complex64)).cuda()
    d_o = torch.empty((S, plan.rx_out_total), dtype=torch.complex64, device="cuda")
    plan.rx(d_x, d_o, S)
    out = d_o.cpu().numpy()
    for u in range(S):
        for m, (L, c, w) in enumerate(zip(Ls, cs, wins)):
            ref = O.rx_continuous(want[u][0], N, L, c, w)
            seg = out[u, plan.rx_out_off[m]:plan.rx_out_off[m] + plan.rx_out_len[m]]
            assert len(seg) == len(ref) and rel_rms(seg, ref) <= TOL, (u, m)


def test_known_answers_on_gpu():  # test_fc_core.cpp:209-253 through the reference-shaped API
    rng = np.random.default_rng(17)
    L, N = 8, 32
    x = rng.standard_normal(24) + 1j * rng.standard_normal(24)
    cfg = api.SubbandConfig(L=L, c=N // 2, window=np.ones(L))
    w = api.tx_continuous([api.CpOfdmSignal(x, [0], L)], [cfg], N, 0.5, 1.0)
    p = api.derive_fc_params(N, L)
    t = (p.L_O + np.arange(24)) * p.I
    assert np.max(np.abs(w.samples[t] - x / np.sqrt(p.I))) < 1e-5
    # L == N loopback is exact (up to fp32)
    L = N = 16
    x = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    cfg = api.SubbandConfig(L=L, c=N // 2, window=np.ones(L))
    w = api.tx_continuous([api.CpOfdmSignal(x, [2], L)], [cfg], N, 0.5, 1.0)
    p = api.derive_fc_params(N, L)
    assert w.useful0 == N // 2 + p.I * 2
    y = api.rx_continuous(w, cfg, p)
    assert np.max(np.abs(y[p.L_O:p.L_O + 40] - x)) < 1e-5
    # zero in, zero out
    cfg = api.SubbandConfig(L=8, c=11, window=api.design_window(8, 6, 1))
    w = api.tx_continuous([api.CpOfdmSignal(np.zeros(16), [0, 0], 8)], [cfg], 32, 0.5, 1.0)
    assert np.all(w.samples == 0)
    assert np.all(api.rx_continuous(w, cfg, api.derive_fc_params(32, 8)) == 0)


def test_continuous_errors():
    cfg = api.SubbandConfig(L=16, c=3, window=np.ones(16))
    with pytest.raises(ValueError):
        api.ContPlan(64, [cfg], [10], 32)  # waveform shorter than one FC block (fc_core.cpp:201)
    with pytest.raises(ValueError):
        api.tx_continuous([], [], 64, 0.5, 1.0)
