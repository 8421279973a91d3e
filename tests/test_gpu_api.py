"""GPU checks of the host-facing layers: the `_fcwave` mirror
(paper_2008_00672_b200.fcwave, proj/python/tests/test_smoke.py:47-70 restated
on the GPU), the reference-shaped Python API against the oracle, the C++ host
library (tests/cpp/host_api_smoke.cpp), and error paths of the device entry
points."""
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2008_00672_b200 as fb
import paper_2008_00672_b200.fcwave as fc
from paper_2008_00672_b200 import _lib, configs

from helpers import rel_rms

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fcwave_mirror_chain_roundtrip():  # test_smoke.py:47-70 on the GPU path
    L, N, c = 16, 1024, 512
    bins = [1, 2, 3, 4, 12, 13, 14, 15]
    cols = []
    for n in range(3):
        col = [0j] * L
        for i, b in enumerate(bins):
            col[b] = np.exp(1j * (0.7 * n + i))
        cols.append(col)
    samples, useful0 = fc.tx_discontinuous(cols, L, N, c, 8, 2, 12)
    rec = fc.rx_discontinuous(samples, useful0, 3, L, N, c, 8, 2, 12)
    num = sum(abs(rec[n][b] - cols[n][b]) ** 2 for n in range(3) for b in bins)
    den = sum(abs(cols[n][b]) ** 2 for n in range(3) for b in bins)
    assert 10 * np.log10(den / num) > 25.0
    rec2 = fc.rx_discontinuous(samples, useful0, 3, L, N, c, 8, 2, 12, True)
    assert max(abs(a - b) for ra, rb in zip(rec, rec2) for a, b in zip(ra, rb)) < 1e-5
    # and against the oracle on the same inputs
    want, u0 = O.tx_discontinuous([np.array(cols)], [L], [c], [O.design_window(L, 12, 2)], O.cp_schedule(15, N, 3), N)
    assert u0 == useful0 and rel_rms(samples, want) <= 1e-5


def test_reference_shaped_multisubband():
    rng = np.random.default_rng(3)
    N, cps = 2048, fb.cp_schedule(fb.make_numerology(15, 2048), 14)
    cfgs = [fb.SubbandConfig(L=512, c=c, window=fb.design_window(512, 288, 4)) for c in (300, 600, 900)]
    grids = [fb.QamGrid(512, [], list(rng.standard_normal((14, 512)) + 1j * rng.standard_normal((14, 512))))
             for _ in cfgs]
    w = fb.tx_discontinuous(grids, cfgs, cps, N, 0.5, 30.72e6)
    want, u0 = O.tx_discontinuous([np.array(g.symbols) for g in grids], [512] * 3, [300, 600, 900],
                                  [c.window for c in cfgs], cps.per_symbol_high_rate, N)
    assert w.useful0 == u0 and rel_rms(w.samples, want) <= 1e-5
    allr = fb.rx_discontinuous_all(w, cfgs, cps, N, 0.5, True)
    for cfg, got in zip(cfgs, allr):
        ref = O.rx_discontinuous(w.samples, w.useful0, cps.per_symbol_high_rate, N, 512, cfg.c, cfg.window, True)
        assert rel_rms(got, ref) <= 1e-5


def test_cpp_host_library():
    exe = os.path.join(ROOT, "tests", "cpp", "host_api_smoke")
    libdir = os.path.join(ROOT, "paper_2008_00672_b200", "lib")
    src = os.path.join(ROOT, "tests", "cpp", "host_api_smoke.cpp")
    subprocess.run(["g++", "-std=c++17", "-O1", src, "-I", os.path.join(ROOT, "include"), "-I",
                    os.path.join(ROOT, "paper_2008_00672_b200", "csrc"), "-L", libdir, "-lfcwave_b200",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_device_entry_error_paths():
    w = configs.config1()
    plan = w.plan()
    S = 2
    grid = torch.zeros((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    wave = torch.zeros((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, 0)  # S = 0 is a no-op
    with pytest.raises(ValueError):
        plan.tx(grid, wave, -1)
    with pytest.raises(ValueError):  # waveform stride smaller than Q
        plan.tx(grid, wave, S, wave_stride=plan.Q - 1)
    with pytest.raises(ValueError):  # waveform too short for the symbol window (rx_segment)
        plan.rx(wave, plan.Q - 1, plan.useful0, grid, S)
    with pytest.raises(ValueError):  # useful0 before the first block
        plan.rx(wave, plan.Q, plan.useful0 - plan.N_L - 1, grid, S)
    with pytest.raises(ValueError):
        plan.gen_qam(1, 0, S, 3, grid)
    with pytest.raises(ValueError):
        fb.Plan(1024, [80, 72], [fb.SubbandConfig(L=16, c=0, window=np.ones(16), l_ofdm=32)])
    with pytest.raises(fb.FcwError) as ei:
        fb.Plan(1024, [80, 72], [fb.SubbandConfig(L=16, c=0, window=np.ones(16))], overlap=0.25)
    assert ei.value.code == _lib.FCW_ENOTSUP


def test_rx_accepts_longer_waveform_and_offset_useful0():
    """A received waveform longer than Q with symbol 0 later than N_L (useful0 is
    the caller's, Waveform::useful0): same columns as the oracle."""
    w = configs.config1()
    plan = w.plan()
    rng = np.random.default_rng(5)
    pad = 37
    wave = rng.standard_normal(plan.Q + 100) + 1j * rng.standard_normal(plan.Q + 100)
    out = plan.rx_host(wave.astype(np.complex64), len(wave), plan.useful0 + pad, 1, fused=True, full=True)[0]
    s = w.subbands[0]
    ref = O.rx_discontinuous(wave, plan.useful0 + pad, w.cp, w.N, s.L, s.c, s.window, True)
    assert rel_rms(out, ref) <= 1e-5


def test_linearity_full_frame():
    """TX is linear: tx(a*g1 + g2) == a*tx(g1) + tx(g2) at the full C5 frame size."""
    w = configs.config5()
    plan = w.plan()
    S = 2
    g = torch.empty((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(11, 0, S, 8, g)
    a = 0.5 - 0.25j
    comb = (a * g[0] + g[1]).unsqueeze(0).contiguous()
    waves = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    wc = torch.empty((1, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(g, waves, S)
    plan.tx(comb, wc, 1)
    torch.cuda.synchronize()
    lhs = wc[0].cpu().numpy().astype(np.complex128)
    rhs = a * waves[0].cpu().numpy().astype(np.complex128) + waves[1].cpu().numpy()
    assert rel_rms(lhs, rhs) <= 1e-5
