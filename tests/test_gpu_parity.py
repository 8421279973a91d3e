"""GPU parity: the sm_100a TX/RX kernels, called through the C ABI, against the
CPU oracle on identical seeded inputs.

Tolerances (BASELINE.json north_star): index maps and block boundaries
bit-exact; time- and frequency-domain samples within relative RMS 1e-5
(complex fp32 on the GPU vs complex128 in the oracle)."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2008_00672_b200 import api, configs

from helpers import oracle_rx, oracle_tx, rel_rms, truncate

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5
SEED = 20080672


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.complex64)).cuda()


def _cases():
    return {
        "c1": configs.config1(),
        "c2": configs.config2(),
        "c4_2slots": truncate(configs.config4(), 28),
        "c5_2slots": truncate(configs.config5(), 28),
    }


@pytest.fixture(scope="module", params=list(_cases().keys()))
def case(request):
    w = _cases()[request.param]
    plan = w.plan()
    S = 2
    grid = torch.empty((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(SEED, 0, S, w.bits_per_symbol, grid)
    torch.cuda.synchronize()
    return w, plan, S, grid


def test_generator_bit_exact(case):
    w, plan, S, grid = case
    want = O.gen_grid(SEED, 0, S, w.B, plan.row_active, w.bits_per_symbol).astype(np.complex64)
    got = grid.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_geometry_bit_exact(case):
    w, plan, S, grid = case
    assert plan.Q == O.combined_length(w.B, w.cp, O.derive_params(w.N, w.subbands[0].L))
    assert plan.useful0 == O.derive_params(w.N, w.subbands[0].L).N_L
    assert plan.sigma().tolist() == [O.symbol_sigma(n, w.cp, w.N) for n in range(w.B)]
    for m, s in enumerate(w.subbands):
        lcp, ex = plan.cp_split(m)
        I = w.N // s.L
        assert [(int(a), int(b)) for a, b in zip(lcp, ex)] == [O.cp_truncate(c, I) for c in w.cp]


def test_tx_parity(case):
    w, plan, S, grid = case
    wave = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, S)
    torch.cuda.synchronize()
    got = wave.cpu().numpy()
    packed = grid.cpu().numpy().astype(np.complex128)
    for u in range(S):
        want, useful0 = oracle_tx(w, packed[u])
        assert useful0 == plan.useful0
        assert len(want) == plan.Q
        assert rel_rms(got[u], want) <= TOL, (w.name, u, rel_rms(got[u], want))


@pytest.mark.parametrize("fused", [False, True])
def test_rx_parity(case, fused):
    w, plan, S, grid = case
    packed = grid.cpu().numpy().astype(np.complex128)
    waves, wants_p, wants_f = [], [], []
    for u in range(S):
        wv, useful0 = oracle_tx(w, packed[u])
        waves.append(wv)
        p, f = oracle_rx(w, wv, useful0, fused)
        wants_p.append(p)
        wants_f.append(f)
    wdev = _dev(np.stack(waves))
    out_p = torch.empty((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    out_f = torch.empty((S, w.B, plan.row_full), dtype=torch.complex64, device="cuda")
    plan.rx(wdev, plan.Q, plan.useful0, out_p, S, fused=fused)
    plan.rx(wdev, plan.Q, plan.useful0, out_f, S, fused=fused, full=True)
    torch.cuda.synchronize()
    for u in range(S):
        assert rel_rms(out_p[u].cpu().numpy(), wants_p[u]) <= TOL
        assert rel_rms(out_f[u].cpu().numpy(), wants_f[u]) <= TOL


# ---------------------------------------------------------------- generic path
def _golden():
    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    return sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith(".npz"))


def _hot_golden():
    return [p for p in _golden() if "packed" in np.load(p).files]


@pytest.mark.parametrize("sched", ["default", "chunk1", "chunk7", "static"])
@pytest.mark.parametrize("path", _hot_golden(), ids=lambda p: os.path.basename(p)[:-4])
def test_gpu_matches_reference_golden_hot_geometry(path, sched, monkeypatch):
    """The UNMODIFIED reference's outputs at the exact geometry of BASELINE
    configs 5 (g7: 23 x L=256, the zero-bin kernel variant) and 4 (g8: 273 x
    L=16), through the same packed-grid plan and kernels bench.py times, under
    every work schedule (chunk1 / chunk7: a TX carry recompute at every run
    start)."""
    if sched.startswith("chunk"):
        monkeypatch.setenv("FCW_CHUNK", sched[5:])
    elif sched == "static":
        monkeypatch.setenv("FCW_SCHED", "static")
    z = np.load(path)
    N, cp = int(z["N"]), z["cp"].tolist()
    Ls, cs = z["Ls"].tolist(), z["cs"].tolist()
    wins = np.split(z["windows"], np.cumsum(Ls)[:-1])
    maps = [m.tolist() for m in np.split(z["active"], np.cumsum(z["n_active"])[:-1])]
    subs = [api.SubbandConfig(L=L, c=c, window=w) for L, c, w in zip(Ls, cs, wins)]
    plan = api.Plan(N, cp, subs, maps)
    S = 3  # three identical units: every unit of a batched launch must match
    grid = _dev(np.broadcast_to(z["packed"], (S,) + z["packed"].shape))
    wave = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, S)
    torch.cuda.synchronize()
    assert plan.Q == len(z["wave"]) and plan.useful0 == int(z["useful0"])
    got = wave.cpu().numpy()
    for u in range(S):
        assert rel_rms(got[u], z["wave"]) <= TOL, (u, rel_rms(got[u], z["wave"]))
    wref = _dev(np.broadcast_to(z["wave"], (S, len(z["wave"]))))
    act = np.concatenate([np.asarray(m) + off for m, off in zip(maps, np.cumsum([0] + Ls[:-1]))])
    for fused in (0, 1):
        want = z[f"rx_full_{fused}"]
        out_p = torch.empty((S, len(cp), plan.row_active), dtype=torch.complex64, device="cuda")
        out_f = torch.empty((S, len(cp), plan.row_full), dtype=torch.complex64, device="cuda")
        plan.rx(wref, plan.Q, plan.useful0, out_p, S, fused=bool(fused))
        plan.rx(wref, plan.Q, plan.useful0, out_f, S, fused=bool(fused), full=True)
        torch.cuda.synchronize()
        for u in range(S):
            assert rel_rms(out_f[u].cpu().numpy(), want) <= TOL, (u, fused)
            assert rel_rms(out_p[u].cpu().numpy(), want[:, act]) <= TOL, (u, fused)


@pytest.mark.parametrize("path", [p for p in _golden() if p not in _hot_golden()],
                         ids=lambda p: os.path.basename(p)[:-4])
def test_gpu_matches_reference_golden(path):
    """The committed outputs of the UNMODIFIED reference (tests/golden) — full
    DFT-bin grids in, reference waveform / RX columns out."""
    z = np.load(path)
    N, cp = int(z["N"]), z["cp"].tolist()
    Ls, cs = z["Ls"].tolist(), z["cs"].tolist()
    wins = np.split(z["windows"], np.cumsum(Ls)[:-1])
    B = len(cp)
    subs = [api.SubbandConfig(L=L, c=c, window=w) for L, c, w in zip(Ls, cs, wins)]
    plan = api.Plan(N, cp, subs)
    grids = np.split(z["grids"], np.cumsum([B * L for L in Ls])[:-1])
    rows = np.concatenate([g.reshape(B, L) for g, L in zip(grids, Ls)], axis=1)
    wave = plan.tx_host(rows.reshape(-1), 1, full=True)[0]
    assert plan.Q == len(z["wave"]) and plan.useful0 == int(z["useful0"])
    assert rel_rms(wave, z["wave"]) <= TOL
    for fused in (0, 1):
        got = plan.rx_host(z["wave"].astype(np.complex64), plan.Q, plan.useful0, 1, fused=bool(fused), full=True)[0]
        off = 0
        for m, L in enumerate(Ls):
            assert rel_rms(got[:, off:off + L], z[f"rx_{m}_{fused}"]) <= TOL, (m, fused)
            off += L


def _random_case(rng, N, Ls, cps):
    subs, maps = [], []
    for L in Ls:
        c = int(rng.integers(0, N))
        subs.append(api.SubbandConfig(L=L, c=c, window=rng.uniform(0, 1, L)))
        maps.append(sorted(rng.choice(L, size=max(1, L // 2), replace=False).tolist()))
    return subs, maps


@pytest.mark.parametrize("N,Ls,cps", [
    (32, [8], [8, 4, 4, 4]),
    (16, [16], [2, 1, 1]),
    (64, [16, 8, 4], [8, 4, 4, 8, 4]),
    (256, [32, 64, 16, 64], [16, 12, 12, 12, 16, 12]),
    (1024, [16, 64, 256], [80, 72, 72, 72]),     # mixed L at a specialised N -> generic kernel
    (2048, [1024, 512], [144] * 6),
    (4096, [32] * 7, [352, 288, 288, 288]),
    (4096, [1024, 64], [352, 288, 288]),
    (4096, [256] * 3, [352, 288, 288, 288]),   # uniform L = 256 with full-support windows (no zero-bin variant)
    (1024, [16], [80, 72, 72]),                # one L = 16 subband: narrowband long transforms
])
def test_random_geometries(N, Ls, cps):
    rng = np.random.default_rng(N + len(Ls))
    subs, maps = _random_case(rng, N, Ls, cps)
    B = len(cps)
    plan = api.Plan(N, cps, subs, maps)
    S = 3
    grid = (rng.standard_normal((S, B, plan.row_active)) + 1j * rng.standard_normal((S, B, plan.row_active)))
    grid = grid.astype(np.complex64)
    wave = plan.tx_host(grid, S)
    w = type("W", (), {})()
    w.subbands, w.active_maps, w.B, w.N, w.cp = subs, maps, B, N, cps
    for u in range(S):
        want, u0 = oracle_tx(w, grid[u].astype(np.complex128))
        assert rel_rms(wave[u], want) <= TOL, u
    for fused in (False, True):
        out = plan.rx_host(wave, plan.Q, plan.useful0, S, fused=fused)
        for u in range(S):
            want_p, _ = oracle_rx(w, wave[u].astype(np.complex128), plan.useful0, fused)
            assert rel_rms(out[u], want_p) <= TOL, (u, fused)


def _zv_case(n_acts, cs, n_tb=4):
    """Uniform L = 256 at N = 4096 with centred active maps and design_window windows: the
    structure the zero-bin (zv) kernels accept."""
    subs, maps = [], []
    for n_act, c in zip(n_acts, cs):
        subs.append(api.SubbandConfig(L=256, c=c, window=api.design_window(256, n_act, n_tb)))
        maps.append(api.centered_active_map(256, n_act, skip_dc=False))
    return subs, maps


@pytest.mark.parametrize("n_acts,cs,variant", [
    # three classes whose pairs differ between TX (one subband per warp) and RX (pairs (0,1), (2,-))
    ([144, 108, 144], [600, 1500, 3200], 1),
    # adjacent subbands sharing transition bins, a narrower one in the middle: mixed class pairs
    ([144, 144, 120, 144, 144], [400, 552, 700, 848, 1000], None),
    # ten adjacent equal subbands: a TX pair round with idle half-warps (slots 10..15 repeat the last subband)
    ([144] * 10, [200 + 144 * i for i in range(10)], 1),
    # ten subbands of six widths: more class pairs than TMEM rows -> the plan falls back to the general kernels
    ([144, 132, 120, 108, 96, 84, 144, 132, 120, 108], [300 + 160 * i for i in range(10)], 0),
])
def test_zero_bin_plans_with_mixed_classes(n_acts, cs, variant):
    """zv plans keep per-lane (weight, slot code) rows of their bin classes in TMEM, one row per
    PAIR of classes that the schedule puts in one warp (fcw_capi.cpp); plans needing more than
    four rows must fall back.  Either way the results match the oracle."""
    N, cps = 4096, [352, 288, 288, 288, 288]
    subs, maps = _zv_case(n_acts, cs)
    rng = np.random.default_rng(sum(n_acts))
    B = len(cps)
    plan = api.Plan(N, cps, subs, maps)
    if variant is not None:
        assert plan.kernel_variant == variant, (plan.kernel_variant, plan.tmem_rows)
    assert plan.tmem_rows <= 4
    S = 2
    grid = (rng.standard_normal((S, B, plan.row_active)) + 1j * rng.standard_normal((S, B, plan.row_active)))
    grid = grid.astype(np.complex64)
    wave = plan.tx_host(grid, S)
    w = type("W", (), {})()
    w.subbands, w.active_maps, w.B, w.N, w.cp = subs, maps, B, N, cps
    for u in range(S):
        want, u0 = oracle_tx(w, grid[u].astype(np.complex128))
        assert rel_rms(wave[u], want) <= TOL, u
    for fused in (False, True):
        out = plan.rx_host(wave, plan.Q, plan.useful0, S, fused=fused)
        for u in range(S):
            want_p, _ = oracle_rx(w, wave[u].astype(np.complex128), plan.useful0, fused)
            assert rel_rms(out[u], want_p) <= TOL, (u, fused)


def test_kernel_smem_attribute_across_plans():
    """One generic kernel, plans with more / less / more dynamic SMEM: the
    kernel's SMEM attribute must never be lowered under a larger plan (it was
    once cached per (kernel, smem) and the smaller plan reset it)."""
    rng = np.random.default_rng(7)
    cps = [144] * 3
    plans = []
    for Ls in ([1024, 512], [512, 64], [1024, 512]):
        subs, maps = _random_case(rng, 2048, Ls, cps)
        plans.append((api.Plan(2048, cps, subs, maps), subs, maps))
    for plan, subs, maps in plans:
        grid = (rng.standard_normal((1, len(cps), plan.row_active))
                + 1j * rng.standard_normal((1, len(cps), plan.row_active))).astype(np.complex64)
        wave = plan.tx_host(grid, 1)
        w = type("W", (), {})()
        w.subbands, w.active_maps, w.B, w.N, w.cp = subs, maps, len(cps), 2048, cps
        want, _ = oracle_tx(w, grid[0].astype(np.complex128))
        assert rel_rms(wave[0], want) <= TOL


@pytest.mark.parametrize("chunk", ["1", "3", "7", "280"])
def test_chunk_boundaries_full_frame(chunk, monkeypatch):
    """Full 280-symbol C5 frame: every CTA-run boundary recomputes the carry of
    the symbol before it; results must not depend on the run length."""
    monkeypatch.setenv("FCW_CHUNK", chunk)
    w = configs.config5()
    plan = w.plan()
    grid = torch.empty((1, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(SEED, 5, 1, w.bits_per_symbol, grid)
    wave = torch.empty((1, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, 1)
    out = torch.empty_like(grid)
    plan.rx(wave, plan.Q, plan.useful0, out, 1, fused=True)
    torch.cuda.synchronize()
    key = ("c5full",)
    if key not in _FULL:
        g = grid[0].cpu().numpy().astype(np.complex128)
        ww, u0 = oracle_tx(w, g)
        _FULL[key] = (ww, oracle_rx(w, wave[0].cpu().numpy().astype(np.complex128), u0, True)[0])
    want_w, want_r = _FULL[key]
    assert rel_rms(wave[0].cpu().numpy(), want_w) <= TOL
    assert rel_rms(out[0].cpu().numpy(), want_r) <= TOL


_FULL: dict = {}


# ------------------------------------------------------- config 3 (mixed)
def test_c3_mixed_numerology():
    """Two numerologies summed on one waveform: glue = two oracle calls + an
    offset sum (parity unpinned by the reference, which cannot express it)."""
    mw = configs.config3()
    plans = mw.plans()
    mixed = mw.mixed(plans)
    S = 2
    grids = []
    for i, (w, p) in enumerate(zip(mw.banks, plans)):
        g = torch.empty((S, w.B, p.row_active), dtype=torch.complex64, device="cuda")
        p.gen_qam(SEED + i, 0, S, mw.bits_per_symbol, g)
        grids.append(g)
    wave = torch.empty((S, mixed.Q), dtype=torch.complex64, device="cuda")
    mixed.tx(grids, wave, S)
    torch.cuda.synchronize()
    assert mixed.Q == 31568 and mw.offsets == [0, 184]
    for u in range(S):
        want = np.zeros(mixed.Q, np.complex128)
        for (w, p), off, g in zip(zip(mw.banks, plans), mw.offsets, grids):
            wv, u0 = oracle_tx(w, g[u].cpu().numpy().astype(np.complex128))
            want[off:off + len(wv)] += wv
        assert rel_rms(wave[u].cpu().numpy(), want) <= TOL
        outs = [torch.empty((S, w.B, p.row_active), dtype=torch.complex64, device="cuda")
                for w, p in zip(mw.banks, plans)]
        mixed.rx(_dev(np.stack([want] * S)), outs, S, fused=True)
        torch.cuda.synchronize()
        for (w, p), off, o in zip(zip(mw.banks, plans), mw.offsets, outs):
            rp, _ = oracle_rx(w, want, off + p.useful0, True)
            assert rel_rms(o[u].cpu().numpy(), rp) <= TOL


def test_mixed_numerology_zero_fills_uncovered_spans():
    """Bank order reversed (the 30 kHz bank first, at offset 184): samples
    [0, 184) and past bank 0's end are only ever ADDED to by bank 1, so the
    composition must zero them first — the output buffer starts as garbage."""
    mw = configs.config3()
    plans = mw.plans()
    banks = [(plans[1], mw.offsets[1]), (plans[0], mw.offsets[0])]
    mixed = api.MixedNumerology(banks)
    S = 2
    grids = []
    for i, (w, p) in enumerate(zip(mw.banks, plans)):
        g = torch.empty((S, w.B, p.row_active), dtype=torch.complex64, device="cuda")
        p.gen_qam(SEED + i, 0, S, mw.bits_per_symbol, g)
        grids.append(g)
    wave = torch.full((S, mixed.Q), 1e3 + 1e3j, dtype=torch.complex64, device="cuda")
    mixed.tx([grids[1], grids[0]], wave, S)
    torch.cuda.synchronize()
    for u in range(S):
        want = np.zeros(mixed.Q, np.complex128)
        for (w, p), off, g in zip(zip(mw.banks, plans), mw.offsets, grids):
            wv, _ = oracle_tx(w, g[u].cpu().numpy().astype(np.complex128))
            want[off:off + len(wv)] += wv
        assert rel_rms(wave[u].cpu().numpy(), want) <= TOL


def test_tx_accumulate_adds():
    w = truncate(configs.config5(), 16)
    plan = w.plan()
    S = 2
    grid = torch.empty((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(SEED, 0, S, w.bits_per_symbol, grid)
    a = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, a, S)
    b = a.clone()
    plan.tx(grid, b, S, accumulate=True)
    torch.cuda.synchronize()
    assert torch.allclose(b, 2 * a, rtol=1e-6, atol=1e-7)


def test_narrowband_wrapping_span():
    """N = 1024, one L = 16 subband whose 16-bin span wraps through bin 0: the
    narrowband long transforms (k0 = c - 8 mod N) against the oracle."""
    rng = np.random.default_rng(11)
    for c in (3, 1020, 512):
        subs = [api.SubbandConfig(L=16, c=c, window=rng.uniform(0.1, 1, 16))]
        maps = [sorted(rng.choice(16, size=12, replace=False).tolist())]
        cps = [80, 72, 72, 72]
        plan = api.Plan(1024, cps, subs, maps)
        S = 5
        grid = (rng.standard_normal((S, len(cps), plan.row_active)) +
                1j * rng.standard_normal((S, len(cps), plan.row_active))).astype(np.complex64)
        wave = plan.tx_host(grid, S)
        w = type("W", (), {})()
        w.subbands, w.active_maps, w.B, w.N, w.cp = subs, maps, len(cps), 1024, cps
        for u in range(S):
            want, _ = oracle_tx(w, grid[u].astype(np.complex128))
            assert rel_rms(wave[u], want) <= TOL, (c, u)
        for fused in (False, True):
            out = plan.rx_host(wave, plan.Q, plan.useful0, S, fused=fused)
            for u in range(S):
                want_p, _ = oracle_rx(w, wave[u].astype(np.complex128), plan.useful0, fused)
                assert rel_rms(out[u], want_p) <= TOL, (c, u, fused)


# ------------------------------------------------- exported index maps (C ABI)
@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c5", "random"])
def test_plan_index_maps_bit_exact(name):
    """fcw_plan_bin_map / fcw_plan_rx_starts against the oracle's maps
    (fc_core.cpp:80-84, fc_sync.cpp:148): bit-exact, every subband."""
    if name == "random":
        rng = np.random.default_rng(5)
        subs = [api.SubbandConfig(L=L, c=int(rng.integers(0, 2048)), window=rng.uniform(0, 1, L))
                for L in (16, 64, 256, 32, 512)]
        cps = [160, 144, 144, 144]
        plan, N, cp = api.Plan(2048, cps, subs), 2048, cps
    else:
        w = configs.get(name)
        subs, plan, N, cp = w.subbands, w.plan(), w.N, w.cp
    for m, s in enumerate(subs):
        q, b = plan.bin_map(m)
        oq, ob = O.bin_map(s.L, s.c, N)
        assert np.array_equal(q, oq) and np.array_equal(b, ob), m
    for off in (0, 37):
        u0 = plan.useful0 + off
        want = O.rx_starts(u0, cp, N, subs[0].L)
        assert np.array_equal(plan.rx_starts(u0), want)
    with pytest.raises(IndexError):
        plan.bin_map(len(subs))


@pytest.mark.parametrize("sched", ["default", "chunk1", "chunk7", "static"])
def test_c4_full_frame(sched, monkeypatch):
    """All 280 symbols of config 4 (273 x L = 16, NR CP 352 / 288) under every
    work schedule: TX against the oracle, and fused + direct RX of the
    oracle's waveform against the oracle."""
    if sched.startswith("chunk"):
        monkeypatch.setenv("FCW_CHUNK", sched[5:])
    elif sched == "static":
        monkeypatch.setenv("FCW_SCHED", "static")
    w = configs.config4()
    plan = w.plan()
    grid = torch.empty((1, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(SEED, 3, 1, w.bits_per_symbol, grid)
    wave = torch.empty((1, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, 1)
    torch.cuda.synchronize()
    key = ("c4full",)
    if key not in _FULL:
        ww, u0 = oracle_tx(w, grid[0].cpu().numpy().astype(np.complex128))
        _FULL[key] = (ww, {f: oracle_rx(w, ww, u0, f)[0] for f in (True, False)})
    want_w, want_r = _FULL[key]
    assert rel_rms(wave[0].cpu().numpy(), want_w) <= TOL
    wref = _dev(want_w[None, :])
    for f in (True, False):
        o = torch.empty_like(grid)
        plan.rx(wref, plan.Q, plan.useful0, o, 1, fused=f)
        torch.cuda.synchronize()
        assert rel_rms(o[0].cpu().numpy(), want_r[f]) <= TOL, f
