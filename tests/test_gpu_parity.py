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
