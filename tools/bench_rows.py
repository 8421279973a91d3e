#!/usr/bin/env python3
"""Measurement of the SURVEY §8 "next" rows built around the path (dev tool;
bench.py keeps the headline contract).  One JSON line per row:

  link  (f1/f3): fcw_link_stats (demap + bit errors + EVM sums) and fcw_awgn /
                 fcw_wave_power on the C5 unit geometry; HBM roofline of the
                 bytes each pass must move.
  cont  (f2):    continuous FC TX + RX (fcw_tx_continuous / fcw_rx_continuous)
                 on the C5 carrier (23 subbands, L = 256, N = 4096) fed with
                 one frame of CP-OFDM low-rate samples per subband and unit.

  python tools/bench_rows.py [--units 64] [--steps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=64)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import torch

    from paper_2008_00672_b200 import api, configs

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    torch.cuda.set_device(0)
    w = configs.get("c5")
    plan = w.plan()
    S = args.units

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.steps

    # ---- f1 / f3: link step on the C5 RX grid and waveform
    grid = torch.empty((S, w.B, plan.row_active), dtype=torch.complex64, device="cuda")
    plan.gen_qam(7, 0, S, w.bits_per_symbol, grid)
    wave = torch.empty((S, plan.Q), dtype=torch.complex64, device="cuda")
    plan.tx(grid, wave, S)
    out = torch.empty_like(grid)
    plan.rx(wave, plan.Q, plan.useful0, out, S, fused=True)
    n_el = S * w.B * plan.row_active
    ms_link = timed(lambda: plan.link_stats(out, S, 7, 0, w.bits_per_symbol))
    ms_awgn = timed(lambda: plan.awgn(wave, plan.Q, S, 1e-3, 3, 0))
    ms_pow = timed(lambda: plan.wave_power(wave, plan.Q, S, plan.useful0, plan.useful0 + plan.frame_samples))
    st = plan.link_stats(out, S, 7, 0, w.bits_per_symbol)
    print(json.dumps({
        "row": "f1/f3 link step", "config": {"workload": "c5 geometry", "units": S, "elements": n_el},
        "link_stats": {"ms": ms_link, "Msymbols_per_s": n_el / ms_link / 1e3,
                       "hbm_gbs": 8 * n_el / ms_link / 1e6, "frac": 8 * n_el / ms_link / 1e6 / peak},
        "awgn": {"ms": ms_awgn, "Msamples_per_s": S * plan.Q / ms_awgn / 1e3,
                 "hbm_gbs": 16 * S * plan.Q / ms_awgn / 1e6, "frac": 16 * S * plan.Q / ms_awgn / 1e6 / peak},
        "wave_power": {"ms": ms_pow, "hbm_gbs": 8 * S * plan.frame_samples / ms_pow / 1e6,
                       "frac": 8 * S * plan.frame_samples / ms_pow / 1e6 / peak},
        "loopback": {"evm_db": st.evm_db(), "ber": st.ber()}, "peak_gbs": peak}))

    # ---- f2: continuous FC on the C5 carrier
    cps = w.cp
    lens = []
    for sb in w.subbands:
        I = w.N // sb.L
        lens.append(sum(sb.L + c // I for c in cps))
    cplan = api.ContPlan(w.N, w.subbands, lens, plan.Q, l_cp0=cps[0] // (w.N // w.subbands[0].L))
    rng = np.random.default_rng(1)
    streams = torch.from_numpy(
        (rng.standard_normal((S, cplan.stream_total)) + 1j * rng.standard_normal((S, cplan.stream_total)))
        .astype(np.complex64)).cuda()
    cw = torch.empty((S, cplan.tx_stride), dtype=torch.complex64, device="cuda")
    co = torch.empty((S, cplan.rx_out_total), dtype=torch.complex64, device="cuda")
    ms_tx = timed(lambda: cplan.tx(streams, cw, S))
    n = min(cplan.tx_stride, cplan.rx_wave_len)
    rx_in = torch.zeros((S, cplan.rx_wave_len), dtype=torch.complex64, device="cuda")
    rx_in[:, :n] = cw[:, :n]
    ms_rx = timed(lambda: cplan.rx(rx_in, co, S))
    samples = S * cplan.tx_len
    alg = 8 * S * (cplan.stream_total + cplan.tx_len) * 2  # TX in+out, RX in+out (low-rate ~ stream size)
    print(json.dumps({
        "row": "f2 continuous FC", "config": {"workload": "c5 carrier, continuous", "units": S,
                                             "stream_total": cplan.stream_total, "tx_len": cplan.tx_len},
        "Msamples_per_s": samples / (ms_tx + ms_rx) / 1e3, "tx_ms": ms_tx, "rx_ms": ms_rx,
        "algorithmic_gbs": alg / (ms_tx + ms_rx) / 1e6, "frac": alg / (ms_tx + ms_rx) / 1e6 / peak}))


if __name__ == "__main__":
    main()
