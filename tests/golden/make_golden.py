"""Generate golden vectors from the UNMODIFIED reference (oracle/_ref, built
from /root/reference/proj/src with the FFTW-API shim).  Run here, where the
reference is mounted:

    make -C oracle && python tests/golden/make_golden.py

Each .npz holds the inputs (N, cp, L/c/window per subband, full grids) and
the reference outputs: the tx_discontinuous waveform and, per subband, the
rx_discontinuous columns of the direct (0) and fused (1) paths.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def case(name, N, Ls, cs, windows, cp, rng, qam_bits=None):
    B = len(cp)
    grids = []
    for L in Ls:
        if qam_bits:
            g = np.zeros((B, L), complex)
            bins = O.centered_active_map(L, L // 2)
            g[:, bins] = [[O.qam_map(qam_bits, int(v)) for v in row]
                          for row in rng.integers(0, 1 << qam_bits, (B, len(bins)))]
        else:
            g = rng.standard_normal((B, L)) + 1j * rng.standard_normal((B, L))
        grids.append(g)
    wave, u0 = O.Ref.tx_discontinuous(grids, Ls, cs, windows, cp, N)
    out = dict(N=N, cp=np.array(cp), Ls=np.array(Ls), cs=np.array(cs), windows=np.concatenate(windows),
               grids=np.concatenate([g.reshape(-1) for g in grids]), wave=wave, useful0=u0)
    for m, (L, c, w) in enumerate(zip(Ls, cs, windows)):
        for fused in (0, 1):
            out[f"rx_{m}_{fused}"] = O.Ref.rx_discontinuous(wave, u0, cp, N, L, c, w, bool(fused))
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, len(wave))


def case_workload(name, w, B, seed):
    """A BASELINE workload's exact geometry (paper_2008_00672_b200.configs with
    the oracle's geometry backend) over its first B symbols, seeded 2^bits-QAM
    on the active bins.  Compact format: the packed grid and all outputs are
    stored as complex64 (the grid is rounded to fp32 BEFORE the reference runs,
    so the reference and the GPU consume identical inputs); outputs are the
    reference's full L-bin RX columns of every subband, concatenated."""
    cp = w.cp[:B]
    A = sum(len(m) for m in w.active_maps)
    packed = O.gen_grid(seed, 0, 1, B, A, w.bits_per_symbol)[0].astype(np.complex64)
    grids, off = [], 0
    for s, bins in zip(w.subbands, w.active_maps):
        g = np.zeros((B, s.L), complex)
        g[:, bins] = packed[:, off:off + len(bins)]
        grids.append(g)
        off += len(bins)
    Ls, cs, wins = [s.L for s in w.subbands], [s.c for s in w.subbands], [s.window for s in w.subbands]
    wave, u0 = O.Ref.tx_discontinuous(grids, Ls, cs, wins, cp, w.N)
    out = dict(N=w.N, cp=np.array(cp), Ls=np.array(Ls), cs=np.array(cs), windows=np.concatenate(wins),
               active=np.concatenate([np.asarray(m, np.int32) for m in w.active_maps]),
               n_active=np.array([len(m) for m in w.active_maps]), packed=packed,
               wave=wave.astype(np.complex64), useful0=u0, seed=seed, bits=w.bits_per_symbol)
    for fused in (0, 1):
        cols = [O.Ref.rx_discontinuous(wave, u0, cp, w.N, L, c, win, bool(fused)) for L, c, win in zip(Ls, cs, wins)]
        out[f"rx_full_{fused}"] = np.concatenate(cols, axis=1).astype(np.complex64)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, len(wave))


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built (needs /root/reference)")
    rng = np.random.default_rng(2008_00672)
    case("g1_c1_minislot", 1024, [16], [512], [O.design_window(16, 12, 2)], [80, 72], rng, qam_bits=2)
    case("g2_dense_L8_N32", 32, [8], [13], [rng.uniform(0, 1, 8)], [8, 4, 4], rng)
    case("g3_identity_L16_N16", 16, [16], [8], [np.ones(16)], [2, 1, 1], rng)
    case("g4_multisub_N256", 256, [32, 64, 16], [10, 77, 200], [rng.uniform(0, 1, L) for L in (32, 64, 16)],
         [16, 12, 12, 12, 12], rng)
    case("g5_c2_slot_N2048", 2048, [512] * 4, [1556, 1844, 84, 432],
         [O.design_window(512, n, 4) for n in (288, 288, 288, 408)], O.cp_schedule(15, 2048, 14), rng, qam_bits=4)
    case("g6_30khz_N4096_L16", 4096, [16] * 3, [2464, 2476, 2488], [O.design_window(16, 12, 2)] * 3,
         [352] + [288] * 13 + [352], rng, qam_bits=8)
    # the hot geometries of BASELINE configs 5 and 4 (the kernels bench.py times)
    from paper_2008_00672_b200 import configs

    geom = O.Geometry()
    case_workload("g7_c5_23sb_L256_N4096", configs.config5(geom=geom), 16, 7)
    case_workload("g8_c4_273sb_L16_N4096", configs.config4(geom=geom), 15, 8)


if __name__ == "__main__":
    main()
