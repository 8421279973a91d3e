// C++ host-library smoke test (the fcwave:: -> fcwave_b200:: swap):
// builds a 2-symbol C1 waveform with tx_discontinuous, analyses it with
// rx_discontinuous (direct and fused) and prints the in-band EVM and the
// fused-vs-direct difference; checks the exception class of a bad input.
#include <cmath>
#include <complex>
#include <cstdio>
#include <stdexcept>

#include "fcwave_b200.hpp"

namespace fw = fcwave_b200;

int main() {
    const int L = 16, N = 1024, c = 512;
    const auto num = fw::make_numerology(15, N);
    const auto cps = fw::cp_schedule(num, 3);
    fw::SubbandConfig cfg;
    cfg.L = L;
    cfg.l_ofdm = L;
    cfg.c = c;
    cfg.window = fw::design_window(L, 12, 2);
    fw::QamGrid g;
    g.l_ofdm = L;
    g.active_map = {1, 2, 3, 4, 12, 13, 14, 15};
    for (int n = 0; n < 3; ++n) {
        fw::cvec col(L, fw::cd(0, 0));
        for (size_t i = 0; i < g.active_map.size(); ++i) col[g.active_map[i]] = std::polar(1.0, 0.7 * n + i);
        g.symbols.push_back(col);
    }
    const fw::Waveform w = fw::tx_discontinuous({g}, {cfg}, cps, N, 0.5, num.fs_hz());
    const auto d = fw::rx_discontinuous(w, cfg, cps, N, 0.5, false);
    const auto f = fw::rx_discontinuous(w, cfg, cps, N, 0.5, true);
    double num_e = 0, den = 0, diff = 0;
    for (int n = 0; n < 3; ++n)
        for (int b : g.active_map) {
            num_e += std::norm(d[n][b] - g.symbols[n][b]);
            den += std::norm(g.symbols[n][b]);
            diff = std::max(diff, std::abs(d[n][b] - f[n][b]));
        }
    // the reference's per-symbol API (fc_sync.hpp:24-75) rebuilds the same
    // waveform and symbol outputs: tx_symbol + combine_symbols ==
    // tx_discontinuous; rx_segment + rx_block_freq + rx_symbol_simplified /
    // rx_symbol_direct == rx_discontinuous
    const auto p = fw::derive_fc_params(N, L, 0.5);
    std::vector<fw::FilteredSymbol> syms;
    for (int n = 0; n < 3; ++n) {
        const auto sp = fw::cp_truncate(cps.per_symbol_high_rate[n], p.I);
        fw::cvec x(L);  // ofdm_modulate (ofdm.cpp:97-106): IDFT_L * sqrt(L) / L
        for (int t = 0; t < L; ++t)
            for (int b = 0; b < L; ++b) x[t] += g.symbols[n][b] * std::polar(1.0, 2 * M_PI * b * t / L) / std::sqrt(double(L));
        fw::cvec sym(x.end() - sp.l_cp, x.end());  // cp_insert
        sym.insert(sym.end(), x.begin(), x.end());
        syms.push_back(fw::tx_symbol(sym, cfg, p, cps, n));
    }
    const fw::Waveform w2 = fw::combine_symbols(syms, cps, p, num.fs_hz());
    double tx_err = 0, tx_ref = 0;
    for (size_t t = 0; t < w.samples.size(); ++t) {
        tx_err += std::norm(w2.samples[t] - w.samples[t]);
        tx_ref += std::norm(w.samples[t]);
    }
    double rx_err = 0, rx_ref = 0;
    for (int n = 0; n < 3; ++n) {
        const auto blk = fw::rx_segment(w, cps, p, n);
        const auto th = fw::symbol_phase(n, c, cps, N);
        const auto g0 = fw::rx_block_freq(blk.y0, cfg, p, fw::block_phase(0, c, p.L_S, L) * th);
        const auto g1 = fw::rx_block_freq(blk.y1, cfg, p, fw::block_phase(1, c, p.L_S, L) * th);
        const auto xs = fw::rx_symbol_simplified(g0, g1, cfg, p);
        const auto xd = fw::rx_symbol_direct(blk.y0, blk.y1, cfg, p, cps, n);
        for (int b = 0; b < L; ++b) {
            rx_err += std::norm(xs[b] - f[n][b]) + std::norm(xd[b] - d[n][b]);
            rx_ref += std::norm(f[n][b]) + std::norm(d[n][b]);
        }
    }
    const double tx_rel = std::sqrt(tx_err / tx_ref), rx_rel = std::sqrt(rx_err / rx_ref);
    std::printf("per-symbol API: tx rel %.2e, rx rel %.2e\n", tx_rel, rx_rel);
    if (!(tx_rel < 1e-5 && rx_rel < 1e-5)) return 2;
    bool threw = false;
    try {
        fw::derive_fc_params(1024, 96, 0.5);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    std::printf("Q=%zu useful0=%lld evm_db=%.2f fused_vs_direct=%.3e invalid_argument=%d\n", w.samples.size(),
                (long long)w.useful0, 10 * std::log10(den / num_e), diff, threw ? 1 : 0);
    return (w.samples.size() == 2632 + 1096 && w.useful0 == 256 && 10 * std::log10(den / num_e) > 25.0 &&
            diff < 1e-5 && threw)
               ? 0
               : 1;
}
