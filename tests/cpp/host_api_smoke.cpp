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
