/*
 * TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * extern "C" driver around the UNMODIFIED reference library compiled from
 * /root/reference/proj/src (see oracle/Makefile; outputs go to oracle/_ref/).
 * It lets the Python tests and bench.py's reference arm call the reference's
 * own hot path:
 *   tx_discontinuous  proj/include/fcwave/fc_sync.hpp:52-54 (fc_sync.cpp:114-143)
 *   rx_discontinuous  proj/include/fcwave/fc_sync.hpp:78-80 (fc_sync.cpp:245-264)
 *   tx_symbol / rx_symbol_direct / rx_block_freq / rx_symbol_simplified
 *                     proj/include/fcwave/fc_sync.hpp:38-75
 * Complex data crosses this boundary as interleaved doubles.  Reference
 * exceptions map to status codes: invalid_argument -> 1, out_of_range -> 2,
 * anything else -> 3; the message is kept in fcwref_last_error().
 */
#include "fcwave/channel.hpp"
#include "fcwave/fc_core.hpp"
#include "fcwave/metrics.hpp"
#include "fcwave/fc_sync.hpp"
#include "fcwave/numerology.hpp"
#include "fcwave/ofdm.hpp"

#include <atomic>
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using fcwave::cd;
using fcwave::cvec;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

cvec to_cvec(const double* p, std::size_t n) {
    cvec v(n);
    for (std::size_t i = 0; i < n; ++i) v[i] = cd{p[2 * i], p[2 * i + 1]};
    return v;
}

void from_cvec(const cvec& v, double* p) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        p[2 * i] = v[i].real();
        p[2 * i + 1] = v[i].imag();
    }
}

fcwave::CpSchedule sched(const int* cp, int B) {
    fcwave::CpSchedule s;
    s.per_symbol_high_rate.assign(cp, cp + B);
    return s;
}

fcwave::SubbandConfig cfg_of(int L, int c, const double* window) {
    fcwave::SubbandConfig cfg;
    cfg.L = L;
    cfg.l_ofdm = L;
    cfg.c = c;
    cfg.window.assign(window, window + L);
    return cfg;
}

}  // namespace

extern "C" {

const char* fcwref_last_error(void) { return g_err.c_str(); }

/* grids: for each subband m, B columns of L_m complex values (full DFT-bin
 * columns, QamGrid::symbols layout ofdm.hpp:27-33), concatenated over m. */
int fcwref_tx(int N, double overlap, const int* cp, int B, int M, const int* Ls, const int* cs,
              const double* windows, const double* grids, double* wave_out, long long cap,
              long long* Q, long long* useful0) {
    return guarded([&] {
        std::vector<fcwave::QamGrid> gs(static_cast<std::size_t>(M));
        std::vector<fcwave::SubbandConfig> cfgs(static_cast<std::size_t>(M));
        std::size_t woff = 0, goff = 0;
        for (int m = 0; m < M; ++m) {
            const int L = Ls[m];
            cfgs[m] = cfg_of(L, cs[m], windows + woff);
            woff += static_cast<std::size_t>(L);
            gs[m].l_ofdm = L;
            for (int n = 0; n < B; ++n) {
                gs[m].symbols.push_back(to_cvec(grids + 2 * goff, static_cast<std::size_t>(L)));
                goff += static_cast<std::size_t>(L);
            }
        }
        const fcwave::Waveform w = fcwave::tx_discontinuous(gs, cfgs, sched(cp, B), N, overlap, 1.0);
        *Q = static_cast<long long>(w.samples.size());
        *useful0 = static_cast<long long>(w.useful0);
        if (wave_out) {
            if (static_cast<long long>(w.samples.size()) > cap)
                throw std::invalid_argument("output capacity too small");
            from_cvec(w.samples, wave_out);
        }
    });
}

int fcwref_rx(int N, double overlap, const int* cp, int B, int L, int c, const double* window,
              const double* wave, long long len, long long useful0, int simplified, double* out) {
    return guarded([&] {
        fcwave::Waveform w;
        w.samples = to_cvec(wave, static_cast<std::size_t>(len));
        w.useful0 = useful0;
        w.fs_hz = 1.0;
        const auto cols = fcwave::rx_discontinuous(w, cfg_of(L, c, window), sched(cp, B), N, overlap,
                                                   simplified != 0);
        for (std::size_t n = 0; n < cols.size(); ++n) from_cvec(cols[n], out + 2 * n * static_cast<std::size_t>(L));
    });
}

int fcwref_tx_symbol(const double* sym, int sym_len, int L, int c, const double* window, int N,
                     double overlap, const int* cp, int B, int n, double* out3n2) {
    return guarded([&] {
        const fcwave::FcParams p = fcwave::derive_fc_params(N, L, overlap);
        const fcwave::FilteredSymbol fs = fcwave::tx_symbol(
            to_cvec(sym, static_cast<std::size_t>(sym_len)), cfg_of(L, c, window), p, sched(cp, B), n);
        from_cvec(fs.samples, out3n2);
    });
}

int fcwref_rx_symbol_direct(const double* y0, const double* y1, int L, int c, const double* window,
                            int N, double overlap, const int* cp, int B, int n, double* out) {
    return guarded([&] {
        const fcwave::FcParams p = fcwave::derive_fc_params(N, L, overlap);
        from_cvec(fcwave::rx_symbol_direct(to_cvec(y0, N), to_cvec(y1, N), cfg_of(L, c, window), p,
                                           sched(cp, B), n),
                  out);
    });
}

int fcwref_rx_block_freq(const double* y, int L, int c, const double* window, int N, double overlap,
                         double ph_re, double ph_im, double* out) {
    return guarded([&] {
        const fcwave::FcParams p = fcwave::derive_fc_params(N, L, overlap);
        from_cvec(fcwave::rx_block_freq(to_cvec(y, N), cfg_of(L, c, window), p, cd{ph_re, ph_im}), out);
    });
}

int fcwref_rx_symbol_simplified(const double* g0, const double* g1, int L, int c, const double* window,
                                int N, double overlap, double* out) {
    return guarded([&] {
        const fcwave::FcParams p = fcwave::derive_fc_params(N, L, overlap);
        from_cvec(fcwave::rx_symbol_simplified(to_cvec(g0, L), to_cvec(g1, L), cfg_of(L, c, window), p),
                  out);
    });
}

/*
 * CPU baseline: the reference's own path over `units` independent
 * (stream, frame) units on `threads` host threads, one unit per task pulled
 * from an atomic counter (the reference's drop pool, scenario.cpp:499-514).
 * Per unit: one tx_discontinuous over all subbands, then rx_discontinuous
 * once per subband (how the reference's callers use it, scenario.cpp:242).
 * grids_packed: [units][B][sum n_active] complex64 active-bin values; they are
 * expanded into full QamGrid columns BEFORE the clock starts.
 * Returns elapsed wall seconds of the TX+RX region (negative on error).
 */
double fcwref_bench_txrx(int N, double overlap, const int* cp, int B, int M, const int* Ls,
                         const int* cs, const double* windows, const int* n_active,
                         const int* active_bins, const float* grids_packed, int units, int threads,
                         int simplified, double* checksum) {
    double elapsed = -1.0;
    const int rc = guarded([&] {
        const fcwave::CpSchedule cps = sched(cp, B);
        std::vector<fcwave::SubbandConfig> cfgs(static_cast<std::size_t>(M));
        std::vector<std::vector<int>> bins(static_cast<std::size_t>(M));
        std::size_t woff = 0, boff = 0;
        int A = 0;
        for (int m = 0; m < M; ++m) {
            cfgs[m] = cfg_of(Ls[m], cs[m], windows + woff);
            woff += static_cast<std::size_t>(Ls[m]);
            bins[m].assign(active_bins + boff, active_bins + boff + n_active[m]);
            boff += static_cast<std::size_t>(n_active[m]);
            A += n_active[m];
        }
        std::vector<std::vector<fcwave::QamGrid>> inputs(static_cast<std::size_t>(units));
        for (int u = 0; u < units; ++u) {
            auto& gs = inputs[u];
            gs.resize(static_cast<std::size_t>(M));
            int aoff = 0;
            for (int m = 0; m < M; ++m) {
                gs[m].l_ofdm = Ls[m];
                gs[m].active_map = bins[m];
                for (int n = 0; n < B; ++n) {
                    cvec col(static_cast<std::size_t>(Ls[m]), cd{0, 0});
                    const float* row = grids_packed + 2 * (static_cast<std::size_t>(u) * B + n) * A;
                    for (int a = 0; a < n_active[m]; ++a)
                        col[bins[m][a]] = cd{row[2 * (aoff + a)], row[2 * (aoff + a) + 1]};
                    gs[m].symbols.push_back(std::move(col));
                }
                aoff += n_active[m];
            }
        }
        std::vector<double> sums(static_cast<std::size_t>(units), 0.0);
        std::atomic<int> next{0};
        std::atomic<int> failed{0};
        auto worker = [&] {
            for (;;) {
                const int u = next.fetch_add(1);
                if (u >= units) break;
                try {
                    const fcwave::Waveform w =
                        fcwave::tx_discontinuous(inputs[u], cfgs, cps, N, overlap, 1.0);
                    double s = 0.0;
                    for (int m = 0; m < M; ++m) {
                        const auto cols = fcwave::rx_discontinuous(w, cfgs[m], cps, N, overlap, simplified != 0);
                        for (const auto& col : cols)
                            for (const cd& v : col) s += v.real();
                    }
                    sums[u] = s;
                } catch (...) {
                    failed.store(1);
                }
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        const int nt = threads < 1 ? 1 : threads;
        for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
        for (auto& th : pool) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        if (failed.load()) throw std::runtime_error("reference worker threw");
        elapsed = std::chrono::duration<double>(t1 - t0).count();
        double total = 0.0;
        for (double s : sums) total += s;
        if (checksum) *checksum = total;
    });
    return rc == 0 ? elapsed : -1.0;
}


/* ---- link step (f1/f3): the reference's own demap / metrics / channel ---- */
int fcwref_qam_demap(int bits_per_symbol, const double* y, int n, unsigned* out) {
    return guarded([&] {
        const fcwave::Modulation m = bits_per_symbol == 2   ? fcwave::Modulation::QPSK
                                     : bits_per_symbol == 4 ? fcwave::Modulation::QAM16
                                                            : fcwave::Modulation::QAM64;
        for (int i = 0; i < n; ++i) out[i] = fcwave::qam_demap(m, cd{y[2 * i], y[2 * i + 1]});
    });
}

int fcwref_qam_map(int bits_per_symbol, const unsigned* sym, int n, double* out) {
    return guarded([&] {
        const fcwave::Modulation m = bits_per_symbol == 2   ? fcwave::Modulation::QPSK
                                     : bits_per_symbol == 4 ? fcwave::Modulation::QAM16
                                                            : fcwave::Modulation::QAM64;
        for (int i = 0; i < n; ++i) {
            const cd v = fcwave::qam_map(m, sym[i]);
            out[2 * i] = v.real();
            out[2 * i + 1] = v.imag();
        }
    });
}

int fcwref_ber(const unsigned char* a, const unsigned char* b, long long n, double* out) {
    return guarded([&] {
        *out = fcwave::ber(std::vector<std::uint8_t>(a, a + n), std::vector<std::uint8_t>(b, b + n));
    });
}

int fcwref_evm_db(const double* ref, const double* rx, long long n, double* out) {
    return guarded([&] { *out = fcwave::evm_db(to_cvec(ref, (std::size_t)n), to_cvec(rx, (std::size_t)n)); });
}

int fcwref_awgn_with_variance(double* wave, long long n, double sigma2, unsigned long long seed) {
    return guarded([&] {
        fcwave::Waveform w;
        w.samples = to_cvec(wave, (std::size_t)n);
        fcwave::awgn_with_variance(w, sigma2, seed);
        from_cvec(w.samples, wave);
    });
}

int fcwref_measure_power(const double* wave, long long n, long long begin, long long end, double* out) {
    return guarded([&] {
        fcwave::Waveform w;
        w.samples = to_cvec(wave, (std::size_t)n);
        *out = fcwave::measure_power(w, begin, end);
    });
}

int fcwref_awgn_noise_variance(const double* wave, long long n, double snr_db, int n_fft, int n_active,
                               double* out) {
    return guarded([&] {
        fcwave::Waveform w;
        w.samples = to_cvec(wave, (std::size_t)n);
        *out = fcwave::awgn_noise_variance(w, snr_db, n_fft, n_active);
    });
}

/* ---- continuous FC (f2): fc_core.hpp:64-77 ---- */
int fcwref_tx_continuous(int N, double overlap, int M, const int* Ls, const int* cs, const double* windows,
                         const double* streams, const long long* lens, int l_cp0, double* wave_out, long long cap,
                         long long* out_len, long long* useful0) {
    return guarded([&] {
        std::vector<fcwave::CpOfdmSignal> sigs;
        std::vector<fcwave::SubbandConfig> cfgs;
        size_t soff = 0, woff = 0;
        for (int m = 0; m < M; ++m) {
            fcwave::CpOfdmSignal sg;
            sg.samples = to_cvec(streams + 2 * soff, (std::size_t)lens[m]);
            sg.cp_lengths = {m == 0 ? l_cp0 : 0};
            sg.l_ofdm = Ls[m];
            sigs.push_back(std::move(sg));
            cfgs.push_back(cfg_of(Ls[m], cs[m], windows + woff));
            soff += (size_t)lens[m];
            woff += (size_t)Ls[m];
        }
        const fcwave::Waveform w = fcwave::tx_continuous(sigs, cfgs, N, overlap, 1.0);
        if ((long long)w.samples.size() > cap) throw std::out_of_range("capacity");
        from_cvec(w.samples, wave_out);
        *out_len = (long long)w.samples.size();
        *useful0 = (long long)w.useful0;
    });
}

int fcwref_rx_continuous(const double* wave, long long len, int N, double overlap, int L, int c,
                         const double* window, double* out, long long cap, long long* n_out) {
    return guarded([&] {
        fcwave::Waveform w;
        w.samples = to_cvec(wave, (std::size_t)len);
        const fcwave::FcParams p = fcwave::derive_fc_params(N, L, overlap);
        const cvec z = fcwave::rx_continuous(w, cfg_of(L, c, window), p);
        if ((long long)z.size() > cap) throw std::out_of_range("capacity");
        from_cvec(z, out);
        *n_out = (long long)z.size();
    });
}

/* ---- Welch PSD (f4): metrics.hpp:75 ---- */
int fcwref_psd(const double* x, long long len, int seg_len, double overlap_frac, double* out) {
    return guarded([&] {
        const std::vector<double> p = fcwave::psd(to_cvec(x, (std::size_t)len), seg_len, overlap_frac);
        std::copy(p.begin(), p.end(), out);
    });
}

/* ---- TDL channel (f3): channel.hpp:34-60 ---- */
int fcwref_draw_tdl(const double* delay_ns, const double* power_lin, int n_taps, double fs_hz,
                    unsigned long long seed, int* delays, double* gains) {
    return guarded([&] {
        fcwave::TdlProfile p;
        for (int k = 0; k < n_taps; ++k) p.taps.push_back({delay_ns[k], power_lin[k]});
        const fcwave::ChannelRealization ch = fcwave::draw_tdl(p, fs_hz, seed);
        for (int k = 0; k < n_taps; ++k) delays[k] = ch.delays_samples[k];
        from_cvec(ch.gains, gains);
    });
}

int fcwref_apply_channel(double* wave, long long len, const int* delays, const double* gains, int n_taps) {
    return guarded([&] {
        fcwave::Waveform w;
        w.samples = to_cvec(wave, (std::size_t)len);
        fcwave::ChannelRealization ch;
        ch.delays_samples.assign(delays, delays + n_taps);
        ch.gains = to_cvec(gains, (std::size_t)n_taps);
        fcwave::apply_channel(w, ch);
        from_cvec(w.samples, wave);
    });
}

}  // extern "C"
