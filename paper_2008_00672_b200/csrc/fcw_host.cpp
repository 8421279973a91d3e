// C++ host library over the C ABI (see fcwave_b200.hpp).  The reference-shaped
// functions convert complex<double> <-> complex64 at the boundary and run the
// GPU pipeline through the host-buffer entry points.
#include "fcwave_b200.hpp"

#include <stdexcept>
#include <string>

namespace fcwave_b200 {

void check(int rc) {
    if (rc == FCW_OK) return;
    const std::string msg = fcw_last_error();
    if (rc == FCW_EINVAL) throw std::invalid_argument(msg);
    if (rc == FCW_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

Numerology make_numerology(int scs_khz, int n_fft) {
    // numerology.cpp:17-27
    auto pow2 = [](int v) { return v >= 1 && (v & (v - 1)) == 0; };
    if (!pow2(n_fft) || n_fft < 16) throw std::invalid_argument("n_fft must be a power of two >= 16");
    if (scs_khz <= 0 || scs_khz % 15 != 0 || !pow2(scs_khz / 15))
        throw std::invalid_argument("scs_khz must be 15*2^k");
    Numerology num;
    num.scs_khz = scs_khz;
    num.n_fft = n_fft;
    num.symbols_per_half_subframe = 7;
    return num;
}

CpSchedule cp_schedule(const Numerology& num, int n_symbols) {
    CpSchedule s;
    s.per_symbol_high_rate.resize(n_symbols > 0 ? n_symbols : 1);
    check(fcw_cp_schedule(num.scs_khz, num.n_fft, n_symbols, s.per_symbol_high_rate.data()));
    return s;
}

CpSchedule nr_cp_schedule(const Numerology& num, int n_symbols) {
    CpSchedule s;
    s.per_symbol_high_rate.resize(n_symbols > 0 ? n_symbols : 1);
    check(fcw_nr_cp_schedule(num.scs_khz, num.n_fft, n_symbols, s.per_symbol_high_rate.data()));
    return s;
}

FcParams derive_fc_params(int N, int L, double overlap) {
    FcParams p{};
    check(fcw_derive_fc_params(N, L, overlap, &p));
    return p;
}

double first_block_overlap(const FcParams& params, int l_cp) {
    double v = 0.0;
    check(fcw_first_block_overlap(&params, l_cp, &v));
    return v;
}

std::vector<double> design_window(int L, int n_pass, int n_tb) {
    std::vector<double> w(L > 0 ? L : 0);
    check(fcw_design_window(L, n_pass, n_tb, w.data()));
    return w;
}

std::vector<int> centered_active_map(int l_ofdm, int n_active, bool skip_dc) {
    std::vector<int> b(n_active > 0 ? n_active : 0);
    check(fcw_centered_active_map(l_ofdm, n_active, skip_dc ? 1 : 0, b.data()));
    return b;
}

CpSplit cp_truncate(int n_cp_high, int I) {
    CpSplit s;
    check(fcw_cp_truncate(n_cp_high, I, &s.l_cp, &s.extrap));
    return s;
}

std::int64_t symbol_sigma(int n, const CpSchedule& cps, int N) {
    return fcw_symbol_sigma(n, cps.per_symbol_high_rate.data(), N);
}

std::int64_t combined_length(int n_symbols, const CpSchedule& cps, const FcParams& p) {
    return fcw_combined_length(n_symbols, cps.per_symbol_high_rate.data(), &p);
}

namespace {

struct PlanHolder {
    fcw_plan* p = nullptr;
    ~PlanHolder() { fcw_plan_destroy(p); }
};

std::vector<fcw_subband> descs(const std::vector<SubbandConfig>& cfgs, const std::vector<std::vector<int>>& maps) {
    std::vector<fcw_subband> d(cfgs.size());
    for (size_t m = 0; m < cfgs.size(); ++m) {
        if (static_cast<int>(cfgs[m].window.size()) != cfgs[m].L)
            throw std::invalid_argument("window length must be L");
        d[m].L = cfgs[m].L;
        d[m].l_ofdm = cfgs[m].l_ofdm;
        d[m].c = cfgs[m].c;
        d[m].n_active = static_cast<int>(maps[m].size());
        d[m].n_tb = cfgs[m].n_tb;
        d[m].active_bins = maps[m].data();
        d[m].window = cfgs[m].window.data();
    }
    return d;
}

std::vector<std::vector<int>> all_bins(const std::vector<SubbandConfig>& cfgs) {
    std::vector<std::vector<int>> maps(cfgs.size());
    for (size_t m = 0; m < cfgs.size(); ++m)
        for (int b = 0; b < cfgs[m].L; ++b) maps[m].push_back(b);
    return maps;
}

}  // namespace

Waveform tx_discontinuous(const std::vector<QamGrid>& grids, const std::vector<SubbandConfig>& cfgs,
                          const CpSchedule& cps, int N, double overlap, double fs_hz) {
    if (grids.size() != cfgs.size() || grids.empty()) throw std::invalid_argument("one config per grid required");
    const int B = static_cast<int>(cps.per_symbol_high_rate.size());
    for (const auto& g : grids)
        if (g.n_symbols() != B) throw std::invalid_argument("grid symbol count must match CP schedule");
    const auto maps = all_bins(cfgs);
    const auto d = descs(cfgs, maps);
    PlanHolder h;
    check(fcw_plan_create(&h.p, N, overlap, cps.per_symbol_high_rate.data(), B, d.data(),
                          static_cast<int>(d.size()), 0));
    fcw_plan_info info{};
    check(fcw_plan_get_info(h.p, &info));
    std::vector<float> in(2 * static_cast<size_t>(B) * info.row_full);
    for (int n = 0; n < B; ++n) {
        size_t off = 2 * static_cast<size_t>(n) * info.row_full;
        for (size_t m = 0; m < grids.size(); ++m) {
            const cvec& col = grids[m].symbols[n];
            if (static_cast<int>(col.size()) != cfgs[m].L) throw std::invalid_argument("grid column size mismatch");
            for (const cd& v : col) {
                in[off++] = static_cast<float>(v.real());
                in[off++] = static_cast<float>(v.imag());
            }
        }
    }
    std::vector<float> out(2 * static_cast<size_t>(info.Q));
    check(fcw_tx_host(h.p, in.data(), out.data(), 1, FCW_GRID_FULL));
    Waveform w;
    w.fs_hz = fs_hz;
    w.useful0 = info.useful0;
    w.samples.resize(info.Q);
    for (int64_t t = 0; t < info.Q; ++t) w.samples[t] = cd(out[2 * t], out[2 * t + 1]);
    return w;
}

std::vector<std::vector<cvec>> rx_discontinuous_all(const Waveform& w, const std::vector<SubbandConfig>& cfgs,
                                                    const CpSchedule& cps, int N, double overlap,
                                                    bool simplified) {
    const int B = static_cast<int>(cps.per_symbol_high_rate.size());
    if (B < 1) throw std::invalid_argument("no symbols");
    if (simplified)
        for (const auto& c : cfgs)
            if (derive_fc_params(N, c.L, overlap).L_S * 2 != c.L)
                throw std::invalid_argument("fused RX path requires 50 % overlap");
    const auto maps = all_bins(cfgs);
    const auto d = descs(cfgs, maps);
    PlanHolder h;
    check(fcw_plan_create(&h.p, N, overlap, cps.per_symbol_high_rate.data(), B, d.data(),
                          static_cast<int>(d.size()), 0));
    fcw_plan_info info{};
    check(fcw_plan_get_info(h.p, &info));
    const int64_t len = static_cast<int64_t>(w.samples.size());
    std::vector<float> in(2 * static_cast<size_t>(len));
    for (int64_t t = 0; t < len; ++t) {
        in[2 * t] = static_cast<float>(w.samples[t].real());
        in[2 * t + 1] = static_cast<float>(w.samples[t].imag());
    }
    std::vector<float> out(2 * static_cast<size_t>(B) * info.row_full);
    check(fcw_rx_host(h.p, in.data(), len, w.useful0, out.data(), 1,
                      FCW_GRID_FULL | (simplified ? FCW_RX_FUSED : 0u)));
    std::vector<std::vector<cvec>> res(cfgs.size(), std::vector<cvec>(B));
    for (int n = 0; n < B; ++n) {
        size_t off = 2 * static_cast<size_t>(n) * info.row_full;
        for (size_t m = 0; m < cfgs.size(); ++m) {
            cvec& col = res[m][n];
            col.resize(cfgs[m].L);
            for (int b = 0; b < cfgs[m].L; ++b, off += 2) col[b] = cd(out[off], out[off + 1]);
        }
    }
    return res;
}

std::vector<cvec> rx_discontinuous(const Waveform& w, const SubbandConfig& cfg, const CpSchedule& cps, int N,
                                   double overlap, bool simplified) {
    return rx_discontinuous_all(w, {cfg}, cps, N, overlap, simplified)[0];
}

Engine::Engine(int N, double overlap, const CpSchedule& cps, const std::vector<SubbandConfig>& cfgs,
               const std::vector<std::vector<int>>& active_maps) {
    if (cfgs.size() != active_maps.size()) throw std::invalid_argument("one active map per subband required");
    const auto d = descs(cfgs, active_maps);
    check(fcw_plan_create(&plan_, N, overlap, cps.per_symbol_high_rate.data(),
                          static_cast<int>(cps.per_symbol_high_rate.size()), d.data(), static_cast<int>(d.size()),
                          0));
}

Engine::~Engine() { fcw_plan_destroy(plan_); }

fcw_plan_info Engine::info() const {
    fcw_plan_info i{};
    check(fcw_plan_get_info(plan_, &i));
    return i;
}

void Engine::tx(const void* grid_dev, void* wave_dev, int S, unsigned flags, void* stream) const {
    check(fcw_tx(plan_, grid_dev, 0, wave_dev, 0, S, flags, stream));
}

void Engine::rx(const void* wave_dev, std::int64_t wave_len, std::int64_t useful0, void* grid_dev, int S,
                unsigned flags, void* stream) const {
    check(fcw_rx(plan_, wave_dev, 0, wave_len, useful0, grid_dev, 0, S, flags, stream));
}

}  // namespace fcwave_b200
