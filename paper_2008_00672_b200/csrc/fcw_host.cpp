// C++ host library over the C ABI (see fcwave_b200.hpp).  The reference-shaped
// functions convert complex<double> <-> complex64 at the boundary and run the
// GPU pipeline through the host-buffer entry points.
#include "fcwave_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
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

// ------------------------------------------------ per-symbol API (device)
namespace {

struct DevBuf {  // complex64 device buffer of n entries
    void* p = nullptr;
    explicit DevBuf(size_t n) {
        if (cudaMalloc(&p, 8 * (n ? n : 1)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    }
    ~DevBuf() { cudaFree(p); }
    void put(const cvec& v) const {
        std::vector<float> f(2 * v.size());
        for (size_t i = 0; i < v.size(); ++i) {
            f[2 * i] = static_cast<float>(v[i].real());
            f[2 * i + 1] = static_cast<float>(v[i].imag());
        }
        if (cudaMemcpy(p, f.data(), 4 * f.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            throw std::runtime_error("cudaMemcpy failed");
    }
    cvec get(size_t n) const {
        std::vector<float> f(2 * n);
        if (cudaMemcpy(f.data(), p, 4 * f.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
            throw std::runtime_error("cudaMemcpy failed");
        cvec v(n);
        for (size_t i = 0; i < n; ++i) v[i] = cd(f[2 * i], f[2 * i + 1]);
        return v;
    }
};

// one-subband plan over `cps` (a one-symbol schedule when the call has none)
struct OnePlan {
    PlanHolder h;
    OnePlan(const SubbandConfig& cfg, const FcParams& p, const std::vector<int>& cp) {
        if (cfg.L != p.L) throw std::invalid_argument("subband L does not match FC params");
        const std::vector<SubbandConfig> cfgs{cfg};  // named: the descriptors point into it
        const std::vector<std::vector<int>> maps = all_bins(cfgs);
        const auto d = descs(cfgs, maps);
        check(fcw_plan_create(&h.p, p.N, p.overlap, cp.data(), static_cast<int>(cp.size()), d.data(), 1, 0));
    }
};

std::vector<int> sched_or_zero(const CpSchedule& cps) {
    return cps.per_symbol_high_rate.empty() ? std::vector<int>{0} : cps.per_symbol_high_rate;
}

}  // namespace

cd symbol_phase(int n, int c, const CpSchedule& cps, int N) {
    double re = 0, im = 0;
    check(fcw_symbol_phase(n, c, cps.per_symbol_high_rate.data(), static_cast<int>(cps.per_symbol_high_rate.size()),
                           N, &re, &im));
    return cd(re, im);
}

cd block_phase(std::int64_t r, int c, int L_S, int L) {
    double re = 0, im = 0;
    check(fcw_block_phase(r, c, L_S, L, &re, &im));
    return cd(re, im);
}

FilteredSymbol tx_symbol(const cvec& sym, const SubbandConfig& cfg, const FcParams& p, const CpSchedule& cps, int n) {
    const int l_cp = static_cast<int>(sym.size()) - p.L;  // fc_sync.cpp:65
    if (l_cp < 0) throw std::invalid_argument("symbol length must be L + L_CP");
    OnePlan pl(cfg, p, sched_or_zero(cps));
    DevBuf in(sym.size()), out(3 * static_cast<size_t>(p.N) / 2);
    in.put(sym);
    check(fcw_tx_symbol(pl.h.p, 0, n, in.p, 0, l_cp, out.p, 0, 1, nullptr));
    FilteredSymbol f;
    f.n = n;
    f.samples = out.get(3 * static_cast<size_t>(p.N) / 2);
    return f;
}

Waveform combine_symbols(const std::vector<FilteredSymbol>& syms, const CpSchedule& cps, const FcParams& p,
                         double fs_hz) {
    if (syms.empty()) throw std::invalid_argument("no symbols");
    const int B = static_cast<int>(syms.size());
    const size_t len = 3 * static_cast<size_t>(p.N) / 2;
    // the device kernel takes symbol n at slot n: the reference's usual call
    // (one FilteredSymbol per schedule entry, in order)
    cvec all(static_cast<size_t>(B) * len);
    std::vector<char> seen(static_cast<size_t>(B), 0);
    for (const auto& s : syms) {
        if (s.samples.size() != len) throw std::invalid_argument("filtered symbol length must be 3N/2");
        if (s.n < 0 || s.n >= B || seen[static_cast<size_t>(s.n)])
            throw std::invalid_argument("combine_symbols: symbols must be n = 0..B-1, each once");
        seen[static_cast<size_t>(s.n)] = 1;
        std::copy(s.samples.begin(), s.samples.end(), all.begin() + static_cast<std::ptrdiff_t>(s.n * len));
    }
    if (static_cast<int>(cps.per_symbol_high_rate.size()) < B) throw std::out_of_range("CP schedule too short");
    CpSchedule head;
    head.per_symbol_high_rate.assign(cps.per_symbol_high_rate.begin(), cps.per_symbol_high_rate.begin() + B);
    SubbandConfig cfg;  // the plan only needs N, the schedule and a subband of size p.L
    cfg.L = cfg.l_ofdm = p.L;
    cfg.window.assign(static_cast<size_t>(p.L), 1.0);
    OnePlan pl(cfg, p, head.per_symbol_high_rate);
    fcw_plan_info info{};
    check(fcw_plan_get_info(pl.h.p, &info));
    DevBuf in(all.size()), out(static_cast<size_t>(info.Q));
    in.put(all);
    check(fcw_combine_symbols(pl.h.p, in.p, 0, out.p, 0, 1, nullptr));
    Waveform w;
    w.fs_hz = fs_hz;
    w.useful0 = p.N_L;
    w.samples = out.get(static_cast<size_t>(info.Q));
    return w;
}

SymbolBlocks rx_segment(const Waveform& w, const CpSchedule& cps, const FcParams& p, int n) {
    // index arithmetic and a copy (no arithmetic on samples): host side
    if (n < 0 || n >= static_cast<int>(cps.per_symbol_high_rate.size()))
        throw std::out_of_range("symbol index outside CP schedule");
    const std::int64_t start = w.useful0 - p.N_L + symbol_sigma(n, cps, p.N);
    if (start < 0 || start + 3 * p.N / 2 > static_cast<std::int64_t>(w.samples.size()))
        throw std::invalid_argument("waveform too short for symbol window");
    SymbolBlocks b;
    b.y0.assign(w.samples.begin() + start, w.samples.begin() + start + p.N);
    b.y1.assign(w.samples.begin() + start + p.N / 2, w.samples.begin() + start + 3 * p.N / 2);
    return b;
}

cvec rx_symbol_direct(const cvec& y0, const cvec& y1, const SubbandConfig& cfg, const FcParams& p,
                      const CpSchedule& cps, int n) {
    if (static_cast<int>(y0.size()) != p.N || static_cast<int>(y1.size()) != p.N)
        throw std::invalid_argument("block length must be N");
    OnePlan pl(cfg, p, sched_or_zero(cps));
    DevBuf a(y0.size()), b(y1.size()), out(static_cast<size_t>(p.L));
    a.put(y0);
    b.put(y1);
    check(fcw_rx_symbol_direct(pl.h.p, 0, n, a.p, b.p, 0, out.p, 0, 1, nullptr));
    return out.get(static_cast<size_t>(p.L));
}

cvec rx_symbol_simplified(const cvec& g0, const cvec& g1, const SubbandConfig& cfg, const FcParams& p) {
    if (static_cast<int>(g0.size()) != p.L || static_cast<int>(g1.size()) != p.L)
        throw std::invalid_argument("frequency blocks must have length L");
    SubbandConfig c2 = cfg;  // (the reference ignores cfg here, fc_sync.cpp:201)
    if (static_cast<int>(c2.window.size()) != p.L) c2.window.assign(static_cast<size_t>(p.L), 1.0);
    c2.L = p.L;
    if (c2.l_ofdm == 0) c2.l_ofdm = p.L;
    OnePlan pl(c2, p, {0});
    DevBuf a(g0.size()), b(g1.size()), out(static_cast<size_t>(p.L));
    a.put(g0);
    b.put(g1);
    check(fcw_rx_symbol_simplified(pl.h.p, 0, a.p, b.p, 0, out.p, 0, 1, nullptr));
    return out.get(static_cast<size_t>(p.L));
}

cvec rx_block_freq(const cvec& y, const SubbandConfig& cfg, const FcParams& p, cd phase) {
    if (static_cast<int>(y.size()) != p.N) throw std::invalid_argument("block length must be N");
    OnePlan pl(cfg, p, {0});
    DevBuf in(y.size()), out(static_cast<size_t>(p.L));
    in.put(y);
    check(fcw_rx_block_freq(pl.h.p, 0, in.p, 0, phase.real(), phase.imag(), out.p, 0, 1, nullptr));
    return out.get(static_cast<size_t>(p.L));
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
