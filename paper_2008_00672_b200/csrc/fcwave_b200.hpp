// fcwave-b200 C++ host library: the reference's data model and entry points
// (proj/include/fcwave/{types,numerology,fc_core,ofdm,fc_sync}.hpp) on top of
// the C ABI (include/fcwave_b200.h).  A reference user switches by replacing
// `fcwave::` with `fcwave_b200::`; the heavy work runs on the GPU.
//
// Errors are the reference's exception classes: FCW_EINVAL ->
// std::invalid_argument, FCW_ERANGE -> std::out_of_range, everything else ->
// std::runtime_error.
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <vector>

#include "fcwave_b200.h"

namespace fcwave_b200 {

using cd = std::complex<double>;
using cvec = std::vector<cd>;

struct Waveform {  // types.hpp:22-26
    cvec samples;
    double fs_hz = 0.0;
    std::int64_t useful0 = 0;
};

struct Numerology {  // numerology.hpp:14-20
    int scs_khz = 15;
    int n_fft = 1024;
    int symbols_per_half_subframe = 7;
    double fs_hz() const { return static_cast<double>(scs_khz) * 1000.0 * n_fft; }
};

struct CpSchedule {  // numerology.hpp:23-31
    std::vector<int> per_symbol_high_rate;
    int total() const {
        int s = 0;
        for (int v : per_symbol_high_rate) s += v;
        return s;
    }
};

using FcParams = fcw_fc_params;  // numerology.hpp:34-41 (same fields)

struct SubbandConfig {  // fc_core.hpp:20-27
    int L = 0;
    int l_ofdm = 0;
    int c = 0;
    int n_active = 0;
    int n_tb = 0;
    std::vector<double> window;
};

struct QamGrid {  // ofdm.hpp:27-33
    int l_ofdm = 0;
    std::vector<int> active_map;
    std::vector<cvec> symbols;
    int n_symbols() const { return static_cast<int>(symbols.size()); }
};

struct CpSplit {  // fc_sync.hpp:13-17
    int l_cp = 0;
    int extrap = 0;
};

Numerology make_numerology(int scs_khz, int n_fft);
CpSchedule cp_schedule(const Numerology& num, int n_symbols);
CpSchedule nr_cp_schedule(const Numerology& num, int n_symbols);
FcParams derive_fc_params(int N, int L, double overlap);
double first_block_overlap(const FcParams& params, int l_cp);
std::vector<double> design_window(int L, int n_pass, int n_tb);
std::vector<int> centered_active_map(int l_ofdm, int n_active, bool skip_dc = true);
CpSplit cp_truncate(int n_cp_high, int I);
std::int64_t symbol_sigma(int n, const CpSchedule& cps, int N);
std::int64_t combined_length(int n_symbols, const CpSchedule& cps, const FcParams& p);

// ---- reference-granularity per-symbol API (fc_sync.hpp:24-75, fc_core.hpp
// block_phase): same signatures; each call runs one item through the per-symbol
// device kernels of fcw_symbol.cu (host vectors in and out).
struct FilteredSymbol {  // fc_sync.hpp:31-35
    cvec samples;
    int n = 0;
};
struct SymbolBlocks {  // fc_sync.hpp:57-59
    cvec y0, y1;
};
cd symbol_phase(int n, int c, const CpSchedule& cps, int N);
cd block_phase(std::int64_t r, int c, int L_S, int L);
FilteredSymbol tx_symbol(const cvec& cp_ofdm_symbol, const SubbandConfig& cfg, const FcParams& p,
                         const CpSchedule& cps, int n);
Waveform combine_symbols(const std::vector<FilteredSymbol>& syms, const CpSchedule& cps, const FcParams& p,
                         double fs_hz);
SymbolBlocks rx_segment(const Waveform& w, const CpSchedule& cps, const FcParams& p, int n);
cvec rx_symbol_direct(const cvec& y0, const cvec& y1, const SubbandConfig& cfg, const FcParams& p,
                      const CpSchedule& cps, int n);
cvec rx_symbol_simplified(const cvec& g0, const cvec& g1, const SubbandConfig& cfg, const FcParams& p);
cvec rx_block_freq(const cvec& y, const SubbandConfig& cfg, const FcParams& p, cd phase);

// fc_sync.hpp:52-54 — one GPU pass over all subbands.
Waveform tx_discontinuous(const std::vector<QamGrid>& grids, const std::vector<SubbandConfig>& cfgs,
                          const CpSchedule& cps, int N, double overlap, double fs_hz);
// fc_sync.hpp:78-80 — one subband, full L-bin columns.
std::vector<cvec> rx_discontinuous(const Waveform& w, const SubbandConfig& cfg, const CpSchedule& cps, int N,
                                   double overlap, bool simplified = false);
// All subbands of `cfgs` in one pass (what a multi-subband receiver wants).
std::vector<std::vector<cvec>> rx_discontinuous_all(const Waveform& w, const std::vector<SubbandConfig>& cfgs,
                                                    const CpSchedule& cps, int N, double overlap,
                                                    bool simplified = false);

// Batched, device-resident engine: one immutable plan, S units per call.
class Engine {
  public:
    Engine(int N, double overlap, const CpSchedule& cps, const std::vector<SubbandConfig>& cfgs,
           const std::vector<std::vector<int>>& active_maps);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    fcw_plan_info info() const;
    // device pointers (complex64), see include/fcwave_b200.h
    void tx(const void* grid_dev, void* wave_dev, int S, unsigned flags = 0, void* stream = nullptr) const;
    void rx(const void* wave_dev, std::int64_t wave_len, std::int64_t useful0, void* grid_dev, int S,
            unsigned flags = FCW_RX_FUSED, void* stream = nullptr) const;
    fcw_plan* raw() const { return plan_; }

  private:
    fcw_plan* plan_ = nullptr;
};

void check(int rc);  // throws the reference's exception class for rc

}  // namespace fcwave_b200
