// Internal definitions shared by the host plan builder and the sm_100a
// kernels.  Not part of the public ABI (include/fcwave_b200.h is).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "fcwave_b200.h"

namespace fcw {

constexpr int kThreads = 256;     // CTA size of both kernels
constexpr int kWarps = kThreads / 32;
constexpr int kMaxN = 4096;       // long transform envelope (SMEM-resident blocks)
constexpr int kMaxL = 1024;       // short transform envelope (warp-resident)
constexpr int kMaxGroups = 9;     // distinct L values: 4..1024
constexpr int kMaxLevels = 8;     // contributor ranks per shared bin
constexpr int kMaxTmemClasses = 4; // bin classes whose per-lane rows fit the TMEM columns of a zv kernel

// Per-subband constants resident in HBM (read through L1).
struct SubDev {
    int L, logL, c, logI;
    int act_off;   // offset of this subband's active bins in a packed grid row
    int n_act;
    int full_off;  // offset of this subband's L bins in a full grid row / table row
    int cmodN;     // c mod N (for the symbol rotator exponent)
    float bp1;     // block_phase(1, c, L/2, L) = +-1 (fc_core.cpp:41-44, lambda = 1/2)
    float tx_scale;  // sqrt(I) / (N sqrt(L)): folds ofdm_modulate sqrt(L)/L, IDFT_N 1/N, tx_symbol sqrt(I)
    float rx_s0;     // sqrt(I) (L/N) / sqrt(L)  (fc_sync.cpp:238-240)
    int cls_off;     // offset of this subband's bin-class row in the class table
    int ext_base;    // first extension slot of this subband's secondary bins
    // zv kernels: the TMEM bin-class row pair this subband's warp reads in TX / RX (KParams::combo);
    // both half-warps of a warp issue one tcgen05.ld, so the two subbands of a pair share the id
    int row_tx, row_rx;
    int pad_[1];
};

// Per-symbol geometry (all integer-exact on the host).
struct SymDev {
    long long sigma;  // symbol_sigma (fc_sync.cpp:86-88)
    int cp;           // N_CP,n
    int own_len;      // samples [sigma_n, sigma_n+own_len) owned by symbol n's tile
    int carry_len;    // leading samples that also receive the previous symbol's block 1
    int smodN;        // (sum_{q=1..n} N_CP,q) mod N
    int pad_[2];
};

struct fc_col;  // continuous-FC column descriptor (below)

// Kernel parameter block (passed by value).
struct KParams {
    int N, B, M;
    int chunk;           // max symbols per run (a TX run recomputes the symbol before it)
    int n_units;         // S: units of this launch
    int teams;           // teams per CTA (teams_per_cta<N>)
    int dynamic;         // 1: runs pulled from item_counter; 0: static balanced ranges
    int n_items, nchunks;  // dynamic mode: S * nchunks runs of `chunk` symbols
    int spec_stride;  // float2 per block spectrum in SMEM (>= N + n_ext, >= N + N/16)
    int scratch_stride;  // float2 per warp scratch
    int stab_len;        // entries of the SMEM short-transform twiddle table (plan Lmax)
    int stage_off;       // TX: offset of the cp.async grid staging buffer in a warp's scratch
    int tw16_len;        // float2 entries of the half-warp FFT_256 twiddle table in SMEM (0 or 512)
    int nb_k0;           // narrowband plans (ZV == 2 kernels): first of the 16 spectrum bins in use
    int row_len;
    int grid_full;
    int fused;
    int accumulate;      // TX: add into the waveform instead of storing (FCW_TX_ACCUMULATE)
    int dbg_skip;        // dev-only timing knob (FCW_DEBUG_SKIP): 1 = short stage, 2 = long transform
    int n_ext, n_zero, n_lvl;
    // zv kernels: TMEM bin-class rows.  Row j holds class combo[j][h] for the lanes of half-warp h
    // (the pairs of classes that the fixed subband-to-warp schedule puts side by side in one warp)
    int n_combo;
    int combo[kMaxTmemClasses][2];
    int lvl_start[kMaxLevels + 1];
    int n_groups;
    int grp_L[kMaxGroups], grp_start[kMaxGroups], grp_count[kMaxGroups];
    long long Q;
    long long rx_base;   // useful0 - N_L
    long long wave_len;
    long long in_stride, out_stride;
    const SubDev* sub;
    const SymDev* sym;
    const int* inv;      // [sum L] DFT bin -> active index or -1
    const int2* cls;     // bin-class rows: per DFT bin b {inv[b] | sec(p0) << 16, bits(w[p0])}, p0 = b ^ L/2
    const int* grp_sub;  // subband ids grouped by L
    const int* fix_tgt;  // [n_ext] target bin of each secondary contribution, rank-ordered
    const int* fix_slot; // [n_ext] its extension slot
    // the same contributions grouped by the long-transform thread that loads the target bin
    // (q mod N/16), rank order kept inside a group: entries [own_start[t], own_start[t + 1])
    const int* own_start;
    const int* own_tgt;
    const int* own_slot;
    const int* zero_list;  // [n_zero] bins no subband touches
    const float2* tw;    // [N] exp(-2 pi i k / N)
    // time-domain I/O of the continuous FC (fcw_cont.cu, cp = 0 plans; null =
    // grid I/O): TX reads each subband's low-rate stream, RX writes each
    // subband's output stream, per subband m at td[m] offsets, pair n = sigma / N
    const fc_col* td;
    const float2* in;
    float2* out;
    int* item_counter;   // per-launch scratch: dynamic run counter
    float2* carry;       // per-launch scratch: gridDim.x * teams * N/2 TX carry buffers
};

struct Plan {
    int device = 0;
    int N = 0, B = 0, M = 0;
    double overlap = 0.5;
    fcw_fc_params pN{};  // N-side geometry (N_L, N_T shared by all subbands)
    long long Q = 0, useful0 = 0, frame_samples = 0;
    int row_active = 0, row_full = 0;
    int chunk = 0;
    std::vector<int> cp;
    std::vector<long long> sigma;
    struct Sub {
        fcw_subband desc;
        std::vector<int> bins;
        std::vector<double> window;
        fcw_fc_params p;
    };
    std::vector<Sub> subs;
    // host images of the device tables
    std::vector<SubDev> h_sub;
    std::vector<SymDev> h_sym;
    std::vector<float> h_win;
    std::vector<int> h_inv, h_dest, h_grp_sub, h_fix, h_zero;
    std::vector<int2> h_cls;
    std::vector<int> h_combo;  // zv plans: flattened (class of half 0, class of half 1) per TMEM row
    std::vector<int> h_fix_slot;
    std::vector<int> h_own_start, h_own_tgt, h_own_slot;  // fix-up list grouped by owner thread
    int n_ext = 0, n_lvl = 0;
    std::vector<int> lvl_start;
    int n_groups = 0;
    int grp_L[kMaxGroups]{}, grp_start[kMaxGroups]{}, grp_count[kMaxGroups]{};
    int Lmax = 0;
    bool zv = false;
    int n_zero_core = 0;  // zero-filled bins (the guard band of a zv plan excluded)
    bool generic = false;  // run the generic (LU = 0) kernels even for a uniform L (continuous-FC TX plans
                           // whose short paths carry the time-domain input only there, fcw_cont.cu)
    bool nb = false;      // narrowband: every subband span within 16 bins [nb_k0, nb_k0 + 16), N = 1024, L = 16
    int nb_k0 = 0;  // uniform L = 256, N = 4096, bins t + 16m (m in [5, 10]) inactive and windowed out
    // device tables (one allocation)
    void* d_blob = nullptr;
    SubDev* d_sub = nullptr;
    SymDev* d_sym = nullptr;
    int *d_inv = nullptr, *d_grp_sub = nullptr, *d_fix = nullptr, *d_zero = nullptr;
    int2* d_cls = nullptr;
    int* d_fix_slot = nullptr;
    int *d_own_start = nullptr, *d_own_tgt = nullptr, *d_own_slot = nullptr;
    float2* d_tw = nullptr;
    // host-buffer pipeline state
    std::mutex host_mu;
    cudaStream_t streams[2] = {nullptr, nullptr};
    void* stage[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    size_t stage_bytes[2][2] = {{0, 0}, {0, 0}};
};

// Continuous-FC column descriptor (fcw_cont.cu): one per subband.
struct fc_col {
    long long in_off;   // TX: offset of this subband's stream in a unit's concatenated streams
    long long len;      // TX: stream length (low-rate samples)
    long long out_off;  // RX: offset of this subband's output stream in a unit's output
    long long len_out;  // RX: R_tot * L_S output samples
    int lt;             // L_T: the block-pair window starts L_T samples before 2 n L_S
    int row;            // full grid row length (sum L_m)
    int full_off;       // this subband's first bin in a full grid row
    int pad_;
};

int set_error(int code, const std::string& msg);
struct fc_col;
int set_cuda_error(cudaError_t e, const char* where);

// fcw_launch.cu
// per-device stream-ordered scratch pool that keeps its memory (no OS
// re-allocation after every synchronisation)
cudaError_t scratch_pool(int dev, cudaMemPool_t* out);
// SM count of the current device (queried once per device; grid sizing and
// the work schedule use it instead of a hard-coded 148).
int device_sms();
template <class T>
cudaError_t scratch_alloc(T** p, size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (e == cudaSuccess) e = scratch_pool(dev, &pool);
    if (e == cudaSuccess) e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, pool, st);
    return e;
}
cudaError_t launch_tx(const Plan& plan, KParams& kp, int S, cudaStream_t st);
cudaError_t launch_rx(const Plan& plan, KParams& kp, int S, cudaStream_t st);
cudaError_t launch_gen_qam(const Plan& plan, uint64_t seed, long long unit0, int S, int bits,
                           float2* out, cudaStream_t st);
bool plan_team_only(const Plan& plan);  // the plan runs the team-only kernels (fcw_launch.cu)
size_t tx_smem_bytes(const Plan& plan);
// fcw_link.cu (link step around the path; blocking where results go to the host)
cudaError_t link_stats(const Plan& p, const float2* grid, long long stride, int S, uint64_t seed, long long unit0,
                       int bits, double* evm_num, double* evm_den, long long* errors, cudaStream_t st);
cudaError_t awgn(float2* wave, long long stride, long long len, int S, double sigma2, uint64_t seed,
                 long long unit0, cudaStream_t st);
cudaError_t wave_power(const float2* wave, long long stride, int S, long long begin, long long end, double* power,
                       cudaStream_t st);
cudaError_t apply_channel(const float2* in, float2* out, long long stride, long long len, int S, const int* delays,
                          const float2* gains, int n_taps, cudaStream_t st);
cudaError_t psd(const float2* wave, long long stride, long long len, int S, int L, double overlap, double* out_host,
                cudaStream_t st);
size_t rx_smem_bytes(const Plan& plan);
void fill_common(const Plan& plan, KParams& kp);
// fcw_capi.cpp: continuous FC with time-domain I/O (fcw_cont.cu)
// reference-granularity per-symbol entry points (fcw_symbol.cu)
cudaError_t sym_tx_symbol(const Plan& p, int m, const float2* sym, long long sym_stride, int l_cp, float2 ph0,
                          float2 ph1, float scale, float2* out, long long out_stride, int S, cudaStream_t st);
cudaError_t sym_combine(const Plan& p, const float2* syms, long long sym_unit_stride, float2* wave,
                        long long wave_stride, int S, cudaStream_t st);
cudaError_t sym_rx_block_freq(const Plan& p, int m, const float2* y, long long y_stride, float2 cph, float2* g,
                              long long g_stride, int S, cudaStream_t st);
cudaError_t sym_rx_simplified(const Plan& p, int m, const float2* g0, const float2* g1, long long g_stride,
                              float scale, float2* out, long long out_stride, int S, cudaStream_t st);
cudaError_t sym_rx_direct(const Plan& p, int m, const float2* y0, const float2* y1, long long y_stride, float2 cph0,
                          float2 cph1, float scale, float2* out, long long out_stride, int S, cudaStream_t st);
void plan_force_generic(fcw_plan* p);
void plan_clear_special(fcw_plan* p);
int tx_time_domain(const fcw_plan* p, const fc_col* td, const float2* streams, long long stream_stride,
                   float2* wave, long long wave_stride, int S, cudaStream_t st);
int rx_time_domain(const fcw_plan* p, const fc_col* td, const float2* wave, long long wave_stride,
                   long long wave_len, long long rx_base, float2* out, long long out_stride, int S,
                   cudaStream_t st);

}  // namespace fcw
