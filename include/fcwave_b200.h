/*
 * fcwave-b200 — C ABI of the B200-native symbol-synchronized FC-F-OFDM
 * TX synthesis / RX analysis hot path (arXiv 2008.00672).
 *
 * This is the drop-in boundary for the reference's operator API
 * (/root/reference/proj/include/fcwave/fc_sync.hpp).  Every entry point names
 * the reference interface it replaces.  Plain C types only: complex samples are
 * interleaved float32 pairs (re, im) ("complex64"), streams are cudaStream_t
 * passed as void*, device and host buffers are plain pointers owned by the
 * caller.
 *
 * Errors: every function returns FCW_OK (0) or a status code; the message is
 * available from fcw_last_error() (thread-local).  The codes mirror the
 * reference's exception classes: FCW_EINVAL <-> std::invalid_argument,
 * FCW_ERANGE <-> std::out_of_range (proj/src/fc_sync.cpp:35-38,62-63,117-125,
 * 137-138,146-151,198-201; proj/src/numerology.cpp:45-54).
 *
 * Threading: a plan is immutable after creation and may be used concurrently
 * from several host threads / CUDA streams with the device entry points
 * (fcw_tx, fcw_rx).  The host-buffer entry points (fcw_tx_host, fcw_rx_host)
 * serialize per plan (they own staging buffers).
 */
#ifndef FCWAVE_B200_H
#define FCWAVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCW_OK 0
#define FCW_EINVAL 1  /* std::invalid_argument in the reference */
#define FCW_ERANGE 2  /* std::out_of_range in the reference */
#define FCW_ECUDA 3   /* CUDA runtime failure (no device, launch error, ...) */
#define FCW_ENOMEM 4  /* device / pinned host allocation failed */
#define FCW_ENOTSUP 5 /* valid for the reference but outside this build's envelope */

/* fcw_tx / fcw_rx flags */
#define FCW_GRID_FULL 1u /* grid rows hold all L_m DFT bins per subband (QamGrid::symbols,
                            ofdm.hpp:27-33) instead of the packed active bins */
#define FCW_RX_FUSED 2u  /* RX by transform decomposition (rx_symbol_simplified,
                            fc_sync.cpp:195-243); default is the direct path
                            (rx_symbol_direct, fc_sync.cpp:158-176) */
#define FCW_TX_ACCUMULATE 4u /* TX adds into the waveform instead of storing it: the
                            reference's subband sum w += sub (fc_sync.cpp:139),
                            e.g. a second numerology's bank at a sample offset */

/* Geometry of one FC bank (FcParams, numerology.hpp:34-41). */
typedef struct fcw_fc_params {
    int L, N;
    double overlap;
    int L_O, L_S, L_L, L_T;
    int N_O, N_S, N_L, N_T;
    int I;
} fcw_fc_params;

/* One subband (SubbandConfig, fc_core.hpp:20-27, plus QamGrid::active_map,
 * ofdm.hpp:27-33).  Copied at plan creation; the caller keeps ownership. */
typedef struct fcw_subband {
    int L;                  /* short transform size L_m (power of two, 4..1024, L | N) */
    int l_ofdm;             /* OFDM transform size; must equal L (fc_sync.cpp:62-63); 0 = L */
    int c;                  /* centre bin on the N-bin grid */
    int n_active;           /* number of active (QAM-bearing) bins */
    int n_tb;               /* transition bins per edge (informational) */
    const int* active_bins; /* n_active DFT-bin indices in [0, L): packed grid order */
    const double* window;   /* L shifted-domain weights (design_window, fc_core.cpp:25-39) */
} fcw_subband;

typedef struct fcw_plan fcw_plan;

typedef struct fcw_plan_info {
    int N, B, M;
    double overlap;
    int64_t Q;             /* combined_length(B) (fc_sync.cpp:90-94): waveform samples per unit */
    int64_t useful0;       /* Waveform::useful0 of the TX output = N_L (fc_sync.cpp:102) */
    int64_t frame_samples; /* sum_n (N + N_CP,n): air-interface samples per unit */
    int row_active;        /* packed grid row length: sum_m n_active */
    int row_full;          /* full grid row length: sum_m L_m */
    int N_L, N_T;
    int chunk;             /* symbols per CTA (launch geometry, informational) */
    int kernel_variant;    /* informational: 0 general, 1 zero-bin L = 256 / N = 4096 (TMEM tables), 2 narrowband, 3 team-only */
    int tmem_rows;         /* zero-bin variant: bin-class row pairs parked in tensor memory (<= 4) */
} fcw_plan_info;

/* ----------------------------------------------------------------- plan */

/* Replaces the per-call geometry of tx_discontinuous / rx_discontinuous
 * (fc_sync.hpp:52-54, 78-80): N, overlap, the explicit CpSchedule
 * (numerology.hpp:23-31) and the subband configs.  Validates exactly the
 * reference preconditions (derive_fc_params numerology.cpp:44-54,
 * zero_pad_symbol fc_sync.cpp:35-38, tx_symbol :62-63, cp_insert ofdm.cpp:109,
 * equal Q/useful0 across subbands fc_sync.cpp:137-138).  Allocates the
 * device-resident tables on the current CUDA device.  flags: reserved, 0. */
int fcw_plan_create(fcw_plan** plan, int N, double overlap, const int* cp_high, int B,
                    const fcw_subband* subbands, int M, unsigned flags);
void fcw_plan_destroy(fcw_plan* plan);
int fcw_plan_get_info(const fcw_plan* plan, fcw_plan_info* info);
/* sigma_n = n N + sum_{q=1..n} N_CP,q (symbol_sigma, fc_sync.cpp:86-88), B entries */
int fcw_plan_sigma(const fcw_plan* plan, int64_t* sigma);
/* per-symbol (l_cp, extrap) of subband m (cp_truncate, fc_sync.cpp:26-32), B entries each */
int fcw_plan_cp_split(const fcw_plan* plan, int m, int* l_cp, int* extrap);
/* subband m bin map: for shifted index p0 in [0, L): q[p0] = (c - ceil(L/2) + p0) mod N
 * and b[p0] = (p0 + L/2) mod L (fc_core.cpp:81-84) */
int fcw_plan_bin_map(const fcw_plan* plan, int m, int* q, int* b);
/* rx block starts: useful0 - N_L + sigma_n (rx_segment, fc_sync.cpp:148), B entries */
int fcw_plan_rx_starts(const fcw_plan* plan, int64_t useful0, int64_t* starts);
int fcw_plan_fc_params(const fcw_plan* plan, int m, fcw_fc_params* out);

/* ------------------------------------------------------ device entry points */

/* TX synthesis of S independent units (antenna stream x frame) — replaces
 * tx_discontinuous (fc_sync.hpp:52-54, fc_sync.cpp:114-143).
 *   grid: device complex64 [S][B][row] with row = row_active (packed, default)
 *         or row_full (FCW_GRID_FULL); grid_unit_stride in complex elements
 *         (0 = B*row).
 *   wave: device complex64 [S][wave_unit_stride] (0 = Q); samples [0, Q) of
 *         each unit are written (or added to, with FCW_TX_ACCUMULATE),
 *         useful0 = N_L.
 * Asynchronous on `stream` (cudaStream_t; NULL = legacy default stream). */
int fcw_tx(const fcw_plan* plan, const void* grid, int64_t grid_unit_stride, void* wave,
           int64_t wave_unit_stride, int S, unsigned flags, void* stream);

/* RX analysis of S units — replaces rx_discontinuous (fc_sync.hpp:78-80,
 * fc_sync.cpp:245-264) for ALL subbands of the plan in one pass (one shared
 * N-point transform per block instead of one per subband).
 *   wave: device complex64 [S][wave_unit_stride] (0 = wave_len), wave_len
 *         samples per unit, first useful sample of symbol 0 at useful0.
 *   grid: device complex64 [S][B][row] (packed active bins, or all L_m bins
 *         with FCW_GRID_FULL = the reference's return layout).
 * flags: FCW_RX_FUSED selects the transform-decomposition path. */
int fcw_rx(const fcw_plan* plan, const void* wave, int64_t wave_unit_stride, int64_t wave_len,
           int64_t useful0, void* grid, int64_t grid_unit_stride, int S, unsigned flags, void* stream);

/* ------------------- reference-granularity per-symbol entry points
 * The reference's finer hot-path API (fc_sync.hpp:38-75), batched over S
 * items (units) of ONE (subband m, symbol n) of the plan, on the device, in
 * complex fp32 (all buffers device complex64; a stride of 0 = contiguous).
 * They run their own generic kernels (fcw_symbol.cu), not the fused
 * whole-frame K-TX / K-RX; use fcw_tx / fcw_rx for throughput. */

/* symbol_phase (fc_sync.hpp:24, fc_sync.cpp:45-50) and block_phase
 * (fc_core.cpp:41-44) in double, bit-exact with the reference. */
int fcw_symbol_phase(int n, int c, const int* cp_high, int B, int N, double* re, double* im);
int fcw_block_phase(int64_t r, int c, int L_S, int L, double* re, double* im);

/* tx_symbol (fc_sync.hpp:41-42): sym [S][sym_stride] holds the CP-OFDM
 * symbol n of subband m, L + l_cp samples (l_cp <= L_L); out [S][out_stride]
 * receives its 3N/2 filtered samples (FilteredSymbol::samples). */
int fcw_tx_symbol(const fcw_plan* plan, int m, int n, const void* sym, int64_t sym_stride, int l_cp, void* out,
                  int64_t out_stride, int S, void* stream);

/* combine_symbols (fc_sync.hpp:46-47): syms [S][B][3N/2] (symbol n at index
 * n, unit stride sym_unit_stride, 0 = B*3N/2) overlap-added at sigma_n into
 * wave [S][wave_stride] (Q samples, useful0 = N_L). */
int fcw_combine_symbols(const fcw_plan* plan, const void* syms, int64_t sym_unit_stride, void* wave,
                        int64_t wave_stride, int S, void* stream);

/* rx_segment (fc_sync.hpp:60): y0 = w[start, +N), y1 = w[start + N/2, +N),
 * start = useful0 - N_L + sigma_n, for S waveforms.  FCW_ERANGE for n outside
 * the CP schedule, FCW_EINVAL when the window leaves the waveform. */
int fcw_rx_segment(const fcw_plan* plan, const void* wave, int64_t wave_stride, int64_t wave_len, int64_t useful0,
                   int n, void* y0, void* y1, int64_t y_stride, int S, void* stream);

/* rx_block_freq (fc_sync.hpp:73): g [S][g_stride] = the L frequency-domain FC
 * outputs of subband m of the N-sample blocks y [S][y_stride], with phase. */
int fcw_rx_block_freq(const fcw_plan* plan, int m, const void* y, int64_t y_stride, double phase_re,
                      double phase_im, void* g, int64_t g_stride, int S, void* stream);

/* rx_symbol_simplified (fc_sync.hpp:69-70), Eq. (30): L bins of subband m
 * from g0, g1 [S][g_stride]. */
int fcw_rx_symbol_simplified(const fcw_plan* plan, int m, const void* g0, const void* g1, int64_t g_stride,
                             void* out, int64_t out_stride, int S, void* stream);

/* rx_symbol_direct (fc_sync.hpp:64-65): L bins of subband m, symbol n, from
 * the blocks y0, y1 [S][y_stride]. */
int fcw_rx_symbol_direct(const fcw_plan* plan, int m, int n, const void* y0, const void* y1, int64_t y_stride,
                         void* out, int64_t out_stride, int S, void* stream);

/* Seeded synthetic QAM grid on the device, bit-identical to the host oracle:
 * per unit u a splitmix64 stream seeded derive_seed(seed, unit0 + u)
 * (channel.cpp:19-48), one draw per bit LSB-first (scenario.cpp:110-128),
 * Gray square QAM of bits_per_symbol in {2,4,6,8} at unit power (ofdm.cpp:55-65,
 * extended to 256-QAM).  Output: packed grid [S][B][row_active]. */
int fcw_gen_qam(const fcw_plan* plan, uint64_t seed, int64_t unit0, int S, int bits_per_symbol,
                void* grid, void* stream);

/* --------------------------------------- link step around the path (f1, f3) */

/* Per-unit link statistics of a received packed grid [S][B][row_active]
 * against the seeded transmit grid of fcw_gen_qam(seed, unit0, bits): the EVM
 * sums sum|y - x|^2, sum|x|^2 (evm_db, metrics.cpp:115-127) and the bit errors
 * of the hard decisions (qam_demap ofdm.cpp:67-78, ber metrics.cpp:105-113),
 * as accumulated per drop in run_scenario (scenario.cpp:469-494).  Decisions
 * are computed in double exactly like the reference; sums are reduced in a
 * fixed order (deterministic).  Blocking: stats go to host memory. */
typedef struct fcw_link_stat {
    double evm_num, evm_den;
    int64_t bit_errors, n_bits;
} fcw_link_stat;
int fcw_link_stats(const fcw_plan* plan, const void* grid, int64_t grid_unit_stride, int S, uint64_t seed,
                   int64_t unit0, int bits_per_symbol, fcw_link_stat* stats, void* stream);

/* awgn_with_variance (channel.cpp:136-141) on S device waveforms in place:
 * unit u draws GaussianRng(derive_seed(seed, unit0 + u)) (channel.cpp:37-48),
 * two draws per sample; v += sqrt(sigma2) * n in double, stored as fp32. */
int fcw_awgn(const fcw_plan* plan, void* wave, int64_t wave_unit_stride, int64_t wave_len, int S, double sigma2,
             uint64_t seed, int64_t unit0, void* stream);

/* draw_tdl (channel.cpp:101-111), host: delays[k] = lround(delay_ns[k] 1e-9 fs),
 * gains[k] = sqrt(power_lin[k]) * GaussianRng(seed).next_complex() (complex
 * as interleaved doubles, 2 n_taps). */
int fcw_draw_tdl(const double* delay_ns, const double* power_lin, int n_taps, double fs_hz, uint64_t seed,
                 int* delays, double* gains);

/* apply_channel (channel.cpp:113-124) on S device waveforms, out of place:
 * out[u][t] = sum_k g[u][k] in[u][t - d[u][k]] (t >= d[u][k]).  delays
 * [S][n_taps] and gains [S][n_taps] (interleaved complex doubles) are host
 * arrays, one tap line per unit, n_taps <= 64.  Blocking. */
int fcw_apply_channel(const void* wave_in, void* wave_out, int64_t wave_unit_stride, int64_t wave_len, int S,
                      const int* delays, const double* gains, int n_taps, void* stream);

/* measure_power (channel.cpp:148-155) per unit: mean |v|^2 over
 * [begin, end) clipped to [0, wave_len).  Blocking: power[S] on the host. */
int fcw_wave_power(const fcw_plan* plan, const void* wave, int64_t wave_unit_stride, int64_t wave_len, int S,
                   int64_t begin, int64_t end, double* power, void* stream);

/* Zero samples [begin, end) of S device waveforms (stream-ordered 2-D
 * memset).  MixedNumerology composition: the spans the first bank does not
 * write before later banks accumulate onto them (there is no reference
 * counterpart; the reference allocates zeroed vectors, fc_sync.cpp:103,133). */
int fcw_wave_zero(void* wave, int64_t wave_unit_stride, int S, int64_t begin, int64_t end, void* stream);

/* Welch PSD (metrics.cpp:128-155, row f4) of S device waveforms of wave_len
 * samples: Hann windows of seg_len (a power of two in [64, 4096]) hopping
 * lround(seg_len (1 - overlap_frac)), |FFT|^2 averaged and scaled by
 * 1 / (n_seg sum w^2).  Per-bin sums in double, deterministic order.
 * Blocking: psd[S][seg_len] (double) on the host. */
int fcw_psd(const void* wave, int64_t wave_unit_stride, int64_t wave_len, int S, int seg_len, double overlap_frac,
            double* psd, void* stream);

/* ------------------------------------ continuous FC filterbank (row f2) */

/* Replaces tx_continuous / rx_continuous (fc_core.hpp:64-77, fc_core.cpp:
 * 155-223): blocks hop L_S = L/2 (low rate) and N_S = N/2 (high rate).  The
 * plan fixes N, overlap (0.5), the subbands (window, c, L; active_bins and
 * n_active are ignored: every bin is carried), the TX low-rate stream length
 * of each subband (CpOfdmSignal::samples.size()), the RX waveform length and
 * the first subband's first low-rate CP length l_cp0 (for useful0,
 * fc_core.cpp:192-196).  Internally a block pair (2n, 2n+1) is one cp = 0
 * symbol of the fused kernels (see fcw_cont.cu). */
typedef struct fcw_cont_plan fcw_cont_plan;
typedef struct fcw_cont_info {
    int N, M;
    int64_t tx_len;       /* reference waveform length: max_m (R_tot,m - 1) N_S + N */
    int64_t tx_stride;    /* samples per unit written by fcw_tx_continuous (>= tx_len; the tail is zero) */
    int64_t useful0;      /* Waveform::useful0 = round(overlap N) + I_0 l_cp0 */
    int64_t stream_total; /* sum_m stream_len[m]: TX input samples per unit */
    int64_t rx_wave_len;  /* RX input samples per unit */
    int64_t rx_out_total; /* sum_m R_tot,m L_S,m: RX output samples per unit */
    int tx_pairs, rx_pairs; /* block pairs per unit */
} fcw_cont_info;
int fcw_cont_plan_create(fcw_cont_plan** plan, int N, double overlap, const fcw_subband* subbands, int M,
                         const int64_t* stream_len, int64_t rx_wave_len, int l_cp0);
void fcw_cont_plan_destroy(fcw_cont_plan* plan);
/* rx_out_len / rx_out_off (M entries each, may be NULL): each subband's RX
 * output length R_tot,m L_S,m and offset in a unit's output row. */
int fcw_cont_plan_get_info(const fcw_cont_plan* plan, fcw_cont_info* info, int64_t* rx_out_len,
                           int64_t* rx_out_off);
/* streams: device complex64 [S][stream_total] (subband streams concatenated
 * in order); wave: device complex64 [S][tx_stride].  Stream-ordered. */
int fcw_tx_continuous(const fcw_cont_plan* plan, const void* streams, void* wave, int S, void* stream);
/* wave: device complex64 [S][rx_wave_len]; out: device complex64
 * [S][rx_out_total], subband m at rx_out_off[m] (rx_continuous per subband). */
int fcw_rx_continuous(const fcw_cont_plan* plan, const void* wave, void* out, int S, void* stream);

/* -------------------------------------------------- host-buffer entry points */

/* Same as fcw_tx / fcw_rx with HOST buffers (pinned via fcw_host_alloc for
 * full PCIe overlap; pageable works but is slower).  Units are streamed in
 * chunks through device staging buffers on two CUDA streams so H2D, kernels
 * and D2H overlap.  Blocking. */
int fcw_tx_host(fcw_plan* plan, const void* grid_host, void* wave_host, int S, unsigned flags);
int fcw_rx_host(fcw_plan* plan, const void* wave_host, int64_t wave_len, int64_t useful0,
                void* grid_host, int S, unsigned flags);
void* fcw_host_alloc(size_t bytes);
void fcw_host_free(void* p);

/* -------------------------------------------- geometry (host, integer-exact) */

int fcw_derive_fc_params(int N, int L, double overlap, fcw_fc_params* out);  /* numerology.cpp:44-70 */
int fcw_cp_schedule(int scs_khz, int n_fft, int n_symbols, int* out);        /* numerology.cpp:29-42 */
/* 5G-NR normal-CP pattern for scs = 15*2^mu kHz: short = 144 N/2048, long =
 * short + 16*2^mu N/2048 on symbols n mod (7*2^mu) == 0 (0.5 ms boundaries).
 * Equals fcw_cp_schedule at 15 kHz; gives 288/352 at 30 kHz, N=4096. */
int fcw_nr_cp_schedule(int scs_khz, int n_fft, int n_symbols, int* out);
int fcw_cp_truncate(int n_cp_high, int I, int* l_cp, int* extrap);           /* fc_sync.cpp:26-32 */
int fcw_first_block_overlap(const fcw_fc_params* p, int l_cp, double* out);  /* numerology.cpp:72-76 */
int fcw_design_window(int L, int n_pass, int n_tb, double* w);              /* fc_core.cpp:25-39 */
int fcw_centered_active_map(int l_ofdm, int n_active, int skip_dc, int* bins); /* ofdm.cpp:80-95 */
int64_t fcw_symbol_sigma(int n, const int* cp_high, int N);                 /* fc_sync.cpp:86-88 */
int64_t fcw_combined_length(int B, const int* cp_high, const fcw_fc_params* p); /* fc_sync.cpp:90-94 */

const char* fcw_last_error(void);
const char* fcw_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FCWAVE_B200_H */
