/*
 * TEST INFRASTRUCTURE ONLY.  This is the CPU oracle for the FC-F-OFDM hot
 * path: a plain-C, double-precision restatement of the reference algorithm
 * (fcwave, arXiv 2008.00672).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it, and only as
 * the checker.  The product library (paper_2008_00672_b200) never links it.
 *
 * Pinning: tests/test_oracle.py checks every function here against the known
 * answers in the reference's own tests (proj/tests/test_{numerology,ofdm,
 * fc_core,fc_sync}.cpp, proj/tests/acceptance.cpp c1-c4,c10,
 * proj/python/tests/test_smoke.py:47-70), against first-principles dense
 * operators (the proj/tests/oracle.hpp construction, restated in numpy), and
 * against the unmodified reference compiled here (oracle/_ref) through the
 * committed golden vectors in tests/golden/.
 *
 * Complex data are interleaved doubles (re, im).  Functions return 0 on
 * success, 1 for the reference's std::invalid_argument cases, 2 for its
 * std::out_of_range cases.
 */
#ifndef FCW_ORACLE_H
#define FCW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int L, N;
    double overlap;
    int L_O, L_S, L_L, L_T;
    int N_O, N_S, N_L, N_T;
    int I;
} fco_params;

int fco_derive_params(int N, int L, double overlap, fco_params* p);
int fco_cp_schedule(int scs_khz, int n_fft, int n_symbols, int* out);
void fco_cp_truncate(int n_cp_high, int I, int* l_cp, int* extrap);
int64_t fco_cp_partial_sum(const int* cp, int n);
int64_t fco_symbol_sigma(int n, const int* cp, int N);
void fco_bin_map(int L, int c, int N, int* q, int* b);
int64_t fco_rx_start(int64_t useful0, int N_L, int n, const int* cp, int N);
int64_t fco_combined_length(int B, const int* cp, const fco_params* p);
int fco_design_window(int L, int n_pass, int n_tb, double* w);
int fco_centered_active_map(int l_ofdm, int n_active, int skip_dc, int* bins);
void fco_block_phase(int64_t r, int c, int L_S, int L, double* re, double* im);
void fco_symbol_phase(int n, int c, const int* cp, int N, double* re, double* im);

/* fc_sync.cpp:34-43 (z length 3L/2) and :52-58 (first-block window) */
int fco_zero_pad_symbol(const double* sym, int sym_len, const fco_params* p, int l_cp, double* z);
int fco_first_block_window(const fco_params* p, int l_cp, double* a);

/* In-place DFT: forward unscaled e^{-j}; inverse e^{+j} with 1/n. */
void fco_fft(double* data, int n, int inverse);

int fco_tx_symbol(const double* sym, int sym_len, int L, int c, const double* window,
                  const fco_params* p, const int* cp, int n, double* out3n2);
/* grids: per subband m, B full columns of L_m complex values, concatenated. */
int fco_tx_discontinuous(int N, double overlap, const int* cp, int B, int M, const int* Ls,
                         const int* cs, const double* windows, const double* grids, double* wave,
                         int64_t cap, int64_t* Q, int64_t* useful0);
int fco_rx_block_freq(const double* y, int L, int c, const double* window, const fco_params* p,
                      double ph_re, double ph_im, double* g);
int fco_rx_symbol_direct(const double* y0, const double* y1, int L, int c, const double* window,
                         const fco_params* p, const int* cp, int n, double* out);
int fco_rx_symbol_simplified(const double* g0, const double* g1, const fco_params* p, double* out);
int fco_rx_discontinuous(const double* wave, int64_t len, int64_t useful0, int N, double overlap,
                         const int* cp, int B, int L, int c, const double* window, int simplified,
                         double* out);

/* Seeded synthetic inputs (channel.cpp:19-48, scenario.cpp:110-128,
 * ofdm.cpp:55-65 extended to 256-QAM).  packed: [units][B][A] complex. */
uint64_t fco_splitmix64(uint64_t* state);
uint64_t fco_derive_seed(uint64_t seed, uint64_t index);
void fco_qam_map(int bits_per_symbol, unsigned symbol_bits, double* re, double* im);
void fco_gen_grid(uint64_t seed, int64_t unit0, int units, int B, int A, int bits_per_symbol,
                  double* packed);

/* Link step around the path (f1/f3): ofdm.cpp:67-78, metrics.cpp:105-127,
 * scenario.cpp:469-494, channel.cpp:37-42,136-155. */
unsigned fco_qam_demap(int bits_per_symbol, double re, double im);
void fco_link_stats(const double* rx, uint64_t seed, int64_t unit0, int units, int B, int A,
                    int bits_per_symbol, double* out, int64_t* errs);
void fco_gauss_complex(uint64_t* state, double* re, double* im);
void fco_awgn(double* wave, int64_t len, double sigma2, uint64_t seed);
double fco_measure_power(const double* wave, int64_t len, int64_t begin, int64_t end);

/* TDL channel (f3): channel.cpp:101-124. */
void fco_draw_tdl(const double* delay_ns, const double* power_lin, int n_taps, double fs_hz, uint64_t seed,
                  int* delays, double* gains);
void fco_apply_channel(const double* w, int64_t len, const int* delays, const double* gains, int n_taps,
                       double* out);

/* Welch PSD (f4): metrics.cpp:128-155. */
int fco_psd(const double* x, int64_t len, int seg_len, double overlap_frac, double* out);

/* Continuous FC filterbank (f2): fc_core.cpp:155-223. */
int fco_continuous_block_count(int stream_len, const fco_params* p);
int fco_tx_continuous(int N, double overlap, int M, const int* Ls, const int* cs, const double* windows,
                      const double* streams, const int64_t* lens, int l_cp0, double* wave, int64_t cap,
                      int64_t* out_len, int64_t* useful0);
int fco_rx_continuous(const double* wave, int64_t len, int N, double overlap, int L, int c,
                      const double* window, double* out, int64_t cap, int64_t* n_out);

#ifdef __cplusplus
}
#endif

#endif
