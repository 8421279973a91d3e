// Launch configuration and the K-GEN generator kernel.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "fcw_device.cuh"

namespace fcw {

KernelPair kernels_n16_l0();
KernelPair kernels_n32_l0();
KernelPair kernels_n64_l0();
KernelPair kernels_n128_l0();
KernelPair kernels_n256_l0();
KernelPair kernels_n512_l0();
KernelPair kernels_n1024_l0();
KernelPair kernels_n2048_l0();
KernelPair kernels_n4096_l0();
KernelPair kernels_n1024_l16();
KernelPair kernels_n1024_l32();
KernelPair kernels_n1024_l64();
KernelPair kernels_n1024_l128();
KernelPair kernels_n1024_l256();
KernelPair kernels_n1024_l512();
KernelPair kernels_n1024_l1024();
KernelPair kernels_n2048_l16();
KernelPair kernels_n2048_l32();
KernelPair kernels_n2048_l64();
KernelPair kernels_n2048_l128();
KernelPair kernels_n2048_l256();
KernelPair kernels_n2048_l512();
KernelPair kernels_n2048_l1024();
KernelPair kernels_n4096_l16();
KernelPair kernels_n4096_l32();
KernelPair kernels_n4096_l64();
KernelPair kernels_n4096_l128();
KernelPair kernels_n4096_l256();
KernelPair kernels_n4096_l512();
KernelPair kernels_n4096_l1024();
KernelPair kernels_n4096_l256z();
KernelPair kernels_n1024_l16n();
KernelPair kernels_n4096_l1024t();
KernelPair kernels_n2048_l512t();
KernelPair kernels_n2048_l1024t();
KernelPair kernels_n1024_l512t();
KernelPair kernels_n1024_l1024t();

namespace {

KernelPair pick_l(int N, int LU) {
#define FCW_PICK_L(NN)                         \
    switch (LU) {                              \
        case 16: return kernels_n##NN##_l16();   \
        case 32: return kernels_n##NN##_l32();   \
        case 64: return kernels_n##NN##_l64();   \
        case 128: return kernels_n##NN##_l128(); \
        case 256: return kernels_n##NN##_l256(); \
        case 512: return kernels_n##NN##_l512(); \
        case 1024: return kernels_n##NN##_l1024(); \
        default: return kernels_n##NN##_l0();    \
    }
    switch (N) {
        case 1024: FCW_PICK_L(1024)
        case 2048: FCW_PICK_L(2048)
        case 4096: FCW_PICK_L(4096)
        default: return KernelPair{nullptr, nullptr, nullptr, nullptr};
    }
#undef FCW_PICK_L
}

KernelPair pick(int N, int LU, bool zv = false, bool nb = false, bool team = false) {
    if (zv && N == 4096 && LU == 256) return kernels_n4096_l256z();
    if (team) {
        if (N == 4096 && LU == 1024) return kernels_n4096_l1024t();
        if (N == 2048 && LU == 512) return kernels_n2048_l512t();
        if (N == 2048 && LU == 1024) return kernels_n2048_l1024t();
        if (N == 1024 && LU == 512) return kernels_n1024_l512t();
        if (N == 1024 && LU == 1024) return kernels_n1024_l1024t();
    }
    if (nb && N == 1024 && LU == 16) return kernels_n1024_l16n();
    switch (N) {
        case 16: return kernels_n16_l0();
        case 32: return kernels_n32_l0();
        case 64: return kernels_n64_l0();
        case 128: return kernels_n128_l0();
        case 256: return kernels_n256_l0();
        case 512: return kernels_n512_l0();
        default: return pick_l(N, LU);
    }
}

// The uniform short size the specialised kernels were built for, or 0.
int uniform_L(const Plan& p) {
    if (p.generic || p.n_groups != 1 || p.N < 1024) return 0;
    const int L = p.grp_L[0];
    return (L >= 16 && L <= 1024) ? L : 0;
}

// Team-only kernels (ZV = 3): uniform L >= 512 with the team-wide short path
// usable (>= 4 points per thread) and at most one subband per two warps of a
// team (use_team_short / tx_short_all in fcw_device.cuh).
bool team_only(const Plan& p) {
    const int LU = uniform_L(p);
    if (LU < 512) return false;  // (continuous TX plans with L >= 512 run the generic kernels: LU = 0)
    const int G = (p.N >= 512 && p.N <= 4096) ? 4096 / p.N : 1, TT = G == 1 ? kThreads : p.N / kPPT;
    if (LU > p.N || LU / TT < 4) return false;
    return 2 * p.M <= TT / 32;
}

// RX with the half-warp L = 256 path keeps a wrap-around copy of bins [0, L)
// at [N, N + L) (rx_kernel, rx_short_half).
bool rx_mirror(const Plan& p) { return uniform_L(p) == 256; }

int spec_stride(const Plan& p, bool mirror = false) {
    int ext = p.n_ext > p.N / 16 ? p.n_ext : p.N / 16;
    if (mirror && ext < p.Lmax) ext = p.Lmax;
    return (p.N + ext + 2 + 1) & ~1;
}

// Warp scratch: one padded buffer of the largest warp-path L, two where a path
// transforms both blocks at once (TX; direct RX at L = 64 and generic plans).
// TX: two FFT buffers (lockstep block DFTs for L <= 256; for L >= 512 the
// second holds the cp.async staging of the next subband's grid values);
// RX: one buffer, two where the direct path needs both blocks' short outputs
// at once (L = 64, generic plans).
int scratch_one(const Plan& p) { return (p.Lmax + p.Lmax / 16 + 2 + 1) & ~1; }
bool team_only(const Plan& p);
int scratch_stride(const Plan& p, int LU, bool tx, bool rx_direct) {
    if (p.Lmax < 64) return 0;
    if (team_only(p)) {
        // tx/rx_short_team: two buffers of L + L/16 + 2 per team, spread over
        // the team's contiguous warp scratch
        const int wpt = (p.N >= 512 && p.N <= 4096) ? kWarps / (4096 / p.N) : kWarps;
        return ((2 * (p.Lmax + p.Lmax / 16 + 2) + wpt - 1) / wpt + 1) & ~1;
    }
    if (tx) return 2 * scratch_one(p);
    // fused L = 256 runs on half-warps: one buffer per half
    const bool two = (rx_direct && (LU == 0 || LU == 64 || p.Lmax == 64)) || p.Lmax == 256;
    return two ? 2 * scratch_one(p) : scratch_one(p);
}

int stab_len(const Plan& p) { return p.Lmax >= 64 ? p.Lmax : 0; }
// per-lane twiddles of the half-warp FFT_256 (uniform L = 256 kernels)
// The plan runs the kernels that keep their twiddles in TMEM (tmem_tw in fcw_device.cuh).
bool tmem_kernels(const Plan& p) { return FCW_TMEM_TW && p.zv && p.N == 4096 && uniform_L(p) == 256; }
// (those kernels read these twiddles from TMEM instead)
int tw16_len(const Plan& p) {
    if ((FCW_TMEM_TW & 1) && tmem_kernels(p)) return 0;
    return uniform_L(p) == 256 ? 512 : 0;
}

// Independent teams per CTA (must match teams_per_cta<N> in fcw_device.cuh).
int teams(const Plan& p) { return (p.N >= 512 && p.N <= 4096) ? 4096 / p.N : 1; }

size_t smem_bytes(const Plan& p, bool tx, bool rx_direct) {
    const int LU = uniform_L(p);
    const size_t f2 = 2 * (size_t)teams(p) * spec_stride(p, !tx && rx_mirror(p)) +
                      (size_t)kWarps * scratch_stride(p, LU, tx, rx_direct) + stab_len(p) +
                      128 /* two-level long twiddles */ + tw16_len(p) + (teams(p) + 1) / 2 /* run-id slots */;
    return f2 * sizeof(float2);
}

// Persistent launch: as many CTAs as can be resident; each team owns a static
// balanced range of the S*B symbols.  The TX carry buffers are per-launch
// stream-ordered scratch, so concurrent launches never share them.
// Resident CTAs per SM for (kernel, smem, device); sets the dynamic-SMEM
// attribute once.  Cached: the queries cost host time on every launch.
// tmem: the kernel allocates tensor memory (tcgen05.alloc).  The occupancy API
// then reports one CTA per SM whatever the kernel needs, although the SM does
// co-schedule such CTAs while their columns fit (measured: two 128-column CTAs
// overlap on every SM), so the count comes from the register / shared-memory /
// TMEM-column budgets instead.
cudaError_t resident_per_sm(KernelFn k, size_t smem, int dev, int* per_sm, bool tmem = false) {
    static std::mutex mu;
    static std::map<std::pair<std::pair<const void*, size_t>, int>, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(std::make_pair(reinterpret_cast<const void*>(k), smem), dev);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *per_sm = it->second;
        return cudaSuccess;
    }
    // The dynamic-SMEM attribute only ever grows: a plan with less SMEM must
    // not lower it under a cached entry of a plan that needs more (which
    // would then launch with "invalid argument").
    static std::map<std::pair<const void*, int>, size_t> attr_max;
    size_t& amax = attr_max[std::make_pair(reinterpret_cast<const void*>(k), dev)];
    cudaError_t e = cudaSuccess;
    if (smem > amax) {
        e = cudaFuncSetAttribute(reinterpret_cast<const void*>(k), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        amax = smem;
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, reinterpret_cast<const void*>(k), kThreads, smem);
    if (e != cudaSuccess) return e;
    if (tmem && *per_sm >= 1) {
        cudaFuncAttributes fa{};
        int regs_sm = 0, smem_sm = 0, smem_rsv = 0;
        e = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(k));
        if (e != cudaSuccess) return e;
        cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
        const int regs_cta = ((fa.numRegs + 7) & ~7) * kThreads;
        const size_t smem_cta = smem + fa.sharedSizeBytes + (size_t)smem_rsv;
        const int by_regs = regs_cta > 0 ? regs_sm / regs_cta : 1;
        const int by_smem = smem_cta > 0 ? (int)((size_t)smem_sm / smem_cta) : 1;
        *per_sm = std::max(1, std::min({by_regs, by_smem, 512 / kTmemCols}));
    }
    cache[key] = *per_sm;
    return cudaSuccess;
}

cudaError_t launch_one(KernelFn k, size_t smem, KParams& kp, bool tx, int N, int G, cudaStream_t st,
                       bool tmem = false) {
    if (!k) return cudaErrorInvalidValue;
#if FCW_DEV_KNOBS
    // dev-only occupancy probe: extra dynamic SMEM per CTA (e.g. 16384 forces one CTA per SM)
    if (const char* pad = std::getenv("FCW_DEV_SMEM_PAD")) smem += (size_t)std::atoi(pad);
#endif
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = resident_per_sm(k, smem, dev, &per_sm, tmem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    // at most the resident CTAs; in dynamic mode no more teams than runs,
    // in static mode no more teams than symbols
    const long long work = kp.dynamic ? kp.n_items : (long long)kp.n_units * kp.B;
    const int grid = (int)std::max(1LL, std::min((work + G - 1) / G, (long long)per_sm * sms));
    const size_t carry_bytes = tx ? (size_t)grid * G * (N / 2) * sizeof(float2) : 0;
    cudaMemPool_t pool;
    e = scratch_pool(dev, &pool);
    if (e != cudaSuccess) return e;
    void* scratch = nullptr;
    e = cudaMallocFromPoolAsync(&scratch, 256 + carry_bytes, pool, st);
    if (e != cudaSuccess) return e;
    kp.item_counter = static_cast<int*>(scratch);
    kp.carry = tx ? reinterpret_cast<float2*>(static_cast<char*>(scratch) + 256) : nullptr;
    e = kp.dynamic ? cudaMemsetAsync(scratch, 0, sizeof(int), st) : cudaSuccess;
    if (e == cudaSuccess) {
        void* args[] = {&kp};
        e = cudaLaunchKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(kThreads), args, smem, st);
    }
    const cudaError_t f = cudaFreeAsync(scratch, st);
    return e != cudaSuccess ? e : f;
}

}  // namespace

// Per-device stream-ordered pool that keeps freed memory (release threshold
// = max): the per-launch scratch is then a sub-microsecond pool hit instead of
// an OS allocation after every synchronisation.
cudaError_t scratch_pool(int dev, cudaMemPool_t* out) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(dev);
    if (it != pools.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    cudaError_t e = cudaMemPoolCreate(&pool, &props);
    if (e != cudaSuccess) return e;
    uint64_t keep = UINT64_MAX;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if (e != cudaSuccess) return e;
    pools[dev] = pool;
    *out = pool;
    return cudaSuccess;
}

int device_sms() {
    static std::mutex mu;
    static std::map<int, int> sms;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lk(mu);
    auto it = sms.find(dev);
    if (it != sms.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
    sms[dev] = n;
    return n;
}

void fill_common(const Plan& p, KParams& kp) {
    kp.N = p.N;
    kp.B = p.B;
    kp.M = p.M;
    kp.spec_stride = spec_stride(p);
    kp.n_ext = p.n_ext;
    // zv kernels never read the guard band, narrowband kernels only bins [nb_k0, nb_k0 + 16)
    kp.n_zero = (p.zv || p.nb) ? p.n_zero_core : (int)p.h_zero.size();
    kp.nb_k0 = p.nb_k0;
    kp.n_lvl = p.n_lvl;
    kp.n_combo = (int)p.h_combo.size() / 2;
    for (int j = 0; j < kMaxTmemClasses; ++j)
        for (int h = 0; h < 2; ++h) kp.combo[j][h] = j < kp.n_combo ? p.h_combo[2 * j + h] : 0;
    for (int i = 0; i <= kMaxLevels; ++i) kp.lvl_start[i] = i < (int)p.lvl_start.size() ? p.lvl_start[i] : p.n_ext;
    kp.n_groups = p.n_groups;
    for (int g = 0; g < kMaxGroups; ++g) {
        kp.grp_L[g] = p.grp_L[g];
        kp.grp_start[g] = p.grp_start[g];
        kp.grp_count[g] = p.grp_count[g];
    }
    kp.Q = p.Q;
    kp.sub = p.d_sub;
    kp.sym = p.d_sym;
    kp.inv = p.d_inv;
    kp.cls = p.d_cls;
    kp.fix_slot = p.d_fix_slot;
    // uniform-L plans iterate subbands directly (identity group order)
    kp.grp_sub = uniform_L(p) ? nullptr : p.d_grp_sub;
    kp.fix_tgt = p.d_fix;
    kp.own_start = p.d_own_start;
    kp.own_tgt = p.d_own_tgt;
    kp.own_slot = p.d_own_slot;
    kp.zero_list = p.d_zero;
    kp.tw = p.d_tw;
    kp.stab_len = stab_len(p);
    kp.tw16_len = tw16_len(p);
    kp.stage_off = p.Lmax >= 64 ? scratch_one(p) : 0;
#if FCW_DEV_KNOBS
    const char* dbg = std::getenv("FCW_DEBUG_SKIP");
    kp.dbg_skip = dbg ? std::atoi(dbg) : 0;
#else
    kp.dbg_skip = 0;
#endif
}

// 0 general, 2 narrowband, 1 zero-bin, 3 team-only: the kernel family `pick` selects (informational)
bool plan_team_only(const Plan& p) { return team_only(p); }
size_t tx_smem_bytes(const Plan& p) { return smem_bytes(p, true, false); }
size_t rx_smem_bytes(const Plan& p) { return smem_bytes(p, false, true); }

cudaError_t launch_tx(const Plan& p, KParams& kp, int S, cudaStream_t st) {
    const int LU = uniform_L(p);
    kp.scratch_stride = scratch_stride(p, LU, true, false);
    kp.spec_stride = spec_stride(p);
    kp.n_units = S;
    kp.teams = teams(p);
    kp.n_items = S * kp.nchunks;
    const KernelPair kp2 = pick(p.N, LU, p.zv, p.nb, team_only(p));
    return launch_one(kp.dynamic ? kp2.tx_d : kp2.tx, smem_bytes(p, true, false), kp, true, p.N, teams(p), st,
                      tmem_kernels(p));
}

cudaError_t launch_rx(const Plan& p, KParams& kp, int S, cudaStream_t st) {
    const int LU = uniform_L(p);
    const bool direct = !kp.fused;
    kp.scratch_stride = scratch_stride(p, LU, false, direct);
    kp.spec_stride = spec_stride(p, rx_mirror(p));
    kp.n_units = S;
    kp.teams = teams(p);
    kp.n_items = S * kp.nchunks;
    const KernelPair kp2 = pick(p.N, LU, p.zv, p.nb, team_only(p));
    return launch_one(kp.dynamic ? kp2.rx_d : kp2.rx, smem_bytes(p, false, direct), kp, false, p.N, teams(p), st,
                      tmem_kernels(p));
}

// K-GEN: one thread per QAM symbol; splitmix64 is counter-based, so draw j of
// unit u is mix(seed_u + (j+1) * gamma) and every draw is independent
// (channel.cpp:19-48, scenario.cpp:110-128, ofdm.cpp:55-65).
__global__ void gen_qam_kernel(uint64_t seed, long long unit0, int S, long long per_unit, int bits,
                               float2* __restrict__ out) {
    const long long total = (long long)S * per_unit;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long u = idx / per_unit, i = idx - u * per_unit;
        uint64_t s = seed ^ (0x9e3779b97f4a7c15ULL * (uint64_t)(unit0 + u + 1));  // derive_seed
        s += 0x9e3779b97f4a7c15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        uint64_t st = z ^ (z >> 31);
        if (st == 0) st = 0x1234567890abcdefULL;  // GaussianRng ctor (channel.cpp:26)
        unsigned sym = 0;
        const uint64_t base = st + (uint64_t)(i * bits) * 0x9e3779b97f4a7c15ULL;
        for (int b = 0; b < bits; ++b) {
            uint64_t x = base + (uint64_t)(b + 1) * 0x9e3779b97f4a7c15ULL;
            x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
            x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
            x ^= x >> 31;
            sym |= (unsigned)(x & 1u) << b;
        }
        const int k = bits / 2, levels = 1 << k;
        const unsigned mask = (1u << k) - 1u;
        unsigned gi = sym & mask, gq = (sym >> k) & mask, li = 0, lq = 0;
        for (; gi; gi >>= 1) li ^= gi;
        for (; gq; gq >>= 1) lq ^= gq;
        const double sc = 1.0 / sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
        out[idx] = make_float2((float)(sc * (2.0 * li + 1 - levels)), (float)(sc * (2.0 * lq + 1 - levels)));
    }
}

cudaError_t launch_gen_qam(const Plan& p, uint64_t seed, long long unit0, int S, int bits, float2* out,
                           cudaStream_t st) {
    const long long per_unit = (long long)p.B * p.row_active;
    const long long total = per_unit * S;
    int grid = (int)((total + 255) / 256);
    const int cap = device_sms() * 64;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    gen_qam_kernel<<<grid, 256, 0, st>>>(seed, unit0, S, per_unit, bits, out);
    return cudaGetLastError();
}

}  // namespace fcw
