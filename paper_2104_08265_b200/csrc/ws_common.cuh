// Shared device-side definitions for the B200 signal-simulation hot path.
//
// Layout of one "event" launch: up to kMaxPlanes independent planes (each a
// run_simulation-equivalent), their depos concatenated into
// "units" (one unit = one depo on one plane). Plane descriptors travel as a
// kernel parameter (EventDesc) so a launch needs no host->device copy.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "wiresim_gpu.h"
#include "ws_fft.cuh"

namespace wsb {

constexpr int kMaxPlanes = 8;
constexpr int kMaxPasses = 12;
constexpr int kMaxWireWeights = 33;  // 2h+1 <= 33 taps of cross-wire coupling
constexpr int kConvThreads = 256;
constexpr int kTwiddleTable = 512;   // [W_M^j | W_M^{64i} | W_Np^j | W_Np^{64i}], 64 + 192 + 64 + 192
constexpr int kMaxFftHalf = 12288;   // M = N'/2 <= 12288 (N' <= 24576 ticks)
constexpr int kKernPad = 192;        // zero taps either side of PlaneDesc::kern (k_gprof window)
#ifndef WS_TILE_ROWS
#define WS_TILE_ROWS 8
#endif
#ifndef WS_TILE_TICKS
#define WS_TILE_TICKS 2048
#endif
#ifndef WS_SEG_SHIFT
#define WS_SEG_SHIFT 11  // one bound per tile row (r2: 16% fewer bound atomics than 64-tick segments, -4% k_direct)
#endif
constexpr int kTileRows = WS_TILE_ROWS;    // direct path tile: kTileRows wire rows x kTileTicks ticks
constexpr int kTileTicks = WS_TILE_TICKS;
constexpr int kSegShiftD = WS_SEG_SHIFT;   // direct path fixed-point bounds per 64-tick segment
constexpr int kSegs = kTileTicks >> kSegShiftD;
constexpr double kFixScale = 4294967296.0;          // 2^32: fixed-point electrons
constexpr int kRecipN = 16384;                      // reciprocal table of the exact fluctuation walk
constexpr double kFixInv = 1.0 / 4294967296.0;

// Per-unit footprint record written by the sample kernel.
struct __align__(16) UnitRec {
    int32_t w0;    // first wire (padded index) of the clipped footprint; -1 = empty
    int32_t t0;    // first tick (padded index)
    int32_t n_w;   // wires
    int32_t n_t;   // ticks
    uint32_t pool; // pool offset (32-bit words) of the profiles: fluct off [raw | eff | tv] (f32), on [wv | tv] (f64)
    uint32_t goff; // direct-path planes: pool offset of g (16-byte aligned; max|g| at g[-1]); else 0
    float a;       // fluct off: q / total; fluct on: unused
    float tsum;    // fluct off: sum of the tick profile, rounded up (>= its max; bounds fixed-point scales)
};

// One entry of a direct-path tile list (k_fill_bands -> k_direct), 80 bytes.
struct __align__(16) TEnt {
    uint32_t tsL;   // first output tick ts (circular, < N) | profile length L << 16
    uint32_t goff;  // pool offset of g (16-byte aligned)
    uint32_t rows;  // covered tile rows [lo, hi): lo | hi << 8
    float gbound;   // >= max|g| (sum of the tick profile x max|kernel|)
    float c[kTileRows];  // a * eff[w] per tile row (0: not covered)
};

// Device view of one plane for one launch.
struct PlaneDesc {
    // geometry (GridSpec, core.hpp:40-58)
    int32_t W, N;              // padded wires, padded ticks
    int32_t pad_w, pad_t;
    double pitch, tick, origin_x, origin_t;
    double n_sigma;
    // response
    int32_t h;                 // wire-weight half width
    int32_t ww_is_one;         // wire_weights == {1.0}: S' == S
    int32_t folded;            // circular wrap folded from a length-Np linear transform
    int32_t Np, M;             // real FFT length, complex half length
    int32_t lo_lag, hi_lag;    // combined kernel lags
    FftPlanDev fft;            // radix passes of the length-M complex transform
    const double* ww;          // 2h+1 wire weights
    const float2* H;           // M+1 response spectrum bins, pre-scaled by 1/M
    const float2* tw;          // split twiddle tables (kTwiddleTable entries, see ws_api.cu)
    const uint16_t* rev;       // rev[k] = slot of spectrum bin k after the DIF transform
    // time-domain path (ws_direct.cu): per-depo response profiles g = tv (*) kernel
    int32_t direct;            // this call: direct path (tiles, pool holds g) instead of the row FFT (bands)
    int32_t n_lags;            // combined kernel length
    const float* kern;         // n_lags combined-kernel taps (lag lo_lag first), kKernPad zeros either side
    float kern_absmax;         // max |kernel tap| (rounded up)
    int32_t n_windows;         // direct: tick windows of kTileTicks per row band
    uint32_t direct_cap;       // direct: k_direct stages at most this many entries at a time
    // impact positions (ws_plane_create_impacts): the wire pitch is split into
    // `impacts` sub-bins; this plane (class) takes the charge of the sub-bins
    // whose bit is set in imp_mask, normalised over all of them
    int32_t impacts;           // 1 = the reference's wire binning (core.cpp:31-32)
    uint32_t imp_mask;
    int32_t stats_owner;       // counts clipped charge / patches (the first class of a plane only)
    // per call
    const ws_depo* depos;
    uint32_t n_units;
    uint32_t unit_base;        // first unit index of this plane
    uint32_t band_base;        // first bin of this plane (FFT: bands of rows_per_band rows; direct: tiles)
    int32_t rows_per_band;     // FFT bands
    int32_t n_bands;           // bins of this plane in this call
    float* frame;              // out: M (nullable when only the charge grid is wanted)
    double* frame64;           // out: M widened to fp64 (readout, nullable)
    void* adc;                 // out: digitized codes, int32 or uint16 per EventDesc::adc_u16 (readout, nullable)
    float* charge_out;         // out: S (nullable)
    const float* charge_in;    // in: S (mode "grid")
    unsigned long long* charge_cnt;  // fluctuation on: the integer charge grid (mode 1 reads it): u64 counts, or
                                     // u32 counts when the plane's depos carry < 2^32 electrons in all (cnt_wide)
    const unsigned long long* cnt_qsum;  // fluctuation on: the plane's sum of min(q, 2^32), set by k_sample
    long long* stats;          // [0] clipped_charge, [1] clipped_patches
    uint32_t* tile_need;       // fixed tile lists: the largest slot + 1 that did not fit (atomicMax, 0 = none)
};

// The count grid's cell width: a cell never holds more electrons than the
// plane's depos carry in all, so below 2^32 electrons u32 cells are exact (the
// reference's ChargeGrid is int64; half the zeroing and the convolution's reads)
__device__ __forceinline__ bool cnt_wide(const PlaneDesc& P)
{
    return !P.cnt_qsum || *P.cnt_qsum >= (1ull << 32);
}

// A cell of the count grid (u64 or u32 cells)
struct CellPtr {
    unsigned char* p;
    int shift;  // 3: u64 cells, 2: u32
    __device__ __forceinline__ void advance(long long n) { p += n << shift; }
    __device__ __forceinline__ void add(int64_t k) const
    {
        if (k <= 0) return;
        if (shift == 3) atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)k);
        else atomicAdd(reinterpret_cast<unsigned*>(p), (unsigned)k);
    }
};
__device__ __forceinline__ CellPtr cell_at(const PlaneDesc& P, size_t i, bool wide)
{
    CellPtr c;
    c.shift = wide ? 3 : 2;
    c.p = reinterpret_cast<unsigned char*>(P.charge_cnt) + (i << c.shift);
    return c;
}
__device__ __forceinline__ unsigned long long count_at(const PlaneDesc& P, size_t i, bool wide)
{
    return wide ? __ldg(P.charge_cnt + i) : (unsigned long long)__ldg(reinterpret_cast<const unsigned*>(P.charge_cnt) + i);
}

struct EventDesc {
    int32_t n_planes;
    int32_t fluctuate;
    int32_t approx;
    int32_t rng_mode;
    uint64_t seed;
    int32_t drift_enabled;
    int32_t mode;              // conv source: 0 accumulate from band lists, 1 charge grid
    double drift_plane_x, drift_speed, drift_dl, drift_dt;
    uint32_t total_units;
    uint32_t total_bands;
    uint32_t list_cap;         // capacity (entries) of the bin lists; more -> kErrRange, convolution skipped
    // direct planes with fixed-capacity tile lists (fluctuation off): the
    // sampler appends each unit's entries to tiles[b * tile_cap + slot],
    // slot from tile_count[b] (no scan, no k_fill_bands); tile_cap 0 = CSR
    uint32_t tile_cap;
    TEnt* tiles;
    uint32_t* tile_count;
    uint32_t* list_need;       // CSR lists: the entry total when it exceeded list_cap (k_fill_bands)
    unsigned* err;             // the call's error flags
    const double* recip;       // recip[j] = RN(1 / j), j < kRecipN (the exact walk's divisions, ws_sample.cu)
    int32_t fl_quorum;         // exact walk: set up new draws once this many 16ths of the live lanes are idle
    // exact walk, per-bin draw records (k_fluct_prep -> k_fluct_walk, 32 B:
    // ws_sample.cu FlRec), allocated from fl_ctr; more than fl_cap ->
    // kErrFluct: those units take the one-pass walk, the host grows the buffer
    double* fl_bins;
    unsigned long long fl_cap;
    unsigned long long* fl_ctr;
    // readout fused into the frame-store epilogues (add_noise + digitize,
    // spectral.cpp:177-196, 228-238): ro = 0 -> plain fp32 frame stores
    int32_t ro;
    int32_t ro_noise;          // 1: white noise from the Philox stream (seed ^ salt, wire), pair p -> draws 2p, 2p+1
    int32_t adc_u16;           // adc element type: 0 int32 (Matrix<int32_t>), 1 uint16
    double ro_sigma;
    uint64_t ro_seed;
    double adc_scale, adc_offset, adc_max;
    PlaneDesc p[kMaxPlanes];
};

// Error / overflow flags shared by kernels (device scalar words).
enum : unsigned { kErrPool = 1u, kErrDomain = 2u, kErrCharge = 4u, kErrRange = 8u, kErrTileCap = 16u,
                  kErrCellOvf = 32u, kErrFluct = 64u };

__device__ __forceinline__ int band_plane(const EventDesc& ev, uint32_t gb)
{
    int p = 0;
#pragma unroll 1
    for (int i = 1; i < ev.n_planes; ++i)
        if (gb >= ev.p[i].band_base) p = i;
    return p;
}

// Pool layout of a fluctuation-off unit (32-bit words, see k_sample):
//   [raw f32 x n_w][eff f32 x n_eff][tv f32 x n_t][pad][gmax f32][g f32 x L, 0-filled to 32k]
// the last two only on direct-path planes (g 16-byte aligned); L = n_t + n_lags - 1.
__device__ __forceinline__ int unit_n_eff(const PlaneDesc& P, int n_w) { return P.ww_is_one ? 0 : n_w + 2 * P.h; }
__device__ __forceinline__ uint32_t unit_tv_off(const PlaneDesc& P, const UnitRec& r)
{
    return r.pool + (uint32_t)(r.n_w + unit_n_eff(P, r.n_w));
}
// Coefficient of unit `r` on wire row w of the (stencilled unless raw) charge:
// a * profile[j], j = (w - first row) mod W, summed over every wrap that lands
// on the row (a tiny grid can be narrower than the stencilled footprint).
// Returns false when the unit does not cover the row.
__device__ __forceinline__ bool row_coef(const PlaneDesc& P, int w, bool raw, const UnitRec& r,
                                         const uint32_t* __restrict__ pool, float& c)
{
    const int h = P.h;
    const bool stencil = !raw && !P.ww_is_one;
    const int lo_row = stencil ? r.w0 - h : r.w0;
    const int n_rows = stencil ? r.n_w + 2 * h : r.n_w;
    int j = w - lo_row;  // lo_row in [-h, W), w in [0, W)
    if (j < 0) j += P.W;
    else if (j >= P.W) j -= P.W;
    if (j >= P.W) j %= P.W;  // grids narrower than the stencil
    if (j >= n_rows) return false;
    const float* prof = reinterpret_cast<const float*>(pool + r.pool) + (stencil ? r.n_w : 0);
    float s = __ldg(&prof[j]);  // one load in the common case: rows' loads can all be in flight
    if (n_rows > P.W)
        for (j += P.W; j < n_rows; j += P.W) s += __ldg(&prof[j]);
    c = s * r.a;
    return true;
}

// Effective rows [w0 - h, w0 + n_w - 1 + h] of a unit modulo W as up to two ranges.
__device__ __forceinline__ void row_ranges(const PlaneDesc& P, int w0, int n_w, int& a0, int& b0, int& a1, int& b1)
{
    const int W = P.W;
    const int lo = w0 - P.h, hi = w0 + n_w - 1 + P.h;
    a1 = 1;
    b1 = 0;  // empty second range
    if (hi - lo + 1 >= W) {
        a0 = 0;
        b0 = W - 1;
    } else if (lo < 0) {
        a0 = lo + W;
        b0 = W - 1;
        a1 = 0;
        b1 = hi;
    } else if (hi >= W) {
        a0 = lo;
        b0 = W - 1;
        a1 = 0;
        b1 = hi - W;
    } else {
        a0 = lo;
        b0 = hi;
    }
}

// Visit each group of B rows the unit's effective rows touch, exactly once.
template <typename F>
__device__ __forceinline__ void for_each_row_group(const PlaneDesc& P, int w0, int n_w, int B, F&& f)
{
    int a0, b0, a1, b1;
    row_ranges(P, w0, n_w, a0, b0, a1, b1);
    const int c0 = a0 / B, c1 = b0 / B;
    for (int c = c0; c <= c1; ++c) f(c);
    if (a1 <= b1) {
        const int d0 = a1 / B, d1 = b1 / B;
        for (int c = d0; c <= d1; ++c)
            if (c < c0 || c > c1) f(c);
    }
}

// Tick windows (kTileTicks each) touched by the circular output span
// [ts, ts + L) mod N, as a bit mask (N <= 32 windows on direct planes).
__device__ __forceinline__ uint32_t span_windows(int ts, int L, int N, int n_windows)
{
    if (L >= N) return n_windows >= 32 ? 0xffffffffu : ((1u << n_windows) - 1u);
    auto range = [](int a, int b) {  // windows a..b
        const uint32_t hi = b >= 31 ? 0xffffffffu : ((2u << b) - 1u);
        return hi & ~((1u << a) - 1u);
    };
    const int e = ts + L - 1;
    if (e < N) return range(ts / kTileTicks, e / kTileTicks);
    return range(ts / kTileTicks, (N - 1) / kTileTicks) | range(0, (e - N) / kTileTicks);
}

// Visit each bin of the unit exactly once: FFT planes bin by bands of
// rows_per_band rows; direct planes by (16-row band, tick window) tiles,
// tile index = band * n_windows + window.
template <typename F>
__device__ __forceinline__ void for_each_bin(const PlaneDesc& P, int w0, int n_w, int t0, int n_t, F&& f)
{
    if (!P.direct) {
        for_each_row_group(P, w0, n_w, P.rows_per_band, f);
        return;
    }
    int ts = t0 + P.lo_lag;
    if (ts < 0) ts += P.N;
    const uint32_t wm = span_windows(ts, n_t + P.n_lags - 1, P.N, P.n_windows);
    for_each_row_group(P, w0, n_w, kTileRows, [&](int rb) {
        for (uint32_t m = wm; m; m &= m - 1) f(rb * P.n_windows + (__ffs(m) - 1));
    });
}

__device__ __forceinline__ int plane_of_unit(const EventDesc& ev, uint32_t u)
{
    int p = 0;
#pragma unroll 1
    for (int i = 1; i < ev.n_planes; ++i)
        if (u >= ev.p[i].unit_base) p = i;
    return p;
}

// ------------------------------------------------------------------ RNG --
// xoshiro256** / splitmix64, bit-identical to rng.cpp:18-76.
__device__ __forceinline__ uint64_t splitmix64_next(uint64_t& s)
{
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Rng {
    int mode;      // 0 substream (xoshiro), 1 philox
    uint64_t s0, s1, s2, s3;
    uint32_t key0, key1, id0, id1;
    uint32_t draw;
    double spare;
    bool have_spare;

    __device__ void init(int m, uint64_t seed, uint64_t id)
    {
        mode = m;
        have_spare = false;
        spare = 0.0;
        draw = 0;
        if (m == WS_RNG_SUBSTREAM) {
            // substream (rng.cpp:64-76)
            uint64_t sm = seed, tag = id;
            (void)splitmix64_next(tag);
            sm ^= splitmix64_next(tag);
            s0 = splitmix64_next(sm);
            s1 = splitmix64_next(sm);
            s2 = splitmix64_next(sm);
            s3 = splitmix64_next(sm);
            if ((s0 | s1 | s2 | s3) == 0) s0 = 0x9e3779b97f4a7c15ULL;
        } else {
            key0 = (uint32_t)seed;
            key1 = (uint32_t)(seed >> 32);
            id0 = (uint32_t)id;
            id1 = (uint32_t)(id >> 32);
        }
    }

    __device__ __forceinline__ uint64_t next_xoshiro()
    {
        const uint64_t result = rotl64(s1 * 5, 7) * 9;
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = rotl64(s3, 45);
        return result;
    }

    // Philox4x32-10; draw i -> ctr (i>>1, id lo, id hi, 0), words 2(i&1), 2(i&1)+1.
    // philox_block: both draws of block j (draws 2j, 2j + 1).
    __device__ __forceinline__ void philox_block(uint32_t j, uint64_t& w01, uint64_t& w23) const
    {
        uint32_t c0 = j, c1 = id0, c2 = id1, c3 = 0u;
        uint32_t k0 = key0, k1 = key1;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
            const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
            const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
            c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        w01 = (uint64_t)c0 << 32 | c1;
        w23 = (uint64_t)c2 << 32 | c3;
    }
    __device__ __forceinline__ uint64_t next_philox()
    {
        const uint32_t i = draw++;
        uint64_t a, b;
        philox_block(i >> 1, a, b);
        return (i & 1u) ? b : a;
    }

    // uniform01 (rng.cpp:51-54)
    __device__ __forceinline__ double uniform()
    {
        const uint64_t x = mode == WS_RNG_SUBSTREAM ? next_xoshiro() : next_philox();
        return (double)(x >> 11) * 0x1.0p-53;
    }

    // StreamSource::normal (rng.hpp:78-90) + box_muller (rng.cpp:56-62)
    __device__ double normal()
    {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        const double u1 = __dsub_rn(1.0, uniform());
        const double u2 = uniform();
        const double r = sqrt(__dmul_rn(-2.0, log(u1)));
        const double a = __dmul_rn(6.283185307179586476925286766559, u2);
        double sn, cs;
        sincos(a, &sn, &cs);
        spare = __dmul_rn(r, sn);
        have_spare = true;
        return __dmul_rn(r, cs);
    }
};

// exp with a correctly rounded subnormal range. CUDA's exp loses the
// subnormal results that glibc returns (e.g. the lgamma-seeded pmf at
// n*log1p(-p) ~ -744, rng.cpp:152-162); scale into the normal range, then let
// one IEEE multiply round into the subnormal grid.
__device__ __forceinline__ double exp_ref(double x)
{
    if (x >= -708.0) return exp(x);
    const double kLn2Hi = 0x1.62e42fefa3800p-1, kLn2Lo = 0x1.ef35793c7673p-45;
    const double y = exp(__dadd_rn(__dadd_rn(x, 512.0 * kLn2Hi), 512.0 * kLn2Lo));
    return __dmul_rn(y, 0x1p-512);
}

// --------------------------------------------------------------- binomial --
// invert_binomial_cdf (rng.cpp:146-170), operation order kept with explicit
// round-to-nearest intrinsics (no FMA contraction).
__device__ __forceinline__ int64_t invert_binomial_cdf(int64_t n, double p, double u)
{
    const double odds = __ddiv_rn(p, __dsub_rn(1.0, p));
    int64_t k = 0;
    double pmf;
    const double log_pmf0 = __dmul_rn((double)n, log1p(-p));
    if (log_pmf0 > -700.0) {
        pmf = exp_ref(log_pmf0);
    } else {
        const double mean = __dmul_rn((double)n, p);
        const double sd = sqrt(__dmul_rn(mean, __dsub_rn(1.0, p)));
        const int64_t k0 = (int64_t)__dsub_rn(mean, __dmul_rn(30.0, sd));
        k = k0 > 0 ? k0 : 0;
        const double nd = (double)n, kd = (double)k;
        double e = __dsub_rn(lgamma(__dadd_rn(nd, 1.0)), lgamma(__dadd_rn(kd, 1.0)));
        e = __dsub_rn(e, lgamma(__dadd_rn(__dsub_rn(nd, kd), 1.0)));
        e = __dadd_rn(e, __dmul_rn(kd, log(p)));
        e = __dadd_rn(e, __dmul_rn(__dsub_rn(nd, kd), log1p(-p)));
        pmf = exp_ref(e);
    }
    double cdf = pmf;
    while (cdf <= u && k < n) {
        pmf = __dmul_rn(pmf, __ddiv_rn(__dmul_rn(odds, (double)(n - k)), (double)(k + 1)));
        ++k;
        cdf = __dadd_rn(cdf, pmf);
    }
    return k;
}

// binomial (rng.cpp:174-193); p in [0,1] guaranteed by the caller's clamp.
__device__ __forceinline__ int64_t binomial(int64_t n, double p, Rng& src)
{
    if (n == 0 || p == 0.0) return 0;
    if (p == 1.0) return n;
    const double mean = __dmul_rn((double)n, p);
    const double var = __dmul_rn(mean, __dsub_rn(1.0, p));
    const double q1 = __dsub_rn(1.0, p);
    const double mn = (q1 < p) ? q1 : p;
    if (__dmul_rn((double)n, mn) > 1e6) {
        const double k = round(__dadd_rn(mean, __dmul_rn(sqrt(var), src.normal())));
        if (k < 0.0) return 0;
        if (k > (double)n) return n;
        return (int64_t)k;
    }
    const double u = src.uniform();
    if (p > 0.5) return n - invert_binomial_cdf(n, q1, u);
    return invert_binomial_cdf(n, p, u);
}

// fluctuate_approx draw (rasterize.cpp:161-169)
__device__ __forceinline__ int64_t binomial_approx(int64_t n, double p, Rng& src)
{
    if (p <= 0.0) return 0;
    if (p >= 1.0) return n;
    const double mean = __dmul_rn((double)n, p);
    const double k = round(__dadd_rn(mean, __dmul_rn(sqrt(__dmul_rn(mean, __dsub_rn(1.0, p))), src.normal())));
    if (k < 0.0) return 0;
    if (k > (double)n) return n;
    return (int64_t)k;
}

// ---------------------------------------------------------------- readout --
// add_noise (white, spectral.cpp:184-196) + digitize (spectral.cpp:228-238)
// of frame samples, fused into the store epilogue of the convolution kernels
// (or run by ws_noise.cu / k_noise_spectrum after them). Noise is added in
// fp64 to the fp32 sample, as the unfused kernels do, so both give the same
// bits; the ADC code is round(v * scale + offset) clamped to [0, 2^bits - 1].
constexpr uint64_t kWhiteNoiseSalt = 0x77686974656e6f69ULL;  // spectral.cpp:21

struct Sink {  // outputs of one plane's samples (any may be null)
    float* frame;
    double* frame64;
    void* adc;
    int adc_u16;
    double scale, offset, max_code;
};

__device__ __forceinline__ int adc_code(double v, double scale, double offset, double max_code)
{
    const double c = round(__dadd_rn(__dmul_rn(v, scale), offset));
    return (int)(c < 0.0 ? 0.0 : (c > max_code ? max_code : c));
}

__device__ __forceinline__ void sink_put(const Sink& k, size_t i, double v)
{
    if (k.frame) k.frame[i] = (float)v;
    if (k.frame64) k.frame64[i] = v;
    if (k.adc) {
        const int c = adc_code(v, k.scale, k.offset, k.max_code);
        if (k.adc_u16) static_cast<uint16_t*>(k.adc)[i] = (uint16_t)c;
        else static_cast<int32_t*>(k.adc)[i] = c;
    }
}

// White-noise pair p of wire w (Philox): the normals of ticks 2p and 2p+1
__device__ __forceinline__ void white_pair(uint64_t seed, int w, int p, double& n0, double& n1)
{
    Rng src;
    src.init(WS_RNG_PHILOX, seed ^ kWhiteNoiseSalt, (uint64_t)w);
    src.draw = 2u * (uint32_t)p;
    n0 = src.normal();
    n1 = src.normal();  // the cached spare
}

// Readout of samples t, t+1 of row w (t even; has1 false past the row end)
__device__ __forceinline__ void readout_pair(const EventDesc& ev, const PlaneDesc& P, int w, int t, float v0, float v1,
                                             bool has1)
{
    double a = (double)v0, b = (double)v1;
    if (ev.ro_noise) {
        double n0, n1;
        white_pair(ev.ro_seed, w, t >> 1, n0, n1);
        a = __dadd_rn(a, __dmul_rn(ev.ro_sigma, n0));
        b = __dadd_rn(b, __dmul_rn(ev.ro_sigma, n1));
    }
    const Sink k{P.frame, P.frame64, P.adc, ev.adc_u16, ev.adc_scale, ev.adc_offset, ev.adc_max};
    const size_t i = (size_t)w * P.N + t;
    sink_put(k, i, a);
    if (has1) sink_put(k, i + 1, b);
}

// Readout of 4 samples t..t+3 of row w (t a multiple of 4, all in the row;
// the row length a multiple of 4): vector stores
__device__ __forceinline__ void readout4(const EventDesc& ev, const PlaneDesc& P, int w, int t, const float v[4])
{
    double x[4] = {(double)v[0], (double)v[1], (double)v[2], (double)v[3]};
    if (ev.ro_noise) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double n0, n1;
            white_pair(ev.ro_seed, w, (t >> 1) + h, n0, n1);
            x[2 * h] = __dadd_rn(x[2 * h], __dmul_rn(ev.ro_sigma, n0));
            x[2 * h + 1] = __dadd_rn(x[2 * h + 1], __dmul_rn(ev.ro_sigma, n1));
        }
    }
    const size_t i = (size_t)w * P.N + t;
    if (P.frame)
        __stcs(reinterpret_cast<float4*>(P.frame + i), make_float4((float)x[0], (float)x[1], (float)x[2], (float)x[3]));
    if (P.frame64) {
        __stcs(reinterpret_cast<double2*>(P.frame64 + i), make_double2(x[0], x[1]));
        __stcs(reinterpret_cast<double2*>(P.frame64 + i) + 1, make_double2(x[2], x[3]));
    }
    if (P.adc) {
        int c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = adc_code(x[j], ev.adc_scale, ev.adc_offset, ev.adc_max);
        if (ev.adc_u16)
            __stcs(reinterpret_cast<uint2*>(static_cast<uint16_t*>(P.adc) + i),
                   make_uint2((uint32_t)c[0] | ((uint32_t)c[1] << 16), (uint32_t)c[2] | ((uint32_t)c[3] << 16)));
        else
            __stcs(reinterpret_cast<int4*>(static_cast<int32_t*>(P.adc) + i), make_int4(c[0], c[1], c[2], c[3]));
    }
}

// sigproc chain (ws_sigproc.cu): one launch over a batch of signal rows
constexpr int kSpMaxRadices = 32;
struct SigprocDesc {
    const double2* data;        // mode 0: rows x n complex; mode 1: rows x n real
    const double2* filter;      // n complex (mode 0)
    double* block;              // out x n (nullable)
    double* medians;            // out (nullable)
    unsigned long long* stats;  // [max |re|, max |im|] as bit patterns (mode 0)
    const double2* tw;          // per-pass tables: pass f (sub-length L_f) holds exp(+2 pi i j / L_f), j < L_f / R_f
    const int* perm;            // natural output index -> position after the DIF passes
    int n, rows, pad, out, mode, nf;
    double inv_n;
    unsigned long long radix[2];  // pass f's radix = (radix[f >> 4] >> (4 * (f & 15))) & 15
};

}  // namespace wsb
