// C-ABI host layer (include/wiresim_gpu.h): contexts, planes (response
// spectrum + FFT plan precomputed once per geometry), workspace management and
// the launch sequence of one event. No exceptions cross the ABI; no CPU
// fallback exists — every path launches the kernels in ws_sample.cu and
// ws_conv.cu or fails with WS_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <functional>
#include <vector>

#include "ws_common.cuh"
#include "wiresim_gpu.h"

using wsb::EventDesc;
using wsb::PlaneDesc;
using wsb::UnitRec;

extern "C" cudaError_t wsb_launch_sample(const EventDesc& ev, UnitRec* recs, uint32_t* pool, uint32_t pool_cap,
                                         uint32_t* pool_ctr, uint32_t* band_count, unsigned* err, cudaStream_t s,
                                         int pdl);
extern "C" cudaError_t wsb_launch_scan(uint32_t* count, uint32_t* off, uint32_t* fill, uint32_t n, cudaStream_t s);
extern "C" cudaError_t wsb_launch_fill(const EventDesc& ev, const UnitRec* recs, const uint32_t* off, uint32_t* fill,
                                       UnitRec* list, wsb::TEnt* tlist, const uint32_t* pool, unsigned* err,
                                       cudaStream_t s);
extern "C" cudaError_t wsb_launch_gprof(const EventDesc& ev, const UnitRec* recs, uint32_t* pool, cudaStream_t s,
                                        int pdl);
extern "C" cudaError_t wsb_launch_noise(const float* in, const wsb::Sink& out, int W, int N, int noise, int rng_mode,
                                        double sigma, uint64_t seed, cudaStream_t s);
extern "C" cudaError_t wsb_launch_counts_out(const unsigned long long* g, void* out, int type, size_t n, unsigned* err,
                                             const unsigned long long* qsum, cudaStream_t s);
extern "C" cudaError_t wsb_launch_noise_spectrum(const wsb::PlaneDesc& P, const double* amp, uint64_t seed, int rng_mode,
                                                 const float* in, const wsb::Sink& out, int variant,
                                                 cudaStream_t stream);
extern "C" size_t wsb_direct_smem(int cap);
extern "C" int wsb_direct_cap();
extern "C" cudaError_t wsb_launch_direct(const EventDesc& ev, const uint32_t* pool, const uint32_t* band_off,
                                         const wsb::TEnt* tlist, size_t smem_bytes, cudaStream_t stream, int pdl);
extern "C" int wsb_conv_tc_nb(const PlaneDesc& P);
extern "C" cudaError_t wsb_launch_conv_tc(const EventDesc& ev, int nb, cudaStream_t s);
extern "C" cudaError_t wsb_launch_conv_tc2(const EventDesc& ev, cudaStream_t s);
extern "C" size_t wsb_fluct_scratch_bytes(uint32_t n);
extern "C" cudaError_t wsb_launch_zero(void* p, size_t bytes, cudaStream_t s);
extern "C" cudaError_t wsb_launch_zero_counts(void* p, size_t cells, const unsigned long long* qsum, cudaStream_t s);
extern "C" cudaError_t wsb_launch_fluctuate(const EventDesc& ev, const UnitRec* recs, const uint32_t* pool,
                                            const uint32_t* order, void* scratch, cudaStream_t s);
extern "C" size_t wsb_sigproc_smem(int n);
extern "C" int wsb_sigproc_max_n();
extern "C" int wsb_sigproc_dft_max_n();
extern "C" cudaError_t wsb_launch_sigproc(const wsb::SigprocDesc& d, cudaStream_t s);
extern "C" size_t wsb_conv_smem(int N, int Np, int M);
extern "C" cudaError_t wsb_launch_conv(const EventDesc& ev, const uint32_t* pool, const uint32_t* band_off,
                                       const UnitRec* band_list, int flags, size_t smem_bytes, int variant,
                                       cudaStream_t stream);

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define WS_CUDA(call)                                                                            \
    do {                                                                                         \
        const cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                                   \
            return set_err(WS_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                           __LINE__);                                                            \
    } while (0)

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kInvSqrt2 = 0.70710678118654752440084436210485;
constexpr int kStatSlots = 256;  // per-call headers in flight before a drain (a 64-event batch fits)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
    cudaError_t reserve(size_t n)
    {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(n, 1);
        cudaError_t e = cudaMalloc(&p, want * sizeof(T));
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace

// per-call device scratch header: [pool_ctr, err, list_need, pad] u32 + stats
// i64[2*kMaxPlanes] + per-plane tile needs (the sizes a re-run needs after an
// overflow: nothing is ever dropped silently)
struct ScratchHeader {
    uint32_t pool_ctr;
    uint32_t err;
    uint32_t list_need;
    uint32_t pad;
    long long stats[2 * wsb::kMaxPlanes];
    uint32_t tile_need[wsb::kMaxPlanes];
    unsigned long long fl_ctr;  // exact walk: draw records allocated (the need after a kErrFluct)
    unsigned long long qsum[wsb::kMaxPlanes];  // fluctuation on: each plane's electrons (count-grid cell width)
};

struct PendingCall {
    ws_timing* timing;
    int slot;
    int n_planes;
    int direct_planes;
    cudaEvent_t ev[6];
    int fluctuate;
    int tag;                               // caller's tag (ws_simulate_events: event index), -1 none
    uint64_t tiles;                        // fixed-list tiles of the call (bands)
    ws_plane* planes[wsb::kMaxPlanes];     // direct-routed planes (null otherwise)
};

// budget of the fixed-capacity tile lists (bands x capacity x 80 B); above it
// the direct path uses exact-size CSR lists
constexpr size_t kFixedTileBudget = size_t(2) << 30;

struct ws_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint64_t launches = 0;
    DevBuf<UnitRec> recs;
    DevBuf<uint32_t> pool;
    DevBuf<uint32_t> band_count, band_off, band_fill;  // per bin (FFT bands / direct tiles)
    DevBuf<UnitRec> band_list;  // CSR lists of full unit records per FFT band (k_fill_bands)
    DevBuf<wsb::TEnt> tile_list;  // CSR lists of direct-path tile entries (k_fill_bands)
    DevBuf<wsb::TEnt> tile_fixed;  // fixed-capacity tile lists (all-direct events, filled by the sampler)
    uint32_t tile_cap_hint = 2048;  // entries per tile; sized from the real count after a kErrTileCap
    bool csr_next = false;      // next call: CSR tile lists (a fixed capacity would exceed kFixedTileBudget)
    int call_tag = -1;          // tag recorded with the next calls (ws_simulate_events: event index)
    std::vector<int> failed_tags;  // tags of calls that overflowed (re-run by their owner)
    size_t list_hint = 0;       // exact CSR list size after a kErrRange
    uint32_t last_list_cap = 0;
    DevBuf<ScratchHeader> header;
    DevBuf<ws_depo> depos;
    DevBuf<float> frames, charges, ro_scratch;
    DevBuf<unsigned long long> counts;  // fluctuation on: the integer charge grids (u64 counts)
    DevBuf<double> recip;               // RN(1/j), j < kRecipN: the exact walk's divisions
    DevBuf<double> fl_bins;             // exact walk: per-bin draw records (32 B each, ws_sample.cu FlRec)
    DevBuf<unsigned char> fl_scratch;   // exact walk: sort keys / values, offsets, CUB temporaries
    size_t fl_hint = 0;                 // records needed by the last overflowing call
    DevBuf<unsigned char> out_stage;  // ws_run_*: device staging of the readout outputs (ADC / fp64 frames)
    DevBuf<double> noise_amp;  // spectrum-mode amplitudes of the last ws_noise_digitize_device
    ScratchHeader* host_slots = nullptr;  // pinned, kStatSlots
    int next_slot = 0;
    std::vector<PendingCall> pending;
    std::vector<cudaEvent_t> event_pool;
    size_t pool_hint = 0;
    int sm_count = 0;
    int conv_variant = 25;                       // k_conv: 25 (3 CTAs/SM, radix <= 25) or 8 (4 CTAs/SM, radix <= 8)
    int conv_path = WS_CONV_AUTO;                // ws_ctx_set_conv_path
    double direct_kappa = 128.0;                 // AUTO: direct if est. depo-row-taps <= kappa x cells (per plane);
                                                 // r2: direct is 2.3x faster than the row FFT at 1M depos per
                                                 // MicroBooNE plane (ratio 43), so only very long kernels take the FFT
    cudaStream_t copy_stream = nullptr;          // D2H of the pipelined batch path
    cudaStream_t aux_stream = nullptr;           // k_gprof, concurrent with binning
    cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
    cudaEvent_t slot_computed[2] = {nullptr, nullptr};
    cudaEvent_t slot_copied[2] = {nullptr, nullptr};
    cudaEvent_t slot_loaded[2] = {nullptr, nullptr};  // ws_run_events: the slot's depos are on the device
    // sigproc chain: plan of the last row length + staging of the host path
    uint64_t sp_n = 0;
    bool sp_dft = false;  // direct-DFT plan (a prime factor > 13)
    std::vector<int8_t> sp_radix;
    DevBuf<double2> sp_tw, sp_data, sp_filter;
    DevBuf<int> sp_perm;
    DevBuf<double> sp_block, sp_med;
    DevBuf<unsigned long long> sp_stats;
    cudaStream_t h2d_stream = nullptr;
    cudaEvent_t sp_loaded[2] = {nullptr, nullptr}, sp_done[2] = {nullptr, nullptr}, sp_copied[2] = {nullptr, nullptr};
};

struct ws_plane {
    ws_ctx* ctx = nullptr;
    int device = 0;  // the context's device (destroy must not touch the context: it may be gone)
    ws_grid_spec grid{};
    double n_sigma = 3.0;
    int W = 0, N = 0, Np = 0, M = 0, folded = 0, h = 0;
    long lo_lag = 0, n_lags = 0, support_ticks = 0, support_wires = 0;
    std::vector<double> kernel;  // combined time-domain kernel
    std::vector<int> radix;
    wsb::FftPlanDev plan{};
    double* d_ww = nullptr;
    float2* d_H = nullptr;
    float* d_kern = nullptr;  // combined kernel taps (fp32) for the direct path
    float kern_absmax = 0.0f;
    int direct_ok = 0;   // eligible for the time-domain path
    int n_windows = 0;   // direct: tick windows per 16-row band
    float2* d_tw = nullptr;
    uint16_t* d_rev = nullptr;
    int ww_is_one = 0;
    // impact positions (ws_plane_create_impacts): sub-bins per pitch and the
    // impacts of this plane's response class; further classes (distinct
    // responses) are child planes run alongside this one into the same frame
    int impacts = 1;
    uint32_t imp_mask = 1u;
    std::vector<ws_plane*> classes;
    int rows_per_band = 4;
    int n_bands = 0;
    size_t smem = 0;
};

namespace {

cudaEvent_t take_event(ws_ctx* c)
{
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// ---------------------------------------------------------------- response --
// Host restatement of the response builder's time-domain kernel
// (spectral.cpp:34-83 field/shaper samples, :98-113 combination and supports),
// with the same validation (:89-92, :117-121). The frequency-domain values are
// produced below for the row transform instead of a 2D fft_2d (:137).

double gauss_pdf(double t, double sigma)
{
    const double z = t / sigma;
    return std::exp(-0.5 * z * z) / (sigma * std::sqrt(kTwoPi));
}

void bin_integrals(double center, double sigma, double lo_edge, double spacing, size_t n, double* vals)
{
    for (size_t i = 0; i < n; ++i) vals[i] = 0.0;
    if (n == 0) return;
    if (sigma <= 0.0) {
        long idx = (long)std::floor((center - lo_edge) / spacing);
        idx = std::clamp<long>(idx, 0, (long)n - 1);
        vals[idx] = 1.0;
        return;
    }
    const double inv = kInvSqrt2 / sigma;
    double prev = std::erf((lo_edge - center) * inv);
    for (size_t i = 0; i < n; ++i) {
        const double next = std::erf((lo_edge + (double)(i + 1) * spacing - center) * inv);
        vals[i] = 0.5 * (next - prev);
        prev = next;
    }
}

int build_kernel(const ws_grid_spec& g, const ws_response& r, std::vector<double>& combined, long& lo_lag,
                 long& support_ticks, long& support_wires)
{
    if (r.shaper_order < 1) return set_err(WS_EINVAL, "build_response: shaper_order must be >= 1");
    if (!r.wire_weights || r.n_wire_weights == 0 || r.n_wire_weights % 2 == 0)
        return set_err(WS_EINVAL, "build_response: wire_weights must have odd length");
    const double tick = g.tick;
    std::vector<double> f;
    long half = 0;
    if (r.field_sigma_t <= 0.0) {
        f = {1.0};
    } else {
        const double sigma = r.field_sigma_t;
        half = (long)std::ceil(8.0 * sigma / tick);
        const size_t n = (size_t)(2 * half + 1);
        f.assign(n, 0.0);
        if (r.plane_kind == WS_COLLECTION) {
            bin_integrals(0.0, sigma, (-(double)half - 0.5) * tick, tick, n, f.data());
            double sum = 0.0;
            for (double v : f) sum += v;
            for (double& v : f) v /= sum;
        } else {
            double pos = 0.0;
            for (size_t i = 0; i < n; ++i) {
                const double lo = ((double)i - (double)half - 0.5) * tick;
                f[i] = gauss_pdf(lo + tick, sigma) - gauss_pdf(lo, sigma);
                if (f[i] > 0.0) pos += f[i];
            }
            for (double& v : f) v /= pos;
        }
    }
    std::vector<double> s;
    if (r.shaper_peaking <= 0.0) {
        s = {1.0};
    } else {
        const double tau = r.shaper_peaking;
        const int order = r.shaper_order;
        for (long k = 0;; ++k) {
            const double t = (double)k * tick;
            const double z = t / tau;
            const double v = std::pow(z, order) * std::exp(-(double)order * (z - 1.0));
            s.push_back(v);
            if (t > tau && v < 1e-14) break;
            if (k > 2000000) return set_err(WS_ERUNTIME, "build_response: shaper tail does not decay");
        }
    }
    double shaper_sum = 0.0;
    for (double v : s) shaper_sum += v;
    const double amplitude = r.gain / shaper_sum;
    const size_t n_lags = f.size() + s.size() - 1;
    combined.assign(n_lags, 0.0);
    for (size_t i = 0; i < f.size(); ++i)
        for (size_t j = 0; j < s.size(); ++j) combined[i + j] += f[i] * s[j] * amplitude;
    lo_lag = -half;
    support_ticks = std::max<long>(-lo_lag, lo_lag + (long)n_lags - 1);
    support_wires = (long)(r.n_wire_weights / 2);
    const uint64_t W = g.n_wires + 2 * g.pad_wires, N = g.n_ticks + 2 * g.pad_ticks;
    if (n_lags > N)
        return set_err(WS_EINVAL, "build_response: kernel time support %zu exceeds the padded tick count %llu", n_lags,
                       (unsigned long long)N);
    if (r.n_wire_weights > W) return set_err(WS_EINVAL, "build_response: wire_weights exceed the padded wire count");
    return WS_OK;
}

bool smooth7(long n)
{
    if (n < 1) return false;
    for (long p : {2L, 3L, 5L, 7L})
        while (n % p == 0) n /= p;
    return n == 1;
}

// Pass plan for the length-m complex transform: the factorisation into
// in-register radices with the fewest shared-memory passes, then the smallest
// largest radix (register pressure), searched exhaustively (m is 7-smooth).
// Radix sets instantiated by the two k_conv variants (ws_conv.cu). The DIF
// pass order puts odd radices last: the final DIF pass (and the first DIT
// pass) has unit stride, where an odd radix keeps the shared-memory accesses
// free of bank conflicts.
const std::vector<int> kRadix25 = {25, 24, 20, 16, 14, 10, 8, 7, 5, 4, 3, 2};
const std::vector<int> kRadix8 = {8, 7, 5, 4, 3, 2};

std::vector<int> plan_radices(int m, const std::vector<int>& kRadices)
{
    std::vector<int> best, cur;
    std::function<void(int)> dfs = [&](int rem) {
        if (rem == 1) {
            const int mx = cur.empty() ? 0 : *std::max_element(cur.begin(), cur.end());
            const int bmx = best.empty() ? 1 << 30 : *std::max_element(best.begin(), best.end());
            if (best.empty() || cur.size() < best.size() || (cur.size() == best.size() && mx < bmx)) best = cur;
            return;
        }
        if (!best.empty() && cur.size() + 1 > best.size()) return;
        for (int r : kRadices)
            if (rem % r == 0 && (cur.empty() || r <= cur.back())) {  // non-increasing: one order per multiset
                cur.push_back(r);
                dfs(rem / r);
                cur.pop_back();
            }
    };
    dfs(m);
    std::stable_sort(best.begin(), best.end(), [](int a, int b) { return (a & 1) < (b & 1); });  // odd last
    return best;
}

int validate_grid(const ws_grid_spec* g)
{
    if (!g) return set_err(WS_EINVAL, "GridSpec: null");
    if (g->n_wires < 1 || g->n_ticks < 1) return set_err(WS_EINVAL, "GridSpec: active grid must be at least 1x1");
    if (!(g->pitch > 0.0)) return set_err(WS_EINVAL, "GridSpec: pitch must be > 0");
    if (!(g->tick > 0.0)) return set_err(WS_EINVAL, "GridSpec: tick must be > 0");
    const uint64_t W = g->n_wires + 2 * g->pad_wires, N = g->n_ticks + 2 * g->pad_ticks;
    if (W > (1u << 30) || N > (1u << 30)) return set_err(WS_EINVAL, "GridSpec: padded grid too large");
    return WS_OK;
}

PlaneDesc plane_desc(const ws_plane* p)
{
    PlaneDesc d{};
    d.W = p->W;
    d.N = p->N;
    d.pad_w = (int)p->grid.pad_wires;
    d.pad_t = (int)p->grid.pad_ticks;
    d.pitch = p->grid.pitch;
    d.tick = p->grid.tick;
    d.origin_x = p->grid.origin_x;
    d.origin_t = p->grid.origin_t;
    d.n_sigma = p->n_sigma;
    d.h = p->h;
    d.ww_is_one = p->ww_is_one;
    d.folded = p->folded;
    d.Np = p->Np;
    d.M = p->M;
    d.lo_lag = (int)p->lo_lag;
    d.hi_lag = (int)(p->lo_lag + p->n_lags - 1);
    d.fft = p->plan;
    d.ww = p->d_ww;
    d.H = p->d_H;
    d.tw = p->d_tw;
    d.rev = p->d_rev;
    d.rows_per_band = p->rows_per_band;
    d.n_lags = (int)p->n_lags;
    d.kern = p->d_kern ? p->d_kern + wsb::kKernPad : nullptr;
    d.kern_absmax = p->kern_absmax;
    d.direct = 0;  // decided per call (run_group)
    d.impacts = p->impacts;
    d.imp_mask = p->imp_mask;
    d.stats_owner = 1;
    d.n_windows = p->n_windows;
    d.direct_cap = (uint32_t)wsb_direct_cap();
    d.n_bands = p->n_bands;
    return d;
}

int check_opts(const ws_sim_options* o)
{
    if (!o) return set_err(WS_EINVAL, "options: null");
    if (o->rng_mode != WS_RNG_SUBSTREAM && o->rng_mode != WS_RNG_PHILOX)
        return set_err(WS_EINVAL, "options: unknown rng mode %d", o->rng_mode);
    if (o->drift.enabled && !(o->drift.drift_speed > 0.0))
        return set_err(WS_EINVAL, "drift_depo: drift_speed must be > 0");
    if (o->charge_type != WS_CHARGE_F32 && o->charge_type != WS_CHARGE_U32 && o->charge_type != WS_CHARGE_I64)
        return set_err(WS_EINVAL, "options: unknown charge type %d", o->charge_type);
    return WS_OK;
}

// Launch one group of <= kMaxPlanes planes. frames/charges are device
// pointers (frames[i] may be null when only charge is wanted).
int finish_pending(ws_ctx* c);

// Readout of a call (run_simulation's add_noise + digitize, pipeline.cpp:420-423)
struct Readout {
    const ws_readout* spec;  // noise model, ADC config, output types
    void* const* adc;        // per plane (nullable entries)
    double* const* frame64;  // per plane (nullable entries)
};

// The noise runs fused in the frame-store epilogues unless it needs a
// sequential per-wire stream (white noise, substream) or its own row IFFT
// (spectrum mode): those run as a second kernel over the fp32 frame.
bool readout_fused(const ws_readout* r)
{
    return r->noise.mode == WS_NOISE_OFF || (r->noise.mode == WS_NOISE_WHITE && r->noise.rng_mode == WS_RNG_PHILOX) ||
           (r->noise.mode == WS_NOISE_WHITE && r->noise.sigma == 0.0);
}

// charges: per plane (nullable array / entries): fluctuation off, the float32
// charge grid S (an extra accumulate pass); fluctuation on, the caller's copy
// of the integer counts in opt->charge_type. counts: fluctuation on, the
// device count grids of the walk (u64, required).
int run_group(ws_ctx* c, uint32_t n, ws_plane* const* planes, const ws_depo* const* depos, const uint64_t* n_depos,
              const ws_sim_options* opt, float* const* frames, float* const* charges, const float* const* charge_in,
              ws_timing* timing, const Readout* ro = nullptr, unsigned long long* const* counts = nullptr)
{
    cudaStream_t s = c->stream;
    EventDesc ev{};
    // the readout is fused into the frame stores of the fluctuation-off
    // kernels; behind a given grid's convolution (k_conv_tc2: four epilogue
    // warps per SM) the fp64 noise math would run at a fraction of the GPU,
    // so that path writes the fp32 frame and the full-GPU pair kernel follows
    const bool grid_conv = charge_in != nullptr || (opt && opt->fluctuate);
    const bool ro_fused = ro && readout_fused(ro->spec) && !grid_conv;
    if (ro_fused) {
        const ws_readout& r = *ro->spec;
        ev.ro = 1;
        ev.ro_noise = r.noise.mode == WS_NOISE_WHITE && r.noise.sigma != 0.0 ? 1 : 0;
        ev.ro_sigma = r.noise.sigma;
        ev.ro_seed = r.noise.seed;
        ev.adc_u16 = r.adc_type == WS_ADC_U16 ? 1 : 0;
        ev.adc_scale = r.adc.scale;
        ev.adc_offset = r.adc.offset;
        ev.adc_max = (double)((1 << r.adc.bits) - 1);
    }
    // an unfused readout noise kernel reads an fp32 frame: the caller's, or scratch
    std::vector<float*> fr32(n, nullptr);
    if (ro && !ro_fused) {
        size_t need = 0;
        for (uint32_t i = 0; i < n; ++i)
            if (!(frames && frames[i])) need += (size_t)planes[i]->W * planes[i]->N;
        WS_CUDA(c->ro_scratch.reserve(need));
        size_t off = 0;
        for (uint32_t i = 0; i < n; ++i) {
            if (frames && frames[i]) {
                fr32[i] = frames[i];
            } else {
                fr32[i] = c->ro_scratch.p + off;
                off += (size_t)planes[i]->W * planes[i]->N;
            }
        }
    }
    ev.n_planes = (int)n;
    ev.fluctuate = opt ? opt->fluctuate : 0;
    ev.approx = opt ? opt->approx : 0;
    ev.rng_mode = opt ? opt->rng_mode : 0;
    ev.seed = opt ? opt->seed : 0;
    ev.drift_enabled = opt ? opt->drift.enabled : 0;
    if (ev.drift_enabled) {
        ev.drift_plane_x = opt->drift.response_plane_x;
        ev.drift_speed = opt->drift.drift_speed;
        ev.drift_dl = opt->drift.diffusion_long;
        ev.drift_dt = opt->drift.diffusion_tran;
    }
    const bool from_grid = charge_in != nullptr;
    ev.mode = (from_grid || ev.fluctuate) ? 1 : 0;
    uint32_t units = 0, bands = 0;
    size_t smem = 0;
    bool want_frame = false, any_direct = false, any_fft = false;
    int max_lags = 0;
    // plane descriptors of the launch: one per plane, plus one per further
    // response class of a plane with impact positions (same depos, tiles and
    // frame; its own response), right after its plane
    uint32_t nd = 0;
    std::vector<uint32_t> desc_of(n);
    std::vector<ws_plane*> desc_plane;
    for (uint32_t i = 0; i < n; ++i) {
        ws_plane* p = planes[i];
        PlaneDesc d = plane_desc(p);
        d.depos = depos ? depos[i] : nullptr;
        d.n_units = depos ? (uint32_t)n_depos[i] : 0u;
        d.unit_base = units;
        d.band_base = bands;
        d.frame = (ro && !ro_fused) ? fr32[i] : (frames ? frames[i] : nullptr);
        if (ro_fused) {
            d.frame64 = ro->frame64 ? ro->frame64[i] : nullptr;
            d.adc = ro->adc ? ro->adc[i] : nullptr;
        }
        // fluctuation on: the walk's integer grid
        d.charge_cnt = (ev.fluctuate && !from_grid) ? counts[i] : nullptr;
        d.charge_out = (charges && !ev.fluctuate) ? charges[i] : nullptr;
        d.charge_in = from_grid ? charge_in[i] : nullptr;
        d.stats = nullptr;
        const bool has_out = d.frame || d.frame64 || d.adc;
        // time-domain path for fluctuation-off frames (not with a charge
        // grid request: that pass bins by FFT bands). AUTO estimates the
        // work as depos x ~12 wire rows x profile taps against the plane's
        // cells (ws_ctx_set_direct_kappa).
        // (A tile list that overflowed - a local density far above the plane
        // average, e.g. a shower - is re-run on the same kernel with the grown
        // lists, so a call's result never depends on the workspace's history.)
        const bool classes = !p->classes.empty();
        if (classes) {
            // distinct per-impact responses: the classes' profiles are summed
            // in k_direct's tiles (the sum over impacts fused into the
            // time-domain convolution)
            if (ev.mode != 0 || d.charge_out)
                return set_err(WS_EINVAL, "impact planes with distinct responses: fluctuation, charge-grid input and "
                                          "charge output are not supported");
            if (c->conv_path == WS_CONV_FFT)
                return set_err(WS_EINVAL, "impact planes with distinct responses run on the time-domain path only");
        }
        if (ev.mode == 0 && has_out && !d.charge_out && p->direct_ok && c->conv_path != WS_CONV_FFT) {
            const double work = (double)d.n_units * 12.0 * (double)(p->n_lags + 16);
            if (classes || c->conv_path == WS_CONV_DIRECT || work <= c->direct_kappa * (double)p->W * (double)p->Np) {
                d.direct = 1;
                d.n_bands = ((p->W + wsb::kTileRows - 1) / wsb::kTileRows) * p->n_windows;
                any_direct = true;
                max_lags = std::max(max_lags, (int)p->n_lags);
            }
        }
        if (nd + 1 + p->classes.size() > (size_t)wsb::kMaxPlanes)
            return set_err(WS_EINVAL, "launch group: more than %d plane descriptors", wsb::kMaxPlanes);
        any_fft = any_fft || !d.direct;
        desc_of[i] = nd;
        desc_plane.push_back(classes ? nullptr : p);
        ev.p[nd++] = d;
        units += d.n_units;
        bands += (uint32_t)d.n_bands;
        smem = std::max(smem, p->smem);
        want_frame = want_frame || has_out;
        for (ws_plane* cp : p->classes) {
            PlaneDesc e = plane_desc(cp);
            e.depos = d.depos;
            e.n_units = d.n_units;
            e.unit_base = units;
            e.band_base = d.band_base;  // the plane's tiles
            e.n_bands = 0;
            e.frame = d.frame;
            e.frame64 = d.frame64;
            e.adc = d.adc;
            e.direct = 1;
            e.stats_owner = 0;
            max_lags = std::max(max_lags, (int)cp->n_lags);
            desc_plane.push_back(nullptr);
            ev.p[nd++] = e;
            units += e.n_units;
        }
    }
    ev.n_planes = (int)nd;
    ev.total_units = units;
    ev.total_bands = bands;

    // workspace
    const size_t pool_need = std::max<size_t>(c->pool_hint, (size_t)units * (96 + (any_direct ? max_lags + 40 : 0)) + 4096);
    WS_CUDA(c->recs.reserve(units));
    WS_CUDA(c->pool.reserve(pool_need));
    {
        // the counts are zeroed by their consumer (k_scan_bands / k_direct)
        // for the next call; a fresh allocation is zeroed here
        const size_t cap0 = c->band_count.cap;
        WS_CUDA(c->band_count.reserve(bands + 1));
        if (c->band_count.cap != cap0)
            WS_CUDA(cudaMemsetAsync(c->band_count.p, 0, sizeof(uint32_t) * c->band_count.cap, s));
    }
    WS_CUDA(c->band_off.reserve(bands + 1));
    WS_CUDA(c->band_fill.reserve(bands + 1));
    int max_h = 0;
    for (uint32_t i = 0; i < nd; ++i) max_h = std::max(max_h, ev.p[i].h);
    // bin lists: ~4.5 entries per unit for 4-row FFT bands, ~2 per unit for
    // 16 x 2048 tiles at typical widths; overflow is detected on the device
    const size_t list_cap = std::min<size_t>(std::max<size_t>(c->list_hint, (size_t)units * (8 + max_h) + 4096),
                                             0xffffffffu);
    ev.list_cap = (uint32_t)list_cap;
    c->last_list_cap = (uint32_t)list_cap;
    if (any_fft) WS_CUDA(c->band_list.reserve(list_cap));
    // all-direct fluctuation-off events: the sampler fills fixed-capacity tile
    // lists (no count scan, no k_fill_bands); WS_TILE_CSR=1 forces the CSR path
    static const bool csr_only = [] {
        const char* v = getenv("WS_TILE_CSR");
        return v && v[0] == '1';
    }();
    const bool fixed_fits = (size_t)bands * c->tile_cap_hint * sizeof(wsb::TEnt) <= kFixedTileBudget;
    const bool use_fixed = any_direct && !any_fft && ev.mode == 0 && !ev.fluctuate && !csr_only && bands > 0 &&
                           want_frame && fixed_fits && !c->csr_next;
    c->csr_next = false;
    ev.tile_cap = 0;
    ev.tiles = nullptr;
    ev.tile_count = c->band_count.p;
    if (use_fixed) {
        WS_CUDA(c->tile_fixed.reserve((size_t)bands * c->tile_cap_hint));
        ev.tile_cap = c->tile_cap_hint;
        ev.tiles = c->tile_fixed.p;
    } else if (any_direct) {
        WS_CUDA(c->tile_list.reserve(list_cap));
    }
    // per-call header in a device ring (zeroed when allocated and after each
    // read-back), copied to the host at synchronize: no per-call memset / D2H
    if (!c->header.p) {
        WS_CUDA(c->header.reserve(kStatSlots));
        WS_CUDA(cudaMemsetAsync(c->header.p, 0, sizeof(ScratchHeader) * kStatSlots, s));
    }
    if ((int)c->pending.size() >= kStatSlots) {
        // ring full: drain (reads and re-zeroes the slots). Inside a batch
        // (tagged calls) an overflow of an earlier event is re-run by the
        // batch at its end; this call still goes ahead.
        const int rc = finish_pending(c);
        if (rc && !(rc == WS_ERANGE && c->call_tag >= 0)) return rc;
    }
    const int slot = c->next_slot;
    c->next_slot = (c->next_slot + 1) % kStatSlots;
    ScratchHeader* hdr = c->header.p + slot;
    for (uint32_t i = 0; i < nd; ++i) {
        ev.p[i].stats = &hdr->stats[2 * i];
        ev.p[i].tile_need = &hdr->tile_need[i];
        ev.p[i].cnt_qsum = ev.p[i].charge_cnt ? &hdr->qsum[i] : nullptr;
    }
    ev.list_need = &hdr->list_need;
    ev.err = &hdr->err;

    PendingCall pc{};
    pc.timing = timing;
    pc.n_planes = (int)nd;
    pc.tag = c->call_tag;
    pc.tiles = bands;
    uint32_t direct_units = 0;  // units on direct planes: the profiles kernel runs iff > 0
    for (uint32_t i = 0; i < nd; ++i) {
        pc.direct_planes += ev.p[i].direct && ev.p[i].stats_owner;
        pc.planes[i] = ev.p[i].direct ? desc_plane[i] : nullptr;
        if (ev.p[i].direct) direct_units += ev.p[i].n_units;
    }
    pc.fluctuate = ev.fluctuate;
    if (timing)
        for (int k = 0; k < 6; ++k) pc.ev[k] = take_event(c);

    if (timing) WS_CUDA(cudaEventRecord(pc.ev[0], s));  // stage timing only

    if (!from_grid) {
        WS_CUDA(wsb_launch_sample(ev, c->recs.p, c->pool.p, (uint32_t)std::min<size_t>(c->pool.cap, 0xffffffffu),
                                  &hdr->pool_ctr, c->band_count.p, &hdr->err, s, timing ? 0 : 1));
        c->launches += units ? 1 : 0;
    }
    // the count grids at the cell width the sampler's electron sums chose (u32
    // below 2^32 electrons per plane), zeroed on the SMs
    if (ev.fluctuate && !from_grid)
        for (uint32_t i = 0; i < nd; ++i)
            if (ev.p[i].charge_cnt) {
                WS_CUDA(wsb_launch_zero_counts(ev.p[i].charge_cnt, (size_t)ev.p[i].W * ev.p[i].N, ev.p[i].cnt_qsum, s));
                c->launches += 1;
            }
    if (timing) WS_CUDA(cudaEventRecord(pc.ev[1], s));  // stage timing only
    if (ev.fluctuate && !from_grid) {
        if (!c->recip.p) {
            std::vector<double> r(wsb::kRecipN);
            r[0] = 0.0;
            for (int j = 1; j < wsb::kRecipN; ++j) r[j] = 1.0 / (double)j;  // IEEE division: RN(1/j)
            WS_CUDA(c->recip.reserve(r.size()));
            WS_CUDA(cudaMemcpy(c->recip.p, r.data(), sizeof(double) * r.size(), cudaMemcpyHostToDevice));
        }
        ev.recip = c->recip.p;
        static const int quorum = [] {
            const char* v = getenv("WS_FLUCT_QUORUM");  // tuning only
            return v ? std::max(1, std::min(16, atoi(v))) : 6;  // (r2 sweeps: 6 best with 7 steps and one settled draw per pass)
        }();
        ev.fl_quorum = quorum;
        if (!ev.approx) {
            // one record per drawn bin; the need is known after an overflow
            const size_t recs_need = std::max<size_t>(c->fl_hint, (size_t)units * 160 + 4096);
            WS_CUDA(c->fl_bins.reserve(4 * recs_need));  // 32-byte records
            ev.fl_bins = c->fl_bins.p;
            ev.fl_cap = c->fl_bins.cap / 4;
            ev.fl_ctr = &hdr->fl_ctr;
        }
        void* scratch = nullptr;
        if (!ev.approx && units) {
            WS_CUDA(c->fl_scratch.reserve(wsb_fluct_scratch_bytes(units)));
            scratch = c->fl_scratch.p;
        }
        WS_CUDA(wsb_launch_fluctuate(ev, c->recs.p, c->pool.p, nullptr, scratch, s));
        c->launches += units ? (ev.approx ? 1 : 7) : 0;  // exact: 4 scheduling-sort kernels, records, walk, normal-branch units
    }
    if (timing) WS_CUDA(cudaEventRecord(pc.ev[2], s));  // stage timing only
    if (ev.mode == 0) {
        if (any_direct && ev.tile_cap) {
            // fixed tile lists: the binning happened in the sampler, the
            // profiles are all that is left before k_direct (same stream)
            WS_CUDA(wsb_launch_gprof(ev, c->recs.p, c->pool.p, s, timing ? 0 : 1));  // programmatic after the sampler
            c->launches += units ? 1 : 0;
        } else if (any_direct) {
            // response profiles on the auxiliary stream, concurrent with the
            // binning (k_direct is the first consumer)
            if (!c->aux_stream) {
                // lowest priority: the binning's blocks (main stream) go first
                // whenever both kernels have blocks waiting
                int lo_prio = 0, hi_prio = 0;
                WS_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
                WS_CUDA(cudaStreamCreateWithPriority(&c->aux_stream, cudaStreamNonBlocking, lo_prio));
                WS_CUDA(cudaEventCreateWithFlags(&c->aux_fork, cudaEventDisableTiming));
                WS_CUDA(cudaEventCreateWithFlags(&c->aux_join, cudaEventDisableTiming));
            }
            WS_CUDA(cudaEventRecord(c->aux_fork, s));
            WS_CUDA(cudaStreamWaitEvent(c->aux_stream, c->aux_fork, 0));
            WS_CUDA(wsb_launch_gprof(ev, c->recs.p, c->pool.p, c->aux_stream, 0));
            WS_CUDA(cudaEventRecord(c->aux_join, c->aux_stream));
            c->launches += units ? 1 : 0;
        }
        if (!ev.tile_cap) {  // CSR lists: scan the counts, then append
            WS_CUDA(wsb_launch_scan(c->band_count.p, c->band_off.p, c->band_fill.p, bands, s));
            WS_CUDA(wsb_launch_fill(ev, c->recs.p, c->band_off.p, c->band_fill.p, c->band_list.p,
                                    c->tile_list.p, c->pool.p, &hdr->err, s));
            c->launches += 1 + (units ? 1 : 0);
        }
        if (any_direct && !ev.tile_cap)
            WS_CUDA(cudaStreamWaitEvent(s, c->aux_join, 0));  // profiles ready (bin stage ends)
    }
    if (timing) WS_CUDA(cudaEventRecord(pc.ev[3], s));  // stage timing only
    if (ev.mode == 0 && charges) {
        // the charge grid is the un-stencilled S: an accumulate-only pass of
        // the row kernel over every band (parity / inspection output)
        WS_CUDA(wsb_launch_conv(ev, c->pool.p, c->band_off.p, c->band_list.p, 2, smem, c->conv_variant, s));
        c->launches += bands ? 1 : 0;
    }
    if (want_frame) {
        // each kernel skips the other's planes
        if (any_direct) {
            // programmatic launch after the profiles kernel on the same stream
            // (fixed tile lists, no charge pass in between). Only when the
            // profiles kernel was launched in this call: otherwise the
            // predecessor could be the previous call's k_direct, which
            // releases its dependents at its start, before it has consumed
            // (and zeroed) the tile counts this launch reads.
            const int pdl = ev.tile_cap != 0 && !(ev.mode == 0 && charges) && direct_units > 0 ? 1 : 0;
            WS_CUDA(wsb_launch_direct(ev, c->pool.p, c->band_off.p, c->tile_list.p, wsb_direct_smem(wsb_direct_cap()),
                                      s, pdl));
            c->launches += bands ? 1 : 0;
        }
        if (any_fft) {
            // a given grid (fluctuation counts / ws_convolve_device): the
            // tensor-core direct convolution when every plane is eligible,
            // else the row FFT
            int nb = 0;
            cudaError_t te = cudaErrorNotSupported;
            if (ev.mode == 1) {
                te = wsb_launch_conv_tc2(ev, s);  // the pipelined kernel, where every plane is eligible
                if (te == cudaErrorNotSupported) {
                    (void)cudaGetLastError();
                    nb = 4;
                    for (uint32_t i = 0; i < nd && nb; ++i)
                        if (!ev.p[i].direct) nb = std::min(nb, wsb_conv_tc_nb(ev.p[i]));
                    te = nb ? wsb_launch_conv_tc(ev, nb, s) : cudaErrorNotSupported;
                }
            }
            if (te == cudaErrorNotSupported) {
                (void)cudaGetLastError();
                te = wsb_launch_conv(ev, c->pool.p, c->band_off.p, c->band_list.p, 1, smem, c->conv_variant, s);
            }
            WS_CUDA(te);
            c->launches += bands ? 1 : 0;
        }
    }
    if (ro && !ro_fused) {
        // readout with a sequential per-wire stream or a spectrum: its own
        // kernel over the fp32 frame (in place), then digitize
        const ws_readout& r = *ro->spec;
        for (uint32_t i = 0; i < n; ++i) {
            const PlaneDesc& d = ev.p[desc_of[i]];
            const wsb::Sink sk{frames && frames[i] ? frames[i] : nullptr, ro->frame64 ? ro->frame64[i] : nullptr,
                               ro->adc ? ro->adc[i] : nullptr, r.adc_type == WS_ADC_U16 ? 1 : 0, r.adc.scale,
                               r.adc.offset, (double)((1 << r.adc.bits) - 1)};
            if (r.noise.mode == WS_NOISE_SPECTRUM) {
                WS_CUDA(c->noise_amp.reserve((size_t)d.N));
                WS_CUDA(cudaMemcpyAsync(c->noise_amp.p, r.noise.amplitude_spectrum, sizeof(double) * d.N,
                                        cudaMemcpyHostToDevice, s));
                WS_CUDA(wsb_launch_noise_spectrum(d, c->noise_amp.p, r.noise.seed, r.noise.rng_mode, d.frame, sk,
                                                  c->conv_variant, s));
            } else {
                const int noisy = r.noise.mode == WS_NOISE_WHITE && r.noise.sigma != 0.0 ? 1 : 0;  // else digitize only
                WS_CUDA(wsb_launch_noise(d.frame, sk, d.W, d.N, noisy, r.noise.rng_mode, r.noise.sigma, r.noise.seed, s));
            }
            c->launches += 1;
        }
    }
    if (ev.fluctuate && !from_grid && charges)
        for (uint32_t i = 0; i < n; ++i) {  // the caller's charge output: the counts in its type
            const PlaneDesc& d = ev.p[desc_of[i]];
            if (!charges[i]) continue;
            WS_CUDA(wsb_launch_counts_out(d.charge_cnt, charges[i], opt->charge_type, (size_t)d.W * d.N, &hdr->err,
                                          d.cnt_qsum, s));
            c->launches += 1;
        }
    if (timing) WS_CUDA(cudaEventRecord(pc.ev[4], s));  // stage timing only
    pc.slot = slot;
    if (timing) WS_CUDA(cudaEventRecord(pc.ev[5], s));  // stage timing only
    c->pending.push_back(pc);
    return WS_OK;
}

int finish_pending(ws_ctx* c)
{
    WS_CUDA(cudaStreamSynchronize(c->stream));
    if (!c->pending.empty()) {
        // the ring's headers of the pending calls -> host, then zero them for reuse
        WS_CUDA(cudaMemcpy(c->host_slots, c->header.p, sizeof(ScratchHeader) * kStatSlots, cudaMemcpyDeviceToHost));
        for (const PendingCall& pc : c->pending)
            WS_CUDA(cudaMemsetAsync(c->header.p + pc.slot, 0, sizeof(ScratchHeader), c->stream));
    }
    // Every call's status is evaluated (the first error is returned): an
    // overflow never yields WS_OK. The workspace is sized from the real needs
    // the device recorded, so a single re-run fits; tagged calls that
    // overflowed are listed for their owner (ws_simulate_events) to re-run.
    int rc = WS_OK;
    for (PendingCall& pc : c->pending) {
        const ScratchHeader& h = c->host_slots[pc.slot];
        int prc = WS_OK;
        char msg[256] = {0};
        if (h.err & wsb::kErrDomain) {
            prc = WS_EDOMAIN;
            snprintf(msg, sizeof msg, "drift_depo: a depo is behind the response plane");
        } else if (h.err & wsb::kErrCharge) {
            prc = WS_EINVAL;
            snprintf(msg, sizeof msg, "fluctuate: charge must be >= 0");
        } else if (h.err & wsb::kErrCellOvf) {
            prc = WS_ERUNTIME;  // (not retried)
            snprintf(msg, sizeof msg, "charge output: a cell exceeds 4294967295 electrons (uint32 charge type; "
                                      "use int64)");
        }
        if (h.err & wsb::kErrPool) {
            c->pool_hint = std::max<size_t>(c->pool_hint, (size_t)h.pool_ctr + 4096);
            if (!prc) {
                prc = WS_ERANGE;
                snprintf(msg, sizeof msg, "workspace: patch pool overflow (%u words needed); grown, re-run the call",
                         h.pool_ctr);
            }
        }
        // fluctuation records beyond the buffer: those units took the one-pass
        // walk (complete result); the next call gets room for all of them
        if (h.err & wsb::kErrFluct) c->fl_hint = std::max<size_t>(c->fl_hint, (size_t)h.fl_ctr + 4096);
        if (h.err & wsb::kErrTileCap) {
            // the real per-tile counts: size the fixed lists from them, or
            // (beyond the budget) take exact-size CSR lists
            uint32_t need = 0;
            for (int i = 0; i < pc.n_planes; ++i) need = std::max(need, h.tile_need[i]);
            uint32_t cap = c->tile_cap_hint;
            while (cap < need && cap < (1u << 30)) cap *= 2;
            // past the fixed-list budget the calls take exact-size CSR lists
            // from now on (fixed_fits is false for the grown hint)
            c->tile_cap_hint = cap;
            if ((size_t)pc.tiles * cap * sizeof(wsb::TEnt) > kFixedTileBudget) c->csr_next = true;
            if (!prc) {
                prc = WS_ERANGE;
                snprintf(msg, sizeof msg,
                         "workspace: tile list overflow (%u entries in one tile, capacity %u); grown, re-run the call",
                         need, c->tile_cap_hint);
            }
        }
        if (h.err & wsb::kErrRange) {
            c->list_hint = std::max<size_t>(c->list_hint, (size_t)h.list_need + 4096);
            if (!prc) {
                prc = WS_ERANGE;
                snprintf(msg, sizeof msg, "workspace: bin lists overflow (%u entries, capacity %u); grown, re-run the call",
                         h.list_need, c->last_list_cap);
            }
        }
        if (prc == WS_ERANGE && pc.tag >= 0) c->failed_tags.push_back(pc.tag);
        if (prc && rc == WS_OK) rc = set_err(prc, "%s", msg);
        if (pc.timing) {
            ws_timing& t = *pc.timing;
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pc.ev[0], pc.ev[1]);
            t.prepare_ms = ms;
            cudaEventElapsedTime(&ms, pc.ev[1], pc.ev[2]);
            t.fluctuate_ms = ms;
            cudaEventElapsedTime(&ms, pc.ev[2], pc.ev[3]);
            t.bin_ms = ms;
            cudaEventElapsedTime(&ms, pc.ev[3], pc.ev[4]);
            t.convolve_ms = ms;
            cudaEventElapsedTime(&ms, pc.ev[0], pc.ev[4]);
            t.total_ms = ms;
            t.clipped_charge = 0;
            t.clipped_patches = 0;
            t.direct_planes = pc.direct_planes;
            for (int i = 0; i < pc.n_planes; ++i) {
                t.clipped_charge += h.stats[2 * i];
                t.clipped_patches += h.stats[2 * i + 1];
            }
        }
        if (pc.timing)
            for (int k = 0; k < 6; ++k) c->event_pool.push_back(pc.ev[k]);
    }
    c->pending.clear();
    return rc;
}

int check_plane_set(ws_ctx* ctx, uint32_t n, ws_plane* const* planes)
{
    if (!ctx) return set_err(WS_EINVAL, "null context");
    if (n == 0) return WS_OK;
    if (!planes) return set_err(WS_EINVAL, "null plane array");
    for (uint32_t i = 0; i < n; ++i)
        if (!planes[i] || planes[i]->ctx != ctx) return set_err(WS_EINVAL, "plane %u does not belong to the context", i);
    return WS_OK;
}

}  // namespace

extern "C" {

const char* ws_last_error(void) { return g_err.c_str(); }
int ws_set_error_message(int code, const char* msg) { return set_err(code, "%s", msg); }
int ws_abi_version(void) { return WS_ABI_VERSION; }

int ws_ctx_create(int device, void* stream, ws_ctx** out)
{
    if (!out) return set_err(WS_EINVAL, "null out pointer");
    *out = nullptr;
    int n = 0;
    WS_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return set_err(WS_ECUDA, "device %d not present (%d devices)", device, n);
    cudaDeviceProp prop{};
    WS_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) return set_err(WS_ECUDA, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);
    WS_CUDA(cudaSetDevice(device));
    ws_ctx* c = new ws_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    if (const char* e = getenv("WS_CONV_VARIANT")) c->conv_variant = atoi(e) == 8 ? 8 : 25;
    if (const char* e = getenv("WS_DIRECT_KAPPA")) c->direct_kappa = atof(e);
    if (stream) {
        c->stream = (cudaStream_t)stream;
    } else {
        // highest priority: within a call, its blocks win over the auxiliary
        // stream's (k_gprof) whenever both have blocks waiting
        int lo_prio = 0, hi_prio = 0;
        cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
        cudaError_t e = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi_prio);
        if (e != cudaSuccess) {
            delete c;
            return set_err(WS_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
        }
        c->own_stream = true;
    }
    cudaError_t e = cudaMallocHost(&c->host_slots, sizeof(ScratchHeader) * kStatSlots);
    if (e != cudaSuccess) {
        delete c;
        return set_err(WS_ECUDA, "cudaMallocHost: %s", cudaGetErrorString(e));
    }
    *out = c;
    return WS_OK;
}

int ws_ctx_destroy(ws_ctx* c)
{
    if (!c) return WS_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->recs.release();
    c->pool.release();
    c->band_count.release();
    c->band_off.release();
    c->band_fill.release();

    c->band_list.release();
    c->tile_list.release();
    c->tile_fixed.release();
    c->header.release();
    c->depos.release();
    c->frames.release();
    c->charges.release();
    c->counts.release();
    c->recip.release();
    c->fl_bins.release();
    c->fl_scratch.release();
    c->ro_scratch.release();
    c->out_stage.release();
    c->noise_amp.release();
    for (PendingCall& pc : c->pending)
        for (cudaEvent_t e : pc.ev) cudaEventDestroy(e);
    for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
    if (c->host_slots) cudaFreeHost(c->host_slots);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    if (c->aux_stream) {
        cudaStreamSynchronize(c->aux_stream);
        cudaStreamDestroy(c->aux_stream);
    }
    if (c->aux_fork) cudaEventDestroy(c->aux_fork);
    if (c->aux_join) cudaEventDestroy(c->aux_join);
    for (int s = 0; s < 2; ++s) {
        if (c->slot_computed[s]) cudaEventDestroy(c->slot_computed[s]);
        if (c->slot_loaded[s]) cudaEventDestroy(c->slot_loaded[s]);
        if (c->slot_copied[s]) cudaEventDestroy(c->slot_copied[s]);
    }
    c->sp_tw.release();
    c->sp_data.release();
    c->sp_filter.release();
    c->sp_perm.release();
    c->sp_block.release();
    c->sp_med.release();
    c->sp_stats.release();
    if (c->h2d_stream) {
        cudaStreamSynchronize(c->h2d_stream);
        cudaStreamDestroy(c->h2d_stream);
    }
    for (int s = 0; s < 2; ++s)
        for (cudaEvent_t e : {c->sp_loaded[s], c->sp_done[s], c->sp_copied[s]})
            if (e) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    (void)cudaGetLastError();  // nothing of this teardown may surface in a later launch check
    return WS_OK;
}

int ws_ctx_synchronize(ws_ctx* c)
{
    if (!c) return set_err(WS_EINVAL, "null context");
    WS_CUDA(cudaSetDevice(c->device));
    return finish_pending(c);
}

void* ws_ctx_stream(ws_ctx* c) { return c ? (void*)c->stream : nullptr; }

int ws_ctx_set_conv_path(ws_ctx* c, int path)
{
    if (!c) return set_err(WS_EINVAL, "null context");
    if (path != WS_CONV_AUTO && path != WS_CONV_FFT && path != WS_CONV_DIRECT)
        return set_err(WS_EINVAL, "unknown convolution path %d", path);
    c->conv_path = path;
    return WS_OK;
}

int ws_ctx_set_direct_kappa(ws_ctx* c, double kappa)
{
    if (!c) return set_err(WS_EINVAL, "null context");
    if (!(kappa >= 0.0)) return set_err(WS_EINVAL, "direct-path threshold must be >= 0");
    c->direct_kappa = kappa;
    return WS_OK;
}
uint64_t ws_ctx_launch_count(const ws_ctx* c) { return c ? c->launches : 0; }

}  // extern "C"

namespace {
int plane_create(ws_ctx* ctx, const ws_grid_spec* grid, const ws_response* response, double n_sigma, ws_plane** out);
}

extern "C" {

int ws_plane_create(ws_ctx* ctx, const ws_grid_spec* grid, const ws_response* response, double n_sigma, ws_plane** out)
{
    return plane_create(ctx, grid, response, n_sigma, out);
}

static bool same_response(const ws_response& a, const ws_response& b)
{
    if (a.plane_kind != b.plane_kind || a.shaper_order != b.shaper_order || a.field_sigma_t != b.field_sigma_t ||
        a.shaper_peaking != b.shaper_peaking || a.gain != b.gain || a.n_wire_weights != b.n_wire_weights)
        return false;
    for (uint64_t i = 0; i < a.n_wire_weights; ++i)
        if (a.wire_weights[i] != b.wire_weights[i]) return false;
    return true;
}

int ws_plane_create_impacts(ws_ctx* ctx, const ws_grid_spec* grid, const ws_response* responses,
                            uint32_t impacts_per_pitch, double n_sigma, ws_plane** out)
{
    if (!ctx || !out || !responses) return set_err(WS_EINVAL, "null argument");
    *out = nullptr;
    if (impacts_per_pitch < 1 || impacts_per_pitch > 32)
        return set_err(WS_EINVAL, "impacts_per_pitch must be in [1, 32] (got %u)", impacts_per_pitch);
    for (uint32_t i = 0; i < impacts_per_pitch; ++i)
        if (!responses[i].wire_weights) return set_err(WS_EINVAL, "impact %u: null wire_weights", i);
    // response classes: impacts with identical responses share one
    std::vector<uint32_t> masks;
    std::vector<uint32_t> first;
    for (uint32_t i = 0; i < impacts_per_pitch; ++i) {
        size_t c = 0;
        while (c < first.size() && !same_response(responses[first[c]], responses[i])) ++c;
        if (c == first.size()) {
            first.push_back(i);
            masks.push_back(0u);
        }
        masks[c] |= 1u << i;
    }
    if (masks.size() > (size_t)wsb::kMaxPlanes)
        return set_err(WS_EINVAL, "at most %d distinct impact responses per plane (got %zu)", wsb::kMaxPlanes,
                       masks.size());
    std::vector<ws_plane*> made;
    for (size_t c = 0; c < masks.size(); ++c) {
        ws_plane* p = nullptr;
        if (int rc = plane_create(ctx, grid, &responses[first[c]], n_sigma, &p)) {
            for (ws_plane* q : made) ws_plane_destroy(q);
            return rc;
        }
        p->impacts = (int)impacts_per_pitch;
        p->imp_mask = masks[c];
        made.push_back(p);
        if (masks.size() > 1 && !p->direct_ok) {
            for (ws_plane* q : made) ws_plane_destroy(q);
            return set_err(WS_EINVAL, "impact responses: distinct per-impact responses run on the time-domain path, "
                                      "which this geometry / kernel length does not support");
        }
    }
    for (size_t c = 1; c < made.size(); ++c) made[0]->classes.push_back(made[c]);
    *out = made[0];
    return WS_OK;
}

}  // extern "C"

namespace {

int plane_create(ws_ctx* ctx, const ws_grid_spec* grid, const ws_response* response, double n_sigma, ws_plane** out)
{
    if (!ctx || !out || !response) return set_err(WS_EINVAL, "null argument");
    *out = nullptr;
    if (int rc = validate_grid(grid)) return rc;
    if (!(n_sigma > 0.0)) return set_err(WS_EINVAL, "map_depo_to_grid: n_sigma must be > 0");
    WS_CUDA(cudaSetDevice(ctx->device));
    ws_plane* p = new ws_plane();
    p->ctx = ctx;
    p->device = ctx->device;
    p->grid = *grid;
    p->n_sigma = n_sigma;
    p->W = (int)(grid->n_wires + 2 * grid->pad_wires);
    p->N = (int)(grid->n_ticks + 2 * grid->pad_ticks);
    if (int rc = build_kernel(*grid, *response, p->kernel, p->lo_lag, p->support_ticks, p->support_wires)) {
        delete p;
        return rc;
    }
    p->n_lags = (long)p->kernel.size();
    // convolve's wrap check (spectral.cpp:147-153)
    if (p->support_ticks > (long)grid->pad_ticks || p->support_wires > (long)grid->pad_wires) {
        const int rc = set_err(WS_EINVAL,
                               "convolve: kernel support (%ld wires, %ld ticks) exceeds the padding; pad_wires >= %ld "
                               "and pad_ticks >= %ld required",
                               p->support_wires, p->support_ticks, p->support_wires, p->support_ticks);
        delete p;
        return rc;
    }
    if ((int)response->n_wire_weights > wsb::kMaxWireWeights) {
        delete p;
        return set_err(WS_EINVAL, "wire_weights: at most %d taps supported", wsb::kMaxWireWeights);
    }
    p->h = (int)(response->n_wire_weights / 2);
    p->ww_is_one = (response->n_wire_weights == 1 && response->wire_weights[0] == 1.0) ? 1 : 0;
    // transform length: the padded tick count itself when it is even and
    // 7-smooth (exact circular convolution), else the smallest even 7-smooth
    // length holding the linear convolution, whose tails are folded back
    // (same circular result).
    if (p->N % 2 == 0 && smooth7(p->N)) {
        p->Np = p->N;
        p->folded = 0;
    } else {
        long L = p->N + p->n_lags - 1;
        if (L % 2) ++L;
        while (!smooth7(L)) L += 2;
        p->Np = (int)L;
        p->folded = 1;
    }
    p->M = p->Np / 2;
    if (p->M > wsb::kMaxFftHalf) {
        delete p;
        return set_err(WS_EINVAL, "padded_ticks %d needs a %d-point transform; at most %d supported", p->N, p->Np,
                       2 * wsb::kMaxFftHalf);
    }
    p->radix = plan_radices(p->M, ctx->conv_variant == 8 ? kRadix8 : kRadix25);
    if (p->radix.empty()) {
        delete p;
        return set_err(WS_EINVAL, "no radix plan for a %d-point transform", p->M);
    }
    if ((int)p->radix.size() > wsb::kMaxPasses) {
        delete p;
        return set_err(WS_EINVAL, "transform plan too deep");
    }
    // response spectrum H[k] = (1/M) sum_lag c_lag exp(-2 pi i k lag / Np), k <= M
    const int Np = p->Np, M = p->M;
    std::vector<double> cs(Np), sn(Np);
    for (int m = 0; m < Np; ++m) {
        const double a = -kTwoPi * (double)m / (double)Np;
        cs[m] = std::cos(a);
        sn[m] = std::sin(a);
    }
    // DIF / DIT pass plan (ws_fft.cuh), the digit-reversal map of the DIF
    // output, and the split twiddle tables [W_M^j | W_M^{64 i} | W_Np^j | W_Np^{64 i}]
    std::vector<float2> tw(wsb::kTwiddleTable);
    std::vector<uint16_t> rev(M);
    {
        wsb::FftPlanDev& pl = p->plan;
        pl = wsb::FftPlanDev{};
        const int P = (int)p->radix.size();
        pl.npass = P;
        auto magic = [](int d) { return d > 1 ? (uint32_t)((0x100000000ULL + d - 1) / d) : 0u; };
        int L = M;
        for (int i = 0; i < P; ++i) {  // DIF pass i: length L, stride S = L / R
            const int R = p->radix[i];
            pl.radix[i] = R;
            pl.dif_s[i] = L / R;
            pl.dif_mg[i] = magic(L / R);
            pl.dif_step[i] = M / L;
            L /= R;
        }
        int lam = 1;
        for (int i = 0; i < P; ++i) {  // DIT pass i runs radix[P-1-i]
            const int R = p->radix[P - 1 - i];
            pl.dit_lam[i] = lam;
            pl.dit_mg[i] = magic(lam);
            pl.dit_step[i] = M / (lam * R);
            lam *= R;
        }
        for (int k = 0; k < M; ++k) {  // pos(k) = sum_p q_p M / (R_0..R_p), k = sum_p q_p R_0..R_{p-1}
            long pos = 0, div = 1, len = M;
            for (int i = 0; i < P; ++i) {
                const int R = p->radix[i];
                len /= R;
                pos += ((k / div) % R) * len;
                div *= R;
            }
            rev[k] = (uint16_t)pos;
        }
        auto put = [&](int at, long idx) { tw[at] = make_float2((float)cs[idx % Np], (float)sn[idx % Np]); };
        for (int j = 0; j < 64; ++j) put(j, 2L * j);                 // W_M^j   (W_M = W_Np^2)
        for (int i = 0; i < 192; ++i) put(64 + i, 2L * 64 * i);      // W_M^{64 i}
        for (int j = 0; j < 64; ++j) put(256 + j, j);                // W_Np^j
        for (int i = 0; i < 192; ++i) put(320 + i, 64L * i);         // W_Np^{64 i}
    }
    std::vector<float2> H(M + 1);
    for (int k = 0; k <= M; ++k) {
        double re = 0.0, im = 0.0;
        for (long i = 0; i < p->n_lags; ++i) {
            long lag = (p->lo_lag + i) % Np;
            if (lag < 0) lag += Np;
            const long idx = (long)(((long long)k * lag) % Np);
            re += p->kernel[i] * cs[idx];
            im += p->kernel[i] * sn[idx];
        }
        H[k] = make_float2((float)(re / M), (float)(im / M));
    }
    std::vector<double> ww(response->wire_weights, response->wire_weights + response->n_wire_weights);
    cudaError_t e = cudaSuccess;
    e = e ? e : cudaMalloc(&p->d_H, sizeof(float2) * (M + 1));
    e = e ? e : cudaMalloc(&p->d_tw, sizeof(float2) * tw.size());
    e = e ? e : cudaMalloc(&p->d_ww, sizeof(double) * ww.size());
    e = e ? e : cudaMemcpy(p->d_H, H.data(), sizeof(float2) * (M + 1), cudaMemcpyHostToDevice);
    e = e ? e : cudaMemcpy(p->d_tw, tw.data(), sizeof(float2) * tw.size(), cudaMemcpyHostToDevice);
    e = e ? e : cudaMemcpy(p->d_ww, ww.data(), sizeof(double) * ww.size(), cudaMemcpyHostToDevice);
    e = e ? e : cudaMalloc(&p->d_rev, sizeof(uint16_t) * M);
    e = e ? e : cudaMemcpy(p->d_rev, rev.data(), sizeof(uint16_t) * M, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        ws_plane_destroy(p);
        return set_err(WS_ECUDA, "plane upload: %s", cudaGetErrorString(e));
    }
    p->n_bands = (p->W + p->rows_per_band - 1) / p->rows_per_band;
    p->smem = wsb_conv_smem(p->N, p->Np, p->M);
    // time-domain path: kernel taps on the device; eligible while a band's
    // fixed-point rows fit in shared memory and the kernel is not huge
    p->n_windows = (p->N + wsb::kTileTicks - 1) / wsb::kTileTicks;
    if (p->n_windows <= 32 && p->n_lags <= 4096 && p->N < 65536) {
        double km = 0.0;
        for (double v : p->kernel) km = std::max(km, std::fabs(v));
        p->kern_absmax = std::nextafter((float)km, INFINITY) * (1.0f + 1e-6f);  // fp32 taps x tv sums stay below
        std::vector<float> kf(p->kernel.size() + 2 * wsb::kKernPad, 0.0f);
        std::copy(p->kernel.begin(), p->kernel.end(), kf.begin() + wsb::kKernPad);
        e = cudaMalloc(&p->d_kern, sizeof(float) * kf.size());
        e = e ? e : cudaMemcpy(p->d_kern, kf.data(), sizeof(float) * kf.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            ws_plane_destroy(p);
            return set_err(WS_ECUDA, "plane upload: %s", cudaGetErrorString(e));
        }
        p->direct_ok = 1;
    }
    if (p->smem > 227 * 1024) {
        ws_plane_destroy(p);
        return set_err(WS_EINVAL, "padded_ticks too large for the shared-memory row transform");
    }
    *out = p;
    return WS_OK;
}

}  // namespace

extern "C" {

int ws_plane_destroy(ws_plane* p)
{
    if (!p) return WS_OK;
    for (ws_plane* c : p->classes) ws_plane_destroy(c);
    cudaSetDevice(p->device);
    if (p->d_H) cudaFree(p->d_H);
    if (p->d_kern) cudaFree(p->d_kern);
    if (p->d_tw) cudaFree(p->d_tw);
    if (p->d_rev) cudaFree(p->d_rev);
    if (p->d_ww) cudaFree(p->d_ww);
    delete p;
    (void)cudaGetLastError();  // nothing of this teardown may surface in a later launch check
    return WS_OK;
}

int ws_plane_get_info(const ws_plane* p, ws_plane_info* info)
{
    if (!p || !info) return set_err(WS_EINVAL, "null argument");
    info->padded_wires = (uint64_t)p->W;
    info->padded_ticks = (uint64_t)p->N;
    info->fft_length = (uint64_t)p->Np;
    info->folded = p->folded;
    info->n_radix_passes = (int32_t)p->radix.size();
    info->support_ticks = p->support_ticks;
    info->support_wires = p->support_wires;
    info->lo_lag = p->lo_lag;
    info->n_lags = p->n_lags;
    info->impacts_per_pitch = p->impacts;
    info->n_response_classes = 1 + (int32_t)p->classes.size();
    return WS_OK;
}

int ws_plane_get_kernel(const ws_plane* p, double* out, uint64_t cap)
{
    if (!p || !out) return set_err(WS_EINVAL, "null argument");
    if (cap < p->kernel.size()) return set_err(WS_ERANGE, "kernel has %zu lags", p->kernel.size());
    std::copy(p->kernel.begin(), p->kernel.end(), out);
    return WS_OK;
}

}  // extern "C"

namespace {

constexpr int kMaxAttempts = 6;  // host paths: re-runs after a workspace overflow (one normally suffices)

int check_readout(const ws_readout* r, uint32_t n_planes, ws_plane* const* planes)
{
    if (!r) return WS_OK;
    const ws_noise_model& m = r->noise;
    if (m.mode != WS_NOISE_OFF && m.mode != WS_NOISE_WHITE && m.mode != WS_NOISE_SPECTRUM)
        return set_err(WS_EINVAL, "add_noise: unknown noise mode %d", m.mode);
    if (m.mode != WS_NOISE_OFF && m.rng_mode != WS_RNG_SUBSTREAM && m.rng_mode != WS_RNG_PHILOX)
        return set_err(WS_EINVAL, "add_noise: unknown rng mode %d", m.rng_mode);
    if (m.sigma < 0.0) return set_err(WS_EINVAL, "add_noise: sigma must be >= 0");
    if (r->adc.bits < 1 || r->adc.bits > 16) return set_err(WS_EINVAL, "digitize: bits must be in [1,16]");
    if (r->frame_type != WS_FRAME_F32 && r->frame_type != WS_FRAME_F64)
        return set_err(WS_EINVAL, "readout: unknown frame type %d", r->frame_type);
    if (r->adc_type != WS_ADC_I32 && r->adc_type != WS_ADC_U16)
        return set_err(WS_EINVAL, "readout: unknown adc type %d", r->adc_type);
    if (m.mode == WS_NOISE_SPECTRUM)
        for (uint32_t i = 0; i < n_planes; ++i) {
            if (!m.amplitude_spectrum || m.n_amplitude != (uint64_t)planes[i]->N)
                return set_err(WS_EINVAL,
                               "add_noise: amplitude_spectrum length %llu does not match the padded tick count %d",
                               (unsigned long long)m.n_amplitude, planes[i]->N);
            if (planes[i]->folded)
                return set_err(WS_EINVAL,
                               "add_noise: spectrum mode needs an even 7-smooth padded tick count (got %d)",
                               planes[i]->N);
        }
    return WS_OK;
}

size_t frame_elem(const ws_readout* r) { return r && r->frame_type == WS_FRAME_F64 ? 8 : 4; }
size_t adc_elem(const ws_readout* r) { return r && r->adc_type == WS_ADC_U16 ? 2 : 4; }

// One event (any number of planes, in launch groups of kMaxPlanes), device
// pointers, asynchronous. frames[i]: fp32 (ro == null or an fp32 readout) or
// fp64 (fp64 readout); adcs[i]: readout codes; charges[i] (nullable array):
// the caller's charge grids (float32 on return).
int event_device(ws_ctx* ctx, uint32_t n_planes, ws_plane* const* planes, const ws_depo* const* depos,
                 const uint64_t* n_depos, const ws_sim_options* opt, const ws_readout* spec, void* const* frames,
                 void* const* adcs, float* const* charges, ws_timing* timing)
{
    std::vector<float*> ch(n_planes, nullptr);
    std::vector<unsigned long long*> cnt(n_planes, nullptr);
    bool user_charge = false;
    if (charges)
        for (uint32_t i = 0; i < n_planes; ++i) {
            ch[i] = charges[i];
            user_charge = user_charge || charges[i];
        }
    if (opt->fluctuate) {
        // the walk's integer grids (u64 counts, internal; copied out in the
        // caller's charge type when asked)
        size_t total = 0;
        for (uint32_t i = 0; i < n_planes; ++i) total += (size_t)planes[i]->W * planes[i]->N;
        WS_CUDA(ctx->counts.reserve(total));
        size_t off = 0;
        for (uint32_t i = 0; i < n_planes; ++i) {
            cnt[i] = ctx->counts.p + off;
            off += (size_t)planes[i]->W * planes[i]->N;
        }
    }
    const bool f64 = spec && spec->frame_type == WS_FRAME_F64;
    std::vector<float*> fr(n_planes, nullptr);
    std::vector<double*> fr64(n_planes, nullptr);
    std::vector<void*> ad(n_planes, nullptr);
    for (uint32_t i = 0; i < n_planes; ++i) {
        void* f = frames ? frames[i] : nullptr;
        if (f64) fr64[i] = static_cast<double*>(f);
        else fr[i] = static_cast<float*>(f);
        ad[i] = adcs ? adcs[i] : nullptr;
    }
    for (uint32_t g = 0, n = 0; g < n_planes; g += n) {
        // launch groups of at most kMaxPlanes plane descriptors (a plane with
        // impact positions takes one per response class)
        uint32_t slots = 0;
        for (n = 0; g + n < n_planes; ++n) {
            const uint32_t k = 1u + (uint32_t)planes[g + n]->classes.size();
            if (n && slots + k > (uint32_t)wsb::kMaxPlanes) break;
            slots += k;
        }
        const Readout ro{spec, ad.data() + g, fr64.data() + g};
        bool any_charge = false;
        for (uint32_t i = g; i < g + n; ++i) any_charge = any_charge || ch[i];
        const int rc = run_group(ctx, n, planes + g, depos + g, n_depos + g, opt, fr.data() + g,
                                 any_charge ? ch.data() + g : nullptr, nullptr, g == 0 ? timing : nullptr,
                                 spec ? &ro : nullptr, opt->fluctuate ? cnt.data() + g : nullptr);
        if (rc) return rc;
    }
    return WS_OK;
}

// Host buffers: events pipelined over two device slots (event e computes
// while event e-1's outputs stream back on the copy stream). Calls whose
// workspace overflowed are re-run (the device recorded the sizes they need),
// at most kMaxAttempts times; an overflow never returns WS_OK.
// frames / adcs / charges: [n_events * n_planes] host pointers (arrays and
// entries nullable).
int events_host(ws_ctx* ctx, uint32_t n_events, uint32_t n_planes, ws_plane* const* planes,
                const ws_depo* const* depos, const uint64_t* n_depos, const ws_sim_options* opt,
                const ws_readout* spec, void* const* frames, void* const* adcs, float* const* charges,
                ws_timing* timing)
{
    if (int rc = check_plane_set(ctx, n_planes, planes)) return rc;
    if (int rc = check_opts(opt)) return rc;
    if (int rc = check_readout(spec, n_planes, planes)) return rc;
    if (n_events == 0 || n_planes == 0) return WS_OK;
    if (!depos || !n_depos) return set_err(WS_EINVAL, "null argument");
    WS_CUDA(cudaSetDevice(ctx->device));
    if (int rc = finish_pending(ctx)) return rc;
    if (!ctx->copy_stream) WS_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    if (!ctx->h2d_stream) WS_CUDA(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
    for (int s = 0; s < 2; ++s) {
        if (!ctx->slot_computed[s]) WS_CUDA(cudaEventCreateWithFlags(&ctx->slot_computed[s], cudaEventDisableTiming));
        if (!ctx->slot_copied[s]) WS_CUDA(cudaEventCreateWithFlags(&ctx->slot_copied[s], cudaEventDisableTiming));
        if (!ctx->slot_loaded[s]) WS_CUDA(cudaEventCreateWithFlags(&ctx->slot_loaded[s], cudaEventDisableTiming));
    }
    const size_t total = (size_t)n_events * n_planes;
    auto any = [&](void* const* a) {
        if (a)
            for (size_t k = 0; k < total; ++k)
                if (a[k]) return true;
        return false;
    };
    const bool want_f = any(frames), want_a = spec && any(adcs);
    const bool want_c = charges && any(reinterpret_cast<void* const*>(charges));
    if (!want_f && !want_a && !want_c) return set_err(WS_EINVAL, "no output requested");
    // per-slot device layout, per plane: [frame][adc][charge]
    std::vector<size_t> off_f(n_planes), off_a(n_planes), off_c(n_planes);
    size_t slot_bytes = 0;
    for (uint32_t i = 0; i < n_planes; ++i) {
        const size_t cells = (size_t)planes[i]->W * planes[i]->N;
        auto put = [&](bool on, size_t el) {
            const size_t o = slot_bytes;
            if (on) slot_bytes += (cells * el + 255) & ~(size_t)255;
            return o;
        };
        off_f[i] = put(want_f, frame_elem(spec));
        off_a[i] = put(want_a, adc_elem(spec));
        off_c[i] = put(want_c, opt->fluctuate && opt->charge_type == WS_CHARGE_I64 ? 8 : 4);
    }
    size_t max_units = 0;
    for (uint32_t e = 0; e < n_events; ++e) {
        size_t u = 0;
        for (uint32_t i = 0; i < n_planes; ++i) u += n_depos[(size_t)e * n_planes + i];
        max_units = std::max(max_units, u);
    }
    WS_CUDA(ctx->depos.reserve(2 * max_units + 1));
    WS_CUDA(ctx->out_stage.reserve(2 * slot_bytes));
    unsigned char* stage = ctx->out_stage.p;
    std::vector<const ws_depo*> dd(n_planes);
    std::vector<void*> df(n_planes), da(n_planes);
    std::vector<float*> dc(n_planes);

    std::vector<uint32_t> todo(n_events);
    for (uint32_t e = 0; e < n_events; ++e) todo[e] = e;
    for (int attempt = 0; attempt < kMaxAttempts && !todo.empty(); ++attempt) {
        ctx->failed_tags.clear();
        int rc = WS_OK;
        for (size_t j = 0; j < todo.size() && rc == WS_OK; ++j) {
            const uint32_t e = todo[j];
            const int slot = (int)(j & 1u);
            rc = [&]() -> int {
                if (j >= 2) WS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->slot_copied[slot], 0));
                // the depos go in on their own stream (a copy engine of their
                // own): this event's H2D overlaps the previous event's compute,
                // once the slot's last user (two events back) has computed
                if (j >= 2) WS_CUDA(cudaStreamWaitEvent(ctx->h2d_stream, ctx->slot_computed[slot], 0));
                size_t uo = (size_t)slot * max_units;
                unsigned char* base = stage + (size_t)slot * slot_bytes;
                for (uint32_t i = 0; i < n_planes; ++i) {
                    const size_t k = (size_t)e * n_planes + i;
                    dd[i] = ctx->depos.p + uo;
                    if (n_depos[k])
                        WS_CUDA(cudaMemcpyAsync(ctx->depos.p + uo, depos[k], sizeof(ws_depo) * n_depos[k],
                                                cudaMemcpyHostToDevice, ctx->h2d_stream));
                    uo += n_depos[k];
                    df[i] = frames && frames[k] ? base + off_f[i] : nullptr;
                    da[i] = want_a && adcs[k] ? base + off_a[i] : nullptr;
                    dc[i] = want_c && charges[k] ? reinterpret_cast<float*>(base + off_c[i]) : nullptr;
                }
                WS_CUDA(cudaEventRecord(ctx->slot_loaded[slot], ctx->h2d_stream));
                WS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->slot_loaded[slot], 0));
                ctx->call_tag = (int)e;
                const int r = event_device(ctx, n_planes, planes, dd.data(), n_depos + (size_t)e * n_planes, opt, spec,
                                           df.data(), da.data(), want_c ? dc.data() : nullptr,
                                           e == 0 ? timing : nullptr);
                ctx->call_tag = -1;
                if (r) return r;
                WS_CUDA(cudaEventRecord(ctx->slot_computed[slot], ctx->stream));
                WS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->slot_computed[slot], 0));
                for (uint32_t i = 0; i < n_planes; ++i) {
                    const size_t k = (size_t)e * n_planes + i, cells = (size_t)planes[i]->W * planes[i]->N;
                    if (df[i])
                        WS_CUDA(cudaMemcpyAsync(frames[k], df[i], cells * frame_elem(spec), cudaMemcpyDeviceToHost,
                                                ctx->copy_stream));
                    if (da[i])
                        WS_CUDA(cudaMemcpyAsync(adcs[k], da[i], cells * adc_elem(spec), cudaMemcpyDeviceToHost,
                                                ctx->copy_stream));
                    if (dc[i])
                        WS_CUDA(cudaMemcpyAsync(charges[k], dc[i],
                                                cells * (opt->fluctuate && opt->charge_type == WS_CHARGE_I64 ? 8 : 4),
                                                cudaMemcpyDeviceToHost, ctx->copy_stream));
                }
                WS_CUDA(cudaEventRecord(ctx->slot_copied[slot], ctx->copy_stream));
                return WS_OK;
            }();
        }
        // every copy has landed before this returns, whatever happened
        const cudaError_t he = cudaStreamSynchronize(ctx->h2d_stream);  // (host depos no longer read)
        cudaError_t ce = cudaStreamSynchronize(ctx->copy_stream);
        if (ce == cudaSuccess) ce = he;
        if (rc == WS_OK && ce != cudaSuccess)
            rc = set_err(WS_ECUDA, "copy stream: %s", cudaGetErrorString(ce));
        const int frc = finish_pending(ctx);
        if (rc == WS_OK || rc == WS_ERANGE) rc = frc;
        if (rc && rc != WS_ERANGE) return rc;
        std::vector<uint32_t> redo;
        for (int t : ctx->failed_tags) redo.push_back((uint32_t)t);
        std::sort(redo.begin(), redo.end());
        redo.erase(std::unique(redo.begin(), redo.end()), redo.end());
        if (rc == WS_ERANGE && redo.empty()) return rc;  // an untagged overflow: nothing to re-run
        todo.swap(redo);
    }
    ctx->failed_tags.clear();
    if (!todo.empty())
        return set_err(WS_ERANGE, "workspace: %zu event(s) still overflow after %d attempts", todo.size(),
                       kMaxAttempts);
    return WS_OK;
}

}  // namespace

extern "C" {

int ws_simulate_event_device(ws_ctx* ctx, uint32_t n_planes, ws_plane* const* planes, const ws_depo* const* depos,
                             const uint64_t* n_depos, const ws_sim_options* opt, float* const* frames,
                             ws_timing* timing)
{
    if (int rc = check_plane_set(ctx, n_planes, planes)) return rc;
    if (int rc = check_opts(opt)) return rc;
    WS_CUDA(cudaSetDevice(ctx->device));
    return event_device(ctx, n_planes, planes, depos, n_depos, opt, nullptr,
                        reinterpret_cast<void* const*>(frames), nullptr, nullptr, timing);
}

int ws_run_event_device(ws_ctx* ctx, uint32_t n_planes, ws_plane* const* planes, const ws_depo* const* depos,
                        const uint64_t* n_depos, const ws_sim_options* opt, const ws_readout* readout,
                        void* const* adcs, void* const* frames, ws_timing* timing)
{
    if (int rc = check_plane_set(ctx, n_planes, planes)) return rc;
    if (int rc = check_opts(opt)) return rc;
    if (!readout) return set_err(WS_EINVAL, "null readout");
    if (int rc = check_readout(readout, n_planes, planes)) return rc;
    WS_CUDA(cudaSetDevice(ctx->device));
    return event_device(ctx, n_planes, planes, depos, n_depos, opt, readout, frames, adcs, nullptr, timing);
}

int ws_simulate_plane_device(ws_plane* p, const ws_depo* depos, uint64_t n, const ws_sim_options* opt, float* frame,
                             float* charge, ws_timing* timing)
{
    if (!p) return set_err(WS_EINVAL, "null plane");
    if (int rc = check_opts(opt)) return rc;
    WS_CUDA(cudaSetDevice(p->ctx->device));
    ws_plane* planes[1] = {p};
    const ws_depo* dp[1] = {depos};
    uint64_t nd[1] = {n};
    void* fr[1] = {frame};
    float* ch[1] = {charge};
    return event_device(p->ctx, 1, planes, dp, nd, opt, nullptr, fr, nullptr, ch, timing);
}

int ws_run_simulation_device(ws_plane* p, const ws_depo* depos, uint64_t n, const ws_sim_options* opt,
                             const ws_readout* readout, void* adc, void* frame, float* charge, ws_timing* timing)
{
    if (!p) return set_err(WS_EINVAL, "null plane");
    if (int rc = check_opts(opt)) return rc;
    if (!readout) return set_err(WS_EINVAL, "null readout");
    ws_plane* planes[1] = {p};
    if (int rc = check_readout(readout, 1, planes)) return rc;
    WS_CUDA(cudaSetDevice(p->ctx->device));
    const ws_depo* dp[1] = {depos};
    uint64_t nd[1] = {n};
    void* fr[1] = {frame};
    void* ad[1] = {adc};
    float* ch[1] = {charge};
    return event_device(p->ctx, 1, planes, dp, nd, opt, readout, fr, ad, ch, timing);
}

int ws_rasterize_device(ws_plane* p, const ws_depo* depos, uint64_t n, const ws_sim_options* opt, float* charge,
                        ws_timing* timing)
{
    if (!p || !charge) return set_err(WS_EINVAL, "null argument");
    if (int rc = check_opts(opt)) return rc;
    WS_CUDA(cudaSetDevice(p->ctx->device));
    ws_plane* planes[1] = {p};
    const ws_depo* dp[1] = {depos};
    uint64_t nd[1] = {n};
    float* chs[1] = {charge};
    unsigned long long* cnt[1] = {nullptr};
    if (opt->fluctuate) {
        WS_CUDA(p->ctx->counts.reserve((size_t)p->W * p->N));
        cnt[0] = p->ctx->counts.p;
    }
    return run_group(p->ctx, 1, planes, dp, nd, opt, nullptr, chs, nullptr, timing, nullptr, cnt);
}

int ws_convolve_device(ws_plane* p, const float* charge, float* frame)
{
    if (!p || !charge || !frame) return set_err(WS_EINVAL, "null argument");
    WS_CUDA(cudaSetDevice(p->ctx->device));
    ws_sim_options o{};
    ws_plane* planes[1] = {p};
    float* fr[1] = {frame};
    const float* ci[1] = {charge};
    return run_group(p->ctx, 1, planes, nullptr, nullptr, &o, fr, nullptr, ci, nullptr);
}

int ws_simulate_event(ws_ctx* ctx, uint32_t n_planes, ws_plane* const* planes, const ws_depo* const* depos,
                      const uint64_t* n_depos, const ws_sim_options* opt, float* const* frames, ws_timing* timing)
{
    if (!frames) return set_err(WS_EINVAL, "null frames");
    return events_host(ctx, 1, n_planes, planes, depos, n_depos, opt, nullptr,
                       reinterpret_cast<void* const*>(frames), nullptr, nullptr, timing);
}

int ws_simulate_events(ws_ctx* ctx, uint32_t n_events, uint32_t n_planes, ws_plane* const* planes,
                       const ws_depo* const* depos, const uint64_t* n_depos, const ws_sim_options* opt,
                       float* const* frames, ws_timing* timing)
{
    if (n_events && n_planes && !frames) return set_err(WS_EINVAL, "null frames");
    return events_host(ctx, n_events, n_planes, planes, depos, n_depos, opt, nullptr,
                       reinterpret_cast<void* const*>(frames), nullptr, nullptr, timing);
}

int ws_run_events(ws_ctx* ctx, uint32_t n_events, uint32_t n_planes, ws_plane* const* planes,
                  const ws_depo* const* depos, const uint64_t* n_depos, const ws_sim_options* opt,
                  const ws_readout* readout, void* const* adcs, void* const* frames, ws_timing* timing)
{
    if (!readout) return set_err(WS_EINVAL, "null readout");
    return events_host(ctx, n_events, n_planes, planes, depos, n_depos, opt, readout, frames, adcs, nullptr, timing);
}

int ws_noise_digitize_device(ws_plane* p, float* frame, const ws_noise_model* noise, double scale, double offset,
                             int32_t bits, int32_t* adc)
{
    if (!p || !frame) return set_err(WS_EINVAL, "null argument");
    const int white = noise && noise->mode == WS_NOISE_WHITE;
    const int spectrum = noise && noise->mode == WS_NOISE_SPECTRUM;
    if (noise && noise->mode != WS_NOISE_OFF && !white && !spectrum)
        return set_err(WS_EINVAL, "add_noise: unknown noise mode %d", noise->mode);
    const wsb::Sink sk{frame, nullptr, adc, 0, scale, offset, (double)((1 << (adc && bits >= 1 && bits <= 16 ? bits : 1)) - 1)};
    if (spectrum) {
        if (noise->rng_mode != WS_RNG_SUBSTREAM && noise->rng_mode != WS_RNG_PHILOX)
            return set_err(WS_EINVAL, "add_noise: unknown rng mode %d", noise->rng_mode);
        if (!noise->amplitude_spectrum || noise->n_amplitude != (uint64_t)p->N)
            return set_err(WS_EINVAL,
                           "add_noise: amplitude_spectrum length %llu does not match the padded tick count %d",
                           (unsigned long long)noise->n_amplitude, p->N);
        if (adc && (bits < 1 || bits > 16)) return set_err(WS_EINVAL, "digitize: bits must be in [1,16]");
        if (p->folded)
            return set_err(WS_EINVAL, "add_noise: spectrum mode needs an even 7-smooth padded tick count (got %d)",
                           p->N);
        ws_ctx* c = p->ctx;
        WS_CUDA(cudaSetDevice(c->device));
        WS_CUDA(c->noise_amp.reserve((size_t)p->N));
        WS_CUDA(cudaMemcpyAsync(c->noise_amp.p, noise->amplitude_spectrum, sizeof(double) * p->N,
                                cudaMemcpyHostToDevice, c->stream));
        const PlaneDesc d = plane_desc(p);
        WS_CUDA(wsb_launch_noise_spectrum(d, c->noise_amp.p, noise->seed, noise->rng_mode, frame, sk, c->conv_variant,
                                          c->stream));
        c->launches += 1;
        return WS_OK;
    }
    if (noise && noise->sigma < 0.0) return set_err(WS_EINVAL, "add_noise: sigma must be >= 0");
    if (noise && noise->rng_mode != WS_RNG_SUBSTREAM && noise->rng_mode != WS_RNG_PHILOX)
        return set_err(WS_EINVAL, "add_noise: unknown rng mode %d", noise->rng_mode);
    if (adc && (bits < 1 || bits > 16)) return set_err(WS_EINVAL, "digitize: bits must be in [1,16]");
    const int do_noise = white && noise->sigma != 0.0;  // sigma 0: the reference returns the input
    if (!do_noise && !adc) return WS_OK;
    ws_ctx* c = p->ctx;
    WS_CUDA(cudaSetDevice(c->device));
    wsb::Sink k = sk;
    if (!do_noise) k.frame = nullptr;  // digitize only: the frame is untouched
    WS_CUDA(wsb_launch_noise(frame, k, p->W, p->N, do_noise, do_noise ? noise->rng_mode : WS_RNG_PHILOX,
                             do_noise ? noise->sigma : 0.0, do_noise ? noise->seed : 0, c->stream));
    c->launches += 1;
    return WS_OK;
}

int ws_simulate_plane(ws_plane* p, const ws_depo* depos, uint64_t n, const ws_sim_options* opt, float* frame,
                      float* charge, ws_timing* timing)
{
    if (!p) return set_err(WS_EINVAL, "null plane");
    ws_plane* planes[1] = {p};
    const ws_depo* dp[1] = {depos};
    uint64_t nd[1] = {n};
    void* fr[1] = {frame};
    float* ch[1] = {charge};
    return events_host(p->ctx, 1, 1, planes, dp, nd, opt, nullptr, fr, nullptr, ch, timing);
}

int ws_run_simulation(ws_plane* p, const ws_depo* depos, uint64_t n, const ws_sim_options* opt,
                      const ws_readout* readout, void* adc, void* frame, float* charge, ws_timing* timing)
{
    if (!p) return set_err(WS_EINVAL, "null plane");
    if (!readout) return set_err(WS_EINVAL, "null readout");
    ws_plane* planes[1] = {p};
    const ws_depo* dp[1] = {depos};
    uint64_t nd[1] = {n};
    void* fr[1] = {frame};
    void* ad[1] = {adc};
    float* ch[1] = {charge};
    return events_host(p->ctx, 1, 1, planes, dp, nd, opt, readout, fr, ad, ch, timing);
}

}  // extern "C"

// ---- signal processing (ws_sigproc.cu) -------------------------------------

namespace {

// plan for row length n: radices (8s, then 4 / 2, then odd primes <= 13),
// output permutation of the in-place DIF passes, split twiddle table
int sigproc_plan(ws_ctx* c, uint64_t n)
{
    if (c->sp_n == n && n) return WS_OK;
    std::vector<int8_t> radix;
    uint64_t m = n;
    int twos = 0;
    while (m % 2 == 0) {
        m /= 2;
        ++twos;
    }
    for (; twos >= 4; twos -= 4) radix.push_back(16);
    if (twos == 3) radix.push_back(8);
    if (twos == 2) radix.push_back(4);
    if (twos == 1) radix.push_back(2);
    for (int p : {3, 5, 7, 11, 13})
        while (m % p == 0) {
            m /= p;
            radix.push_back((int8_t)p);
        }
    if (m != 1) {
        // a prime factor > 13: the direct inverse DFT, twiddles exp(+2 pi i m / n), m < n
        if (n > (uint64_t)wsb_sigproc_dft_max_n())
            return set_err(WS_EINVAL, "sigproc: row length %llu has a prime factor > 13 and exceeds the direct "
                           "path's %d samples", (unsigned long long)n, wsb_sigproc_dft_max_n());
        std::vector<double2> tw(n);
        for (uint64_t j = 0; j < n; ++j) {
            const long double a = 6.283185307179586476925286766559L * (long double)j / (long double)n;
            tw[j] = make_double2((double)cosl(a), (double)sinl(a));
        }
        WS_CUDA(c->sp_tw.reserve(n));
        WS_CUDA(cudaMemcpyAsync(c->sp_tw.p, tw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
        WS_CUDA(cudaStreamSynchronize(c->stream));
        c->sp_radix.clear();
        c->sp_dft = true;
        c->sp_n = n;
        return WS_OK;
    }
    c->sp_dft = false;
    if ((int)radix.size() > wsb::kSpMaxRadices) return set_err(WS_EINVAL, "sigproc: too many radix passes");
    std::vector<int> perm(n);
    for (uint64_t k = 0; k < n; ++k) {
        uint64_t kk = k, S = n, pos = 0;
        for (int8_t R : radix) {
            S /= (uint64_t)R;
            pos += (kk % (uint64_t)R) * S;
            kk /= (uint64_t)R;
        }
        perm[k] = (int)pos;
    }
    std::vector<double2> tw;  // per pass: exp(+2 pi i j / L), j < L / R
    uint64_t L = n;
    for (int8_t R : radix) {
        const uint64_t S = L / (uint64_t)R;
        for (uint64_t j = 0; j < S; ++j) {
            const long double a = 6.283185307179586476925286766559L * (long double)j / (long double)L;
            tw.push_back(make_double2((double)cosl(a), (double)sinl(a)));
        }
        L = S;
    }
    if (tw.empty()) tw.push_back(make_double2(1.0, 0.0));
    const size_t n_tw = tw.size();
    WS_CUDA(c->sp_perm.reserve(n));
    WS_CUDA(c->sp_tw.reserve(n_tw));
    WS_CUDA(cudaMemcpyAsync(c->sp_perm.p, perm.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    WS_CUDA(cudaMemcpyAsync(c->sp_tw.p, tw.data(), sizeof(double2) * n_tw, cudaMemcpyHostToDevice, c->stream));
    WS_CUDA(cudaStreamSynchronize(c->stream));  // host vectors go out of scope
    c->sp_radix = radix;
    c->sp_n = n;
    return WS_OK;
}

int sigproc_validate(const ws_signal_batch* b, uint64_t filter_len)
{
    if (!b) return set_err(WS_EINVAL, "null batch");
    // SignalBatch::validate (sigproc.hpp:24-28), apply_filter (sigproc.cpp:14-17)
    if (b->cols < 1) return set_err(WS_EINVAL, "SignalBatch: need at least one column");
    if (b->pad_rows + b->out_rows > b->rows)
        return set_err(WS_EINVAL, "SignalBatch: pad_rows + out_rows exceeds the row count");
    if (filter_len != b->cols)
        return set_err(WS_EINVAL, "apply_filter: filter length %llu does not match %llu columns",
                       (unsigned long long)filter_len, (unsigned long long)b->cols);
    if (b->cols > (uint64_t)wsb_sigproc_max_n())
        return set_err(WS_EINVAL, "sigproc: row length %llu exceeds the GPU path's %d samples",
                       (unsigned long long)b->cols, wsb_sigproc_max_n());
    if (b->rows > 0x7fffffffull) return set_err(WS_EINVAL, "sigproc: too many rows");
    if (b->rows && !b->data) return set_err(WS_EINVAL, "null batch data");
    return WS_OK;
}

wsb::SigprocDesc sigproc_desc(ws_ctx* c, const double* data, uint64_t rows, int pad, int out, const double2* filter,
                              double* block, double* medians)
{
    wsb::SigprocDesc d{};
    d.data = reinterpret_cast<const double2*>(data);
    d.filter = filter;
    d.block = block;
    d.medians = medians;
    d.stats = c->sp_stats.p;
    d.tw = c->sp_tw.p;
    d.perm = c->sp_perm.p;
    d.n = (int)c->sp_n;
    d.rows = (int)rows;
    d.pad = pad;
    d.out = out;
    d.mode = c->sp_dft ? 2 : 0;
    d.nf = (int)c->sp_radix.size();
    d.inv_n = 1.0 / (double)c->sp_n;  // fft.cpp:99
    for (int i = 0; i < d.nf; ++i)  // 4 bits per pass, radix 16 encoded as 1
        d.radix[i >> 4] |= (unsigned long long)(c->sp_radix[i] == 16 ? 1 : c->sp_radix[i]) << (4 * (i & 15));
    return d;
}

int sigproc_residue(ws_ctx* c, double* max_rel_imag)
{
    unsigned long long st[2];
    WS_CUDA(cudaMemcpyAsync(st, c->sp_stats.p, sizeof st, cudaMemcpyDeviceToHost, c->stream));
    WS_CUDA(cudaStreamSynchronize(c->stream));
    double peak, resid;
    std::memcpy(&peak, &st[0], sizeof peak);
    std::memcpy(&resid, &st[1], sizeof resid);
    *max_rel_imag = peak > 0.0 ? resid / peak : resid;
    if (*max_rel_imag > 1e-6)  // idft_rows_to_real's report (sigproc.cpp:66-68)
        std::fprintf(stderr, "idft_rows_to_real: imaginary residue %.3e relative (input not Hermitian?)\n",
                     *max_rel_imag);
    return WS_OK;
}

}  // namespace

extern "C" {

uint64_t ws_sigproc_max_cols(void) { return (uint64_t)wsb_sigproc_max_n(); }

int ws_sigproc_chain_device(ws_ctx* c, const ws_signal_batch* b, const double* filter, uint64_t filter_len,
                            double* block, double* medians, double* max_rel_imag)
{
    if (!c) return set_err(WS_EINVAL, "null context");
    if (int rc = sigproc_validate(b, filter_len)) return rc;
    if (!filter) return set_err(WS_EINVAL, "null filter");
    if (b->out_rows && !block) return set_err(WS_EINVAL, "null block");
    WS_CUDA(cudaSetDevice(c->device));
    if (int rc = sigproc_plan(c, b->cols)) return rc;
    WS_CUDA(c->sp_stats.reserve(2));
    WS_CUDA(cudaMemsetAsync(c->sp_stats.p, 0, 2 * sizeof(unsigned long long), c->stream));
    const wsb::SigprocDesc d = sigproc_desc(c, b->data, b->rows, (int)b->pad_rows, (int)b->out_rows,
                                            reinterpret_cast<const double2*>(filter), block, medians);
    WS_CUDA(wsb_launch_sigproc(d, c->stream));
    if (b->rows) c->launches += 1;
    if (max_rel_imag) return sigproc_residue(c, max_rel_imag);
    return WS_OK;
}

int ws_sigproc_chain(ws_ctx* c, const ws_signal_batch* b, const double* filter, uint64_t filter_len,
                     int filter_complex, double* block, double* medians, double* max_rel_imag)
{
    if (!c) return set_err(WS_EINVAL, "null context");
    if (int rc = sigproc_validate(b, filter_len)) return rc;
    if (!filter) return set_err(WS_EINVAL, "null filter");
    if (b->out_rows && !block) return set_err(WS_EINVAL, "null block");
    WS_CUDA(cudaSetDevice(c->device));
    if (int rc = finish_pending(c)) return rc;
    const uint64_t n = b->cols;
    if (int rc = sigproc_plan(c, n)) return rc;
    // filter -> complex on the device (a real filter gets zero imaginary parts)
    std::vector<double2> f(n);
    for (uint64_t i = 0; i < n; ++i)
        f[i] = filter_complex ? make_double2(filter[2 * i], filter[2 * i + 1]) : make_double2(filter[i], 0.0);
    WS_CUDA(c->sp_filter.reserve(n));
    WS_CUDA(cudaMemcpyAsync(c->sp_filter.p, f.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, c->stream));
    WS_CUDA(c->sp_stats.reserve(2));
    WS_CUDA(cudaMemsetAsync(c->sp_stats.p, 0, 2 * sizeof(unsigned long long), c->stream));
    WS_CUDA(c->sp_med.reserve(std::max<uint64_t>(b->out_rows, 1)));
    // rows stream through two staging slots: H2D (h2d_stream) -> chain (main) -> D2H (copy_stream)
    if (!c->h2d_stream) WS_CUDA(cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking));
    if (!c->copy_stream) WS_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int s = 0; s < 2; ++s)
        for (cudaEvent_t* e : {&c->sp_loaded[s], &c->sp_done[s], &c->sp_copied[s]})
            if (!*e) WS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(b->rows, (8u << 20) / (16 * n)));
    WS_CUDA(c->sp_data.reserve(2 * chunk * n));
    WS_CUDA(c->sp_block.reserve(2 * chunk * n));
    WS_CUDA(cudaEventRecord(c->sp_done[0], c->stream));  // filter / stats / plan uploads precede every chunk
    WS_CUDA(cudaStreamWaitEvent(c->h2d_stream, c->sp_done[0], 0));
    const uint64_t pad = b->pad_rows, out = b->out_rows;
    int k = 0;
    for (uint64_t r0 = 0; r0 < b->rows; r0 += chunk, ++k) {
        const int slot = k & 1;
        const uint64_t nr = std::min(chunk, b->rows - r0);
        double2* din = c->sp_data.p + (size_t)slot * chunk * n;
        double* dblk = c->sp_block.p + (size_t)slot * chunk * n;
        // slot reuse: the chain of chunk k - 2 has read din, its block has left dblk
        if (k >= 2) {
            WS_CUDA(cudaStreamWaitEvent(c->h2d_stream, c->sp_done[slot], 0));
            WS_CUDA(cudaStreamWaitEvent(c->stream, c->sp_copied[slot], 0));
        }
        WS_CUDA(cudaMemcpyAsync(din, b->data + 2 * r0 * n, sizeof(double2) * nr * n, cudaMemcpyHostToDevice,
                                c->h2d_stream));
        WS_CUDA(cudaEventRecord(c->sp_loaded[slot], c->h2d_stream));
        WS_CUDA(cudaStreamWaitEvent(c->stream, c->sp_loaded[slot], 0));
        const uint64_t o0 = std::max(r0, pad), o1 = std::min(r0 + nr, pad + out);  // block rows of this chunk
        const int n_out = o1 > o0 ? (int)(o1 - o0) : 0;
        const int pad_in_chunk = n_out ? (int)(o0 - r0) : (int)nr;
        const wsb::SigprocDesc d =
            sigproc_desc(c, reinterpret_cast<const double*>(din), nr, pad_in_chunk, n_out, c->sp_filter.p, dblk,
                         medians && n_out ? c->sp_med.p + (o0 - pad) : nullptr);
        WS_CUDA(wsb_launch_sigproc(d, c->stream));
        c->launches += 1;
        WS_CUDA(cudaEventRecord(c->sp_done[slot], c->stream));
        if (n_out) {
            WS_CUDA(cudaStreamWaitEvent(c->copy_stream, c->sp_done[slot], 0));
            WS_CUDA(cudaMemcpyAsync(block + (o0 - pad) * n, dblk, sizeof(double) * (size_t)n_out * n,
                                    cudaMemcpyDeviceToHost, c->copy_stream));
        }
        WS_CUDA(cudaEventRecord(c->sp_copied[slot], c->copy_stream));
    }
    if (medians && out) {
        WS_CUDA(cudaMemcpyAsync(medians, c->sp_med.p, sizeof(double) * out, cudaMemcpyDeviceToHost, c->stream));
    }
    WS_CUDA(cudaStreamSynchronize(c->copy_stream));
    WS_CUDA(cudaStreamSynchronize(c->stream));
    if (max_rel_imag) return sigproc_residue(c, max_rel_imag);
    return WS_OK;
}

int ws_row_medians_device(ws_ctx* c, const double* m, uint64_t rows, uint64_t cols, double* medians)
{
    if (!c) return set_err(WS_EINVAL, "null context");
    if (cols < 1) return set_err(WS_EINVAL, "row_median: empty input");
    if (cols > (uint64_t)wsb_sigproc_max_n())
        return set_err(WS_EINVAL, "row_median: row length %llu exceeds the GPU path's %d samples",
                       (unsigned long long)cols, wsb_sigproc_max_n());
    if (rows > 0x7fffffffull) return set_err(WS_EINVAL, "row_median: too many rows");
    if (rows && (!m || !medians)) return set_err(WS_EINVAL, "null argument");
    WS_CUDA(cudaSetDevice(c->device));
    wsb::SigprocDesc d{};
    d.data = reinterpret_cast<const double2*>(m);
    d.medians = medians;
    d.n = (int)cols;
    d.rows = (int)rows;
    d.out = (int)rows;
    d.mode = 1;
    WS_CUDA(wsb_launch_sigproc(d, c->stream));
    if (rows) c->launches += 1;
    return WS_OK;
}

}  // extern "C"
