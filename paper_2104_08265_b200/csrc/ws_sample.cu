// Per-depo sampling (K1 front half), depo -> wire-band binning, and the
// sequential-binomial fluctuation walk (K2).
//
// Compiled with --fmad=false: every double expression below keeps the
// reference's operation order and rounding (no FMA contraction), so the
// footprints and bin integrals are the reference's, and the fluctuation walk
// reproduces its integer draws.
#include "ws_common.cuh"

#include <algorithm>


namespace wsb {

__device__ __forceinline__ int lane_id() { return (int)(threadIdx.x & 31); }

constexpr double kInvSqrt2 = 0.70710678118654752440084436210485;

struct Footprint {
    int w0, n_w, t0, n_t;
    bool clipped, empty;
};

// map_depo_to_grid (core.cpp:25-41) + the clip of sample_patch (rasterize.cpp:68-80)
__device__ __forceinline__ Footprint footprint(const PlaneDesc& P, const ws_depo& d)
{
    const long cw = (long)P.pad_w + (long)floor((d.x - P.origin_x) / P.pitch);
    const long ct = (long)P.pad_t + (long)floor((d.t - P.origin_t) / P.tick);
    const long hw = d.sigma_x <= 0.0 ? 0 : (long)ceil(P.n_sigma * d.sigma_x / P.pitch);
    const long ht = d.sigma_t <= 0.0 ? 0 : (long)ceil(P.n_sigma * d.sigma_t / P.tick);
    const long wlo = cw - hw, whi = cw + hw, tlo = ct - ht, thi = ct + ht;
    const long max_w = (long)P.W - 1, max_t = (long)P.N - 1;
    const long wl = wlo > 0 ? wlo : 0, wh = whi < max_w ? whi : max_w;
    const long tl = tlo > 0 ? tlo : 0, th = thi < max_t ? thi : max_t;
    Footprint f;
    f.clipped = wl != wlo || wh != whi || tl != tlo || th != thi;
    f.empty = wl > wh || tl > th;
    f.w0 = (int)wl;
    f.t0 = (int)tl;
    f.n_w = f.empty ? 0 : (int)(wh - wl + 1);
    f.n_t = f.empty ? 0 : (int)(th - tl + 1);
    return f;
}

// drift_depo (rasterize.cpp:22-42); returns false if the depo is behind the plane.
__device__ __forceinline__ bool drift(const EventDesc& ev, ws_depo& d)
{
    if (d.x < ev.drift_plane_x) return false;
    const double dx = d.x - ev.drift_plane_x;
    const double drift_time = dx / ev.drift_speed;
    d.t = d.t + drift_time;
    d.x = ev.drift_plane_x;
    const double v2 = ev.drift_speed * ev.drift_speed;
    d.sigma_t = sqrt(d.sigma_t * d.sigma_t + 2.0 * ev.drift_dl * drift_time / v2);
    d.sigma_x = sqrt(d.sigma_x * d.sigma_x + 2.0 * ev.drift_dt * drift_time);
    return true;
}

// gauss_bin_integrals (rasterize.cpp:44-64), one thread, reference order.
// Returns sum and max of the n values; writes them through `put(i, v)`.
template <typename Put>
__device__ __forceinline__ void bin_integrals(double center, double sigma, double lo_edge, double spacing, int n,
                                              Put&& put, double& sum, double& vmax)
{
    sum = 0.0;
    vmax = 0.0;
    if (sigma <= 0.0) {
        long idx = (long)floor((center - lo_edge) / spacing);
        idx = idx < 0 ? 0 : (idx > n - 1 ? n - 1 : idx);
        for (int i = 0; i < n; ++i) put(i, i == idx ? 1.0 : 0.0);
        sum = 1.0;
        vmax = 1.0;
        return;
    }
    const double inv = kInvSqrt2 / sigma;
    double prev = erf((lo_edge - center) * inv);
    for (int i = 0; i < n; ++i) {
        const double next = erf((lo_edge + (double)(i + 1) * spacing - center) * inv);
        const double v = 0.5 * (next - prev);
        prev = next;
        put(i, v);
        sum += v;
        vmax = v > vmax ? v : vmax;
    }
}

// Fluctuation-off bin integrals in fp32 (the north star's fp32 mode): one
// erfcf per edge, differences formed on the side of the centre where they
// do not cancel (the tails keep their relative accuracy). Used when both
// widths are at least a quarter bin, so every edge argument is within
// |x| < 5 and nothing underflows; narrower depos take the fp64 path.
template <typename Put>
__device__ __forceinline__ void bin_integrals_f32(double center, double sigma, double lo_edge, double spacing, int n,
                                                  Put&& put, double& sum, double& vmax)
{
    const double inv = kInvSqrt2 / sigma;
    const float x0 = (float)((lo_edge - center) * inv), dx = (float)(spacing * inv);
    float xp = x0, cp = erfcf(fabsf(x0));
    float s = 0.0f, m = 0.0f, fi = 1.0f;  // float counter: no I2F on the XU pipe
    for (int i = 0; i < n; ++i, fi += 1.0f) {
        const float xn = fmaf(fi, dx, x0);
        const float cn = erfcf(fabsf(xn));
        // erf(xn) - erf(xp) with erf(x) = sign(x) (1 - erfc|x|)
        const float diff = xp >= 0.0f ? cp - cn : (xn <= 0.0f ? cn - cp : 2.0f - cn - cp);
        const float v = 0.5f * diff;
        put(i, v);
        s += v;
        m = fmaxf(m, v);
        xp = xn;
        cp = cn;
    }
    sum = s;
    vmax = m;
}

// Wire-direction integrals at impact resolution (ws_plane_create_impacts):
// the footprint's n_w wires are split into `imp` sub-bins each (impact i of
// wire j spans [lo + (j imp + i) pitch / imp, + pitch / imp)), each sub-bin
// the Gaussian's integral (gauss_bin_integrals' rule at the finer spacing;
// sigma <= 0 puts the delta in its containing sub-bin). out[j] = the sum over
// the sub-bins of wire j whose impact is in `mask` (this response class);
// all4 = {sum, max} over the class's wires and {sum, max} over every
// sub-bin (the normalisation and the emptiness test of sample_patch,
// rasterize.cpp:101-118, run over all impacts). The sub-bin integrals of a
// wire telescope to its wire-bin integral: with one class the result is the
// reference's wire profile up to rounding.
template <typename T, typename Put>
__device__ __noinline__ void impact_integrals(double center, double sigma, double lo_edge, double pitch, int n_w, int imp,
                                              uint32_t mask, Put&& put, double* all4)
{
    double sc = 0.0, mc = 0.0, sa = 0.0, ma = 0.0;
    const int nk = n_w * imp;
    const double sub = pitch / (double)imp;
    if (sigma <= 0.0) {
        long idx = (long)floor((center - lo_edge) / sub);
        idx = idx < 0 ? 0 : (idx > nk - 1 ? nk - 1 : idx);
        for (int j = 0; j < n_w; ++j) put(j, (T)0);
        const bool in = (mask >> (idx % imp)) & 1u;
        if (in) put((int)(idx / imp), (T)1);
        sc = mc = in ? 1.0 : 0.0;
        sa = ma = 1.0;
    } else if constexpr (sizeof(T) == 8) {
        const double inv = kInvSqrt2 / sigma;
        double prev = erf((lo_edge - center) * inv);
        for (int j = 0; j < n_w; ++j) {
            double w = 0.0;
            for (int i = 0; i < imp; ++i) {
                const double next = erf((lo_edge + (double)(j * imp + i + 1) * sub - center) * inv);
                const double v = 0.5 * (next - prev);
                prev = next;
                sa += v;
                ma = v > ma ? v : ma;
                if ((mask >> i) & 1u) w += v;
            }
            put(j, (T)w);
            sc += w;
            mc = w > mc ? w : mc;
        }
    } else {
        // fp32 (fluctuation off): one erfcf per edge, each difference on the
        // side of the centre where it does not cancel (bin_integrals_f32)
        const double inv = kInvSqrt2 / sigma;
        const float x0 = (float)((lo_edge - center) * inv), dx = (float)(sub * inv);
        float xp = x0, cp = erfcf(fabsf(x0)), fi = 1.0f;
        float fsa = 0.0f, fma = 0.0f, fsc = 0.0f, fmc = 0.0f;
        for (int j = 0; j < n_w; ++j) {
            float w = 0.0f;
            for (int i = 0; i < imp; ++i, fi += 1.0f) {
                const float xn = fmaf(fi, dx, x0);
                const float cn = erfcf(fabsf(xn));
                const float diff = xp >= 0.0f ? cp - cn : (xn <= 0.0f ? cn - cp : 2.0f - cn - cp);
                const float v = 0.5f * diff;
                fsa += v;
                fma = fmaxf(fma, v);
                if ((mask >> i) & 1u) w += v;
                xp = xn;
                cp = cn;
            }
            put(j, (T)w);
            fsc += w;
            fmc = fmaxf(fmc, w);
        }
        sc = fsc;
        mc = fmc;
        sa = fsa;
        ma = fma;
    }
    all4[0] = sc;
    all4[1] = mc;
    all4[2] = sa;
    all4[3] = ma;
}

// fp64 bin integrals out of line (fluctuation on, and narrow depos with it
// off): their register demand stays out of the common fp32 path.
// out = {sum_w, max_w, sum_t, max_t}
template <bool kInline>
__device__ __forceinline__ void sample_f64_body(const ws_depo* d, double wire_edge, double pitch, int n_w, double tick_edge,
                                        double tick, int n_t, double* wv64, double* tv64, float* wv32, float* tv32,
                                        double* out)
{
    double sw, mw, st, mt;
    if (wv64) {
        bin_integrals(d->x, d->sigma_x, wire_edge, pitch, n_w, [&](int i, double v) { wv64[i] = v; }, sw, mw);
        bin_integrals(d->t, d->sigma_t, tick_edge, tick, n_t, [&](int i, double v) { tv64[i] = v; }, st, mt);
    } else {
        bin_integrals(d->x, d->sigma_x, wire_edge, pitch, n_w, [&](int i, double v) { wv32[i] = (float)v; }, sw, mw);
        bin_integrals(d->t, d->sigma_t, tick_edge, tick, n_t, [&](int i, double v) { tv32[i] = (float)v; }, st, mt);
    }
    out[0] = sw;
    out[1] = mw;
    out[2] = st;
    out[3] = mt;
}

__device__ __noinline__ void sample_f64_ool(const ws_depo* d, double wire_edge, double pitch, int n_w, double tick_edge,
                                            double tick, int n_t, float* wv32, float* tv32, double* out)
{
    sample_f64_body<false>(d, wire_edge, pitch, n_w, tick_edge, tick, n_t, nullptr, nullptr, wv32, tv32, out);
}

// Fluctuation-off sampling of a plane with impact positions (out of line):
// the class's wire profile at impact resolution (fp32 for wide depos, fp64
// for narrow ones, as the wire-binned path), the tick profile as usual.
// out6 = {sum, max} of the class's wire profile, {sum, max} over all
// impacts, {sum, max} of the tick profile.
// (scalars only: a PlaneDesc reference would copy the kernel parameters to the stack)
__device__ __noinline__ void sample_impacts_ool(const ws_depo* d, double pitch, double tick, int imp, uint32_t mask,
                                                double wire_edge, double tick_edge, int n_w, int n_t, bool fast,
                                                float* wv, float* tv, double* out6)
{
    double a4[4], st, mt;
    if (fast) {
        impact_integrals<float>(d->x, d->sigma_x, wire_edge, pitch, n_w, imp, mask, [&](int i, float v) { wv[i] = v; },
                                a4);
        bin_integrals_f32(d->t, d->sigma_t, tick_edge, tick, n_t, [&](int i, float v) { tv[i] = v; }, st, mt);
    } else {
        impact_integrals<double>(d->x, d->sigma_x, wire_edge, pitch, n_w, imp, mask,
                                 [&](int i, double v) { wv[i] = (float)v; }, a4);
        bin_integrals(d->t, d->sigma_t, tick_edge, tick, n_t, [&](int i, double v) { tv[i] = (float)v; }, st, mt);
    }
    for (int k = 0; k < 4; ++k) out6[k] = a4[k];
    out6[4] = st;
    out6[5] = mt;
}

// One thread per unit: footprint (map_depo_to_grid + clip), bin integrals
// into the pool, emptiness (sample_patch's total <= 0 test), clipped-charge
// bookkeeping and, with fluctuation off, the normalised separable profiles
// and the band counts.
//
// Pool layout per unit (32-bit words):
//   fluctuation on : [wv f64 x n_w][tv f64 x n_t]                 (8-byte aligned)
//   fluctuation off: [raw f32 x n_w][eff f32 x n_eff][tv f32 x n_t]
//                    (+ [g f32 x L][max|g|] on direct-path planes, filled by
//                    k_fill_bands; L = n_t + n_lags - 1)
// with raw = wv (the un-stencilled wire profile), eff = the profile after the
// cross-wire stencil (absent when wire_weights == {1}); rec.a = q / total with
// total = sum_w wv * sum_t tv.
// kFluct = false (the fluctuation-off hot path): fp32 profiles, 64 registers
// for occupancy, the rare fp64 fallback out of line; kFluct = true: fp64.
template <bool kFluct>
__global__ void __launch_bounds__(128, kFluct ? 1 : 8) k_sample(const EventDesc ev, UnitRec* __restrict__ recs, uint32_t* __restrict__ pool, uint32_t pool_cap,
                         uint32_t* __restrict__ pool_ctr, uint32_t* __restrict__ band_count,
                         unsigned* __restrict__ err)
{
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= ev.total_units) return;
    const int pi = plane_of_unit(ev, u);
    const PlaneDesc& P = ev.p[pi];
    ws_depo d = P.depos[u - P.unit_base];
    if constexpr (kFluct) {
        // the plane's electrons in all, each depo capped at 2^32 (cnt_wide:
        // below 2^32 the count grid takes u32 cells); one atomic per warp when
        // the warp's units share a plane
        if (P.cnt_qsum) {
            unsigned long long qq = d.q > 0 ? min((unsigned long long)d.q, 1ull << 32) : 0ull;
            const unsigned act = __activemask();
            const int lead = __ffs(act) - 1;
            if (__all_sync(act, pi == __shfl_sync(act, pi, lead))) {
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long t = __shfl_down_sync(act, qq, o);
                    if ((threadIdx.x & 31) + o < 32 && (act >> ((threadIdx.x & 31) + o)) & 1u) qq += t;
                }
                if ((int)(threadIdx.x & 31) == lead && qq)
                    atomicAdd(const_cast<unsigned long long*>(P.cnt_qsum), qq);
            } else if (qq) {
                atomicAdd(const_cast<unsigned long long*>(P.cnt_qsum), qq);
            }
        }
    }
    UnitRec rec;
    rec.w0 = -1;
    rec.t0 = 0;
    rec.n_w = 0;
    rec.n_t = 0;
    rec.pool = 0;
    rec.goff = 0;
    rec.a = 0.0f;
    rec.tsum = 0.0f;
    if (ev.drift_enabled && !drift(ev, d)) {
        atomicOr(err, kErrDomain);
        recs[u] = rec;
        return;
    }
    if (d.q < 0) atomicOr(err, kErrCharge);
    const Footprint f = footprint(P, d);
    if (f.clipped && P.stats_owner) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[1]), 1ULL);
    if (f.empty) {
        if (P.stats_owner) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[0]), (unsigned long long)d.q);
        recs[u] = rec;
        return;
    }
    const int h = P.h;
    const int n_eff = P.ww_is_one ? 0 : f.n_w + 2 * h;
    // fluctuation off on a direct-path plane: room for g = tv (*) kernel and max|g| (k_fill_bands)
    const bool with_g = !kFluct && ev.mode == 0 && P.direct;
    const uint32_t L = (uint32_t)(f.n_t + P.n_lags - 1);
    const uint32_t need = kFluct ? (uint32_t)(2 * (f.n_w + f.n_t) + 1)
                                       : (uint32_t)(f.n_w + n_eff + f.n_t) + (with_g ? ((L + 31u) & ~31u) + 4u : 0u);
    uint32_t off = atomicAdd(pool_ctr, need);
    if ((uint64_t)off + need > pool_cap) {
        atomicOr(err, kErrPool);
        recs[u] = rec;
        return;
    }
    const double wire_edge = P.origin_x + ((double)f.w0 - (double)P.pad_w) * P.pitch;
    const double tick_edge = P.origin_t + ((double)f.t0 - (double)P.pad_t) * P.tick;
    double sw, mw, st, mt;
    if constexpr (kFluct) {
        double o4[4];
        off += off & 1u;  // 8-byte alignment
        double* wv = reinterpret_cast<double*>(pool + off);
        if (P.impacts > 1) {
            // one response class (the host allows fluctuation only then):
            // the wire profile summed over the impact sub-bins
            double a4[4];
            impact_integrals<double>(d.x, d.sigma_x, wire_edge, P.pitch, f.n_w, P.impacts, P.imp_mask,
                                     [&](int i, double v) { wv[i] = v; }, a4);
            bin_integrals(d.t, d.sigma_t, tick_edge, P.tick, f.n_t, [&](int i, double v) { wv[f.n_w + i] = v; }, st,
                          mt);
            sw = a4[0];
            mw = a4[1];
        } else {
            sample_f64_body<true>(&d, wire_edge, P.pitch, f.n_w, tick_edge, P.tick, f.n_t, wv, wv + f.n_w, nullptr,
                                  nullptr, o4);
            sw = o4[0];
            mw = o4[1];
            st = o4[2];
            mt = o4[3];
        }
    } else if (!(d.sigma_x * 4.0 >= P.pitch && d.sigma_t * 4.0 >= P.tick)) {
        double o4[4];
        float* raw = reinterpret_cast<float*>(pool + off);
        sample_f64_ool(&d, wire_edge, P.pitch, f.n_w, tick_edge, P.tick, f.n_t, raw, raw + f.n_w + n_eff, o4);
        sw = o4[0];
        mw = o4[1];
        st = o4[2];
        mt = o4[3];
    } else {
        float* raw = reinterpret_cast<float*>(pool + off);
        float* tv = raw + f.n_w + n_eff;
        bin_integrals_f32(d.x, d.sigma_x, wire_edge, P.pitch, f.n_w, [&](int i, float v) { raw[i] = v; }, sw, mw);
        bin_integrals_f32(d.t, d.sigma_t, tick_edge, P.tick, f.n_t, [&](int i, float v) { tv[i] = v; }, st, mt);
    }
    // sum_w sum_t wv*tv > 0  <=>  max(wv)*max(tv) > 0 (all terms >= 0, products monotone)
    if (!(mw * mt > 0.0)) {
        // numerically empty (rasterize.cpp:111-116) -> clipped charge (pipeline.cpp:339-340)
        if (P.stats_owner) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[0]), (unsigned long long)d.q);
        recs[u] = rec;
        return;
    }
    if constexpr (!kFluct) {
        // S = q * p = a * wv[w] * tv[t] with a = q / total; a is applied by
        // the consumer (k_conv), so the profiles are stored unscaled
        const double a = (double)d.q / (sw * st);
        float* raw = reinterpret_cast<float*>(pool + off);
        if (n_eff) {
            float* eff = raw + f.n_w;
            for (int j = 0; j < n_eff; ++j) {
                float e = 0.0f;
                for (int dw = -h; dw <= h; ++dw) {
                    const int i = j - h - dw;
                    if (i >= 0 && i < f.n_w) e = fmaf((float)P.ww[dw + h], raw[i], e);
                }
                eff[j] = e;
            }
        }
        rec.a = (float)a;
        rec.tsum = __double2float_ru(st);
    }
    rec.w0 = f.w0;
    rec.t0 = f.t0;
    rec.n_w = f.n_w;
    rec.n_t = f.n_t;
    rec.pool = off;
    recs[u] = rec;
    if (!kFluct && ev.mode == 0)
        for_each_bin(P, f.w0, f.n_w, f.t0, f.n_t, [&](int c) { atomicAdd(&band_count[P.band_base + c], 1u); });
}

// The direct-path tile entries of one unit (every lane of the warp calls it;
// `live` false for lanes without a unit): a TEnt per (8-row group x window)
// tile the unit touches, with its row coefficients a eff[w]. Slots come from
// counter[] (warp-aggregated over the lanes that share a tile); put(b, slot,
// entry) stores them (CSR offsets in k_fill_bands, fixed-capacity lists in
// k_sample_off).
// base: the unit's profile words [raw][eff][tv] (global with kLdg, or the
// staging copy in shared memory / the unit's own global writes without).
template <bool kLdg, typename Put>
__device__ __forceinline__ void emit_tile_entries(const PlaneDesc& P, const UnitRec& rec, bool live,
                                                  const float* base, uint32_t* __restrict__ counter, Put&& put)
{
    auto ld = [&](const float* a) { return kLdg ? __ldg(a) : *a; };
    // row_coef (ws_common.cuh) on `base`: a * profile[j], j = (w - first row) mod W, every wrap summed
    auto coef = [&](int w, float& c) {
        const bool stencil = !P.ww_is_one;
        const int lo = stencil ? rec.w0 - P.h : rec.w0;
        const int nrw = stencil ? rec.n_w + 2 * P.h : rec.n_w;
        int j = w - lo;
        if (j < 0) j += P.W;
        else if (j >= P.W) j -= P.W;
        if (j >= P.W) j %= P.W;
        if (j >= nrw) return false;
        const float* pr = base + (stencil ? rec.n_w : 0);
        float acc = ld(&pr[j]);
        if (nrw > P.W)
            for (j += P.W; j < nrw; j += P.W) acc += ld(&pr[j]);
        c = acc * rec.a;
        return true;
    };
    const int L = rec.n_t + P.n_lags - 1;
    int ts = rec.t0 + P.lo_lag;
    if (ts < 0) ts += P.N;
    const uint32_t goff = rec.goff;
    // the unit's (stencilled) wire rows; units whose rows do not wrap around
    // the padded grid read their profile with branch-free predicated loads
    const bool stencil = !P.ww_is_one;
    const int lo_row = stencil ? rec.w0 - P.h : rec.w0;
    const int n_rows = stencil ? rec.n_w + 2 * P.h : rec.n_w;
    const bool simple = lo_row >= 0 && lo_row + n_rows <= P.W;
    const float* prof = base + (stencil ? rec.n_w : 0);
    // the entry for tile (row group c / n_windows, window c % n_windows)
    auto make_entry = [&](int c) {
        const int r0 = (c / P.n_windows) * kTileRows, nr = min(kTileRows, P.W - r0);
        TEnt d;
        d.tsL = (uint32_t)ts | ((uint32_t)L << 16);
        d.goff = goff;
        d.gbound = __fmul_ru(rec.tsum, P.kern_absmax);
        int rlo = kTileRows, rhi = 0;
        if (simple) {
#pragma unroll
            for (int r = 0; r < kTileRows; ++r) {
                const int j = r0 + r - lo_row;
                const bool in = r < nr && j >= 0 && j < n_rows;
                const float v = in ? ld(&prof[in ? j : 0]) : 0.0f;
                d.c[r] = v * rec.a;  // row_coef's product
            }
#pragma unroll
            for (int r = 0; r < kTileRows; ++r)
                if (d.c[r] != 0.0f) {
                    rlo = min(rlo, r);
                    rhi = r + 1;
                }
        } else {
#pragma unroll
            for (int r = 0; r < kTileRows; ++r) {
                float cr = 0.0f;
                if (r < nr && coef(r0 + r, cr) && cr != 0.0f) {
                    rlo = min(rlo, r);
                    rhi = r + 1;
                }
                d.c[r] = cr;
            }
        }
        d.rows = (uint32_t)rlo | ((uint32_t)max(rhi, rlo) << 8);
        return d;
    };
    // common case (rows not wrapping, <= 4 row groups x <= 2 windows): all the
    // slot atomics issued back to back before any entry is written, instead of
    // one dependent global round trip per entry
    const uint32_t wm = span_windows(ts, L, P.N, P.n_windows);
    const int g0 = lo_row / kTileRows, g1 = (lo_row + n_rows - 1) / kTileRows;
    const bool fast = live && simple && __popc(wm) <= 2 && g1 - g0 < 4;
    const unsigned act = __ballot_sync(0xffffffffu, fast);
    if (fast) {
        {
            const int w0 = __ffs(wm) - 1, w1 = __popc(wm) > 1 ? 31 - __clz(wm) : -1;
            // consecutive depos (one track) mostly share tiles: one atomic per
            // distinct tile of the warp, ranks by match mask
            uint32_t slot[8];
            const unsigned lt = (1u << lane_id()) - 1u;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int g = g0 + (k >> 1), w = (k & 1) ? w1 : w0;
                const bool valid = g <= g1 && w >= 0;
                const unsigned vm = __ballot_sync(act, valid);
                slot[k] = 0u;
                if (valid) {
                    const uint32_t b = P.band_base + g * P.n_windows + w;
                    const unsigned peers = __match_any_sync(vm, b);
                    const int leader = __ffs(peers) - 1;
                    uint32_t base = 0;
                    if (lane_id() == leader) base = atomicAdd(&counter[b], (unsigned)__popc(peers));
                    base = __shfl_sync(peers, base, leader);
                    slot[k] = base + __popc(peers & lt);
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int g = g0 + (k >> 1), w = (k & 1) ? w1 : w0;
                if (g <= g1 && w >= 0) {
                    const int c = g * P.n_windows + w;
                    put(P.band_base + c, slot[k], make_entry(c));
                }
            }
            return;
        }
    }
    if (!live) return;
    for_each_bin(P, rec.w0, rec.n_w, rec.t0, rec.n_t, [&](int c) {
        const uint32_t b = P.band_base + c;
        put(b, atomicAdd(&counter[b], 1u), make_entry(c));
    });
}

// Fluctuation-off sampling (the hot path), one thread per unit as k_sample,
// but the profiles [raw][eff][tv] are written through shared memory: every
// lane stages its unit's words, then the warp copies unit after unit with
// coalesced stores (per-lane scattered 4-byte stores were the limiter:
// 8.4M L2 sectors for 50 MB). Lanes past the warp's staging capacity write
// directly. On all-direct events the kernel also appends every unit's tile
// entries to the fixed-capacity per-tile lists (emit_tile_entries), which
// replaces the count scan and k_fill_bands.
constexpr int kSampleThreads = 128;
constexpr int kStageWarp = 32 * 52;  // staged profile words per warp

// kImp: some plane of the call has impact positions (a separate
// instantiation: the wire-binned hot path keeps its registers)
template <bool kImp>
__global__ void __launch_bounds__(kSampleThreads, 8)
k_sample_off(const EventDesc ev, UnitRec* __restrict__ recs, uint32_t* __restrict__ pool, uint32_t pool_cap,
             uint32_t* __restrict__ pool_ctr, uint32_t* __restrict__ band_count, unsigned* __restrict__ err)
{
    extern __shared__ float s_stage[];
    asm volatile("griddepcontrol.launch_dependents;");  // the profiles kernel may set up meanwhile
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    const bool in_range = u < ev.total_units;
    const int pi = in_range ? plane_of_unit(ev, u) : 0;
    const PlaneDesc& P = ev.p[pi];
    ws_depo d{};
    if (in_range) d = P.depos[u - P.unit_base];
    UnitRec rec;
    rec.w0 = -1;
    rec.t0 = 0;
    rec.n_w = 0;
    rec.n_t = 0;
    rec.pool = 0;
    rec.goff = 0;
    rec.a = 0.0f;
    rec.tsum = 0.0f;
    bool live = in_range;
    if (live && ev.drift_enabled && !drift(ev, d)) {
        atomicOr(err, kErrDomain);
        live = false;
    }
    Footprint f{};
    if (live) {
        if (d.q < 0) atomicOr(err, kErrCharge);
        f = footprint(P, d);
        if (f.clipped && P.stats_owner) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[1]), 1ULL);
        if (f.empty) {
            if (P.stats_owner) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[0]), (unsigned long long)d.q);
            live = false;
        }
    }
    const int h = P.h;
    const int n_eff = live && !P.ww_is_one ? f.n_w + 2 * h : 0;
    // warp-contiguous allocation, one atomic per warp: the 32 units' profiles
    // back to back [base, base + W), then their g regions (direct planes:
    // 8 header words, g[-1] = max|g|, then ceil32(L) taps: every g starts on a
    // 32-byte DRAM sector, so the profile writes never leave a partial sector
    // (a read-modify-write under HBM3's ECC; r2: 72 -> see DESIGN)
    const uint32_t words = live ? (uint32_t)(f.n_w + n_eff + f.n_t) : 0u;
    const uint32_t gneed = (live && ev.mode == 0 && P.direct) ? (((uint32_t)(f.n_t + P.n_lags - 1) + 31u) & ~31u) + 8u
                                                               : 0u;
    uint32_t wex = words, gex = gneed;  // inclusive scans -> exclusive below
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a = __shfl_up_sync(0xffffffffu, wex, o), b = __shfl_up_sync(0xffffffffu, gex, o);
        if (lane >= o) {
            wex += a;
            gex += b;
        }
    }
    const uint32_t w_tot = __shfl_sync(0xffffffffu, wex, 31), g_tot = __shfl_sync(0xffffffffu, gex, 31);
    wex -= words;
    gex -= gneed;
    const uint32_t w_pad = (w_tot + 3u) & ~3u;
    uint32_t base = 0;
    if (lane == 0 && w_tot + g_tot) base = atomicAdd(pool_ctr, w_pad + g_tot + 8u);
    base = __shfl_sync(0xffffffffu, base, 0);
    const uint32_t gbase = (base + w_pad + 7u) & ~7u;  // 32-byte aligned
    if ((uint64_t)base + w_pad + g_tot + 8u > pool_cap && (w_tot + g_tot)) {
        if (live) atomicOr(err, kErrPool);
        live = false;
    }
    const uint32_t off = base + wex;
    // everything above touched only this call's header slot; the pool, the
    // records and the tile lists may still be in use by the previous call's
    // k_direct when this kernel was launched programmatically behind it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const bool fast = live && d.sigma_x * 4.0 >= P.pitch && d.sigma_t * 4.0 >= P.tick;
    // the staged prefix of the warp's profile words (compact, same order as the pool)
    const bool staged = live && wex + words <= (uint32_t)kStageWarp;  // a prefix of the lanes
    float* stage = s_stage + warp * kStageWarp;
    double sw = 0.0, mw = 0.0, st = 0.0, mt = 0.0;
    double sw_all = 0.0, mw_all = 0.0;  // over every impact (== sw, mw without impact positions)
    float* raw = reinterpret_cast<float*>(pool + off);
    if (live) {
        rec.goff = gneed ? gbase + gex + 8u : 0u;
        const double wire_edge = P.origin_x + ((double)f.w0 - (double)P.pad_w) * P.pitch;
        const double tick_edge = P.origin_t + ((double)f.t0 - (double)P.pad_t) * P.tick;
        float* dst = staged ? stage + wex : raw;
        if (kImp && P.impacts > 1) {
            double o6[6];
            sample_impacts_ool(&d, P.pitch, P.tick, P.impacts, P.imp_mask, wire_edge, tick_edge, f.n_w, f.n_t, fast, dst,
                               dst + f.n_w + n_eff, o6);
            sw = o6[0];
            mw = o6[1];
            sw_all = o6[2];
            mw_all = o6[3];
            st = o6[4];
            mt = o6[5];
        } else if (fast) {
            float* tv = dst + f.n_w + n_eff;
            bin_integrals_f32(d.x, d.sigma_x, wire_edge, P.pitch, f.n_w, [&](int i, float v) { dst[i] = v; }, sw,
                              mw);
            bin_integrals_f32(d.t, d.sigma_t, tick_edge, P.tick, f.n_t, [&](int i, float v) { tv[i] = v; }, st, mt);
        } else {
            double o4[4];
            sample_f64_ool(&d, wire_edge, P.pitch, f.n_w, tick_edge, P.tick, f.n_t, dst, dst + f.n_w + n_eff, o4);
            sw = o4[0];
            mw = o4[1];
            st = o4[2];
            mt = o4[3];
        }
        if (!kImp || P.impacts == 1) {
            sw_all = sw;
            mw_all = mw;
        }
        if (n_eff) {
            float* eff = dst + f.n_w;
            for (int j = 0; j < n_eff; ++j) {
                float e = 0.0f;
                for (int dw = -h; dw <= h; ++dw) {
                    const int i = j - h - dw;
                    if (i >= 0 && i < f.n_w) e = fmaf((float)P.ww[dw + h], dst[i], e);
                }
                eff[j] = e;
            }
        }
    }
    // coalesced write-out of the staged prefix [base, base + n_staged)
    __syncwarp();
    uint32_t n_staged = staged ? wex + words : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) n_staged = max(n_staged, __shfl_xor_sync(0xffffffffu, n_staged, o));
    float* pw = reinterpret_cast<float*>(pool) + base;
    for (uint32_t k = lane; k < n_staged; k += 32) pw[k] = stage[k];
    // sum_w sum_t wv*tv > 0  <=>  max(wv)*max(tv) > 0; numerically empty
    // (rasterize.cpp:111-116) -> clipped charge (pipeline.cpp:339-340)
    bool emit = live;
    if (live && !(mw_all * mt > 0.0)) {
        if (P.stats_owner) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[0]), (unsigned long long)d.q);
        emit = false;
    } else if (kImp && live && !(mw * mt > 0.0)) {
        emit = false;  // impact positions: none of the depo's charge falls in this class's sub-bins
    }
    if (emit) {
        // S = q * p = a * wv[w] * tv[t] with a = q / total (applied by the consumers);
        // the total runs over every impact sub-bin
        rec.a = (float)((double)d.q / (sw_all * st));
        rec.tsum = __double2float_ru(st);
        rec.w0 = f.w0;
        rec.t0 = f.t0;
        rec.n_w = f.n_w;
        rec.n_t = f.n_t;
        rec.pool = off;
    } else {
        rec.goff = 0;
    }
    if (in_range) recs[u] = rec;
    if (ev.mode != 0) return;  // warp-uniform
    const bool fixed = emit && ev.tile_cap != 0 && P.direct;
    if (emit && !fixed)  // counts for the CSR lists (k_scan_bands -> k_fill_bands)
        for_each_bin(P, f.w0, f.n_w, f.t0, f.n_t, [&](int c) { atomicAdd(&band_count[P.band_base + c], 1u); });
    if (__any_sync(0xffffffffu, fixed)) {
        // fixed-capacity tile lists: this warp's entries straight away (the
        // profile from the staging copy, or the lane's own global writes)
        const float* prof = staged ? stage + wex : raw;
        const uint32_t cap = ev.tile_cap;
        emit_tile_entries<false>(P, rec, fixed, prof, ev.tile_count, [&](uint32_t b, uint32_t slot, const TEnt& e) {
            if (slot < cap) {
                ev.tiles[(size_t)b * cap + slot] = e;
            } else {
                // never dropped silently: the host sizes the re-run from the
                // real count (or routes the dense plane to the row FFT)
                atomicOr(err, kErrTileCap);
                atomicMax(P.tile_need, slot + 1u);
            }
        });
    }
}

// Exclusive scan of bin counts (single block); resets the fill cursors.
__global__ void __launch_bounds__(1024) k_scan_bands(uint32_t* __restrict__ count, uint32_t* __restrict__ off,
                                                    uint32_t* __restrict__ fill, uint32_t n)
{
    // one pass: each thread scans kPer consecutive counts in registers, the
    // block scans the 1024 partial sums (two warp-shuffle levels), carry
    // across passes only for n > 1024 * kPer
    constexpr int kPer = 8;
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll 1
    for (uint32_t base = 0; base < n; base += 1024u * kPer) {
        const uint32_t i0 = base + threadIdx.x * kPer;
        uint32_t v[kPer], sum = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            v[k] = i0 + k < n ? count[i0 + k] : 0u;
            sum += v[k];
        }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        __syncthreads();  // carry / warp_sums of the previous pass consumed
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t t = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            warp_sums[lane] = t;
        }
        __syncthreads();
        uint32_t run = carry + (wid ? warp_sums[wid - 1] : 0u) + x - sum;
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (i0 + k < n) {
                off[i0 + k] = run;
                fill[i0 + k] = 0;
                count[i0 + k] = 0;  // zero for the next call (no memset per call)
                run += v[k];
            }
        __syncthreads();
        if (threadIdx.x == 1023) carry = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) off[n] = carry;
}

// Thread per unit: append the unit to the list of every bin it touches.
// FFT planes list the unit record per band; direct planes list, per tile,
// the entry k_direct consumes: tick span, profile offset and the
// coefficient a eff[w] of each tile row (independent of k_gprof, which may
// run concurrently on the auxiliary stream). Lists larger
// than ev.list_cap (the scan's total) flag kErrRange and write nothing.
__global__ void k_fill_bands(const EventDesc ev, const UnitRec* __restrict__ recs, const uint32_t* __restrict__ off,
                             uint32_t* __restrict__ fill, UnitRec* __restrict__ list, TEnt* __restrict__ tlist,
                             const uint32_t* __restrict__ pool, unsigned* __restrict__ err)
{
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (off[ev.total_bands] > ev.list_cap) {  // grid-uniform
        if (u == 0) {
            atomicOr(err, kErrRange);
            *ev.list_need = off[ev.total_bands];  // the exact size for the re-run
        }
        return;
    }
    // no early exits below: the warp-collective tile-slot allocation needs every lane
    bool live = u < ev.total_units;
    UnitRec rec{};
    if (live) rec = recs[u];
    live = live && rec.w0 >= 0;
    const PlaneDesc& P = ev.p[plane_of_unit(ev, live ? u : 0)];
    if (live && !P.direct) {
        for_each_bin(P, rec.w0, rec.n_w, rec.t0, rec.n_t, [&](int c) {
            const uint32_t b = P.band_base + c;
            list[off[b] + atomicAdd(&fill[b], 1u)] = rec;  // full record: k_conv streams the list
        });
        live = false;
    }
    emit_tile_entries<true>(P, rec, live, reinterpret_cast<const float*>(pool + rec.pool), fill,
                            [&](uint32_t b, uint32_t slot, const TEnt& e) { tlist[off[b] + slot] = e; });
}

// RN(t / d) for the walk's pmf recursion (rng.cpp:165-168: pmf *= odds * (n -
// k) / (k + 1)), d = k + 1 an integer: with y = RN(1/d) from a table, q =
// RN(t y) is within one ulp of t/d, the residual r = t - q d is exact (one
// FMA), and RN(q + r y) is the correctly rounded quotient (Markstein's
// theorem, round-to-nearest, no under/overflow: t is a moderate odds ratio
// times n - k). Three dependent fp64 operations instead of the IEEE division
// sequence; the same bits as the reference's division (checked on the full
// configs[2] event, tests/test_gpu_fullsize.py). Larger d: the division.
constexpr double kMarksteinMin = 0x1p-900;  // t >= this: q and the residual stay normal
__device__ __forceinline__ double div_rn_y(double t, double d, double y)
{
    const double q = __dmul_rn(t, y);
    const double r = __fma_rn(-q, d, t);
    return __fma_rn(r, y, q);
}

// Electron counts into the integer charge grid (the reference's ChargeGrid is
// int64, core.hpp:94-99): integer reductions (fire and forget: the walk never
// waits on them), exact and order independent, into u64 cells or - when the
// plane's depos carry fewer than 2^32 electrons - u32 cells (CellPtr).

// Fluctuation walk, one thread per unit: sample_patch's exact probabilities
// (rasterize.cpp:101-118) then fluctuate_sequential (rasterize.cpp:124-149)
// with the reference binomial (rng.cpp:146-193) or the Gaussian approximation
// (rasterize.cpp:159-170); counts scattered with integer atomics (CellPtr).
__global__ void k_fluctuate(const EventDesc ev, const UnitRec* __restrict__ recs, const uint32_t* __restrict__ pool,
                            const uint32_t* __restrict__ order)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ev.total_units) return;
    const uint32_t u = order ? order[i] : i;
    const UnitRec rec = recs[u];
    if (rec.w0 < 0) return;
    const PlaneDesc& P = ev.p[plane_of_unit(ev, u)];
    const ws_depo d = P.depos[u - P.unit_base];
    const double* wv = reinterpret_cast<const double*>(pool + rec.pool);
    const double* tv = wv + rec.n_w;
    const int n_w = rec.n_w, n_t = rec.n_t;
    double total = 0.0;
    for (int w = 0; w < n_w; ++w) {
        const double pw = wv[w];
        for (int t = 0; t < n_t; ++t) total += pw * tv[t];
    }
    const double norm = 1.0 / total;
    Rng src;
    src.init(ev.rng_mode, ev.seed, (uint64_t)d.id);
    const bool wide = cnt_wide(P);
    const int N = P.N;
    int64_t remaining = d.q;
    double p_rem = 1.0;
    const int last = n_w * n_t - 1;
    for (int b = 0; b < last; ++b) {
        if (remaining == 0) break;
        const int w = b / n_t, t = b - w * n_t;
        const double pi = (wv[w] * tv[t]) * norm;
        double p = 1.0;
        if (p_rem > 0.0) {
            p = pi / p_rem;
            p = p < 0.0 ? 0.0 : (p > 1.0 ? 1.0 : p);
        }
        const int64_t k = ev.approx ? binomial_approx(remaining, p, src) : binomial(remaining, p, src);
        cell_at(P, (size_t)(rec.w0 + w) * N + rec.t0 + t, wide).add(k);
        remaining -= k;
        p_rem -= pi;
    }
    if (remaining) cell_at(P, (size_t)(rec.w0 + n_w - 1) * N + rec.t0 + n_t - 1, wide).add(remaining);
}

// Exact fluctuation (fluctuate_sequential with the reference binomial), the
// same per-depo operation sequence as k_fluctuate, scheduled for SIMT: the
// nested loop (bins x CDF-walk steps) diverges per bin (the warp pays the
// longest walk of every bin), so each lane runs a state machine instead -
// lanes walk their current draw one step per iteration and only when a
// quarter of the warp's live lanes have finished their draws does the warp
// set up the next draws (RNG, pmf seed) together. The integer grid is
// unchanged (same draws, same order per depo; exact integer atomics).
// Scheduling orders of the exact walk, by bucket (counting) sort: units by
// descending charge (the walk is ~q steps: warps of similar charge keep their
// lanes busy together) and by descending bin count (k_fluct_prep's per-lane
// work). Only the schedule depends on these orders, never the counts (each
// unit's draws come from its own stream), so buckets need not be exact and
// the order inside a bucket may vary. No memsets: a large CUB sort's
// cudaMemsetAsync calls queue on a copy engine behind the previous event's
// frame copies (end-to-end calls).
constexpr int kFlBq = 1056;  // charge buckets: 0 (q <= 0), then log2 x 32 sub-buckets
constexpr int kFlBb = 4096;  // bin-count buckets (counts >= 4095 share the last)
__device__ __forceinline__ uint32_t fl_bucket_q(int64_t q)
{
    if (q <= 0) return 0u;
    const uint64_t v = (uint64_t)q;
    const int l = 63 - __clzll((long long)v);
    const uint32_t frac = l >= 5 ? (uint32_t)(v >> (l - 5)) & 31u : (uint32_t)(v << (5 - l)) & 31u;
    return min(1u + 32u * (uint32_t)l + frac, (uint32_t)kFlBq - 1u);
}
__global__ void k_fluct_hist_zero(uint32_t* __restrict__ hist, uint32_t* __restrict__ n_slow)
{
    for (int i = threadIdx.x; i < kFlBq + kFlBb; i += blockDim.x) hist[i] = 0u;
    if (threadIdx.x == 0) n_slow[0] = 0u;
}
// Both histograms are counted per block in shared memory (kFlPer units per
// thread) and added to the global ones once per non-empty bucket: hot buckets
// (a track's depos share them) no longer serialise on one global atomic
// address per warp (r2: keys + scatter 100 -> < 40 us per C3 event)
constexpr int kFlSortThreads = 1024, kFlPer = 4;
__global__ void __launch_bounds__(kFlSortThreads) k_fluct_keys(const EventDesc ev, const UnitRec* __restrict__ recs,
                                                               uint32_t* __restrict__ bq, uint32_t* __restrict__ bb,
                                                               uint32_t* __restrict__ hist)
{
    __shared__ uint32_t h[kFlBq + kFlBb];
    for (int i = threadIdx.x; i < kFlBq + kFlBb; i += kFlSortThreads) h[i] = 0u;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kFlPer; ++k) {
        const uint32_t u = (blockIdx.x * kFlPer + k) * kFlSortThreads + threadIdx.x;
        if (u < ev.total_units) {
            const PlaneDesc& P = ev.p[plane_of_unit(ev, u)];
            const UnitRec r = recs[u];
            const int64_t q = r.w0 >= 0 ? P.depos[u - P.unit_base].q : 0;
            const uint32_t kq = (uint32_t)kFlBq - 1u - fl_bucket_q(q);  // descending
            const uint32_t kb =
                (uint32_t)kFlBb - 1u - (r.w0 >= 0 ? min((uint32_t)(r.n_w * r.n_t), (uint32_t)kFlBb - 1u) : 0u);
            bq[u] = kq;
            bb[u] = kb;
            atomicAdd(&h[kq], 1u);
            atomicAdd(&h[kFlBq + kb], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kFlBq + kFlBb; i += kFlSortThreads)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}
// exclusive scans of both histograms, in place (one block)
__global__ void __launch_bounds__(1024) k_fluct_hist_scan(uint32_t* __restrict__ hist)
{
    __shared__ uint32_t part[1024];
    for (int h = 0; h < 2; ++h) {
        uint32_t* a = hist + (h ? kFlBq : 0);
        const int n = h ? kFlBb : kFlBq;
        const int per = (n + 1023) / 1024, i0 = threadIdx.x * per;
        uint32_t sum = 0;
        for (int i = i0; i < min(i0 + per, n); ++i) sum += a[i];
        part[threadIdx.x] = sum;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const uint32_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
            __syncthreads();
            part[threadIdx.x] += v;
            __syncthreads();
        }
        uint32_t run = part[threadIdx.x] - sum;
        for (int i = i0; i < min(i0 + per, n); ++i) {
            const uint32_t c = a[i];
            a[i] = run;
            run += c;
        }
        __syncthreads();
    }
}
__global__ void __launch_bounds__(kFlSortThreads) k_fluct_scatter(uint32_t n, const uint32_t* __restrict__ bq,
                                                                  const uint32_t* __restrict__ bb,
                                                                  uint32_t* __restrict__ hist, uint32_t* __restrict__ by_q,
                                                                  uint32_t* __restrict__ by_b)
{
    // ranks inside the block's share of each bucket, then one global claim
    // per non-empty bucket (the order inside a bucket is free)
    __shared__ uint32_t h[kFlBq + kFlBb];
    for (int i = threadIdx.x; i < kFlBq + kFlBb; i += kFlSortThreads) h[i] = 0u;
    __syncthreads();
    uint32_t kq[kFlPer], kb[kFlPer], rq[kFlPer], rb[kFlPer];
#pragma unroll
    for (int k = 0; k < kFlPer; ++k) {
        const uint32_t u = (blockIdx.x * kFlPer + k) * kFlSortThreads + threadIdx.x;
        if (u < n) {
            kq[k] = bq[u];
            kb[k] = kFlBq + bb[u];
            rq[k] = atomicAdd(&h[kq[k]], 1u);
            rb[k] = atomicAdd(&h[kb[k]], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kFlBq + kFlBb; i += kFlSortThreads)
        if (h[i]) h[i] = atomicAdd(&hist[i], h[i]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kFlPer; ++k) {
        const uint32_t u = (blockIdx.x * kFlPer + k) * kFlSortThreads + threadIdx.x;
        if (u < n) {
            by_q[h[kq[k]] + rq[k]] = u;
            by_b[h[kb[k]] + rb[k]] = u;
        }
    }
}

// n_list (nullable): the number of entries of `order` (device), else total_units
__global__ void __launch_bounds__(128) k_fluctuate_exact(const EventDesc ev, const UnitRec* __restrict__ recs,
                                                          const uint32_t* __restrict__ pool,
                                                          const uint32_t* __restrict__ order,
                                                          const uint32_t* __restrict__ n_list)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    bool done = i >= (n_list ? *n_list : ev.total_units);
    const uint32_t u = done ? 0u : (order ? order[i] : i);
    UnitRec rec{};
    if (!done) rec = recs[u];
    done = done || rec.w0 < 0;
    const PlaneDesc& P = ev.p[plane_of_unit(ev, done ? 0 : u)];
    ws_depo d{};
    if (!done) d = P.depos[u - P.unit_base];
    const double* wv = reinterpret_cast<const double*>(pool + rec.pool);
    const double* tv = wv + rec.n_w;
    const int n_t = rec.n_t;
    double norm = 0.0;
    if (!done) {
        double total = 0.0;
        for (int w = 0; w < rec.n_w; ++w) {
            const double pw = wv[w];
            for (int t = 0; t < n_t; ++t) total += pw * tv[t];
        }
        norm = 1.0 / total;
    }
    Rng src;
    src.init(ev.rng_mode, ev.seed, (uint64_t)d.id);
    const int N = P.N;
    const int last = rec.n_w * n_t - 1;
    int64_t remaining = d.q;
    double p_rem = 1.0, pi = 0.0;
    int b = 0;
    // the draw in progress (invert_binomial_cdf's loop state)
    bool walking = false, flip = false;
    int64_t n = 0;
    double odds = 0.0, pmf = 0.0, cdf = 0.0, uu = 0.0, kd = 0.0, nd = 0.0, nk = 0.0, k1 = 0.0;
    int kr = 0;

    // bin b = (bw, bt), tracked incrementally (no integer division per draw)
    int bw = 0, bt = 0;
    const bool wide = cnt_wide(P);
    CellPtr cellp = cell_at(P, (size_t)rec.w0 * N + rec.t0, wide);  // grid[w0 + bw][t0 + bt]
    auto commit = [&](int64_t k) {  // bin b drew k electrons
        cellp.add(k);
        remaining -= k;
        p_rem -= pi;
        ++b;
        if (++bt == n_t) {
            bt = 0;
            ++bw;
            cellp.advance(N - (n_t - 1));
        } else {
            cellp.advance(1);
        }
    };
    // draws until one needs a CDF walk (or the depo is finished)
    auto setup = [&]() {
        while (!done && !walking) {
            if (remaining == 0 || b >= last) {
                if (remaining)  // the last bin takes the rest
                    cell_at(P, (size_t)(rec.w0 + rec.n_w - 1) * N + rec.t0 + n_t - 1, wide).add(remaining);
                done = true;
                break;
            }
            pi = (wv[bw] * tv[bt]) * norm;
            double p = 1.0;
            if (p_rem > 0.0) {
                p = pi / p_rem;
                p = p < 0.0 ? 0.0 : (p > 1.0 ? 1.0 : p);
            }
            // binomial (rng.cpp:174-193)
            n = remaining;
            if (p == 0.0) {
                commit(0);
                continue;
            }
            if (p == 1.0) {
                commit(n);
                continue;
            }
            const double mean = __dmul_rn((double)n, p);
            const double var = __dmul_rn(mean, __dsub_rn(1.0, p));
            const double q1 = __dsub_rn(1.0, p);
            const double mn = (q1 < p) ? q1 : p;
            if (__dmul_rn((double)n, mn) > 1e6) {
                const double k = round(__dadd_rn(mean, __dmul_rn(sqrt(var), src.normal())));
                commit(k < 0.0 ? 0 : (k > (double)n ? n : (int64_t)k));
                continue;
            }
            uu = src.uniform();
            flip = p > 0.5;
            const double pp = flip ? q1 : p;
            // invert_binomial_cdf (rng.cpp:146-170): the pmf seed
            odds = __ddiv_rn(pp, __dsub_rn(1.0, pp));
            int64_t k = 0;
            const double log_pmf0 = __dmul_rn((double)n, log1p(-pp));
            if (log_pmf0 > -700.0) {
                pmf = exp_ref(log_pmf0);
            } else {
                const double m2 = __dmul_rn((double)n, pp);
                const double sd = sqrt(__dmul_rn(m2, __dsub_rn(1.0, pp)));
                const int64_t k0 = (int64_t)__dsub_rn(m2, __dmul_rn(30.0, sd));
                k = k0 > 0 ? k0 : 0;
                const double nn = (double)n, kk = (double)k;
                double e = __dsub_rn(lgamma(__dadd_rn(nn, 1.0)), lgamma(__dadd_rn(kk, 1.0)));
                e = __dsub_rn(e, lgamma(__dadd_rn(__dsub_rn(nn, kk), 1.0)));
                e = __dadd_rn(e, __dmul_rn(kk, log(pp)));
                e = __dadd_rn(e, __dmul_rn(__dsub_rn(nn, kk), log1p(-pp)));
                pmf = exp_ref(e);
            }
            cdf = pmf;
            if (cdf <= uu && k < n) {
                walking = true;
                kd = (double)k;
                nd = (double)n;
                nk = (double)(n - k);  // exact integers below 2^53: the reference's casts
                k1 = (double)(k + 1);
                // table index of the next divisor; tiny odds (t = odds (n - k)
                // near the subnormal range) keep the IEEE division
                kr = k + 1 < (int64_t)kRecipN && odds >= kMarksteinMin ? (int)(k + 1) : kRecipN;
            } else {
                commit(flip ? n - k : k);
            }
        }
    };

#pragma unroll 1
    for (;;) {
        setup();
        const unsigned alive = __ballot_sync(0xffffffffu, !done);
        if (!alive) break;
        const int quorum = max(1, (__popc(alive) * ev.fl_quorum) >> 4);  // this share of the live lanes idle: set up together
#pragma unroll 1
        for (;;) {
            if (walking) {
                // kWalk CDF steps per iteration. The recursion factor
                // f_i = RN(RN(odds (n - k - i)) / (k + i + 1)) does not depend
                // on the pmf: the kWalk factors are independent (pipelined),
                // and only pmf *= f, cdf += pmf and the stop test (the
                // reference's loop condition, evaluated after every step)
                // form the serial chain. Steps past the stop are discarded.
                constexpr int kWalk = 4;
                double f[kWalk];
                if (kr + kWalk <= kRecipN) {  // divisors k + 1 .. k + kWalk from the table
#pragma unroll
                    for (int i = 0; i < kWalk; ++i)
                        f[i] = div_rn_y(__dmul_rn(odds, nk - (double)i), k1 + (double)i, __ldg(&ev.recip[kr + i]));
                } else {
#pragma unroll
                    for (int i = 0; i < kWalk; ++i) f[i] = __ddiv_rn(__dmul_rn(odds, nk - (double)i), k1 + (double)i);
                }
                double p = pmf, c = cdf, kk = kd;
                bool go = true;
#pragma unroll
                for (int i = 0; i < kWalk; ++i) {
                    if (go) {
                        p = __dmul_rn(p, f[i]);
                        c = __dadd_rn(c, p);
                        kk += 1.0;
                        go = c <= uu && kk < nd;
                    }
                }
                const double adv = kk - kd;
                pmf = p;
                cdf = c;
                kd = kk;
                nk -= adv;
                k1 += adv;
                kr += (int)adv;
                if (!go) {
                    walking = false;
                    const int64_t k = (int64_t)kd;
                    commit(flip ? n - k : k);
                }
            }
            const unsigned wk = __ballot_sync(0xffffffffu, walking);
            if (wk == 0 || __popc(alive & ~wk) >= quorum) break;
        }
    }
}


// ---- exact walk, two passes -------------------------------------------------
// The draws of a depo are sequential only through n = remaining: every other
// input of bin b's draw - its conditional probability p_b (the running p_rem
// subtraction, rasterize.cpp:141-147), pp = min(p, 1 - p), log1p(-pp) and the
// uniform it consumes (bins with p in (0, 1) consume one each, in bin order,
// as long as no draw can take binomial's normal branch: q min(p, 1 - p) <=
// 1e6 for every bin, since n <= q) - is fixed by the patch. k_fluct_prep
// computes them for all bins, one lane per unit with the same work per bin;
// k_fluct_walk then runs only what depends on n: n log1p(-pp), the pmf seed
// exp(n log1p(-pp)) (lgamma seed past -700) and the CDF walk. The reference's
// operations and their order are unchanged (the same values are computed,
// some earlier). Units that could reach the normal branch, and units whose
// records do not fit the buffer, take the one-pass walk (k_fluctuate_exact)
// whole (kErrFluct only tells the host to grow the buffer).
constexpr uint32_t kFlNone = 0xffffffffu;
#ifndef WS_FLWALK_MINB
#define WS_FLWALK_MINB 6  // 80 registers, 24 warps per SM (r2 re-sweep with skip records: 6 x 10 steps 3.20 ms, 7 x 7 3.36, 7 x 9 3.30, 8 x 7 3.52)
#endif
#ifndef WS_FLWALK_PF
#define WS_FLWALK_PF 3
#endif
#ifndef WS_FLWALK_PF2
#define WS_FLWALK_PF2 0
#endif
enum : uint32_t { kFlDraw = 0u, kFlDrawFlip = 1u, kFlZero = 2u, kFlAll = 3u, kFlSkip = 4u };
#ifndef WS_FL_SKIP
#define WS_FL_SKIP 1  // runs of certain-zero draws as one skip record (0: off)
#endif
#ifndef WS_FL_CHEAPMAX
#define WS_FL_CHEAPMAX 1
#endif
#ifndef WS_PREP_UNROLL
#define WS_PREP_UNROLL 4  // (r2: 964 -> 902 us per C3 event; the draws of four bins overlap)
#endif
constexpr int kPrepUnroll = WS_PREP_UNROLL;

// One bin's draw inputs, 32 B (one sector).
struct __align__(32) FlRec {
    double pp;   // min(p, 1 - p) (the walk's p, rng.cpp:191-192)
    double lg;   // log1p(-pp)
    double u;    // the draw's uniform
    float lnu;   // logf(u) (|error| < 7.7e-6; +inf below u = 1e-30): k = 0 test without exp
    uint32_t cls;  // kFlDraw / kFlDrawFlip (p > 0.5) / kFlZero (p == 0) / kFlAll (p == 1)
};
static_assert(sizeof(FlRec) == 32, "one sector per record");
// a run of m draws that take 0 electrons: class kFlSkip, m in the lnu slot
// and, in the first slot, the cell advance over the run and the tick the run ends on
__device__ __forceinline__ void fl_skip_record(FlRec* r, uint32_t m, int adv, int bt_end)
{
    reinterpret_cast<double2*>(r)[0] = make_double2(__hiloint2double(bt_end, adv), 0.0);
    reinterpret_cast<double2*>(r)[1] = make_double2(0.0, __hiloint2double((int)kFlSkip, (int)m));
}

#ifndef WS_PREP_MINB
#define WS_PREP_MINB 1
#endif
__global__ void __launch_bounds__(128, WS_PREP_MINB) k_fluct_prep(const EventDesc ev, const UnitRec* __restrict__ recs,
                                                     const uint32_t* __restrict__ pool,
                                                     const uint32_t* __restrict__ order, uint32_t* __restrict__ offs,
                                                     uint32_t* __restrict__ slow, uint32_t* __restrict__ n_slow,
                                                     uint32_t* __restrict__ cursor, uint32_t first)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if (i == 0) *cursor = first;  // k_fluct_walk's unit cursor (its lanes start with units [0, first))
    const bool in = i < ev.total_units;
    const uint32_t u = in ? order[i] : 0u;  // units by bin count: the lanes of a warp do similar work
    UnitRec rec{};
    rec.w0 = -1;
    if (in) rec = recs[u];
    const bool live = in && rec.w0 >= 0;
    const uint32_t need = live ? (uint32_t)(rec.n_w * rec.n_t - 1) : 0u;  // draws: every bin but the last
    // warp-aggregated allocation of the records
    uint32_t incl = need;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && tot) base = atomicAdd(ev.fl_ctr, (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 31);
    if (!in) return;
    if (!live) {
        offs[u] = kFlNone;
        return;
    }
    const unsigned long long off = base + incl - need;
    if (off + need > ev.fl_cap || off + need > 0xfffffffeull) {
        atomicOr(ev.err, kErrFluct);
        offs[u] = kFlNone;
        slow[atomicAdd(n_slow, 1u)] = u;
        return;
    }
    const PlaneDesc& P = ev.p[plane_of_unit(ev, u)];
    const ws_depo d = P.depos[u - P.unit_base];
    const double* wv = reinterpret_cast<const double*>(pool + rec.pool);
    const double* tv = wv + rec.n_w;
    const int n_t = rec.n_t;
    double total = 0.0;
    for (int w = 0; w < rec.n_w; ++w) {
        const double pw = wv[w];
        for (int t = 0; t < n_t; ++t) total += pw * tv[t];
    }
    const double norm = 1.0 / total;
    Rng src;
    src.init(ev.rng_mode, ev.seed, (uint64_t)d.id);
    // uniform01 (rng.cpp:51-54); Philox: each block computed once for its two draws
    uint64_t odd_half = 0;
    auto uniform = [&]() -> double {
        if (ev.rng_mode == WS_RNG_SUBSTREAM) return src.uniform();
        const uint32_t k = src.draw++;
        uint64_t x = odd_half;
        if (!(k & 1u)) src.philox_block(k >> 1, x, odd_half);
        return (double)(x >> 11) * 0x1.0p-53;
    };
    const double qd = (double)d.q;
    FlRec* out = reinterpret_cast<FlRec*>(ev.fl_bins) + off;
    double p_rem = 1.0;
    bool slow_unit = false;
    int bw = 0, bt = 0;
    int zs = -1, zbw = 0, zbt = 0;  // first record of the current run of certain-zero draws, its bin
    const bool can_skip = (long long)rec.n_w * P.N < (1ll << 31);  // a skip's cell advance fits its int32 slot
    // the bin's weights are loaded one bin ahead (bin need, the last, is in
    // range): the L1 latency hides behind the previous bin's draw (r2: prep
    // 0.89 -> 0.85 ms per C3 event)
    double cw = wv[0], ct = tv[0];
#pragma unroll kPrepUnroll
    for (uint32_t b = 0; b < need; ++b) {
        const double pi = (cw * ct) * norm;
        {
            const int nt = bt + 1 == n_t ? 0 : bt + 1;
            const int nw = bt + 1 == n_t ? bw + 1 : bw;
            cw = wv[nw];
            ct = tv[nt];
        }
        double p = 1.0;
        if (p_rem > 0.0) {
            p = pi / p_rem;
            p = p < 0.0 ? 0.0 : (p > 1.0 ? 1.0 : p);
        }
        FlRec r;
        r.pp = 0.0;
        r.lg = 0.0;
        r.u = 0.0;
        r.lnu = 0.0f;
        r.cls = p == 0.0 ? kFlZero : kFlAll;
        if (p > 0.0 && p < 1.0) {
            const double q1 = __dsub_rn(1.0, p);
            const double mn = (q1 < p) ? q1 : p;
            slow_unit |= __dmul_rn(qd, mn) > 1e6;
            r.cls = p > 0.5 ? kFlDrawFlip : kFlDraw;
            r.pp = p > 0.5 ? q1 : p;
            r.lg = log1p(-r.pp);
            r.u = uniform();
            // log(u) for the walk's k = 0 test: |logf - ln u| <= 1 ulp (<= 7.6e-6
            // at u >= 1e-30) + the float rounding of u (6e-8); +inf disables the
            // test for smaller u
            r.lnu = r.u >= 1e-30 ? logf((float)r.u) : INFINITY;
        }
        double4 v0 = make_double4(r.pp, r.lg, r.u, 0.0);
        reinterpret_cast<uint32_t*>(&v0.w)[0] = __float_as_uint(r.lnu);
        reinterpret_cast<uint32_t*>(&v0.w)[1] = r.cls;
#if WS_FL_SKIP
        // a draw that takes 0 electrons for any n <= q (n log1p(-pp) >=
        // q log1p(-pp) passes the walk's k = 0 test) or p == 0: a run of them
        // is one skip record (the run's first slot; the others are never read
        // and never written)
        const double xq = __dmul_rn(qd, r.lg);
        const bool cz = can_skip && (r.cls == kFlZero || (r.cls == kFlDraw && xq > -700.0 && xq > (double)r.lnu + 4e-5));
        if (cz) {
            if (zs < 0) {
                zs = (int)b;
                zbw = bw;
                zbt = bt;
            }
        } else {
            if (zs >= 0) {
                fl_skip_record(out + zs, (uint32_t)((int)b - zs), (bw - zbw) * P.N + (bt - zbt), bt);
                zs = -1;
            }
            reinterpret_cast<double2*>(out + b)[0] = make_double2(v0.x, v0.y);
            reinterpret_cast<double2*>(out + b)[1] = make_double2(v0.z, v0.w);
        }
#else
        reinterpret_cast<double2*>(out + b)[0] = make_double2(v0.x, v0.y);
        reinterpret_cast<double2*>(out + b)[1] = make_double2(v0.z, v0.w);
#endif
        p_rem -= pi;
        if (++bt == n_t) {
            bt = 0;
            ++bw;
        }
    }
#if WS_FL_SKIP
    if (zs >= 0) fl_skip_record(out + zs, (uint32_t)((int)need - zs), (bw - zbw) * P.N + (bt - zbt), bt);
#endif
    if (slow_unit) {
        offs[u] = kFlNone;
        slow[atomicAdd(n_slow, 1u)] = u;
    } else {
        offs[u] = (uint32_t)off;
    }
}

// The walk over k_fluct_prep's records: persistent lanes (a grid that fills
// the GPU once) take units from a shared cursor over the charge-sorted
// order, so a lane whose depo is finished takes the next one instead of
// idling until its warp's longest depo ends. Per lane the state machine of
// k_fluctuate_exact: setting up draws is a loop over the records that settles
// the cheap ones without exp (p == 0, p == 1, and k = 0 when n log1p(-pp) >
// log(u) + 4e-5: then (1 - pp)^n > u for the reference's exp as for ours) and
// stops at the first draw that needs its pmf seed; the warp's seeds are then
// computed together, and the warp walks until a quorum of its lanes is idle.
// The walk takes kWalk CDF steps per iteration: the recursion factors are
// independent, the serial chain is pmf *= f, cdf += pmf, and as the CDF never
// decreases the stop is the first step with cdf > u.
#ifdef WS_WALK_PROF
__device__ unsigned long long g_walkprof[16];
#endif
__global__ void __launch_bounds__(128, WS_FLWALK_MINB) k_fluct_walk(const EventDesc ev, const UnitRec* __restrict__ recs,
                                                     const uint32_t* __restrict__ order,
                                                     const uint32_t* __restrict__ offs, uint32_t* __restrict__ cursor)
{
    const int lane = threadIdx.x & 31;
    // the lane's unit
    bool has = false, exhausted = false;
    int64_t remaining = 0;
    int n_t = 0, last = 0, b = 0, bt = 0, N = 0;
    CellPtr cellp{nullptr, 3}, lastp{nullptr, 3};
    const FlRec* rp = nullptr;
    // the draw in progress
    bool walking = false, flip = false;
    int64_t n = 0;
    double odds = 0.0, pmf = 0.0, cdf = 0.0, uu = 0.0, kd = 0.0, nd = 0.0, nk = 0.0, k1 = 0.0;
    int kr = 0;

    auto take = [&](uint32_t idx) {  // start unit order[idx] (if it has records)
        if (idx >= ev.total_units) {
            exhausted = true;
            return;
        }
        const uint32_t u = order[idx];
        const uint32_t off = offs[u];
        if (off == kFlNone) return;  // empty, or the one-pass walk's
        const UnitRec rec = recs[u];
        const PlaneDesc& P = ev.p[plane_of_unit(ev, u)];
        remaining = P.depos[u - P.unit_base].q;
        N = P.N;
        n_t = rec.n_t;
        last = rec.n_w * n_t - 1;
        b = 0;
        bt = 0;
        const bool wide = cnt_wide(P);
        cellp = cell_at(P, (size_t)rec.w0 * N + rec.t0, wide);
        lastp = cell_at(P, (size_t)(rec.w0 + rec.n_w - 1) * N + rec.t0 + n_t - 1, wide);
        rp = reinterpret_cast<const FlRec*>(ev.fl_bins) + off;
        has = true;
    };
    auto commit = [&](int64_t k) {
        cellp.add(k);
        remaining -= k;
        ++b;
        ++rp;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + WS_FLWALK_PF));
        if (WS_FLWALK_PF2 > 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + WS_FLWALK_PF2));
        if (++bt == n_t) {
            bt = 0;
            cellp.advance(N - (n_t - 1));
        } else {
            cellp.advance(1);
        }
    };
    take(blockIdx.x * blockDim.x + threadIdx.x);

    int64_t kdone = -1;  // a draw the walk finished, committed by the next setup (all idle lanes together)
#ifdef WS_WALK_PROF
    unsigned long long wp[16] = {};
#endif
    auto setup = [&]() {
#ifdef WS_WALK_PROF
        const long long wp_c = clock64();
#endif
        if (kdone >= 0) {
            commit(kdone);
            kdone = -1;
        }
#ifdef WS_WALK_PROF
        __syncwarp();
        wp[11] += clock64() - wp_c;
        const long long wp_l = clock64();
#endif
        bool seed = false;  // the current draw needs its pmf seed
        double pp = 0.0, lg = 0.0, x = 0.0;
#pragma unroll 1
        for (;;) {
            // lanes without a unit take the next ones (one atomic per warp)
            const unsigned want = __ballot_sync(0xffffffffu, !has && !exhausted);
#ifdef WS_WALK_PROF
            wp[13] += 1;
            if (want) wp[8] += 1;
#endif
            if (want) {
                uint32_t base = 0;
                if (lane == __ffs(want) - 1) base = atomicAdd(cursor, (uint32_t)__popc(want));
                base = __shfl_sync(0xffffffffu, base, __ffs(want) - 1);
                if (want & (1u << lane)) take(base + __popc(want & ((1u << lane) - 1u)));
                continue;
            }
            // cheap draws until one needs its seed, the unit ends, or the lane walks
            // at most WS_FL_CHEAPMAX settled draws per lane per setup pass: a
            // lane with a long run of p = 0 / p = 1 / k = 0 draws no longer holds
            // the warp in setup; it settles one and counts as idle for the quorum
            // (r2: walk 4.40 -> 4.13 ms per C3 event with quorum 8/16)
            int cheap = 0;
            while (has && !walking && !seed && cheap++ < WS_FL_CHEAPMAX) {
#ifdef WS_WALK_PROF
                wp[14] += 1;
#endif
                if (remaining == 0 || b >= last) {
                    if (remaining) lastp.add(remaining);  // the last bin takes the rest
                    has = false;
                    break;
                }
                const double2 ra = __ldg(reinterpret_cast<const double2*>(rp));
                const double2 rb = __ldg(reinterpret_cast<const double2*>(rp) + 1);
                const uint32_t cls = __double2hiint(rb.y);
                n = remaining;
                if (cls == kFlSkip) {  // a run of m draws that take 0 electrons
                    const int m = __double2loint(rb.y);
                    cellp.advance((long long)__double2loint(ra.x));  // (prep: rows x N + ticks)
                    bt = __double2hiint(ra.x);
                    b += m;
                    rp += m;
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + WS_FLWALK_PF));
                    continue;
                }
                if (cls == kFlZero) {
                    commit(0);
                    continue;
                }
                if (cls == kFlAll) {
                    commit(n);
                    continue;
                }
                flip = cls == kFlDrawFlip;
                pp = ra.x;
                lg = ra.y;
                x = __dmul_rn((double)n, lg);
                if (x > -700.0 && x > (double)__int_as_float(__double2loint(rb.y)) + 4e-5) {
                    commit(flip ? n : 0);  // (1 - pp)^n > u: k = 0
                    continue;
                }
                uu = rb.x;
                seed = true;
            }
            if (!__any_sync(0xffffffffu, !has && !exhausted)) break;
        }
#ifdef WS_WALK_PROF
        __syncwarp();
        wp[12] += clock64() - wp_l;
        const long long wp_sd = clock64();
        wp[10] += __popc(__ballot_sync(0xffffffffu, seed));
#endif
        if (seed) {
            // invert_binomial_cdf (rng.cpp:146-170): the pmf seed
            odds = __ddiv_rn(pp, __dsub_rn(1.0, pp));
            int64_t k = 0;
            if (x > -700.0) {
                pmf = exp_ref(x);
            } else {
                const double m2 = __dmul_rn((double)n, pp);
                const double sd = sqrt(__dmul_rn(m2, __dsub_rn(1.0, pp)));
                const int64_t k0 = (int64_t)__dsub_rn(m2, __dmul_rn(30.0, sd));
                k = k0 > 0 ? k0 : 0;
                const double nn = (double)n, kk = (double)k;
                double e = __dsub_rn(lgamma(__dadd_rn(nn, 1.0)), lgamma(__dadd_rn(kk, 1.0)));
                e = __dsub_rn(e, lgamma(__dadd_rn(__dsub_rn(nn, kk), 1.0)));
                e = __dadd_rn(e, __dmul_rn(kk, log(pp)));
                e = __dadd_rn(e, __dmul_rn(__dsub_rn(nn, kk), lg));
                pmf = exp_ref(e);
            }
            cdf = pmf;
            if (cdf <= uu && k < n) {
                walking = true;
                kd = (double)k;
                nd = (double)n;
                nk = (double)(n - k);
                k1 = (double)(k + 1);
                kr = k + 1 < (int64_t)kRecipN && odds >= kMarksteinMin ? (int)(k + 1) : kRecipN;
            } else {
                commit(flip ? n - k : k);
            }
        }
#ifdef WS_WALK_PROF
        __syncwarp();
        wp[9] += clock64() - wp_sd;
#endif
    };

#ifndef WS_FL_KWALK
#define WS_FL_KWALK 10  // CDF steps per iteration (sweeps: 7 at 72 registers before skip records, 10 at 80 after: 9 / 10 / 11 / 12 = 3.24 / 3.20 / 3.22 / 3.27 ms)
#endif
    constexpr int kWalk = WS_FL_KWALK;
#ifdef WS_WALK_PROF
    const long long wp_t0 = clock64();
#endif
#pragma unroll 1
    for (;;) {
#ifdef WS_WALK_PROF
        const long long wp_s = clock64();
        setup();
        wp[0] += clock64() - wp_s;
        wp[4] += 1;
#else
        setup();
#endif
        const unsigned alive = __ballot_sync(0xffffffffu, has);  // (lanes without a unit are exhausted)
        if (!alive) break;
        const int quorum = max(1, (__popc(alive) * ev.fl_quorum) >> 4);
#ifdef WS_WALK_PROF
        wp[5] += __popc(alive);
        wp[7] += __popc(__ballot_sync(0xffffffffu, walking));
        const long long wp_w = clock64();
#endif
#pragma unroll 1
        for (;;) {
#ifdef WS_WALK_PROF
            wp[2] += 1;
            wp[3] += __popc(__ballot_sync(0xffffffffu, walking));
#endif
            if (walking) {
                double f[kWalk];
                if (kr + kWalk <= kRecipN) {
#pragma unroll
                    for (int j = 0; j < kWalk; ++j)
                        f[j] = div_rn_y(__dmul_rn(odds, nk - (double)j), k1 + (double)j, __ldg(&ev.recip[kr + j]));
                } else {
#pragma unroll
                    for (int j = 0; j < kWalk; ++j) f[j] = __ddiv_rn(__dmul_rn(odds, nk - (double)j), k1 + (double)j);
                }
                if (nk >= (double)kWalk) {
                    // k + kWalk <= n: only the cdf test can stop these steps
                    double pm = pmf, c = cdf;
                    int adv = 0;
#pragma unroll
                    for (int j = 0; j < kWalk; ++j) {
                        pm = __dmul_rn(pm, f[j]);
                        c = __dadd_rn(c, pm);
                        adv += c <= uu ? 1 : 0;  // monotone: counts the steps before the stop
                    }
                    if (adv == kWalk && nk > (double)kWalk) {  // (k + kWalk == n ends the walk too)
                        pmf = pm;
                        cdf = c;
                        kd += (double)kWalk;
                        nk -= (double)kWalk;
                        k1 += (double)kWalk;
                        kr += kWalk;
                    } else {
                        walking = false;
                        const int64_t k = (int64_t)kd + min(adv + 1, kWalk);
                        kdone = flip ? n - k : k;
                    }
                } else {
                    double pm = pmf, c = cdf, kk = kd;
                    bool go = true;
#pragma unroll
                    for (int j = 0; j < kWalk; ++j) {
                        if (go) {
                            pm = __dmul_rn(pm, f[j]);
                            c = __dadd_rn(c, pm);
                            kk += 1.0;
                            go = c <= uu && kk < nd;
                        }
                    }
                    const double adv = kk - kd;
                    pmf = pm;
                    cdf = c;
                    kd = kk;
                    nk -= adv;
                    k1 += adv;
                    kr += (int)adv;
                    if (!go) {
                        walking = false;
                        const int64_t k = (int64_t)kd;
                        kdone = flip ? n - k : k;
                    }
                }
            }
            const unsigned wk = __ballot_sync(0xffffffffu, walking);
            if (wk == 0 || __popc(alive & ~wk) >= quorum) break;
        }
#ifdef WS_WALK_PROF
        wp[1] += clock64() - wp_w;
#endif
    }
#ifdef WS_WALK_PROF
    wp[6] = clock64() - wp_t0;
    if (lane == 0)
        for (int i = 0; i < 16; ++i) atomicAdd(&g_walkprof[i], wp[i]);
#endif
}

}  // namespace wsb

#ifdef WS_WALK_PROF
#include <cstdio>
// tools/walkprof.py (a -DWS_WALK_PROF build): where the walk's warps spend their cycles
extern "C" void wsb_walk_prof_dump()
{
    unsigned long long h[16];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, wsb::g_walkprof, sizeof(h));
    fprintf(stderr, "walkprof setup_cyc %llu walk_cyc %llu total_cyc %llu | walk_iters %llu walking_lanes/iter %.2f | setups %llu alive/setup %.2f walking_after_setup %.2f\n",
            h[0], h[1], h[6], h[2], h[2] ? (double)h[3] / h[2] : 0.0, h[4], h[4] ? (double)h[5] / h[4] : 0.0,
            h[4] ? (double)h[7] / h[4] : 0.0);
    fprintf(stderr, "walkprof take_passes %llu seed_cyc %llu seeding_lanes/setup %.2f commit_cyc %llu loop_cyc %llu loop_passes %llu cheap_lane_iters %llu\n",
            h[8], h[9], h[4] ? (double)h[10] / h[4] : 0.0, h[11], h[12], h[13], h[14]);
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(wsb::g_walkprof, z, sizeof(z));
}
#endif

extern "C" cudaError_t wsb_launch_sample(const wsb::EventDesc& ev, wsb::UnitRec* recs, uint32_t* pool, uint32_t pool_cap,
                                         uint32_t* pool_ctr, uint32_t* band_count, unsigned* err, cudaStream_t s,
                                         int pdl)
{
    if (ev.total_units == 0) return cudaSuccess;
    const uint32_t threads = 128;
    const uint32_t blocks = (ev.total_units + threads - 1) / threads;
    if (ev.fluctuate) {
        wsb::k_sample<true><<<blocks, threads, 0, s>>>(ev, recs, pool, pool_cap, pool_ctr, band_count, err);
    } else {
        constexpr size_t smem = sizeof(float) * (wsb::kSampleThreads / 32) * wsb::kStageWarp;
        const unsigned grid = (ev.total_units + wsb::kSampleThreads - 1) / wsb::kSampleThreads;
        bool imp = false;
        for (int i = 0; i < ev.n_planes; ++i) imp = imp || ev.p[i].impacts > 1;
        const auto kfn = imp ? wsb::k_sample_off<true> : wsb::k_sample_off<false>;
        if (!pdl) {
            kfn<<<grid, wsb::kSampleThreads, smem, s>>>(ev, recs, pool, pool_cap, pool_ctr, band_count, err);
            return cudaGetLastError();
        }
        // programmatic launch behind the previous call's k_direct (footprints
        // and pool allocation overlap its tail; griddepcontrol.wait guards the rest)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(wsb::kSampleThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kfn, ev, recs, pool, pool_cap, pool_ctr, band_count, err);
    }
    return cudaGetLastError();
}

// Zero n 16-byte words on the SMs (a large cudaMemsetAsync may run on a copy
// engine, where it queues behind the previous event's frame copies)
namespace wsb {
__global__ void k_zero16(uint4* __restrict__ p, size_t n)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(0u, 0u, 0u, 0u);
}
}  // namespace wsb

// Zero a count grid of `cells` cells at the width cnt_wide chose (after k_sample)
namespace wsb {
__global__ void k_zero_counts(uint4* __restrict__ p, size_t cells, const unsigned long long* __restrict__ qsum)
{
    const bool wide = !qsum || *qsum >= (1ull << 32);
    const size_t n = ((cells << (wide ? 3 : 2)) + 15) / 16;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(0u, 0u, 0u, 0u);
}
}  // namespace wsb

extern "C" cudaError_t wsb_launch_zero_counts(void* p, size_t cells, const unsigned long long* qsum, cudaStream_t s)
{
    if (cells == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t n = (cells * 8 + 15) / 16;
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)sms * 8);
    wsb::k_zero_counts<<<blocks, 256, 0, s>>>(static_cast<uint4*>(p), cells, qsum);
    return cudaGetLastError();
}

extern "C" cudaError_t wsb_launch_zero(void* p, size_t bytes, cudaStream_t s)
{
    if (bytes == 0) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(p) | bytes) & 15) return cudaMemsetAsync(p, 0, bytes, s);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t n = bytes / 16;
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)sms * 8);
    wsb::k_zero16<<<blocks, 256, 0, s>>>(static_cast<uint4*>(p), n);
    return cudaGetLastError();
}

extern "C" cudaError_t wsb_launch_scan(uint32_t* count, uint32_t* off, uint32_t* fill, uint32_t n, cudaStream_t s)
{
    wsb::k_scan_bands<<<1, 1024, 0, s>>>(count, off, fill, n);
    return cudaGetLastError();
}

extern "C" cudaError_t wsb_launch_fill(const wsb::EventDesc& ev, const wsb::UnitRec* recs, const uint32_t* off,
                                       uint32_t* fill, wsb::UnitRec* list, wsb::TEnt* tlist, const uint32_t* pool,
                                       unsigned* err, cudaStream_t s)
{
    if (ev.total_units == 0) return cudaSuccess;
    wsb::k_fill_bands<<<(ev.total_units + 255) / 256, 256, 0, s>>>(ev, recs, off, fill, list, tlist, pool, err);
    return cudaGetLastError();
}

// Scratch of the exact walk for n units: bucket keys, the two schedules,
// record offsets, the normal-branch list, counters and the bucket histograms.
extern "C" size_t wsb_fluct_scratch_bytes(uint32_t n)
{
    return sizeof(uint32_t) * (6 * (size_t)n + 4 + wsb::kFlBq + wsb::kFlBb);
}

// scratch: wsb_fluct_scratch_bytes(ev.total_units) bytes of device memory the
// caller keeps (a context buffer: no allocation per call)
extern "C" cudaError_t wsb_launch_fluctuate(const wsb::EventDesc& ev, const wsb::UnitRec* recs, const uint32_t* pool,
                                            const uint32_t* order, void* scratch, cudaStream_t s)
{
    if (ev.total_units == 0) return cudaSuccess;
    if (ev.approx) {
        wsb::k_fluctuate<<<(ev.total_units + 127) / 128, 128, 0, s>>>(ev, recs, pool, order);
        return cudaGetLastError();
    }
    // exact walk: the units in descending charge for the walk and by bin count
    // for the records (bucket sorts in the caller's scratch), the per-bin
    // records (k_fluct_prep), the walk (k_fluct_walk), then the units that
    // could take binomial's normal branch (k_fluctuate_exact)
    const uint32_t n = ev.total_units;
    uint32_t* buf = static_cast<uint32_t*>(scratch);
    uint32_t *bq = buf, *bb = buf + n, *v_out = buf + 2 * (size_t)n, *b_order = buf + 3 * (size_t)n;
    uint32_t *offs = buf + 4 * (size_t)n, *slow = buf + 5 * (size_t)n;
    uint32_t *n_slow = buf + 6 * (size_t)n, *cursor = n_slow + 1, *hist = n_slow + 4;
    const unsigned blocks = (n + 127) / 128;
    cudaError_t e = cudaSuccess;
    wsb::k_fluct_hist_zero<<<1, 1024, 0, s>>>(hist, n_slow);
    constexpr unsigned per_block = wsb::kFlSortThreads * wsb::kFlPer;
    wsb::k_fluct_keys<<<(n + per_block - 1) / per_block, wsb::kFlSortThreads, 0, s>>>(ev, recs, bq, bb, hist);
    wsb::k_fluct_hist_scan<<<1, 1024, 0, s>>>(hist);
    wsb::k_fluct_scatter<<<(n + per_block - 1) / per_block, wsb::kFlSortThreads, 0, s>>>(n, bq, bb, hist, v_out,
                                                                                          b_order);
    if (e == cudaSuccess) {
        // persistent walk: one resident wave of lanes pulling units from a cursor
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wsb::k_fluct_walk, 128, 0);
        const unsigned wblocks = std::min<unsigned>(blocks, (unsigned)(sms * std::max(per_sm, 1)));
        wsb::k_fluct_prep<<<blocks, 128, 0, s>>>(ev, recs, pool, b_order, offs, slow, n_slow, cursor, wblocks * 128u);
        wsb::k_fluct_walk<<<wblocks, 128, 0, s>>>(ev, recs, v_out, offs, cursor);
        wsb::k_fluctuate_exact<<<blocks, 128, 0, s>>>(ev, recs, pool, slow, n_slow);
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}
