/* TEST INFRASTRUCTURE — NOT PRODUCT CODE. See wsoracle.h for scope and pinning.
 *
 * Compile with -O2 -ffp-contract=off (oracle/Makefile): the expressions below
 * keep the reference's operation order so every double is bit-identical to
 * the reference built with the same flags.
 */
#define _GNU_SOURCE
#include "wsoracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return 1;
}

const char* wso_last_error(void) { return g_err; }

static const double kTwoPi = 6.283185307179586476925286766559;
static const double kInvSqrt2 = 0.70710678118654752440084436210485;

/* ---------------------------------------------------------------- rng ---- */

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.cpp:18-24 */
uint64_t wso_splitmix64_next(uint64_t* state)
{
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.cpp:26-35 */
void wso_seed_state(uint64_t seed, uint64_t s[4])
{
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) s[i] = wso_splitmix64_next(&sm);
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 0x9e3779b97f4a7c15ULL;
}

/* rng.cpp:64-76 */
void wso_substream(uint64_t seed, uint64_t stream_id, uint64_t s[4])
{
    uint64_t sm = seed;
    uint64_t tag = stream_id;
    (void)wso_splitmix64_next(&tag);
    sm ^= wso_splitmix64_next(&tag);
    for (int i = 0; i < 4; ++i) s[i] = wso_splitmix64_next(&sm);
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 0x9e3779b97f4a7c15ULL;
}

/* rng.cpp:37-49 (xoshiro256**) */
uint64_t wso_next_u64(uint64_t s[4])
{
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

/* rng.cpp:51-54 */
double wso_uniform01(uint64_t s[4]) { return (double)(wso_next_u64(s) >> 11) * 0x1.0p-53; }

/* Philox4x32-10 (Salmon et al. SC'11; Random123). Not in the reference: the
 * shared counter-based stream of the north star. KATs in
 * tests/test_oracle.py. */
void wso_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void wso_src_init(wso_src* src, int mode, uint64_t seed, uint64_t id)
{
    memset(src, 0, sizeof *src);
    src->mode = mode;
    src->seed = seed;
    src->id = id;
    if (mode == 0) wso_substream(seed, id, src->s); /* rasterize.cpp:191 */
}

/* StreamSource::uniform (rng.hpp:76) or the Philox counter layout:
 * draw i -> ctr (i>>1, id lo, id hi, 0), key (seed lo, seed hi),
 * u64 = word[2(i&1)] << 32 | word[2(i&1)+1], u = (u64 >> 11) * 2^-53. */
double wso_src_uniform(wso_src* src)
{
    if (src->mode == 0) return wso_uniform01(src->s);
    const uint64_t i = src->draw++;
    const uint32_t ctr[4] = {(uint32_t)(i >> 1), (uint32_t)src->id, (uint32_t)(src->id >> 32), 0u};
    const uint32_t key[2] = {(uint32_t)src->seed, (uint32_t)(src->seed >> 32)};
    uint32_t o[4];
    wso_philox4x32_10(ctr, key, o);
    const int h = (int)(i & 1u) * 2;
    const uint64_t u64 = ((uint64_t)o[h] << 32) | o[h + 1];
    return (double)(u64 >> 11) * 0x1.0p-53;
}

/* StreamSource::normal (rng.hpp:78-90) + box_muller (rng.cpp:56-62) */
double wso_src_normal(wso_src* src)
{
    if (src->have_spare) {
        src->have_spare = 0;
        return src->spare;
    }
    const double u1 = 1.0 - wso_src_uniform(src);
    const double u2 = wso_src_uniform(src);
    const double r = sqrt(-2.0 * log(u1));
    src->spare = r * sin(kTwoPi * u2);
    src->have_spare = 1;
    return r * cos(kTwoPi * u2);
}

/* rng.cpp:146-170 */
static int64_t invert_binomial_cdf(int64_t n, double p, double u)
{
    const double odds = p / (1.0 - p);
    int64_t k = 0;
    double pmf;
    const double log_pmf0 = (double)n * log1p(-p);
    if (log_pmf0 > -700.0) {
        pmf = exp(log_pmf0);
    } else {
        const double mean = (double)n * p;
        const double sd = sqrt(mean * (1.0 - p));
        const int64_t k0 = (int64_t)(mean - 30.0 * sd);
        k = k0 > 0 ? k0 : 0;
        const double nd = (double)n;
        const double kd = (double)k;
        pmf = exp(lgamma(nd + 1.0) - lgamma(kd + 1.0) - lgamma(nd - kd + 1.0) + kd * log(p) +
                  (nd - kd) * log1p(-p));
    }
    double cdf = pmf;
    while (cdf <= u && k < n) {
        pmf *= odds * (double)(n - k) / (double)(k + 1);
        ++k;
        cdf += pmf;
    }
    return k;
}

/* rng.cpp:174-193 */
int wso_binomial(int64_t n, double p, wso_src* src, int64_t* k)
{
    if (n < 0) return fail("binomial: n must be >= 0");
    if (p < 0.0 || p > 1.0) return fail("binomial: p must be in [0,1]");
    if (n == 0 || p == 0.0) { *k = 0; return 0; }
    if (p == 1.0) { *k = n; return 0; }
    const double mean = (double)n * p;
    const double var = mean * (1.0 - p);
    const double mn = p < 1.0 - p ? p : 1.0 - p;
    if ((double)n * mn > 1e6) {
        const double kk = round(mean + sqrt(var) * wso_src_normal(src));
        *k = kk < 0.0 ? 0 : (kk > (double)n ? n : (int64_t)kk);
        return 0;
    }
    const double u = wso_src_uniform(src);
    if (p > 0.5) *k = n - invert_binomial_cdf(n, 1.0 - p, u);
    else *k = invert_binomial_cdf(n, p, u);
    return 0;
}

/* ---------------------------------------------------------- rasterize ---- */

static int validate_grid(const wso_grid* g)
{
    if (g->n_wires < 1 || g->n_ticks < 1) return fail("GridSpec: active grid must be at least 1x1");
    if (!(g->pitch > 0.0)) return fail("GridSpec: pitch must be > 0");
    if (!(g->tick > 0.0)) return fail("GridSpec: tick must be > 0");
    return 0;
}

/* core.cpp:9-21 */
static long floor_index(double coord, double origin, double spacing) { return (long)floor((coord - origin) / spacing); }
static long half_extent(double n_sigma, double sigma, double spacing)
{
    if (sigma <= 0.0) return 0;
    return (long)ceil(n_sigma * sigma / spacing);
}

/* core.cpp:25-41 -> {center_wire, center_tick, wire_lo, wire_hi, tick_lo, tick_hi} */
int wso_map_depo(const wso_grid* g, const wso_depo* d, double n_sigma, long out6[6])
{
    if (validate_grid(g)) return 1;
    if (!(n_sigma > 0.0)) return fail("map_depo_to_grid: n_sigma must be > 0");
    const long cw = (long)g->pad_wires + floor_index(d->x, g->origin_x, g->pitch);
    const long ct = (long)g->pad_ticks + floor_index(d->t, g->origin_t, g->tick);
    const long hw = half_extent(n_sigma, d->sigma_x, g->pitch);
    const long ht = half_extent(n_sigma, d->sigma_t, g->tick);
    out6[0] = cw; out6[1] = ct;
    out6[2] = cw - hw; out6[3] = cw + hw;
    out6[4] = ct - ht; out6[5] = ct + ht;
    return 0;
}

/* rasterize.cpp:22-42 */
int wso_drift_depo(const wso_depo* d, const wso_drift* p, wso_depo* out)
{
    if (!(p->drift_speed > 0.0)) return fail("drift_depo: drift_speed must be > 0");
    if (d->x < p->response_plane_x)
        return fail("drift_depo: depo %lld at x=%f mm is behind the response plane at %f mm", (long long)d->id, d->x,
                    p->response_plane_x);
    const double dx = d->x - p->response_plane_x;
    const double drift_time = dx / p->drift_speed;
    *out = *d;
    out->t = d->t + drift_time;
    out->x = p->response_plane_x;
    const double v2 = p->drift_speed * p->drift_speed;
    out->sigma_t = sqrt(d->sigma_t * d->sigma_t + 2.0 * p->diffusion_long * drift_time / v2);
    out->sigma_x = sqrt(d->sigma_x * d->sigma_x + 2.0 * p->diffusion_tran * drift_time);
    return 0;
}

/* rasterize.cpp:44-64 */
void wso_gauss_bin_integrals(double center, double sigma, double lo_edge, double spacing, size_t n, double* vals)
{
    for (size_t i = 0; i < n; ++i) vals[i] = 0.0;
    if (n == 0) return;
    if (sigma <= 0.0) {
        long idx = (long)floor((center - lo_edge) / spacing);
        if (idx < 0) idx = 0;
        if (idx > (long)n - 1) idx = (long)n - 1;
        vals[idx] = 1.0;
        return;
    }
    const double inv = kInvSqrt2 / sigma;
    double prev = erf((lo_edge - center) * inv);
    for (size_t i = 0; i < n; ++i) {
        const double next = erf((lo_edge + (double)(i + 1) * spacing - center) * inv);
        vals[i] = 0.5 * (next - prev);
        prev = next;
    }
}

/* rasterize.cpp:66-120. meta = {wire_offset, tick_offset, n_w, n_t, clipped};
 * an empty patch has n_w = n_t = 0 and *captured = 0. */
int wso_sample_patch(const wso_grid* g, const wso_depo* d, double n_sigma, long meta[5], double* values,
                     size_t cap, double* captured)
{
    long fp[6];
    if (wso_map_depo(g, d, n_sigma, fp)) return 1;
    const long max_w = (long)(g->n_wires + 2 * g->pad_wires) - 1;
    const long max_t = (long)(g->n_ticks + 2 * g->pad_ticks) - 1;
    const long wire_lo = fp[2] > 0 ? fp[2] : 0;
    const long wire_hi = fp[3] < max_w ? fp[3] : max_w;
    const long tick_lo = fp[4] > 0 ? fp[4] : 0;
    const long tick_hi = fp[5] < max_t ? fp[5] : max_t;
    meta[0] = 0; meta[1] = 0; meta[2] = 0; meta[3] = 0;
    meta[4] = (wire_lo != fp[2] || wire_hi != fp[3] || tick_lo != fp[4] || tick_hi != fp[5]) ? 1 : 0;
    *captured = 0.0;
    if (wire_lo > wire_hi || tick_lo > tick_hi) return 0;
    const size_t n_w = (size_t)(wire_hi - wire_lo + 1);
    const size_t n_t = (size_t)(tick_hi - tick_lo + 1);
    if (n_w * n_t > cap) return fail("sample_patch: patch of %zu bins exceeds cap %zu", n_w * n_t, cap);
    const double wire_edge = g->origin_x + ((double)wire_lo - (double)g->pad_wires) * g->pitch;
    const double tick_edge = g->origin_t + ((double)tick_lo - (double)g->pad_ticks) * g->tick;
    double* wv = (double*)malloc(sizeof(double) * (n_w + n_t));
    if (!wv) return fail("sample_patch: out of memory");
    double* tv = wv + n_w;
    wso_gauss_bin_integrals(d->x, d->sigma_x, wire_edge, g->pitch, n_w, wv);
    wso_gauss_bin_integrals(d->t, d->sigma_t, tick_edge, g->tick, n_t, tv);
    double total = 0.0;
    for (size_t w = 0; w < n_w; ++w) {
        const double pw = wv[w];
        for (size_t t = 0; t < n_t; ++t) {
            const double v = pw * tv[t];
            values[w * n_t + t] = v;
            total += v;
        }
    }
    free(wv);
    if (total <= 0.0) return 0; /* numerically empty */
    const double norm = 1.0 / total;
    for (size_t i = 0; i < n_w * n_t; ++i) values[i] *= norm;
    meta[0] = wire_lo; meta[1] = tick_lo;
    meta[2] = (long)n_w; meta[3] = (long)n_t;
    *captured = total;
    return 0;
}

/* rasterize.cpp:124-170 (fluctuate_sequential with binomial / Gaussian-approx draws) */
int wso_fluctuate(const double* p, size_t n, int64_t q, wso_src* src, int approx, int64_t* out)
{
    if (q < 0) return fail("fluctuate: charge must be >= 0");
    for (size_t i = 0; i < n; ++i) out[i] = 0;
    if (n == 0) return 0;
    int64_t remaining = q;
    double p_rem = 1.0;
    const size_t last = n - 1;
    for (size_t i = 0; i < last; ++i) {
        if (remaining == 0) break;
        double pi = 1.0;
        if (p_rem > 0.0) {
            pi = p[i] / p_rem;
            pi = pi < 0.0 ? 0.0 : (pi > 1.0 ? 1.0 : pi);
        }
        int64_t k;
        if (approx) {
            if (pi <= 0.0) k = 0;
            else if (pi >= 1.0) k = remaining;
            else {
                const double mean = (double)remaining * pi;
                const double kk = round(mean + sqrt(mean * (1.0 - pi)) * wso_src_normal(src));
                k = kk < 0.0 ? 0 : (kk > (double)remaining ? remaining : (int64_t)kk);
            }
        } else if (wso_binomial(remaining, pi, src, &k)) {
            return 1;
        }
        out[i] = k;
        remaining -= k;
        p_rem -= p[i];
    }
    out[last] += remaining;
    return 0;
}

/* ---------------------------------------------- charge grids (scatter) ---- */

#define PATCH_CAP (1u << 20)

static size_t padded_w(const wso_grid* g) { return (size_t)(g->n_wires + 2 * g->pad_wires); }
static size_t padded_t(const wso_grid* g) { return (size_t)(g->n_ticks + 2 * g->pad_ticks); }

/* Fluctuation off: S += q * p over sample_patch (rasterize.cpp:66-120), drift
 * first when given (pipeline.cpp:358-362), empty patches add q to the clipped
 * charge (pipeline.cpp:339-340). S is accumulated (caller zeroes it). */
int wso_charge_fluct_off(const wso_grid* g, const wso_depo* d, size_t n, double n_sigma, const wso_drift* drift,
                         double* s, int64_t* clipped_charge)
{
    double* vals = (double*)malloc(sizeof(double) * PATCH_CAP);
    if (!vals) return fail("out of memory");
    const size_t cols = padded_t(g);
    int64_t clipped = 0;
    for (size_t i = 0; i < n; ++i) {
        wso_depo dd = d[i];
        if (drift && wso_drift_depo(&d[i], drift, &dd)) { free(vals); return 1; }
        long meta[5];
        double cap;
        if (wso_sample_patch(g, &dd, n_sigma, meta, vals, PATCH_CAP, &cap)) { free(vals); return 1; }
        if (meta[2] == 0) { clipped += dd.q; continue; }
        const double q = (double)dd.q;
        for (long w = 0; w < meta[2]; ++w)
            for (long t = 0; t < meta[3]; ++t)
                s[(size_t)(meta[0] + w) * cols + (size_t)(meta[1] + t)] += q * vals[w * meta[3] + t];
    }
    free(vals);
    if (clipped_charge) *clipped_charge = clipped;
    return 0;
}

/* Fluctuation on: rasterize_depo (rasterize.cpp:172-205) in substream mode
 * (rng_mode 0) or with the Philox source (rng_mode 1); exact binomial or the
 * Gaussian approximation; scatter_add (scatter.cpp:27-36). */
int wso_charge_fluct_on(const wso_grid* g, const wso_depo* d, size_t n, double n_sigma, const wso_drift* drift,
                        int rng_mode, int approx, uint64_t seed, int64_t* s, int64_t* clipped_charge)
{
    double* vals = (double*)malloc(sizeof(double) * PATCH_CAP);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * PATCH_CAP);
    if (!vals || !cnt) { free(vals); free(cnt); return fail("out of memory"); }
    const size_t cols = padded_t(g);
    int64_t clipped = 0;
    int rc = 0;
    for (size_t i = 0; i < n && !rc; ++i) {
        wso_depo dd = d[i];
        if (drift && wso_drift_depo(&d[i], drift, &dd)) { rc = 1; break; }
        long meta[5];
        double cap;
        if (wso_sample_patch(g, &dd, n_sigma, meta, vals, PATCH_CAP, &cap)) { rc = 1; break; }
        if (meta[2] == 0) { clipped += dd.q; continue; }
        if (dd.q < 0) { rc = fail("fluctuate: charge must be >= 0"); break; }
        wso_src src;
        wso_src_init(&src, rng_mode, seed, (uint64_t)dd.id);
        const size_t nb = (size_t)(meta[2] * meta[3]);
        if (wso_fluctuate(vals, nb, dd.q, &src, approx, cnt)) { rc = 1; break; }
        for (long w = 0; w < meta[2]; ++w)
            for (long t = 0; t < meta[3]; ++t)
                s[(size_t)(meta[0] + w) * cols + (size_t)(meta[1] + t)] += cnt[w * meta[3] + t];
    }
    free(vals);
    free(cnt);
    if (!rc && clipped_charge) *clipped_charge = clipped;
    return rc;
}

/* ------------------------------------------------------------ response ---- */

static double gauss_pdf(double t, double sigma)
{
    const double z = t / sigma;
    return exp(-0.5 * z * z) / (sigma * sqrt(kTwoPi)); /* spectral.cpp:24-28 */
}

/* Combined time-domain kernel over lags [lo_lag, lo_lag + n_lags):
 * field_samples (spectral.cpp:34-64) convolved with shaper_samples
 * (spectral.cpp:68-83), scaled by gain / sum(shaper) (spectral.cpp:98-107);
 * validation and supports as build_response (spectral.cpp:87-121). */
int wso_response_td(const wso_grid* g, const wso_response* r, double* combined, size_t cap, long* lo_lag,
                    size_t* n_lags, long* support_ticks, long* support_wires)
{
    if (validate_grid(g)) return 1;
    if (r->shaper_order < 1) return fail("build_response: shaper_order must be >= 1");
    if (r->n_wire_weights == 0 || r->n_wire_weights % 2 == 0)
        return fail("build_response: wire_weights must have odd length");
    const double tick = g->tick;

    /* field */
    long half = 0;
    size_t nf = 1;
    double* f = NULL;
    if (r->field_sigma_t <= 0.0) {
        f = (double*)malloc(sizeof(double));
        f[0] = 1.0;
    } else {
        const double sigma = r->field_sigma_t;
        half = (long)ceil(8.0 * sigma / tick);
        nf = (size_t)(2 * half + 1);
        f = (double*)malloc(sizeof(double) * nf);
        if (r->plane_kind == 1) {
            const double lo = (-(double)half - 0.5) * tick;
            wso_gauss_bin_integrals(0.0, sigma, lo, tick, nf, f);
            double sum = 0.0;
            for (size_t i = 0; i < nf; ++i) sum += f[i];
            for (size_t i = 0; i < nf; ++i) f[i] /= sum;
        } else {
            double pos = 0.0;
            for (size_t i = 0; i < nf; ++i) {
                const double lo = ((double)i - (double)half - 0.5) * tick;
                const double hi = lo + tick;
                f[i] = gauss_pdf(hi, sigma) - gauss_pdf(lo, sigma);
                if (f[i] > 0.0) pos += f[i];
            }
            for (size_t i = 0; i < nf; ++i) f[i] /= pos;
        }
    }

    /* shaper */
    size_t ns = 0, scap = 1024;
    double* s = (double*)malloc(sizeof(double) * scap);
    if (r->shaper_peaking <= 0.0) {
        s[0] = 1.0;
        ns = 1;
    } else {
        const double tau = r->shaper_peaking;
        const int order = r->shaper_order;
        for (long k = 0;; ++k) {
            const double t = (double)k * tick;
            const double z = t / tau;
            const double v = pow(z, (double)order) * exp(-(double)order * (z - 1.0));
            if (ns == scap) { scap *= 2; s = (double*)realloc(s, sizeof(double) * scap); }
            s[ns++] = v;
            if (t > tau && v < 1e-14) break;
            if (k > 2000000) { free(f); free(s); return fail("build_response: shaper tail does not decay"); }
        }
    }
    double shaper_sum = 0.0;
    for (size_t j = 0; j < ns; ++j) shaper_sum += s[j];
    const double amplitude = r->gain / shaper_sum;

    const size_t nl = nf + ns - 1;
    *lo_lag = -half;
    *n_lags = nl;
    *support_ticks = (-*lo_lag) > (*lo_lag + (long)nl - 1) ? -*lo_lag : *lo_lag + (long)nl - 1;
    *support_wires = (long)(r->n_wire_weights / 2);
    int rc = 0;
    if (nl > padded_t(g))
        rc = fail("build_response: kernel time support %zu exceeds the padded tick count %zu", nl, padded_t(g));
    else if (r->n_wire_weights > padded_w(g))
        rc = fail("build_response: wire_weights exceed the padded wire count");
    else if (combined) {
        if (nl > cap) rc = fail("build_response: cap %zu < %zu lags", cap, nl);
        else {
            for (size_t i = 0; i < nl; ++i) combined[i] = 0.0;
            for (size_t i = 0; i < nf; ++i)
                for (size_t j = 0; j < ns; ++j) combined[i + j] += f[i] * s[j] * amplitude;
        }
    }
    free(f);
    free(s);
    return rc;
}

/* convolve (spectral.cpp:141-175) restated as the direct 2D circular sum it
 * computes: kernel_td[dw mod W][lag mod T] = ww[dw] * combined[lag]
 * (spectral.cpp:123-135), M = kernel_td (*) S circularly. fp64; equals the
 * reference FFT path to ~1e-13 relative (test_oracle.py). */
int wso_convolve_direct(const wso_grid* g, const wso_response* r, const double* s, double* m)
{
    const size_t W = padded_w(g), T = padded_t(g);
    long lo_lag, st, sw;
    size_t nl;
    if (wso_response_td(g, r, NULL, 0, &lo_lag, &nl, &st, &sw)) return 1;
    if (st > (long)g->pad_ticks || sw > (long)g->pad_wires)
        return fail("convolve: kernel support (%ld wires, %ld ticks) exceeds the padding", sw, st);
    double* k = (double*)malloc(sizeof(double) * nl);
    if (wso_response_td(g, r, k, nl, &lo_lag, &nl, &st, &sw)) { free(k); return 1; }
    unsigned char* nz = (unsigned char*)calloc(W, 1);
    for (size_t w = 0; w < W; ++w)
        for (size_t t = 0; t < T; ++t)
            if (s[w * T + t] != 0.0) { nz[w] = 1; break; }
    const long h = (long)(r->n_wire_weights / 2);
    for (size_t w = 0; w < W; ++w) {
        double* out = m + w * T;
        for (size_t t = 0; t < T; ++t) out[t] = 0.0;
        for (long dw = -h; dw <= h; ++dw) {
            const double ww = r->wire_weights[dw + h];
            if (ww == 0.0) continue;
            const size_t src_row = (size_t)((((long)w - dw) % (long)W + (long)W) % (long)W);
            if (!nz[src_row]) continue;
            const double* src = s + src_row * T;
            for (size_t i = 0; i < nl; ++i) {
                const double kv = ww * k[i];
                const long lag = lo_lag + (long)i;
                const size_t sh = (size_t)(((lag % (long)T) + (long)T) % (long)T);
                /* out[t] += kv * src[(t - sh) mod T] */
                for (size_t t = sh; t < T; ++t) out[t] += kv * src[t - sh];
                for (size_t t = 0; t < sh; ++t) out[t] += kv * src[t + T - sh];
            }
        }
    }
    free(nz);
    free(k);
    return 0;
}

/* --------------------------------------------------- noise / digitize ---- */

/* add_noise white mode (spectral.cpp:188-196): per-wire substream of
 * (seed ^ kWhiteNoiseSalt, wire), row[t] += sigma * normal(). */
int wso_add_white_noise_rng(const wso_grid* g, double sigma, uint64_t seed, int rng_mode, double* m);

int wso_add_white_noise(const wso_grid* g, double sigma, uint64_t seed, double* m)
{
    return wso_add_white_noise_rng(g, sigma, seed, 0, m);
}

/* add_noise white mode with the per-wire stream of rng_mode: 0 the
 * reference's substream(seed ^ salt, w) (spectral.cpp:188-195), 1 the shared
 * Philox stream keyed by (seed ^ salt, w) (no reference equivalent: the GPU's
 * parallel mode, restated here as its checker) */
int wso_add_white_noise_rng(const wso_grid* g, double sigma, uint64_t seed, int rng_mode, double* m)
{
    if (sigma < 0.0) return fail("add_noise: sigma must be >= 0");
    if (sigma == 0.0) return 0;
    const size_t W = padded_w(g), T = padded_t(g);
    for (size_t w = 0; w < W; ++w) {
        wso_src src;
        wso_src_init(&src, rng_mode, seed ^ 0x77686974656e6f69ULL, (uint64_t)w);
        double* row = m + w * T;
        for (size_t t = 0; t < T; ++t) row[t] += sigma * wso_src_normal(&src);
    }
    return 0;
}

/* digitize (spectral.cpp:228-238) */
int wso_digitize(const double* m, size_t n, double scale, double offset, int bits, int32_t* adc)
{
    if (bits < 1 || bits > 16) return fail("digitize: bits must be in [1,16]");
    const double max_code = (double)((1 << bits) - 1);
    for (size_t i = 0; i < n; ++i) {
        const double v = round(m[i] * scale + offset);
        adc[i] = (int32_t)(v < 0.0 ? 0.0 : (v > max_code ? max_code : v));
    }
    return 0;
}

uint64_t wso_fnv1a64(const void* data, size_t nbytes)
{
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (size_t i = 0; i < nbytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* ------------------------------------------------------------------------
 * Signal processing (sigproc.cpp:12-118): filter -> inverse DFT along rows ->
 * block cut -> per-row medians.
 *
 * The DFT is a plain recursive mixed-radix decimation in time (smallest prime
 * factor first, O(n * sum of prime factors)); it is not the reference's
 * FftPlan but computes the same unscaled forward transform
 * X[k] = sum_j x[j] exp(-2 pi i jk / n) (fft.cpp:50), and the inverse by the
 * reference's conjugation identity with the 1/n factor applied as a multiply
 * (fft.cpp:96-100).
 */

/* out = DFT_n of x[0], x[stride], ...; scratch holds n complex values. The
 * children ping-pong between out and scratch. tw[j] = exp(-2 pi i j / N) of
 * the root length N (a multiple of n). */
static void dft_forward_rec(const double* x, size_t stride, size_t n, double* out, double* scratch,
                            const double* tw, size_t N)
{
    if (n == 1) {
        out[0] = x[0];
        out[1] = x[1];
        return;
    }
    size_t p = 2;
    while (p * p <= n && n % p) ++p;
    if (n % p) p = n;
    const size_t m = n / p, step = N / n;
    for (size_t q = 0; q < p; ++q) dft_forward_rec(x + 2 * q * stride, stride * p, m, scratch + 2 * q * m, out, tw, N);
    for (size_t k = 0; k < n; ++k) {
        double re = 0.0, im = 0.0;
        const size_t kk = k % m;
        for (size_t q = 0; q < p; ++q) {
            const size_t j = ((q * k) % n) * step;
            const double c = tw[2 * j], s = tw[2 * j + 1];
            const double a = scratch[2 * (q * m + kk)], b = scratch[2 * (q * m + kk) + 1];
            re += a * c - b * s;
            im += a * s + b * c;
        }
        out[2 * k] = re;
        out[2 * k + 1] = im;
    }
}

/* forward unscaled DFT of n complex (interleaved) values, out-of-place;
 * tw from dft_twiddles(n) */
static int dft_forward(const double* x, size_t n, double* out, const double* tw)
{
    double* work = (double*)malloc(sizeof(double) * 2 * n);
    if (!work) return fail("sigproc: out of memory");
    dft_forward_rec(x, 1, n, out, work, tw, n);
    free(work);
    return 0;
}

static double* dft_twiddles(size_t n)
{
    double* tw = (double*)malloc(sizeof(double) * 2 * n);
    if (!tw) return NULL;
    for (size_t j = 0; j < n; ++j) {
        const double ang = -2.0 * M_PI * (double)j / (double)n; /* fft.cpp:50 */
        tw[2 * j] = cos(ang);
        tw[2 * j + 1] = sin(ang);
    }
    return tw;
}

static int cmp_double(const void* a, const void* b)
{
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* row_median_by_sort (sigproc.cpp:95-102): must equal row_median exactly */
double wso_row_median(const double* v, size_t n)
{
    double* w = (double*)malloc(sizeof(double) * (n ? n : 1));
    memcpy(w, v, sizeof(double) * n);
    qsort(w, n, sizeof(double), cmp_double);
    const double r = (n % 2) ? w[n / 2] : (w[n / 2 - 1] + w[n / 2]) / 2.0;
    free(w);
    return r;
}

int wso_sigproc_chain(const double* data, size_t rows, size_t cols, size_t pad_rows, size_t out_rows,
                      const double* filter, double* block, double* medians, double* max_rel_imag)
{
    /* SignalBatch::validate (sigproc.hpp:24-28) */
    if (cols < 1) return fail("SignalBatch: need at least one column");
    if (pad_rows + out_rows > rows) return fail("SignalBatch: pad_rows + out_rows exceeds the row count");
    double* line = (double*)malloc(sizeof(double) * 2 * cols);
    double* spec = (double*)malloc(sizeof(double) * 2 * cols);
    double* tw = dft_twiddles(cols);
    if (!line || !spec || !tw) {
        free(line);
        free(spec);
        free(tw);
        return fail("sigproc: out of memory");
    }
    const double inv = 1.0 / (double)cols;
    double peak = 0.0, residue = 0.0;
    int rc = 0;
    for (size_t r = 0; r < rows && !rc; ++r) {
        const double* src = data + 2 * r * cols;
        for (size_t c = 0; c < cols; ++c) {
            /* apply_filter (sigproc.cpp:12-24), then conj for the inverse (fft.cpp:97) */
            const double a = src[2 * c], b = src[2 * c + 1], fc = filter[2 * c], fd = filter[2 * c + 1];
            line[2 * c] = a * fc - b * fd;
            line[2 * c + 1] = -(a * fd + b * fc);
        }
        rc = dft_forward(line, cols, spec, tw);
        if (rc) break;
        const int in_block = r >= pad_rows && r < pad_rows + out_rows;
        for (size_t c = 0; c < cols; ++c) {
            const double re = spec[2 * c] * inv, im = -spec[2 * c + 1] * inv;
            if (fabs(re) > peak) peak = fabs(re);
            if (fabs(im) > residue) residue = fabs(im);
            if (in_block) block[(r - pad_rows) * cols + c] = re;
        }
    }
    free(line);
    free(spec);
    free(tw);
    if (rc) return rc;
    if (medians)
        for (size_t r = 0; r < out_rows; ++r) medians[r] = wso_row_median(block + r * cols, cols);
    if (max_rel_imag) *max_rel_imag = peak > 0.0 ? residue / peak : residue;
    return 0;
}
