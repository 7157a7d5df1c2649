// Signal processing chain of the paper's Listing 1 (sigproc.cpp:104-118):
// per-row filter multiply -> inverse DFT along the row (real part kept) ->
// block cut [pad_rows, pad_rows + out_rows) -> per-row median.
//
// One CTA per signal row, the whole row resident in shared memory as
// complex fp64 (16 B x n; 96 KB at the paper's n = 6000, two CTAs per SM):
//   load     row x filter (coalesced 16-B loads, streaming), natural order
//   FFT      in-place mixed-radix decimation in frequency (radices 8/4/2 first,
//            then odd primes <= 13; the filter is applied in the first pass),
//            exp(+2 pi i/L) twiddles from per-pass tables (coalesced L1
//            loads); no scratch buffer
//   store    the DIF output is in digit-reversed order: a gather through the
//            plan's permutation writes the block row coalesced (x 1/n, the
//            reference's conjugation identity, fft.cpp:96-100) and leaves the
//            real part in place for the median; max |re| / max |im| feed the
//            imaginary-residue report (sigproc.cpp:33-69)
//   median   radix select on the order-preserving 64-bit keys of the row's
//            values: a 2048-bin histogram over the row's [min, max] locates
//            the central rank(s); their bins' elements are ranked by counting
//            (exact radix select on the 64-bit keys as the fallback); even
//            lengths average the two central order statistics
//            (sigproc.cpp:80-93)
// The median does not need the values in natural order, which is what lets
// the whole chain run in one buffer.
#include "ws_common.cuh"

#include <atomic>

namespace wsb {

constexpr int kSpThreads = 256;
constexpr int kSpBinsLog = 11;
constexpr int kSpBins = 1 << kSpBinsLog;

// cos / sin (2 pi m / R) for the odd radices, m < R: offsets 3:0 5:3 7:8 11:15 13:26
__constant__ double2 c_sproot[39];

template <int R>
__device__ __forceinline__ constexpr int sp_root_off()
{
    return R == 3 ? 0 : R == 5 ? 3 : R == 7 ? 8 : R == 11 ? 15 : 26;
}

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 c_muli(double2 a) { return make_double2(-a.y, a.x); }  // a * (+i)

// y_q = sum_r x_r exp(+2 pi i q r / R), in place
template <int R>
__device__ __forceinline__ void sp_dft(double2* x)
{
    if constexpr (R == 2) {
        const double2 t = x[0];
        x[0] = c_add(t, x[1]);
        x[1] = c_sub(t, x[1]);
    } else if constexpr (R == 4) {
        const double2 t0 = c_add(x[0], x[2]), t1 = c_sub(x[0], x[2]);
        const double2 t2 = c_add(x[1], x[3]), t3 = c_muli(c_sub(x[1], x[3]));
        x[0] = c_add(t0, t2);
        x[2] = c_sub(t0, t2);
        x[1] = c_add(t1, t3);
        x[3] = c_sub(t1, t3);
    } else if constexpr (R == 8) {
        double2 e[4] = {x[0], x[2], x[4], x[6]}, o[4] = {x[1], x[3], x[5], x[7]};
        sp_dft<4>(e);
        sp_dft<4>(o);
        constexpr double h = 0.70710678118654752440084436210485;
        o[1] = make_double2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y));
        o[2] = c_muli(o[2]);
        o[3] = make_double2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            x[q] = c_add(e[q], o[q]);
            x[q + 4] = c_sub(e[q], o[q]);
        }
    } else if constexpr (R == 16) {
        // 16 = 4 x 4: X[k1 + 4 k2] = sum_n2 W16^(n2 k1) W4^(n2 k2) sum_n1 x[4 n1 + n2] W4^(n1 k1)
        double2 a[4][4];
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {
            double2 t[4] = {x[n2], x[4 + n2], x[8 + n2], x[12 + n2]};
            sp_dft<4>(t);
#pragma unroll
            for (int k1 = 0; k1 < 4; ++k1) a[n2][k1] = t[k1];
        }
        constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
        // twiddles W16^m = exp(+2 pi i m / 16), m = n2 k1
        const double2 w[10] = {{1.0, 0.0}, {c1, s1}, {h, h}, {s1, c1}, {0.0, 1.0},
                               {-s1, c1}, {-h, h}, {-c1, s1}, {-1.0, 0.0}, {-c1, -s1}};
#pragma unroll
        for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
            for (int k1 = 1; k1 < 4; ++k1) a[n2][k1] = c_mul(a[n2][k1], w[n2 * k1]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            double2 t[4] = {a[0][k1], a[1][k1], a[2][k1], a[3][k1]};
            sp_dft<4>(t);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = t[k2];
        }
    } else {
        constexpr int H = (R - 1) / 2;
        double2 s[H + 1], d[H + 1];
        double2 y0 = x[0];
#pragma unroll
        for (int r = 1; r <= H; ++r) {
            s[r] = c_add(x[r], x[R - r]);
            d[r] = c_sub(x[r], x[R - r]);
            y0 = c_add(y0, s[r]);
        }
        const double2 x0 = x[0];
#pragma unroll
        for (int q = 1; q <= H; ++q) {
            double2 a = x0, b = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 1; r <= H; ++r) {
                const double2 w = c_sproot[sp_root_off<R>() + (q * r) % R];
                a.x = fma(s[r].x, w.x, a.x);
                a.y = fma(s[r].y, w.x, a.y);
                b.x = fma(d[r].x, w.y, b.x);
                b.y = fma(d[r].y, w.y, b.y);
            }
            x[q] = make_double2(a.x - b.y, a.y + b.x);
            x[R - q] = make_double2(a.x + b.y, a.y - b.x);
        }
        x[0] = y0;
    }
}

__device__ __forceinline__ double2 sp_filter_mul(double2 v, double2 f)
{
    // std::complex operator*= (apply_filter, sigproc.cpp:20), no contraction
    return make_double2(__dsub_rn(__dmul_rn(v.x, f.x), __dmul_rn(v.y, f.y)),
                        __dadd_rn(__dmul_rn(v.x, f.y), __dmul_rn(v.y, f.x)));
}

// One decimation-in-frequency pass over sub-transforms of length L:
// butterflies of radix R at stride S = L / R, then the exp(+2 pi i q j / L)
// twiddles (w^q by recurrence from the pass's table tw[j] = exp(+2 pi i j / L),
// coalesced through L1), in place. The
// first pass (L = n) applies the filter to its inputs.
// U butterflies of one pass at once (independent chains for the scheduler)
template <int R, bool kFilter, int U>
__device__ __forceinline__ void sp_bfly(double2* buf, const double2* tw, const double2* __restrict__ filter, int L,
                                        int S, uint32_t magic, int b0)
{
    double2 x[U][R];
    double2* p[U];
    int j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int b = b0 + u * kSpThreads;
        const int blk = S == 1 ? b : (int)__umulhi((uint32_t)b, magic);
        j[u] = b - blk * S;
        p[u] = buf + blk * L + j[u];
#pragma unroll
        for (int r = 0; r < R; ++r) x[u][r] = p[u][r * S];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if constexpr (kFilter) {
#pragma unroll
            for (int r = 0; r < R; ++r) x[u][r] = sp_filter_mul(x[u][r], __ldg(filter + j[u] + r * S));
        }
        sp_dft<R>(x[u]);
        // exp(+2 pi i q j / L) by recurrence from tw[j] (tw[0] = 1: exact)
        const double2 w1 = __ldg(tw + j[u]);
        double2 w = w1;
        x[u][1] = c_mul(x[u][1], w1);
#pragma unroll
        for (int q = 2; q < R; ++q) {
            w = c_mul(w, w1);
            x[u][q] = c_mul(x[u][q], w);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) p[u][r * S] = x[u][r];
}

// One decimation-in-frequency pass over sub-transforms of length L:
// butterflies of radix R at stride S = L / R, then the exp(+2 pi i q j / L)
// twiddles (w^q by recurrence from the pass's table tw[j] = exp(+2 pi i j / L),
// coalesced through L1), in place. The first pass (L = n) applies the filter
// to its inputs. Butterflies touch disjoint elements, so two per thread are
// in flight at once for radices <= 5.
template <int R, bool kFilter>
__device__ __forceinline__ void sp_pass(double2* buf, const double2* tw, const double2* __restrict__ filter, int n,
                                        int L)
{
    const int S = L / R, nb = n / R;
    const uint32_t magic = 0xffffffffu / (uint32_t)S + 1u;  // b / S for b, S < 2^15
    int b = threadIdx.x;
    if constexpr (R <= 5) {
        for (; b + kSpThreads < nb; b += 2 * kSpThreads) sp_bfly<R, kFilter, 2>(buf, tw, filter, L, S, magic, b);
    }
    for (; b < nb; b += kSpThreads) sp_bfly<R, kFilter, 1>(buf, tw, filter, L, S, magic, b);
}

// the wide odd radices out of line: their register demand stays out of the hot passes
template <int R>
__device__ __noinline__ void sp_pass_wide(double2* buf, const double2* tw, int n, int L)
{
    sp_pass<R, false>(buf, tw, nullptr, n, L);
}

template <bool kFilter>
__device__ __forceinline__ void sp_pass_any(int R, double2* buf, const double2* tw, const double2* filter, int n, int L)
{
    switch (R) {
        case 2: sp_pass<2, kFilter>(buf, tw, filter, n, L); break;
        case 3: sp_pass<3, kFilter>(buf, tw, filter, n, L); break;
        case 4: sp_pass<4, kFilter>(buf, tw, filter, n, L); break;
        case 5: sp_pass<5, kFilter>(buf, tw, filter, n, L); break;
        case 7: sp_pass<7, kFilter>(buf, tw, filter, n, L); break;
        case 8: sp_pass<8, kFilter>(buf, tw, filter, n, L); break;
        case 16: sp_pass<16, kFilter>(buf, tw, filter, n, L); break;
        case 11: sp_pass_wide<11>(buf, tw, n, L); break;  // filtered beforehand
        default: sp_pass_wide<13>(buf, tw, n, L); break;
    }
}

__device__ __forceinline__ unsigned long long sp_key(double v)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double sp_key_value(unsigned long long k)
{
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

constexpr int kSpCand = 512;  // candidates finished by rank counting

struct SpSelect {
    uint32_t hist[kSpBins];
    uint32_t warp_sum[kSpThreads / 32];
    uint32_t bin, cum, cnt, cnt_less;
    unsigned long long key, max_less;
    unsigned long long red[2 * (kSpThreads / 32)];
    double wmin[kSpThreads / 32], wmax[kSpThreads / 32];
    uint32_t bin_lo, cum_lo, bin_hi, cum_hi, n_cand;
    unsigned long long rank_key[2];
    unsigned long long cand[kSpCand];
    unsigned long long bar;  // mbarrier of the row's bulk copy
};

// key of the rank-k (0-based) element of buf[0..n).x
__device__ unsigned long long sp_select(const double* v, int st, int n, uint32_t k, SpSelect& s)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long prefix = 0, hmask = 0;
    int shift = 64;
    while (shift > 0) {
        const int w = shift < kSpBinsLog ? shift : kSpBinsLog;
        shift -= w;
        const uint32_t mask = (1u << w) - 1;
        for (int i = tid; i < kSpBins; i += kSpThreads) s.hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += kSpThreads) {
            const unsigned long long key = sp_key(v[i * st]);
            if ((key & hmask) == prefix) atomicAdd(&s.hist[(uint32_t)(key >> shift) & mask], 1u);
        }
        __syncthreads();
        constexpr int kPer = kSpBins / kSpThreads;
        uint32_t loc[kPer], sum = 0;
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            loc[e] = s.hist[tid * kPer + e];
            sum += loc[e];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s.warp_sum[warp] = incl;
        __syncthreads();
        uint32_t base = incl - sum;
        for (int v = 0; v < warp; ++v) base += s.warp_sum[v];
        if (k >= base && k < base + sum) {
#pragma unroll
            for (int e = 0; e < kPer; ++e) {
                if (k < base + loc[e]) {
                    s.bin = tid * kPer + e;
                    s.cum = base;
                    s.cnt = loc[e];
                    break;
                }
                base += loc[e];
            }
        }
        __syncthreads();
        const uint32_t bin = s.bin, cnt = s.cnt;
        k -= s.cum;
        prefix |= (unsigned long long)bin << shift;
        hmask |= (unsigned long long)mask << shift;
        if (cnt == 1 && shift > 0) {  // the rank's bin holds one element: find it
            for (int i = tid; i < n; i += kSpThreads) {
                const unsigned long long key = sp_key(v[i * st]);
                if ((key & hmask) == prefix) s.key = key;
            }
            __syncthreads();
            const unsigned long long key = s.key;
            __syncthreads();
            return key;
        }
    }
    return prefix;
}

// row_median (sigproc.cpp:80-93) of buf[0..n).x
__device__ __noinline__ double sp_median(const double* v, int st, int n, SpSelect& s)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long upper = sp_select(v, st, n, (uint32_t)(n / 2), s);
    if (n & 1) return sp_key_value(upper);
    // the rank n/2 - 1 element: upper again unless exactly n/2 elements are below it
    uint32_t cnt = 0;
    unsigned long long mx = 0;
    for (int i = tid; i < n; i += kSpThreads) {
        const unsigned long long key = sp_key(v[i * st]);
        if (key < upper) {
            ++cnt;
            mx = key > mx ? key : mx;
        }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = v > mx ? v : mx;
    }
    if (lane == 0) {
        s.red[warp] = cnt;
        s.red[kSpThreads / 32 + warp] = mx;
    }
    __syncthreads();
    uint32_t below = 0;
    unsigned long long max_below = 0;
    for (int v = 0; v < kSpThreads / 32; ++v) {
        below += (uint32_t)s.red[v];
        max_below = s.red[kSpThreads / 32 + v] > max_below ? s.red[kSpThreads / 32 + v] : max_below;
    }
    __syncthreads();
    const unsigned long long lower = below == (uint32_t)(n / 2) ? max_below : upper;
    return (sp_key_value(lower) + sp_key_value(upper)) / 2.0;
}

// row_median via a value-range histogram: bins of (v - lo) * 2048 / (hi - lo)
// are monotone in v, so the rank(s) n/2 (and n/2 - 1) fall in known bins; the
// elements of those bins (usually a handful) are compacted and ranked by
// counting. More than kSpCand candidates (heavy ties, extreme ranges) take the
// exact radix select instead. lo / hi: the row's min / max, known to all threads.
__device__ __noinline__ double sp_median_fast(const double* v, int st, int n, double lo, double hi, SpSelect& s)
{
    if (!(hi > lo)) return lo;  // constant row (or no usable range)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double scale = (double)kSpBins / (hi - lo);
    if (!(scale > 0.0) || isinf(scale)) return sp_median(v, st, n, s);
    // round((v - lo) * scale) through the 2^52 magic constant: one FFMA on the
    // fp64 pipe instead of an F2I conversion; rounding is monotone, which is
    // all the binning needs
    auto bin_of = [&](double v) {
        const uint32_t b = (uint32_t)__double2loint(fma(v - lo, scale, 0x1p52));
        return (int)(b < (uint32_t)kSpBins - 1 ? b : (uint32_t)kSpBins - 1);
    };
    for (int i = tid; i < kSpBins; i += kSpThreads) s.hist[i] = 0;
    if (tid == 0) s.n_cand = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kSpThreads) atomicAdd(&s.hist[bin_of(v[i * st])], 1u);
    __syncthreads();
    constexpr int kPer = kSpBins / kSpThreads;
    uint32_t loc[kPer], sum = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        loc[e] = s.hist[tid * kPer + e];
        sum += loc[e];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s.warp_sum[warp] = incl;
    __syncthreads();
    uint32_t base = incl - sum;
    for (int v = 0; v < warp; ++v) base += s.warp_sum[v];
    const uint32_t k_hi = (uint32_t)(n / 2), k_lo = (n & 1) ? k_hi : k_hi - 1;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        if (k_lo >= base && k_lo < base + loc[e]) {
            s.bin_lo = tid * kPer + e;
            s.cum_lo = base;
        }
        if (k_hi >= base && k_hi < base + loc[e]) {
            s.bin_hi = tid * kPer + e;
            s.cum_hi = base + loc[e];  // through bin_hi
        }
        base += loc[e];
    }
    __syncthreads();
    const int b_lo = (int)s.bin_lo, b_hi = (int)s.bin_hi;
    const uint32_t c0 = s.cum_lo, n_c = s.cum_hi - c0;
    if (n_c > (uint32_t)kSpCand) return sp_median(v, st, n, s);
    for (int i = tid; i < n; i += kSpThreads) {
        const double x = v[i * st];
        const int b = bin_of(x);
        if (b >= b_lo && b <= b_hi) s.cand[atomicAdd(&s.n_cand, 1u)] = sp_key(x);
    }
    __syncthreads();
    for (int t = tid; t < (int)n_c; t += kSpThreads) {
        const unsigned long long key = s.cand[t];
        uint32_t less = 0, eq = 0;
        for (uint32_t j = 0; j < n_c; ++j) {
            const unsigned long long o = s.cand[j];
            less += o < key;
            eq += o == key;
        }
        const uint32_t r_lo = k_lo - c0, r_hi = k_hi - c0;
        if (r_lo >= less && r_lo < less + eq) s.rank_key[0] = key;
        if (r_hi >= less && r_hi < less + eq) s.rank_key[1] = key;
    }
    __syncthreads();
    const double a = sp_key_value(s.rank_key[0]), b = sp_key_value(s.rank_key[1]);
    __syncthreads();
    return (n & 1) ? b : (a + b) / 2.0;
}

// CTA-wide min / max, result in every thread
__device__ __forceinline__ void sp_minmax(double& lo, double& hi, SpSelect& s)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
        s.wmin[warp] = lo;
        s.wmax[warp] = hi;
    }
    __syncthreads();
#pragma unroll
    for (int v = 0; v < kSpThreads / 32; ++v) {
        lo = fmin(lo, s.wmin[v]);
        hi = fmax(hi, s.wmax[v]);
    }
}

// Rows whose length has a prime factor > 13 (the reference takes them through
// Bluestein, fft.cpp:140-160): the inverse DFT directly, O(n^2) per row in
// fp64, twiddles exp(+2 pi i j k / n) reseeded from a table (d.tw) every 64
// k and advanced by complex multiplies in between. Same outputs as the chain: block row,
// residue statistics, medians. Shared: the filtered row (16 n) + the real
// parts (8 n) + the selection scratch.
__global__ void __launch_bounds__(kSpThreads) k_sigproc_dft(const SigprocDesc d)
{
    extern __shared__ __align__(16) unsigned char dft_smem[];
    const int n = d.n, tid = threadIdx.x, lane = tid & 31;
    double2* X = reinterpret_cast<double2*>(dft_smem);
    double* re_s = reinterpret_cast<double*>(X + n);
    SpSelect& sel = *reinterpret_cast<SpSelect*>(dft_smem + (((size_t)n * 24 + 15) & ~(size_t)15));
    const int row = blockIdx.x, out_row = row - d.pad;
    const bool in_block = out_row >= 0 && out_row < d.out;
    const double2* src = d.data + (size_t)row * n;
    for (int c = tid; c < n; c += kSpThreads) X[c] = sp_filter_mul(__ldcs(src + c), __ldg(d.filter + c));
    __syncthreads();
    double peak = 0.0, resid = 0.0, lo = INFINITY, hi = -INFINITY;
    double* dst = in_block && d.block ? d.block + (size_t)out_row * n : nullptr;
    constexpr int kJ = 4;  // outputs per thread per sweep: one X[k] load feeds four independent chains
    for (int j0 = tid; j0 < n; j0 += kJ * kSpThreads) {
        double ar[kJ], ai[kJ];
        int m[kJ], jj[kJ];  // m = j k mod n
#pragma unroll
        for (int q = 0; q < kJ; ++q) {
            ar[q] = ai[q] = 0.0;
            m[q] = 0;
            jj[q] = min(j0 + q * kSpThreads, n - 1);  // past n: a duplicate, not stored
        }
        // twiddle w = exp(+2 pi i j k / n): reseeded from the table every 64
        // k, advanced by one complex multiply in between (error ~64 ulp)
        double2 st[kJ];
#pragma unroll
        for (int q = 0; q < kJ; ++q) st[q] = __ldg(d.tw + jj[q]);
        for (int k0 = 0; k0 < n; k0 += 64) {
            double2 w[kJ];
#pragma unroll
            for (int q = 0; q < kJ; ++q) w[q] = __ldg(d.tw + m[q]);
            const int k1 = min(k0 + 64, n);
            for (int k = k0; k < k1; ++k) {
                const double2 x = X[k];
#pragma unroll
                for (int q = 0; q < kJ; ++q) {
                    ar[q] = fma(x.x, w[q].x, fma(-x.y, w[q].y, ar[q]));
                    ai[q] = fma(x.x, w[q].y, fma(x.y, w[q].x, ai[q]));
                    w[q] = c_mul(w[q], st[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < kJ; ++q) m[q] = (int)(((long long)m[q] + 64ll * jj[q]) % n);
        }
#pragma unroll
        for (int q = 0; q < kJ; ++q) {
            const int j = j0 + q * kSpThreads;
            if (j >= n) break;
            const double re = ar[q] * d.inv_n, im = ai[q] * d.inv_n;
            peak = fmax(peak, fabs(re));
            resid = fmax(resid, fabs(im));
            lo = fmin(lo, re);
            hi = fmax(hi, re);
            re_s[j] = re;
            if (dst) __stcs(dst + j, re);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
        resid = fmax(resid, __shfl_xor_sync(0xffffffffu, resid, o));
    }
    if (lane == 0) {
        atomicMax(d.stats, (unsigned long long)__double_as_longlong(peak));
        atomicMax(d.stats + 1, (unsigned long long)__double_as_longlong(resid));
    }
    if (!in_block || !d.medians) return;
    sp_minmax(lo, hi, sel);  // includes the barrier after the re_s stores
    const double med = sp_median_fast(re_s, 1, n, lo, hi, sel);
    if (tid == 0) d.medians[out_row] = med;
}

__global__ void __launch_bounds__(kSpThreads, 2) k_sigproc(const SigprocDesc d)
{
    extern __shared__ __align__(16) unsigned char sp_smem[];
    const int n = d.n;
    double2* buf = reinterpret_cast<double2*>(sp_smem);
    SpSelect& sel = *reinterpret_cast<SpSelect*>(buf + n);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = blockIdx.x;
    const int out_row = row - d.pad;
    const bool in_block = out_row >= 0 && out_row < d.out;

    if (d.mode == 1) {  // row medians of a real matrix
        const double* src = reinterpret_cast<const double*>(d.data) + (size_t)row * n;
        double lo = INFINITY, hi = -INFINITY;
        for (int c = tid; c < n; c += kSpThreads) {
            const double v = __ldcs(src + c);
            buf[c].x = v;
            lo = fmin(lo, v);
            hi = fmax(hi, v);
        }
        sp_minmax(lo, hi, sel);  // includes the barrier after the stores
        const double med = sp_median_fast(reinterpret_cast<const double*>(buf), 2, n, lo, hi, sel);
        if (tid == 0) d.medians[row] = med;
        return;
    }

    // the row: one bulk async copy into shared memory (completion on an
    // mbarrier) while the threads stage the twiddle table
    const double2* src = d.data + (size_t)row * n;
    const uint32_t s_buf = (uint32_t)__cvta_generic_to_shared(buf);
    const uint32_t s_bar = (uint32_t)__cvta_generic_to_shared(&sel.bar);
    const bool bulk = ((reinterpret_cast<uintptr_t>(d.data) & 15) == 0);
    if (bulk && tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(s_bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    if (bulk) {
        if (tid == 0) {
            const uint32_t bytes = (uint32_t)n * 16u;
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(s_bar), "r"(bytes) : "memory");
            constexpr uint32_t kChunk = 32768;
            for (uint32_t off = 0; off < bytes; off += kChunk) {
                const uint32_t sz = bytes - off < kChunk ? bytes - off : kChunk;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        s_buf + off),
                    "l"(reinterpret_cast<const char*>(src) + off), "r"(sz), "r"(s_bar)
                    : "memory");
            }
        }
    } else {
        for (int c = tid; c < n; c += kSpThreads) buf[c] = __ldcs(src + c);
    }
    if (bulk) {
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(s_bar)
                : "memory");
    }
    __syncthreads();
    if (bulk && tid == 0) asm volatile("mbarrier.inval.shared.b64 [%0];" ::"r"(s_bar) : "memory");

    const int r0c = (int)(d.radix[0] & 15);
    if (d.nf == 0 || (r0c > 8)) {  // radix 16 (code 1) fuses the filter too  // no pass (n == 1) or a first radix too wide to fuse the filter into
        for (int c = tid; c < n; c += kSpThreads) buf[c] = sp_filter_mul(buf[c], __ldg(d.filter + c));
        __syncthreads();
    }
    int L = n;
    const double2* tw = d.tw;  // per-pass twiddle tables, back to back
    for (int f = 0; f < d.nf; ++f) {
        const int rc = (int)(((f < 16 ? d.radix[0] : d.radix[1]) >> (4 * (f & 15))) & 15);
        const int R = rc == 1 ? 16 : rc;  // code 1 = radix 16
        if (f == 0)
            sp_pass_any<true>(R, buf, tw, d.filter, n, L);
        else
            sp_pass_any<false>(R, buf, tw, d.filter, n, L);
        L /= R;
        tw += L;  // this pass's table had S = L_new entries
        __syncthreads();
    }

    // natural-order gather: block row, residue statistics, real part kept in place
    double peak = 0.0, resid = 0.0, lo = INFINITY, hi = -INFINITY;
    double* dst = in_block && d.block ? d.block + (size_t)out_row * n : nullptr;
    for (int i = tid; i < n; i += kSpThreads) {
        const int p = __ldg(d.perm + i);
        const double2 v = buf[p];
        const double re = v.x * d.inv_n, im = v.y * d.inv_n;
        peak = fmax(peak, fabs(re));
        resid = fmax(resid, fabs(im));
        lo = fmin(lo, re);
        hi = fmax(hi, re);
        if (dst) __stcs(dst + i, re);
        buf[p].x = re;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
        resid = fmax(resid, __shfl_xor_sync(0xffffffffu, resid, o));
    }
    if (lane == 0) {  // non-negative doubles order as their bit patterns
        atomicMax(d.stats, (unsigned long long)__double_as_longlong(peak));
        atomicMax(d.stats + 1, (unsigned long long)__double_as_longlong(resid));
    }
    (void)warp;
    if (!in_block || !d.medians) return;
    sp_minmax(lo, hi, sel);
    const double med = sp_median_fast(reinterpret_cast<const double*>(buf), 2, n, lo, hi, sel);
    if (tid == 0) d.medians[out_row] = med;
}

}  // namespace wsb

extern "C" size_t wsb_sigproc_smem(int n)
{
    return sizeof(double2) * (size_t)n + sizeof(wsb::SpSelect);
}

extern "C" int wsb_sigproc_dft_max_n()
{
    // the direct-DFT path (lengths with a prime factor > 13)
    return (int)((227 * 1024 - sizeof(wsb::SpSelect) - 16) / 24);
}

extern "C" int wsb_sigproc_max_n()
{
    // largest row that fits one CTA's shared memory (227 KB opt-in)
    int n = 0;
    while (wsb_sigproc_smem(n + 64) <= 227 * 1024) n += 64;
    return n;
}

extern "C" cudaError_t wsb_sigproc_setup()
{
    static std::atomic<unsigned long long> ready{0};  // per-device attribute setup (idempotent)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (ready & (1ull << dev)) return cudaSuccess;
    double2 roots[39];
    const int rs[5] = {3, 5, 7, 11, 13}, off[5] = {0, 3, 8, 15, 26};
    for (int i = 0; i < 5; ++i)
        for (int m = 0; m < rs[i]; ++m) {
            const long double a = 6.283185307179586476925286766559L * m / rs[i];
            roots[off[i] + m] = make_double2((double)cosl(a), (double)sinl(a));
        }
    e = cudaMemcpyToSymbol(wsb::c_sproot, roots, sizeof roots);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(wsb::k_sigproc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(wsb::k_sigproc_dft, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    ready |= 1ull << dev;
    return cudaSuccess;
}

extern "C" cudaError_t wsb_launch_sigproc(const wsb::SigprocDesc& d, cudaStream_t s)
{
    cudaError_t e = wsb_sigproc_setup();
    if (e != cudaSuccess) return e;
    if (d.rows == 0) return cudaSuccess;
    if (d.mode == 2) {
        const size_t smem = (((size_t)d.n * 24 + 15) & ~(size_t)15) + sizeof(wsb::SpSelect);
        wsb::k_sigproc_dft<<<d.rows, wsb::kSpThreads, smem, s>>>(d);
    } else {
        wsb::k_sigproc<<<d.rows, wsb::kSpThreads, wsb_sigproc_smem(d.n), s>>>(d);
    }
    return cudaGetLastError();
}
