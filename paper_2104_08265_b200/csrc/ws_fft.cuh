// Shared-memory mixed-radix Stockham FFT (complex fp32) for one tick row.
//
// Replaces the reference's recursive double FFT (fft.cpp:116-161) on the hot
// path. The transform length M is 7-smooth and planned on the host
// (ws_api.cu: plan_passes) into few passes of large radices (2..40, composite
// radices run as two nested small DFTs in registers), so a row needs ~3
// shared-memory round trips per transform instead of log2(M). Passes
// ping-pong between two M-element buffers (16*M bytes of shared memory, the
// footprint of the row's fixed-point accumulator, which they alias).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace wsb {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by -i
__device__ __forceinline__ float2 cmul_mi(float2 a) { return make_float2(a.y, -a.x); }

// Twiddles W_R^m = exp(-2 pi i m / R) of the composite in-register DFTs, filled
// by the host (ws_api.cu). After full unrolling every index is a compile-time
// constant, so the values become constant-bank operands of the FMAs.
constexpr int kCompositeTwiddles = 512;
static __constant__ float2 c_wr[kCompositeTwiddles];
// offset of W_R^0 in c_wr for composite R (host and device share this map)
__host__ __device__ constexpr int comp_off(int R)
{
    return R == 10 ? 0 : R == 14 ? 10 : R == 16 ? 24 : R == 20 ? 40 : R == 24 ? 60 : R == 25 ? 84 : R == 28 ? 109
         : R == 32 ? 137 : R == 35 ? 169 : R == 40 ? 204 : R == 49 ? 244 : -1;
}

// Forward DFT of size R in registers: X_k = sum_n x_n exp(-2 pi i n k / R).
template <int R>
struct Dft;

template <>
struct Dft<2> {
    static __device__ __forceinline__ void run(float2* v)
    {
        const float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template <>
struct Dft<4> {
    static __device__ __forceinline__ void run(float2* v)
    {
        const float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        const float2 s13 = cadd(v[1], v[3]), d13 = cmul_mi(csub(v[1], v[3]));
        v[0] = cadd(s02, s13);
        v[2] = csub(s02, s13);
        v[1] = cadd(d02, d13);
        v[3] = csub(d02, d13);
    }
};

template <>
struct Dft<8> {
    static __device__ __forceinline__ void run(float2* v)
    {
        constexpr float r = 0.70710678118654752440f;
        float2 a[4], b[4];
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            a[n] = cadd(v[n], v[n + 4]);
            b[n] = csub(v[n], v[n + 4]);
        }
        // b[n] *= exp(-2 pi i n / 8)
        b[1] = make_float2(r * (b[1].x + b[1].y), r * (b[1].y - b[1].x));
        b[2] = cmul_mi(b[2]);
        b[3] = make_float2(r * (b[3].y - b[3].x), -r * (b[3].x + b[3].y));
        Dft<4>::run(a);
        Dft<4>::run(b);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = a[k];
            v[2 * k + 1] = b[k];
        }
    }
};

// Odd prime radix via the symmetric-pair form: with a_m = x_m + x_{R-m},
// b_m = x_m - x_{R-m}: X_k = x_0 + sum_m a_m cos(2 pi k m / R) - i sum_m b_m sin(...).
template <int R>
struct OddDft {
    static __device__ __forceinline__ float cosv(int km);
    static __device__ __forceinline__ float sinv(int km);
};

template <>
__device__ __forceinline__ float OddDft<3>::cosv(int km)
{
    return (km % 3 == 0) ? 1.0f : -0.5f;
}
template <>
__device__ __forceinline__ float OddDft<3>::sinv(int km)
{
    const int r = km % 3;
    return r == 0 ? 0.0f : (r == 1 ? 0.86602540378443864676f : -0.86602540378443864676f);
}

template <>
__device__ __forceinline__ float OddDft<5>::cosv(int km)
{
    const int r = km % 5;
    return r == 0 ? 1.0f : (r == 1 || r == 4) ? 0.30901699437494742410f : -0.80901699437494742410f;
}
template <>
__device__ __forceinline__ float OddDft<5>::sinv(int km)
{
    const int r = km % 5;
    return r == 0 ? 0.0f
         : r == 1 ? 0.95105651629515357212f
         : r == 2 ? 0.58778525229247312917f
         : r == 3 ? -0.58778525229247312917f
                  : -0.95105651629515357212f;
}

template <>
__device__ __forceinline__ float OddDft<7>::cosv(int km)
{
    const int r = km % 7;
    return r == 0 ? 1.0f
         : (r == 1 || r == 6) ? 0.62348980185873353053f
         : (r == 2 || r == 5) ? -0.22252093395631440429f
                              : -0.90096886790241912624f;
}
template <>
__device__ __forceinline__ float OddDft<7>::sinv(int km)
{
    const int r = km % 7;
    return r == 0 ? 0.0f
         : r == 1 ? 0.78183148246802980871f
         : r == 2 ? 0.97492791218182360702f
         : r == 3 ? 0.43388373911755812048f
         : r == 4 ? -0.43388373911755812048f
         : r == 5 ? -0.97492791218182360702f
                  : -0.78183148246802980871f;
}

template <int R>
struct DftOdd {
    static __device__ __forceinline__ void run(float2* v)
    {
        constexpr int H = (R - 1) / 2;
        float2 a[H], b[H];
        float2 s = v[0];
#pragma unroll
        for (int m = 1; m <= H; ++m) {
            a[m - 1] = cadd(v[m], v[R - m]);
            b[m - 1] = csub(v[m], v[R - m]);
            s = cadd(s, a[m - 1]);
        }
        float2 out[R];
        out[0] = s;
#pragma unroll
        for (int k = 1; k <= H; ++k) {
            float2 re = v[0], im = make_float2(0.f, 0.f);
#pragma unroll
            for (int m = 1; m <= H; ++m) {
                const float c = OddDft<R>::cosv(k * m), sn = OddDft<R>::sinv(k * m);
                re.x += a[m - 1].x * c;
                re.y += a[m - 1].y * c;
                im.x += b[m - 1].x * sn;
                im.y += b[m - 1].y * sn;
            }
            // X_k = re - i*im ; X_{R-k} = re + i*im
            out[k] = make_float2(re.x + im.y, re.y - im.x);
            out[R - k] = make_float2(re.x - im.y, re.y + im.x);
        }
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = out[k];
    }
};

template <>
struct Dft<3> : DftOdd<3> {};
template <>
struct Dft<5> : DftOdd<5> {};
template <>
struct Dft<7> : DftOdd<7> {};

// Composite R = A*B in registers (Cooley-Tukey, n = n1 + A n2, k = k2 + B k1):
// DFT_B over n2 for every n1, twiddle by W_R^{n1 k2}, DFT_A over n1. Works in
// place: X[k2 + B k1] ends in slot k1 + A k2, exposed through pos().
template <int A, int B>
struct DftComp {
    static __host__ __device__ constexpr int pos(int r) { return (r / B) + A * (r % B); }
    static __device__ __forceinline__ void run(float2* v)
    {
        constexpr int R = A * B;
        constexpr int off = comp_off(R);
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {
            float2 t[B];
#pragma unroll
            for (int n2 = 0; n2 < B; ++n2) t[n2] = v[n1 + A * n2];
            Dft<B>::run(t);
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2)
                v[n1 + A * k2] = (n1 * k2 == 0) ? t[k2] : cmul(t[k2], c_wr[off + (n1 * k2) % R]);
        }
#pragma unroll
        for (int k2 = 0; k2 < B; ++k2) {
            float2 z[A];
#pragma unroll
            for (int n1 = 0; n1 < A; ++n1) z[n1] = v[n1 + A * k2];
            Dft<A>::run(z);
#pragma unroll
            for (int k1 = 0; k1 < A; ++k1) v[k1 + A * k2] = z[k1];
        }
    }
};

// slot of output X[r] after Dft<R>::run (identity unless composite)
template <int R>
struct DftPos {
    static __host__ __device__ constexpr int pos(int r) { return r; }
};

template <> struct DftPos<10> : DftComp<2, 5> {};
template <> struct DftPos<14> : DftComp<2, 7> {};
template <> struct DftPos<16> : DftComp<4, 4> {};
template <> struct DftPos<20> : DftComp<4, 5> {};
template <> struct DftPos<24> : DftComp<8, 3> {};
template <> struct DftPos<25> : DftComp<5, 5> {};
template <> struct DftPos<28> : DftComp<4, 7> {};
template <> struct DftPos<32> : DftComp<8, 4> {};

template <> struct Dft<10> : DftComp<2, 5> {};
template <> struct Dft<14> : DftComp<2, 7> {};
template <> struct Dft<16> : DftComp<4, 4> {};
template <> struct Dft<20> : DftComp<4, 5> {};
template <> struct Dft<24> : DftComp<8, 3> {};
template <> struct Dft<25> : DftComp<5, 5> {};
template <> struct Dft<28> : DftComp<4, 7> {};
template <> struct Dft<32> : DftComp<8, 4> {};
template <> struct Dft<35> : DftComp<5, 7> {};
template <> struct Dft<40> : DftComp<8, 5> {};

// ---------------------------------------------------------------------------
// In-place mixed-radix DIF / DIT pair for convolution (no digit reversal pass).
//
// DIF (Sande-Tukey) with radices R_0..R_{P-1}: pass p has sub-transforms of
// length L_p = M / (R_0..R_{p-1}) and stride S_p = L_p / R_p; butterfly
// (block b, offset j < S_p) reads x[b L_p + j + r S_p], runs DFT_R, multiplies
// output q by W_{L_p}^{j q}, writes back to the same slots. The result X[k]
// lands at pos(k) = sum_p q_p M / (R_0..R_p) for k = sum_p q_p R_0..R_{p-1}.
// DIT (Cooley-Tukey) with the radices reversed consumes exactly that order and
// returns natural order: butterfly (b, j < Lam_p) pre-multiplies x_r by
// W_{Lam_p R}^{j r}, runs DFT_R, writes back. Each butterfly touches only its
// own slots, so a pass needs a single barrier and one row of shared memory.
struct FftPlanDev {
    int npass;
    int radix[12];        // DIF order; DIT runs radix[npass-1-p] at pass p
    int dif_s[12];        // S_p
    uint32_t dif_mg[12];  // ceil(2^32 / S_p)
    int dif_step[12];     // M / L_p: W_{L_p}^{jq} = W_M^{jq step}
    int dit_lam[12];      // Lam_p
    uint32_t dit_mg[12];  // ceil(2^32 / Lam_p)
    int dit_step[12];     // M / (Lam_p R)
};

// W_M^m from two 64-way shared-memory tables: lo[j] = W_M^j, hi[i] = W_M^{64 i}.
struct TwiddleSplit {
    const float2* lo;
    const float2* hi;
    __device__ __forceinline__ float2 operator()(int m) const { return cmul(hi[m >> 6], lo[m & 63]); }
};

__device__ __forceinline__ int fast_div(int a, int d, uint32_t mg) { return d > 1 ? (int)__umulhi((uint32_t)a, mg) : a; }

template <int R, int NT>
__device__ __forceinline__ void dif_pass(float2* __restrict__ x, int M, int S, uint32_t mg, int step,
                                         const TwiddleSplit& tw)
{
    const int L = S * R;
#pragma unroll 1
    for (int g = threadIdx.x; g < M / R; g += NT) {
        const int b = fast_div(g, S, mg);
        const int j = g - b * S;
        float2* p = x + b * L + j;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = p[r * S];
        Dft<R>::run(v);
        if (j) {
            const int dm = j * step;
            int m = dm;
#pragma unroll
            for (int q = 1; q < R; ++q, m += dm) v[DftPos<R>::pos(q)] = cmul(v[DftPos<R>::pos(q)], tw(m));
        }
#pragma unroll
        for (int q = 0; q < R; ++q) p[q * S] = v[DftPos<R>::pos(q)];
    }
}

template <int R, int NT>
__device__ __forceinline__ void dit_pass(float2* __restrict__ x, int M, int Lam, uint32_t mg, int step,
                                         const TwiddleSplit& tw)
{
    const int L = Lam * R;
#pragma unroll 1
    for (int g = threadIdx.x; g < M / R; g += NT) {
        const int b = fast_div(g, Lam, mg);
        const int j = g - b * Lam;
        float2* p = x + b * L + j;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = p[r * Lam];
        if (j) {
            const int dm = j * step;
            int m = dm;
#pragma unroll
            for (int r = 1; r < R; ++r, m += dm) v[r] = cmul(v[r], tw(m));
        }
        Dft<R>::run(v);
#pragma unroll
        for (int q = 0; q < R; ++q) p[q * Lam] = v[DftPos<R>::pos(q)];
    }
}

#define WSB_RADIX_SWITCH(R_, CALL)                     \
    switch (R_) {                                      \
        case 2: CALL(2); break;                        \
        case 3: CALL(3); break;                        \
        case 4: CALL(4); break;                        \
        case 5: CALL(5); break;                        \
        case 7: CALL(7); break;                        \
        case 8: CALL(8); break;                        \
        default:                                       \
            if constexpr (MAXR >= 25) {                \
                switch (R_) {                          \
                    case 10: CALL(10); break;          \
                    case 14: CALL(14); break;          \
                    case 16: CALL(16); break;          \
                    case 20: CALL(20); break;          \
                    case 24: CALL(24); break;          \
                    default: CALL(25); break;          \
                }                                      \
            }                                          \
            break;                                     \
    }

// forward DFT, natural order in, digit-reversed (pos) order out
template <int NT, int MAXR>
__device__ __forceinline__ void fft_dif(float2* x, int M, const FftPlanDev& pl, const TwiddleSplit& tw)
{
#pragma unroll 1
    for (int p = 0; p < pl.npass; ++p) {
        const int S = pl.dif_s[p], st = pl.dif_step[p];
        const uint32_t mg = pl.dif_mg[p];
#define WSB_DIF(R) dif_pass<R, NT>(x, M, S, mg, st, tw)
        WSB_RADIX_SWITCH(pl.radix[p], WSB_DIF)
#undef WSB_DIF
        __syncthreads();
    }
}

// forward DFT, digit-reversed (pos) order in, natural order out
template <int NT, int MAXR>
__device__ __forceinline__ void fft_dit(float2* x, int M, const FftPlanDev& pl, const TwiddleSplit& tw)
{
#pragma unroll 1
    for (int p = 0; p < pl.npass; ++p) {
        const int lam = pl.dit_lam[p], st = pl.dit_step[p];
        const uint32_t mg = pl.dit_mg[p];
#define WSB_DIT(R) dit_pass<R, NT>(x, M, lam, mg, st, tw)
        WSB_RADIX_SWITCH(pl.radix[pl.npass - 1 - p], WSB_DIT)
#undef WSB_DIT
        __syncthreads();
    }
}

}  // namespace wsb
