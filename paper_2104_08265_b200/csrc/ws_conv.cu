// Fused accumulate + FFT convolution kernel (K3, with K1's scatter fused in).
//
// One CTA owns a band of `rows_per_band` consecutive wire rows of one plane and
// walks them one row at a time, entirely in shared memory:
//
//   1. source the charge row S[w, 0:N)
//        mode 0 (fluctuation off): scatter-add every depo patch that covers
//               the row from the band's depo list (the reference's
//               sample_patch -> scatter_add, rasterize.cpp:66-120 +
//               scatter.cpp:27-36), accumulating q*p in int64 fixed point
//               (2^-32 e-) so the sum is exact and order independent; the
//               cross-wire stencil (spectral.cpp:124-135) is applied to the
//               separable wire profile, S'[w] = sum_dw ww[dw] S[w-dw];
//        mode 1: load S rows from a charge grid (fluctuation on / convolve
//               only), same stencil;
//   2. real FFT of length Np along ticks as a complex FFT of length M = Np/2
//      (row samples paired (2n, 2n+1), so every channel's roundoff is relative
//      to its own norm — never FFT across wires);
//   3. untangle to the half spectrum, multiply by the response spectrum H
//      (ResponseKernel values, spectral.cpp:137 / convolve :160), re-tangle;
//   4. inverse FFT (forward FFT of the conjugate), fold the circular wrap when
//      Np > N, write the frame row (convolve :172-173).
//
// S never touches HBM in mode 0: the only DRAM traffic is the frame write
// (4 B/cell) plus the depo records.
#include "ws_common.cuh"

namespace wsb {

constexpr int kLoBits = 20;              // fixed point split: v = hi * 2^20 + lo
constexpr uint32_t kLoMask = (1u << kLoBits) - 1;
constexpr int kChunk = 4095;             // band entries per pass: lo holds 4096 * 2^20 < 2^32
constexpr float kFix = 16777216.0f;      // 2^24 fixed-point electrons
constexpr float kFixInvF = 1.0f / 16777216.0f;

__device__ __forceinline__ int band_plane(const EventDesc& ev, uint32_t gb)
{
    int p = 0;
#pragma unroll 1
    for (int i = 1; i < ev.n_planes; ++i)
        if (gb >= ev.p[i].band_base) p = i;
    return p;
}

// Scatter-add every band entry that covers row w into the row accumulator,
// one thread per (entry, row): v = c * tv[t] in 2^-24 e- fixed point, split
// into a signed hi word (v >> 20) and an unsigned lo word (v & 0xFFFFF), both
// added with native shared-memory int32 atomics (ATOMS.ADD). Integer sums are
// order independent, so the row is bitwise reproducible for any schedule.
// raw: accumulate the un-stencilled S (charge-grid output) instead of S'.
// Split v (an integer-valued fp32, the 2^-24 e- fixed-point bin value) into
// hi = floor(v / 2^20) and lo = v - hi 2^20 in [0, 2^20) with fp32 ops only
// (magic-number conversions, exact while |hi| < 2^22, i.e. a bin below
// ~2.6e5 e-; larger bins take the 64-bit conversion).
__device__ __forceinline__ void split_fixed(float v, int& hi, uint32_t& lo)
{
    const float hf = floorf(v * (1.0f / 1048576.0f));
    if (fabsf(hf) < 4194304.0f) {
        const float lf = fmaf(-hf, 1048576.0f, v);                      // exact, in [0, 2^20)
        hi = __float_as_int(hf + 12582912.0f) - 0x4B400000;             // 1.5 * 2^23 magic
        lo = (uint32_t)__float_as_int(lf + 8388608.0f) & 0x7FFFFFu;     // 2^23 magic
    } else {
        const long long x = __float2ll_rn(v);
        hi = (int)(x >> kLoBits);
        lo = (uint32_t)x & kLoMask;
    }
}

// Band list entries are full unit records (copied by k_fill), so the scan
// streams them coalesced instead of chasing an index into the record table.
template <int NT>
__device__ __forceinline__ void accumulate_row(const PlaneDesc& P, int w, bool raw, uint32_t* acc_lo, int* acc_hi,
                                               const uint32_t* __restrict__ pool, const UnitRec* __restrict__ list,
                                               uint32_t lo, uint32_t hi, int dbg)
{
    const int W = P.W;
    const int h = P.h;
    const bool stencil = !raw && !P.ww_is_one;
#pragma unroll 1
    for (uint32_t i = lo + threadIdx.x; i < hi; i += NT) {
        const int4 r = __ldg(reinterpret_cast<const int4*>(&list[i]));
        const int w0 = r.x, t0 = r.y, n_w = r.z, n_t = r.w;
        const int lo_row = stencil ? w0 - h : w0;
        const int n_rows = stencil ? n_w + 2 * h : n_w;
        int j = (w - lo_row) % W;
        if (j < 0) j += W;
        if (j >= n_rows) continue;
        const uint32_t off = __ldg(&list[i].pool);
        const float* prof = reinterpret_cast<const float*>(pool + off) + (stencil ? n_w : 0);
        const float* tv = reinterpret_cast<const float*>(pool + off) + n_w + (P.ww_is_one ? 0 : n_w + 2 * h);
        float c = 0.0f;
        for (; j < n_rows; j += W) c += __ldg(&prof[j]);  // a wrap can land twice on a tiny grid
        c *= (float)__ldg(&list[i].a) * kFix;              // q / total, 2^24 fixed point
        // profile loads in batches of 8 so their latencies overlap
#pragma unroll 1
        for (int tb = 0; tb < n_t; tb += 8) {
            float tvv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                tvv[k] = tb + k < n_t ? ((dbg & 32) ? 0.25f : __ldg(&tv[tb + k])) : 0.0f;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (tb + k < n_t) {
                    int vh;
                    uint32_t vl;
                    split_fixed(rintf(c * tvv[k]), vh, vl);
                    if (dbg & 16) {  // profiling only: racy plain adds, to price the atomics
                        acc_lo[t0 + tb + k] += vl;
                        acc_hi[t0 + tb + k] += vh;
                    } else {
                        atomicAdd(&acc_lo[t0 + tb + k], vl);
                        atomicAdd(&acc_hi[t0 + tb + k], vh);
                    }
                }
            }
        }
    }
}

// NT = 256: 16 warps/SM, <= 128 registers, passes of radix <= 25 (3 passes at
// M = 4900); NT = 512: 32 warps/SM, <= 64 registers, radix <= 8 (more passes).
template <int NT, int MAXR>
__global__ void __launch_bounds__(NT, 2)
k_conv(const EventDesc ev, const UnitRec* __restrict__ recs, const uint32_t* __restrict__ pool,
       const uint32_t* __restrict__ band_off, const UnitRec* __restrict__ band_list, int flags)
{
    // flags bit 0: produce the frame; bit 1: raw-charge pass (no wire stencil)
    const bool want_frame = flags & 1;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t gb = blockIdx.x;
    const int pi = band_plane(ev, gb);
    const PlaneDesc& P = ev.p[pi];
    const int band = (int)(gb - P.band_base);
    const int W = P.W, N = P.N, Np = P.Np, M = P.M;
    const int r0 = band * P.rows_per_band;
    const int r1 = min(r0 + P.rows_per_band, W);
    const int tid = threadIdx.x;
    // row workspace (8 * max(N, Np) bytes): the fixed-point accumulator
    // acc_lo[N] | acc_hi[N], aliased by the float row xs[Np] (xs[t] sits on
    // acc_lo[t]) and by the two FFT buffers bufA[M] | bufB[M].
    uint32_t* acc_lo = reinterpret_cast<uint32_t*>(smem);
    int* acc_hi = reinterpret_cast<int*>(smem) + N;
    float2* bufA = reinterpret_cast<float2*>(smem);
    float2* bufB = bufA + M;
    float* xs = reinterpret_cast<float*>(smem);
    const bool raw = flags & 2;
    // split twiddle tables after the workspace (read before the first barrier use)
    float2* s_tw = reinterpret_cast<float2*>(smem + (((size_t)8 * (size_t)max(N, Np) + 15) & ~(size_t)15));
    for (int i = tid; i < kTwiddleTable; i += NT) s_tw[i] = __ldg(&P.tw[i]);
    const TwiddleSplit tw_m{s_tw, s_tw + 64};         // W_M
    const TwiddleSplit tw_np{s_tw + 256, s_tw + 320};  // W_Np

#pragma unroll 1
    for (int w = r0; w < r1; ++w) {
        // the charge grid is the raw S: written by the pass that accumulates without the stencil
        float* crow = (P.charge_out && (raw || P.ww_is_one)) ? P.charge_out + (size_t)w * N : nullptr;
        if (ev.mode == 0) {
            {
                int4* z4 = reinterpret_cast<int4*>(smem);
                const int n4 = (2 * N + 3) / 4;
                for (int i = tid; i < n4; i += NT) z4[i] = make_int4(0, 0, 0, 0);
            }
            __syncthreads();
            const uint32_t lo = band_off[gb], hi = band_off[gb + 1];
#pragma unroll 1
            for (uint32_t c0 = lo; c0 < hi; c0 += kChunk) {
                if (c0 != lo) {
                    // carry lo into hi so the next chunk cannot overflow the lo words
                    __syncthreads();
                    for (int t = tid; t < N; t += NT) {
                        acc_hi[t] += (int)(acc_lo[t] >> kLoBits);
                        acc_lo[t] &= kLoMask;
                    }
                    __syncthreads();
                }
                if (!(flags & 8))  // profiling switch: skip the scatter
                    accumulate_row<NT>(P, w, raw, acc_lo, acc_hi, pool, band_list, c0, min(hi, c0 + kChunk),
                                   flags & 48);
            }
            __syncthreads();
            // fixed point -> fp32 in place (xs[t] overlays acc_lo[t], same thread):
            // normalise lo < 2^20, then one rounding of hi 2^20 + lo (FFMA)
            for (int t = tid; t < N; t += NT) {
                const uint32_t l = acc_lo[t];
                const int hh = acc_hi[t] + (int)(l >> kLoBits);
                const float lf = __int_as_float(0x4B000000 | (l & kLoMask)) - 8388608.0f;
                const float x = fmaf(__int2float_rn(hh), 1048576.0f, lf) * kFixInvF;
                xs[t] = x;
                if (crow) __stcs(&crow[t], x);
            }
            if (Np > N) {
                __syncthreads();  // acc_hi (overlaid by xs[N..Np)) fully read
                for (int t = N + tid; t < Np; t += NT) xs[t] = 0.0f;
            }
        } else {
            // charge grid source with the cross-wire stencil
            for (int t = tid; t < Np; t += NT) {
                float s = 0.0f;
                if (t < N) {
                    for (int dw = -P.h; dw <= P.h; ++dw) {
                        int src = (w - dw) % W;
                        if (src < 0) src += W;
                        s += (float)P.ww[dw + P.h] * __ldg(&P.charge_in[(size_t)src * N + t]);
                    }
                }
                xs[t] = s;
            }
        }
        __syncthreads();
        if (!want_frame) continue;
        if (flags & 4) {  // profiling switch: skip the transforms, store S
            for (int t = tid; t < N; t += NT) P.frame[(size_t)w * N + t] = xs[t];
            __syncthreads();
            continue;
        }

        float2* z = fft_forward<NT, MAXR>(bufA, bufB, M, P.fft, tw_m);

        // untangle -> multiply by H -> re-tangle (conjugated for the inverse)
#pragma unroll 2
        for (int k = tid; k <= M / 2; k += NT) {
            if (k == 0) {
                const float2 z0 = z[0];
                const float x0 = z0.x + z0.y, xm = z0.x - z0.y;  // X[0], X[M]
                const float2 h0 = __ldg(&P.H[0]), hm = __ldg(&P.H[M]);
                const float2 y0 = cscale(h0, x0), ym = cscale(hm, xm);
                const float2 ye = cscale(cadd(y0, ym), 0.5f);
                const float2 yo = cscale(csub(y0, ym), 0.5f);
                // Z' = ye + i*yo ; store conj(Z')
                z[0] = make_float2(ye.x - yo.y, -(ye.y + yo.x));
            } else {
                const int kk = M - k;
                const float2 a = z[k], b = z[kk];
                const float2 wk = tw_np(k);                   // exp(-2 pi i k / Np)
                const float2 wkk = make_float2(-wk.x, wk.y);  // exp(-2 pi i (M-k) / Np) = -conj(wk)
                // X[k] = E + W^k O with E = (a + conj b)/2, O = (a - conj b)/(2i)
                const float2 e1 = cscale(cadd(a, cconj(b)), 0.5f);
                const float2 o1 = cscale(csub(a, cconj(b)), 0.5f);
                const float2 xk = cadd(e1, cmul(wk, make_float2(o1.y, -o1.x)));
                const float2 e2 = cscale(cadd(b, cconj(a)), 0.5f);
                const float2 o2 = cscale(csub(b, cconj(a)), 0.5f);
                const float2 xkk = cadd(e2, cmul(wkk, make_float2(o2.y, -o2.x)));
                const float2 yk = cmul(xk, __ldg(&P.H[k]));
                const float2 ykk = cmul(xkk, __ldg(&P.H[kk]));
                // Z'[k] = YE + i YO, YE = (Y[k] + conj Y[M-k])/2, YO = (Y[k] - conj Y[M-k]) conj(W^k) / 2
                const float2 ye1 = cscale(cadd(yk, cconj(ykk)), 0.5f);
                const float2 yo1 = cmul(cscale(csub(yk, cconj(ykk)), 0.5f), cconj(wk));
                const float2 ye2 = cscale(cadd(ykk, cconj(yk)), 0.5f);
                const float2 yo2 = cmul(cscale(csub(ykk, cconj(yk)), 0.5f), cconj(wkk));
                z[k] = make_float2(ye1.x - yo1.y, -(ye1.y + yo1.x));
                if (kk != k) z[kk] = make_float2(ye2.x - yo2.y, -(ye2.y + yo2.x));
            }
        }
        __syncthreads();

        float2* other = (z == bufA) ? bufB : bufA;
        const float2* y2 = fft_forward<NT, MAXR>(z, other, M, P.fft, tw_m);

        // y[2n] = Re res[n], y[2n+1] = -Im res[n]  (1/M folded into H)
        float* frow = P.frame + (size_t)w * N;
        const float* yr = reinterpret_cast<const float*>(y2);
        const int hi_wrap = P.hi_lag;           // t < hi_wrap: + y[t + N]
        const int lo_wrap = N + P.lo_lag;       // t >= lo_wrap: + y[t - N + Np]
#pragma unroll 4
        for (int t = tid; t < N; t += NT) {
            float y = (t & 1) ? -yr[t] : yr[t];
            if (P.folded) {
                if (t < hi_wrap) {
                    const int tt = t + N;
                    y += (tt & 1) ? -yr[tt] : yr[tt];
                }
                if (t >= lo_wrap) {
                    const int tt = t - N + Np;
                    y += (tt & 1) ? -yr[tt] : yr[tt];
                }
            }
            __stcs(&frow[t], y);  // streaming store: the frame must not evict the band data from L2
        }
        __syncthreads();
    }
}

}  // namespace wsb

// launch helper used by ws_api.cu
extern "C" cudaError_t wsb_launch_conv(const wsb::EventDesc& ev, const wsb::UnitRec* recs, const uint32_t* pool,
                                       const uint32_t* band_off, const wsb::UnitRec* band_list, int flags,
                                       size_t smem_bytes, int threads, cudaStream_t stream)
{
    // once per device: shared-memory opt-in and the composite-radix twiddles
    static unsigned long long ready = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(ready & (1ull << dev))) {
        e = cudaFuncSetAttribute(wsb::k_conv<256, 25>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(wsb::k_conv<512, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        float2 host[wsb::kCompositeTwiddles] = {};
        for (int R : {10, 14, 16, 20, 24, 25, 28, 32, 35, 40, 49}) {
            const int off = wsb::comp_off(R);
            for (int m = 0; m < R; ++m) {
                const double a = -6.283185307179586476925286766559 * (double)m / (double)R;
                host[off + m] = make_float2((float)cos(a), (float)sin(a));
            }
        }
        e = cudaMemcpyToSymbol(wsb::c_wr, host, sizeof(host));
        if (e != cudaSuccess) return e;
        ready |= 1ull << dev;
    }
    if (ev.total_bands == 0) return cudaSuccess;
    if (threads == 512)
        wsb::k_conv<512, 8><<<ev.total_bands, 512, smem_bytes, stream>>>(ev, recs, pool, band_off, band_list, flags);
    else
        wsb::k_conv<256, 25><<<ev.total_bands, 256, smem_bytes, stream>>>(ev, recs, pool, band_off, band_list, flags);
    return cudaGetLastError();
}
