// Fused scatter + FFT convolution kernel (k_conv: K1's scatter fused into K3).
//
// One CTA owns a band of `rows_per_band` consecutive wire rows of one plane and
// walks them one row at a time, entirely in one row of shared memory
// (4 B/tick), so several rows are in flight per SM:
//
//   1. source the charge row S[w, 0:N)
//        mode 0 (fluctuation off): scatter-add every depo patch that covers
//               the row from the band's depo list (the reference's
//               sample_patch -> scatter_add, rasterize.cpp:66-120 +
//               scatter.cpp:27-36), with the cross-wire stencil applied to
//               the separable wire profile, S'[w] = sum_dw ww[dw] S[w-dw]
//               (spectral.cpp:124-135). Accumulation is int32 fixed point at a
//               per-row power-of-two scale chosen from a rigorous bound (each
//               covering depo adds ceil(|c| max(tv)) to the 64-tick segments it
//               touches; the largest segment bound maps to 2^30), so no sum can
//               overflow for any depo count, one native shared-memory atomic
//               (ATOMS.ADD) per bin suffices, and the row is bitwise
//               reproducible for any schedule;
//        mode 1: load S rows from a charge grid (fluctuation on / convolve
//               only), same stencil;
//   2. real FFT of length Np along ticks as a complex FFT of length M = Np/2
//      (sample pairs (2n, 2n+1), so each channel's roundoff is relative to its
//      own norm — never FFT across wires), in place, DIF
//      (natural in, digit-reversed out);
//   3. untangle to the half spectrum, multiply by the response spectrum H
//      (ResponseKernel values, spectral.cpp:137 / convolve :160), re-tangle,
//      all in digit-reversed positions;
//   4. inverse as a forward DIT of the conjugate (digit-reversed in, natural
//      out), fold of the circular wrap when Np > N, frame row store
//      (convolve :172-173).
//
// S never touches HBM in mode 0: the only DRAM traffic is the frame write
// (4 B/cell) plus the depo records.
#include "ws_common.cuh"

#include <atomic>

namespace wsb {

constexpr int kSegShift = 6;  // 64-tick bound segments

// One covering (entry, row) pair.
struct Cover {
    float c;       // a * (stencilled) wire weight of this row
    int t0, n_t;
    uint32_t tvo;  // pool offset of the tick profile
};

// Does band entry i cover row w? raw: the un-stencilled S (charge output).
__device__ __forceinline__ bool cover_of(const PlaneDesc& P, int w, bool raw, const UnitRec* __restrict__ list,
                                         const uint32_t* __restrict__ pool, uint32_t i, Cover& cv, float& tmax)
{
    const int4 r = __ldg(reinterpret_cast<const int4*>(&list[i]));
    const int w0 = r.x, n_w = r.z;
    const int h = P.h;
    const bool stencil = !raw && !P.ww_is_one;
    const int lo_row = stencil ? w0 - h : w0;
    const int n_rows = stencil ? n_w + 2 * h : n_w;
    int j = (w - lo_row) % P.W;
    if (j < 0) j += P.W;
    if (j >= n_rows) return false;
    const uint32_t off = __ldg(&list[i].pool);
    const float2 at = __ldg(reinterpret_cast<const float2*>(&list[i].a));  // a, tsum (>= max of the tick profile)
    const float* prof = reinterpret_cast<const float*>(pool + off) + (stencil ? n_w : 0);
    float c = 0.0f;
    for (; j < n_rows; j += P.W) c += __ldg(&prof[j]);  // a wrap can land twice on a tiny grid
    cv.c = c * at.x;
    cv.t0 = r.y;
    cv.n_t = r.w;
    cv.tvo = off + n_w + (P.ww_is_one ? 0 : n_w + 2 * h);
    tmax = at.y;
    return true;
}

constexpr int kKeep = 4;  // covering entries per thread carried from the bound pass

template <int NT>
__device__ __forceinline__ void scatter_row(const PlaneDesc& P, int w, bool raw, int* acc, unsigned* segb, int* s_red,
                                            int nseg, const uint32_t* __restrict__ pool,
                                            const UnitRec* __restrict__ list, uint32_t lo, uint32_t hi, float& inv)
{
    const int tid = threadIdx.x;
    // pass 1: bounds per 64-tick segment in units of 2^ue electrons (rounded
    // up); the first kKeep covers of this thread stay in registers for pass
    // 2. The row's total of all cover bounds (>= every segment sum) decides
    // whether a 32-bit sum could overflow (extreme charges only): then the
    // pass re-runs with a 2^16 coarser unit.
    Cover keep[kKeep];
    int keep_at[kKeep];
    int nkeep, kdone, ue = 0;
#pragma unroll 1
    for (;;) {
        nkeep = 0;
        kdone = 0x7fffffff;  // iterations <= kdone are fully classified
        double tot = 0.0;
#pragma unroll 1
        for (uint32_t i = lo + tid, k = 0; i < hi; i += NT, ++k) {
            Cover cv;
            float tm;
            if (!cover_of(P, w, raw, list, pool, i, cv, tm)) continue;
            const float bu = ceilf(ldexpf(fabsf(cv.c) * tm, -ue)) + 1.0f;
            tot += (double)bu;
            const unsigned b = (unsigned)fminf(bu, 4.0e9f);
            const int s0 = cv.t0 >> kSegShift, s1 = (cv.t0 + cv.n_t - 1) >> kSegShift;
            for (int s = s0; s <= s1; ++s) atomicAdd(&segb[s], b);
            if (nkeep < kKeep) {
                keep[nkeep] = cv;
                keep_at[nkeep] = (int)k;
                if (++nkeep == kKeep) kdone = (int)k;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        double* s_tot = reinterpret_cast<double*>(s_red);  // NT / 32 <= 16 doubles
        if ((tid & 31) == 0) s_tot[tid >> 5] = tot;
        __syncthreads();
        tot = 0.0;
#pragma unroll
        for (int q = 0; q < NT / 32; ++q) tot += s_tot[q];
        __syncthreads();  // s_red is reused below
        if (tot < 4294967296.0) break;
        ue += 16;
        for (int i = tid; i < nseg; i += NT) segb[i] = 0u;
        __syncthreads();
    }
    // scale: the largest segment bound maps below 2^30
    unsigned mx = 0u;
    for (int i = tid; i < nseg; i += NT) mx = max(mx, segb[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) s_red[tid >> 5] = (int)mx;
    __syncthreads();
    mx = 0u;
#pragma unroll
    for (int q = 0; q < NT / 32; ++q) mx = max(mx, (unsigned)s_red[q]);
    const int sh = 30 - (32 - __clz(mx) + ue);  // bound < 2^(32-clz+ue)  =>  bound 2^sh < 2^30
    const float scale = ldexpf(1.0f, sh);
    inv = ldexpf(1.0f, -sh);
    // pass 2: scatter, one int32 shared atomic per bin
    int kk = 0;
#pragma unroll 1
    for (uint32_t i = lo + tid, k = 0; i < hi; i += NT, ++k) {
        Cover cv;
        float tm;
        if ((int)k <= kdone) {  // classified in pass 1: a kept cover or not covering
            if (kk >= nkeep || keep_at[kk] != (int)k) continue;
            cv = keep[kk++];
        } else if (!cover_of(P, w, raw, list, pool, i, cv, tm)) {
            continue;
        }
        const float cs = cv.c * scale;
        const float* tv = reinterpret_cast<const float*>(pool + cv.tvo);
#pragma unroll 1
        for (int tb = 0; tb < cv.n_t; tb += 8) {
            float tvv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) tvv[q] = tb + q < cv.n_t ? __ldg(&tv[tb + q]) : 0.0f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (tb + q < cv.n_t) atomicAdd(&acc[cv.t0 + tb + q], __float2int_rn(cs * tvv[q]));
        }
    }
}

template <int NT, int MAXR, int MINB>
__global__ void __launch_bounds__(NT, MINB)
k_conv(const EventDesc ev, const uint32_t* __restrict__ pool, const uint32_t* __restrict__ band_off,
       const UnitRec* __restrict__ band_list, int flags)
{
    // flags bit 0: produce the frame; bit 1: raw-charge pass (no wire stencil)
    extern __shared__ __align__(16) unsigned char smem[];
    const bool want_frame = flags & 1;
    const bool raw = flags & 2;
    const uint32_t gb = blockIdx.x;
    const PlaneDesc& P = ev.p[band_plane(ev, gb)];
    if (P.direct) return;  // tiles of a time-domain plane (k_direct)
    if (ev.mode == 0 && __ldg(&band_off[ev.total_bands]) > ev.list_cap) return;  // lists overflowed (kErrRange)
    const int band = (int)(gb - P.band_base);
    const int W = P.W, N = P.N, Np = P.Np, M = P.M;
    const int r0 = band * P.rows_per_band;
    const int r1 = min(r0 + P.rows_per_band, W);
    const int tid = threadIdx.x;
    const int nseg = (N + 63) >> kSegShift;
    // layout: row (4*Np bytes: int32 accumulator / float row / complex
    // half-length spectrum, all in place) | segment bounds | twiddles |
    // digit-reversal table | reduce scratch
    int* acc = reinterpret_cast<int*>(smem);
    float* xs = reinterpret_cast<float*>(smem);
    float2* buf = reinterpret_cast<float2*>(smem);
    size_t off = ((size_t)4 * Np + 15) & ~(size_t)15;
    unsigned* segb = reinterpret_cast<unsigned*>(smem + off);
    off += ((size_t)4 * nseg + 15) & ~(size_t)15;
    float2* s_tw = reinterpret_cast<float2*>(smem + off);
    off += sizeof(float2) * kTwiddleTable;
    uint16_t* s_rev = reinterpret_cast<uint16_t*>(smem + off);
    off += ((size_t)2 * M + 15) & ~(size_t)15;
    int* s_red = reinterpret_cast<int*>(smem + off);
    for (int i = tid; i < kTwiddleTable; i += NT) s_tw[i] = __ldg(&P.tw[i]);
    for (int i = tid; i < M; i += NT) s_rev[i] = __ldg(&P.rev[i]);
    const TwiddleSplit tw_m{s_tw, s_tw + 64};         // W_M
    const TwiddleSplit tw_np{s_tw + 256, s_tw + 320};  // W_Np
    const uint32_t lo = ev.mode == 0 ? band_off[gb] : 0u, hi = ev.mode == 0 ? band_off[gb + 1] : 0u;

#pragma unroll 1
    for (int w = r0; w < r1; ++w) {
                float* crow = (P.charge_out && raw) ? P.charge_out + (size_t)w * N : nullptr;
        if (ev.mode == 0) {
            {
                int4* z4 = reinterpret_cast<int4*>(smem);
                for (int i = tid; i < (Np + 3) / 4; i += NT) z4[i] = make_int4(0, 0, 0, 0);
                for (int i = tid; i < nseg; i += NT) segb[i] = 0u;
            }
            __syncthreads();
            float inv;
            scatter_row<NT>(P, w, raw, acc, segb, s_red, nseg, pool, band_list, lo, hi, inv);
            __syncthreads();
            for (int t = tid; t < N; t += NT) {  // int -> float in place (same index, same thread)
                const float x = (float)acc[t] * inv;
                xs[t] = x;
                if (crow) __stcs(&crow[t], x);
            }
        } else {
            for (int t = tid; t < Np; t += NT) {
                float s = 0.0f;
                if (t < N) {
                    for (int dw = -P.h; dw <= P.h; ++dw) {
                        int src = (w - dw) % W;
                        if (src < 0) src += W;
                        // the integer grid of the fluctuation walk, or a float grid (ws_convolve_device)
                        const float q = P.charge_cnt ? (float)count_at(P, (size_t)src * N + t, cnt_wide(P))
                                                     : __ldg(&P.charge_in[(size_t)src * N + t]);
                        s += (float)P.ww[dw + P.h] * q;
                    }
                }
                xs[t] = s;
            }
        }
        __syncthreads();
        if (!want_frame || !(P.frame || P.frame64 || P.adc)) continue;  // (block-uniform)

        fft_dif<NT, MAXR>(buf, M, P.fft, tw_m);

        // untangle -> multiply by H -> re-tangle (conjugated for the inverse);
        // spectrum bin k lives at s_rev[k]
#pragma unroll 2
        for (int k = tid; k <= M / 2; k += NT) {
            if (k == 0) {
                const int p0 = s_rev[0];
                const float2 z0 = buf[p0];
                const float x0 = z0.x + z0.y, xm = z0.x - z0.y;  // X[0], X[M]
                const float2 y0 = cscale(__ldg(&P.H[0]), x0), ym = cscale(__ldg(&P.H[M]), xm);
                const float2 ye = cscale(cadd(y0, ym), 0.5f);
                const float2 yo = cscale(csub(y0, ym), 0.5f);
                buf[p0] = make_float2(ye.x - yo.y, -(ye.y + yo.x));  // conj(ye + i yo)
            } else {
                const int kk = M - k;
                const int pk = s_rev[k], pkk = s_rev[kk];
                const float2 a = buf[pk], b = buf[pkk];
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
                buf[pk] = make_float2(ye1.x - yo1.y, -(ye1.y + yo1.x));
                if (kk != k) buf[pkk] = make_float2(ye2.x - yo2.y, -(ye2.y + yo2.x));
            }
        }
        __syncthreads();

        fft_dit<NT, MAXR>(buf, M, P.fft, tw_m);

        // y[2n] = Re res[n], y[2n+1] = -Im res[n]  (1/M folded into H)
        const int hi_wrap = P.hi_lag;      // t < hi_wrap: + y[t + N]
        const int lo_wrap = N + P.lo_lag;  // t >= lo_wrap: + y[t - N + Np]
        auto sample = [&](int t) {
            float y = (t & 1) ? -xs[t] : xs[t];
            if (P.folded) {
                if (t < hi_wrap) {
                    const int tt = t + N;
                    y += (tt & 1) ? -xs[tt] : xs[tt];
                }
                if (t >= lo_wrap) {
                    const int tt = t - N + Np;
                    y += (tt & 1) ? -xs[tt] : xs[tt];
                }
            }
            return y;
        };
        if (!ev.ro) {
            float* frow = P.frame + (size_t)w * N;
#pragma unroll 4
            for (int t = tid; t < N; t += NT) __stcs(&frow[t], sample(t));  // streaming store: keep the band data in L2
        } else {
            // fused readout (noise + digitize, fp64 frame), one tick pair per thread
            for (int t = 2 * tid; t < N; t += 2 * NT) {
                const bool has1 = t + 1 < N;
                readout_pair(ev, P, w, t, sample(t), has1 ? sample(t + 1) : 0.0f, has1);
            }
        }
        __syncthreads();
    }
}

// Spectrum-mode electronics noise (the reference's add_noise, NoiseMode::
// spectrum, spectral.cpp:198-225): one CTA per wire row synthesises the
// waveform IFFT_N(X) with X[k] = amp[k] e^{2 pi i u_k} Hermitian-completed
// (X[0], X[N/2] real: amp cos(2 pi u)), u_k the row's k-th uniform of the
// reference's stream substream(seed ^ kSpectrumNoiseSalt, w) (drawn by one
// thread: the stream is sequential) or of the Philox stream (one draw per
// thread), and adds it to the frame row (optionally digitizing). The
// half-length real inverse transform is k_conv's second half: re-tangle of
// the half spectrum into the digit-reversed layout, DIT of the conjugate.
// Needs an even, 7-smooth padded tick count (Np == N).
template <int NT, int MAXR>
__global__ void __launch_bounds__(NT)
k_noise_spectrum(const PlaneDesc P, const double* __restrict__ amp, uint64_t seed, int rng_mode, const float* in,
                 const Sink out)
{
    constexpr uint64_t kSpectrumNoiseSalt = 0x737065636e6f6973ULL;  // spectral.cpp:22
    extern __shared__ __align__(16) unsigned char smem[];
    const int w = blockIdx.x, tid = threadIdx.x;
    const int N = P.N, M = P.M;
    float2* buf = reinterpret_cast<float2*>(smem);
    float* xs = reinterpret_cast<float*>(smem);
    size_t off = ((size_t)8 * M + 15) & ~(size_t)15;
    float2* s_tw = reinterpret_cast<float2*>(smem + off);
    off += sizeof(float2) * kTwiddleTable;
    uint16_t* s_rev = reinterpret_cast<uint16_t*>(smem + off);
    off += ((size_t)2 * M + 15) & ~(size_t)15;
    double* s_u = reinterpret_cast<double*>(smem + off);  // M + 1 uniforms
    for (int i = tid; i < kTwiddleTable; i += NT) s_tw[i] = __ldg(&P.tw[i]);
    for (int i = tid; i < M; i += NT) s_rev[i] = __ldg(&P.rev[i]);
    const TwiddleSplit tw_m{s_tw, s_tw + 64};
    const TwiddleSplit tw_np{s_tw + 256, s_tw + 320};
    if (rng_mode == WS_RNG_SUBSTREAM) {
        if (tid == 0) {
            Rng src;
            src.init(WS_RNG_SUBSTREAM, seed ^ kSpectrumNoiseSalt, (uint64_t)w);
            for (int k = 0; k <= M; ++k) s_u[k] = src.uniform();
        }
    } else {
        for (int k = tid; k <= M; k += NT) {
            Rng src;
            src.init(WS_RNG_PHILOX, seed ^ kSpectrumNoiseSalt, (uint64_t)w);
            src.draw = (uint32_t)k;
            s_u[k] = src.uniform();
        }
    }
    __syncthreads();
    // Y[k] = X[k] / M (k_conv's spectrum scaling: the DIT below then yields IFFT_N(X), 1/N included)
    const double kTwoPiD = 6.283185307179586476925286766559;
    auto Y = [&](int k) {
        const double a = amp[k] / (double)M;
        if (k == 0 || k == M) return make_float2((float)(a * cos(kTwoPiD * s_u[k])), 0.0f);
        double sn, cs;
        sincos(kTwoPiD * s_u[k], &sn, &cs);
        return make_float2((float)(a * cs), (float)(a * sn));
    };
    for (int k = tid; k <= M / 2; k += NT) {
        if (k == 0) {
            const float2 y0 = Y(0), ym = Y(M);
            const float2 ye = cscale(cadd(y0, ym), 0.5f);
            const float2 yo = cscale(csub(y0, ym), 0.5f);
            buf[s_rev[0]] = make_float2(ye.x - yo.y, -(ye.y + yo.x));  // conj(ye + i yo)
        } else {
            const int kk = M - k;
            const float2 wk = tw_np(k);
            const float2 wkk = make_float2(-wk.x, wk.y);
            const float2 yk = Y(k), ykk = Y(kk);
            const float2 ye1 = cscale(cadd(yk, cconj(ykk)), 0.5f);
            const float2 yo1 = cmul(cscale(csub(yk, cconj(ykk)), 0.5f), cconj(wk));
            const float2 ye2 = cscale(cadd(ykk, cconj(yk)), 0.5f);
            const float2 yo2 = cmul(cscale(csub(ykk, cconj(yk)), 0.5f), cconj(wkk));
            buf[s_rev[k]] = make_float2(ye1.x - yo1.y, -(ye1.y + yo1.x));
            if (kk != k) buf[s_rev[kk]] = make_float2(ye2.x - yo2.y, -(ye2.y + yo2.x));
        }
    }
    __syncthreads();
    fft_dit<NT, MAXR>(buf, M, P.fft, tw_m);
    // y[2n] = Re res[n], y[2n+1] = -Im res[n]; add to the row (fp64), digitize
    const size_t base = (size_t)w * N;
    for (int t = tid; t < N; t += NT) {
        const float y = (t & 1) ? -xs[t] : xs[t];
        sink_put(out, base + t, __dadd_rn((double)in[base + t], (double)y));
    }
}

}  // namespace wsb

extern "C" size_t wsb_conv_smem(int N, int Np, int M)
{
    const int nseg = (N + 63) >> wsb::kSegShift;
    return (((size_t)4 * Np + 15) & ~(size_t)15) + (((size_t)4 * nseg + 15) & ~(size_t)15) +
           sizeof(float2) * wsb::kTwiddleTable + (((size_t)2 * M + 15) & ~(size_t)15) + 4 * 32;
}

// Variants: 256 threads x 3 CTAs/SM (85 registers, radices up to 25) or
// 256 threads x 4 CTAs/SM (64 registers, radices up to 8).
// Once per device: the composite-radix twiddles in constant memory (every
// kernel that runs the row FFT needs them) and the shared-memory opt-ins.
static cudaError_t conv_device_setup()
{
    static std::atomic<unsigned long long> ready{0};  // per-device attribute setup (idempotent)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (ready & (1ull << dev)) return cudaSuccess;
    e = cudaFuncSetAttribute(wsb::k_conv<256, 25, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(wsb::k_conv<256, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(wsb::k_noise_spectrum<256, 25>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(wsb::k_noise_spectrum<256, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    float2 host[wsb::kCompositeTwiddles] = {};
    for (int R : {10, 14, 16, 20, 24, 25, 28, 32, 35, 40, 49}) {
        const int o = wsb::comp_off(R);
        for (int m = 0; m < R; ++m) {
            const double a = -6.283185307179586476925286766559 * (double)m / (double)R;
            host[o + m] = make_float2((float)cos(a), (float)sin(a));
        }
    }
    e = cudaMemcpyToSymbol(wsb::c_wr, host, sizeof(host));
    if (e != cudaSuccess) return e;
    ready |= 1ull << dev;
    return cudaSuccess;
}

extern "C" cudaError_t wsb_launch_conv(const wsb::EventDesc& ev, const uint32_t* pool, const uint32_t* band_off,
                                       const wsb::UnitRec* band_list, int flags, size_t smem_bytes, int variant,
                                       cudaStream_t stream)
{
    cudaError_t e = conv_device_setup();
    if (e != cudaSuccess) return e;
    if (ev.total_bands == 0) return cudaSuccess;
    if (variant == 8)
        wsb::k_conv<256, 8, 4><<<ev.total_bands, 256, smem_bytes, stream>>>(ev, pool, band_off, band_list, flags);
    else
        wsb::k_conv<256, 25, 3><<<ev.total_bands, 256, smem_bytes, stream>>>(ev, pool, band_off, band_list, flags);
    return cudaGetLastError();
}

extern "C" size_t wsb_noise_spectrum_smem(int M)
{
    return (((size_t)8 * M + 15) & ~(size_t)15) + sizeof(float2) * wsb::kTwiddleTable + (((size_t)2 * M + 15) & ~(size_t)15) +
           sizeof(double) * ((size_t)M + 1);
}

extern "C" cudaError_t wsb_launch_noise_spectrum(const wsb::PlaneDesc& P, const double* amp, uint64_t seed, int rng_mode,
                                                 const float* in, const wsb::Sink& out, int variant,
                                                 cudaStream_t stream)
{
    const size_t smem = wsb_noise_spectrum_smem(P.M);
    cudaError_t e = conv_device_setup();  // composite-radix twiddles (the DIT below uses them)
    if (e != cudaSuccess) return e;
    if (variant == 8)
        wsb::k_noise_spectrum<256, 8><<<P.W, 256, smem, stream>>>(P, amp, seed, rng_mode, in, out);
    else
        wsb::k_noise_spectrum<256, 25><<<P.W, 256, smem, stream>>>(P, amp, seed, rng_mode, in, out);
    return cudaGetLastError();
}
