// Electronics noise + digitization of a frame (the reference's add_noise
// white mode, spectral.cpp:177-196, and digitize, spectral.cpp:228-238), the
// first "next" stage after the convolution.
//
// Compiled with --fmad=false: the noisy sample m + sigma * n and the ADC code
// round(v * scale + offset) keep the reference's fp64 operation order.
//   rng substream: each wire's normals are the reference's own stream
//     StreamSource(substream(seed ^ kWhiteNoiseSalt, w)) in order (Box-Muller
//     pairs, cached spare); the stream is sequential, so one thread walks a row.
//   rng philox:    the shared counter-based stream keyed by (seed ^ salt, w):
//     tick pair p draws uniforms 2p and 2p+1 (one Philox4x32-10 call), so
//     every pair is independent: one thread per pair.
// The frame is updated in place (float32); the ADC codes (int32, the
// reference's Matrix<int32_t>, or uint16) are computed from the fp64 noisy
// value. The same readout runs fused in the convolution kernels' epilogues
// (ws_common.cuh readout_pair / readout4) for the Philox stream.
#include "ws_common.cuh"

#include <algorithm>

namespace wsb {

struct NoiseArgs {
    const float* in;  // the frame samples (fp32)
    Sink out;         // noisy frame (may alias `in`), fp64 frame, ADC codes
    int W, N;
    int noise;        // 0 off, 1 white
    int rng_mode;
    double sigma;
    uint64_t seed;
};

__global__ void k_noise_rows(const NoiseArgs a)
{
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= a.W) return;
    Rng src;
    src.init(WS_RNG_SUBSTREAM, a.seed ^ kWhiteNoiseSalt, (uint64_t)w);
    const size_t base = (size_t)w * a.N;
    for (int t = 0; t < a.N; ++t) {
        double v = (double)a.in[base + t];
        if (a.noise) v = __dadd_rn(v, __dmul_rn(a.sigma, src.normal()));
        sink_put(a.out, base + t, v);
    }
}

__global__ void k_noise_pairs(const NoiseArgs a)
{
    const int half = (a.N + 1) >> 1;
    const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (size_t)a.W * half) return;
    const int w = (int)(g / half), p = (int)(g - (size_t)w * half);
    const size_t base = (size_t)w * a.N + 2 * (size_t)p;
    double n0 = 0.0, n1 = 0.0;
    if (a.noise) {
        Rng src;
        src.init(a.rng_mode, a.seed ^ kWhiteNoiseSalt, (uint64_t)w);
        src.draw = 2u * (uint32_t)p;  // philox: the pair's two uniforms
        n0 = src.normal();
        n1 = src.normal();  // the cached spare
    }
    const bool has1 = 2 * p + 1 < a.N;
    const double v0 = (double)a.in[base], v1 = has1 ? (double)a.in[base + 1] : 0.0;
    sink_put(a.out, base, a.noise ? __dadd_rn(v0, __dmul_rn(a.sigma, n0)) : v0);
    if (has1) sink_put(a.out, base + 1, a.noise ? __dadd_rn(v1, __dmul_rn(a.sigma, n1)) : v1);
}

// Digitize only (no noise), a float4 of samples per thread: the frame's
// samples -> fp32 / fp64 frame and ADC codes (the reference's fp64 rounding,
// adc_code), 16-byte loads and 8-/16-byte stores. n4: the samples / 4 (the
// frame is contiguous: W x N padded samples).
__global__ void k_digitize4(const float4* __restrict__ in, const Sink k, size_t n4)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldcs(in + i);
        const double x[4] = {(double)v.x, (double)v.y, (double)v.z, (double)v.w};
        if (k.frame && k.frame != reinterpret_cast<const float*>(in)) reinterpret_cast<float4*>(k.frame)[i] = v;
        if (k.frame64) {
            reinterpret_cast<double2*>(k.frame64)[2 * i] = make_double2(x[0], x[1]);
            reinterpret_cast<double2*>(k.frame64)[2 * i + 1] = make_double2(x[2], x[3]);
        }
        if (k.adc) {
            int c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) c[j] = adc_code(x[j], k.scale, k.offset, k.max_code);
            if (k.adc_u16)
                reinterpret_cast<uint2*>(k.adc)[i] =
                    make_uint2((uint32_t)c[0] | ((uint32_t)c[1] << 16), (uint32_t)c[2] | ((uint32_t)c[3] << 16));
            else
                reinterpret_cast<int4*>(k.adc)[i] = make_int4(c[0], c[1], c[2], c[3]);
        }
    }
}

// integer charge grid (fluctuation on, u64 counts) -> the caller's charge
// output: float32 (type 0), uint32 (1; a count past 2^32 - 1 flags
// kErrCellOvf) or int64 (2, the reference's ChargeGrid)
__global__ void k_counts_out(const unsigned long long* __restrict__ g, void* out, int type, size_t n, unsigned* err,
                             const unsigned long long* __restrict__ qsum)
{
    bool ovf = false;
    const bool wide = !qsum || *qsum >= (1ull << 32);  // the grid's cell width (cnt_wide)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const unsigned long long v = wide ? g[i] : (unsigned long long)reinterpret_cast<const unsigned*>(g)[i];
        if (type == 0) {
            static_cast<float*>(out)[i] = (float)v;
        } else if (type == 1) {
            ovf |= v > 0xffffffffull;
            static_cast<uint32_t*>(out)[i] = (uint32_t)v;
        } else {
            static_cast<long long*>(out)[i] = (long long)v;
        }
    }
    if (__any_sync(0xffffffffu, ovf) && (threadIdx.x & 31) == 0) atomicOr(err, kErrCellOvf);
}

}  // namespace wsb

// add_noise (white) + digitize: `in` -> sink (frame in place when noisy, fp64
// frame, ADC codes); rng substream walks each wire's sequential stream
extern "C" cudaError_t wsb_launch_noise(const float* in, const wsb::Sink& out, int W, int N, int noise, int rng_mode,
                                        double sigma, uint64_t seed, cudaStream_t s)
{
    const wsb::NoiseArgs a{in, out, W, N, noise, rng_mode, sigma, seed};
    const size_t n = (size_t)W * N;
    const auto aligned = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (!noise && n % 4 == 0 && aligned(in) && aligned(out.frame) && aligned(out.frame64) && aligned(out.adc)) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const size_t n4 = n / 4;
        wsb::k_digitize4<<<(unsigned)std::min<size_t>((n4 + 255) / 256, (size_t)sms * 16), 256, 0, s>>>(
            reinterpret_cast<const float4*>(in), out, n4);
    } else if (noise && rng_mode == WS_RNG_SUBSTREAM) {
        wsb::k_noise_rows<<<(W + 63) / 64, 64, 0, s>>>(a);
    } else {
        const size_t pairs = (size_t)W * ((N + 1) / 2);
        wsb::k_noise_pairs<<<(unsigned)((pairs + 255) / 256), 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

extern "C" cudaError_t wsb_launch_counts_out(const unsigned long long* g, void* out, int type, size_t n, unsigned* err,
                                             const unsigned long long* qsum, cudaStream_t s)
{
    if (!n) return cudaSuccess;
    wsb::k_counts_out<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(g, out, type, n, err, qsum);
    return cudaGetLastError();
}
