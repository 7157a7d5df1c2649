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
// reference's Matrix<int32_t>) are computed from the fp64 noisy value.
#include "ws_common.cuh"

namespace wsb {

constexpr uint64_t kWhiteNoiseSalt = 0x77686974656e6f69ULL;  // spectral.cpp:21

struct NoiseArgs {
    float* frame;
    int32_t* adc;     // nullable
    int W, N;
    int noise;        // 0 off, 1 white
    int rng_mode;
    double sigma;
    uint64_t seed;
    double scale, offset, max_code;
};

__device__ __forceinline__ void emit(const NoiseArgs& a, size_t i, double v)
{
    if (a.noise) a.frame[i] = (float)v;
    if (a.adc) {
        const double c = round(__dadd_rn(__dmul_rn(v, a.scale), a.offset));
        a.adc[i] = (int32_t)(c < 0.0 ? 0.0 : (c > a.max_code ? a.max_code : c));
    }
}

__global__ void k_noise_rows(const NoiseArgs a)
{
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= a.W) return;
    Rng src;
    src.init(WS_RNG_SUBSTREAM, a.seed ^ kWhiteNoiseSalt, (uint64_t)w);
    const size_t base = (size_t)w * a.N;
    for (int t = 0; t < a.N; ++t) {
        double v = (double)a.frame[base + t];
        if (a.noise) v = __dadd_rn(v, __dmul_rn(a.sigma, src.normal()));
        emit(a, base + t, v);
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
    emit(a, base, a.noise ? __dadd_rn((double)a.frame[base], __dmul_rn(a.sigma, n0)) : (double)a.frame[base]);
    if (2 * p + 1 < a.N)
        emit(a, base + 1,
             a.noise ? __dadd_rn((double)a.frame[base + 1], __dmul_rn(a.sigma, n1)) : (double)a.frame[base + 1]);
}

}  // namespace wsb

extern "C" cudaError_t wsb_launch_noise(float* frame, int32_t* adc, int W, int N, int noise, int rng_mode, double sigma,
                                        uint64_t seed, double scale, double offset, double max_code, cudaStream_t s)
{
    const wsb::NoiseArgs a{frame, adc, W, N, noise, rng_mode, sigma, seed, scale, offset, max_code};
    if (noise && rng_mode == WS_RNG_SUBSTREAM) {
        wsb::k_noise_rows<<<(W + 63) / 64, 64, 0, s>>>(a);
    } else {
        const size_t pairs = (size_t)W * ((N + 1) / 2);
        wsb::k_noise_pairs<<<(unsigned)((pairs + 255) / 256), 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}
