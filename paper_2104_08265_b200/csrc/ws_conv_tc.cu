// Convolution of a charge grid on the 5th-generation tensor cores (k_conv_tc):
// the reference's convolve (spectral.cpp:141-175) for an existing grid S
// (the fluctuation walk's integer counts, or a float grid given to
// ws_convolve_device), as a direct circular convolution along ticks
//   D[w, t] = sum_l k[l] S[w, (t - l) mod N]
// followed by the cross-wire stencil M[w] = sum_dw ww[dw] D[w - dw mod W]
// (kernel_td's wire rows, spectral.cpp:124-135). It replaces the row FFT of
// k_conv in mode 1; the result is the same circular convolution, with no
// constraint on the tick count.
//
// One CTA owns 32 - 2h wire rows x 128 nb ticks. Along ticks the product is
// a Toeplitz GEMM per 128-tick sub-block:
//   D[128 x 32] = A[128 x K] . B[K x 32],  A[m][k] = k(m + c - k),  B[k][n] = S[row n][t0 - c + k]
// with K = ceil8(128 + c - lo_lag) input ticks (c = ceil8(hi_lag)). Every
// 8-wide K step of A is the same matrix shifted by 8 rows, so A is one
// (128 + K - 8) x 8 matrix E in shared memory and step j starts 8 (J-1-j)
// rows into it: the kernel is staged once per CTA (12 KB per TF32 part at 129
// lags) instead of a 128 x K Toeplitz block. B is the tile's input window
// (32 rows x 128 nb + K - 128 ticks) in the canonical K-major layout; the
// sub-blocks' windows overlap and start 128 ticks apart. tcgen05.mma
// kind::tf32 (M = 128, N = 32, K = 8), issued by one thread, accumulates in
// TMEM (32 columns per sub-block).
//
// Exactness: the kernel taps are split into TF32 hi + lo parts (2 passes;
// ~2^-22 relative per tap). Integer counts enter exactly: a tile whose
// counts fit 11 bits is one round; larger counts run one round per 11-bit
// chunk (chunk << 11 rho is exact in TF32), all into the same accumulator. A
// float grid runs its TF32 hi part (2 passes) and its lo part (1 pass).
//
// Epilogue: warp w reads its TMEM lane quadrant (32 ticks) x 32 columns
// (tcgen05.ld 32x32b.x32), applies the stencil across columns in registers
// and stores each output row with coalesced stores (or the fused readout:
// noise + digitize, fp64 frame).
#include "ws_common.cuh"

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <type_traits>

namespace wsb {

constexpr int kTcThreads = 256;
constexpr int kTcN = 32;   // MMA N: wire rows of a tile including the stencil halo
constexpr int kTcM = 128;  // MMA M: output ticks of a sub-block
constexpr int kTcMaxH = 2;  // stencil half widths with an instantiation (wire_weights of 1, 3, 5 taps)

struct TcGeom {
    int c, K, J, RE, kwin;
};

__host__ __device__ inline TcGeom tc_geom(int lo_lag, int n_lags, int nb)
{
    TcGeom g;
    const int hi = lo_lag + n_lags - 1;
    g.c = hi >= 0 ? (hi + 7) / 8 * 8 : -((-hi) / 8 * 8);  // ceil8(hi)
    g.K = (kTcM + g.c - lo_lag + 7) / 8 * 8;
    g.J = g.K / 8;
    g.RE = kTcM + 8 * (g.J - 1);
    g.kwin = kTcM * nb + g.K - kTcM;
    return g;
}

__host__ __device__ inline size_t tc_smem(const TcGeom& g) { return (size_t)2 * g.RE * 32 + (size_t)kTcN * g.kwin * 4; }

__device__ __forceinline__ uint32_t tc_tf32(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// KSRC 0: the u64 count grid (P.charge_cnt); 1: a float grid (P.charge_in)
template <int H, int KSRC>
__global__ void __launch_bounds__(kTcThreads, 2) k_conv_tc(const EventDesc ev, int nb)
{
    constexpr int R = kTcN - 2 * H;  // output rows per tile
    const PlaneDesc& P = ev.p[blockIdx.y];
    if (P.direct || !P.frame && !P.frame64 && !P.adc) return;
    const int W = P.W, Nt = P.N;
    const int tt = (Nt + kTcM * nb - 1) / (kTcM * nb);
    const int tiles = ((W + R - 1) / R) * tt;
    if ((int)blockIdx.x >= tiles) return;
    const int ri = blockIdx.x / tt, ti = blockIdx.x - ri * tt;  // tick tiles fastest: neighbours share halos in L2
    const int r0 = ri * R, T0 = ti * kTcM * nb;
    const int nr = min(R, W - r0);
    const int lo = P.lo_lag, hi = P.lo_lag + P.n_lags - 1;
    const TcGeom g = tc_geom(lo, P.n_lags, nb);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    extern __shared__ __align__(128) unsigned char tc_smem_buf[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tc_smem_buf);
    const uint32_t e_hi = sbase, e_lo = e_hi + (uint32_t)g.RE * 32u, bsm = e_lo + (uint32_t)g.RE * 32u;
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ unsigned long long s_max;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    const uint32_t cols = nb == 1 ? 32u : nb == 2 ? 64u : 128u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                     "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_max = 0ull;
    }

    // A: E[r][kk] = k(r + c - 8 (J - 1) - kk), TF32 hi and lo parts, K-major
    // canonical layout (core matrices of 8 rows x 4 taps; K chunk kq at kq RE/8 x 128 B)
    const int ebase = g.c - 8 * (g.J - 1);
    for (int i = tid; i < 2 * g.RE; i += kTcThreads) {
        const int r = i >> 1, kq = i & 1;
        uint32_t vh[4], vl[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int l = r + ebase - (4 * kq + q);
            const float v = (l >= lo && l <= hi) ? __ldg(&P.kern[l - lo]) : 0.0f;
            vh[q] = tc_tf32(v);
            vl[q] = tc_tf32(v - __uint_as_float(vh[q]));
        }
        const uint32_t o = (uint32_t)(((kq * (g.RE >> 3) + (r >> 3)) << 7) + ((r & 7) << 4));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(e_hi + o), "r"(vh[0]), "r"(vh[1]), "r"(vh[2]),
                     "r"(vh[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(e_lo + o), "r"(vl[0]), "r"(vl[1]), "r"(vl[2]),
                     "r"(vl[3]));
    }

    // B: the input window, rows n = lane (source row r0 - H + n mod W), four
    // ticks per item; round rho of a count grid holds the 11-bit chunk rho of
    // every count (exact in TF32), round 1 of a float grid its TF32 residue
    int s0 = (T0 - g.c) % Nt;
    if (s0 < 0) s0 += Nt;
    const int n = lane;
    const bool row_live = n < nr + 2 * H;
    int sw = (r0 - H + n) % W;
    if (sw < 0) sw += W;
    const int nk4 = g.kwin >> 2;
    const bool vec = (Nt & 3) == 0;
    auto load_round = [&](int rho) {
        unsigned long long mx = 0ull;
        // items k4 = warp + 8 i, four ticks each; kB items' loads in flight per batch
        constexpr int kB = 4;
        using raw_t = typename std::conditional<KSRC == 0, ulonglong2, float4>::type;
        for (int k0 = warp; k0 < nk4; k0 += kB * (kTcThreads / 32)) {
            raw_t ra[kB], rb[kB];
            int sv[kB];
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int k4 = k0 + b * (kTcThreads / 32);
                int s = s0 + 4 * k4;
                s -= s >= Nt ? Nt : 0;
                if (s >= Nt) s %= Nt;  // windows longer than the row
                sv[b] = (row_live && k4 < nk4) ? ((vec && s + 3 < Nt) ? s : -1 - s) : INT_MIN;
                if (sv[b] >= 0) {
                    if constexpr (KSRC == 0) {
                        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(P.charge_cnt + (size_t)sw * Nt + s);
                        ra[b] = __ldg(src);
                        rb[b] = __ldg(src + 1);
                    } else {
                        ra[b] = __ldg(reinterpret_cast<const float4*>(P.charge_in + (size_t)sw * Nt + s));
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < kB; ++b) {
                const int k4 = k0 + b * (kTcThreads / 32);
                if (k4 >= nk4) break;
                uint32_t v[4] = {0u, 0u, 0u, 0u};
                if (sv[b] != INT_MIN) {
                    if constexpr (KSRC == 0) {
                        unsigned long long c4[4];
                        if (sv[b] >= 0) {
                            c4[0] = ra[b].x; c4[1] = ra[b].y; c4[2] = rb[b].x; c4[3] = rb[b].y;
                        } else {  // unaligned / wrapping: scalar loads
                            const int s = -1 - sv[b];
                            const unsigned long long* src = P.charge_cnt + (size_t)sw * Nt;
#pragma unroll
                            for (int q = 0; q < 4; ++q) c4[q] = __ldg(src + (s + q) % Nt);
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            mx = c4[q] > mx ? c4[q] : mx;
                            const uint32_t ch = (uint32_t)((c4[q] >> (11 * rho)) & 2047ull);
                            v[q] = __float_as_uint((float)ch) + ((uint32_t)(11 * rho) << 23) * (ch != 0u);  // ch 2^(11 rho)
                        }
                    } else {
                        float x4[4];
                        if (sv[b] >= 0) {
                            x4[0] = ra[b].x; x4[1] = ra[b].y; x4[2] = ra[b].z; x4[3] = ra[b].w;
                        } else {
                            const int s = -1 - sv[b];
                            const float* src = P.charge_in + (size_t)sw * Nt;
#pragma unroll
                            for (int q = 0; q < 4; ++q) x4[q] = __ldg(src + (s + q) % Nt);
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t h4 = tc_tf32(x4[q]);
                            v[q] = rho == 0 ? h4 : tc_tf32(x4[q] - __uint_as_float(h4));
                        }
                    }
                }
                const uint32_t o = bsm + (uint32_t)(((k4 * (kTcN >> 3) + (n >> 3)) << 7) + ((n & 7) << 4));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(o), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                             "r"(v[3]));
            }
        }
        if constexpr (KSRC == 0)
            if (rho == 0) {
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
                    mx = t > mx ? t : mx;
                }
                if (lane == 0) atomicMax(&s_max, mx);
            }
    };
    load_round(0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    int rounds = 2;  // float grid: hi part, then the TF32 residue
    if constexpr (KSRC == 0) {
        const unsigned long long m = s_max;
        rounds = 1;
        while (rounds < 6 && (m >> (11 * rounds)) != 0ull) ++rounds;
    }
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcN >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
    const uint32_t lbo_a = (uint32_t)(g.RE >> 3) * 128u, lbo_b = (kTcN >> 3) * 128u;
    const int nbv = min(nb, (Nt - T0 + kTcM - 1) / kTcM);  // sub-blocks inside the row
#pragma unroll 1
    for (int rho = 0; rho < rounds; ++rho) {
        if (rho > 0) {
            load_round(rho);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (tid == 0) {
            // descriptors advance by constant byte offsets (>> 4 in the start field)
            const int parts = (KSRC == 1 && rho == 1) ? 1 : 2;  // the residue times the hi taps only
            const uint64_t da0 = tc_desc(e_hi + (uint32_t)(g.J - 1) * 128u, lbo_a, 128);
            const uint64_t dl = (uint64_t)((e_lo - e_hi) >> 4);
            for (int jb = 0; jb < nbv; ++jb) {
                uint64_t da = da0, db = tc_desc(bsm + (uint32_t)(32 * jb) * lbo_b, lbo_b, 128);
                const uint32_t d = tmem + (uint32_t)(kTcN * jb);
                uint32_t acc = rho ? 1u : 0u;
#pragma unroll 4
                for (int j = 0; j < g.J; ++j) {
                    tc_mma(d, da, db, idesc, acc);
                    if (parts == 2) tc_mma(d, da + dl, db, idesc, 1u);
                    acc = 1u;
                    da -= 128u >> 4;          // E rows 8 earlier
                    db += (2u * lbo_b) >> 4;  // the window 8 ticks later
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                         : "memory");
        }
        {
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(bar), "r"((uint32_t)(rho & 1))
                    : "memory");
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }

    // epilogue: warp w owns TMEM lanes 32 (w & 3) .. + 31 (ticks) of the
    // sub-blocks jb = w >> 2, w >> 2 + 2, ...
    float ww[2 * H + 1];
#pragma unroll
    for (int e = 0; e <= 2 * H; ++e) ww[e] = (float)P.ww[e];
    const int q4 = warp & 3;
    for (int jb = warp >> 2; jb < nbv; jb += kTcThreads / 128) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(kTcN * jb)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int t = T0 + kTcM * jb + 32 * q4 + lane;
        float out[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float s = 0.0f;
#pragma unroll
            for (int e = 0; e <= 2 * H; ++e) s = __fmaf_rn(ww[e], __uint_as_float(v[r + 2 * H - e]), s);
            out[r] = s;
        }
        if (!ev.ro) {
            if (t < Nt) {
                float* dst = P.frame + (size_t)r0 * Nt + t;
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (r < nr) __stcs(dst + (size_t)r * Nt, out[r]);
            }
        } else {
            // fused readout on tick pairs (t even on even lanes)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float nxt = __shfl_down_sync(0xffffffffu, out[r], 1);
                if (r < nr && !(lane & 1) && t < Nt) readout_pair(ev, P, r0 + r, t, out[r], nxt, t + 1 < Nt);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}

}  // namespace wsb

// Sub-blocks per tile for a plane on the tensor-core path (the largest that
// fits two CTAs per SM, else one), or 0 when it is not eligible (kernel taps
// absent, stencil wider than 5 taps, window too large).
extern "C" int wsb_conv_tc_nb(const wsb::PlaneDesc& P)
{
    static const int off = [] {
        const char* v = getenv("WS_CONV_TC");  // 0: the row FFT for every grid convolution (A/B)
        return v && atoi(v) == 0;
    }();
    if (off || !P.kern || P.h > wsb::kTcMaxH || P.n_lags < 1) return 0;
    for (int nb : {4, 2, 1}) {
        const size_t sm = wsb::tc_smem(wsb::tc_geom(P.lo_lag, P.n_lags, nb));
        if (sm + 1024 <= 112 * 1024 || (nb == 1 && sm + 1024 <= 226 * 1024)) return nb;
    }
    for (int nb : {4, 2, 1})
        if (wsb::tc_smem(wsb::tc_geom(P.lo_lag, P.n_lags, nb)) + 1024 <= 226 * 1024) return nb;
    return 0;
}

// Mode-1 convolution of every non-direct plane of the event on the tensor
// cores; the caller checked wsb_conv_tc_nb > 0 for each (nb: their minimum).
extern "C" cudaError_t wsb_launch_conv_tc(const wsb::EventDesc& ev, int nb, cudaStream_t s)
{
    static std::atomic<unsigned long long> ready{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(ready & (1ull << dev))) {
        for (auto f : {wsb::k_conv_tc<0, 0>, wsb::k_conv_tc<1, 0>, wsb::k_conv_tc<2, 0>, wsb::k_conv_tc<0, 1>,
                       wsb::k_conv_tc<1, 1>, wsb::k_conv_tc<2, 1>}) {
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
            if (e != cudaSuccess) return e;
        }
        ready |= 1ull << dev;
    }
    size_t smem = 0;
    int max_tiles = 0, h = -1, src = -1;
    for (int i = 0; i < ev.n_planes; ++i) {
        const wsb::PlaneDesc& P = ev.p[i];
        if (P.direct) continue;
        if (h >= 0 && (P.h != h || (P.charge_cnt ? 0 : 1) != src)) return cudaErrorNotSupported;  // one instantiation per launch
        h = P.h;
        src = P.charge_cnt ? 0 : 1;
        smem = std::max(smem, wsb::tc_smem(wsb::tc_geom(P.lo_lag, P.n_lags, nb)));
        const int R = wsb::kTcN - 2 * P.h;
        max_tiles = std::max(max_tiles, ((P.W + R - 1) / R) * ((P.N + wsb::kTcM * nb - 1) / (wsb::kTcM * nb)));
    }
    if (h < 0 || max_tiles == 0) return cudaSuccess;
    const dim3 grid((unsigned)max_tiles, (unsigned)ev.n_planes);
    using K = void (*)(const wsb::EventDesc, int);
    const K fns[2][3] = {{wsb::k_conv_tc<0, 0>, wsb::k_conv_tc<1, 0>, wsb::k_conv_tc<2, 0>},
                         {wsb::k_conv_tc<0, 1>, wsb::k_conv_tc<1, 1>, wsb::k_conv_tc<2, 1>}};
    fns[src][h]<<<grid, wsb::kTcThreads, smem, s>>>(ev, nb);
    return cudaGetLastError();
}
