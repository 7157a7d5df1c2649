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

#include <cuda.h>
#include <cudaTypedefs.h>

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
    const bool wide = KSRC == 0 && cnt_wide(P);  // u64 or u32 count cells
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
                        if (wide) {
                            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(P.charge_cnt + (size_t)sw * Nt + s);
                            ra[b] = __ldg(src);
                            rb[b] = __ldg(src + 1);
                        } else {  // u32 cells: four in one 16-byte load
                            const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(
                                reinterpret_cast<const unsigned*>(P.charge_cnt) + (size_t)sw * Nt + s));
                            ra[b] = make_ulonglong2(w4.x, w4.y);
                            rb[b] = make_ulonglong2(w4.z, w4.w);
                        }
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
#pragma unroll
                            for (int q = 0; q < 4; ++q) c4[q] = count_at(P, (size_t)sw * Nt + (s + q) % Nt, wide);
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


// ---- k_conv_tc2: the same convolution as a persistent warp-specialised pipeline
//
// k_conv_tc re-reads its 4 KB Toeplitz operand from shared memory for every
// 128 x 32 x 8 MMA and loads, converts, multiplies and stores one tile after
// another, so the tensor pipe idles while a tile loads and shared-memory
// bandwidth caps it when it runs (r2c: 0.79 ms per C3 event, 24% of warps
// active). Here one CTA per SM walks a list of work items (plane, strip of
// 128 wire rows, chunk of eight 128-tick sub-blocks), N = 128 wire rows per
// MMA (tools/ubench_umma.cu: 64 cycles per 128x128x8 TF32 MMA, 46 at N = 32),
// and four roles overlap, connected by mbarriers:
//   warp 0 (loader): per "slab" (16 ticks x 128 rows = two MMA K steps) two
//     TMA 2D boxes of the count grid (u64 or u32 cells) or float grid into a
//     4-deep raw ring; planes whose layout rules TMA out (a wire stencil wraps
//     rows, N % 8 != 0, an unaligned base) take cp.async per wire row (warps
//     0-3) instead;
//   warps 4-11 (converters, two groups taking alternate slabs, one wire row
//     per thread): raw values -> TF32 hi (plus a lo part where a value does
//     not fit 11 bits) in a 4-slot MMA ring. Loading and converting are
//     separate warps because the generic -> async proxy fence the converters
//     need compiles to MEMBAR.ALL.CTA, which waits for every load the thread
//     has in flight;
//   warp 16 (one elected lane): per slab, the MMAs of every sub-block whose K
//     range contains it (<= 3 for J <= 48) into a ring of four 128-column TMEM
//     accumulators; tcgen05.commit releases the slab and, after a sub-block's
//     last K step, hands its accumulator to the epilogue;
//   warps 12-15 (epilogue, one TMEM lane quadrant each): tcgen05.ld, the
//     cross-wire stencil in registers, predicated coalesced stores with a
//     running offset (or the fused readout; the end-to-end calls digitize
//     with the full-GPU pair kernel instead, ws_api.cu).
// Exactness as in k_conv_tc: taps split TF32 hi + lo; counts below 2^11 are
// one TF32 value, below 2^22 exactly hi + lo (the 11-bit halves), above that
// hi + lo within 2^-22 relative (the frame tolerance is 1e-5); float grids hi
// + lo. Products hi x hi, lo(tap) x hi, hi(tap) x lo accumulate in fp32.
constexpr int kT2N = 128;        // MMA N: wire rows of a strip including the stencil halo
constexpr int kT2SK = 2;         // K steps (8 ticks each) per slab
constexpr int kT2Slots = 4;      // slab ring depth (a power of two)
constexpr int kT2Acc = 4;        // TMEM accumulators of 128 columns
constexpr int kT2MaxJ = 48;      // K steps per sub-block: <= 3 accumulators live per slab
constexpr int kT2Groups = 2;     // converter groups of 4 warps (one wire row per thread) taking alternate slabs
constexpr int kT2EpiWarp = 4 + 4 * kT2Groups;  // first of the 4 epilogue warps (warp & 3 = TMEM lane quadrant)
constexpr int kT2MmaWarp = kT2EpiWarp + 4;
constexpr int kT2Threads = 32 * (kT2MmaWarp + 1);
constexpr int kT2Raw = 4;        // raw ring (TMA / cp.async landing slots) depth
constexpr uint32_t kT2RawHalf = kT2N * 64;  // one K step of a raw slot: 128 wire rows x 8 ticks (u64 64 B/row, f32 32 B)
constexpr uint32_t kT2RawSlot = kT2SK * kT2RawHalf;
constexpr uint32_t kT2Step = kT2N * 8 * 4;  // one K step of one TF32 part: 4 KB
constexpr uint32_t kT2Part = kT2SK * kT2Step;  // one TF32 part of a slab
constexpr uint32_t kT2SlotBytes = 2 * kT2Part;  // [hi | lo]

// K steps per sub-block rounded up to whole slabs (the extra steps meet zero
// taps: E is zero outside the kernel's lags) and E's rows.
struct T2Geom {
    int c, J, RE;
};
__host__ __device__ inline T2Geom t2_geom(int lo_lag, int n_lags)
{
    const TcGeom g = tc_geom(lo_lag, n_lags, 1);
    T2Geom r;
    r.c = g.c;
    r.J = (g.J + kT2SK - 1) / kT2SK * kT2SK;
    r.RE = kTcM + 8 * (r.J - 1);
    return r;
}

struct alignas(64) T2Plan {
    int np;                       // planes on this path
    int chunk;                    // sub-blocks per work item
    int pl[kMaxPlanes];           // their EventDesc indices
    int item0[kMaxPlanes + 1];    // first work item of each (item0[np] = total)
    int chunks[kMaxPlanes];       // work items per strip
    uint32_t eoff[kMaxPlanes];    // shared byte offset of the plane's E (hi; lo at + RE * 32)
    int tma;                      // 1: slab halves are TMA box loads (8 ticks x 128 rows) through tm[]
    CUtensorMap tm[kMaxPlanes];   // the planes' input grids as 2D tensors (ticks, wire rows): u64 counts / floats
    CUtensorMap tm32[kMaxPlanes]; // the count grids viewed as u32 cells (cnt_wide false)
};

#ifdef WS_T2_PROF
// per-role wait cycles (tools: bring-up profiling only)
__device__ unsigned long long g_t2prof[16];
#define T2_PROF_DECL unsigned long long t2p_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; const long long t2p_t0 = clock64();
#define T2_WAIT(b, par, k) do { const long long _c = clock64(); t2_wait(b, par); t2p_acc[k] += clock64() - _c; } while (0)
#define T2_PROF_FLUSH(base) do { if ((threadIdx.x & 31) == 0) { for (int _i = 0; _i < 3; ++_i) atomicAdd(&g_t2prof[(base) + _i], t2p_acc[_i]); atomicAdd(&g_t2prof[(base) + 3], (unsigned long long)(clock64() - t2p_t0)); } } while (0)
#else
#define T2_PROF_DECL
#define T2_WAIT(b, par, k) t2_wait(b, par)
#define T2_PROF_FLUSH(base)
#endif
__device__ __forceinline__ void t2_wait(uint32_t bar, uint32_t parity)
{
    uint32_t done = 0, spins = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (++spins == (1u << 28)) __trap();  // a pipeline bug fails the launch instead of hanging the GPU
    }
}
__device__ __forceinline__ bool elect_one()
{
    uint32_t p;
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; selp.u32 %0, 1, 0, e; }" : "=r"(p));
    return p != 0u;
}
__device__ __forceinline__ void t2_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void t2_commit(uint32_t bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Geometry of one work item (every role derives it the same way).
struct T2Item {
    int k;        // plan plane index
    int r0, nr;   // first output row, output rows
    int T0;       // first output tick
    int nsub;     // sub-blocks
    int nslab;    // input slabs of 16 ticks = 8 (nsub - 1) + J / 2
    int S0;       // input tick of slab 0 (T0 - c), not reduced
    int J, RE;    // K steps per sub-block (even), E rows
};

template <int H>
__device__ __forceinline__ T2Item t2_item(const EventDesc& ev, const T2Plan& plan, int it)
{
    T2Item I;
    int k = 0;
    while (k + 1 < plan.np && it >= plan.item0[k + 1]) ++k;
    const PlaneDesc& P = ev.p[plan.pl[k]];
    const int local = it - plan.item0[k];
    const int strip = local / plan.chunks[k], ch = local - strip * plan.chunks[k];
    constexpr int R = kT2N - 2 * H;
    I.k = k;
    I.r0 = strip * R;
    I.nr = min(R, P.W - I.r0);
    const int nsub_row = (P.N + kTcM - 1) / kTcM;
    const int sb0 = ch * plan.chunk;
    I.nsub = min(plan.chunk, nsub_row - sb0);
    I.T0 = sb0 * kTcM;
    const T2Geom g = t2_geom(P.lo_lag, P.n_lags);
    I.J = g.J;
    I.RE = g.RE;
    I.nslab = (kTcM / (8 * kT2SK)) * (I.nsub - 1) + g.J / kT2SK;
    I.S0 = I.T0 - g.c;
    return I;
}

// KSRC 0: u64 counts (P.charge_cnt); 1: float grid (P.charge_in)
template <int H, int KSRC>
__global__ void __launch_bounds__(kT2Threads, 1) k_conv_tc2(const EventDesc ev, const __grid_constant__ T2Plan plan)
{
    constexpr int kSlabsPerSub = kTcM / (8 * kT2SK);  // 8: a sub-block starts every 8 slabs
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_items = plan.item0[plan.np];

    extern __shared__ __align__(1024) unsigned char t2_buf[];
    __shared__ __align__(8) unsigned long long s_full[kT2Slots], s_empty[kT2Slots], s_accf[kT2Acc], s_acce[kT2Acc];
    __shared__ __align__(8) unsigned long long s_rfull[kT2Raw], s_rempty[kT2Raw];
    __shared__ uint32_t s_tag[kT2Slots];
    __shared__ uint32_t s_tmem;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(t2_buf);
    const uint32_t ring = sbase;  // kT2Slots x [hi part | lo part], a part = kT2SK K steps of 4 KB
    const uint32_t raw = sbase + kT2Slots * kT2SlotBytes;  // kT2Raw x kT2SK x 128 rows x (8 ticks of u64 / u32 / f32)
    auto bar = [](unsigned long long* b) { return (uint32_t)__cvta_generic_to_shared(b); };
    // shared addresses of the barrier arrays, once (cvta reads the CTA id register)
    const uint32_t a_full = bar(s_full), a_empty = bar(s_empty), a_accf = bar(s_accf), a_acce = bar(s_acce);
    const uint32_t a_rfull = bar(s_rfull), a_rempty = bar(s_rempty);

    if (warp == kT2MmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                     "r"(kT2Acc * 128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < kT2Slots; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(bar(&s_full[i])));  // one converter group
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar(&s_empty[i])));
            s_tag[i] = 0u;
        }
        for (int i = 0; i < kT2Raw; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar(&s_rfull[i])),
                         "r"(plan.tma ? 1 : kT2N));  // the TMA issuer, or every loader thread
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(bar(&s_rempty[i])));  // one converter group
        }
        for (int i = 0; i < kT2Acc; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar(&s_accf[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(bar(&s_acce[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // lo parts of the ring start zeroed (converters keep them zero unless used)
    for (uint32_t i = tid; i < kT2Slots * (kT2Part / 16); i += kT2Threads) {
        const uint32_t slot = i / (kT2Part / 16), w = i - slot * (kT2Part / 16);
        asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(ring + slot * kT2SlotBytes + kT2Part + 16u * w),
                     "r"(0u));
    }
    // E of every plane: E[r][kk] = k(r + c - 8 (J - 1) - kk), TF32 hi and lo
    for (int k = 0; k < plan.np; ++k) {
        const PlaneDesc& P = ev.p[plan.pl[k]];
        const T2Geom g = t2_geom(P.lo_lag, P.n_lags);
        const int lo = P.lo_lag, hi = P.lo_lag + P.n_lags - 1;
        const int ebase = g.c - 8 * (g.J - 1);
        const uint32_t e_hi = sbase + plan.eoff[k], e_lo = e_hi + (uint32_t)g.RE * 32u;
        for (int i = tid; i < 2 * g.RE; i += kT2Threads) {
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
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(e_hi + o), "r"(vh[0]), "r"(vh[1]),
                         "r"(vh[2]), "r"(vh[3]));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(e_lo + o), "r"(vl[0]), "r"(vl[1]),
                         "r"(vl[2]), "r"(vl[3]));
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    T2_PROF_DECL

    if (warp < 4) {
        // ---- loaders: the kT2SK K steps (8 ticks x 128 wire rows each) of
        // every slab into the raw ring, many slabs in flight, completion on
        // mbarriers: TMA boxes from one thread, else cp.async per wire row
        const int n = tid;
        uint32_t gs = 0;
        if (plan.tma) {
            if (tid == 0)
                for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
                    const T2Item I = t2_item<H>(ev, plan, it);
                    const int Nt = ev.p[plan.pl[I.k]].N;
                    const bool wide = KSRC == 0 && cnt_wide(ev.p[plan.pl[I.k]]);
                    const uint64_t tmap = reinterpret_cast<uint64_t>(KSRC == 0 && !wide ? &plan.tm32[I.k] : &plan.tm[I.k]);
                    int st = I.S0 % Nt;
                    st = st < 0 ? st + Nt : st;
                    for (int s = 0; s < I.nslab; ++s, ++gs) {
                        const uint32_t rs = gs % kT2Raw, use = gs / kT2Raw;
                        if (use > 0) T2_WAIT((a_rempty + 8u * (rs)), (use - 1) & 1u, 0);
                        const uint32_t fb = (a_rfull + 8u * (rs));
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                                     "r"(kT2SK * kT2N * 8u * (wide ? 8u : 4u))
                                     : "memory");
#pragma unroll
                        for (int h = 0; h < kT2SK; ++h) {  // (N % 8 == 0: a K step never wraps; steps may)
                            asm volatile(
                                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                                    raw + rs * kT2RawSlot + h * kT2RawHalf),
                                "l"(tmap), "r"(st), "r"(I.r0), "r"(fb)
                                : "memory");
                            st += 8;
                            if (st >= Nt) st -= Nt;
                        }
                    }
                }
        } else {
            for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
                const T2Item I = t2_item<H>(ev, plan, it);
                const PlaneDesc& P = ev.p[plan.pl[I.k]];
                const int Nt = P.N, W = P.W;
                int sw = (I.r0 - H + n) % W;
                sw = sw < 0 ? sw + W : sw;
                const bool live = n < I.nr + 2 * H;
                const bool wide = KSRC == 0 && cnt_wide(P);
                const int E = wide ? 8 : 4;  // bytes per cell
                const int rawq = E / 2;      // 16-byte words per 8-tick row
                const uint32_t rowb = 16u * (uint32_t)rawq;
                const size_t off = (size_t)sw * Nt;
                const unsigned char* row = KSRC == 0 ? reinterpret_cast<const unsigned char*>(P.charge_cnt) + off * E
                                                     : reinterpret_cast<const unsigned char*>(P.charge_in + off);
                int st = I.S0 % Nt;
                st = st < 0 ? st + Nt : st;
                for (int s = 0; s < I.nslab; ++s, ++gs) {
                    const uint32_t rs = gs % kT2Raw, use = gs / kT2Raw;
                    if (use > 0) T2_WAIT((a_rempty + 8u * (rs)), (use - 1) & 1u, 0);
                    bool async = false;
#pragma unroll
                    for (int h = 0; h < kT2SK; ++h) {
                        const uint32_t dst = raw + rs * kT2RawSlot + h * kT2RawHalf + (uint32_t)n * rowb;
                        if (live && st + 8 <= Nt && ((st | Nt) & (16 / E - 1)) == 0) {
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                if (q < rawq)
                                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * q),
                                                 "l"(row + (size_t)st * E + 16 * q)
                                                 : "memory");
                            async = true;
                        } else {
                            // wrapping / unaligned / dead rows: plain loads and stores
                            uint32_t v[16];
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                int t = st + i;
                                while (t >= Nt) t -= Nt;
                                if (KSRC == 0 && wide) {
                                    const unsigned long long x =
                                        live ? __ldg(reinterpret_cast<const unsigned long long*>(row) + t) : 0ull;
                                    v[2 * i] = (uint32_t)x;
                                    v[2 * i + 1] = (uint32_t)(x >> 32);
                                } else {  // u32 counts or floats: the 32-bit word
                                    v[i] = live ? __ldg(reinterpret_cast<const unsigned*>(row) + t) : 0u;
                                }
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                if (q < rawq)
                                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16u * q),
                                                 "r"(v[4 * q]), "r"(v[4 * q + 1]), "r"(v[4 * q + 2]), "r"(v[4 * q + 3])
                                                 : "memory");
                        }
                        st += 8;
                        while (st >= Nt) st -= Nt;
                    }
                    // the arrive fires when this thread's copies have landed
                    // (at once if it made none); its plain stores precede it
                    if (async)
                        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"((a_rfull + 8u * (rs)))
                                     : "memory");
                    else
                        t2_arrive((a_rfull + 8u * (rs)));
                }
            }
        }
    } else if (warp < kT2EpiWarp) {
        // ---- converters: group gp takes the slabs gs = gp mod kT2Groups; thread
        // n converts wire row n to TF32 (hi part, plus a lo part where a value
        // does not fit 11 bits) into the MMA ring
        const int n = tid & (kT2N - 1), gp = (warp - 4) >> 2;
        uint32_t dirty = 0u;  // slots whose lo part this warp wrote non-zero
        uint32_t gs = 0;
        for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
          const T2Item I = t2_item<H>(ev, plan, it);
          // u64 or u32 count cells (cnt_wide), or floats: a raw row is 8 ticks
          const bool wide = KSRC == 0 && cnt_wide(ev.p[plan.pl[I.k]]);
          const uint32_t rowb = wide ? 64u : 32u;
          for (int s = 0; s < I.nslab; ++s, ++gs) {
            if ((int)(gs % kT2Groups) != gp) continue;
            const uint32_t rs = gs % kT2Raw;
            T2_WAIT((a_rfull + 8u * (rs)), (gs / kT2Raw) & 1u, 0);
            uint4 rw[kT2SK][4];
#pragma unroll
            for (int h = 0; h < kT2SK; ++h) {
                const uint32_t src = raw + rs * kT2RawSlot + h * kT2RawHalf + (uint32_t)n * rowb;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q < 2 || wide)
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(rw[h][q].x), "=r"(rw[h][q].y), "=r"(rw[h][q].z), "=r"(rw[h][q].w)
                                     : "r"(src + 16u * q)
                                     : "memory");
            }
            __syncwarp();
            if (lane == 0) t2_arrive((a_rempty + 8u * (rs)));
            uint32_t vh[kT2SK][8], vl[kT2SK][8];
            uint32_t any_lo = 0u;
#pragma unroll
            for (int h = 0; h < kT2SK; ++h) {
                float x[8];
                if (KSRC == 0 && wide) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        x[2 * q] = (float)(((unsigned long long)rw[h][q].y << 32) | rw[h][q].x);
                        x[2 * q + 1] = (float)(((unsigned long long)rw[h][q].w << 32) | rw[h][q].z);
                    }
                } else if (KSRC == 0) {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        x[4 * q] = (float)rw[h][q].x;
                        x[4 * q + 1] = (float)rw[h][q].y;
                        x[4 * q + 2] = (float)rw[h][q].z;
                        x[4 * q + 3] = (float)rw[h][q].w;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        x[4 * q] = __uint_as_float(rw[h][q].x);
                        x[4 * q + 1] = __uint_as_float(rw[h][q].y);
                        x[4 * q + 2] = __uint_as_float(rw[h][q].z);
                        x[4 * q + 3] = __uint_as_float(rw[h][q].w);
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    vh[h][i] = tc_tf32(x[i]);
                    vl[h][i] = tc_tf32(x[i] - __uint_as_float(vh[h][i]));
                    any_lo |= vl[h][i] << 1;  // (sign bit dropped: -0 is 0)
                }
            }
            const bool need = __any_sync(0xffffffffu, any_lo != 0u);
            const uint32_t slot = gs % kT2Slots, use = gs / kT2Slots;
            if (use > 0) T2_WAIT((a_empty + 8u * (slot)), (use - 1) & 1u, 1);
            const uint32_t base = ring + slot * kT2SlotBytes + (uint32_t)(((n >> 3) << 7) + ((n & 7) << 4));
            const uint32_t bit = 1u << slot;
            const bool wlo = need || (dirty & bit);
#pragma unroll
            for (int h = 0; h < kT2SK; ++h) {
                const uint32_t b = base + h * kT2Step;
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b), "r"(vh[h][0]), "r"(vh[h][1]),
                             "r"(vh[h][2]), "r"(vh[h][3]));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b + 2048u), "r"(vh[h][4]), "r"(vh[h][5]),
                             "r"(vh[h][6]), "r"(vh[h][7]));
                if (wlo) {
                    if (!need)
#pragma unroll
                        for (int i = 0; i < 8; ++i) vl[h][i] = 0u;
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b + kT2Part), "r"(vl[h][0]),
                                 "r"(vl[h][1]), "r"(vl[h][2]), "r"(vl[h][3]));
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b + kT2Part + 2048u), "r"(vl[h][4]),
                                 "r"(vl[h][5]), "r"(vl[h][6]), "r"(vl[h][7]));
                }
            }
            if (wlo) dirty = need ? (dirty | bit) : (dirty & ~bit);
            // generic-proxy writes -> the tensor core's async proxy (this
            // thread has no global loads in flight: the fence is cheap)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if (need) atomicMax(&s_tag[slot], (use << 1) | 1u);
                t2_arrive((a_full + 8u * (slot)));
            }
          }
        }
    } else if (warp == kT2MmaWarp) {
        // ---- MMA issuer: the whole warp runs the loop, one elected lane issues
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kT2N >> 3) << 17) |
                               ((uint32_t)(kTcM >> 4) << 24);
        const uint64_t dring = tc_desc(ring, 2048u, 128u);  // slot 0, hi part, K step 0 (descriptor units of 16 B)
        uint32_t gs = 0, gsub = 0;
        for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
            const T2Item I = t2_item<H>(ev, plan, it);
            const uint32_t e_hi = sbase + plan.eoff[I.k];
            const uint64_t da0 = tc_desc(e_hi + (uint32_t)(I.J - 1) * 128u, (uint32_t)(I.RE >> 3) * 128u, 128u);
            const uint64_t dlo = (uint64_t)(((uint32_t)I.RE * 32u) >> 4);  // E lo part
            const int js = I.J / kT2SK;  // slabs per sub-block
            int jlo = 0, jhi = 0;        // sub-blocks whose K range holds slab s
            for (int s = 0; s < I.nslab; ++s, ++gs) {
                const uint32_t slot = gs & (kT2Slots - 1), use = gs / kT2Slots;
                if (s == kSlabsPerSub * (jhi + 1) && jhi + 1 < I.nsub) ++jhi;
                if (s - kSlabsPerSub * jlo == js) ++jlo;
                T2_WAIT((a_full + 8u * (slot)), use & 1u, 0);
                const bool two = s_tag[slot] == ((use << 1) | 1u);  // some warp wrote a lo part
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t db0 = dring + (uint64_t)(slot * (kT2SlotBytes >> 4));
                for (int jb = jlo; jb <= jhi; ++jb) {
                    const int j0 = kT2SK * (s - kSlabsPerSub * jb);  // the slab's first K step in sub-block jb
                    const uint32_t g = gsub + (uint32_t)jb, ab = g & (kT2Acc - 1), v = g / kT2Acc;
                    if (j0 == 0 && v > 0) {
                        T2_WAIT((a_acce + 8u * (ab)), (v - 1) & 1u, 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    }
                    const uint32_t d = tmem + ab * 128u;
#ifdef WS_T2_PROF
                    const long long t2p_m = clock64();
#endif
                    if (elect_one()) {
#pragma unroll
                        for (int h = 0; h < kT2SK; ++h) {
                            const uint64_t dah = da0 - (uint64_t)(8 * (j0 + h)), dal = dah + dlo;  // E rows 8 j earlier
                            const uint64_t db = db0 + (uint64_t)(h * (kT2Step >> 4));
                            tc_mma(d, dah, db, idesc, (j0 + h) > 0 ? 1u : 0u);
                            tc_mma(d, dal, db, idesc, 1u);
                            if (two) tc_mma(d, dah, db + (kT2Part >> 4), idesc, 1u);
                        }
                        if (j0 + kT2SK == I.J) t2_commit((a_accf + 8u * (ab)));
                    }
                    __syncwarp();
#ifdef WS_T2_PROF
                    t2p_acc[2] += clock64() - t2p_m;
#endif
                }
                if (elect_one()) t2_commit((a_empty + 8u * (slot)));
                __syncwarp();
            }
            gsub += (uint32_t)I.nsub;
        }
    } else {
        // ---- epilogue: warp (kT2EpiWarp + q) drains TMEM lanes 32 q .. 32 q + 31 (ticks)
        const int q4 = warp & 3;
        uint32_t gsub = 0;
        for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
            const T2Item I = t2_item<H>(ev, plan, it);
            const PlaneDesc& P = ev.p[plan.pl[I.k]];
            const int Nt = P.N;
            float* const frame = P.frame;
            const bool ro = ev.ro != 0;
            const int cmax = I.nr + 2 * H;  // columns past the plane's last output row are not stored
            float ww[2 * H + 1];
#pragma unroll
            for (int e = 0; e <= 2 * H; ++e) ww[e] = (float)P.ww[e];
            for (int jb = 0; jb < I.nsub; ++jb) {
                const uint32_t g = gsub + (uint32_t)jb, ab = g % kT2Acc, v = g / kT2Acc;
                T2_WAIT((a_accf + 8u * (ab)), v & 1u, 0);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const int t = I.T0 + kTcM * jb + 32 * q4 + lane;
                const bool tv = t < Nt;
                float carry[2 * H + 1];
#pragma unroll
                for (int e = 0; e <= 2 * H; ++e) carry[e] = 0.0f;
#pragma unroll 1
                for (int ck = 0; ck < kT2N / 32; ++ck) {
                    uint32_t x[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                        "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                        "[%32];"
                        : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]),
                          "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]),
                          "=r"(x[15]), "=r"(x[16]), "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]), "=r"(x[21]),
                          "=r"(x[22]), "=r"(x[23]), "=r"(x[24]), "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]),
                          "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
                        : "r"(tmem + ((uint32_t)(32 * q4) << 16) + ab * 128u + (uint32_t)(32 * ck)));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (!ro) {
                        // plain stores: one running offset (row r0 + col - 2H, tick t), predicated
                        long long off = (long long)(I.r0 - 2 * H + 32 * ck) * Nt + t;
#pragma unroll
                        for (int cc = 0; cc < 32; ++cc, off += Nt) {
                            const int col = 32 * ck + cc;  // the last input column of output row col - 2H
                            float out = 0.0f;
#pragma unroll
                            for (int e = 0; e <= 2 * H; ++e)
                                out = __fmaf_rn(ww[e], cc - e >= 0 ? __uint_as_float(x[cc - e]) : carry[2 * H + cc - e], out);
                            if (tv && col >= 2 * H && col < cmax) __stcs(frame + off, out);
                        }
                    } else {
                        // fused readout (noise + digitize) on tick pairs: even lanes
                        // take their odd neighbour's value; stencil unrolled over
                        // the chunk's columns, the readout call kept out of line
                        float outv[32];
#pragma unroll
                        for (int cc = 0; cc < 32; ++cc) {
                            float out = 0.0f;
#pragma unroll
                            for (int e = 0; e <= 2 * H; ++e)
                                out = __fmaf_rn(ww[e], cc - e >= 0 ? __uint_as_float(x[cc - e]) : carry[2 * H + cc - e], out);
                            outv[cc] = out;
                        }
                        float nxtv[32];
#pragma unroll
                        for (int cc = 0; cc < 32; ++cc) nxtv[cc] = __shfl_down_sync(0xffffffffu, outv[cc], 1);
                        if (!(lane & 1) && tv) {
#pragma unroll 1
                            for (int cc = 0; cc < 32; ++cc) {
                                const int o = 32 * ck + cc - 2 * H;
                                if (o >= 0 && o < I.nr) readout_pair(ev, P, I.r0 + o, t, outv[cc], nxtv[cc], t + 1 < Nt);
                            }
                        }
                    }
                    // the last 2H columns feed the next chunk's first outputs
#pragma unroll
                    for (int e = 0; e < 2 * H; ++e) carry[e] = __uint_as_float(x[32 - 2 * H + e]);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) t2_arrive((a_acce + 8u * (ab)));
            }
            gsub += (uint32_t)I.nsub;
        }
    }
    T2_PROF_FLUSH(warp < 4 ? 0 : warp < kT2EpiWarp ? 4 : warp < kT2MmaWarp ? 8 : 12);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == kT2MmaWarp) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kT2Acc * 128));
    }
}

}  // namespace wsb

// Sub-blocks per tile for a plane on the tensor-core path (the largest that
// fits two CTAs per SM, else one), or 0 when it is not eligible (kernel taps
// absent, stencil wider than 5 taps, window too large).
extern "C" int wsb_conv_tc_nb(const wsb::PlaneDesc& P)
{
    const char* v = getenv("WS_CONV_TC");  // 0: the row FFT for every grid convolution (A/B, tests)
    if ((v && atoi(v) == 0) || !P.kern || P.h > wsb::kTcMaxH || P.n_lags < 1) return 0;
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

// The pipelined tensor-core convolution (k_conv_tc2) of every non-direct plane
// of the event: cudaErrorNotSupported when a plane is not eligible (stencil
// wider than 5 taps, more than kT2MaxJ K steps, shared memory) - the caller
// then takes k_conv_tc / the row FFT.
extern "C" cudaError_t wsb_launch_conv_tc2(const wsb::EventDesc& ev, cudaStream_t s)
{
    using namespace wsb;
    const char* off = getenv("WS_CONV_TC2");  // 0: the one-tile-at-a-time kernel (A/B, tests)
    if (off && atoi(off) == 0) return cudaErrorNotSupported;
    T2Plan plan{};
    static const int chunk = [] {
        const char* v = getenv("WS_CONV_TC2_CHUNK");  // sub-blocks per work item (tuning only)
        return v ? std::max(1, std::min(64, atoi(v))) : 8;
    }();
    plan.chunk = chunk;
    uint32_t eoff = kT2Slots * kT2SlotBytes + kT2Raw * kT2RawSlot;
    int h = -1, src = -1;
    for (int i = 0; i < ev.n_planes; ++i) {
        const PlaneDesc& P = ev.p[i];
        if (P.direct || !P.frame && !P.frame64 && !P.adc) continue;
        if (!P.kern || P.n_lags < 1 || P.h > kTcMaxH) return cudaErrorNotSupported;
        const int si = P.charge_cnt ? 0 : 1;
        if (h >= 0 && (P.h != h || si != src)) return cudaErrorNotSupported;
        h = P.h;
        src = si;
        const T2Geom g = t2_geom(P.lo_lag, P.n_lags);
        if (g.J > kT2MaxJ) return cudaErrorNotSupported;
        const int k = plan.np++;
        plan.pl[k] = i;
        plan.eoff[k] = eoff;
        eoff += (uint32_t)(2 * g.RE * 32);
        const int R = kT2N - 2 * P.h;
        const int strips = (P.W + R - 1) / R, nsub = (P.N + kTcM - 1) / kTcM;
        plan.chunks[k] = (nsub + plan.chunk - 1) / plan.chunk;
        plan.item0[k + 1] = plan.item0[k] + strips * plan.chunks[k];
    }
    if (plan.np == 0) return cudaSuccess;
    // TMA box loads where every plane allows them: no wire stencil (no row
    // wrap), N % 8 == 0 (no slab wraps), 16-byte aligned rows and base
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    const char* tv = getenv("WS_CONV_TC2_TMA");  // 0: cp.async loads (A/B, tests)
    plan.tma = encode && h == 0 && !(tv && atoi(tv) == 0) ? 1 : 0;
    for (int k = 0; k < plan.np && plan.tma; ++k) {
        const PlaneDesc& P = ev.p[plan.pl[k]];
        const void* base = src == 0 ? (const void*)P.charge_cnt : (const void*)P.charge_in;
        const size_t esz = src == 0 ? 8 : 4;
        if (P.N % 8 || ((size_t)P.N * esz) % 16 || reinterpret_cast<uintptr_t>(base) % 16) {
            plan.tma = 0;
            break;
        }
        const cuuint64_t dims[2] = {(cuuint64_t)P.N, (cuuint64_t)P.W};
        const cuuint64_t strides[1] = {(cuuint64_t)P.N * esz};
        const cuuint32_t box[2] = {8u, (cuuint32_t)kT2N};
        const cuuint32_t estr[2] = {1u, 1u};
        if (encode(&plan.tm[k], src == 0 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            plan.tma = 0;
        const cuuint64_t strides32[1] = {(cuuint64_t)P.N * 4};
        if (src == 0 && ((size_t)P.N * 4) % 16) plan.tma = 0;
        if (src == 0 && plan.tma &&
            encode(&plan.tm32[k], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides32, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            plan.tma = 0;
    }
    const size_t smem = eoff;
    if (smem > 224 * 1024) return cudaErrorNotSupported;
    static std::atomic<unsigned long long> ready{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(ready & (1ull << dev))) {
        for (auto f : {k_conv_tc2<0, 0>, k_conv_tc2<1, 0>, k_conv_tc2<2, 0>, k_conv_tc2<0, 1>, k_conv_tc2<1, 1>,
                       k_conv_tc2<2, 1>}) {
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
            if (e != cudaSuccess) return e;
        }
        ready |= 1ull << dev;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int items = plan.item0[plan.np];
    using K = void (*)(const EventDesc, const T2Plan);
    const K fns[2][3] = {{k_conv_tc2<0, 0>, k_conv_tc2<1, 0>, k_conv_tc2<2, 0>},
                         {k_conv_tc2<0, 1>, k_conv_tc2<1, 1>, k_conv_tc2<2, 1>}};
    fns[src][h]<<<std::min(items, sms), kT2Threads, smem, s>>>(ev, plan);
    return cudaGetLastError();
}

#ifdef WS_T2_PROF
#include <cstdio>
extern "C" void wsb_t2_prof_dump()
{
    unsigned long long h[16];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, wsb::g_t2prof, sizeof(h));
    const char* role[4] = {"loader", "convert", "epilogue", "mma"};
    for (int r = 0; r < 4; ++r)
        fprintf(stderr, "t2prof %-8s total %14llu  wait0 %14llu  wait1 %14llu  x2 %14llu\n", role[r], h[4 * r + 3], h[4 * r],
                h[4 * r + 1], h[4 * r + 2]);
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(wsb::g_t2prof, z, sizeof(z));
}
#endif
