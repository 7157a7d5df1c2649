// Per-depo response profiles for the time-domain path on the tensor cores.
//
// Every unit (depo on a direct-path plane) needs g[j] = sum_k tv[k] h[j - k],
// j < L = n_t + n_lags - 1: its tick profile tv (n_t <= 32 bins,
// sample_patch's bin integrals, rasterize.cpp:91-92) convolved with the
// plane's combined time kernel h (build_response's time-domain kernel,
// spectral.cpp:98-113). For 16 units at a time this is a dense GEMM
//   G[16 x N] = TV[16 x K] . T[K x N],  T[k][j] = h[j - k]  (Toeplitz, K <= 32),
// run as mma.sync m16n8k8 TF32 with the 3-pass split (a_hi b_hi + a_hi b_lo +
// a_lo b_hi, fp32 accumulate: ~fp32 accuracy). The Toeplitz operand is never
// materialised: B fragments read the kernel's hi/lo TF32 parts from shared
// memory at offset j - k. g is zero-filled up to a multiple of 32 taps (the
// kernel is zero-padded) and max|g| goes to g[-1]. Units with n_t > 32 (very
// wide depos) take a per-warp SIMT loop.
#include "ws_common.cuh"

#include <atomic>

#include <algorithm>
#include <cstdlib>

namespace wsb {

constexpr int kGpWarps = 4;
constexpr int kGpPre = 32;  // kernel taps staged before index 0 (j - k >= -31)
constexpr int kGpPost = 16; // taps past the last tile (the paired tile loop's spare tile)

__device__ __forceinline__ uint32_t tf32_rna(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void mma_tf32(float* c, const uint32_t* a, uint32_t b0, uint32_t b1)
{
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// The n tiles (8 output taps each) of one 16-unit group with KS k steps. B
// fragments depend on n - ks only, so a window of the last KS fragments
// slides along n (one new fragment = 4 shared loads per tile); the three
// TF32 passes accumulate into one chain per tile.
template <int KS>
__device__ __forceinline__ void gp_tiles(const uint32_t* hh, const uint32_t* hl, const uint32_t (*ah)[4],
                                         const uint32_t (*al)[4], int nt_n, int gq, int tq, const bool* mine,
                                         const int* lp, float* const* gp, float* gmax)
{
    // fragment for m = n - ks: b0 (k = tq, j = gq) = h[8 m + gq - tq], b1 = h[8 m + gq - tq - 4]
    uint32_t bh0[KS], bh1[KS], bl0[KS], bl1[KS];
    const int x0 = gq - tq + kGpPre;
#pragma unroll
    for (int i = 0; i + 1 < KS; ++i) {  // the window as of n = -1: slot i holds m = -1 - i (zero-padded taps)
        const int x = x0 - 8 * (i + 1);
        bh0[i] = hh[x];
        bh1[i] = hh[x - 4];
        bl0[i] = hl[x];
        bl1[i] = hl[x - 4];
    }
    // two tiles per iteration (independent MMA chains); an odd count computes
    // one spare tile past the end (padded taps, stores predicated off)
#pragma unroll 1
    for (int n = 0; n < nt_n; n += 2) {
        float c[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int t = 0; t < 2; ++t) {
#pragma unroll
            for (int i = KS - 1; i > 0; --i) {
                bh0[i] = bh0[i - 1];
                bh1[i] = bh1[i - 1];
                bl0[i] = bl0[i - 1];
                bl1[i] = bl1[i - 1];
            }
            const int x = x0 + 8 * (n + t);
            bh0[0] = hh[x];
            bh1[0] = hh[x - 4];
            bl0[0] = hl[x];
            bl1[0] = hl[x - 4];
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                mma_tf32(c[t], ah[ks], bh0[ks], bh1[ks]);
                mma_tf32(c[t], ah[ks], bl0[ks], bl1[ks]);
                mma_tf32(c[t], al[ks], bh0[ks], bh1[ks]);
            }
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            // C (16 x 8): c0, c1 -> row gq, taps 8n + 2tq, +1; c2, c3 -> row gq + 8
            const int j = 8 * (n + t) + 2 * tq;
            if (mine[0] && j < lp[0]) *reinterpret_cast<float2*>(gp[0] + j) = make_float2(c[t][0], c[t][1]);
            if (mine[1] && j < lp[1]) *reinterpret_cast<float2*>(gp[1] + j) = make_float2(c[t][2], c[t][3]);
            if (n + t < nt_n) {
                gmax[0] = fmaxf(gmax[0], fmaxf(fabsf(c[t][0]), fabsf(c[t][1])));
                gmax[1] = fmaxf(gmax[1], fmaxf(fabsf(c[t][2]), fabsf(c[t][3])));
            }
        }
    }
}

__global__ void __launch_bounds__(32 * kGpWarps)
k_gprof(const EventDesc ev, const UnitRec* __restrict__ recs, uint32_t* __restrict__ pool)
{
    const PlaneDesc& P = ev.p[blockIdx.y];
    if (!P.direct || P.n_units == 0) return;
    const int nl = P.n_lags;
    const int ntap = (nl + 31 + 31) & ~31;  // >= ceil32(L) for every n_t <= 32
    // kernel tap i, -kGpPre <= i < ntap, split into TF32 hi + lo parts
    extern __shared__ uint32_t s_hk[];
    uint32_t* hh = s_hk;
    uint32_t* hl = s_hk + (ntap + kGpPre + kGpPost);
    for (int x = threadIdx.x; x < ntap + kGpPre + kGpPost; x += blockDim.x) {
        const float v = __ldg(&P.kern[x - kGpPre]);  // zero-padded by kKernPad >= 192 taps
        const uint32_t hi = tf32_rna(v);
        hh[x] = hi;
        hl[x] = tf32_rna(v - __uint_as_float(hi));
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;  // mma fragment coordinates
    const int n_groups = (int)((P.n_units + 15) / 16);
    const int stride = gridDim.x * kGpWarps;
    // the fields of this thread's two records (rows gq, gq + 8), the next
    // group's prefetched while the current one computes
    struct Rec {
        int w0, n_w, n_t;
        uint32_t pool, goff;
    };
    auto load_rec = [&](int grp, Rec* out) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t ul = (uint32_t)grp * 16 + gq + 8 * h;
            out[h].w0 = -1;
            if (grp < n_groups && ul < P.n_units) {
                const int4 a = __ldg(reinterpret_cast<const int4*>(recs + P.unit_base + ul));
                const int4 b = __ldg(reinterpret_cast<const int4*>(recs + P.unit_base + ul) + 1);
                out[h].w0 = a.x;
                out[h].n_w = a.z;
                out[h].n_t = a.w;
                out[h].pool = (uint32_t)b.x;
                out[h].goff = (uint32_t)b.y;
            }
        }
    };
    Rec nxt[2];
    load_rec(blockIdx.x * kGpWarps + warp, nxt);
    for (int grp = blockIdx.x * kGpWarps + warp; grp < n_groups; grp += stride) {
        Rec cur[2] = {nxt[0], nxt[1]};
        load_rec(grp + stride, nxt);
        // this thread's two units: rows gq and gq + 8 of the group
        const float* tv[2];
        float* gp[2];
        int nt[2], lp[2];
        bool mine[2], wide[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            mine[h] = false;
            wide[h] = false;
            nt[h] = 0;
            lp[h] = 0;
            tv[h] = nullptr;
            gp[h] = nullptr;
            if (cur[h].w0 >= 0) {
                const uint32_t tvo = cur[h].pool + (uint32_t)(cur[h].n_w + unit_n_eff(P, cur[h].n_w));
                tv[h] = reinterpret_cast<const float*>(pool + tvo);
                gp[h] = reinterpret_cast<float*>(pool + cur[h].goff);
                wide[h] = cur[h].n_t > 32;
                mine[h] = !wide[h];
                nt[h] = mine[h] ? cur[h].n_t : 0;
                lp[h] = (cur[h].n_t + nl - 1 + 31) & ~31;
            }
        }
        // k steps (8 taps of tv each) and n tiles (8 output taps) the group needs
        int ks_n = (max(nt[0], nt[1]) + 7) >> 3;
        int nt_n = max(mine[0] ? lp[0] : 0, mine[1] ? lp[1] : 0) >> 3;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            ks_n = max(ks_n, __shfl_xor_sync(0xffffffffu, ks_n, o));
            nt_n = max(nt_n, __shfl_xor_sync(0xffffffffu, nt_n, o));
        }
        // A fragments (row-major 16 x 8 per k step): a0 (gq, tq), a1 (gq+8, tq),
        // a2 (gq, tq+4), a3 (gq+8, tq+4); hi and lo TF32 parts
        uint32_t ah[4][4], al[4][4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int h = e & 1, k = 8 * ks + tq + 4 * (e >> 1);
                const float v = (ks < ks_n && k < nt[h]) ? tv[h][k] : 0.0f;
                ah[ks][e] = tf32_rna(v);
                al[ks][e] = tf32_rna(v - __uint_as_float(ah[ks][e]));
            }
        }
        float gmax[2] = {0.0f, 0.0f};
        switch (ks_n) {
            case 1: gp_tiles<1>(hh, hl, ah, al, nt_n, gq, tq, mine, lp, gp, gmax); break;
            case 2: gp_tiles<2>(hh, hl, ah, al, nt_n, gq, tq, mine, lp, gp, gmax); break;
            case 3: gp_tiles<3>(hh, hl, ah, al, nt_n, gq, tq, mine, lp, gp, gmax); break;
            default: gp_tiles<4>(hh, hl, ah, al, nt_n, gq, tq, mine, lp, gp, gmax); break;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            gmax[h] = fmaxf(gmax[h], __shfl_xor_sync(0xffffffffu, gmax[h], 1));
            gmax[h] = fmaxf(gmax[h], __shfl_xor_sync(0xffffffffu, gmax[h], 2));
            if (mine[h] && tq == 0) gp[h][-1] = gmax[h];
        }
        // wide tick profiles (n_t > 32): the whole warp, one unit at a time
        if (!__any_sync(0xffffffffu, wide[0] || wide[1])) continue;
#pragma unroll 1
        for (int src = 0; src < 32; src += 4) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const bool w = __shfl_sync(0xffffffffu, wide[h], src);
                if (!w) continue;  // lane 4 gq (tq == 0) speaks for rows gq, gq + 8
                const float* tvw = reinterpret_cast<const float*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(tv[h]), src));
                float* gw = reinterpret_cast<float*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(gp[h]), src));
                const int lpw = __shfl_sync(0xffffffffu, lp[h], src);
                const UnitRec rec = recs[P.unit_base + (uint32_t)grp * 16 + (src >> 2) + 8 * h];
                const int ntr = rec.n_t, L = ntr + nl - 1;
                float gm = 0.0f;
                for (int jj = lane; jj < lpw; jj += 32) {
                    const int k0 = jj - nl + 1 > 0 ? jj - nl + 1 : 0, k1 = jj < ntr - 1 ? jj : ntr - 1;
                    float sum = 0.0f;
                    for (int k = k0; k <= k1; ++k) sum = __fmaf_rn(tvw[k], __ldg(&P.kern[jj - k]), sum);
                    gw[jj] = jj < L ? sum : 0.0f;
                    gm = fmaxf(gm, fabsf(sum));
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
                if (lane == 0) gw[-1] = gm;
            }
        }
    }
}

}  // namespace wsb

extern "C" int wsb_gprof_umma_n(const wsb::EventDesc& ev);
extern "C" cudaError_t wsb_launch_gprof_umma(const wsb::EventDesc& ev, const wsb::UnitRec* recs, uint32_t* pool,
                                             int N, cudaStream_t s, int pdl);

extern "C" cudaError_t wsb_launch_gprof(const wsb::EventDesc& ev, const wsb::UnitRec* recs, uint32_t* pool,
                                        cudaStream_t s, int pdl)
{
    // tcgen05 path (ws_gprof_umma.cu) unless a kernel is too long for it or
    // WS_GPROF_MMASYNC=1 selects the warp-level mma.sync kernel below
    static const bool mmasync = [] {
        const char* v = getenv("WS_GPROF_MMASYNC");
        return v && v[0] == '1';
    }();
    if (!mmasync) {
        const int N = wsb_gprof_umma_n(ev);
        if (N > 0) return wsb_launch_gprof_umma(ev, recs, pool, N, s, pdl);
    }
    uint32_t max_units = 0;
    int max_lags = 0;
    for (int i = 0; i < ev.n_planes; ++i)
        if (ev.p[i].direct) {
            max_units = max_units > ev.p[i].n_units ? max_units : ev.p[i].n_units;
            max_lags = max_lags > ev.p[i].n_lags ? max_lags : ev.p[i].n_lags;
        }
    if (max_units == 0) return cudaSuccess;
    const int ntap = (max_lags + 62) & ~31;
    const size_t smem = 2 * sizeof(uint32_t) * (size_t)(ntap + wsb::kGpPre + wsb::kGpPost);
    static std::atomic<unsigned long long> ready{0};  // per-device attribute setup (idempotent)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(ready & (1ull << dev))) {
        e = cudaFuncSetAttribute(wsb::k_gprof, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        if (e != cudaSuccess) return e;
        ready |= 1ull << dev;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned groups = (max_units + 15) / 16;
    // persistent warps (a few groups each, the next group's records in flight)
    const unsigned blocks = std::min((groups + wsb::kGpWarps - 1) / wsb::kGpWarps, (unsigned)sms * 6u);
    const dim3 grid(blocks, (unsigned)ev.n_planes);
    wsb::k_gprof<<<grid, 32 * wsb::kGpWarps, smem, s>>>(ev, recs, pool);
    return cudaGetLastError();
}
