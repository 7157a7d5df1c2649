// Per-depo response profiles on the 5th-generation tensor cores (tcgen05).
//
// g_u = tv_u (*) h for 128 units u at a time is one GEMM
//   G[128 x N] = TV[128 x 32] . T[32 x N],  T[k][j] = h[j - k]   (Toeplitz)
// (N = ceil32(n_lags + 31) output taps, n_t <= 32 tick taps), issued by one
// thread as tcgen05.mma kind::tf32 with the fp32 accumulator in TMEM. TF32
// operands in the 3-pass split (hi.hi + hi.lo + lo.hi, all into the same
// accumulator: ~fp32 accuracy), 12 MMAs of 128 x N x 8 per tile. Operands are
// staged in shared memory in the canonical K-major no-swizzle layout (core
// matrices of 8 rows x 16 bytes); the Toeplitz T is rebuilt per CTA from the
// plane's zero-padded kernel. The epilogue reads the accumulator back with
// tcgen05.ld (warp w owns TMEM lanes 32w..32w+31 = units) and writes each
// unit's ceil32(L) taps. This replaces the warp-level mma.sync kernel
// (k_gprof), whose TF32 rate on sm_100 was its limiter. Units with n_t > 32
// compute their profile with a scalar loop in the epilogue.
#include "ws_common.cuh"

#include <atomic>
#include <cstdlib>

#include <algorithm>

namespace wsb {

constexpr int kUmM = 128;  // units per tile (UMMA M)
constexpr int kUmK = 32;   // tick-profile taps (UMMA K = 4 steps of 8)
constexpr int kUmThreads = 256;  // two warps per TMEM lane quadrant

__device__ __forceinline__ uint32_t um_tf32(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// byte offset of element (row r, k) in a K-major SWIZZLE_NONE operand of R rows:
// core matrix (k / 4, r / 8) of 8 rows x 16 bytes, K-chunks R/8 core matrices apart
__device__ __forceinline__ uint32_t um_off(int r, int kc, int R) { return ((kc * (R >> 3) + (r >> 3)) << 7) + ((r & 7) << 4); }

// shared-memory matrix descriptor (sm100): start, leading (K) and stride (M/N)
// byte offsets >> 4, version 1, no swizzle
__device__ __forceinline__ uint64_t um_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void um_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

__device__ __forceinline__ bool elect_sync_one()
{
    uint32_t p;
    asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; selp.u32 %0, 1, 0, e; }" : "=r"(p));
    return p != 0u;
}

__global__ void __launch_bounds__(kUmThreads) k_gprof_umma(const EventDesc ev, const UnitRec* __restrict__ recs,
                                                           uint32_t* __restrict__ pool, int N)
{
    const PlaneDesc& P = ev.p[blockIdx.y];
    if (!P.direct || P.n_units == 0) return;
    const int nl = P.n_lags;
    const int tid = threadIdx.x, warp = tid >> 5;

    // layout: A hi | A lo (128 x 32 each) | B hi | B lo (N x 32 each), 128-byte aligned
    extern __shared__ __align__(128) unsigned char um_smem[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(um_smem);
    const uint32_t a_hi = sbase, a_lo = a_hi + kUmM * kUmK * 4;
    const uint32_t b_hi = a_lo + kUmM * kUmK * 4, b_lo = b_hi + (uint32_t)N * kUmK * 4;
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_bar;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);

    // TMEM accumulator (N fp32 columns x 128 lanes) and the completion barrier
    if (warp == 0) {
        const uint32_t cols = N <= 32 ? 32u : N <= 64 ? 64u : N <= 128 ? 128u : 256u;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                     "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // B = the plane's Toeplitz kernel, hi and lo TF32 parts: row n, taps k..k+3
    for (int i = tid; i < N * (kUmK / 4); i += kUmThreads) {
        const int n = i % N, kc = i / N;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float v = __ldg(&P.kern[n - (4 * kc + q)]);  // zero-padded both sides
            hi[q] = um_tf32(v);
            lo[q] = um_tf32(v - __uint_as_float(hi[q]));
        }
        const uint32_t o = um_off(n, kc, N);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b_hi + o), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]),
                     "r"(hi[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b_lo + o), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]),
                     "r"(lo[3]));
    }
    // TMEM address to all threads
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kUmM >> 4) << 24);
    const uint32_t lbo_a = (kUmM / 8) * 128, lbo_b = (uint32_t)(N / 8) * 128;
    // thread -> unit row (tid & 127) and half (tid >> 7): K taps 16 h..16 h+15
    // when staging, output columns [h N/2, (h+1) N/2) in the epilogue
    const int row = tid & (kUmM - 1), half = tid >> 7;
    const uint32_t trow = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    const int n_tiles = (int)((P.n_units + kUmM - 1) / kUmM);

    // persistent over this plane's tiles; B (and the TMEM allocation) stay
    // this thread's unit of a tile (row tid): record and tick profile (0 past
    // n_t; wide units 0); the next tile's are loaded while this one's
    // accumulator drains
    constexpr int kH = kUmK / 2;
    auto fetch = [&](int tile, UnitRec& rec, float* vals) {
        const uint32_t ul = (uint32_t)tile * kUmM + (uint32_t)row;
        rec = UnitRec{};
        rec.w0 = -1;
        if (tile < n_tiles && ul < P.n_units) rec = recs[P.unit_base + ul];
        const bool ok = rec.w0 >= 0 && rec.n_t <= kUmK;
        const float* t = reinterpret_cast<const float*>(pool + rec.pool + (uint32_t)(rec.n_w + unit_n_eff(P, rec.n_w)));
#pragma unroll
        for (int k = 0; k < kH; ++k) vals[k] = ok && kH * half + k < rec.n_t ? __ldg(t + kH * half + k) : 0.0f;
    };
    // the records and tick profiles come from the previous kernel (k_sample_off);
    // with a programmatic launch the TMEM / barrier / Toeplitz setup above
    // overlapped its tail
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the sampler has completed: a programmatically launched successor
    // (k_direct) may now run its profile-independent prologue (it reads the
    // sampler's tile lists), waiting for this grid before the profiles
    asm volatile("griddepcontrol.launch_dependents;");
    UnitRec rec_n;
    float vals_n[kH];
    fetch(blockIdx.x, rec_n, vals_n);
#pragma unroll 1
    for (int tile = blockIdx.x, it = 0; tile < n_tiles; tile += gridDim.x, ++it) {
        const UnitRec rec = rec_n;
        float vals[kH];
#pragma unroll
        for (int k = 0; k < kH; ++k) vals[k] = vals_n[k];
        const bool live = rec.w0 >= 0;
        const float* tv =
            reinterpret_cast<const float*>(pool + rec.pool + (uint32_t)(rec.n_w + unit_n_eff(P, rec.n_w)));
        const int nt = live && rec.n_t <= kUmK ? rec.n_t : 0;
#pragma unroll
        for (int kq = 0; kq < kH / 4; ++kq) {
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float v = vals[4 * kq + q];
                hi[q] = um_tf32(v);
                lo[q] = um_tf32(v - __uint_as_float(hi[q]));
            }
            const uint32_t o = um_off(row, (kH / 4) * half + kq, kUmM);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a_hi + o), "r"(hi[0]), "r"(hi[1]),
                         "r"(hi[2]), "r"(hi[3]));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a_lo + o), "r"(lo[0]), "r"(lo[1]),
                         "r"(lo[2]), "r"(lo[3]));
        }
        // operands visible to the tensor core (async proxy); the previous
        // tile's TMEM reads are complete (fence before the barrier)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (tid == 0) {
            // 3 passes x 4 K steps (8 taps = two 16-byte K chunks per step)
            const uint32_t as[3] = {a_hi, a_hi, a_lo}, bs[3] = {b_hi, b_lo, b_hi};
#pragma unroll
            for (int pass = 0; pass < 3; ++pass)
#pragma unroll
                for (int s = 0; s < kUmK / 8; ++s)
                    um_mma(tmem, um_desc(as[pass] + 2u * s * lbo_a, lbo_a, 128),
                           um_desc(bs[pass] + 2u * s * lbo_b, lbo_b, 128), idesc, (pass | s) ? 1u : 0u);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                         : "memory");
        }
        fetch(tile + gridDim.x, rec_n, vals_n);  // in flight while the MMAs run
        {
            uint32_t done = 0;
            const uint32_t parity = (uint32_t)(it & 1);
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(bar), "r"(parity)
                    : "memory");
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

        // epilogue: accumulator rows -> g (ceil32(L) taps per unit). TMEM gives
        // lane = unit row; a per-warp shared transpose turns each 16-column
        // chunk into 8-row x 64-byte float4 stores (full sectors)
        const int lp = live ? (rec.n_t + nl - 1 + 15) & ~15 : 0;  // k_direct reads taps < L only
        float* g = reinterpret_cast<float*>(pool + rec.goff);
        const int lane = tid & 31;
        float* stg = reinterpret_cast<float*>(um_smem) + warp * (32 * 20);  // A area (free now)
        float* rg[4];
        int rlp[4];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            const int src = 8 * rr + (lane >> 2);
            rg[rr] = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(g), src));
            rlp[rr] = __shfl_sync(0xffffffffu, nt > 0 ? lp : 0, src);
        }
        const int cq = 4 * (lane & 3);
        for (int c0 = half * (N / 2); c0 < (half + 1) * (N / 2); c0 += 16) {
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                "%13, %14, %15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15])
                : "r"(trow + (uint32_t)c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int q = 0; q < 4; ++q)
                reinterpret_cast<uint4*>(stg + lane * 20)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            __syncwarp();
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const int r8 = 8 * rr + (lane >> 2);
                const float4 x = *reinterpret_cast<const float4*>(stg + r8 * 20 + cq);
                if (c0 + cq < rlp[rr]) *reinterpret_cast<float4*>(rg[rr] + c0 + cq) = x;
            }
            __syncwarp();
        }
        if (half == 0 && live && rec.n_t > kUmK) {  // wide tick profile: scalar
            const int L = rec.n_t + nl - 1;
            for (int j = 0; j < lp; ++j) {
                const int k0 = j - nl + 1 > 0 ? j - nl + 1 : 0, k1 = j < rec.n_t - 1 ? j : rec.n_t - 1;
                float sum = 0.0f;
                for (int k = k0; k <= k1; ++k) sum = __fmaf_rn(__ldg(tv + k), __ldg(&P.kern[j - k]), sum);
                g[j] = j < L ? sum : 0.0f;
            }
        }
        __syncthreads();  // the transpose staging (A lo area) is free for the next tile's operands
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        const uint32_t cols = N <= 32 ? 32u : N <= 64 ? 64u : N <= 128 ? 128u : 256u;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
    }
}


// ---- k_gprof_umma2: the same GEMM as a warp-specialised pipeline ----------
// k_gprof_umma stages a tile, multiplies, waits and drains it in turn (two CTAs
// per SM: 9 us per 128-unit tile, 18% issue-active, r2c). Here one CTA per SM
// keeps three stages in flight over the tiles of one plane:
//   warps 0-7 (producers, two groups of 4 taking alternate tiles, one unit
//     per thread): record + tick profile loads one tile ahead, TF32 hi / lo
//     split into a ring of three A operand slots;
//   warp 16 (one elected lane): the 12 MMAs of a tile into one of two
//     256-column TMEM accumulators; commits release the A slot and hand the
//     accumulator to the epilogue;
//   warps 8-15 (epilogue, two per TMEM lane quadrant, half the columns each):
//     tcgen05.ld, the per-warp transpose into full-sector float4 stores of g.
// The bound is the profile write (~111 MB per MicroBooNE event).
constexpr int kG2Slots = 3;
constexpr int kG2EpiWarp = 8, kG2MmaWarp = 16;
constexpr int kG2Threads = 32 * (kG2MmaWarp + 1);
constexpr uint32_t kG2APart = kUmM * kUmK * 4;  // 16 KB: one TF32 part of A

__device__ __forceinline__ void g2_wait(uint32_t bar, uint32_t parity)
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

__global__ void __launch_bounds__(kG2Threads, 1) k_gprof_umma2(const EventDesc ev, const UnitRec* __restrict__ recs,
                                                               uint32_t* __restrict__ pool, int N)
{
    const PlaneDesc& P = ev.p[blockIdx.y];
    if (!P.direct || P.n_units == 0) return;
    const int nl = P.n_lags;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_tiles = (int)((P.n_units + kUmM - 1) / kUmM);
    const int my_tiles = (int)blockIdx.x < n_tiles ? (n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

    // layout: B hi | B lo (N x 32 each) | A ring (kG2Slots x [hi | lo]) | epilogue staging (8 warps x 32 x 20)
    extern __shared__ __align__(128) unsigned char g2_smem[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(g2_smem);
    const uint32_t b_hi = sbase, b_lo = b_hi + (uint32_t)N * kUmK * 4;
    const uint32_t a_ring = b_lo + (uint32_t)N * kUmK * 4;
    float* stg_base = reinterpret_cast<float*>(g2_smem + 2 * (size_t)N * kUmK * 4 + (size_t)kG2Slots * 2 * kG2APart);
    __shared__ __align__(8) unsigned long long s_afull[kG2Slots], s_aempty[kG2Slots], s_accf[2], s_acce[2];
    __shared__ uint32_t s_tmem;
    const uint32_t a_afull = (uint32_t)__cvta_generic_to_shared(s_afull), a_aempty = (uint32_t)__cvta_generic_to_shared(s_aempty);
    const uint32_t a_accf = (uint32_t)__cvta_generic_to_shared(s_accf), a_acce = (uint32_t)__cvta_generic_to_shared(s_acce);

    if (warp == kG2MmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < kG2Slots; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(a_afull + 8u * i));  // one producer group
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a_aempty + 8u * i));
        }
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a_accf + 8u * i));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(a_acce + 8u * i));  // the epilogue warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // B = the plane's Toeplitz kernel, hi and lo TF32 parts: row n, taps k..k+3
    for (int i = tid; i < N * (kUmK / 4); i += kG2Threads) {
        const int n = i % N, kc = i / N;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float v = __ldg(&P.kern[n - (4 * kc + q)]);  // zero-padded both sides
            hi[q] = um_tf32(v);
            lo[q] = um_tf32(v - __uint_as_float(hi[q]));
        }
        const uint32_t o = um_off(n, kc, N);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b_hi + o), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]),
                     "r"(hi[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b_lo + o), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]),
                     "r"(lo[3]));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    // the records and tick profiles come from the previous kernel (k_sample_off);
    // with a programmatic launch the setup above overlapped its tail
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the sampler has completed: a programmatically launched successor
    // (k_direct) may now run its profile-independent prologue
    asm volatile("griddepcontrol.launch_dependents;");

    if (warp < kG2EpiWarp) {
        // ---- producers: group gp takes the CTA's tiles j = gp mod 2; thread
        // row = the unit of the tile; loads one tile ahead
        const int row = tid & (kUmM - 1), gp = warp >> 2;
        // the record of tile j, then its tick profile (loaded a group step
        // after its record: neither load chain stalls the thread)
        auto fetch_rec = [&](int j) {
            const int tile = (int)blockIdx.x + j * (int)gridDim.x;
            const uint32_t ul = (uint32_t)tile * kUmM + (uint32_t)row;
            UnitRec rec{};
            rec.w0 = -1;
            if (j < my_tiles && ul < P.n_units) rec = recs[P.unit_base + ul];
            return rec;
        };
        auto fetch_tv = [&](const UnitRec& rec, float* vals) {
            const bool ok = rec.w0 >= 0 && rec.n_t <= kUmK;
            const float* t = reinterpret_cast<const float*>(pool + rec.pool + (uint32_t)(rec.n_w + unit_n_eff(P, rec.n_w)));
#pragma unroll
            for (int k = 0; k < kUmK; ++k) vals[k] = ok && k < rec.n_t ? __ldg(t + k) : 0.0f;
#ifdef WS_G2_NOLOAD  // (timing decomposition only: results wrong)
            if (rec.n_t != 12345)
#pragma unroll
                for (int k = 0; k < kUmK; ++k) vals[k] = k < 8 ? 1.0f : 0.0f;
#endif
        };
        float vn[kUmK];
        fetch_tv(fetch_rec(gp), vn);
        UnitRec rn = fetch_rec(gp + 2);
        for (int j = gp; j < my_tiles; j += 2) {
            float v[kUmK];
#pragma unroll
            for (int k = 0; k < kUmK; ++k) v[k] = vn[k];
            fetch_tv(rn, vn);       // the group's next tile, in flight
            rn = fetch_rec(j + 4);  // and the record after it
            const uint32_t slot = (uint32_t)j % kG2Slots, use = (uint32_t)j / kG2Slots;
            if (use > 0) g2_wait(a_aempty + 8u * slot, (use - 1) & 1u);
            const uint32_t ah = a_ring + slot * 2u * kG2APart, al = ah + kG2APart;
#pragma unroll
            for (int kq = 0; kq < kUmK / 4; ++kq) {
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    hi[q] = um_tf32(v[4 * kq + q]);
                    lo[q] = um_tf32(v[4 * kq + q] - __uint_as_float(hi[q]));
                }
                const uint32_t o = um_off(row, kq, kUmM);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ah + o), "r"(hi[0]), "r"(hi[1]),
                             "r"(hi[2]), "r"(hi[3]));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(al + o), "r"(lo[0]), "r"(lo[1]),
                             "r"(lo[2]), "r"(lo[3]));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a_afull + 8u * slot) : "memory");
        }
    } else if (warp == kG2MmaWarp) {
        // ---- MMA issuer: 3 passes x 4 K steps per tile (hi.hi + hi.lo + lo.hi)
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kUmM >> 4) << 24);
        const uint32_t lbo_a = (kUmM / 8) * 128, lbo_b = (uint32_t)(N / 8) * 128;
        for (int j = 0; j < my_tiles; ++j) {
            const uint32_t slot = (uint32_t)j % kG2Slots, use = (uint32_t)j / kG2Slots, ab = (uint32_t)j & 1u;
            g2_wait(a_afull + 8u * slot, use & 1u);
            if (j >= 2) g2_wait(a_acce + 8u * ab, (uint32_t)((j >> 1) - 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t ah = a_ring + slot * 2u * kG2APart, al = ah + kG2APart;
            if (elect_sync_one()) {
                const uint32_t as[3] = {ah, ah, al}, bs[3] = {b_hi, b_lo, b_hi};
#pragma unroll
                for (int pass = 0; pass < 3; ++pass)
#pragma unroll
                    for (int k = 0; k < kUmK / 8; ++k)
                        um_mma(tmem + ab * 256u, um_desc(as[pass] + 2u * k * lbo_a, lbo_a, 128),
                               um_desc(bs[pass] + 2u * k * lbo_b, lbo_b, 128), idesc, (pass | k) ? 1u : 0u);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 a_aempty + 8u * slot)
                             : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 a_accf + 8u * ab)
                             : "memory");
            }
            __syncwarp();
        }
    } else {
        // ---- epilogue: warp 8 + 4 half + q drains lanes 32 q.. (units) x columns [half N/2, (half+1) N/2)
        const int q = warp & 3, half = (warp - kG2EpiWarp) >> 2;
        float* stg = stg_base + (warp - kG2EpiWarp) * (32 * 20);
        const int cq = 4 * (lane & 3);
        auto fetch_rec = [&](int j) {
            const uint32_t ul = (uint32_t)((int)blockIdx.x + j * (int)gridDim.x) * kUmM + (uint32_t)(32 * q + lane);
            UnitRec rec{};
            rec.w0 = -1;
            if (j < my_tiles && ul < P.n_units) rec = recs[P.unit_base + ul];
            return rec;
        };
        UnitRec rn = fetch_rec(0);
        for (int j = 0; j < my_tiles; ++j) {
            const uint32_t ab = (uint32_t)j & 1u;
            const UnitRec rec = rn;
            rn = fetch_rec(j + 1);  // in flight while this tile drains
            const bool live = rec.w0 >= 0;
            const int nt = live && rec.n_t <= kUmK ? rec.n_t : 0;
            const int lp = live ? (rec.n_t + nl - 1 + 15) & ~15 : 0;  // k_direct reads taps < L only
            float* g = reinterpret_cast<float*>(pool + rec.goff);
            float* rg[4];
            int rlp[4];
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const int src = 8 * rr + (lane >> 2);
                rg[rr] = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(g), src));
                rlp[rr] = __shfl_sync(0xffffffffu, nt > 0 ? lp : 0, src);
            }
            g2_wait(a_accf + 8u * ab, (uint32_t)(j >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + ab * 256u;
            for (int c0 = half * (N / 2); c0 < (half + 1) * (N / 2); c0 += 16) {
                uint32_t v[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                    "%13, %14, %15}, [%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15])
                    : "r"(trow + (uint32_t)c0));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int qq = 0; qq < 4; ++qq)
                    reinterpret_cast<uint4*>(stg + lane * 20)[qq] =
                        make_uint4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
                __syncwarp();
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    const int r8 = 8 * rr + (lane >> 2);
                    const float4 x = *reinterpret_cast<const float4*>(stg + r8 * 20 + cq);
#ifndef WS_G2_NOSTORE  // (timing decomposition only: results wrong)
                    if (c0 + cq < rlp[rr]) __stcs(reinterpret_cast<float4*>(rg[rr] + c0 + cq), x);
#else
                    if (c0 + cq < rlp[rr] && x.x == 12345.0f) __stcs(reinterpret_cast<float4*>(rg[rr] + c0 + cq), x);
#endif
                }
                __syncwarp();
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a_acce + 8u * ab) : "memory");
            if (half == 0 && live && rec.n_t > kUmK) {  // wide tick profile: scalar
                const float* tv = reinterpret_cast<const float*>(pool + rec.pool + (uint32_t)(rec.n_w + unit_n_eff(P, rec.n_w)));
                const int L = rec.n_t + nl - 1;
                for (int jj = 0; jj < lp; ++jj) {
                    const int k0 = jj - nl + 1 > 0 ? jj - nl + 1 : 0, k1 = jj < rec.n_t - 1 ? jj : rec.n_t - 1;
                    float sum = 0.0f;
                    for (int k = k0; k <= k1; ++k) sum = __fmaf_rn(__ldg(tv + k), __ldg(&P.kern[jj - k]), sum);
                    g[jj] = jj < L ? sum : 0.0f;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == kG2MmaWarp) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

}  // namespace wsb

// N (output taps per unit) of the UMMA path for the event, or 0 when a plane's
// kernel is too long for it (then k_gprof runs)
extern "C" int wsb_gprof_umma_n(const wsb::EventDesc& ev)
{
    int max_lags = 0;
    for (int i = 0; i < ev.n_planes; ++i)
        if (ev.p[i].direct) max_lags = max_lags > ev.p[i].n_lags ? max_lags : ev.p[i].n_lags;
    const int N = (max_lags + 31 + 31) & ~31;
    return N <= 256 ? N : 0;
}

extern "C" cudaError_t wsb_launch_gprof_umma(const wsb::EventDesc& ev, const wsb::UnitRec* recs, uint32_t* pool,
                                             int N, cudaStream_t s, int pdl)
{
    uint32_t max_units = 0;
    for (int i = 0; i < ev.n_planes; ++i)
        if (ev.p[i].direct) max_units = max_units > ev.p[i].n_units ? max_units : ev.p[i].n_units;
    if (max_units == 0) return cudaSuccess;
    const size_t smem = (size_t)2 * wsb::kUmK * 4 * (wsb::kUmM + (size_t)N);
    static std::atomic<unsigned long long> ready{0};  // per-device attribute setup (idempotent)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(ready & (1ull << dev))) {
        e = cudaFuncSetAttribute(wsb::k_gprof_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
        if (e != cudaSuccess) return e;
        ready |= 1ull << dev;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned tiles = (max_units + wsb::kUmM - 1) / wsb::kUmM;
    const char* v1 = getenv("WS_GPROF_V1");  // 1: the one-tile-at-a-time kernel (A/B, tests)
    if (!(v1 && atoi(v1) == 1)) {
        static std::atomic<unsigned long long> ready2{0};
        const size_t smem2 = (size_t)2 * wsb::kUmK * 4 * N + (size_t)wsb::kG2Slots * 2 * wsb::kG2APart +
                             (size_t)8 * 32 * 20 * 4;
        if (!(ready2 & (1ull << dev))) {
            e = cudaFuncSetAttribute(wsb::k_gprof_umma2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            if (e != cudaSuccess) return e;
            ready2 |= 1ull << dev;
        }
        // one CTA per SM, the SMs split over the plane descriptors
        const unsigned per_plane = std::max(1u, (unsigned)sms / (unsigned)ev.n_planes);
        const dim3 grid2(std::min(tiles, per_plane), (unsigned)ev.n_planes);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid2;
        cfg.blockDim = dim3(wsb::kG2Threads);
        cfg.dynamicSmemBytes = smem2;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, wsb::k_gprof_umma2, ev, recs, pool, N);
    }
    // persistent: two CTAs per SM over the planes (B staged once per CTA)
    const unsigned per_plane = std::max(1u, (unsigned)(2 * sms) / (unsigned)ev.n_planes);
    const dim3 grid(std::min(tiles, per_plane), (unsigned)ev.n_planes);
    if (!pdl) {
        wsb::k_gprof_umma<<<grid, wsb::kUmThreads, smem, s>>>(ev, recs, pool, N);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(wsb::kUmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, wsb::k_gprof_umma, ev, recs, pool, N);
}
