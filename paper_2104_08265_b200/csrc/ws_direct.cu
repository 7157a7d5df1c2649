// Time-domain ("direct") scatter + convolution (k_direct), the alternative
// to the row FFT of k_conv for planes whose depo load is light relative to
// their cell count (ws_api.cu routes each plane of a call).
//
// The reference convolves the whole charge grid with the response
// (convolve, spectral.cpp:141-175): M[w] = sum_dw ww[dw] (S[w - dw] (*) k)
// circularly along ticks, with S a sum of separable depo patches
// S = sum_d a_d wv_d[w] tv_d[t] (sample_patch, rasterize.cpp:66-120). By
// linearity, M[w, t] = sum_d a_d eff_d[w] g_d[t - t0_d - lo_lag] with
// eff_d the stencilled wire profile and g_d = tv_d (*) k the depo's tick
// profile convolved with the combined time kernel (L = n_t + n_lags - 1
// taps, computed once per depo by k_gprof_umma and shared by all its wire rows).
//
// One CTA (640 threads, two per SM) owns a tile of kTileRows wire rows x
// kTileTicks ticks of the frame in shared memory as int32 fixed point. The
// sampler (fixed-capacity lists) or k_fill_bands (CSR lists) has listed the
// tile's depos (tick span, profile offset, max|g|, per-row coefficients). The CTA
// stages the list, bounds every row (per 64-tick segment sum of |terms|,
// largest term; one thread per entry x row) to fix a per-row power-of-two
// scale, then one warp per entry loads the depo's profile into registers
// (the next entry's load in flight behind the current one's atomics) and adds
// round(c_w g_j) to every covered row with native shared atomics. The
// integer sums are exact, so the frame is bitwise reproducible for any
// schedule. Lanes whose tick falls outside the window write to a row margin
// that is discarded. Work ~ depos x rows x L instead of cells x log(ticks).
// Launched programmatically behind the profiles kernel: everything before the
// accumulation (zeroing, staging, bounds) overlaps its tail.
#include "ws_common.cuh"

#include <algorithm>
#include <atomic>

namespace wsb {

constexpr int kQ = 5;                          // profile taps per lane in registers: L <= 160 fast path
constexpr int kSlot = 32 * kQ;                 // taps of the register fast path
constexpr int kMargin = kSlot;                 // discard margins either side of every row
constexpr int kRowStride = kMargin + kTileTicks + kMargin;  // ints per tile row
#ifndef WS_DIRECT_THREADS
#define WS_DIRECT_THREADS 640
#endif
#ifndef WS_DIRECT_MINB
#define WS_DIRECT_MINB 2
#endif
constexpr int kDirectThreads = WS_DIRECT_THREADS;  // x kDirectMinB CTAs per SM
constexpr int kDirectMinB = WS_DIRECT_MINB;

// Fixed-point term round(c g). WS_DIRECT_MAGIC: one FFMA with the magic
// 1.5 * 2^23 (the mantissa bits hold the rounded value; needs |c g| < 2^22,
// so single terms cap the row scale) + one IADD; WS_DIRECT_F2I: FMUL +
// F2I.RNI on the quarter-rate conversion pipe (r1j: 45% busy, 283 us);
// default: one DFMA (below; 259 us). The last two allow any term the
// segment sums allow, so the scale is set by those alone.
#if defined(WS_DIRECT_MAGIC)
constexpr bool kTermBudget = true;
using gtap_t = float;
__device__ __forceinline__ int fix_rn(float c, float g)
{
    return __float_as_int(__fmaf_rn(c, g, 12582912.0f)) - 0x4B400000;
}
#elif defined(WS_DIRECT_F2I)
constexpr bool kTermBudget = false;
using gtap_t = float;
__device__ __forceinline__ int fix_rn(float c, float g) { return __float2int_rn(c * g); }
#else
// default: one DFMA with the magic 1.5 * 2^52: the low word of the sum is
// round(c g) of the EXACT product (24 x 24 bits fit the 53-bit mantissa) for
// any |c g| < 2^51. B200's FP64 pipe runs at half the FP32 rate, so a term
// costs one half-rate DFMA instead of an FMUL plus a quarter-rate F2I; the
// taps are widened once per entry and the coefficient once per row.
constexpr bool kTermBudget = false;
using gtap_t = double;
__device__ __forceinline__ int fix_rn_d(double c, double g)
{
    return __double2loint(__fma_rn(c, g, 6755399441055744.0));
}
__device__ __forceinline__ int fix_rn(float c, float g) { return fix_rn_d((double)c, (double)g); }
#endif

__device__ __forceinline__ void red_shared(uint32_t saddr, int v)
{
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

// red.shared with a compile-time byte offset folded into the instruction
template <int OFF>
__device__ __forceinline__ void red_shared_off(uint32_t saddr, int v)
{
    asm volatile("red.shared.add.s32 [%0+%2], %1;" ::"r"(saddr), "r"(v), "n"(OFF) : "memory");
}

// Rows [rlo, rhi) of one profile (gv: taps lane + 32 q, q < NQ; a0: the
// lane's byte address of tap 0 in row 0): per row one LDS of the
// coefficient, one address add, then per tap one FFMA rounding + one IADD +
// one RED with the tap offset as an instruction immediate.
template <int NQ>
__device__ __forceinline__ void scatter_rows(const float* __restrict__ c, int rlo, int rhi, uint32_t a0,
                                             const gtap_t* gv)
{
    uint32_t ar = a0 + (uint32_t)rlo * (4u * kRowStride);
#pragma unroll 1
    for (int r = rlo; r < rhi; ++r, ar += 4u * kRowStride) {
#if defined(WS_DIRECT_MAGIC) || defined(WS_DIRECT_F2I)
        const float cs = c[r];
#define WS_TERM(q) fix_rn(cs, gv[q])
#else
        const double cs = (double)c[r];
#define WS_TERM(q) fix_rn_d(cs, gv[q])
#endif
        red_shared_off<0>(ar, WS_TERM(0));
        if constexpr (NQ > 1) red_shared_off<128>(ar, WS_TERM(1));
        if constexpr (NQ > 2) red_shared_off<256>(ar, WS_TERM(2));
        if constexpr (NQ > 3) red_shared_off<384>(ar, WS_TERM(3));
        if constexpr (NQ > 4) red_shared_off<512>(ar, WS_TERM(4));
#undef WS_TERM
    }
}

// The same with the row loop unrolled for a known row count (the common
// profile lengths): per row one LDS with an immediate offset and one
// widening, then the taps' DFMA + RED with immediate row / tap offsets; no
// loop counter, no per-row address arithmetic.
#if !defined(WS_DIRECT_MAGIC) && !defined(WS_DIRECT_F2I)
template <int NQ, int R, int NR>
struct RowsUnrolled {
    static __device__ __forceinline__ void run(const float* __restrict__ c, uint32_t ar, const gtap_t* gv)
    {
        if constexpr (R < NR) {
            constexpr int RB = 4 * kRowStride * R;
            const double cs = (double)c[R];
            red_shared_off<RB>(ar, fix_rn_d(cs, gv[0]));
            if constexpr (NQ > 1) red_shared_off<RB + 128>(ar, fix_rn_d(cs, gv[1]));
            if constexpr (NQ > 2) red_shared_off<RB + 256>(ar, fix_rn_d(cs, gv[2]));
            if constexpr (NQ > 3) red_shared_off<RB + 384>(ar, fix_rn_d(cs, gv[3]));
            if constexpr (NQ > 4) red_shared_off<RB + 512>(ar, fix_rn_d(cs, gv[4]));
            RowsUnrolled<NQ, R + 1, NR>::run(c, ar, gv);
        }
    }
};
template <int NQ>
__device__ __forceinline__ void scatter_rows_unrolled(const float* __restrict__ c, int rlo, int rhi, uint32_t a0,
                                                      const gtap_t* gv)
{
    static_assert(kTileRows <= 16, "row groups of at most 8, twice");
    if (rhi - rlo > 8) {  // (16-row tiles) the first 8 rows, then the rest
        RowsUnrolled<NQ, 0, 8>::run(c + rlo, a0 + (uint32_t)rlo * (4u * kRowStride), gv);
        rlo += 8;
    }
    const uint32_t ar = a0 + (uint32_t)rlo * (4u * kRowStride);
    const float* cr = c + rlo;
    switch (rhi - rlo) {
        case 8: RowsUnrolled<NQ, 0, 8>::run(cr, ar, gv); break;
        case 7: RowsUnrolled<NQ, 0, 7>::run(cr, ar, gv); break;
        case 6: RowsUnrolled<NQ, 0, 6>::run(cr, ar, gv); break;
        case 5: RowsUnrolled<NQ, 0, 5>::run(cr, ar, gv); break;
        case 4: RowsUnrolled<NQ, 0, 4>::run(cr, ar, gv); break;
        case 3: RowsUnrolled<NQ, 0, 3>::run(cr, ar, gv); break;
        case 2: RowsUnrolled<NQ, 0, 2>::run(cr, ar, gv); break;
        default: RowsUnrolled<NQ, 0, 1>::run(cr, ar, gv); break;
    }
}
#endif

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* gptr)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

// kRO: the fused readout (noise + digitize, fp64 frame) in the frame store;
// a separate instantiation so the plain fp32 store keeps its registers
template <int NT, bool kRO>
__global__ void __launch_bounds__(NT, kDirectMinB)
k_direct(const EventDesc ev, const uint32_t* __restrict__ pool, const uint32_t* __restrict__ band_off,
         const TEnt* __restrict__ tlist)
{
    constexpr int R = kTileRows;
    constexpr int NW = NT / 32;
    static_assert(NW >= R && kSegs <= 32 && (R & (R - 1)) == 0, "one warp per row computes the scales");
    constexpr int kRShift = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
    const uint32_t gb = blockIdx.x;
    const PlaneDesc& P = ev.p[band_plane(ev, gb)];
    // the next call's sampler may launch now (it waits for this grid before
    // touching the pool, the records or the tile lists)
    asm volatile("griddepcontrol.launch_dependents;");
    if (!P.direct) return;
    const bool fixed = ev.tile_cap != 0;  // fixed-capacity tile lists filled by the sampler
    if (!fixed && __ldg(&band_off[ev.total_bands]) > ev.list_cap) return;
    const int tile = (int)(gb - P.band_base);
    const int W = P.W, N = P.N;
    const int rb = tile / P.n_windows, win = tile - rb * P.n_windows;
    const int r0 = rb * R, nr = min(R, W - r0);
    const int ws = win * kTileTicks, wlen = min(kTileTicks, N - ws);
    const int cap = (int)P.direct_cap;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // layout: fixed-point rows [R][kRowStride] (the first kMargin ints of a
    // row are the discard margin) | segment bounds [R][kSegs] | staged entries [cap]
    extern __shared__ __align__(16) unsigned char smem[];
    int* acc = reinterpret_cast<int*>(smem);
    unsigned* segb = reinterpret_cast<unsigned*>(acc + R * kRowStride);
    TEnt* ent = reinterpret_cast<TEnt*>(segb + R * kSegs);
    __shared__ unsigned s_tmax[R];  // max single term per row (float bits)
    __shared__ float s_scale[R], s_inv[R];
    __shared__ int s_ovf;

    const uint32_t sacc = (uint32_t)__cvta_generic_to_shared(acc);
    {
        constexpr int kZ = R * kRowStride / 4;  // 16-byte words of the rows
#pragma unroll 4
        for (int i = tid; i < kZ; i += NT)
            asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(sacc + 16u * (uint32_t)i), "r"(0) : "memory");
        for (int i = tid; i < R * kSegs; i += NT) segb[i] = 0u;
        if (tid < R) s_tmax[tid] = 0u;
        if (tid == 0) s_ovf = 0;
    }

    const uint32_t lo = fixed ? gb * ev.tile_cap : __ldg(&band_off[gb]);
    const int n = fixed ? (int)min(ev.tile_count[gb], ev.tile_cap) : (int)(__ldg(&band_off[gb + 1]) - lo);
    if (fixed) tlist = ev.tiles;
    const uint32_t s_ent = (uint32_t)__cvta_generic_to_shared(ent);

    // entries [c0, c0 + cnt) of the tile list -> staging (coalesced async copies)
    auto stage = [&](int c0, int cnt) {
        __syncthreads();
        const int4* src = reinterpret_cast<const int4*>(tlist + lo + c0);
        constexpr int kV = sizeof(TEnt) / 16;
        for (int i = tid; i < cnt * kV; i += NT) cp_async16(s_ent + 16u * (uint32_t)i, src + i);
        cp_commit();
        cp_wait<0>();
        __syncthreads();
    };

    // the first chunk's profiles -> L2 while the bounds and scales are
    // worked out (the warps' one-entry-ahead loads then hit L2, not DRAM)
#ifndef WS_DIRECT_NOPF
    if (n > 0) {
        const int cnt0 = min(cap, n);
        stage(0, cnt0);
        for (int i = tid; i < cnt0 * kQ; i += NT) {
            const int e = i / kQ, q = i - e * kQ;
            const TEnt& d = ent[e];
            if (32 * q < (int)(d.tsL >> 16))
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const float*>(pool + d.goff) + 32 * q));
        }
    }
#endif
    // bounds of every row, one thread per (entry, row): per 64-tick segment
    // of the window the sum of |a eff g| in units of 2^ue (rounded up) over the
    // entries whose span touches it, and the largest single term; ue grows if
    // a 32-bit bound overflows (extreme charges only)
    int ue = 0;
#pragma unroll 1
#ifdef WS_DIRECT_NOBOUNDS  // (timing decomposition only: results wrong)
    for (; false;) {
#else
    for (;;) {
#endif
#pragma unroll 1
        for (int c0 = 0; c0 < n; c0 += cap) {
            const int cnt = min(cap, n - c0);
#ifndef WS_DIRECT_NOPF
            if (n > cap && !(c0 == 0 && ue == 0)) stage(c0, cnt);  // (chunk 0 staged above)
#else
            if (n > cap || (c0 == 0 && ue == 0)) stage(c0, cnt);
#endif
#pragma unroll 1
            for (int i = tid; i < cnt * R; i += NT) {
                const TEnt& d = ent[i >> kRShift];
                const int r = i & (R - 1);
                const float t = __fmul_ru(fabsf(d.c[r]), d.gbound);  // >= every |a eff g| of the row
                if (!(t > 0.0f)) continue;
                const float tu = ceilf(ldexpf(t, -ue));
                if (tu >= 4294967296.0f) {
                    s_ovf = 1;
                    continue;
                }
                const unsigned v = (unsigned)tu;
                const int ts = (int)(d.tsL & 0xffffu), L = (int)(d.tsL >> 16);
                bool ovf = false;
                auto piece = [&](int x, int y, unsigned m) {  // global ticks [x, y)
                    const int a0 = max(x, ws) - ws, e0 = min(y, ws + wlen) - ws;
                    for (int sg = a0 >> kSegShiftD; a0 < e0 && sg <= ((e0 - 1) >> kSegShiftD); ++sg)
                        ovf |= atomicAdd(&segb[r * kSegs + sg], m) > 0xffffffffu - m;
                };
                if (L >= N) {  // the profile wraps onto itself: each wrap counted
                    const unsigned long long m = (unsigned long long)v * (unsigned long long)(L / N + 1);
                    ovf |= m > 0xffffffffull;
                    piece(0, N, (unsigned)min(m, 0xffffffffull));
                } else {
                    piece(ts, min(ts + L, N), v);
                    if (ts + L > N) piece(0, ts + L - N, v);
                }
                if (ue == 0) atomicMax(&s_tmax[r], __float_as_uint(t));
                if (ovf) s_ovf = 1;
            }
        }
        __syncthreads();
        if (!s_ovf) break;
        ue += 16;
        for (int i = tid; i < R * kSegs; i += NT) segb[i] = 0u;
        __syncthreads();
        if (tid == 0) s_ovf = 0;
    }
    // per-row scale 2^sh: the largest segment bound below 2^29 (and, with the
    // one-FFMA rounding, every single term below 2^22), so partial sums
    // (bound + rounding of <= 2^28 terms) stay inside int32
    if (warp < R) {
        unsigned mx = lane < kSegs ? segb[warp * kSegs + lane] : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) {
            const int bits = 32 - __clz(mx) + ue;  // bound < 2^bits
            int sh = 29 - bits;
            const float tm = __uint_as_float(s_tmax[warp]);
            if (kTermBudget && tm > 0.0f) sh = min(sh, 21 - ilogbf(tm));  // tm < 2^(e+1): tm 2^sh < 2^22 (fix_rn range)
            s_scale[warp] = ldexpf(1.0f, sh);
            s_inv[warp] = ldexpf(1.0f, -sh);
        }
    }
    __syncthreads();
    if (fixed && tid == 0) ev.tile_count[gb] = 0;  // every thread has read it: zero for the next call

    // the profiles come from the previous kernel (k_gprof_umma): with a
    // programmatic launch everything above overlapped its tail
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // accumulate, one warp per entry: lane j adds round(c_w g[j] scale_w) to
    // tick ts + j of every covered row (consecutive lanes -> consecutive
    // banks); ticks outside the window go to the lane's margin slot. Each
    // warp holds its entry's profile in registers, the next one in flight.
    constexpr uint32_t row_bytes = 4u * kRowStride;

    auto scatter = [&](const TEnt& d, const gtap_t* gv) {  // d: staged, coefficients pre-scaled
        const uint32_t tsL = d.tsL, rows = d.rows;
        const int ts = (int)(tsL & 0xffffu), L = (int)(tsL >> 16);
        const int rlo = (int)(rows & 0xffu), rhi = (int)(rows >> 8);
        if (L <= kSlot && ts + L <= N) {
            // fast path (no circular wrap): tap j of the profile lands on
            // window tick ts - ws + j; taps outside the window land in the
            // row margins, taps past L add 0 (g is 0-filled to 32 k taps)
            const uint32_t a0 = sacc + 4u * (uint32_t)(kMargin + ts - ws + lane);
            static_assert(kQ == 5, "scatter_rows handles up to 5 taps per lane");
            switch ((L + 31) >> 5) {  // 32-tap groups in g's 0-filled length (warp-uniform)
#if !defined(WS_DIRECT_MAGIC) && !defined(WS_DIRECT_F2I) && !defined(WS_DIRECT_ROWLOOP)
                case 5: scatter_rows_unrolled<5>(d.c, rlo, rhi, a0, gv); break;
                case 4: scatter_rows_unrolled<4>(d.c, rlo, rhi, a0, gv); break;
#else
                case 5: scatter_rows<5>(d.c, rlo, rhi, a0, gv); break;
                case 4: scatter_rows<4>(d.c, rlo, rhi, a0, gv); break;
#endif
                case 3: scatter_rows<3>(d.c, rlo, rhi, a0, gv); break;
                case 2: scatter_rows<2>(d.c, rlo, rhi, a0, gv); break;
                default: scatter_rows<1>(d.c, rlo, rhi, a0, gv); break;
            }
        } else {
            // long profiles / spans wrapping past the row end: 32-tap steps
            // from global memory, general wrap
            const float* g = reinterpret_cast<const float*>(pool + d.goff);
#pragma unroll 1
            for (int base = 0; base < L; base += 32) {
                const int j = base + lane;
                const int loc = (ts + j) % N - ws;
                if (j < L && (unsigned)loc < (unsigned)wlen) {
                    const float gj = __ldg(&g[j]);
                    for (int r = rlo; r < rhi; ++r) {
                        const float cs = d.c[r];
                        if (cs != 0.0f) red_shared(sacc + (uint32_t)r * row_bytes + 4u * (kMargin + loc), fix_rn(cs, gj));
                    }
                }
            }
        }
    };

#pragma unroll 1
#ifdef WS_DIRECT_NOLOOP  // (timing decomposition only: results wrong)
    for (int c0 = 0; c0 < 0; c0 += cap) {
#else
    for (int c0 = 0; c0 < n; c0 += cap) {
#endif
        const int cnt = min(cap, n - c0);
        if (n > cap) stage(c0, cnt);
        // coefficients -> fixed-point units of their row
        for (int i = tid; i < cnt * R; i += NT) ent[i >> kRShift].c[i & (R - 1)] *= s_scale[i & (R - 1)];
        __syncthreads();
        // profile of local entry e -> registers (tap lane + 32 q < L, 0 past
        // the profile); one entry ahead
        auto load_g = [&](int e, float* gv) {
            int lc = 0;
            const float* src = nullptr;
            if (e < cnt) {
                const TEnt& d = ent[e];
                lc = (int)(d.tsL >> 16) - lane;  // tap lane + 32 q exists iff 32 q < L - lane
                src = reinterpret_cast<const float*>(pool + d.goff) + lane;
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) gv[q] = 32 * q < lc ? __ldg(src + 32 * q) : 0.0f;
        };
        float gn[kQ];
        load_g(warp, gn);
#pragma unroll 1
        for (int e = warp; e < cnt; e += NW) {
            gtap_t gv[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) gv[q] = (gtap_t)gn[q];
            load_g(e + NW, gn);
#ifndef WS_DIRECT_NOSCATTER  // (timing decomposition only: results wrong)
            scatter(ent[e], gv);
#else
            if (gv[0] == (gtap_t)12345.0) scatter(ent[e], gv);
#endif
        }
    }
    __syncthreads();

    // frame rows of the window (convolve's real part, spectral.cpp:172-173),
    // streaming stores; one flattened (row, 16-byte word) loop. With a
    // readout (ev.ro) the same words go through noise + digitize instead.
#ifdef WS_DIRECT_NOSTORE  // (timing decomposition only: results wrong)
    if (acc[tid] == 0x7fffffff) P.frame[tid] = 1.0f;
    return;
#endif
    if constexpr (kRO) {
        if ((N & 3) == 0) {
            constexpr int kW = kTileTicks / 4;
            const int wlen4 = wlen >> 2;
            for (int i = tid; i < nr * kW; i += NT) {
                const int r = i / kW, c4 = i - r * kW;
                if (c4 >= wlen4) continue;
                const int* a = acc + r * kRowStride + kMargin + 4 * c4;
                const float inv = s_inv[r];
                const float v[4] = {(float)a[0] * inv, (float)a[1] * inv, (float)a[2] * inv, (float)a[3] * inv};
                readout4(ev, P, r0 + r, ws + 4 * c4, v);
            }
        } else {  // N even or odd: tick pairs (ws is even)
            for (int r = 0; r < nr; ++r)
                for (int t = 2 * tid; t < wlen; t += 2 * NT) {
                    const int* a = acc + r * kRowStride + kMargin;
                    const bool has1 = t + 1 < wlen;
                    readout_pair(ev, P, r0 + r, ws + t, (float)a[t] * s_inv[r], has1 ? (float)a[t + 1] * s_inv[r] : 0.0f,
                                 has1);
                }
        }
    } else if ((N & 3) == 0) {  // ws is a multiple of 4 as well: whole 16-byte words
        constexpr int kW = kTileTicks / 4;
        const int wlen4 = wlen >> 2;
        for (int i = tid; i < nr * kW; i += NT) {
            const int r = i / kW, c4 = i - r * kW;  // kW a power of two: shifts
            if (c4 >= wlen4) continue;
            int4 v;
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(sacc + 4u * (uint32_t)(r * kRowStride + kMargin + 4 * c4)));
            const float inv = s_inv[r];
            __stcs(reinterpret_cast<float4*>(P.frame + (size_t)(r0 + r) * N + ws) + c4,
                   make_float4((float)v.x * inv, (float)v.y * inv, (float)v.z * inv, (float)v.w * inv));
        }
    } else {
        for (int r = 0; r < nr; ++r)
            for (int t = tid; t < wlen; t += NT)
                __stcs(P.frame + (size_t)(r0 + r) * N + ws + t, (float)acc[r * kRowStride + kMargin + t] * s_inv[r]);
    }
}

}  // namespace wsb

// Shared memory of k_direct with room for `cap` staged entries; wsb_direct_cap
// gives the cap that fills the SM (tiles with more entries are staged in chunks).
extern "C" size_t wsb_direct_smem(int cap)
{
    return sizeof(int) * wsb::kTileRows * wsb::kRowStride + sizeof(unsigned) * wsb::kTileRows * wsb::kSegs +
           sizeof(wsb::TEnt) * (size_t)cap;
}

extern "C" int wsb_direct_cap()
{
    const size_t limit = (228 * 1024) / wsb::kDirectMinB - 2 * 1024;  // kDirectMinB CTAs per SM (1 KB reserved per CTA, static smem)
    return (int)((limit - wsb_direct_smem(0)) / sizeof(wsb::TEnt));
}

extern "C" cudaError_t wsb_launch_direct(const wsb::EventDesc& ev, const uint32_t* pool, const uint32_t* band_off,
                                         const wsb::TEnt* tlist, size_t smem_bytes, cudaStream_t stream, int pdl)
{
    constexpr int NT = wsb::kDirectThreads;
    static std::atomic<unsigned long long> ready{0};  // per-device attribute setup (idempotent)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(ready & (1ull << dev))) {
        for (auto f : {wsb::k_direct<NT, false>, wsb::k_direct<NT, true>}) {
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
            if (e != cudaSuccess) return e;
            e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            if (e != cudaSuccess) return e;
        }
        ready |= 1ull << dev;
    }
    const auto KFN = ev.ro ? wsb::k_direct<NT, true> : wsb::k_direct<NT, false>;
    if (ev.total_bands == 0) return cudaSuccess;
    if (!pdl) {
        KFN<<<ev.total_bands, NT, smem_bytes, stream>>>(ev, pool, band_off, tlist);
        return cudaGetLastError();
    }
    // programmatic dependent launch: the tiles' prologue (zeroing, staging,
    // bounds) runs while the previous kernel drains; griddepcontrol.wait
    // guards the profile reads
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ev.total_bands);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, KFN, ev, pool, band_off, tlist);
}
