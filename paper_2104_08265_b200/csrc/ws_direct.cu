// Time-domain ("direct") scatter + convolution for bands whose depo load is
// light (k_direct), the sparse-event alternative to the row FFT of k_conv.
//
// The reference convolves the whole charge grid with the response
// (convolve, spectral.cpp:141-175): M[w] = sum_dw ww[dw] (S[w - dw] (*) k)
// circularly along ticks, with S a sum of separable depo patches
// S = sum_d a_d wv_d[w] tv_d[t] (sample_patch, rasterize.cpp:66-120). By
// linearity, M[w, t] = sum_d a_d eff_d[w] g_d[t - t0_d - lo_lag] with
// eff_d the stencilled wire profile and g_d = tv_d (*) k the depo's tick
// profile convolved with the combined time kernel (n_t + n_lags - 1 taps,
// computed once per depo by k_fill_bands and shared by all its wire rows).
// One CTA owns a band of kDirectRows wire rows: it stages the band's entries
// in shared memory with per-row bounds (pass 1), then accumulates every
// covering depo's scaled g into int32 fixed-point rows in shared memory (one
// FFMA rounding + one native shared atomic per tap, exact integer sums, so
// deterministic for any schedule; pass 2), then writes the frame rows. Work is ~ depos x rows x (n_t + n_lags) instead of cells x
// log(ticks), so sparse bands skip the FFT entirely; k_scan_bands routes each
// band to the cheaper kernel.
#include "ws_common.cuh"

#include <algorithm>

namespace wsb {

constexpr int kDirectRows = 4;  // == rows_per_band
constexpr int kSegShiftD = 6;   // 64-tick bound segments
constexpr int kQ = 5;           // profile taps per lane in registers (fast path: n_t + n_lags - 1 <= 160)
constexpr int kTail = 32 * kQ;  // row overhang: the fast path writes ticks [ts, ts + 160) unwrapped
constexpr int kRing = 3;        // profile fetches in flight per warp
constexpr int kDirectThreads = 512;

// One staged band-list entry (bound pass -> accumulate pass), 24 bytes.
struct __align__(8) DEnt {
    uint32_t tsL;   // first output tick ts (circular, < N) | profile length L << 16
    uint32_t goff;  // pool offset of g (16-byte aligned)
    float c[kDirectRows];  // a * eff[w] for each row of the band (0: not covered)
};

// x -> round-to-nearest int for |x| < 2^22 in one FFMA: the magic 1.5 * 2^23
// pins the exponent, so the mantissa bits hold the rounded value.
__device__ __forceinline__ int fix_rn(float c, float g)
{
    return __float_as_int(__fmaf_rn(c, g, 12582912.0f)) - 0x4B400000;
}

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

__device__ __forceinline__ void red_shared(uint32_t saddr, int v)
{
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}

// Add b to the bound of every segment the circular span [ts, ts + L) mod N
// touches; returns true if a 32-bit bound overflowed.
__device__ __forceinline__ bool add_span32(unsigned* seg, int ts, int L, int N, int nseg, unsigned b)
{
    bool ovf = false;
    auto add = [&](int s, unsigned v) { ovf |= atomicAdd(&seg[s], v) > 0xffffffffu - v; };
    if (L >= N) {  // the profile wraps onto itself: every segment, each wrap counted
        const unsigned long long m = (unsigned long long)b * (unsigned long long)(L / N + 1);
        ovf |= m > 0xffffffffull;
        for (int s = 0; s < nseg; ++s) add(s, (unsigned)min(m, 0xffffffffull));
        return ovf;
    }
    const int e = ts + L - 1;
    if (e < N) {
        for (int s = ts >> kSegShiftD; s <= (e >> kSegShiftD); ++s) add(s, b);
    } else {
        for (int s = ts >> kSegShiftD; s <= ((N - 1) >> kSegShiftD); ++s) add(s, b);
        for (int s = 0; s <= ((e - N) >> kSegShiftD); ++s) add(s, b);
    }
    return ovf;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1)
k_direct(const EventDesc ev, const uint32_t* __restrict__ pool, const uint32_t* __restrict__ band_off,
         const UnitRec* __restrict__ band_list, const uint32_t* __restrict__ map, const uint32_t* __restrict__ map_count)
{
    constexpr int R = kDirectRows;
    constexpr int NW = NT / 32;
    constexpr int D = kRing;
    if (blockIdx.x >= __ldg(map_count)) return;
    const uint32_t gb = __ldg(&map[blockIdx.x]);
    const PlaneDesc& P = ev.p[band_plane(ev, gb)];
    const int band = (int)(gb - P.band_base);
    const int W = P.W, N = P.N;
    const int r0 = band * R;
    const int nr = min(R, W - r0);
    const int Ns = (N + kTail + 3) & ~3;  // row stride: N ticks + the unwrapped overhang
    const int nseg = (N + 63) >> kSegShiftD;
    const int cap = (int)P.direct_cap;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // layout: fixed-point rows [R][Ns] (ticks N.. hold the overhang, folded
    // back before the store) | segment bounds [R][nseg] | profile ring
    // [NW][D][kTail] | staged entries [cap]
    extern __shared__ __align__(16) unsigned char smem[];
    int* acc = reinterpret_cast<int*>(smem);
    size_t off = (size_t)4 * R * Ns;
    unsigned* segb = reinterpret_cast<unsigned*>(smem + off);
    off += ((size_t)4 * R * nseg + 15) & ~(size_t)15;
    float* ring = reinterpret_cast<float*>(smem + off);
    off += sizeof(float) * NW * D * kTail;
    DEnt* ent = reinterpret_cast<DEnt*>(smem + off);
    __shared__ unsigned s_tmax[R];  // max single term per row (float bits)
    __shared__ float s_scale[R], s_inv[R];
    __shared__ int s_ovf;

    {
        int4* z = reinterpret_cast<int4*>(acc);
        for (int i = tid; i < R * Ns / 4; i += NT) z[i] = make_int4(0, 0, 0, 0);
        for (int i = tid; i < R * nseg; i += NT) segb[i] = 0u;
        if (tid < R) s_tmax[tid] = 0u;
        if (tid == 0) s_ovf = 0;
    }
    __syncthreads();

    const uint32_t lo = __ldg(&band_off[gb]);
    const int n = (int)(__ldg(&band_off[gb + 1]) - lo);
    const int lo_lag = P.lo_lag, nl = P.n_lags;

    // one band-list entry -> staged form (+ max|g| for the bounds)
    auto make_ent = [&](int e, float& gmax) {
        const UnitRec rec = band_list[lo + e];
        DEnt d;
        const int L = rec.n_t + nl - 1;
        int ts = rec.t0 + lo_lag;
        if (ts < 0) ts += N;
        d.tsL = (uint32_t)ts | ((uint32_t)L << 16);
        d.goff = unit_g_off(P, rec);
        gmax = __uint_as_float(__ldg(&pool[d.goff + L]));
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float c = 0.0f;
            if (r < nr) row_coef(P, r0 + r, false, rec, pool, c);
            d.c[r] = c;
        }
        return d;
    };

    // bound every row over all entries: per 64-tick segment the sum of
    // |a eff g| in units of 2^ue (rounded up), and the largest single term;
    // ue grows if a 32-bit segment bound overflows (extreme charges only).
    // A band that fits the staging area keeps its entries from this pass.
    int ue = 0;
#pragma unroll 1
    for (;;) {
#pragma unroll 1
        for (int e = tid; e < n; e += NT) {
            float gmax;
            const DEnt d = make_ent(e, gmax);
            if (n <= cap && ue == 0) ent[e] = d;
            const int ts = (int)(d.tsL & 0xffffu), L = (int)(d.tsL >> 16);
            bool ovf = false;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float t = fabsf(d.c[r]) * gmax;
                if (!(t > 0.0f)) continue;
                const float tu = ceilf(ldexpf(t, -ue));
                if (tu >= 4294967296.0f) {
                    ovf = true;
                    continue;
                }
                ovf |= add_span32(segb + r * nseg, ts, L, N, nseg, (unsigned)tu);
                if (ue == 0) atomicMax(&s_tmax[r], __float_as_uint(t));
            }
            if (ovf) s_ovf = 1;
        }
        __syncthreads();
        if (!s_ovf) break;
        ue += 16;
        for (int i = tid; i < R * nseg; i += NT) segb[i] = 0u;
        __syncthreads();
        if (tid == 0) s_ovf = 0;
        __syncthreads();
    }
    // per-row scale 2^sh: every single term below 2^21 (one-FFMA rounding,
    // fix_rn) and the largest segment bound below 2^29, so partial sums
    // (bound + rounding of <= 2^28 terms) stay inside int32
    if (warp < nr) {
        unsigned mx = 0u;
        for (int s = lane; s < nseg; s += 32) mx = max(mx, segb[warp * nseg + s]);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) {
            const int bits = 32 - __clz(mx) + ue;  // bound < 2^bits
            int sh = 29 - bits;
            const float tm = __uint_as_float(s_tmax[warp]);
            if (tm > 0.0f) sh = min(sh, 20 - ilogbf(tm));  // tm < 2^(e+1): tm 2^sh < 2^21
            s_scale[warp] = ldexpf(1.0f, sh);
            s_inv[warp] = ldexpf(1.0f, -sh);
        }
    }
    __syncthreads();
    float scale[R];
#pragma unroll
    for (int r = 0; r < R; ++r) scale[r] = s_scale[r];

    // accumulate, one warp per entry: lane j adds a eff[w] g[j] to tick ts + j
    // of every covered row (consecutive lanes -> consecutive banks). Each
    // warp streams its entries' profiles through a D-deep cp.async ring in
    // shared memory, so D profile fetches per warp are in flight.
    const uint32_t sacc = (uint32_t)__cvta_generic_to_shared(acc);
    const uint32_t row_bytes = 4u * (uint32_t)Ns;
    float* my_ring = ring + (size_t)warp * D * kTail;
    const uint32_t s_ring = (uint32_t)__cvta_generic_to_shared(my_ring);

    auto scatter = [&](const DEnt& d, const float* gv) {
        const int ts = (int)(d.tsL & 0xffffu), L = (int)(d.tsL >> 16);
        float cs[R];
#pragma unroll
        for (int r = 0; r < R; ++r) cs[r] = d.c[r] * scale[r];
        if (L <= kTail) {
            // fast path: ticks ts + j, j < 160, unwrapped into the row
            // overhang; lanes past the profile add 0 (their gv is 0)
            const uint32_t a0 = sacc + 4u * (uint32_t)(ts + lane);
            const bool q4 = L > 32 * (kQ - 1);  // warp-uniform
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (cs[r] == 0.0f) continue;  // warp-uniform
                const uint32_t ar = a0 + (uint32_t)r * row_bytes;
#pragma unroll
                for (int q = 0; q < kQ - 1; ++q) red_shared(ar + 128u * q, fix_rn(cs[r], gv[q]));
                if (q4) red_shared(ar + 128u * (kQ - 1), fix_rn(cs[r], gv[kQ - 1]));
            }
        } else {
            // long profiles: 32-tap steps from global memory, general wrap
            const float* g = reinterpret_cast<const float*>(pool + d.goff);
#pragma unroll 1
            for (int base = 0; base < L; base += 32) {
                const int j = base + lane;
                if (j < L) {
                    const float gj = __ldg(&g[j]);
                    const uint32_t t = (uint32_t)((ts + j) % N);
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (cs[r] != 0.0f) red_shared(sacc + (uint32_t)r * row_bytes + 4u * t, fix_rn(cs[r], gj));
                }
            }
        }
    };

#pragma unroll 1
    for (int c0 = 0; c0 < n; c0 += cap) {
        const int cnt = min(cap, n - c0);
        if (n > cap) {  // restage this chunk (bands beyond the staging capacity)
            __syncthreads();
            for (int e = tid; e < cnt; e += NT) {
                float gmax;
                ent[e] = make_ent(c0 + e, gmax);
            }
            __syncthreads();
        }
        // profile fetch of local entry e into ring slot s (one commit group)
        auto fetch = [&](int e, int s) {
            if (e < cnt) {
                const DEnt& d = ent[e];
                const int n4 = min(((int)(d.tsL >> 16) + 3) >> 2, kTail / 4);
                const float* src = reinterpret_cast<const float*>(pool + d.goff);
                for (int i = lane; i < n4; i += 32) cp_async16(s_ring + 4u * (uint32_t)(s * kTail + 4 * i), src + 4 * i);
            }
            cp_commit();
        };
#pragma unroll
        for (int k = 0; k < D; ++k) fetch(warp + NW * k, k);
        int s = 0;
#pragma unroll 1
        for (int e = warp; e < cnt; e += NW) {
            cp_wait<D - 1>();
            __syncwarp();
            const DEnt d = ent[e];
            const int L = (int)(d.tsL >> 16);
            float gv[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const int j = lane + 32 * q;
                gv[q] = j < L ? my_ring[s * kTail + j] : 0.0f;
            }
            __syncwarp();
            fetch(e + NW * D, s);
            s = s + 1 == D ? 0 : s + 1;
            scatter(d, gv);
        }
        cp_wait<0>();
    }
    __syncthreads();
    // fold the overhang back onto the row start (circular wrap, exact)
    if (N >= kTail) {
        for (int i = tid; i < R * kTail; i += NT) {
            const int r = i / kTail, t = i - r * kTail;
            acc[r * Ns + t] += acc[r * Ns + N + t];
        }
    } else if (tid < R) {  // rows shorter than the overhang (tiny grids)
        for (int t = 0; t < kTail; ++t) acc[tid * Ns + t % N] += acc[tid * Ns + N + t];
    }
    __syncthreads();

    // frame rows (convolve's real part, spectral.cpp:172-173), streaming stores
    for (int r = 0; r < nr; ++r) {
        const float inv = s_inv[r];
        const int* row = acc + r * Ns;
        float* frow = P.frame + (size_t)(r0 + r) * N;
        if ((N & 3) == 0) {
            const int4* a4 = reinterpret_cast<const int4*>(row);
            float4* f4 = reinterpret_cast<float4*>(frow);
            for (int i = tid; i < N / 4; i += NT) {
                const int4 v = a4[i];
                __stcs(&f4[i], make_float4((float)v.x * inv, (float)v.y * inv, (float)v.z * inv, (float)v.w * inv));
            }
        } else {
            for (int t = tid; t < N; t += NT) __stcs(&frow[t], (float)row[t] * inv);
        }
    }
}

}  // namespace wsb

// Shared memory of k_direct for padded_ticks N with room for `cap` staged
// entries; wsb_direct_cap gives the cap that fills the SM (bands with more
// entries are staged in chunks).
extern "C" size_t wsb_direct_smem(int N, int cap)
{
    const size_t Ns = ((size_t)N + wsb::kTail + 3) & ~(size_t)3;
    const size_t nseg = ((size_t)N + 63) >> wsb::kSegShiftD;
    return 4 * wsb::kDirectRows * Ns + ((4 * wsb::kDirectRows * nseg + 15) & ~(size_t)15) +
           sizeof(float) * (wsb::kDirectThreads / 32) * wsb::kRing * wsb::kTail + sizeof(wsb::DEnt) * (size_t)cap;
}

extern "C" int wsb_direct_cap(int N)
{
    const size_t limit = 225 * 1024;
    const size_t base = wsb_direct_smem(N, 0);
    if (base >= limit) return 0;
    return (int)std::min<size_t>((limit - base) / sizeof(wsb::DEnt), 8192);
}

extern "C" cudaError_t wsb_launch_direct(const wsb::EventDesc& ev, const uint32_t* pool, const uint32_t* band_off,
                                         const wsb::UnitRec* band_list, const uint32_t* map, const uint32_t* map_count,
                                         size_t smem_bytes, cudaStream_t stream)
{
    constexpr int NT = wsb::kDirectThreads;
    static unsigned long long ready = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(ready & (1ull << dev))) {
        e = cudaFuncSetAttribute(wsb::k_direct<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
        if (e != cudaSuccess) return e;
        ready |= 1ull << dev;
    }
    if (ev.total_bands == 0) return cudaSuccess;
    wsb::k_direct<NT><<<ev.total_bands, NT, smem_bytes, stream>>>(ev, pool, band_off, band_list, map, map_count);
    return cudaGetLastError();
}
