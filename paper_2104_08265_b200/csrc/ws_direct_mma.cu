// Time-domain convolution on the 5th-generation tensor cores (k_direct_mma):
// the same sum as k_direct (ws_direct.cu),
//   M[w, t] = sum_d c_d[w] g_d[t - ts_d]   (circular in t; c = a eff, g = tv (*) kernel),
// evaluated per 16-row x 2048-tick tile as dense products on tcgen05 instead
// of per-tap shared-memory atomics. For each 128-tick chunk j of the tile,
//   D_j[128 ticks x 16 rows] += G_j[128 x K] . C_j[K x 16]
// where the K columns are the depo profile segments touching the chunk
// (G_j[t][k] = g_k(128 j + t - start_k), 0 outside the profile) and C_j[k][r]
// their tile-row coefficients. D lives in TMEM (16 chunks x 16 fp32 columns =
// 256 columns; two CTAs per SM), the operands in shared memory (canonical
// K-major no-swizzle layout, as k_gprof_umma), double-buffered: the 256
// threads build chunk j+1's operands while one thread's MMAs for chunk j run
// (kind::tf32, 3-pass hi.hi + hi.lo + lo.hi: fp32-level accuracy, a fixed
// order: the frame is deterministic). Each profile tap is written to shared
// memory once per chunk it touches (two stores: hi, lo), the row
// coefficients are applied by the tensor core. The epilogue reads D back with
// tcgen05.ld (warp quadrant = 32 ticks, 8 rows per warp half) and writes the
// frame rows with coalesced stores. No fixed-point bound pass is needed.
//
// Tile lists: the sampler's per-(8-row group, window) lists (fixed capacity,
// or CSR from k_fill_bands); a CTA takes the two groups of its 16 rows.
// Profiles wrapping past the row end appear once per wrap (segment copies
// shifted by -N), so every circular case is covered.
#include "ws_common.cuh"

#include <atomic>

namespace wsb {

constexpr int kDmThreads = 256;
constexpr int kDmRows = 16;                    // tile rows (UMMA N)
constexpr int kDmChunk = 128;                  // ticks per chunk (UMMA M)
constexpr int kDmChunks = kTileTicks / kDmChunk;  // 16
constexpr int kDmKB = 32;                      // segments per MMA K-block (4 K-steps of 8)
constexpr int kDmCap = 256;                    // entries staged per batch (one per thread)
constexpr int kDmSegCap = 512;                 // segments per batch
constexpr int kDmListCap = 2048;               // (chunk, segment) pairs per batch

__device__ __forceinline__ uint32_t dm_tf32(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ uint32_t dm_off(int r, int kc, int R) { return ((kc * (R >> 3) + (r >> 3)) << 7) + ((r & 7) << 4); }
__device__ __forceinline__ uint64_t dm_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void dm_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}
__device__ __forceinline__ void dm_wait(uint32_t bar, uint32_t parity)
{
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(bar), "r"(parity)
                     : "memory");
}

// tile index -> (plane, 16-row group, window): tiles of plane i follow its
// predecessors' ceil(groups / 2) x n_windows
__device__ __forceinline__ int dm_tile(const EventDesc& ev, uint32_t gb, int& rb16, int& win)
{
    uint32_t base = 0;
    int pi = -1;
#pragma unroll 1
    for (int i = 0; i < ev.n_planes; ++i) {
        const PlaneDesc& P = ev.p[i];
        if (!P.direct || !P.stats_owner) continue;  // impact classes share their plane's tiles
        const uint32_t groups = (uint32_t)(P.W + kTileRows - 1) / kTileRows;
        const uint32_t n = ((groups + 1) / 2) * (uint32_t)P.n_windows;
        if (gb < base + n) {
            pi = i;
            const uint32_t l = gb - base;
            rb16 = (int)(l / (uint32_t)P.n_windows);
            win = (int)(l - (uint32_t)rb16 * (uint32_t)P.n_windows);
            break;
        }
        base += n;
    }
    return pi;
}

template <bool kRO>
__global__ void __launch_bounds__(kDmThreads, 2)
k_direct_mma(const EventDesc ev, const uint32_t* __restrict__ pool, const uint32_t* __restrict__ band_off,
             const TEnt* __restrict__ tlist)
{
    // the next call's sampler may launch now (it waits for this grid before
    // touching the pool, the records or the tile lists)
    asm volatile("griddepcontrol.launch_dependents;");
    int rb16 = 0, win = 0;
    const int pi = dm_tile(ev, blockIdx.x, rb16, win);
    if (pi < 0) return;
    const PlaneDesc& P = ev.p[pi];
    const bool fixed = ev.tile_cap != 0;
    if (!fixed && __ldg(&band_off[ev.total_bands]) > ev.list_cap) return;
    const int W = P.W, N = P.N;
    const int r0 = rb16 * kDmRows;
    const int ws = win * kTileTicks, wlen = min(kTileTicks, N - ws);
    const int nchunks = (wlen + kDmChunk - 1) / kDmChunk;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int groups = (W + kTileRows - 1) / kTileRows;

    // layout: A[2][hi, lo] (128 x 32 tf32 each) | B[2][hi, lo] (16 x 32) | staged entries | segments | lists
    extern __shared__ __align__(128) unsigned char dm_smem[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(dm_smem);
    constexpr uint32_t kA = kDmChunk * kDmKB * 4, kB = kDmRows * kDmKB * 4;
    auto a_addr = [&](int s, int part) { return sbase + (uint32_t)(2 * s + part) * kA; };
    auto b_addr = [&](int s, int part) { return sbase + 4u * kA + (uint32_t)(2 * s + part) * kB; };
    TEnt* ent = reinterpret_cast<TEnt*>(dm_smem + 4 * kA + 4 * kB);
    int* seg_start = reinterpret_cast<int*>(ent + kDmCap);  // first tick of the segment, window-relative
    int* seg_len = seg_start + kDmSegCap;                   // profile length L
    uint32_t* seg_goff = reinterpret_cast<uint32_t*>(seg_len + kDmSegCap);  // pool offset of g
    int* seg_ent = reinterpret_cast<int*>(seg_goff + kDmSegCap);            // staged entry | group << 16
    uint16_t* list = reinterpret_cast<uint16_t*>(seg_ent + kDmSegCap);      // per chunk: segment ids
    __shared__ int s_off[kDmChunks + 1];
    __shared__ int s_wcnt[2][kDmThreads / 32][kDmChunks];  // per (round, warp, chunk) segment counts
    __shared__ uint32_t s_wsum[kDmThreads / 32];
    __shared__ int s_n[2];
    __shared__ uint32_t s_lo[2];
    __shared__ int s_take;
    __shared__ uint32_t s_tmem;
    __shared__ uint32_t s_written;  // chunks whose accumulator holds data
    __shared__ __align__(8) unsigned long long s_bar[2];
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&s_bar[0]);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                     "r"(256u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar0));
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar0 + 8u));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_written = 0u;
    }
    // the two 8-row groups' lists
    if (tid < 2) {
        const int g = 2 * rb16 + tid;
        int n = 0;
        uint32_t lo = 0;
        if (g < groups) {
            const uint32_t b = P.band_base + (uint32_t)g * (uint32_t)P.n_windows + (uint32_t)win;
            if (fixed) {
                lo = b * ev.tile_cap;
                n = (int)min(ev.tile_count[b], ev.tile_cap);
            } else {
                lo = __ldg(&band_off[b]);
                n = (int)(__ldg(&band_off[b + 1]) - lo);
            }
        }
        s_n[tid] = n;
        s_lo[tid] = lo;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (fixed && tid < 2 && 2 * rb16 + tid < groups)  // every thread has read the counts: zero for the next call
        ev.tile_count[P.band_base + (uint32_t)(2 * rb16 + tid) * (uint32_t)P.n_windows + (uint32_t)win] = 0u;
    const TEnt* src = fixed ? ev.tiles : tlist;
    const int nA = s_n[0], nB = s_n[1], ntot = nA + nB;

    // the profiles come from the previous kernel (k_gprof_umma)
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // M = 128, N = 16, fp32 accumulate, tf32 operands, both K-major
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kDmRows >> 3) << 17) |
                           ((uint32_t)(kDmChunk >> 4) << 24);
    constexpr uint32_t lbo_a = (kDmChunk / 8) * 128, lbo_b = (kDmRows / 8) * 128;
    int it = 0;  // MMA groups issued (operand slot = it & 1)

#pragma unroll 1
    for (int e0 = 0; e0 < ntot;) {
        // stage up to kDmCap entries (group A's then group B's)
        const int cnt = min(kDmCap, ntot - e0);
        for (int i = tid; i < cnt * (int)(sizeof(TEnt) / 16); i += kDmThreads) {
            const int e = e0 + i / (int)(sizeof(TEnt) / 16), q = i % (int)(sizeof(TEnt) / 16);
            const TEnt* s = e < nA ? src + s_lo[0] + e : src + s_lo[1] + (e - nA);
            reinterpret_cast<int4*>(ent)[i] = __ldg(reinterpret_cast<const int4*>(s) + q);
        }
        __syncthreads();
        // segments: one per wrap of an entry's profile over the row that
        // touches the window; cost of an entry = (segments << 16) | (chunk,
        // segment) pairs. A block scan places them in entry order; the batch
        // takes the longest prefix that fits both budgets.
        uint32_t cost = 0;
        const int me = tid;  // kDmCap == kDmThreads: one entry per thread
        if (me < cnt) {
            const TEnt& d = ent[me];
            const int ts = (int)(d.tsL & 0xffffu), L = (int)(d.tsL >> 16);
            for (int c = 0;; ++c) {
                const int a = ts - ws - c * N;
                if (a + L <= 0) break;
                if (a < wlen) cost += (1u << 16) + (uint32_t)((min(a + L, wlen) - 1) / kDmChunk - max(a, 0) / kDmChunk + 1);
            }
        }
        uint32_t incl = cost;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[warp] = incl;
        if (tid == 0) s_take = cnt;
        __syncthreads();
        uint32_t wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += s_wsum[w];
        incl += wbase;
        const uint32_t excl = incl - cost;
        const bool fits = (incl >> 16) <= (uint32_t)kDmSegCap && (incl & 0xffffu) <= (uint32_t)kDmListCap;
        // first entry that does not fit (entries are a prefix: costs are >= 0)
        if (me < cnt && !fits && (me == 0 || (((excl >> 16) <= (uint32_t)kDmSegCap) &&
                                              (excl & 0xffffu) <= (uint32_t)kDmListCap)))
            s_take = max(me, 1);
        __syncthreads();
        const int take = s_take;
        int nseg = 0;
        {
            // total segments of the taken prefix: the scan value of entry take - 1
            __shared__ uint32_t s_tot;
            if (me == take - 1) s_tot = incl;
            __syncthreads();
            nseg = (int)(s_tot >> 16);
        }
        if (me < take) {
            const TEnt& d = ent[me];
            const int ts = (int)(d.tsL & 0xffffu), L = (int)(d.tsL >> 16);
            int sidx = (int)(excl >> 16);
            for (int c = 0;; ++c) {
                const int a = ts - ws - c * N;
                if (a + L <= 0) break;
                if (a < wlen) {
                    seg_start[sidx] = a;
                    seg_len[sidx] = L;
                    seg_goff[sidx] = d.goff;
                    seg_ent[sidx] = me | ((e0 + me) < nA ? 0 : (1 << 16));
                    ++sidx;
                }
            }
        }
        __syncthreads();
        // per-chunk segment lists in segment order (deterministic MMA K order):
        // positions from ballot prefix counts over (round, warp, lane)
        uint32_t cmask[2] = {0u, 0u};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int sg = r * kDmThreads + tid;
            if (sg < nseg) {
                const int a = seg_start[sg], L = seg_len[sg];
                const int j0 = max(a, 0) / kDmChunk, j1 = (min(a + L, wlen) - 1) / kDmChunk;
                cmask[r] = ((2u << j1) - 1u) & ~((1u << j0) - 1u);
            }
#pragma unroll
            for (int j = 0; j < kDmChunks; ++j) {
                const unsigned bal = __ballot_sync(0xffffffffu, (cmask[r] >> j) & 1u);
                if (lane == 0) s_wcnt[r][warp][j] = __popc(bal);
            }
        }
        __syncthreads();
        if (tid < kDmChunks) {  // per chunk: running offsets over (round, warp)
            int tot = 0;
            for (int r = 0; r < 2; ++r)
                for (int w = 0; w < kDmThreads / 32; ++w) {
                    const int c = s_wcnt[r][w][tid];
                    s_wcnt[r][w][tid] = tot;
                    tot += c;
                }
            s_off[tid + 1] = tot;  // chunk sizes (prefix below)
        }
        __syncthreads();
        if (tid == 0) {
            s_off[0] = 0;
            for (int j = 0; j < kDmChunks; ++j) s_off[j + 1] += s_off[j];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int sg = r * kDmThreads + tid;
#pragma unroll
            for (int j = 0; j < kDmChunks; ++j) {
                const unsigned bal = __ballot_sync(0xffffffffu, (cmask[r] >> j) & 1u);
                if ((cmask[r] >> j) & 1u)
                    list[s_off[j] + s_wcnt[r][warp][j] + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)sg;
            }
        }
        __syncthreads();

        // groups = (chunk, K-block of 32 segments); each thread's 16 profile
        // values of group g + 1 are loaded (in flight) while it writes group
        // g's operands; the operands go to slot it & 1, one thread issues the MMAs
        int ng = 0;
        for (int j = 0; j < nchunks; ++j) ng += (s_off[j + 1] - s_off[j] + kDmKB - 1) / kDmKB;
        auto group = [&](int g, int& j, int& kb) {  // g-th (chunk, block) in chunk order
            for (j = 0; j < nchunks; ++j) {
                const int nb = (s_off[j + 1] - s_off[j] + kDmKB - 1) / kDmKB;
                if (g < nb) break;
                g -= nb;
            }
            kb = g * kDmKB;
        };
        const int tA = tid & 63, kq0 = tid >> 6;  // thread: ticks tA, tA + 64; segment quads kq0, kq0 + 4
        auto load_group = [&](int g, float* v) {
            int j, kb;
            group(g, j, kb);
            const int lo = s_off[j], kn = min(kDmKB, s_off[j + 1] - lo - kb);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = 4 * (kq0 + 4 * h2) + q;
                    int st = 1 << 30, ln = 0;
                    const float* gp = nullptr;
                    if (k < kn) {
                        const int sg = list[lo + kb + k];
                        st = seg_start[sg] - j * kDmChunk;  // tap index = t - st
                        ln = seg_len[sg];
                        gp = reinterpret_cast<const float*>(pool + seg_goff[sg]);
                    }
#pragma unroll
                    for (int t2 = 0; t2 < 2; ++t2) {
                        const int tau = tA + 64 * t2 - st;
                        v[8 * h2 + 4 * t2 + q] = (tau >= 0 && tau < ln) ? __ldg(gp + tau) : 0.0f;
                    }
                }
        };
        float vn[16];
        if (ng > 0) load_group(0, vn);
#pragma unroll 1
        for (int g = 0; g < ng; ++g) {
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = vn[i];
            if (g + 1 < ng) load_group(g + 1, vn);
            int j, kb;
            group(g, j, kb);
            const int lo = s_off[j], kn = min(kDmKB, s_off[j + 1] - lo - kb);
            const int slot = it & 1;
            if (it >= 2) dm_wait(bar0 + 8u * (uint32_t)slot, (uint32_t)(((it - 2) >> 1) & 1));
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                for (int t2 = 0; t2 < 2; ++t2) {
                    uint32_t hi[4], lo4[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float x = v[8 * h2 + 4 * t2 + q];
                        hi[q] = dm_tf32(x);
                        lo4[q] = dm_tf32(x - __uint_as_float(hi[q]));
                    }
                    const uint32_t o = dm_off(tA + 64 * t2, kq0 + 4 * h2, kDmChunk);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a_addr(slot, 0) + o), "r"(hi[0]),
                                 "r"(hi[1]), "r"(hi[2]), "r"(hi[3]));
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a_addr(slot, 1) + o), "r"(lo4[0]),
                                 "r"(lo4[1]), "r"(lo4[2]), "r"(lo4[3]));
                }
            // B: (tile row n, 4 segments): the segment's coefficient of row n
            if (tid < kDmRows * (kDmKB / 4)) {
                const int nr = tid & (kDmRows - 1), kq = tid >> 4;
                uint32_t hi[4], lo4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = 4 * kq + q;
                    float c = 0.0f;
                    if (k < kn) {
                        const int se = seg_ent[list[lo + kb + k]];
                        if ((nr >> 3) == (se >> 16)) c = ent[se & 0xffff].c[nr & 7];
                    }
                    hi[q] = dm_tf32(c);
                    lo4[q] = dm_tf32(c - __uint_as_float(hi[q]));
                }
                const uint32_t o = dm_off(nr, kq, kDmRows);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b_addr(slot, 0) + o), "r"(hi[0]),
                             "r"(hi[1]), "r"(hi[2]), "r"(hi[3]));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(b_addr(slot, 1) + o), "r"(lo4[0]),
                             "r"(lo4[1]), "r"(lo4[2]), "r"(lo4[3]));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (tid == 0) {
                const uint32_t d = tmem + (uint32_t)(j * kDmRows);
                const bool first = !((s_written >> j) & 1u);
                const uint32_t as[3] = {a_addr(slot, 0), a_addr(slot, 0), a_addr(slot, 1)};
                const uint32_t bs[3] = {b_addr(slot, 0), b_addr(slot, 1), b_addr(slot, 0)};
                const int ksteps = (kn + 7) >> 3;
#pragma unroll 1
                for (int pass = 0; pass < 3; ++pass)
#pragma unroll 1
                    for (int s = 0; s < ksteps; ++s)
                        dm_mma(d, dm_desc(as[pass] + 2u * s * lbo_a, lbo_a, 128),
                               dm_desc(bs[pass] + 2u * s * lbo_b, lbo_b, 128), idesc,
                               (first && pass == 0 && s == 0) ? 0u : 1u);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 bar0 + 8u * (uint32_t)slot)
                             : "memory");
                s_written |= 1u << j;
            }
            ++it;
        }
        e0 += take;
        __syncthreads();  // staging areas are rewritten by the next batch (the MMAs read only A / B)
    }

    // all MMAs done (a commit tracks every earlier tcgen05 op of the thread)
    if (it > 0) dm_wait(bar0 + 8u * (uint32_t)((it - 1) & 1), (uint32_t)(((it - 1) >> 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    __syncthreads();
    const uint32_t written = s_written;

    // epilogue: warp (quadrant q, half h) reads ticks 32 q .. 32 q + 31 of a
    // chunk, rows 8 h .. 8 h + 7; one coalesced 128-byte store per row
    const int q4 = warp & 3, h = warp >> 2;
#pragma unroll 1
    for (int j = 0; j < nchunks; ++j) {
        uint32_t v[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        if ((written >> j) & 1u) {
            const uint32_t taddr = tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(j * kDmRows + 8 * h);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                           "=r"(v[7])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        const int t = j * kDmChunk + 32 * q4 + lane;
        if (t >= wlen) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = r0 + 8 * h + i;
            if (row >= W) break;
            const float x = __uint_as_float(v[i]);
            if constexpr (kRO) {
                // fused readout: this lane's sample of its tick pair (the pair's
                // normals recomputed per lane; noise only when requested)
                const int tg = ws + t;
                double val = (double)x;
                if (ev.ro_noise) {
                    double n0, n1;
                    white_pair(ev.ro_seed, row, tg >> 1, n0, n1);
                    val = __dadd_rn(val, __dmul_rn(ev.ro_sigma, (tg & 1) ? n1 : n0));
                }
                const Sink k{P.frame, P.frame64, P.adc, ev.adc_u16, ev.adc_scale, ev.adc_offset, ev.adc_max};
                sink_put(k, (size_t)row * N + tg, val);
            } else {
                __stcs(P.frame + (size_t)row * N + ws + t, x);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
}

}  // namespace wsb

extern "C" size_t wsb_direct_mma_smem()
{
    using namespace wsb;
    return 4 * (size_t)kDmChunk * kDmKB * 4 + 4 * (size_t)kDmRows * kDmKB * 4 + sizeof(TEnt) * kDmCap +
           4 * sizeof(int) * kDmSegCap + sizeof(uint16_t) * kDmListCap;
}

// 16-row tiles of the direct planes of the call
extern "C" uint32_t wsb_direct_mma_tiles(const wsb::EventDesc& ev)
{
    uint32_t n = 0;
    for (int i = 0; i < ev.n_planes; ++i) {
        const wsb::PlaneDesc& P = ev.p[i];
        if (!P.direct || !P.stats_owner) continue;
        const uint32_t groups = (uint32_t)(P.W + wsb::kTileRows - 1) / wsb::kTileRows;
        n += ((groups + 1) / 2) * (uint32_t)P.n_windows;
    }
    return n;
}

extern "C" cudaError_t wsb_launch_direct_mma(const wsb::EventDesc& ev, const uint32_t* pool, const uint32_t* band_off,
                                             const wsb::TEnt* tlist, cudaStream_t stream, int pdl)
{
    static std::atomic<unsigned long long> ready{0};  // per-device attribute setup (idempotent)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const size_t smem = wsb_direct_mma_smem();
    if (!(ready & (1ull << dev))) {
        for (auto f : {wsb::k_direct_mma<false>, wsb::k_direct_mma<true>}) {
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        ready |= 1ull << dev;
    }
    const uint32_t tiles = wsb_direct_mma_tiles(ev);
    if (tiles == 0) return cudaSuccess;
    const auto kfn = ev.ro ? wsb::k_direct_mma<true> : wsb::k_direct_mma<false>;
    if (!pdl) {
        kfn<<<tiles, wsb::kDmThreads, smem, stream>>>(ev, pool, band_off, tlist);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(tiles);
    cfg.blockDim = dim3(wsb::kDmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kfn, ev, pool, band_off, tlist);
}
