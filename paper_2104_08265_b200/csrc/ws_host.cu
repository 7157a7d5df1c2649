// Host-side helpers of the C ABI: pinned allocations and the synthetic depo
// generator (input synthesis, not part of the timed hot path).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "wiresim_gpu.h"

namespace {

uint64_t splitmix64_next(uint64_t& s)
{
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct Xoshiro {
    uint64_t s[4];
    explicit Xoshiro(uint64_t seed)
    {
        // seed_state (rng.cpp:26-35)
        uint64_t sm = seed;
        for (auto& w : s) w = splitmix64_next(sm);
        if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 0x9e3779b97f4a7c15ULL;
    }
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    double uniform()
    {
        const uint64_t result = rotl(s[1] * 5, 7) * 9;
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return (double)(result >> 11) * 0x1.0p-53;
    }
};

}  // namespace

extern "C" int ws_set_error_message(int code, const char* msg);

extern "C" int ws_host_alloc(uint64_t bytes, void** out)
{
    if (!out) return ws_set_error_message(WS_EINVAL, "null out pointer");
    const cudaError_t e = cudaMallocHost(out, bytes ? bytes : 1);
    if (e != cudaSuccess) return ws_set_error_message(WS_ECUDA, cudaGetErrorString(e));
    return WS_OK;
}

extern "C" int ws_host_free(void* p)
{
    if (p) cudaFreeHost(p);
    return WS_OK;
}

extern "C" int ws_gen_depos_uniform(uint64_t n, uint64_t seed, const ws_grid_spec* g, const double* r, ws_depo* out)
{
    if (!g || (!out && n)) return ws_set_error_message(WS_EINVAL, "null argument");
    if (g->n_wires < 1 || g->n_ticks < 1 || !(g->pitch > 0.0) || !(g->tick > 0.0))
        return ws_set_error_message(WS_EINVAL, "GridSpec: invalid");
    const int64_t q_min = r ? (int64_t)r[0] : 1000, q_max = r ? (int64_t)r[1] : 10000;
    const double st0 = r ? r[2] : 0.5, st1 = r ? r[3] : 1.5, sx0 = r ? r[4] : 2.5, sx1 = r ? r[5] : 7.5;
    if (q_min < 0 || q_max < q_min) return ws_set_error_message(WS_EINVAL, "gen_depos: bad charge range");
    Xoshiro st(seed);
    const double t_span = (double)g->n_ticks * g->tick;
    const double x_span = (double)g->n_wires * g->pitch;
    for (uint64_t i = 0; i < n; ++i) {
        ws_depo& d = out[i];
        d.id = (int64_t)i;
        d.t = g->origin_t + st.uniform() * t_span;
        d.x = g->origin_x + st.uniform() * x_span;
        d.q = q_min + (int64_t)(st.uniform() * (double)(q_max - q_min + 1));
        d.sigma_t = st0 + st.uniform() * (st1 - st0);
        d.sigma_x = sx0 + st.uniform() * (sx1 - sx0);
    }
    return WS_OK;
}
