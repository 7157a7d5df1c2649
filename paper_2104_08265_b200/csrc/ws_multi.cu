// Multi-GPU sharding behind the C ABI (include/wiresim_gpu.h, ws_multi_*):
// one context per listed device, the same plane geometries on each, and a
// host thread per device. Work units are independent — whole events, or
// (anode-face, plane) runs (one plane per run) — so there is no
// collective on the data path: each device thread runs its shard through the
// pipelined host-buffer path (events_host in ws_api.cu) and its device-to-host
// copies land in the caller's own (disjoint) output buffers, which is the
// final frame gather. Results are placement-invariant: the RNG streams are
// keyed by (seed, depo id), never by device or order.
//
// Sharding: longest-processing-time first over the devices, cost of a unit =
// cells + kDepoCost x depos (the time-domain path's per-depo work against its
// frame write; ws_multi_cost), ties broken by device index.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "wiresim_gpu.h"

extern "C" int ws_set_error_message(int code, const char* msg);

struct ws_multi {
    std::vector<int> devices;
    std::vector<ws_ctx*> ctx;
    std::vector<std::vector<ws_plane*>> planes;  // [device][plane spec]
    std::vector<uint64_t> cells;                 // per plane spec
    uint32_t n_planes = 0;
};

namespace {

constexpr double kDepoCost = 900.0;  // cells-equivalent of one depo on one plane (fitted to the r2 C5 sweep: ~0.9-1.3 ns per depo-plane vs ~1 ps per cell)

int fail(int code, const std::string& msg) { return ws_set_error_message(code, msg.c_str()); }

// LPT: units in decreasing cost, each to the least-loaded device
std::vector<uint32_t> lpt(const std::vector<double>& cost, uint32_t n_dev)
{
    std::vector<uint32_t> order(cost.size());
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cost[a] > cost[b]; });
    std::vector<double> load(n_dev, 0.0);
    std::vector<uint32_t> dev(cost.size(), 0);
    for (uint32_t u : order) {
        const uint32_t d = (uint32_t)(std::min_element(load.begin(), load.end()) - load.begin());
        dev[u] = d;
        load[d] += cost[u];
    }
    return dev;
}

// run fn(d) on one host thread per device; the first failing device's status
// and message are returned on the calling thread
template <class F>
int on_devices(uint32_t n_dev, F&& fn)
{
    std::vector<int> rc(n_dev, WS_OK);
    std::vector<std::string> msg(n_dev);
    std::vector<std::thread> th;
    th.reserve(n_dev);
    for (uint32_t d = 0; d < n_dev; ++d)
        th.emplace_back([&, d] {
            rc[d] = fn(d);
            if (rc[d]) msg[d] = ws_last_error();  // thread-local: carried to the caller
        });
    for (auto& t : th) t.join();
    for (uint32_t d = 0; d < n_dev; ++d)
        if (rc[d]) return fail(rc[d], "device " + std::to_string(d) + ": " + msg[d]);
    return WS_OK;
}

}  // namespace

extern "C" {

double ws_multi_cost(uint64_t cells, uint64_t n_depos) { return (double)cells + kDepoCost * (double)n_depos; }

int ws_multi_create(uint32_t n_devices, const int* devices, uint32_t n_planes, const ws_grid_spec* grids,
                    const ws_response* responses, double n_sigma, ws_multi** out)
{
    if (!out || !devices || n_devices == 0) return fail(WS_EINVAL, "ws_multi_create: no devices");
    if (n_planes && (!grids || !responses)) return fail(WS_EINVAL, "ws_multi_create: null plane specs");
    *out = nullptr;
    ws_multi* m = new ws_multi();
    m->devices.assign(devices, devices + n_devices);
    m->n_planes = n_planes;
    m->ctx.assign(n_devices, nullptr);
    m->planes.assign(n_devices, std::vector<ws_plane*>(n_planes, nullptr));
    for (uint32_t i = 0; i < n_planes; ++i)
        m->cells.push_back((grids[i].n_wires + 2 * grids[i].pad_wires) * (grids[i].n_ticks + 2 * grids[i].pad_ticks));
    int rc = WS_OK;
    for (uint32_t d = 0; d < n_devices && rc == WS_OK; ++d) {
        rc = ws_ctx_create(devices[d], nullptr, &m->ctx[d]);
        for (uint32_t i = 0; i < n_planes && rc == WS_OK; ++i)
            rc = ws_plane_create(m->ctx[d], &grids[i], &responses[i], n_sigma, &m->planes[d][i]);
    }
    if (rc) {
        const std::string msg = ws_last_error();
        ws_multi_destroy(m);
        return fail(rc, msg);
    }
    *out = m;
    return WS_OK;
}

int ws_multi_destroy(ws_multi* m)
{
    if (!m) return WS_OK;
    for (size_t d = 0; d < m->ctx.size(); ++d) {
        for (ws_plane* p : m->planes[d]) ws_plane_destroy(p);
        ws_ctx_destroy(m->ctx[d]);
    }
    delete m;
    return WS_OK;
}

uint32_t ws_multi_device_count(const ws_multi* m) { return m ? (uint32_t)m->ctx.size() : 0u; }
ws_ctx* ws_multi_context(ws_multi* m, uint32_t i) { return m && i < m->ctx.size() ? m->ctx[i] : nullptr; }
ws_plane* ws_multi_plane(ws_multi* m, uint32_t device_index, uint32_t plane)
{
    return m && device_index < m->ctx.size() && plane < m->n_planes ? m->planes[device_index][plane] : nullptr;
}

int ws_multi_set_conv_path(ws_multi* m, int path)
{
    if (!m) return fail(WS_EINVAL, "null multi");
    for (ws_ctx* c : m->ctx)
        if (int rc = ws_ctx_set_conv_path(c, path)) return rc;
    return WS_OK;
}

int ws_multi_run_events(ws_multi* m, uint32_t n_events, const ws_depo* const* depos, const uint64_t* n_depos,
                        const ws_sim_options* opt, const ws_readout* readout, void* const* adcs, void* const* frames,
                        uint32_t* event_device, ws_timing* timing)
{
    if (!m) return fail(WS_EINVAL, "null multi");
    if (n_events == 0) return WS_OK;
    if (!depos || !n_depos) return fail(WS_EINVAL, "null argument");
    const uint32_t P = m->n_planes, D = (uint32_t)m->ctx.size();
    std::vector<double> cost(n_events, 0.0);
    for (uint32_t e = 0; e < n_events; ++e)
        for (uint32_t i = 0; i < P; ++i) cost[e] += ws_multi_cost(m->cells[i], n_depos[(size_t)e * P + i]);
    const std::vector<uint32_t> dev = lpt(cost, D);
    if (event_device) std::copy(dev.begin(), dev.end(), event_device);
    return on_devices(D, [&](uint32_t d) -> int {
        std::vector<const ws_depo*> dd;
        std::vector<uint64_t> nd;
        std::vector<void*> aa, ff;
        for (uint32_t e = 0; e < n_events; ++e) {
            if (dev[e] != d) continue;
            for (uint32_t i = 0; i < P; ++i) {
                const size_t k = (size_t)e * P + i;
                dd.push_back(depos[k]);
                nd.push_back(n_depos[k]);
                aa.push_back(adcs ? adcs[k] : nullptr);
                ff.push_back(frames ? frames[k] : nullptr);
            }
        }
        const uint32_t ne = P ? (uint32_t)(dd.size() / P) : 0u;
        if (ne == 0) return WS_OK;
        ws_timing* t = d == 0 ? timing : nullptr;
        if (readout)
            return ws_run_events(m->ctx[d], ne, P, m->planes[d].data(), dd.data(), nd.data(), opt, readout,
                                 adcs ? aa.data() : nullptr, frames ? ff.data() : nullptr, t);
        return ws_simulate_events(m->ctx[d], ne, P, m->planes[d].data(), dd.data(), nd.data(), opt,
                                  reinterpret_cast<float* const*>(ff.data()), t);
    });
}

int ws_multi_run_units(ws_multi* m, uint32_t n_units, const uint32_t* plane_of, const ws_depo* const* depos,
                       const uint64_t* n_depos, const ws_sim_options* opt, const ws_readout* readout,
                       void* const* adcs, void* const* frames, uint32_t* unit_device)
{
    if (!m) return fail(WS_EINVAL, "null multi");
    if (n_units == 0) return WS_OK;
    if (!plane_of || !depos || !n_depos) return fail(WS_EINVAL, "null argument");
    const uint32_t D = (uint32_t)m->ctx.size();
    std::vector<double> cost(n_units);
    for (uint32_t u = 0; u < n_units; ++u) {
        if (plane_of[u] >= m->n_planes)
            return fail(WS_EINVAL, "unit " + std::to_string(u) + ": plane index out of range");
        cost[u] = ws_multi_cost(m->cells[plane_of[u]], n_depos[u]);
    }
    const std::vector<uint32_t> dev = lpt(cost, D);
    if (unit_device) std::copy(dev.begin(), dev.end(), unit_device);
    return on_devices(D, [&](uint32_t d) -> int {
        // a device's units form one "event" of independent planes (launch
        // groups of up to 8 planes, host-buffer path)
        std::vector<ws_plane*> pl;
        std::vector<const ws_depo*> dd;
        std::vector<uint64_t> nd;
        std::vector<void*> aa, ff;
        for (uint32_t u = 0; u < n_units; ++u) {
            if (dev[u] != d) continue;
            pl.push_back(m->planes[d][plane_of[u]]);
            dd.push_back(depos[u]);
            nd.push_back(n_depos[u]);
            aa.push_back(adcs ? adcs[u] : nullptr);
            ff.push_back(frames ? frames[u] : nullptr);
        }
        if (pl.empty()) return WS_OK;
        const uint32_t n = (uint32_t)pl.size();
        if (readout)
            return ws_run_events(m->ctx[d], 1, n, pl.data(), dd.data(), nd.data(), opt, readout,
                                 adcs ? aa.data() : nullptr, frames ? ff.data() : nullptr, nullptr);
        return ws_simulate_event(m->ctx[d], n, pl.data(), dd.data(), nd.data(), opt,
                                 reinterpret_cast<float* const*>(ff.data()), nullptr);
    });
}

}  // extern "C"
