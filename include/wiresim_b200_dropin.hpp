// wiresim_b200_dropin.hpp — run_simulation with the reference's OWN types:
// include it after the reference headers (<wiresim/pipeline.hpp>), pass a real
// wiresim::SimConfig and std::vector<wiresim::Depo>, get a wiresim::SimResult
// back, computed on the B200 through the C ABI (wiresim_gpu.h). Nothing here
// needs the reference library at link time; only its headers.
//
//   #include <wiresim/pipeline.hpp>
//   #include "wiresim_b200_dropin.hpp"
//   wiresim::SimResult r = wiresim_b200::run_simulation(config, depos);   // was wiresim::run_simulation
//
// Mapping of SimConfig (pipeline.hpp:36-50):
//   grid, response, n_sigma, drift       -> ws_plane_create / ws_sim_options (same meaning)
//   rng.mode substream                   -> WS_RNG_SUBSTREAM: the reference's own per-depo stream; the
//                                           integer charge grid is identical (rasterize.cpp:190-193)
//   rng.mode pool                        -> fluctuate_approx (rasterize.cpp:159-170) with normals from
//                                           per-depo streams (no 1.6 GB pool; statistically equivalent)
//   rng.mode inline_stream               -> std::invalid_argument: its draws are order-dependent
//                                           (the reference refuses it with workers > 1, pipeline.cpp:65-68)
//   noise, adc                           -> ws_readout (add_noise + digitize, spectral.cpp:177-238),
//                                           noise seed = rng.seed as in pipeline.cpp:421
//   workers, dispatch, batch_size, scatter -> no meaning on the GPU (results never depend on them)
// SimResult (pipeline.hpp:94-99): adc (Matrix<int32_t>), charge (int64 counts),
// clipped_charge, and the TimingReport fields this path measures (device
// times in seconds: rasterization_total_s = sample + fluctuate, scatter_add_s
// = binning, ft_s = convolution, total_s).
//
// Simulator caches the context and one plane per distinct (grid, response,
// n_sigma): the response spectrum is built once, the device workspace is
// reused across calls (the reference rebuilds the response every call,
// pipeline.cpp:417).
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "wiresim_gpu.h"

namespace wiresim_b200 {

namespace dropin_detail {

inline void check(int rc)
{
    if (rc == WS_OK) return;
    const std::string msg = ws_last_error();
    switch (rc) {
        case WS_EINVAL: throw std::invalid_argument(msg);
        case WS_ERANGE: throw std::out_of_range(msg);
        case WS_EDOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

inline bool same_grid(const wiresim::GridSpec& a, const wiresim::GridSpec& b)
{
    return a.n_wires == b.n_wires && a.n_ticks == b.n_ticks && a.pad_wires == b.pad_wires &&
           a.pad_ticks == b.pad_ticks && a.pitch == b.pitch && a.tick == b.tick && a.origin_x == b.origin_x &&
           a.origin_t == b.origin_t;
}

inline bool same_response(const wiresim::ResponseParams& a, const wiresim::ResponseParams& b)
{
    return a.plane_kind == b.plane_kind && a.field_sigma_t == b.field_sigma_t &&
           a.shaper_peaking == b.shaper_peaking && a.shaper_order == b.shaper_order && a.gain == b.gain &&
           a.wire_weights == b.wire_weights;
}

}  // namespace dropin_detail

class Simulator {
  public:
    explicit Simulator(int device = 0) { dropin_detail::check(ws_ctx_create(device, nullptr, &m_ctx)); }
    ~Simulator()
    {
        for (auto& e : m_planes) ws_plane_destroy(e.plane);
        ws_ctx_destroy(m_ctx);
    }
    Simulator(const Simulator&) = delete;
    Simulator& operator=(const Simulator&) = delete;
    ws_ctx* context() const { return m_ctx; }

    wiresim::SimResult run(const wiresim::SimConfig& config, const std::vector<wiresim::Depo>& depos)
    {
        static_assert(sizeof(wiresim::Depo) == sizeof(ws_depo), "wiresim::Depo must keep its 48-byte layout");
        using dropin_detail::check;
        config.grid.validate();  // GridSpec::validate is inline in core.hpp
        if (config.n_sigma <= 0.0) throw std::invalid_argument("config: n_sigma must be > 0");
        if (config.adc.bits < 1 || config.adc.bits > 16)
            throw std::invalid_argument("config: adc.bits must be in [1,16]");
        if (config.rng.mode == wiresim::RngMode::inline_stream)
            throw std::invalid_argument(
                "config: inline rng draws are order-dependent and therefore serial-only; "
                "use pool or substream mode on the GPU");
        ws_plane* plane = plane_for(config);
        ws_sim_options o{};
        o.fluctuate = 1;  // the reference always fluctuates (rasterize.cpp:182-202)
        o.approx = config.rng.mode == wiresim::RngMode::pool ? 1 : 0;
        o.rng_mode = WS_RNG_SUBSTREAM;
        o.charge_type = WS_CHARGE_I64;  // the exact counts straight into ChargeGrid's int64 matrix
        o.seed = config.rng.seed;
        o.drift.enabled = config.drift.enabled ? 1 : 0;
        o.drift.response_plane_x = config.drift.response_plane_x;
        o.drift.drift_speed = config.drift.drift_speed;
        o.drift.diffusion_long = config.drift.diffusion_long;
        o.drift.diffusion_tran = config.drift.diffusion_tran;
        ws_readout ro{};
        ro.noise.mode = config.noise.mode == wiresim::NoiseMode::off     ? WS_NOISE_OFF
                        : config.noise.mode == wiresim::NoiseMode::white ? WS_NOISE_WHITE
                                                                         : WS_NOISE_SPECTRUM;
        ro.noise.rng_mode = WS_RNG_SUBSTREAM;  // the reference's per-wire streams
        ro.noise.sigma = config.noise.sigma;
        ro.noise.seed = config.rng.seed;
        ro.noise.amplitude_spectrum = config.noise.amplitude_spectrum.data();
        ro.noise.n_amplitude = config.noise.amplitude_spectrum.size();
        ro.adc.scale = config.adc.scale;
        ro.adc.offset = config.adc.offset;
        ro.adc.bits = config.adc.bits;
        ro.frame_type = WS_FRAME_F32;
        ro.adc_type = WS_ADC_I32;

        const std::size_t W = config.grid.padded_wires(), T = config.grid.padded_ticks();
        wiresim::SimResult res{wiresim::Matrix<std::int32_t>(W, T), wiresim::TimingReport{},
                               wiresim::ChargeGrid(config.grid), 0};
        ws_timing t{};
        check(ws_run_simulation(plane, reinterpret_cast<const ws_depo*>(depos.data()), depos.size(), &o, &ro,
                                res.adc.data.data(), nullptr, reinterpret_cast<float*>(res.charge.counts.data.data()),
                                &t));
        res.clipped_charge = t.clipped_charge;
        res.timing.rasterization_total_s = 1e-3 * (t.prepare_ms + t.fluctuate_ms);
        res.timing.sampling_2d_s = 1e-3 * t.prepare_ms;
        res.timing.fluctuation_s = 1e-3 * t.fluctuate_ms;
        res.timing.scatter_add_s = 1e-3 * t.bin_ms;
        res.timing.ft_s = 1e-3 * t.convolve_ms;
        res.timing.total_s = 1e-3 * t.total_ms;
        res.timing.rng_mode = config.rng.mode == wiresim::RngMode::pool ? "pool" : "substream";
        res.timing.dispatch_mode = "b200";
        res.timing.workers = 1;
        res.timing.clipped_patch_count = t.clipped_patches;
        return res;
    }

  private:
    struct Entry {
        wiresim::GridSpec grid;
        wiresim::ResponseParams response;
        double n_sigma;
        ws_plane* plane;
    };

    ws_plane* plane_for(const wiresim::SimConfig& c)
    {
        for (auto& e : m_planes)
            if (e.n_sigma == c.n_sigma && dropin_detail::same_grid(e.grid, c.grid) &&
                dropin_detail::same_response(e.response, c.response))
                return e.plane;
        const ws_grid_spec g{c.grid.n_wires, c.grid.n_ticks, c.grid.pad_wires, c.grid.pad_ticks,
                             c.grid.pitch,   c.grid.tick,    c.grid.origin_x,  c.grid.origin_t};
        ws_response r{};
        r.plane_kind = c.response.plane_kind == wiresim::PlaneKind::collection ? WS_COLLECTION : WS_INDUCTION;
        r.shaper_order = c.response.shaper_order;
        r.field_sigma_t = c.response.field_sigma_t;
        r.shaper_peaking = c.response.shaper_peaking;
        r.gain = c.response.gain;
        r.wire_weights = c.response.wire_weights.data();
        r.n_wire_weights = c.response.wire_weights.size();
        ws_plane* p = nullptr;
        dropin_detail::check(ws_plane_create(m_ctx, &g, &r, c.n_sigma, &p));
        m_planes.push_back(Entry{c.grid, c.response, c.n_sigma, p});
        return p;
    }

    ws_ctx* m_ctx = nullptr;
    std::vector<Entry> m_planes;
};

// Drop-in for wiresim::run_simulation (pipeline.hpp:104): one Simulator per
// host thread on device 0, kept for the thread's lifetime.
inline wiresim::SimResult run_simulation(const wiresim::SimConfig& config, const std::vector<wiresim::Depo>& depos)
{
    thread_local std::unique_ptr<Simulator> sim;
    if (!sim) sim = std::make_unique<Simulator>(0);
    return sim->run(config, depos);
}

}  // namespace wiresim_b200
