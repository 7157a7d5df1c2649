// wiresim_b200.hpp — header-only C++ mirror of the reference `wiresim`
// interface for the hot path, on top of the C ABI in wiresim_gpu.h.
//
// A caller of the reference keeps its types and call shape:
//
//   wiresim::SimResult r = wiresim::run_simulation(config, depos);   // reference (CPU)
//   wiresim_b200::SimResult g = wiresim_b200::run_simulation(config, depos);   // B200
//
// Types mirror /root/reference/proj/include/wiresim: GridSpec (core.hpp:40-58),
// Depo (core.hpp:63-70, same 48-byte layout, so a std::vector<wiresim::Depo>
// is accepted as is), ResponseParams (spectral.hpp:18-26), DriftParams
// (rasterize.hpp:16-23), RngConfig / SimConfig (pipeline.hpp:24-50). Errors
// are rethrown as the exception types the reference throws
// (std::invalid_argument, std::out_of_range, std::domain_error,
// std::runtime_error). The frame is the pre-noise measurement M of
// convolve (spectral.hpp:47), float32, padded wire x tick, row-major.
#pragma once

#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "wiresim_gpu.h"

namespace wiresim_b200 {

struct GridSpec {
    std::size_t n_wires = 1000;
    std::size_t n_ticks = 6000;
    std::size_t pad_wires = 100;
    std::size_t pad_ticks = 100;
    double pitch = 5.0;
    double tick = 0.5;
    double origin_x = 0.0;
    double origin_t = 0.0;
    std::size_t padded_wires() const { return n_wires + 2 * pad_wires; }
    std::size_t padded_ticks() const { return n_ticks + 2 * pad_ticks; }
};

using Depo = ws_depo;  // {id, t, x, q, sigma_t, sigma_x} == wiresim::Depo

enum class PlaneKind { induction, collection };

struct ResponseParams {
    PlaneKind plane_kind = PlaneKind::collection;
    double field_sigma_t = 1.0;
    double shaper_peaking = 2.0;
    int shaper_order = 2;
    double gain = 14.0;
    std::vector<double> wire_weights{1.0};
};

struct DriftParams {
    double response_plane_x = 0.0;
    double drift_speed = 1.6;
    double diffusion_long = 0.0068;
    double diffusion_tran = 0.0088;
    bool enabled = false;
};

enum class RngMode { substream, philox };

struct RngConfig {
    RngMode mode = RngMode::substream;
    std::uint64_t seed = 12345;
};

struct SimConfig {
    GridSpec grid;
    DriftParams drift;
    ResponseParams response;
    double n_sigma = 3.0;
    RngConfig rng;
    bool fluctuate = true;  // the reference always fluctuates (rasterize.cpp:182-202)
    bool approx = false;    // fluctuate_approx (rasterize.cpp:159-170)
};

struct Frame {
    GridSpec spec;
    std::size_t rows = 0, cols = 0;
    std::vector<float> data;  // row-major, row = wire
    float at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
};

struct SimResult {
    Frame frame;                 // M (pre-noise), float32
    Frame charge;                // S (charge grid), float32 (exact integers with fluctuation)
    std::int64_t clipped_charge = 0;
    std::int64_t clipped_patch_count = 0;
    ws_timing timing{};
};

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

inline ws_grid_spec to_c(const GridSpec& g)
{
    return ws_grid_spec{g.n_wires, g.n_ticks, g.pad_wires, g.pad_ticks, g.pitch, g.tick, g.origin_x, g.origin_t};
}

inline ws_sim_options to_c(const SimConfig& c)
{
    ws_sim_options o{};
    o.fluctuate = c.fluctuate ? 1 : 0;
    o.approx = c.approx ? 1 : 0;
    o.rng_mode = c.rng.mode == RngMode::philox ? WS_RNG_PHILOX : WS_RNG_SUBSTREAM;
    o.seed = c.rng.seed;
    o.drift.enabled = c.drift.enabled ? 1 : 0;
    o.drift.response_plane_x = c.drift.response_plane_x;
    o.drift.drift_speed = c.drift.drift_speed;
    o.drift.diffusion_long = c.drift.diffusion_long;
    o.drift.diffusion_tran = c.drift.diffusion_tran;
    return o;
}

// RAII context: one device + stream + workspace.
class Context {
  public:
    explicit Context(int device = 0, void* stream = nullptr) { check(ws_ctx_create(device, stream, &m_ctx)); }
    ~Context() { ws_ctx_destroy(m_ctx); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    ws_ctx* get() const { return m_ctx; }
    void synchronize() { check(ws_ctx_synchronize(m_ctx)); }

  private:
    ws_ctx* m_ctx = nullptr;
};

// RAII plane: geometry + response precomputed once (replaces the per-call
// build_response of run_simulation, pipeline.cpp:417).
class Plane {
  public:
    Plane(Context& ctx, const GridSpec& grid, const ResponseParams& r, double n_sigma = 3.0) : m_grid(grid)
    {
        const ws_grid_spec g = to_c(grid);
        ws_response resp{};
        resp.plane_kind = r.plane_kind == PlaneKind::collection ? WS_COLLECTION : WS_INDUCTION;
        resp.shaper_order = r.shaper_order;
        resp.field_sigma_t = r.field_sigma_t;
        resp.shaper_peaking = r.shaper_peaking;
        resp.gain = r.gain;
        resp.wire_weights = r.wire_weights.data();
        resp.n_wire_weights = r.wire_weights.size();
        check(ws_plane_create(ctx.get(), &g, &resp, n_sigma, &m_plane));
    }
    ~Plane() { ws_plane_destroy(m_plane); }
    Plane(const Plane&) = delete;
    Plane& operator=(const Plane&) = delete;
    ws_plane* get() const { return m_plane; }
    const GridSpec& grid() const { return m_grid; }

    // raster -> scatter -> convolve, host buffers (the reference's data flow)
    template <class D>
    SimResult simulate(const SimConfig& config, const std::vector<D>& depos, bool want_charge = true) const
    {
        static_assert(sizeof(D) == sizeof(ws_depo) && std::is_standard_layout_v<D>,
                      "depo type must have wiresim::Depo's layout");
        SimResult res;
        const std::size_t W = m_grid.padded_wires(), T = m_grid.padded_ticks();
        res.frame = Frame{m_grid, W, T, std::vector<float>(W * T)};
        if (want_charge) res.charge = Frame{m_grid, W, T, std::vector<float>(W * T)};
        const ws_sim_options o = to_c(config);
        check(ws_simulate_plane(m_plane, reinterpret_cast<const ws_depo*>(depos.data()), depos.size(), &o,
                                res.frame.data.data(), want_charge ? res.charge.data.data() : nullptr, &res.timing));
        res.clipped_charge = res.timing.clipped_charge;
        res.clipped_patch_count = res.timing.clipped_patches;
        return res;
    }

  private:
    GridSpec m_grid;
    ws_plane* m_plane = nullptr;
};

// run_simulation (pipeline.hpp:104) up to the pre-noise frame.
template <class D>
SimResult run_simulation(const SimConfig& config, const std::vector<D>& depos, int device = 0)
{
    Context ctx(device);
    Plane plane(ctx, config.grid, config.response, config.n_sigma);
    return plane.simulate(config, depos);
}

// ---- signal processing (sigproc.hpp, the paper's Listing 1) ---------------
// SignalBatch (sigproc.hpp:17-29): rows x cols complex spectra (row-major),
// pad_rows guard rows before the out_rows of interest.
struct SignalBatch {
    std::size_t rows = 0, cols = 0;
    std::vector<std::complex<double>> data;
    std::size_t pad_rows = 0;
    std::size_t out_rows = 0;
};

// ChainResult (sigproc.hpp:53-57): block (out_rows x cols, row-major), one
// median per block row, the imaginary-residue diagnostic.
struct ChainResult {
    std::size_t rows = 0, cols = 0;
    std::vector<double> block;
    std::vector<double> medians;
    double max_rel_imag = 0.0;
};

// sigproc_chain (sigproc.cpp:104-118) on the GPU: filter -> inverse DFT along
// rows -> block [pad_rows, pad_rows + out_rows) -> row medians. The reference's
// invalid_argument cases (filter length, pad + out > rows) throw the same type.
inline ChainResult sigproc_chain(Context& ctx, const SignalBatch& batch,
                                 const std::vector<std::complex<double>>& filter)
{
    ChainResult r;
    r.rows = batch.out_rows;
    r.cols = batch.cols;
    r.block.resize(batch.out_rows * batch.cols);
    r.medians.resize(batch.out_rows);
    ws_signal_batch b{reinterpret_cast<const double*>(batch.data.data()), batch.rows, batch.cols, batch.pad_rows,
                      batch.out_rows};
    check(ws_sigproc_chain(ctx.get(), &b, reinterpret_cast<const double*>(filter.data()), filter.size(), 1,
                           r.block.data(), r.medians.data(), &r.max_rel_imag));
    return r;
}

// load_depos (pipeline.cpp:226-262): the native CSV reader, same validation and
// std::runtime_error messages. Depo must be layout-compatible with ws_depo.
template <class D = ws_depo>
std::vector<D> load_depos(const std::string& path)
{
    static_assert(sizeof(D) == sizeof(ws_depo), "Depo layout must match ws_depo");
    ws_depo* p = nullptr;
    std::uint64_t n = 0;
    check(ws_load_depos_csv(path.c_str(), 0, &p, &n));
    std::vector<D> out(n);
    if (n) std::memcpy(static_cast<void*>(out.data()), p, n * sizeof(ws_depo));
    ws_free_depos(p, 0);
    return out;
}

}  // namespace wiresim_b200
