// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI harness around the UNMODIFIED reference library (`wiresim`, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu-baseline / reference arm
// load the resulting oracle/_ref/libwsref.so, and only as the checker or as the
// timed CPU reference -- never as the product path.
//
// Every entry point calls public reference functions; the only glue is what the
// reference itself lacks:
//   * fluctuation-off charge: sample_patch (rasterize.cpp:66-120) -> S += q*p in
//     fp64, skipping empty patches (pipeline.cpp:339-340);
//   * real-valued convolve: fft_2d (fft.cpp:171-198) forward, * build_response
//     values (spectral.cpp:87-139), inverse, real part -- mirrors convolve
//     (spectral.cpp:155-173), which only accepts the int64 ChargeGrid;
//   * PhiloxSource : RandomSource (rng.hpp:62-67), the shared counter-based
//     stream the GPU path implements bit-identically.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <string>
#include <thread>
#include <vector>
#include <unistd.h>

#include "wiresim/core.hpp"
#include "wiresim/fft.hpp"
#include "wiresim/pipeline.hpp"
#include "wiresim/rasterize.hpp"
#include "wiresim/rng.hpp"
#include "wiresim/scatter.hpp"
#include "wiresim/sigproc.hpp"
#include "wiresim/spectral.hpp"
#include "wiresim/threading.hpp"

using namespace wiresim;

namespace {

thread_local std::string g_err;

struct wsr_grid {
    std::uint64_t n_wires, n_ticks, pad_wires, pad_ticks;
    double pitch, tick, origin_x, origin_t;
};

struct wsr_response {
    std::int32_t plane_kind;  // 0 induction, 1 collection
    std::int32_t shaper_order;
    double field_sigma_t;
    double shaper_peaking;
    double gain;
    const double* wire_weights;
    std::uint64_t n_wire_weights;
};

static_assert(sizeof(Depo) == 48, "Depo layout");

GridSpec to_spec(const wsr_grid* g)
{
    GridSpec s;
    s.n_wires = g->n_wires;
    s.n_ticks = g->n_ticks;
    s.pad_wires = g->pad_wires;
    s.pad_ticks = g->pad_ticks;
    s.pitch = g->pitch;
    s.tick = g->tick;
    s.origin_x = g->origin_x;
    s.origin_t = g->origin_t;
    return s;
}

ResponseParams to_resp(const wsr_response* r)
{
    ResponseParams p;
    p.plane_kind = r->plane_kind == 0 ? PlaneKind::induction : PlaneKind::collection;
    p.field_sigma_t = r->field_sigma_t;
    p.shaper_peaking = r->shaper_peaking;
    p.shaper_order = r->shaper_order;
    p.gain = r->gain;
    p.wire_weights.assign(r->wire_weights, r->wire_weights + r->n_wire_weights);
    return p;
}

std::vector<Depo> to_depos(const Depo* d, std::uint64_t n)
{
    return std::vector<Depo>(d, d + n);
}

// Philox4x32-10 (Salmon et al., SC'11), the shared counter-based stream.
// key = (seed lo, seed hi); draw i uses block ctr = (i >> 1, id lo, id hi, 0)
// and words (2*(i&1), 2*(i&1)+1) as (hi, lo) of a u64; u = (u64 >> 11) * 2^-53
// mirrors uniform01 (rng.cpp:51-54).
void philox4x32_10(const std::uint32_t ctr_in[4], const std::uint32_t key_in[2], std::uint32_t out[4])
{
    std::uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    std::uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        const std::uint64_t p0 = static_cast<std::uint64_t>(0xD2511F53u) * c0;
        const std::uint64_t p1 = static_cast<std::uint64_t>(0xCD9E8D57u) * c2;
        const std::uint32_t hi0 = static_cast<std::uint32_t>(p0 >> 32), lo0 = static_cast<std::uint32_t>(p0);
        const std::uint32_t hi1 = static_cast<std::uint32_t>(p1 >> 32), lo1 = static_cast<std::uint32_t>(p1);
        const std::uint32_t n0 = hi1 ^ c1 ^ k0;
        const std::uint32_t n1 = lo1;
        const std::uint32_t n2 = hi0 ^ c3 ^ k1;
        const std::uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

class PhiloxSource final : public RandomSource {
  public:
    PhiloxSource(std::uint64_t seed, std::uint64_t id) : m_seed(seed), m_id(id) {}
    double uniform() override
    {
        const std::uint64_t i = m_draw++;
        const std::uint32_t ctr[4] = {static_cast<std::uint32_t>(i >> 1), static_cast<std::uint32_t>(m_id),
                                      static_cast<std::uint32_t>(m_id >> 32), 0u};
        const std::uint32_t key[2] = {static_cast<std::uint32_t>(m_seed), static_cast<std::uint32_t>(m_seed >> 32)};
        std::uint32_t o[4];
        philox4x32_10(ctr, key, o);
        const int h = static_cast<int>(i & 1u) * 2;
        const std::uint64_t u64 = (static_cast<std::uint64_t>(o[h]) << 32) | o[h + 1];
        return static_cast<double>(u64 >> 11) * 0x1.0p-53;
    }
    double normal() override
    {
        // StreamSource pairing semantics (rng.hpp:78-90)
        if (m_have_spare) {
            m_have_spare = false;
            return m_spare;
        }
        const double u1 = 1.0 - uniform();
        const double u2 = uniform();
        auto [z0, z1] = box_muller(u1, u2);
        m_spare = z1;
        m_have_spare = true;
        return z0;
    }

  private:
    std::uint64_t m_seed, m_id, m_draw = 0;
    double m_spare = 0.0;
    bool m_have_spare = false;
};

template <typename F>
int guarded(F&& f)
{
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown exception";
        return 1;
    }
}

double now_s()
{
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

const char* wsr_last_error() { return g_err.c_str(); }

void wsr_philox4x32_10(const std::uint32_t* ctr, const std::uint32_t* key, std::uint32_t* out)
{
    philox4x32_10(ctr, key, out);
}

// Fills `out` with `count` draws from substream(seed, id) (mode 0) or
// PhiloxSource(seed, id) (mode 1): kind 0 uniforms, kind 1 normals.
int wsr_draws(int mode, int kind, std::uint64_t seed, std::uint64_t id, std::uint64_t count, double* out)
{
    return guarded([&] {
        if (mode == 0) {
            StreamSource src(substream(seed, id));
            for (std::uint64_t i = 0; i < count; ++i) out[i] = kind ? src.normal() : src.uniform();
        } else {
            PhiloxSource src(seed, id);
            for (std::uint64_t i = 0; i < count; ++i) out[i] = kind ? src.normal() : src.uniform();
        }
    });
}

// binomial(n, p) draws (rng.cpp:174-193) from substream(seed, id).
int wsr_binomials(std::int64_t n, double p, std::uint64_t seed, std::uint64_t id, std::uint64_t count,
                  std::int64_t* out)
{
    return guarded([&] {
        StreamSource src(substream(seed, id));
        for (std::uint64_t i = 0; i < count; ++i) out[i] = binomial(n, p, src);
    });
}

int wsr_map_depo(const wsr_grid* g, const Depo* d, double n_sigma, long* out6)
{
    return guarded([&] {
        const GridFootprint fp = map_depo_to_grid(*d, to_spec(g), n_sigma);
        out6[0] = fp.center_wire; out6[1] = fp.center_tick;
        out6[2] = fp.wire_lo; out6[3] = fp.wire_hi;
        out6[4] = fp.tick_lo; out6[5] = fp.tick_hi;
    });
}

int wsr_drift(const Depo* d, const double* drift4, Depo* out)
{
    return guarded([&] {
        DriftParams p;
        p.response_plane_x = drift4[0];
        p.drift_speed = drift4[1];
        p.diffusion_long = drift4[2];
        p.diffusion_tran = drift4[3];
        p.enabled = true;
        *out = drift_depo(*d, p);
    });
}

// sample_patch (rasterize.cpp:66-120). meta = {wire_offset, tick_offset, n_w, n_t, clipped};
// values holds n_w*n_t doubles (cap elements available).
int wsr_sample_patch(const wsr_grid* g, const Depo* d, double n_sigma, long* meta, double* values,
                     std::uint64_t cap, double* captured)
{
    return guarded([&] {
        const SampledPatch sp = sample_patch(*d, to_spec(g), n_sigma);
        meta[0] = sp.patch.wire_offset;
        meta[1] = sp.patch.tick_offset;
        meta[2] = static_cast<long>(sp.patch.n_w);
        meta[3] = static_cast<long>(sp.patch.n_t);
        meta[4] = sp.clipped ? 1 : 0;
        if (sp.patch.values.size() > cap) throw std::out_of_range("wsr_sample_patch: cap too small");
        std::copy(sp.patch.values.begin(), sp.patch.values.end(), values);
        *captured = sp.captured_mass;
    });
}

// Full reference run_simulation (pipeline.cpp:345-427). rng_mode: 0 inline, 1 pool, 2 substream.
int wsr_run_simulation(const wsr_grid* g, const wsr_response* r, const Depo* d, std::uint64_t n, double n_sigma,
                       int rng_mode, std::uint64_t seed, std::uint64_t slice_len, int dispatch, int workers,
                       int scatter_atomic, int drift_enabled, const double* drift4, int noise_mode,
                       double noise_sigma, const double* noise_spectrum, std::uint64_t n_spectrum,
                       double adc_scale, double adc_offset, int adc_bits, std::int64_t* charge_out,
                       std::int32_t* adc_out, std::int64_t* clipped_charge, double* timing6)
{
    return guarded([&] {
        SimConfig c;
        c.grid = to_spec(g);
        c.response = to_resp(r);
        c.n_sigma = n_sigma;
        c.rng.mode = rng_mode == 0 ? RngMode::inline_stream : rng_mode == 1 ? RngMode::pool : RngMode::substream;
        c.rng.seed = seed;
        c.rng.slice_len = slice_len;
        c.dispatch = dispatch ? DispatchMode::per_depo : DispatchMode::batched;
        c.workers = workers;
        c.scatter = scatter_atomic ? ScatterStrategy::atomic : ScatterStrategy::banded;
        if (drift_enabled) {
            c.drift.enabled = true;
            c.drift.response_plane_x = drift4[0];
            c.drift.drift_speed = drift4[1];
            c.drift.diffusion_long = drift4[2];
            c.drift.diffusion_tran = drift4[3];
        }
        c.noise.mode = noise_mode == 0 ? NoiseMode::off : noise_mode == 1 ? NoiseMode::white : NoiseMode::spectrum;
        c.noise.sigma = noise_sigma;
        if (noise_spectrum) c.noise.amplitude_spectrum.assign(noise_spectrum, noise_spectrum + n_spectrum);
        c.adc.scale = adc_scale;
        c.adc.offset = adc_offset;
        c.adc.bits = adc_bits;
        const SimResult res = run_simulation(c, to_depos(d, n));
        if (charge_out) std::copy(res.charge.counts.data.begin(), res.charge.counts.data.end(), charge_out);
        if (adc_out) std::copy(res.adc.data.begin(), res.adc.data.end(), adc_out);
        if (clipped_charge) *clipped_charge = res.clipped_charge;
        if (timing6) {
            timing6[0] = res.timing.rasterization_total_s;
            timing6[1] = res.timing.sampling_2d_s;
            timing6[2] = res.timing.fluctuation_s;
            timing6[3] = res.timing.scatter_add_s;
            timing6[4] = res.timing.ft_s;
            timing6[5] = res.timing.total_s;
        }
    });
}

// ResponseKernel (spectral.cpp:87-139): complex values (interleaved, W_p x T_p) and supports.
int wsr_build_response(const wsr_grid* g, const wsr_response* r, double* values_c128, long* support2)
{
    return guarded([&] {
        const ResponseKernel k = build_response(to_spec(g), to_resp(r));
        if (values_c128) std::memcpy(values_c128, k.values.data.data(), k.values.data.size() * sizeof(cdouble));
        support2[0] = k.support_ticks;
        support2[1] = k.support_wires;
    });
}

// convolve (spectral.cpp:141-175) on an int64 charge grid.
int wsr_convolve_int(const wsr_grid* g, const wsr_response* r, const std::int64_t* s, double* m, int workers)
{
    return guarded([&] {
        const GridSpec spec = to_spec(g);
        ChargeGrid cg(spec);
        std::copy(s, s + cg.counts.data.size(), cg.counts.data.begin());
        const ResponseKernel k = build_response(spec, to_resp(r));
        const MeasurementGrid mg = convolve(cg, k, workers);
        std::copy(mg.samples.data.begin(), mg.samples.data.end(), m);
    });
}

// Real-valued S through the same FT / multiply / IFT as convolve (spectral.cpp:155-173).
int wsr_convolve_real(const wsr_grid* g, const wsr_response* r, const double* s, double* m, int workers)
{
    return guarded([&] {
        const GridSpec spec = to_spec(g);
        const ResponseKernel k = build_response(spec, to_resp(r));
        Matrix<cdouble> spec_m(spec.padded_wires(), spec.padded_ticks());
        for (std::size_t i = 0; i < spec_m.data.size(); ++i) spec_m.data[i] = cdouble{s[i], 0.0};
        spec_m = fft_2d(spec_m, FftDirection::forward, workers);
        for (std::size_t i = 0; i < spec_m.data.size(); ++i) spec_m.data[i] *= k.values.data[i];
        spec_m = fft_2d(spec_m, FftDirection::inverse, workers);
        for (std::size_t i = 0; i < spec_m.data.size(); ++i) m[i] = spec_m.data[i].real();
    });
}

// Fluctuation-off charge: sample_patch -> S += q * p (fp64), empty patches
// count as clipped charge (pipeline.cpp:339-340). Optional drift first
// (pipeline.cpp:358-362).
int wsr_fluct_off_charge(const wsr_grid* g, const Depo* d, std::uint64_t n, double n_sigma, int drift_enabled,
                         const double* drift4, double* s, std::int64_t* clipped_charge)
{
    return guarded([&] {
        const GridSpec spec = to_spec(g);
        const std::size_t cols = spec.padded_ticks();
        DriftParams dp;
        if (drift_enabled) {
            dp.response_plane_x = drift4[0];
            dp.drift_speed = drift4[1];
            dp.diffusion_long = drift4[2];
            dp.diffusion_tran = drift4[3];
        }
        std::int64_t clipped = 0;
        for (std::uint64_t i = 0; i < n; ++i) {
            const Depo depo = drift_enabled ? drift_depo(d[i], dp) : d[i];
            const SampledPatch sp = sample_patch(depo, spec, n_sigma);
            if (sp.patch.empty()) {
                clipped += depo.q;
                continue;
            }
            const double q = static_cast<double>(depo.q);
            for (std::size_t w = 0; w < sp.patch.n_w; ++w)
                for (std::size_t t = 0; t < sp.patch.n_t; ++t)
                    s[(static_cast<std::size_t>(sp.patch.wire_offset) + w) * cols +
                      static_cast<std::size_t>(sp.patch.tick_offset) + t] += q * sp.patch.at(w, t);
        }
        if (clipped_charge) *clipped_charge = clipped;
    });
}

// Fluctuation-on charge with the shared Philox stream: unmodified
// fluctuate / fluctuate_approx (rasterize.cpp:153-170) fed by PhiloxSource,
// then scatter_add (scatter.cpp:27-36). approx: 0 exact binomial, 1 Gaussian approx.
int wsr_fluct_philox_charge(const wsr_grid* g, const Depo* d, std::uint64_t n, double n_sigma, std::uint64_t seed,
                            int approx, std::int64_t* s, std::int64_t* clipped_charge)
{
    return guarded([&] {
        const GridSpec spec = to_spec(g);
        ChargeGrid cg(spec);
        std::int64_t clipped = 0;
        for (std::uint64_t i = 0; i < n; ++i) {
            const SampledPatch sp = sample_patch(d[i], spec, n_sigma);
            PhiloxSource src(seed, static_cast<std::uint64_t>(d[i].id));
            const std::int64_t q = sp.patch.empty() ? 0 : d[i].q;
            const CountPatch cp = approx ? fluctuate_approx(sp.patch, q, src) : fluctuate(sp.patch, q, src);
            if (sp.patch.empty()) clipped += d[i].q;
            scatter_add(cg, cp);
        }
        std::copy(cg.counts.data.begin(), cg.counts.data.end(), s);
        if (clipped_charge) *clipped_charge = clipped;
    });
}

// gen_depos (pipeline.cpp:264-294) round-tripped through its CSV file and
// load_depos (pipeline.cpp:226-262), exactly as the CLI does.
int wsr_gen_depos(std::uint64_t n, std::uint64_t seed, const wsr_grid* g, Depo* out)
{
    return guarded([&] {
        char tmpl[] = "/tmp/wsr_depos_XXXXXX";
        const int fd = mkstemp(tmpl);
        if (fd < 0) throw std::runtime_error("mkstemp failed");
        close(fd);
        const std::filesystem::path path(tmpl);
        gen_depos(n, seed, to_spec(g), DepoGenRanges{}, path);
        const std::vector<Depo> depos = load_depos(path);
        std::filesystem::remove(path);
        std::copy(depos.begin(), depos.end(), out);
    });
}

// gen_depos (pipeline.cpp:264-294) to a CSV file, unmodified (golden input files).
int wsr_gen_depos_csv(std::uint64_t n, std::uint64_t seed, const wsr_grid* g, const char* path)
{
    return guarded([&] { gen_depos(n, seed, to_spec(g), DepoGenRanges{}, path); });
}

int wsr_load_depos(const char* path, Depo* out, std::uint64_t cap, std::uint64_t* n_out)
{
    return guarded([&] {
        const std::vector<Depo> depos = load_depos(path);
        *n_out = depos.size();
        if (depos.size() > cap) throw std::out_of_range("wsr_load_depos: cap too small");
        std::copy(depos.begin(), depos.end(), out);
    });
}

// add_noise (spectral.cpp:177-226) then digitize (spectral.cpp:228-238) on a double frame.
int wsr_noise_digitize(const wsr_grid* g, const double* m, int noise_mode, double sigma, const double* spectrum,
                       std::uint64_t n_spectrum, std::uint64_t seed, double scale, double offset, int bits,
                       double* m_noisy, std::int32_t* adc, int workers)
{
    return guarded([&] {
        const GridSpec spec = to_spec(g);
        MeasurementGrid mg(spec);
        std::copy(m, m + mg.samples.data.size(), mg.samples.data.begin());
        NoiseModel model;
        model.mode = noise_mode == 0 ? NoiseMode::off : noise_mode == 1 ? NoiseMode::white : NoiseMode::spectrum;
        model.sigma = sigma;
        if (spectrum) model.amplitude_spectrum.assign(spectrum, spectrum + n_spectrum);
        const MeasurementGrid noisy = add_noise(mg, model, seed, workers);
        if (m_noisy) std::copy(noisy.samples.data.begin(), noisy.samples.data.end(), m_noisy);
        if (adc) {
            const Matrix<std::int32_t> a = digitize(noisy, scale, offset, bits);
            std::copy(a.data.begin(), a.data.end(), adc);
        }
    });
}

// CPU reference timing of the fluctuation-off hot path, each stage with the
// reference's own parallel primitives at `workers` threads:
//   sample  : sample_patch per depo, parallel_for over depos (as rasterize_range, pipeline.cpp:328-331)
//   scatter : fp64 q*p accumulation, wire-banded ownership (as scatter_banded, scatter.cpp:42-59)
//   convolve: fft_2d fwd (workers) * R * fft_2d inv (workers), real part (spectral.cpp:155-173)
// The response kernel is built once per plane (wsr_plane_create, timed into
// build_s) and reused: it is per-geometry and cacheable.
struct WsrPlane {
    GridSpec spec;
    ResponseKernel kernel;
    double build_s = 0.0;
};

void* wsr_plane_create(const wsr_grid* g, const wsr_response* r, double* build_s)
{
    WsrPlane* p = nullptr;
    const int rc = guarded([&] {
        p = new WsrPlane();
        p->spec = to_spec(g);
        const double t0 = now_s();
        p->kernel = build_response(p->spec, to_resp(r));
        p->build_s = now_s() - t0;
    });
    if (rc) {
        delete p;
        return nullptr;
    }
    if (build_s) *build_s = p->build_s;
    return p;
}

void wsr_plane_destroy(void* p) { delete static_cast<WsrPlane*>(p); }

// times = {sample_s, scatter_s, convolve_s}
int wsr_plane_time_fluct_off(void* handle, const Depo* d, std::uint64_t n, double n_sigma, int workers, double* m_out,
                             double* times)
{
    return guarded([&] {
        const WsrPlane& P = *static_cast<WsrPlane*>(handle);
        const GridSpec& spec = P.spec;
        const std::vector<Depo> depos = to_depos(d, n);
        std::vector<SampledPatch> patches(n);
        const double t0 = now_s();
        parallel_for(n, workers, [&](std::size_t lo, std::size_t hi, int) {
            for (std::size_t i = lo; i < hi; ++i) patches[i] = sample_patch(depos[i], spec, n_sigma);
        });
        const double t1 = now_s();
        const std::size_t rows = spec.padded_wires(), cols = spec.padded_ticks();
        Matrix<cdouble> grid(rows, cols);
        parallel_for(rows, workers, [&](std::size_t band_lo, std::size_t band_hi, int) {
            for (std::size_t i = 0; i < n; ++i) {
                const ProbPatch& p = patches[i].patch;
                if (p.empty()) continue;
                const std::size_t plo = static_cast<std::size_t>(p.wire_offset);
                const std::size_t lo = std::max(band_lo, plo), hi = std::min(band_hi, plo + p.n_w);
                const double q = static_cast<double>(depos[i].q);
                for (std::size_t w = lo; w < hi; ++w) {
                    cdouble* dst = grid.row_ptr(w) + p.tick_offset;
                    const double* src = p.values.data() + (w - plo) * p.n_t;
                    for (std::size_t t = 0; t < p.n_t; ++t) dst[t] += q * src[t];
                }
            }
        });
        const double t2 = now_s();
        grid = fft_2d(grid, FftDirection::forward, workers);
        for (std::size_t i = 0; i < grid.data.size(); ++i) grid.data[i] *= P.kernel.values.data[i];
        grid = fft_2d(grid, FftDirection::inverse, workers);
        if (m_out)
            for (std::size_t i = 0; i < grid.data.size(); ++i) m_out[i] = grid.data[i].real();
        const double t3 = now_s();
        times[0] = t1 - t0;
        times[1] = t2 - t1;
        times[2] = t3 - t2;
    });
}

// One-shot variant (builds the response, timed separately into times[3]).
int wsr_time_fluct_off(const wsr_grid* g, const wsr_response* r, const Depo* d, std::uint64_t n, double n_sigma,
                       int workers, double* m_out, double* times)
{
    void* p = wsr_plane_create(g, r, &times[3]);
    if (!p) return 1;
    const int rc = wsr_plane_time_fluct_off(p, d, n, n_sigma, workers, m_out, times);
    wsr_plane_destroy(p);
    return rc;
}

// sigproc_chain (sigproc.cpp:104-118), unmodified; data/filter are interleaved
// complex. seconds (nullable) = wall time of the chain call alone.
int wsr_sigproc_chain(const double* data, std::uint64_t rows, std::uint64_t cols, std::uint64_t pad_rows,
                      std::uint64_t out_rows, const double* filter, int workers, double* block, double* medians,
                      double* max_rel_imag, double* seconds)
{
    return guarded([&] {
        SignalBatch batch;
        batch.data = Matrix<cdouble>(rows, cols);
        std::memcpy(static_cast<void*>(batch.data.data.data()), data, sizeof(double) * 2 * rows * cols);
        batch.pad_rows = pad_rows;
        batch.out_rows = out_rows;
        std::vector<cdouble> f(cols);
        std::memcpy(static_cast<void*>(f.data()), filter, sizeof(double) * 2 * cols);
        const auto t0 = std::chrono::steady_clock::now();
        const ChainResult r = sigproc_chain(batch, f, workers);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (block) std::copy(r.block.data.begin(), r.block.data.end(), block);
        if (medians) std::copy(r.medians.begin(), r.medians.end(), medians);
        if (max_rel_imag) *max_rel_imag = r.max_rel_imag;
    });
}

double wsr_row_median(const double* v, std::uint64_t n, int by_sort)
{
    const std::span<const double> s(v, n);
    return by_sort ? row_median_by_sort(s) : row_median(s);
}

}  // extern "C"
