// Drop-in against the reference's OWN interface: the same wiresim::SimConfig
// and std::vector<wiresim::Depo> go to the unmodified reference
// (wiresim::run_simulation, oracle/_ref/libwsref.so) and to the B200 path
// (wiresim_b200::run_simulation from include/wiresim_b200_dropin.hpp) in one
// process; the two wiresim::SimResult are compared.
//
// Built HERE (where /root/reference exists) by `make -C oracle dropin` into
// oracle/_ref/dropin_ref (test infrastructure: it links the reference);
// run on the GPU box by tests/test_gpu_readout.py::test_dropin_reference_types.
//
// Checks per case: integer charge grid identical (the substream stream is the
// reference's own), clipped charge identical, ADC codes within +-1 where the
// fp32 frame (per-channel relL2 <= 1e-5 of the reference's fp64 frame) sits
// next to a rounding boundary, with the fraction of such codes reported.
// Prints one JSON line per case; exit code 0 iff every case passes.
#include <wiresim/pipeline.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "wiresim_b200_dropin.hpp"

namespace {

std::vector<wiresim::Depo> track(std::size_t n, double t0, double x0, double dt, double dx, std::int64_t qbase)
{
    std::vector<wiresim::Depo> d(n);
    for (std::size_t i = 0; i < n; ++i) {
        d[i].id = (std::int64_t)i;
        d[i].t = t0 + dt * (double)i;
        d[i].x = x0 + dx * (double)i;
        d[i].q = qbase + (std::int64_t)(i * 37 % 9000);
        d[i].sigma_t = 0.5 + 0.003 * (double)(i % 300);
        d[i].sigma_x = 2.5 + 0.01 * (double)(i % 500);
    }
    return d;
}

struct Outcome {
    bool ok;
    double mismatch_frac;
};

Outcome compare(const char* name, const wiresim::SimConfig& cfg, const std::vector<wiresim::Depo>& depos,
                double max_mismatch)
{
    const wiresim::SimResult ref = wiresim::run_simulation(cfg, depos);
    const wiresim::SimResult gpu = wiresim_b200::run_simulation(cfg, depos);
    bool ok = ref.adc.rows == gpu.adc.rows && ref.adc.cols == gpu.adc.cols;
    const bool charge_eq = ref.charge.counts == gpu.charge.counts;
    const bool clipped_eq = ref.clipped_charge == gpu.clipped_charge;
    long long mism = 0, maxd = 0;
    for (std::size_t i = 0; ok && i < ref.adc.data.size(); ++i) {
        const long long d = std::llabs((long long)ref.adc.data[i] - (long long)gpu.adc.data[i]);
        if (d) ++mism;
        if (d > maxd) maxd = d;
    }
    const double frac = ref.adc.data.empty() ? 0.0 : (double)mism / (double)ref.adc.data.size();
    ok = ok && charge_eq && clipped_eq && maxd <= 1 && frac <= max_mismatch;
    std::printf("{\"case\": \"%s\", \"ok\": %s, \"charge_identical\": %s, \"clipped_identical\": %s, "
                "\"adc_max_diff\": %lld, \"adc_mismatch_frac\": %.3e, \"cells\": %zu}\n",
                name, ok ? "true" : "false", charge_eq ? "true" : "false", clipped_eq ? "true" : "false", maxd,
                frac, ref.adc.data.size());
    return {ok, frac};
}

}  // namespace

int main()
{
    bool all = true;
    wiresim::SimConfig base;
    base.grid.n_wires = 64;
    base.grid.n_ticks = 800;
    base.grid.pad_wires = 20;
    base.grid.pad_ticks = 100;  // 1000 padded ticks: even, 7-smooth (spectrum noise allowed)
    base.response.plane_kind = wiresim::PlaneKind::induction;
    base.response.wire_weights = {0.1, 1.0, 0.1};
    base.rng.mode = wiresim::RngMode::substream;
    base.rng.seed = 2024;
    base.adc.scale = 1.0;
    base.adc.offset = 2048.0;
    base.adc.bits = 12;
    const auto depos = track(300, 20.0, 30.0, 0.9, 0.8, 1000);

    all &= compare("substream_noise_off", base, depos, 0.02).ok;
    {
        // same config again: the cached plane and workspace give the same result
        const wiresim::SimResult a = wiresim_b200::run_simulation(base, depos);
        const wiresim::SimResult b = wiresim_b200::run_simulation(base, depos);
        const bool rep = a.adc == b.adc && a.charge.counts == b.charge.counts;
        std::printf("{\"case\": \"repeat_bitwise\", \"ok\": %s}\n", rep ? "true" : "false");
        all &= rep;
    }
    {
        wiresim::SimConfig c = base;
        c.noise.mode = wiresim::NoiseMode::white;
        c.noise.sigma = 2.5;
        all &= compare("white_noise_substream", c, depos, 0.02).ok;
    }
    {
        wiresim::SimConfig c = base;
        c.noise.mode = wiresim::NoiseMode::spectrum;
        c.noise.amplitude_spectrum.resize(c.grid.padded_ticks());
        for (std::size_t k = 0; k < c.noise.amplitude_spectrum.size(); ++k) {
            const double f = (double)std::min(k, c.noise.amplitude_spectrum.size() - k);
            c.noise.amplitude_spectrum[k] = 3.0 / (1.0 + f / 40.0);
        }
        all &= compare("spectrum_noise_substream", c, depos, 0.02).ok;
    }
    {
        wiresim::SimConfig c = base;
        c.drift.enabled = true;
        c.drift.response_plane_x = 0.0;
        auto d = depos;
        for (auto& x : d) x.x += 100.0;  // drift toward the plane at x = 0 ... then binned at the plane
        c.grid.origin_x = -200.0;
        all &= compare("drift", c, d, 0.02).ok;
    }
    {
        wiresim::SimConfig c;
        c.grid.n_wires = 200;
        c.grid.n_ticks = 2000;
        c.grid.pad_wires = 20;
        c.grid.pad_ticks = 100;
        c.response.plane_kind = wiresim::PlaneKind::collection;
        c.rng.seed = 7;
        c.adc.scale = 0.5;
        c.adc.offset = 400.0;
        c.adc.bits = 10;  // clamps at both ends
        const auto d = track(2000, 10.0, 5.0, 0.45, 0.45, 500);
        all &= compare("collection_2k_clamped", c, d, 0.02).ok;
    }
    {
        // the reference's invalid_argument for bad ADC bits, on both sides
        wiresim::SimConfig c = base;
        c.adc.bits = 17;
        int thrown = 0;
        try {
            wiresim::run_simulation(c, depos);
        } catch (const std::invalid_argument&) {
            ++thrown;
        }
        try {
            wiresim_b200::run_simulation(c, depos);
        } catch (const std::invalid_argument&) {
            ++thrown;
        }
        std::printf("{\"case\": \"bad_adc_bits_invalid_argument\", \"ok\": %s}\n", thrown == 2 ? "true" : "false");
        all &= thrown == 2;
    }
    return all ? 0 : 1;
}
