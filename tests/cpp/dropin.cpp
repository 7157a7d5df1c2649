// C++ drop-in check: the reference-shaped C++ interface (include/wiresim_b200.hpp)
// over the C ABI. Simulates one plane and writes the frame (float32, padded,
// row-major) to argv[1]; exit code 0 on success. Built and run by
// tests/test_gpu_parity.py::test_cpp_dropin.
#include <complex>
#include <cstdio>
#include <string>
#include <vector>

#include "wiresim_b200.hpp"

int main(int argc, char** argv)
{
    if (argc < 2) return 2;
    wiresim_b200::SimConfig cfg;
    cfg.grid.n_wires = 64;
    cfg.grid.n_ticks = 800;
    cfg.grid.pad_wires = 20;
    cfg.response.plane_kind = wiresim_b200::PlaneKind::induction;
    cfg.response.wire_weights = {0.1, 1.0, 0.1};
    cfg.fluctuate = false;
    std::vector<wiresim_b200::Depo> depos(std::vector<wiresim_b200::Depo>::size_type(300));
    for (std::size_t i = 0; i < depos.size(); ++i) {
        depos[i].id = (int64_t)i;
        depos[i].t = 20.0 + 0.9 * (double)i;
        depos[i].x = 30.0 + 0.8 * (double)i;
        depos[i].q = 1000 + (int64_t)(i * 37 % 9000);
        depos[i].sigma_t = 0.5 + 0.003 * (double)i;
        depos[i].sigma_x = 2.5 + 0.01 * (double)i;
    }
    try {
        const wiresim_b200::SimResult r = wiresim_b200::run_simulation(cfg, depos);
        FILE* f = std::fopen(argv[1], "wb");
        if (!f) return 3;
        std::fwrite(r.frame.data.data(), sizeof(float), r.frame.data.size(), f);
        std::fclose(f);
        std::printf("frame %zux%zu clipped %lld\n", r.frame.rows, r.frame.cols, (long long)r.clipped_charge);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    // depo CSV ingestion (load_depos, pipeline.cpp:226-262) through the C++ mirror
    {
        const std::string csv = std::string(argv[1]) + ".csv";
        if (ws_save_depos_csv(csv.c_str(), reinterpret_cast<const ws_depo*>(depos.data()), depos.size()) != WS_OK)
            return 5;
        const std::vector<wiresim_b200::Depo> back = wiresim_b200::load_depos<wiresim_b200::Depo>(csv);
        if (back.size() != depos.size()) return 6;
        for (std::size_t i = 0; i < back.size(); ++i)
            if (back[i].t != depos[i].t || back[i].x != depos[i].x || back[i].q != depos[i].q ||
                back[i].sigma_t != depos[i].sigma_t || back[i].sigma_x != depos[i].sigma_x)
                return 7;
        FILE* f = std::fopen(csv.c_str(), "w");
        std::fputs("id,t,x\n", f);
        std::fclose(f);
        try {
            wiresim_b200::load_depos<wiresim_b200::Depo>(csv);
            return 8;
        } catch (const std::runtime_error&) {
        }
    }
    // sigproc_chain (sigproc.cpp:104-118): a Hermitian row (spectrum of a real
    // impulse at sample 3) through an identity filter comes back as the impulse
    {
        wiresim_b200::Context ctx;
        wiresim_b200::SignalBatch b;
        b.rows = 2;
        b.cols = 12;
        b.pad_rows = 1;
        b.out_rows = 1;
        b.data.resize(b.rows * b.cols);
        for (std::size_t r = 0; r < b.rows; ++r)
            for (std::size_t k = 0; k < b.cols; ++k)
                b.data[r * b.cols + k] = std::polar(1.0, -2.0 * 3.14159265358979323846 * 3.0 * (double)k / 12.0);
        const std::vector<std::complex<double>> ones(b.cols, 1.0);
        const wiresim_b200::ChainResult c = wiresim_b200::sigproc_chain(ctx, b, ones);
        for (std::size_t t = 0; t < b.cols; ++t)
            if (std::abs(c.block[t] - (t == 3 ? 1.0 : 0.0)) > 1e-12) return 9;
        if (c.medians.size() != 1 || std::abs(c.medians[0]) > 1e-12) return 10;
        try {
            wiresim_b200::sigproc_chain(ctx, b, std::vector<std::complex<double>>(5, 1.0));
            return 11;
        } catch (const std::invalid_argument&) {
        }
    }
    // the reference's exception categories cross back as the same C++ types
    try {
        wiresim_b200::SimConfig bad = cfg;
        bad.response.wire_weights = {1.0, 1.0};
        wiresim_b200::run_simulation(bad, depos);
        return 4;
    } catch (const std::invalid_argument&) {
    }
    return 0;
}
