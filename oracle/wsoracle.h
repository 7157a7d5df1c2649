/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU restatement (plain C11, libm) of the reference hot path
 * (/root/reference/proj, `wiresim`): rasterize -> fluctuate -> scatter-add ->
 * response build -> circular convolution, plus the noise / digitize epilogue.
 * Each function cites the reference file:line it restates. It is the checker
 * for the CUDA path; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here bit-for-bit
 * against the unmodified reference compiled into oracle/_ref/libwsref.so and
 * against committed golden vectors in tests/golden/ (generated from that
 * library by tests/golden/make_golden.py), including the survey anchor
 * FNV-1a(S) = 9be5e6dc3d524726 for gen_depos(10000, seed 7) on a 480x6000 grid.
 *
 * Struct layouts are identical to the product ABI (include/wiresim_gpu.h).
 */
#ifndef WSORACLE_H
#define WSORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t n_wires, n_ticks, pad_wires, pad_ticks;
    double pitch, tick, origin_x, origin_t;
} wso_grid;

typedef struct {
    int64_t id;
    double t, x;
    int64_t q;
    double sigma_t, sigma_x;
} wso_depo;

typedef struct {
    int32_t plane_kind; /* 0 induction, 1 collection */
    int32_t shaper_order;
    double field_sigma_t, shaper_peaking, gain;
    const double* wire_weights;
    uint64_t n_wire_weights;
} wso_response;

typedef struct {
    double response_plane_x, drift_speed, diffusion_long, diffusion_tran;
} wso_drift;

/* random source: mode 0 = xoshiro256** substream, 1 = Philox4x32-10 */
typedef struct {
    int mode;
    uint64_t s[4];
    uint64_t seed, id, draw;
    double spare;
    int have_spare;
} wso_src;

const char* wso_last_error(void);

uint64_t wso_splitmix64_next(uint64_t* state);
void wso_seed_state(uint64_t seed, uint64_t s[4]);
void wso_substream(uint64_t seed, uint64_t stream_id, uint64_t s[4]);
uint64_t wso_next_u64(uint64_t s[4]);
double wso_uniform01(uint64_t s[4]);
void wso_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void wso_src_init(wso_src* src, int mode, uint64_t seed, uint64_t id);
double wso_src_uniform(wso_src* src);
double wso_src_normal(wso_src* src);
int wso_binomial(int64_t n, double p, wso_src* src, int64_t* k);

int wso_map_depo(const wso_grid* g, const wso_depo* d, double n_sigma, long out6[6]);
int wso_drift_depo(const wso_depo* d, const wso_drift* p, wso_depo* out);
void wso_gauss_bin_integrals(double center, double sigma, double lo_edge, double spacing, size_t n, double* vals);
int wso_sample_patch(const wso_grid* g, const wso_depo* d, double n_sigma, long meta[5], double* values,
                     size_t cap, double* captured);
int wso_fluctuate(const double* p, size_t n, int64_t q, wso_src* src, int approx, int64_t* out);

int wso_charge_fluct_off(const wso_grid* g, const wso_depo* d, size_t n, double n_sigma, const wso_drift* drift,
                         double* s, int64_t* clipped_charge);
int wso_charge_fluct_on(const wso_grid* g, const wso_depo* d, size_t n, double n_sigma, const wso_drift* drift,
                        int rng_mode, int approx, uint64_t seed, int64_t* s, int64_t* clipped_charge);

int wso_response_td(const wso_grid* g, const wso_response* r, double* combined, size_t cap, long* lo_lag,
                    size_t* n_lags, long* support_ticks, long* support_wires);
int wso_convolve_direct(const wso_grid* g, const wso_response* r, const double* s, double* m);

int wso_add_white_noise_rng(const wso_grid* g, double sigma, uint64_t seed, int rng_mode, double* m);
int wso_add_white_noise(const wso_grid* g, double sigma, uint64_t seed, double* m);
int wso_digitize(const double* m, size_t n, double scale, double offset, int bits, int32_t* adc);

uint64_t wso_fnv1a64(const void* data, size_t nbytes);

/* sigproc (sigproc.cpp:12-118). data: rows x cols complex (interleaved re,im),
 * filter: cols complex. block: out_rows x cols, medians: out_rows (nullable).
 * max_rel_imag = max |imag| / max |real| over all rows (workers = 1). */
double wso_row_median(const double* v, size_t n);
int wso_sigproc_chain(const double* data, size_t rows, size_t cols, size_t pad_rows, size_t out_rows,
                      const double* filter, double* block, double* medians, double* max_rel_imag);

#ifdef __cplusplus
}
#endif
#endif
