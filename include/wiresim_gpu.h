/*
 * wiresim_gpu.h — C ABI of the B200-native Wire-Cell signal-simulation hot path
 * (rasterize -> scatter-add -> FFT convolution), a drop-in for the
 * raster/scatter/convolve section of the reference `wiresim` library
 * (/root/reference/proj). Plain C types only: pointers, sizes, PODs. No
 * exceptions cross this boundary; every call returns a ws_status and leaves a
 * thread-local message readable with ws_last_error().
 *
 * Reference interfaces each entry point replaces (file:line under proj/):
 *
 *   ws_plane_create        build_response(GridSpec, ResponseParams)     include/wiresim/spectral.hpp:43
 *                          (spectral.cpp:87-139; precomputed once per plane
 *                          instead of once per run_simulation, pipeline.cpp:417)
 *                          + convolve's support check                   src/spectral.cpp:147-153
 *   ws_rasterize           rasterize_depo over all depos + scatter_add_parallel
 *                          include/wiresim/rasterize.hpp:74-76, scatter.hpp:25-26
 *                          (pipeline.cpp:374-413)
 *   ws_convolve            convolve(ChargeGrid, ResponseKernel, workers)  include/wiresim/spectral.hpp:47
 *   ws_simulate_plane      run_simulation(SimConfig, vector<Depo>) up to the
 *                          pre-noise frame                               include/wiresim/pipeline.hpp:104
 *                          (pipeline.cpp:345-419)
 *   ws_simulate_event      N independent planes (one plane per run)
 *   ws_noise_digitize_device add_noise (white) + digitize              include/wiresim/spectral.hpp:61-65
 *   ws_run_simulation      run_simulation(SimConfig, vector<Depo>) whole: raster -> scatter ->
 *                          convolve -> add_noise -> digitize, SimResult::adc
 *                          (pipeline.cpp:345-427, pipeline.hpp:94-104)
 *   ws_run_events          the same for a batch of events (pipelined host buffers)
 *
 * Data layout (identical to the reference's):
 *   ws_depo     == wiresim::Depo       (core.hpp:63-70), 48 B AoS
 *   ws_grid_spec== wiresim::GridSpec   (core.hpp:40-58)
 *   frames      row-major padded grid, row = wire, column = tick (core.hpp:17-35,
 *               94-107), padded_wires x padded_ticks; float32 on this side.
 *
 * Functions suffixed _device take device pointers and are asynchronous on the
 * context's stream; the others take host pointers and return when the result
 * is in host memory. There is no CPU fallback: without a usable sm_100 device
 * every call fails with WS_ECUDA.
 */
#ifndef WIRESIM_GPU_H
#define WIRESIM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WS_ABI_VERSION 2

typedef enum ws_status {
    WS_OK = 0,
    WS_EINVAL = 1,   /* std::invalid_argument in the reference */
    WS_ERANGE = 2,   /* std::out_of_range */
    WS_EDOMAIN = 3,  /* std::domain_error (e.g. drift_depo behind the plane) */
    WS_ERUNTIME = 4, /* std::runtime_error */
    WS_ECUDA = 5,    /* CUDA runtime / device failure (no CPU fallback) */
    WS_ENOMEM = 6
} ws_status;

typedef struct ws_grid_spec {
    uint64_t n_wires, n_ticks, pad_wires, pad_ticks;
    double pitch;    /* mm per wire */
    double tick;     /* us per tick */
    double origin_x; /* mm, low edge of wire 0 */
    double origin_t; /* us, low edge of tick 0 */
} ws_grid_spec;

typedef struct ws_depo {
    int64_t id;     /* RNG stream key */
    double t;       /* us */
    double x;       /* mm */
    int64_t q;      /* electrons */
    double sigma_t; /* us */
    double sigma_x; /* mm */
} ws_depo;

enum { WS_INDUCTION = 0, WS_COLLECTION = 1 };

typedef struct ws_response {
    int32_t plane_kind; /* WS_INDUCTION | WS_COLLECTION */
    int32_t shaper_order;
    double field_sigma_t;  /* us; 0 = single-bin delta */
    double shaper_peaking; /* us; 0 = single-sample delta */
    double gain;           /* output units per electron */
    const double* wire_weights; /* odd length, centred on lag 0 */
    uint64_t n_wire_weights;
} ws_response;

typedef struct ws_drift {
    int32_t enabled;
    int32_t reserved;
    double response_plane_x, drift_speed, diffusion_long, diffusion_tran;
} ws_drift;

enum { WS_RNG_SUBSTREAM = 0, /* reference xoshiro256** substream(seed, depo.id), rng.cpp:64-76 */
       WS_RNG_PHILOX = 1 };  /* shared Philox4x32-10 stream keyed by (seed, depo.id) */

enum { WS_CHARGE_F32 = 0, WS_CHARGE_U32 = 1, WS_CHARGE_I64 = 2 };

typedef struct ws_sim_options {
    int32_t fluctuate;   /* 0: S = q * p (fp32, fixed-point accumulated); 1: binomial fluctuation */
    int32_t approx;      /* fluctuation sampler: 0 exact binomial (fluctuate), 1 Gaussian approx (fluctuate_approx) */
    int32_t rng_mode;    /* WS_RNG_* */
    int32_t charge_type; /* charge outputs with fluctuation on: WS_CHARGE_F32 (float32), WS_CHARGE_U32
                            (exact counts; a cell past 2^32-1 is a WS_ERUNTIME) or WS_CHARGE_I64 (the
                            reference's int64 ChargeGrid, core.hpp:94-99; 8 B per cell). Fluctuation off:
                            float32 always. */
    uint64_t seed;       /* SimConfig::rng.seed */
    ws_drift drift;      /* SimConfig::drift */
} ws_sim_options;

/* NoiseModel (spectral.hpp:51-55). White: per-wire normals of sigma (output
 * units). Spectrum: per wire, IFFT of amplitude_spectrum[k] with uniform
 * random phases, Hermitian-completed (host array of padded-ticks doubles;
 * needs an even 7-smooth padded tick count). rng_mode WS_RNG_SUBSTREAM is the
 * reference's own per-wire stream substream(seed ^ salt, wire) (sequential
 * per wire), WS_RNG_PHILOX the counter-based stream keyed by (seed ^ salt,
 * wire) (parallel). */
enum { WS_NOISE_OFF = 0, WS_NOISE_WHITE = 1, WS_NOISE_SPECTRUM = 2 };
typedef struct ws_noise_model {
    int32_t mode;
    int32_t rng_mode;
    double sigma;
    uint64_t seed;
    const double* amplitude_spectrum; /* spectrum mode: host pointer, n_amplitude == padded ticks */
    uint64_t n_amplitude;
} ws_noise_model;

/* AdcConfig (pipeline.hpp:30-34): code = clamp(round(v * scale + offset), 0, 2^bits - 1) */
typedef struct ws_adc_config {
    double scale;
    double offset;
    int32_t bits; /* 1..16 */
    int32_t reserved;
} ws_adc_config;

enum { WS_FRAME_F32 = 0, WS_FRAME_F64 = 1 };
enum { WS_ADC_I32 = 0, /* SimResult::adc's Matrix<int32_t> */
       WS_ADC_U16 = 1 }; /* the same codes in 2 bytes (bits <= 16) */

/* The readout stage of run_simulation after the convolution
 * (pipeline.cpp:420-423): m = add_noise(m, noise, seed), adc = digitize(m,
 * adc). White noise from the Philox stream and digitize run fused in the
 * convolution kernels' frame stores; white noise from the reference's
 * sequential per-wire substream and spectrum noise run as a second kernel
 * over the fp32 frame. The noise seed is noise.seed (the reference passes
 * SimConfig::rng.seed). frame_type selects the element type of frame
 * outputs: WS_FRAME_F64 widens the fp32 result (MeasurementGrid is double;
 * the values carry fp32 precision). */
typedef struct ws_readout {
    ws_noise_model noise; /* mode WS_NOISE_OFF: no noise */
    ws_adc_config adc;
    int32_t frame_type;   /* WS_FRAME_F32 | WS_FRAME_F64 */
    int32_t adc_type;     /* WS_ADC_I32 | WS_ADC_U16 */
} ws_readout;

typedef struct ws_timing {
    float prepare_ms;    /* sample: footprints + erf integrals (+ drift) */
    float fluctuate_ms;  /* fluctuation walk + integer scatter (0 when off) */
    float bin_ms;        /* depo -> band / tile binning (+ the response profiles on a second stream) */
    float convolve_ms;   /* fused accumulate + FFT convolution */
    float total_ms;      /* device time of the whole call */
    int32_t direct_planes; /* planes convolved by the time-domain kernel (the rest: row FFT) */
    int64_t clipped_patches; /* TimingReport::clipped_patch_count */
    int64_t clipped_charge;  /* SimResult::clipped_charge */
} ws_timing;

typedef struct ws_plane_info {
    uint64_t padded_wires, padded_ticks;
    uint64_t fft_length;     /* real transform length along ticks (== padded_ticks when circular) */
    int32_t folded;          /* 1 if the circular wrap is folded from a longer linear transform */
    int32_t n_radix_passes;
    int64_t support_ticks, support_wires; /* ResponseKernel::support_* */
    int64_t lo_lag, n_lags;               /* combined time kernel lags [lo_lag, lo_lag + n_lags) */
    int32_t impacts_per_pitch;            /* 1 unless made by ws_plane_create_impacts */
    int32_t n_response_classes;           /* distinct per-impact responses */
} ws_plane_info;

typedef struct ws_ctx ws_ctx;
typedef struct ws_plane ws_plane;

const char* ws_last_error(void);
int ws_abi_version(void);

/* Context: one device, one stream, reusable device workspace. Not thread-safe;
 * use one context per host thread. `stream` (cudaStream_t) may be NULL to
 * create a private non-blocking stream. */
int ws_ctx_create(int device, void* stream, ws_ctx** out);
int ws_ctx_destroy(ws_ctx* ctx);
int ws_ctx_synchronize(ws_ctx* ctx);
void* ws_ctx_stream(ws_ctx* ctx);
/* Convolution path for fluctuation-off frames. AUTO routes every band of
 * wire rows to the cheaper of the two kernels from its depo load (sparse
 * bands: time-domain accumulation of per-depo response profiles; dense
 * bands: per-row FFT); FFT and DIRECT force one kernel (testing, tuning).
 * Both compute the reference's circular convolution (spectral.cpp:141-175). */
enum { WS_CONV_AUTO = 0, WS_CONV_FFT = 1, WS_CONV_DIRECT = 2 };
int ws_ctx_set_conv_path(ws_ctx* ctx, int path);
/* AUTO routing threshold: a band takes the time-domain kernel while the sum
 * of its depos' response-profile lengths is <= kappa x transform length. */
int ws_ctx_set_direct_kappa(ws_ctx* ctx, double kappa);
/* Number of CUDA kernels this context has launched so far. */
uint64_t ws_ctx_launch_count(const ws_ctx* ctx);

/* Plane: geometry + response precomputed on the device (response spectrum,
 * FFT plan, twiddles). Validation mirrors build_response and convolve. A
 * plane is used with its context only; destroying it never touches the
 * context (either may be destroyed first), but a plane whose context is gone
 * can only be destroyed. */
int ws_plane_create(ws_ctx* ctx, const ws_grid_spec* grid, const ws_response* response, double n_sigma,
                    ws_plane** out);
/* Impact positions (north star (3); WCT's per-impact field response, which
 * the reference replaces by one response per plane): each
 * wire pitch is split into impacts_per_pitch equal sub-bins, impact i of wire
 * w spanning [origin_x + (w - pad_wires + i / P) pitch, + pitch / P). Depos
 * are sampled at impact resolution (the Gaussian's integral over every
 * sub-bin, normalised over the footprint's sub-bins) and responses[i] — its
 * own time kernel K_i and wire weights ww_i — applies to the charge S_i
 * binned at impact i:  M[w] = sum_i sum_dw ww_i[dw] (K_i (*) S_i[w - dw]).
 * Impacts with identical responses form one class, whose sub-bins are summed
 * to wires before the convolution (one class, e.g. 10 identical responses,
 * telescopes to the reference's wire binning, core.cpp:25-41 with
 * spectral.cpp:124-135, and runs every path: both kernels, fluctuation).
 * Several classes run on the time-domain path: each class's per-depo
 * profiles are added into the same frame tiles (the sum over impact
 * positions fused into k_direct's accumulation); fluctuation and charge
 * outputs need a single class. impacts_per_pitch in [1, 32], at most 8
 * classes. ws_plane_create is impacts_per_pitch = 1. */
int ws_plane_create_impacts(ws_ctx* ctx, const ws_grid_spec* grid, const ws_response* responses,
                            uint32_t impacts_per_pitch, double n_sigma, ws_plane** out);
int ws_plane_destroy(ws_plane* plane);
int ws_plane_get_info(const ws_plane* plane, ws_plane_info* info);
/* Combined time-domain kernel samples (n_lags doubles, lag lo_lag first). */
int ws_plane_get_kernel(const ws_plane* plane, double* out, uint64_t cap);

/* Charge grid only (raster + scatter), device pointers. charge: padded
 * float32 frame; with fluctuation the values are exact integers. */
int ws_rasterize_device(ws_plane* plane, const ws_depo* depos, uint64_t n, const ws_sim_options* opt,
                        float* charge, ws_timing* timing);
/* Convolution of an existing charge grid (float32, padded) into a frame. */
int ws_convolve_device(ws_plane* plane, const float* charge, float* frame);

/* raster -> scatter -> convolve for one plane, device pointers, asynchronous.
 * charge (nullable) additionally receives the charge grid. timing (nullable)
 * is filled at the next ws_ctx_synchronize, which also reports errors found
 * on the device: WS_ERANGE for a workspace overflow (the workspace is then
 * sized from what the device recorded; call again), never a silently
 * truncated result. */
int ws_simulate_plane_device(ws_plane* plane, const ws_depo* depos, uint64_t n, const ws_sim_options* opt,
                             float* frame, float* charge, ws_timing* timing);

/* Host-buffer drop-in for run_simulation's hot section: depos and frame in
 * host memory (pinned recommended), synchronous. Workspace overflows are
 * re-run internally; WS_ERANGE only if they persist (never WS_OK with a
 * partial result). */
int ws_simulate_plane(ws_plane* plane, const ws_depo* depos, uint64_t n, const ws_sim_options* opt, float* frame,
                      float* charge, ws_timing* timing);

/* Several independent planes (e.g. U, V, W of one event) in one batch of
 * launches. Arrays have n_planes entries; all planes must share the context. */
int ws_simulate_event_device(ws_ctx* ctx, uint32_t n_planes, ws_plane* const* planes, const ws_depo* const* depos,
                             const uint64_t* n_depos, const ws_sim_options* opt, float* const* frames,
                             ws_timing* timing);
int ws_simulate_event(ws_ctx* ctx, uint32_t n_planes, ws_plane* const* planes, const ws_depo* const* depos,
                      const uint64_t* n_depos, const ws_sim_options* opt, float* const* frames, ws_timing* timing);

/* A batch of events through the host-buffer path, pipelined: event e is
 * simulated while the frames of event e-1 stream back to the host on a
 * second stream (PCIe D2H of the fp32 frames dominates end-to-end time).
 * depos / n_depos / frames are [n_events * n_planes], event-major. timing
 * (nullable) describes the first event. Frames should be pinned. */
int ws_simulate_events(ws_ctx* ctx, uint32_t n_events, uint32_t n_planes, ws_plane* const* planes,
                       const ws_depo* const* depos, const uint64_t* n_depos, const ws_sim_options* opt,
                       float* const* frames, ws_timing* timing);

/* run_simulation (pipeline.cpp:345-427) for one plane, host buffers,
 * synchronous: adc (padded wires x padded ticks, int32 or uint16 per
 * readout->adc_type) is SimResult::adc; frame (nullable) the noisy frame
 * before digitization (fp32 or fp64 per readout->frame_type); charge
 * (nullable) the charge grid S (float32; with fluctuation the exact counts
 * in opt->charge_type: float32, uint32 or int64).
 * Workspace overflows are re-run internally (never WS_OK with a partial
 * result). */
int ws_run_simulation(ws_plane* plane, const ws_depo* depos, uint64_t n, const ws_sim_options* opt,
                      const ws_readout* readout, void* adc, void* frame, float* charge, ws_timing* timing);
/* The same with device pointers, asynchronous: a workspace overflow is
 * reported as WS_ERANGE by the next ws_ctx_synchronize (sized for the
 * re-run; call again). */
int ws_run_simulation_device(ws_plane* plane, const ws_depo* depos, uint64_t n, const ws_sim_options* opt,
                             const ws_readout* readout, void* adc, void* frame, float* charge, ws_timing* timing);
/* Several planes of one event (device pointers, asynchronous); arrays of
 * n_planes, adcs / frames entries nullable. */
int ws_run_event_device(ws_ctx* ctx, uint32_t n_planes, ws_plane* const* planes, const ws_depo* const* depos,
                        const uint64_t* n_depos, const ws_sim_options* opt, const ws_readout* readout,
                        void* const* adcs, void* const* frames, ws_timing* timing);
/* A batch of events, host buffers, pipelined like ws_simulate_events:
 * depos / n_depos / adcs / frames are [n_events * n_planes], event-major
 * (adcs, frames and their entries nullable). With WS_ADC_U16 and no frames
 * the device-to-host traffic is 2 B per cell. */
int ws_run_events(ws_ctx* ctx, uint32_t n_events, uint32_t n_planes, ws_plane* const* planes,
                  const ws_depo* const* depos, const uint64_t* n_depos, const ws_sim_options* opt,
                  const ws_readout* readout, void* const* adcs, void* const* frames, ws_timing* timing);

/* add_noise + digitize of a plane's frame (device pointers, asynchronous):
 * the frame gets the noise in place (float32); adc (nullable) receives
 * clamp(round(v * scale + offset), 0, 2^bits - 1) of the noisy fp64 sample
 * (spectral.cpp:177-196, 228-238). noise may be NULL (digitize only). */
int ws_noise_digitize_device(ws_plane* plane, float* frame, const ws_noise_model* noise, double scale, double offset,
                             int32_t bits, int32_t* adc);

/* ---- several GPUs of one node (ws_multi.cu) -------------------------------
 * One context per entry of `devices` (a device may be listed twice: two
 * streams on it) with the same n_planes plane specs on each, and a host
 * thread per device. Work units are independent (events, or (anode-face,
 * plane) runs), so nothing is exchanged between GPUs: each thread runs its
 * shard through the pipelined host-buffer path and its device-to-host copies
 * land in the caller's disjoint output buffers (the final frame gather).
 * Sharding is longest-processing-time first by ws_multi_cost. Results are
 * bitwise independent of the placement (RNG streams keyed by seed and depo
 * id). SURVEY.md §8(e); BASELINE.json configs[3] (faces) and configs[4]. */
typedef struct ws_multi ws_multi;
int ws_multi_create(uint32_t n_devices, const int* devices, uint32_t n_planes, const ws_grid_spec* grids,
                    const ws_response* responses, double n_sigma, ws_multi** out);
int ws_multi_destroy(ws_multi* m);
uint32_t ws_multi_device_count(const ws_multi* m);
ws_ctx* ws_multi_context(ws_multi* m, uint32_t device_index);
ws_plane* ws_multi_plane(ws_multi* m, uint32_t device_index, uint32_t plane);
int ws_multi_set_conv_path(ws_multi* m, int path);
/* cost model of one plane run: cells + 900 x depos (fitted to the 1k-1M depo sweep) */
double ws_multi_cost(uint64_t cells, uint64_t n_depos);
/* Whole events over the devices: depos / n_depos / adcs / frames are
 * [n_events * n_planes] (as ws_run_events). readout NULL: fp32 frames (as
 * ws_simulate_events; adcs ignored). event_device (nullable, n_events) gets
 * each event's device index. timing (nullable): the first event of device 0. */
int ws_multi_run_events(ws_multi* m, uint32_t n_events, const ws_depo* const* depos, const uint64_t* n_depos,
                        const ws_sim_options* opt, const ws_readout* readout, void* const* adcs, void* const* frames,
                        uint32_t* event_device, ws_timing* timing);
/* Independent plane runs (e.g. 12 faces x 3 planes): unit u uses plane spec
 * plane_of[u]; arrays are [n_units]. unit_device (nullable) gets each unit's
 * device index. */
int ws_multi_run_units(ws_multi* m, uint32_t n_units, const uint32_t* plane_of, const ws_depo* const* depos,
                       const uint64_t* n_depos, const ws_sim_options* opt, const ws_readout* readout,
                       void* const* adcs, void* const* frames, uint32_t* unit_device);

/* Pinned host memory for the host-buffer entry points (cudaMallocHost). */
int ws_host_alloc(uint64_t bytes, void** out);
int ws_host_free(void* p);

/* Synthetic depos placed uniformly inside the active grid, the reference's
 * gen_depos (pipeline.cpp:264-294, DepoGenRanges defaults pipeline.hpp:83-87)
 * without the CSV round trip (its %.17g text is exact). ranges6 = {q_min,
 * q_max, sigma_t_min, sigma_t_max, sigma_x_min, sigma_x_max} or NULL. */
int ws_gen_depos_uniform(uint64_t n, uint64_t seed, const ws_grid_spec* grid, const double* ranges6, ws_depo* out);

/* ---- signal processing (sigproc.hpp, the paper's Listing 1) ------------
 * A batch of constant-length signals, one row per signal (SignalBatch,
 * sigproc.hpp:17-29): data is rows x cols complex128, interleaved (re, im),
 * row-major; pad_rows guard rows precede the out_rows of interest. */
typedef struct ws_signal_batch {
    const double* data;
    uint64_t rows, cols, pad_rows, out_rows;
} ws_signal_batch;

/* sigproc_chain (sigproc.cpp:104-118): out[r] = Re(IDFT_row(data[r] * filter))
 * for r in [pad_rows, pad_rows + out_rows) -> block (out_rows x cols, fp64),
 * and medians[r] = row_median(block[r]) (nullable). The inverse DFT is the
 * reference's (1/n scaled, fft.cpp:96-100) along each row; all rows are
 * transformed so *max_rel_imag (nullable; max |imag| / max |real| over the
 * batch, i.e. idft_rows_to_real with workers = 1) is the reference's
 * diagnostic, printed to stderr as it does when > 1e-6. filter: filter_len
 * complex128 values (== cols, else WS_EINVAL like apply_filter). Validation
 * follows SignalBatch::validate. Rows up to ws_sigproc_max_cols() samples
 * whose length factors into primes <= 13 take the mixed-radix row FFT; other
 * lengths (up to ~9.1k samples) a direct O(n^2) inverse DFT per row.
 * _device: device pointers, asynchronous unless max_rel_imag is non-null. */
int ws_sigproc_chain_device(ws_ctx* ctx, const ws_signal_batch* batch, const double* filter, uint64_t filter_len,
                            double* block, double* medians, double* max_rel_imag);
/* Host buffers (pinned recommended); filter_complex = 0 takes a real filter
 * (apply_filter's double overload, sigproc.cpp:26-30). Rows are streamed in
 * chunks so the H2D, the chain and the D2H overlap. */
int ws_sigproc_chain(ws_ctx* ctx, const ws_signal_batch* batch, const double* filter, uint64_t filter_len,
                     int filter_complex, double* block, double* medians, double* max_rel_imag);
/* row_median (sigproc.cpp:80-93) of each row of a real rows x cols matrix
 * (device pointers, asynchronous). */
int ws_row_medians_device(ws_ctx* ctx, const double* m, uint64_t rows, uint64_t cols, double* medians);
uint64_t ws_sigproc_max_cols(void);

/* Depo CSV ingestion: load_depos (pipeline.cpp:226-262), same header, row
 * format ("id,t_us,x_mm,q,sigma_t_us,sigma_x_mm", %ld,%lf,%lf,%ld,%lf,%lf) and
 * the same validation (bad header, malformed row, id != row index, negative
 * charge or width; blank lines skipped), each a WS_ERUNTIME with the
 * reference's message. *out is pinned (cudaMallocHost) when pinned != 0, so it
 * can feed ws_simulate_* directly; release it with ws_free_depos(p, pinned). */
int ws_load_depos_csv(const char* path, int pinned, ws_depo** out, uint64_t* n);
int ws_free_depos(ws_depo* p, int pinned);
/* The CSV writer of gen_depos (pipeline.cpp:270-293): %.17g fields, so a
 * save -> load round trip is exact. Ids must equal the row index. */
int ws_save_depos_csv(const char* path, const ws_depo* depos, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif /* WIRESIM_GPU_H */
