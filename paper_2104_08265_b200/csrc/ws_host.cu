// Host-side helpers of the C ABI: pinned allocations, the synthetic depo
// generator and the depo CSV format (input synthesis and ingestion, not part of
// the timed hot path).
#include <cuda_runtime.h>

#include <cerrno>
#include <charconv>
#include <cinttypes>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

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

// ---------------------------------------------------------------------------
// Depo CSV ingestion (load_depos, pipeline.cpp:226-262) and the writer side of
// gen_depos (pipeline.cpp:270-293). The file is read in one fread and parsed in
// place with from_chars (correctly rounded, so bit-identical to the reference's
// sscanf("%lf")); the result can land directly in pinned memory for the async
// H2D of the host-buffer entry points.

namespace {

constexpr const char* kDepoHeader = "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm";

// sscanf conversions skip leading white space and accept a '+' sign.
const char* skip_ws_sign(const char* p, const char* e, bool allow_plus)
{
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\v' || *p == '\f' || *p == '\r')) ++p;
    if (allow_plus && p + 1 < e && *p == '+' && *(p + 1) != '-' && *(p + 1) != '+') ++p;
    return p;
}

bool parse_i64(const char*& p, const char* e, int64_t& v)
{
    p = skip_ws_sign(p, e, true);
    const auto r = std::from_chars(p, e, v);
    if (r.ec != std::errc()) return false;
    p = r.ptr;
    return true;
}

bool parse_f64(const char*& p, const char* e, double& v)
{
    p = skip_ws_sign(p, e, true);
    const auto r = std::from_chars(p, e, v);
    if (r.ec != std::errc() && r.ec != std::errc::result_out_of_range) return false;
    p = r.ptr;
    return true;
}

// One data row: "%ld,%lf,%lf,%ld,%lf,%lf" and nothing after it (the
// reference's trailing %c makes any extra character a malformed row).
bool parse_row(const char* p, const char* e, ws_depo& d)
{
    auto comma = [&]() {
        if (p < e && *p == ',') {
            ++p;
            return true;
        }
        return false;
    };
    return parse_i64(p, e, d.id) && comma() && parse_f64(p, e, d.t) && comma() && parse_f64(p, e, d.x) &&
           comma() && parse_i64(p, e, d.q) && comma() && parse_f64(p, e, d.sigma_t) && comma() &&
           parse_f64(p, e, d.sigma_x) && p == e;
}

int load_error(const char* path, size_t lineno, const std::string& what)
{
    std::string m = std::string("load_depos: ") + path;
    if (lineno) m += ": line " + std::to_string(lineno);
    m += ": " + what;
    return ws_set_error_message(WS_ERUNTIME, m.c_str());
}

}  // namespace

extern "C" int ws_load_depos_csv(const char* path, int pinned, ws_depo** out, uint64_t* n_out)
{
    if (!path || !out || !n_out) return ws_set_error_message(WS_EINVAL, "null argument");
    *out = nullptr;
    *n_out = 0;
    FILE* f = std::fopen(path, "rb");
    if (!f) return ws_set_error_message(WS_ERUNTIME, (std::string("load_depos: cannot open ") + path).c_str());
    std::string buf;
    char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.append(chunk, got);
    const bool read_err = std::ferror(f);
    std::fclose(f);
    if (read_err) return ws_set_error_message(WS_ERUNTIME, (std::string("load_depos: cannot read ") + path).c_str());
    if (buf.empty()) return ws_set_error_message(WS_ERUNTIME, (std::string("load_depos: ") + path + " is empty").c_str());

    const char* p = buf.data();
    const char* const end = p + buf.size();
    auto next_line = [&](const char*& b, const char*& e) {
        b = p;
        const void* nl = std::memchr(p, '\n', (size_t)(end - p));
        e = nl ? (const char*)nl : end;
        p = nl ? e + 1 : end;
    };
    const char *b, *e;
    next_line(b, e);
    if ((size_t)(e - b) != std::strlen(kDepoHeader) || std::memcmp(b, kDepoHeader, (size_t)(e - b)) != 0)
        return load_error(path, 1, "bad header \"" + std::string(b, e) + "\"");

    std::vector<ws_depo> depos;
    depos.reserve(buf.size() / 64 + 1);
    size_t lineno = 1;
    while (p < end) {
        next_line(b, e);
        ++lineno;
        if (b == e) continue;
        ws_depo d{};
        if (!parse_row(b, e, d)) return load_error(path, lineno, "malformed row \"" + std::string(b, e) + "\"");
        const int64_t row_index = (int64_t)depos.size();
        if (d.id != row_index)
            return load_error(path, lineno, "id " + std::to_string(d.id) + " must equal the row index " +
                                                std::to_string(row_index));
        if (d.q < 0) return load_error(path, lineno, "negative charge " + std::to_string(d.q));
        if (d.sigma_t < 0.0 || d.sigma_x < 0.0) return load_error(path, lineno, "negative width");
        depos.push_back(d);
    }
    const size_t bytes = depos.size() * sizeof(ws_depo);
    void* mem = nullptr;
    if (pinned) {
        const int rc = ws_host_alloc(bytes, &mem);
        if (rc != WS_OK) return rc;
    } else {
        mem = std::malloc(bytes ? bytes : 1);
        if (!mem) return ws_set_error_message(WS_ENOMEM, "load_depos: out of host memory");
    }
    if (bytes) std::memcpy(mem, depos.data(), bytes);
    *out = static_cast<ws_depo*>(mem);
    *n_out = depos.size();
    return WS_OK;
}

extern "C" int ws_free_depos(ws_depo* p, int pinned)
{
    if (!p) return WS_OK;
    if (pinned) return ws_host_free(p);
    std::free(p);
    return WS_OK;
}

extern "C" int ws_save_depos_csv(const char* path, const ws_depo* d, uint64_t n)
{
    if (!path || (!d && n)) return ws_set_error_message(WS_EINVAL, "null argument");
    for (uint64_t i = 0; i < n; ++i)
        if (d[i].id != (int64_t)i)
            return ws_set_error_message(WS_EINVAL, "save_depos: id must equal the row index (load_depos rule)");
    FILE* f = std::fopen(path, "wb");
    if (!f) return ws_set_error_message(WS_ERUNTIME, (std::string("gen_depos: cannot open ") + path).c_str());
    std::string out = std::string(kDepoHeader) + "\n";
    char line[256];
    for (uint64_t i = 0; i < n; ++i) {
        const int k = std::snprintf(line, sizeof line, "%" PRIu64 ",%.17g,%.17g,%" PRId64 ",%.17g,%.17g\n", i,
                                    d[i].t, d[i].x, d[i].q, d[i].sigma_t, d[i].sigma_x);
        out.append(line, (size_t)k);
        if (out.size() > (1u << 22) || i + 1 == n) {
            if (std::fwrite(out.data(), 1, out.size(), f) != out.size()) {
                std::fclose(f);
                return ws_set_error_message(WS_ERUNTIME, (std::string("gen_depos: short write to ") + path).c_str());
            }
            out.clear();
        }
    }
    if (n == 0 && std::fwrite(out.data(), 1, out.size(), f) != out.size()) {
        std::fclose(f);
        return ws_set_error_message(WS_ERUNTIME, (std::string("gen_depos: short write to ") + path).c_str());
    }
    if (std::fclose(f) != 0)
        return ws_set_error_message(WS_ERUNTIME, (std::string("gen_depos: short write to ") + path).c_str());
    return WS_OK;
}
