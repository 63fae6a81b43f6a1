// dpd_capi.cu -- C-ABI (include/dpd.h) and the per-context step engine.
//
// The engine owns all device memory of one (sub)domain, launches every kernel of the
// step on one CUDA stream, and reports device-side errors through a small error word that
// is read back once per synchronising call (no per-step host sync).  See DESIGN.md §5-§6.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dpd.h"
#include "dpd_force_tile.cuh"
#include "dpd_kernels.cuh"

using namespace dpd;

namespace {

enum KernelId {
    KID_PACK = 0,
    KID_BIN,
    KID_SCAN,
    KID_SCATTER,
    KID_FORCE,
    KID_GATHER,
    KID_DEBUG,
    KID_COUNT
};
const char *kKernelNames[KID_COUNT] = {"pack", "bin", "scan", "scatter", "force", "gather", "debug"};

template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t cap = 0; // elements
    cudaError_t reserve(size_t n)
    {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n, 1);
        cudaError_t e = cudaMalloc(&p, want * sizeof(T));
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct PendingTiming {
    cudaEvent_t a, b;
    int kid;
};

} // namespace

struct dpd_ctx {
    // parameters
    double box[3];
    double rc, a, gamma, kT, power, dt;
    uint64_t seed;
    double body_f = 0.0;
    int kmode = 2;
    int force_impl = 0; // 0: tiled production kernel, 1: reference thread-per-particle kernel
    Geom geom{};
    PairP pp{};
    FixP fix{};
    float origin[3] = {0, 0, 0};
    // state
    int64_t n = 0;
    int64_t step = 0;
    bool primed = false; // after set: next kick is dt/2
    bool dense_ids = false;
    int cur = 0; // which of the double buffers holds the current state
    DevBuf<float4> pos[2], vel[2], frc[2];
    DevBuf<int> rank, count, start;
    DevBuf<unsigned long long> scan_state;
    DevBuf<unsigned> scan_epoch;
    DevBuf<int> err;
    DevBuf<float> stage;
    int *h_err = nullptr; // pinned
    // execution
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool timing = false;
    std::vector<PendingTiming> pending;
    std::vector<cudaEvent_t> event_pool;
    double t_ms[KID_COUNT] = {0};
    int64_t t_launches[KID_COUNT] = {0};
    int64_t launches = 0;
    int64_t fallback[3] = {0, 0, 0}; // tiled-kernel fallbacks: staged / home / list capacity
    std::string last_error;
};

namespace {

int fail(dpd_ctx *c, int code, const char *fmt, ...)
{
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->last_error = buf;
    }
    return code;
}

#define CUDA_TRY(c, expr)                                                                            \
    do {                                                                                             \
        cudaError_t e_ = (expr);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return fail((c), DPD_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),  \
                        __FILE__, __LINE__);                                                         \
    } while (0)

cudaEvent_t get_event(dpd_ctx *c)
{
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Launch helper: optional event pair around the launch, launch counting, error check.
template <class F>
int launch(dpd_ctx *c, int kid, F &&f)
{
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->timing) {
        a = get_event(c);
        b = get_event(c);
        cudaEventRecord(a, c->stream);
    }
    f();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return fail(c, DPD_ERR_CUDA, "launch of %s failed: %s", kKernelNames[kid], cudaGetErrorString(e));
    if (c->timing) {
        cudaEventRecord(b, c->stream);
        c->pending.push_back({a, b, kid});
    }
    c->launches += 1;
    return DPD_OK;
}

#define TRY(x)                      \
    do {                            \
        int r_ = (x);               \
        if (r_ != DPD_OK) return r_; \
    } while (0)

int resolve_timing(dpd_ctx *c)
{
    for (auto &p : c->pending) {
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        c->t_ms[p.kid] += ms;
        c->t_launches[p.kid] += 1;
        c->event_pool.push_back(p.a);
        c->event_pool.push_back(p.b);
    }
    c->pending.clear();
    return DPD_OK;
}

// Synchronise and translate the device error word.
int sync_check(dpd_ctx *c)
{
    CUDA_TRY(c, cudaMemcpyAsync(c->h_err, c->err.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    resolve_timing(c);
    if (c->h_err[4] | c->h_err[5] | c->h_err[6]) {
        for (int k = 0; k < 3; ++k) c->fallback[k] += c->h_err[4 + k];
        CUDA_TRY(c, cudaMemsetAsync(c->err.p + 4, 0, 4 * sizeof(int), c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    if (c->h_err[0] != 0) {
        const int flags = c->h_err[0], id = c->h_err[1];
        cudaMemsetAsync(c->err.p, 0, 4 * sizeof(int), c->stream);
        cudaStreamSynchronize(c->stream);
        if (flags & ERR_NONFINITE)
            return fail(c, DPD_ERR_NUMERIC, "non-finite value (particle id %d) at step <= %lld", id,
                        (long long)c->step);
        if (flags & ERR_CAPACITY) return fail(c, DPD_ERR_CAPACITY, "device buffer capacity exceeded");
        if (flags & ERR_RANGE)
            return fail(c, DPD_ERR_NUMERIC, "particle id %d moved more than one box length in a step", id);
        return fail(c, DPD_ERR_NUMERIC, "device error flags 0x%x", flags);
    }
    return DPD_OK;
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)std::max<int64_t>(1, (n + b - 1) / b); }

int ensure_capacity(dpd_ctx *c, int64_t n)
{
    const size_t want = (size_t)std::max<int64_t>(n, 1);
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(c, c->pos[b].reserve(want));
        CUDA_TRY(c, c->vel[b].reserve(want));
        CUDA_TRY(c, c->frc[b].reserve(want));
    }
    CUDA_TRY(c, c->rank.reserve(want));
    return DPD_OK;
}

IntegP integ(const dpd_ctx *c, float dt_drift, float kick)
{
    IntegP ip;
    ip.dt = dt_drift;
    ip.kick = kick;
    ip.body_f = (float)c->body_f;
    ip.x_half = (float)(0.5 * c->box[0] - c->origin[0]);
    return ip;
}

// Cell-list build of the current buffers into the other buffer set (a1-a4); flips cur.
int rebuild(dpd_ctx *c, const IntegP &ip)
{
    const int n = (int)c->n;
    const int s = c->cur, d = 1 - c->cur;
    const Geom g = c->geom;
    if (n > 0) {
        TRY(launch(c, KID_BIN, [&] {
            k_bin<<<nblk(n, 256), 256, 0, c->stream>>>(c->pos[s].p, c->vel[s].p, c->frc[s].p, n, g, ip, c->count.p,
                                                      c->rank.p, c->err.p);
        }));
    }
    const int ntile = (g.ncell + kScanTile - 1) / kScanTile;
    TRY(launch(c, KID_SCAN, [&] {
        k_scan<<<ntile, kScanThreads, 0, c->stream>>>(c->count.p, c->start.p, g.ncell, c->scan_state.p,
                                                      c->scan_epoch.p);
    }));
    if (n > 0) {
        TRY(launch(c, KID_SCATTER, [&] {
            k_scatter<<<nblk(n, 256), 256, 0, c->stream>>>(c->pos[s].p, c->vel[s].p, c->frc[s].p, n, g, ip,
                                                          c->start.p, c->rank.p, c->pos[d].p, c->vel[d].p,
                                                          c->frc[d].p);
        }));
    }
    c->cur = d;
    return DPD_OK;
}

// Force pass on the current buffers at RNG step index `step` (a5).
int force_pass(dpd_ctx *c, int64_t step, float4 *frc_out, PairRec rec, bool record)
{
    const int n = (int)c->n;
    if (n == 0) return DPD_OK;
    const int b = c->cur;
    const uint32_t s_lo = (uint32_t)(uint64_t)step, s_hi = (uint32_t)((uint64_t)step >> 32);
    const Geom g = c->geom;
    const PairP pp = c->pp;
    if (c->force_impl == 0) {
        const FixP fx = c->fix;
        const int ntile = ((g.n[0] + FT_BX - 1) / FT_BX) * ((g.n[1] + FT_BY - 1) / FT_BY) *
                          ((g.n[2] + FT_BZ - 1) / FT_BZ);
        const size_t smem = sizeof(ForceTileSmem);
        return launch(c, record ? KID_DEBUG : KID_FORCE, [&] {
#define DPD_TILE(R, K)                                                                                              \
    k_force_tile<R, K><<<ntile, FT_NTHR, smem, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, c->start.p, g, pp,  \
                                                            fx, s_lo, s_hi, rec, c->err.p)
            if (record) {
                switch (c->kmode) {
                case 0: DPD_TILE(true, 0); break;
                case 1: DPD_TILE(true, 1); break;
                default: DPD_TILE(true, 2); break;
                }
            } else {
                switch (c->kmode) {
                case 0: DPD_TILE(false, 0); break;
                case 1: DPD_TILE(false, 1); break;
                default: DPD_TILE(false, 2); break;
                }
            }
#undef DPD_TILE
        });
    }
    return launch(c, record ? KID_DEBUG : KID_FORCE, [&] {
        const unsigned grid = nblk(n, 128);
        if (record) {
            switch (c->kmode) {
            case 0: k_force_ref<true, 0><<<grid, 128, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, c->start.p, n, g, pp, s_lo, s_hi, rec); break;
            case 1: k_force_ref<true, 1><<<grid, 128, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, c->start.p, n, g, pp, s_lo, s_hi, rec); break;
            default: k_force_ref<true, 2><<<grid, 128, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, c->start.p, n, g, pp, s_lo, s_hi, rec); break;
            }
        } else {
            switch (c->kmode) {
            case 0: k_force_ref<false, 0><<<grid, 128, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, c->start.p, n, g, pp, s_lo, s_hi, rec); break;
            case 1: k_force_ref<false, 1><<<grid, 128, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, c->start.p, n, g, pp, s_lo, s_hi, rec); break;
            default: k_force_ref<false, 2><<<grid, 128, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, c->start.p, n, g, pp, s_lo, s_hi, rec); break;
            }
        }
    });
}

int validate_params(dpd_ctx *c, const double box[3], double rc, double a, double gamma, double kT, double power,
                    double dt)
{
    const double vals[] = {box[0], box[1], box[2], rc, a, gamma, kT, power, dt};
    for (double v : vals)
        if (!std::isfinite(v)) return fail(c, DPD_ERR_CONFIG, "non-finite parameter");
    if (!(rc > 0)) return fail(c, DPD_ERR_CONFIG, "rc must be > 0 (got %g)", rc);
    for (int k = 0; k < 3; ++k)
        if (!(box[k] >= 3.0 * rc))
            return fail(c, DPD_ERR_CONFIG, "box[%d] = %g must be >= 3 rc = %g (S:70)", k, box[k], 3 * rc);
    if (!(a >= 0) || !(gamma >= 0) || !(kT >= 0)) return fail(c, DPD_ERR_CONFIG, "a, gamma, kT must be >= 0");
    if (!(power > 0 && power <= 1)) return fail(c, DPD_ERR_CONFIG, "power must lie in (0, 1] (got %g)", power);
    if (!(dt > 0)) return fail(c, DPD_ERR_CONFIG, "dt must be > 0 (got %g)", dt);
    return DPD_OK;
}

// Geometry of a (sub)domain of extent ext_len with the given split flags.
int setup_geometry(dpd_ctx *c, const double len[3], const int split[3])
{
    Geom g{};
    int64_t ncell = 1;
    for (int k = 0; k < 3; ++k) {
        const int nd = (int)std::floor(len[k] / c->rc);
        if (nd < 3) return fail(c, DPD_ERR_CONFIG, "subdomain needs >= 3 cells per dimension (dim %d: %d)", k, nd);
        g.n[k] = nd;
        g.split[k] = split[k];
        g.off[k] = split[k] ? 1 : 0;
        g.ext[k] = nd + 2 * g.off[k];
        g.L[k] = (float)len[k];
        volatile float nf = (float)nd, lf = (float)len[k];
        g.inv_h[k] = nf / lf;
        ncell *= g.ext[k];
    }
    if (ncell > (int64_t)1 << 30) return fail(c, DPD_ERR_CONFIG, "too many cells (%lld)", (long long)ncell);
    g.ncell = (int)ncell;
    c->geom = g;
    return DPD_OK;
}

int init_ctx(dpd_ctx *c, const double box[3], double rc, double a, double gamma, double kT, double power, double dt,
             uint64_t seed)
{
    TRY(validate_params(c, box, rc, a, gamma, kT, power, dt));
    for (int k = 0; k < 3; ++k) c->box[k] = box[k];
    c->rc = rc;
    c->a = a;
    c->gamma = gamma;
    c->kT = kT;
    c->power = power;
    c->dt = dt;
    c->seed = seed;
    c->kmode = (power == 0.5) ? 0 : (power == 1.0 ? 1 : 2);
    PairP pp;
    pp.a = (float)a;
    pp.gamma = (float)gamma;
    pp.sig_dt = (float)(std::sqrt(2.0 * gamma * kT) / std::sqrt(dt));
    pp.inv_rc = (float)(1.0 / rc);
    pp.rc2 = (float)(rc * rc);
    pp.power = (float)power;
    pp.seed_fold = (uint32_t)seed ^ (uint32_t)(seed >> 32);
    c->pp = pp;
    // Fixed-point scale of the tiled kernel: bound a single pair's force
    // magnitude by a + 6.7 sigma/sqrt(dt) (|xi| <= 6.66 with 32-bit u1) + 20 gamma
    // max(1, sqrt(kT)) (relative speed), keep |f scale| < 2^21; larger magnitudes are
    // detected on the device and reported as DPD_ERR_NUMERIC.
    {
        const double bound = a + 6.7 * (double)pp.sig_dt + 20.0 * gamma * std::max(1.0, std::sqrt(kT)) + 1e-30;
        int k = (int)std::floor(std::log2(std::ldexp(1.0, 21) / bound));
        k = std::min(20, std::max(-20, k));
        c->fix.scale = (float)std::ldexp(1.0, k);
        c->fix.inv_scale = (float)std::ldexp(1.0, -k);
        c->fix.mag_lim = (float)std::ldexp(1.0, 21 - k);
    }
    {
        // two tiles per SM need the maximum shared-memory carveout (2 x (smem + 1 KB) <= 228 KB)
        const int smem = (int)sizeof(ForceTileSmem);
        const void *fns[6] = {(const void *)k_force_tile<false, 0>, (const void *)k_force_tile<false, 1>,
                              (const void *)k_force_tile<false, 2>, (const void *)k_force_tile<true, 0>,
                              (const void *)k_force_tile<true, 1>,  (const void *)k_force_tile<true, 2>};
        for (const void *f : fns) {
            CUDA_TRY(c, cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            CUDA_TRY(c, cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             (int)cudaSharedmemCarveoutMaxShared));
        }
    }
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    CUDA_TRY(c, c->err.reserve(8));
    CUDA_TRY(c, cudaMemset(c->err.p, 0, 8 * sizeof(int)));
    CUDA_TRY(c, cudaMallocHost(&c->h_err, 8 * sizeof(int)));
    CUDA_TRY(c, c->scan_epoch.reserve(1));
    CUDA_TRY(c, cudaMemset(c->scan_epoch.p, 0, sizeof(unsigned)));
    return DPD_OK;
}

int alloc_grid(dpd_ctx *c)
{
    const int ncell = c->geom.ncell;
    CUDA_TRY(c, c->count.reserve((size_t)ncell + 16));
    CUDA_TRY(c, c->start.reserve((size_t)ncell + 16));
    const int ntile = (ncell + kScanTile - 1) / kScanTile;
    CUDA_TRY(c, c->scan_state.reserve((size_t)ntile));
    CUDA_TRY(c, cudaMemset(c->count.p, 0, sizeof(int) * c->count.cap));
    CUDA_TRY(c, cudaMemset(c->scan_state.p, 0, sizeof(unsigned long long) * c->scan_state.cap));
    return DPD_OK;
}

} // namespace

// =========================================================================================
// C-ABI
// =========================================================================================
extern "C" {

int dpd_create(const double box[3], double rc, double a, double gamma, double kT, double power, double dt,
               uint64_t seed, dpd_ctx **out)
{
    if (!out || !box) return DPD_ERR_ARG;
    *out = nullptr;
    dpd_ctx *c = new dpd_ctx();
    int r = init_ctx(c, box, rc, a, gamma, kT, power, dt, seed);
    if (r == DPD_OK) {
        const int split[3] = {0, 0, 0};
        r = setup_geometry(c, box, split);
    }
    if (r == DPD_OK) r = alloc_grid(c);
    if (r != DPD_OK) {
        // keep the message reachable: hand back the context only on success
        static thread_local std::string msg;
        msg = c->last_error;
        dpd_destroy(c);
        fprintf(stderr, "dpd_create: %s\n", msg.c_str());
        return r;
    }
    *out = c;
    return DPD_OK;
}

void dpd_destroy(dpd_ctx *c)
{
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (int b = 0; b < 2; ++b) {
        c->pos[b].release();
        c->vel[b].release();
        c->frc[b].release();
    }
    c->rank.release();
    c->count.release();
    c->start.release();
    c->scan_state.release();
    c->scan_epoch.release();
    c->err.release();
    c->stage.release();
    for (auto &p : c->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    if (c->h_err) cudaFreeHost(c->h_err);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char *dpd_last_error(const dpd_ctx *c) { return c ? c->last_error.c_str() : "null context"; }

int dpd_set_stream(dpd_ctx *c, void *stream)
{
    if (!c) return DPD_ERR_ARG;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    c->own_stream = false;
    if (stream) {
        c->stream = (cudaStream_t)stream;
    } else {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    return DPD_OK;
}

int dpd_set_option(dpd_ctx *c, const char *name, int64_t value)
{
    if (!c || !name) return DPD_ERR_ARG;
    if (strcmp(name, "force_kernel") == 0) {
        if (value < 0 || value > 1) return fail(c, DPD_ERR_ARG, "force_kernel must be 0 (tiled) or 1 (reference)");
        c->force_impl = (int)value;
        return DPD_OK;
    }
    return fail(c, DPD_ERR_ARG, "unknown option '%s'", name);
}

int dpd_get_stat(dpd_ctx *c, const char *name, int64_t *value)
{
    if (!c || !name || !value) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (strcmp(name, "fallback_tiles") == 0) {
        *value = c->fallback[0] + c->fallback[1] + c->fallback[2];
        return DPD_OK;
    }
    if (strcmp(name, "fallback_staged") == 0) { *value = c->fallback[0]; return DPD_OK; }
    if (strcmp(name, "fallback_home") == 0) { *value = c->fallback[1]; return DPD_OK; }
    if (strcmp(name, "fallback_list") == 0) { *value = c->fallback[2]; return DPD_OK; }
    return fail(c, DPD_ERR_ARG, "unknown statistic '%s'", name);
}

int dpd_set_body_force(dpd_ctx *c, double f)
{
    if (!c) return DPD_ERR_ARG;
    if (!std::isfinite(f)) return fail(c, DPD_ERR_CONFIG, "body force must be finite");
    c->body_f = f;
    return DPD_OK;
}

int dpd_set_particles_ex(dpd_ctx *c, int64_t n, const float *pos, const float *vel, const int32_t *ids, int64_t step0)
{
    if (!c) return DPD_ERR_ARG;
    if (n < 0 || n > (int64_t)INT32_MAX / 2) return fail(c, DPD_ERR_ARG, "bad particle count %lld", (long long)n);
    if (n > 0 && (!pos || !vel)) return fail(c, DPD_ERR_ARG, "null pos/vel");
    if (step0 < 0) return fail(c, DPD_ERR_ARG, "step0 must be >= 0");
    TRY(ensure_capacity(c, n));
    // dense-id check (host): ids must be a permutation of 0..n-1 for id-order getters
    bool dense = true;
    if (ids) {
        std::vector<char> seen((size_t)n, 0);
        for (int64_t i = 0; i < n; ++i) {
            const int32_t id = ids[i];
            if (id < 0) return fail(c, DPD_ERR_ARG, "negative id at %lld", (long long)i);
            if (id >= n || seen[(size_t)id]) { dense = false; continue; }
            seen[(size_t)id] = 1;
        }
    }
    c->dense_ids = dense;
    c->n = n;
    c->step = step0;
    c->cur = 0;
    // staging: pos3, vel3 (+ ids)
    const size_t words = (size_t)std::max<int64_t>(n, 1) * 7;
    CUDA_TRY(c, c->stage.reserve(words));
    float *d_pos = c->stage.p, *d_vel = c->stage.p + 3 * (size_t)n;
    int32_t *d_ids = ids ? reinterpret_cast<int32_t *>(c->stage.p + 6 * (size_t)n) : nullptr;
    if (n > 0) {
        CUDA_TRY(c, cudaMemcpyAsync(d_pos, pos, sizeof(float) * 3 * n, cudaMemcpyDefault, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(d_vel, vel, sizeof(float) * 3 * n, cudaMemcpyDefault, c->stream));
        if (ids) CUDA_TRY(c, cudaMemcpyAsync(d_ids, ids, sizeof(int32_t) * n, cudaMemcpyDefault, c->stream));
        const Geom g = c->geom;
        TRY(launch(c, KID_PACK, [&] {
            k_pack_input<<<nblk(n, 256), 256, 0, c->stream>>>(d_pos, d_vel, d_ids, n, g, c->pos[0].p, c->vel[0].p,
                                                              c->frc[0].p, c->err.p);
        }));
    }
    // sort into cells without moving (dt = 0, kick = 0), then prime F_0 at s = step0
    TRY(rebuild(c, integ(c, 0.0f, 0.0f)));
    TRY(force_pass(c, c->step, c->frc[c->cur].p, PairRec{nullptr, nullptr, 0}, false));
    c->primed = true;
    return sync_check(c);
}

int dpd_set_particles(dpd_ctx *c, int64_t n, const float *pos, const float *vel)
{
    return dpd_set_particles_ex(c, n, pos, vel, nullptr, 0);
}

int dpd_step_async(dpd_ctx *c, int64_t nsteps)
{
    if (!c) return DPD_ERR_ARG;
    if (nsteps < 0) return fail(c, DPD_ERR_ARG, "nsteps must be >= 0");
    for (int64_t it = 0; it < nsteps; ++it) {
        const float kick = c->primed ? (float)(0.5 * c->dt) : (float)c->dt;
        TRY(rebuild(c, integ(c, (float)c->dt, kick)));
        c->step += 1;
        TRY(force_pass(c, c->step, c->frc[c->cur].p, PairRec{nullptr, nullptr, 0}, false));
        c->primed = false;
    }
    return DPD_OK;
}

int dpd_step(dpd_ctx *c, int64_t nsteps)
{
    TRY(dpd_step_async(c, nsteps));
    return sync_check(c);
}

int dpd_sync(dpd_ctx *c)
{
    if (!c) return DPD_ERR_ARG;
    return sync_check(c);
}

int dpd_get_count(const dpd_ctx *c, int64_t *n)
{
    if (!c || !n) return DPD_ERR_ARG;
    *n = c->n;
    return DPD_OK;
}

int dpd_get_step(const dpd_ctx *c, int64_t *step)
{
    if (!c || !step) return DPD_ERR_ARG;
    *step = c->step;
    return DPD_OK;
}

int dpd_get_grid(const dpd_ctx *c, int32_t dims[3])
{
    if (!c || !dims) return DPD_ERR_ARG;
    for (int k = 0; k < 3; ++k) dims[k] = c->geom.n[k];
    return DPD_OK;
}

static int gather(dpd_ctx *c, int64_t n, float *pos, float *vel, float *f, int by_id)
{
    TRY(sync_check(c));
    const int64_t cnt = c->n;
    if (cnt == 0) return DPD_OK;
    const size_t words = (size_t)cnt * 9;
    CUDA_TRY(c, c->stage.reserve(words));
    float *d_pos = pos ? c->stage.p : nullptr;
    float *d_vel = vel ? c->stage.p + 3 * (size_t)cnt : nullptr;
    float *d_f = f ? c->stage.p + 6 * (size_t)cnt : nullptr;
    const float hk = c->primed ? 0.0f : (float)(0.5 * c->dt);
    const int b = c->cur;
    const float x_half = (float)(0.5 * c->box[0] - c->origin[0]);
    const float3 org = make_float3(c->origin[0], c->origin[1], c->origin[2]);
    TRY(launch(c, KID_GATHER, [&] {
        k_gather_id<<<nblk(cnt, 256), 256, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, c->frc[b].p, (int)cnt, hk,
                                                           (float)c->body_f, x_half, org, d_pos, d_vel, d_f, by_id);
    }));
    (void)n;
    if (pos) CUDA_TRY(c, cudaMemcpyAsync(pos, d_pos, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    if (vel) CUDA_TRY(c, cudaMemcpyAsync(vel, d_vel, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    if (f) CUDA_TRY(c, cudaMemcpyAsync(f, d_f, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return DPD_OK;
}

int dpd_get_particles(dpd_ctx *c, int64_t n, float *pos, float *vel)
{
    if (!c) return DPD_ERR_ARG;
    if (n != c->n) return fail(c, DPD_ERR_ARG, "n = %lld but the context holds %lld", (long long)n, (long long)c->n);
    if (!c->dense_ids) return fail(c, DPD_ERR_ARG, "ids are not dense 0..n-1; use dpd_get_particles_ex");
    return gather(c, n, pos, vel, nullptr, 1);
}

int dpd_get_forces(dpd_ctx *c, int64_t n, float *f)
{
    if (!c) return DPD_ERR_ARG;
    if (n != c->n) return fail(c, DPD_ERR_ARG, "n = %lld but the context holds %lld", (long long)n, (long long)c->n);
    if (!c->dense_ids) return fail(c, DPD_ERR_ARG, "ids are not dense 0..n-1; use dpd_get_forces_ex");
    return gather(c, n, nullptr, nullptr, f, 1);
}

int dpd_get_state(dpd_ctx *c, int64_t cap, float *pos, float *uhalf, float *f, int32_t *ids, int64_t *n)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n) *n = c->n;
    const int64_t cnt = c->n;
    if (cap < cnt) return fail(c, DPD_ERR_ARG, "cap %lld < count %lld", (long long)cap, (long long)cnt);
    if (cnt == 0) return DPD_OK;
    CUDA_TRY(c, c->stage.reserve((size_t)cnt * 10));
    float *dp = c->stage.p, *du = dp + 3 * cnt, *df = du + 3 * cnt;
    int32_t *di = reinterpret_cast<int32_t *>(df + 3 * cnt);
    const int b = c->cur;
    TRY(launch(c, KID_GATHER, [&] {
        k_state<<<nblk(cnt, 256), 256, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, c->frc[b].p, (int)cnt, dp, du, df,
                                                      di);
    }));
    if (pos) CUDA_TRY(c, cudaMemcpyAsync(pos, dp, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    if (uhalf) CUDA_TRY(c, cudaMemcpyAsync(uhalf, du, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    if (f) CUDA_TRY(c, cudaMemcpyAsync(f, df, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    if (ids) CUDA_TRY(c, cudaMemcpyAsync(ids, di, sizeof(int32_t) * cnt, cudaMemcpyDefault, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return DPD_OK;
}

int dpd_debug_cells(dpd_ctx *c, int32_t *cell_of_id, int32_t *count, int32_t *start)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    const int ncell = c->geom.ncell;
    const int64_t cnt = c->n;
    if (cell_of_id && !c->dense_ids) return fail(c, DPD_ERR_ARG, "cell_of_id needs dense ids");
    std::vector<int32_t> st((size_t)ncell + 1);
    CUDA_TRY(c, cudaMemcpy(st.data(), c->start.p, sizeof(int32_t) * (ncell + 1), cudaMemcpyDeviceToHost));
    if (start) memcpy(start, st.data(), sizeof(int32_t) * (ncell + 1));
    if (count)
        for (int i = 0; i < ncell; ++i) count[i] = st[i + 1] - st[i];
    if (cell_of_id && cnt > 0) {
        CUDA_TRY(c, c->stage.reserve((size_t)cnt));
        int32_t *d = reinterpret_cast<int32_t *>(c->stage.p);
        const int b = c->cur;
        const Geom g = c->geom;
        TRY(launch(c, KID_DEBUG, [&] {
            k_ids_cells<<<nblk(cnt, 256), 256, 0, c->stream>>>(c->pos[b].p, (int)cnt, g, nullptr, d);
        }));
        CUDA_TRY(c, cudaMemcpyAsync(cell_of_id, d, sizeof(int32_t) * cnt, cudaMemcpyDefault, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    return DPD_OK;
}

int dpd_debug_pairs(dpd_ctx *c, int64_t cap, uint32_t *quad, int64_t *npairs)
{
    if (!c || cap < 0) return DPD_ERR_ARG;
    TRY(sync_check(c));
    DevBuf<uint4> q;
    DevBuf<unsigned long long> cntb;
    DevBuf<float4> fscratch;
    CUDA_TRY(c, q.reserve((size_t)std::max<int64_t>(cap, 1)));
    CUDA_TRY(c, cntb.reserve(1));
    CUDA_TRY(c, fscratch.reserve((size_t)std::max<int64_t>(c->n, 1)));
    CUDA_TRY(c, cudaMemsetAsync(cntb.p, 0, sizeof(unsigned long long), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(fscratch.p, 0, sizeof(float4) * fscratch.cap, c->stream));
    int r = force_pass(c, c->step, fscratch.p, PairRec{q.p, cntb.p, (long long)cap}, true);
    unsigned long long total = 0;
    if (r == DPD_OK) {
        cudaMemcpyAsync(&total, cntb.p, sizeof total, cudaMemcpyDeviceToHost, c->stream);
        cudaStreamSynchronize(c->stream);
        const int64_t k = std::min<int64_t>((int64_t)total, cap);
        if (quad && k > 0) cudaMemcpy(quad, q.p, sizeof(uint4) * k, cudaMemcpyDeviceToHost);
        if (npairs) *npairs = (int64_t)total;
    }
    q.release();
    cntb.release();
    fscratch.release();
    if (r != DPD_OK) return r;
    return sync_check(c);
}

int dpd_set_timing(dpd_ctx *c, int enable)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    c->timing = enable != 0;
    for (int k = 0; k < KID_COUNT; ++k) {
        c->t_ms[k] = 0.0;
        c->t_launches[k] = 0;
    }
    return DPD_OK;
}

int dpd_get_timing(dpd_ctx *c, int kid, double *total_ms, int64_t *launches)
{
    if (!c || kid < 0 || kid >= KID_COUNT) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (total_ms) *total_ms = c->t_ms[kid];
    if (launches) *launches = c->t_launches[kid];
    return DPD_OK;
}

const char *dpd_kernel_name(int kid) { return (kid >= 0 && kid < KID_COUNT) ? kKernelNames[kid] : nullptr; }

int dpd_get_launch_count(const dpd_ctx *c, int64_t *launches)
{
    if (!c || !launches) return DPD_ERR_ARG;
    *launches = c->launches;
    return DPD_OK;
}

// ---- debug: device Philox / pair words (T0 on the GPU) ----------------------------------
int dpd_debug_philox(int64_t n, const uint32_t *ctr, const uint32_t *key, uint32_t *out)
{
    if (n <= 0) return n == 0 ? DPD_OK : DPD_ERR_ARG;
    uint2 *dc, *dout;
    uint32_t *dk;
    if (cudaMalloc(&dc, sizeof(uint2) * n) != cudaSuccess) return DPD_ERR_CUDA;
    cudaMalloc(&dk, sizeof(uint32_t) * n);
    cudaMalloc(&dout, sizeof(uint2) * n);
    cudaMemcpy(dc, ctr, sizeof(uint2) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, key, sizeof(uint32_t) * n, cudaMemcpyHostToDevice);
    k_philox2<<<nblk(n, 128), 128>>>(dc, dk, dout, (int)n);
    cudaError_t e = cudaMemcpy(out, dout, sizeof(uint2) * n, cudaMemcpyDeviceToHost);
    cudaFree(dc);
    cudaFree(dk);
    cudaFree(dout);
    return e == cudaSuccess ? DPD_OK : DPD_ERR_CUDA;
}

int dpd_debug_pair_words(int64_t n, const uint32_t *quad_in, uint64_t seed, uint32_t *words, float *xi)
{
    if (n <= 0) return n == 0 ? DPD_OK : DPD_ERR_ARG;
    uint4 *din;
    uint2 *dw;
    float *dxi;
    if (cudaMalloc(&din, sizeof(uint4) * n) != cudaSuccess) return DPD_ERR_CUDA;
    cudaMalloc(&dw, sizeof(uint2) * n);
    cudaMalloc(&dxi, sizeof(float) * n);
    cudaMemcpy(din, quad_in, sizeof(uint4) * n, cudaMemcpyHostToDevice);
    k_pair_words<<<nblk(n, 128), 128>>>(din, (uint32_t)seed ^ (uint32_t)(seed >> 32), dxi, dw, (int)n);
    cudaMemcpy(words, dw, sizeof(uint2) * n, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaMemcpy(xi, dxi, sizeof(float) * n, cudaMemcpyDeviceToHost);
    cudaFree(din);
    cudaFree(dw);
    cudaFree(dxi);
    return e == cudaSuccess ? DPD_OK : DPD_ERR_CUDA;
}

// ---- multi-GPU entry points (filled in by the decomposition layer) -----------------------
int dpd_nccl_unique_id(uint8_t id[128])
{
    (void)id;
    return DPD_ERR_CONFIG;
}

int dpd_create_dist(const double box[3], double rc, double a, double gamma, double kT, double power, double dt,
                    uint64_t seed, int rank, int world, const int32_t grid[3], const uint8_t nccl_id[128],
                    dpd_ctx **out)
{
    (void)box; (void)rc; (void)a; (void)gamma; (void)kT; (void)power; (void)dt; (void)seed;
    (void)rank; (void)world; (void)grid; (void)nccl_id;
    if (out) *out = nullptr;
    return DPD_ERR_CONFIG;
}

int dpd_create_group(const double box[3], double rc, double a, double gamma, double kT, double power, double dt,
                     uint64_t seed, const int32_t grid[3], dpd_ctx **out)
{
    (void)box; (void)rc; (void)a; (void)gamma; (void)kT; (void)power; (void)dt; (void)seed; (void)grid; (void)out;
    return DPD_ERR_CONFIG;
}

int dpd_group_step(dpd_ctx **ctxs, int nctx, int64_t nsteps)
{
    (void)ctxs; (void)nctx; (void)nsteps;
    return DPD_ERR_CONFIG;
}

int dpd_get_particles_ex(dpd_ctx *c, int64_t cap, float *pos, float *vel, int32_t *ids, int64_t *n)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n) *n = c->n;
    if (cap < c->n) return fail(c, DPD_ERR_ARG, "cap %lld < count %lld", (long long)cap, (long long)c->n);
    TRY(gather(c, c->n, pos, vel, nullptr, 0));
    if (ids && c->n > 0) {
        int32_t *d = reinterpret_cast<int32_t *>(c->stage.p);
        const int b = c->cur;
        const Geom g = c->geom;
        TRY(launch(c, KID_GATHER, [&] {
            k_ids_cells<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->pos[b].p, (int)c->n, g, d, nullptr);
        }));
        CUDA_TRY(c, cudaMemcpyAsync(ids, d, sizeof(int32_t) * c->n, cudaMemcpyDefault, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    return DPD_OK;
}

int dpd_get_forces_ex(dpd_ctx *c, int64_t cap, float *f, int32_t *ids, int64_t *n)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n) *n = c->n;
    if (cap < c->n) return fail(c, DPD_ERR_ARG, "cap %lld < count %lld", (long long)cap, (long long)c->n);
    TRY(gather(c, c->n, nullptr, nullptr, f, 0));
    if (ids && c->n > 0) {
        int32_t *d = reinterpret_cast<int32_t *>(c->stage.p);
        const int b = c->cur;
        const Geom g = c->geom;
        TRY(launch(c, KID_GATHER, [&] {
            k_ids_cells<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->pos[b].p, (int)c->n, g, d, nullptr);
        }));
        CUDA_TRY(c, cudaMemcpyAsync(ids, d, sizeof(int32_t) * c->n, cudaMemcpyDefault, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    return DPD_OK;
}

} // extern "C"
