// dpd_capi.cu -- C-ABI (include/dpd.h) and the per-(sub)domain step engine.
//
// The engine owns all device memory of one (sub)domain, launches every kernel of the step
// on one CUDA stream (plus a communication stream in multi-GPU runs), and reports
// device-side errors through a small error word that is read back once per synchronising
// call (no per-step host sync).  Particle counts live on the device (the last entry of the
// cell-start array), so migration never needs a host round trip.  See DESIGN.md §5-§7.
//
// One step (GW velocity Verlet, C-6):
//   a1-a2  k_bin          kick + drift + wrap, cell histogram; leavers -> migration messages
//   a10    exchange(mig)  NCCL send/recv (or device copies inside an in-process group)
//          k_bin_recv     received migrants -> histogram
//   a3     k_scan         exclusive scan of the counts
//   a4     k_scatter (+ k_scatter_recv)  cell-sorted copy
//   a7     k_ghost_pack_cells   boundary-layer particles -> ghost messages
//   a8     exchange(ghost) on the comm stream, overlapped with
//   a5     k_force_tile   local-local half-stencil pairs
//   a9     k_ghost_bin/scan/scatter + k_force_halo_cells   one-sided local-ghost pairs
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#ifdef DPD_HAVE_NCCL
#include <nccl.h>
#endif

#include "../../include/dpd.h"
#include "dpd_dist.cuh"
#include "dpd_force_tile.cuh"
#include "dpd_kernels.cuh"
#include "dpd_sched.h"

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
    KID_MIGRATE,
    KID_GHOST_PACK,
    KID_GHOST_SORT,
    KID_HALO,
    KID_NCCL, // NCCL send/recv groups (timed, not counted as this library's launches)
    KID_COUNT
};
const char *kKernelNames[KID_COUNT] = {"pack",    "bin",        "scan",       "scatter", "force", "gather",
                                       "debug",   "migrate",    "ghost_pack", "ghost_sort", "halo", "nccl"};

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

template <class T>
struct ScopedBuf : DevBuf<T> {
    ScopedBuf() = default;
    ScopedBuf(const ScopedBuf &) = delete;
    ScopedBuf &operator=(const ScopedBuf &) = delete;
    ~ScopedBuf() { this->release(); }
};

struct PendingTiming {
    cudaEvent_t a, b;
    int kid;
};

// Message area of one kind (ghosts or migrants): 27 direction slots, see Msgs.
struct MsgArea {
    DevBuf<char> send, recv;
    Msgs ms{}, mr{}; // device views of send / recv
    size_t bytes[27] = {0};
    int maxcap = 0;
};

} // namespace

// Asynchronous snapshot dumps (NEXT-4): one device staging block, `depth + 1` pinned host
// slots and the I/O worker (IoQueue) writing <prefix>_r<rank>_s<step>.dpd files.
struct DumpSlot {
    char *host = nullptr;
    cudaEvent_t copied = nullptr;
    bool busy = false;
};

struct DumpState {
    std::string prefix;
    int depth = 4;
    int device = 0;
    int64_t every = 0;
    int64_t cap = 0;           // particles per staging block / slot
    int64_t delay_us = 0;      // simulated slow disk (tests)
    char *dev = nullptr;       // device staging block
    cudaEvent_t staged_free = nullptr; // last D2H of the staging block finished
    std::vector<DumpSlot> slots;
    std::mutex m;
    std::condition_variable cv;
    dpd::IoQueue *q = nullptr;
    int64_t submitted = 0;
    int last_slot = -1;
};

struct dpd_ctx {
    // parameters
    double box[3];   // global box
    double sub[3];   // subdomain extent
    double rc, a, gamma, kT, power, dt;
    uint64_t seed;
    double body_f = 0.0;
    int kmode = 2;
    int nspecies = 1;   // NEXT-2 species matrix size (kmode 3 when > 1)
    int body_mode = 0;  // 0: periodic Poiseuille, 1: uniform +f along z
    int frozen_mask = 0; // NEXT-3: species that never move (frozen wall layer)
    int nwall = 0;       // NEXT-3 SDF primitives (global frame)
    int wtype[DPD_MAX_WALLS] = {0};
    float wprm[DPD_MAX_WALLS][4] = {};
    float wvel[DPD_MAX_WALLS][3] = {};
    int force_impl = 0; // 0: tiled production kernel, 1: reference thread-per-particle kernel (cross-check)
    int nsm = 148;
    Geom geom{};
    PairP pp{};
    FixP fix{};
    float origin[3] = {0, 0, 0};
    // decomposition
    bool dist = false;
    int rank = 0, world = 1, grid[3] = {1, 1, 1}, coord[3] = {0, 0, 0};
    int peer_to[27], peer_from[27]; // rank at coord + D / coord - D (periodic), -1 if unused
    MsgArea mig, gh;
    double cap_factor = 1.0;
    bool msgs_ready = false;
    DevBuf<int> rank_in, gcount, gstart, grank;
    DevBuf<int> blist; // [0]: count, then the packed coordinates of the non-empty boundary cells (row a9)
    DevBuf<float4> gpos, gvel;
    DevBuf<unsigned long long> gscan_state;
    int64_t gcap = 0;
#ifdef DPD_HAVE_NCCL
    ncclComm_t nccl = nullptr;
#endif
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_ghost = nullptr;
    dpd_ctx **group = nullptr; // in-process group (device-copy transport), shared by members
    int group_n = 0;
    // state
    int64_t n = 0;     // local particle count as of the last synchronisation
    int64_t n_cap = 0; // capacity of the particle arrays
    int64_t step = 0;
    bool primed = false;     // after set: next kick is dt/2
    bool need_prime = false; // in-process group: forces not yet computed after set
    bool dense_ids = false;
    int cur = 0;  // which of the double buffers holds the current particles
    int scur = 0; // which start array describes them (start[scur][ncell] = count)
    DevBuf<float4> pos[2], vel[2], frc[2];
    DevBuf<int> rank_buf, count, start[2];
    DevBuf<unsigned long long> scan_state;
    DevBuf<unsigned> scan_epoch;
    DevBuf<int> err;
    DevBuf<float> stage;
    int *h_err = nullptr; // pinned: [0..7] error word, [8] local count
    // execution
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool timing = false;
    std::vector<PendingTiming> pending;
    std::vector<cudaEvent_t> event_pool;
    double t_ms[KID_COUNT] = {0};
    int64_t t_launches[KID_COUNT] = {0};
    int64_t launches = 0;
    int64_t fallback[3] = {0, 0, 0}; // tiled kernel: staged / home capacity tiles, full-list particles
    std::string last_error;
    // NEXT-4: the step as a task graph and asynchronous dumps
    dpd::TaskGraph *step_graph[2] = {nullptr, nullptr}; // [0] plain step, [1] step + snapshot
    dpd::TaskGraph *group_graph = nullptr;               // member 0 of an in-process group: its task-graph step
    int group_graph_mode = 0; // member 0: dpd_group_step runs the production task graph (option "group_task_graph")
    IntegP ip_step{};
    cudaStream_t copy_stream = nullptr;
    DumpState *dump = nullptr;
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

#ifdef DPD_HAVE_NCCL
#define NCCL_TRY(c, expr)                                                                            \
    do {                                                                                             \
        ncclResult_t r_ = (expr);                                                                    \
        if (r_ != ncclSuccess)                                                                       \
            return fail((c), DPD_ERR_COMM, "%s failed: %s", #expr, ncclGetErrorString(r_));          \
    } while (0)
#endif

#define TRY(x)                      \
    do {                            \
        int r_ = (x);               \
        if (r_ != DPD_OK) return r_; \
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
int launch(dpd_ctx *c, int kid, F &&f, cudaStream_t st = nullptr)
{
    if (!st) st = c->stream; // the stream f() launches on (timing events go there too)
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->timing) {
        a = get_event(c);
        b = get_event(c);
        cudaEventRecord(a, st);
    }
    f();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return fail(c, DPD_ERR_CUDA, "launch of %s failed: %s", kKernelNames[kid], cudaGetErrorString(e));
    if (c->timing) {
        cudaEventRecord(b, st);
        c->pending.push_back({a, b, kid});
    }
    c->launches += 1;
    return DPD_OK;
}

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

inline int *count_ptr(dpd_ctx *c) { return c->start[c->scur].p + c->geom.ncell; }

// Synchronise, read the local count and translate the device error word.
int sync_check(dpd_ctx *c)
{
    CUDA_TRY(c, cudaMemcpyAsync(c->h_err, c->err.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_err + 8, count_ptr(c), sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    resolve_timing(c);
    c->n = c->h_err[8];
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
        if (flags & ERR_CAPACITY)
            return fail(c, DPD_ERR_CAPACITY, "device buffer capacity exceeded (particles, ghosts or migrants)");
        if (flags & ERR_SPECIES)
            return fail(c, DPD_ERR_ARG, "species index out of range (particle id %d; %d species)", id, c->nspecies);
        if (flags & ERR_IDRANGE)
            return fail(c, DPD_ERR_ARG, "particle id %d out of range: ids must be >= 0, and < 2^30 with a species "
                        "matrix", id);
        if (flags & ERR_RANGE)
            return fail(c, DPD_ERR_NUMERIC,
                        "particle id %d moved more than one (sub)domain in a step or a pair force left the "
                        "fixed-point range", id);
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
    CUDA_TRY(c, c->rank_buf.reserve(want));
    c->n_cap = (int64_t)c->pos[0].cap;
    return DPD_OK;
}

IntegP integ(const dpd_ctx *c, float dt_drift, float kick)
{
    IntegP ip{};
    ip.dt = dt_drift;
    ip.kick = kick;
    ip.body_f = (float)c->body_f;
    ip.x_half = (float)(0.5 * c->box[0] - c->origin[0]);
    ip.body_mode = c->body_mode;
    ip.frozen_mask = c->frozen_mask;
    ip.nwall = c->nwall;
    for (int k = 0; k < DPD_MAX_WALLS; ++k) {
        ip.wtype[k] = c->wtype[k];
        for (int q = 0; q < 4; ++q) ip.wprm[k][q] = c->wprm[k][q];
        for (int q = 0; q < 3; ++q) ip.wvel[k][q] = c->wvel[k][q];
    }
    for (int k = 0; k < 3; ++k) ip.origin[k] = c->origin[k];
    return ip;
}

Msgs no_msgs()
{
    Msgs m{};
    m.base = nullptr;
    return m;
}

// ---- phases of one step -------------------------------------------------------------------

// a1-a2: kick-drift and histogram (leavers into the migration messages).  with_mig = false
// when re-binning a freshly set state (dt = 0: nobody moves, no messages).
int phase_bin(dpd_ctx *c, const IntegP &ip, bool with_mig = true)
{
    const Geom g = c->geom;
    const int s = c->cur;
    with_mig = with_mig && c->dist;
    const Msgs mig = with_mig ? c->mig.ms : no_msgs();
    if (with_mig) {
        TRY(launch(c, KID_MIGRATE, [&] { k_zero_headers<<<1, 32, 0, c->stream>>>(mig); }));
    }
    const bool lean = !c->dist && ip.nwall == 0 && ip.frozen_mask == 0;
    return launch(c, KID_BIN, [&] {
        if (lean)
            k_bin<true><<<nblk(c->n_cap, 256), 256, 0, c->stream>>>(c->pos[s].p, c->vel[s].p, c->frc[s].p, count_ptr(c),
                                                                    g, ip, c->count.p, c->rank_buf.p, mig, c->err.p);
        else
            k_bin<false><<<nblk(c->n_cap, 256), 256, 0, c->stream>>>(c->pos[s].p, c->vel[s].p, c->frc[s].p, count_ptr(c),
                                                                     g, ip, c->count.p, c->rank_buf.p, mig, c->err.p);
    });
}

// a10 (received side) + a3 + a4: histogram of the migrants, scan, scatter; flips cur/scur.
// The target force buffer frc[d] must be zero: inside a step the previous force pass zeroed
// it (k_force_tile's fzero); a re-sort outside a step (set, carve) passes zero_target.
int phase_sort(dpd_ctx *c, const IntegP &ip, bool with_mig = true, bool zero_target = false)
{
    const Geom g = c->geom;
    const int s = c->cur, d = 1 - c->cur;
    const int ss = c->scur, sd = 1 - c->scur;
    if (zero_target && c->n_cap > 0)
        CUDA_TRY(c, cudaMemsetAsync(c->frc[d].p, 0, sizeof(float4) * (size_t)c->n_cap, c->stream));
    with_mig = with_mig && c->dist;
    if (with_mig) {
        const dim3 grid(nblk(c->mig.maxcap, 256), 27);
        const Msgs mr = c->mig.mr;
        TRY(launch(c, KID_MIGRATE, [&] {
            k_bin_recv<<<grid, 256, 0, c->stream>>>(mr, g, c->mig.maxcap, c->count.p, c->rank_in.p, c->err.p);
        }));
    }
    const int ntile = (g.ncell + kScanTile - 1) / kScanTile;
    TRY(launch(c, KID_SCAN, [&] {
        k_scan<<<ntile, kScanThreads, 0, c->stream>>>(c->count.p, c->start[sd].p, g.ncell, c->scan_state.p,
                                                      c->scan_epoch.p);
    }));
    const bool lean = !c->dist && ip.nwall == 0 && ip.frozen_mask == 0; // as phase_bin: identical advance
    TRY(launch(c, KID_SCATTER, [&] {
        if (lean)
            k_scatter<true><<<nblk(c->n_cap, 256), 256, 0, c->stream>>>(
                c->pos[s].p, c->vel[s].p, c->frc[s].p, c->start[ss].p + g.ncell, g, ip, c->start[sd].p, c->rank_buf.p,
                c->pos[d].p, c->vel[d].p, (int)c->n_cap, c->err.p);
        else
            k_scatter<false><<<nblk(c->n_cap, 256), 256, 0, c->stream>>>(
                c->pos[s].p, c->vel[s].p, c->frc[s].p, c->start[ss].p + g.ncell, g, ip, c->start[sd].p, c->rank_buf.p,
                c->pos[d].p, c->vel[d].p, (int)c->n_cap, c->err.p);
    }));
    if (with_mig) {
        const dim3 grid(nblk(c->mig.maxcap, 256), 27);
        const Msgs mr = c->mig.mr;
        TRY(launch(c, KID_MIGRATE, [&] {
            k_scatter_recv<<<grid, 256, 0, c->stream>>>(mr, g, c->mig.maxcap, c->start[sd].p, c->rank_in.p,
                                                        c->pos[d].p, c->vel[d].p, (int)c->n_cap, c->err.p);
        }));
    }
    c->cur = d;
    c->scur = sd;
    return DPD_OK;
}

// a7: boundary layers -> ghost messages.
int phase_ghost_pack(dpd_ctx *c, cudaStream_t st = nullptr)
{
    // reads only the sorted arrays and the cell starts, writes only the ghost messages and the
    // boundary-cell list: in the step graph it runs on the communication stream, concurrently
    // with the local forces
    if (!st) st = c->stream;
    const Geom g = c->geom;
    const Msgs gs = c->gh.ms;
    CUDA_TRY(c, c->blist.reserve((size_t)g.ncell + 1));
    CUDA_TRY(c, cudaMemsetAsync(c->blist.p, 0, sizeof(int), st));
    TRY(launch(c, KID_GHOST_PACK, [&] { k_zero_headers<<<1, 32, 0, st>>>(gs); }, st));
    // the boundary cells as disjoint boxes, one per split dimension (GpPlan in dpd_dist.cuh)
    GpPlan pl{};
    int total = 0;
    for (int k = 0; k < 3; ++k) {
        if (!g.split[k]) continue;
        const int x = pl.nbox++;
        pl.dimk[x] = k;
        int cells = 1;
        for (int d = 0; d < 3; ++d) {
            if (d == k) {
                pl.lo[x][d] = 0;
                pl.ext[x][d] = 2; // {0, n - 1}
            } else if (g.split[d] && d < k) {
                pl.lo[x][d] = 1;
                pl.ext[x][d] = g.n[d] - 2; // inner range: its faces belong to box d
            } else {
                pl.lo[x][d] = 0;
                pl.ext[x][d] = g.n[d];
            }
            cells *= pl.ext[x][d];
        }
        total += cells;
        pl.end[x] = total;
    }
    if (pl.nbox == 0 || total == 0) return DPD_OK;
    const unsigned grid = (unsigned)(((int64_t)total * kGpSub + kGpThreads - 1) / kGpThreads);
    return launch(
        c, KID_GHOST_PACK,
        [&] {
            k_ghost_pack_cells<<<grid, kGpThreads, 0, st>>>(c->pos[c->cur].p, c->vel[c->cur].p, c->start[c->scur].p, g,
                                                            gs, c->blist.p, c->err.p, pl);
        },
        st);
}

// a5: local-local pairs at RNG step index `step`.
// Per-step key on the host (C-7): k_s = fmix32(s_lo ^ seed_lo ^ fmix32(s_hi)) ^ seed_hi; the
// tiled kernel receives the ten round keys k_s + r W as a parameter (dpd_device.cuh RoundKeys).
RoundKeys host_round_keys(uint32_t s_lo, uint32_t s_hi, const PairP &pp)
{
    const uint32_t ks = step_key(s_lo, s_hi, pp.seed_lo, pp.seed_hi);
    RoundKeys K;
    for (int r = 0; r < 10; ++r) K.k[r] = ks + (uint32_t)r * kPhilox2W;
    return K;
}

PairP scaled_pair(PairP pp, float scale)
{
    pp.a *= scale;
    pp.gamma *= scale;
    pp.sig_dt *= scale;
    for (int t = 0; t < DPD_MAX_SPECIES * DPD_MAX_SPECIES; ++t) {
        pp.sa[t] *= scale;
        pp.sg[t] *= scale;
        pp.ss[t] *= scale;
    }
    return pp;
}

int force_pass(dpd_ctx *c, int64_t step, float4 *frc_out, PairRec rec, bool record)
{
    const int b = c->cur;
    const uint32_t s_lo = (uint32_t)(uint64_t)step, s_hi = (uint32_t)((uint64_t)step >> 32);
    const Geom g = c->geom;
    const PairP pp = c->pp;
    // the step's force pass also zeroes the other force buffer (the next sort's target)
    float4 *fzero = (frc_out == c->frc[b].p) ? c->frc[1 - b].p : nullptr;
    const int nzero = fzero ? (int)c->n_cap : 0;
    if (c->force_impl == 0 || c->dist) {
        const FixP fx = c->fix;
        // the tiled kernel works in fixed-point units: a, gamma, sigma/sqrt(dt) pre-multiplied
        // by the power-of-two scale (exact), so one FFMA per component quantises
        const PairP pp = scaled_pair(c->pp, fx.scale);
        const RoundKeys rk = host_round_keys(s_lo, s_hi, c->pp);
        const dim3 tgrid((g.n[0] + FT_BX - 1) / FT_BX, (g.n[1] + FT_BY - 1) / FT_BY, (g.n[2] + FT_BZ - 1) / FT_BZ);
        const size_t smem = sizeof(ForceTileSmem);
        const int *st = c->start[c->scur].p;
        return launch(c, record ? KID_DEBUG : KID_FORCE, [&] {
#define DPD_TILE(R, K)                                                                                              \
    k_force_tile<R, K><<<tgrid, FT_NTHR, smem, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, st, g, pp, fx, rk, rec, \
                                                            c->err.p, fzero, nzero)
            if (record) {
                switch (c->kmode) {
                case 0: DPD_TILE(true, 0); break;
                case 1: DPD_TILE(true, 1); break;
                case 2: DPD_TILE(true, 2); break;
                default: DPD_TILE(true, 3); break;
                }
            } else {
                switch (c->kmode) {
                case 0: DPD_TILE(false, 0); break;
                case 1: DPD_TILE(false, 1); break;
                case 2: DPD_TILE(false, 2); break;
                default: DPD_TILE(false, 3); break;
                }
            }
#undef DPD_TILE
        });
    }
    if (fzero && nzero > 0) CUDA_TRY(c, cudaMemsetAsync(fzero, 0, sizeof(float4) * (size_t)nzero, c->stream));
    const int n = (int)c->n;
    if (n == 0) return DPD_OK;
    const int *st = c->start[c->scur].p;
    return launch(c, record ? KID_DEBUG : KID_FORCE, [&] {
        const unsigned grid = nblk(n, 128);
#define DPD_REF(R, K)                                                                                               \
    k_force_ref<R, K><<<grid, 128, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, frc_out, st, n, g, pp, s_lo, s_hi, rec)
        if (record) {
            switch (c->kmode) {
            case 0: DPD_REF(true, 0); break;
            case 1: DPD_REF(true, 1); break;
            case 2: DPD_REF(true, 2); break;
            default: DPD_REF(true, 3); break;
            }
        } else {
            switch (c->kmode) {
            case 0: DPD_REF(false, 0); break;
            case 1: DPD_REF(false, 1); break;
            case 2: DPD_REF(false, 2); break;
            default: DPD_REF(false, 3); break;
            }
        }
#undef DPD_REF
    });
}

// a9 (first half): received ghosts -> halo cells (bin, scan, scatter) on stream st.  Touches
// only ghost buffers, so in the step graph it runs on the communication stream right after
// the exchange, concurrently with the local forces.
int phase_ghost_sort(dpd_ctx *c, cudaStream_t st)
{
    const Geom g = c->geom;
    const Msgs gr = c->gh.mr;
    const dim3 grid(nblk(c->gh.maxcap, 256), 27);
    TRY(launch(
        c, KID_GHOST_SORT,
        [&] { k_ghost_bin<<<grid, 256, 0, st>>>(gr, g, c->gh.maxcap, c->gcount.p, c->grank.p, c->err.p); }, st));
    const int ntile = (g.ncell + kScanTile - 1) / kScanTile;
    TRY(launch(
        c, KID_GHOST_SORT,
        [&] {
            k_scan<<<ntile, kScanThreads, 0, st>>>(c->gcount.p, c->gstart.p, g.ncell, c->gscan_state.p,
                                                   c->scan_epoch.p + 1);
        },
        st));
    return launch(
        c, KID_GHOST_SORT,
        [&] {
            k_ghost_scatter<<<grid, 256, 0, st>>>(gr, g, c->gh.maxcap, c->gstart.p, c->grank.p, c->gpos.p, c->gvel.p);
        },
        st);
}

// a9 (second half): one-sided local-ghost forces (after the local forces, same stream).
int phase_halo_force(dpd_ctx *c, int64_t step, cudaStream_t st = nullptr)
{
    if (!st) st = c->stream;
    const Geom g = c->geom;
    const uint32_t s_lo = (uint32_t)(uint64_t)step, s_hi = (uint32_t)((uint64_t)step >> 32);
    const PairP pp = c->pp;
    const int b = c->cur;
    return launch(c, KID_HALO, [&] {
        // grid-stride over the boundary list (its length lives on the device)
        const unsigned nbh = (unsigned)c->nsm * 16; // grid-stride over the boundary cells (count on device)
#define DPD_HALO(K)                                                                                                 \
    k_force_halo_cells<K><<<nbh, 32 * kHcWarps, 0, st>>>(c->pos[b].p, c->vel[b].p, c->frc[b].p, c->blist.p,  \
                                                                c->start[c->scur].p, c->gpos.p, c->gvel.p,          \
                                                                c->gstart.p, g, pp, c->fix.scale, c->fix.inv_scale, \
                                                                c->fix.mag_lim, s_lo, s_hi, c->err.p)
        switch (c->kmode) {
        case 0: DPD_HALO(0); break;
        case 1: DPD_HALO(1); break;
        case 2: DPD_HALO(2); break;
        default: DPD_HALO(3); break;
        }
#undef DPD_HALO
    }, st);
}

// a9 on the context's stream (prime, in-process group).
int phase_halo(dpd_ctx *c, int64_t step)
{
    TRY(phase_ghost_sort(c, c->stream));
    return phase_halo_force(c, step);
}

// ---- transports ---------------------------------------------------------------------------
// Message of direction d travels from rank r to peer_to[d] and lands in that rank's receive
// slot d.  Both ends post their sends / receives in increasing d, so NCCL matches them in
// order even when several directions connect the same pair of ranks (2 ranks along a
// dimension); the in-process group copies send slot d of every member to recv slot d of
// peer_to[d].

int exchange_nccl(dpd_ctx *c, MsgArea &m, cudaStream_t st)
{
#ifdef DPD_HAVE_NCCL
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (c->timing) {
        ea = get_event(c);
        eb = get_event(c);
        cudaEventRecord(ea, st);
    }
    NCCL_TRY(c, ncclGroupStart());
    for (int d = 0; d < 27; ++d) {
        if (m.bytes[d] == 0) continue;
        NCCL_TRY(c, ncclSend(m.send.p + m.ms.off[d], m.bytes[d], ncclChar, c->peer_to[d], c->nccl, st));
        NCCL_TRY(c, ncclRecv(m.recv.p + m.mr.off[d], m.bytes[d], ncclChar, c->peer_from[d], c->nccl, st));
    }
    NCCL_TRY(c, ncclGroupEnd());
    if (c->timing) {
        cudaEventRecord(eb, st);
        c->pending.push_back({ea, eb, KID_NCCL});
    }
    return DPD_OK;
#else
    (void)m;
    (void)st;
    return fail(c, DPD_ERR_COMM, "libdpd was built without NCCL");
#endif
}

// st: the stream of the copy (default: the group's shared compute stream); padded: copy the
// capacity-padded slots, the volume the NCCL transport sends (the group's task-graph step).
int exchange_group(dpd_ctx **g, int n, bool ghosts, cudaStream_t st = nullptr, bool padded = false)
{
    // one k_group_copy launch per kCopyJobs messages
    CopyJobs jobs;
    int nj = 0;
    if (!st) st = g[0]->stream;
    auto flush = [&]() -> int {
        if (nj == 0) return DPD_OK;
        dpd_ctx *c = g[0];
        TRY(launch(c, ghosts ? KID_GHOST_PACK : KID_MIGRATE,
                   [&] { k_group_copy<<<dim3(padded ? 64 : 16, nj), 256, 0, st>>>(jobs); }, st));
        nj = 0;
        return DPD_OK;
    };
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        MsgArea &m = ghosts ? c->gh : c->mig;
        for (int d = 0; d < 27; ++d) {
            if (m.bytes[d] == 0) continue;
            dpd_ctx *p = g[c->peer_to[d]];
            MsgArea &pm = ghosts ? p->gh : p->mig;
            if (pm.mr.cap[d] != m.ms.cap[d]) return fail(c, DPD_ERR_CONFIG, "group message capacities differ");
            jobs.j[nj].src = reinterpret_cast<const int4 *>(m.send.p + m.ms.off[d]);
            jobs.j[nj].dst = reinterpret_cast<int4 *>(pm.recv.p + pm.mr.off[d]);
            jobs.j[nj].cap = m.ms.cap[d];
            jobs.j[nj].full = padded ? 1 : 0;
            if (++nj == kCopyJobs) TRY(flush());
        }
    }
    return flush();
}

// ---- message buffers ------------------------------------------------------------------------
// Capacities from the global number density rho: a ghost message holds the particles of a
// one-cell layer of its face / edge / corner, a migration message the leavers of one step
// (|u| dt << h).  1.25 x mean + 8 sqrt(mean) + 64 keeps overflow > 8 sigma away.
int setup_messages(dpd_ctx *c, double rho)
{
    const Geom &g = c->geom;
    const double h[3] = {c->sub[0] / g.n[0], c->sub[1] / g.n[1], c->sub[2] / g.n[2]};
    const double vmax = 4.0 * std::sqrt(std::max(c->kT, 1e-6)) + 1.0; // per-component speed bound
    size_t goff = 0, moff = 0;
    int gmax = 0, mmax = 0;
    for (int d = 0; d < 27; ++d) {
        const int D[3] = {d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1};
        bool used = d != 13;
        double vol_g = 1.0, vol_m = 1.0;
        for (int k = 0; k < 3; ++k) {
            if (D[k] != 0 && !g.split[k]) used = false;
            vol_g *= D[k] ? h[k] : c->sub[k];
            vol_m *= D[k] ? std::min(h[k], vmax * c->dt) : c->sub[k];
        }
        int capg = 0, capm = 0;
        if (used) {
            const double mg = rho * vol_g * c->cap_factor, mm = rho * vol_m * c->cap_factor;
            capg = (int)std::ceil(1.25 * mg + 8.0 * std::sqrt(mg) + 64.0);
            capm = (int)std::ceil(1.25 * mm + 8.0 * std::sqrt(mm) + 64.0);
        }
        c->gh.ms.cap[d] = c->gh.mr.cap[d] = capg;
        c->mig.ms.cap[d] = c->mig.mr.cap[d] = capm;
        c->gh.ms.off[d] = c->gh.mr.off[d] = (int)goff;
        c->mig.ms.off[d] = c->mig.mr.off[d] = (int)moff;
        c->gh.bytes[d] = capg ? 16 + 32 * (size_t)capg : 0;
        c->mig.bytes[d] = capm ? 16 + 32 * (size_t)capm : 0;
        goff += c->gh.bytes[d];
        moff += c->mig.bytes[d];
        gmax = std::max(gmax, capg);
        mmax = std::max(mmax, capm);
    }
    if (goff > ((size_t)1 << 31) || moff > ((size_t)1 << 31))
        return fail(c, DPD_ERR_CONFIG, "message buffers too large");
    c->gh.maxcap = gmax;
    c->mig.maxcap = mmax;
    CUDA_TRY(c, c->gh.send.reserve(goff + 16));
    CUDA_TRY(c, c->gh.recv.reserve(goff + 16));
    CUDA_TRY(c, c->mig.send.reserve(moff + 16));
    CUDA_TRY(c, c->mig.recv.reserve(moff + 16));
    CUDA_TRY(c, cudaMemset(c->gh.send.p, 0, goff + 16));
    CUDA_TRY(c, cudaMemset(c->gh.recv.p, 0, goff + 16));
    CUDA_TRY(c, cudaMemset(c->mig.send.p, 0, moff + 16));
    CUDA_TRY(c, cudaMemset(c->mig.recv.p, 0, moff + 16));
    c->gh.ms.base = c->gh.send.p;
    c->gh.mr.base = c->gh.recv.p;
    c->mig.ms.base = c->mig.send.p;
    c->mig.mr.base = c->mig.recv.p;
    CUDA_TRY(c, c->rank_in.reserve((size_t)27 * std::max(mmax, 1)));
    CUDA_TRY(c, c->grank.reserve((size_t)27 * std::max(gmax, 1)));
    int64_t gtot = 0;
    for (int d = 0; d < 27; ++d) gtot += c->gh.ms.cap[d];
    c->gcap = gtot;
    if (gtot >= ((int64_t)1 << 22))
        return fail(c, DPD_ERR_CAPACITY, "ghost capacity %lld exceeds the halo kernel's 2^22 ghost index range",
                    (long long)gtot);
    CUDA_TRY(c, c->gpos.reserve((size_t)std::max<int64_t>(gtot, 1)));
    CUDA_TRY(c, c->gvel.reserve((size_t)std::max<int64_t>(gtot, 1)));
    c->msgs_ready = true;
    return DPD_OK;
}

// ---- asynchronous snapshot (NEXT-4) ------------------------------------------------------
size_t dump_bytes(int64_t cap) { return 16 + (size_t)cap * 28; }

// Snapshot of the current state into the device staging block (on the compute stream, after
// the previous copy-out of that block).
int dump_snapshot(dpd_ctx *c, cudaStream_t st)
{
    DumpState *d = c->dump;
    if (c->n_cap > d->cap) {
        // a larger state: wait for the writer to finish with every slot, then re-allocate
        {
            std::unique_lock<std::mutex> lk(d->m);
            d->cv.wait(lk, [d] {
                for (auto &sl : d->slots)
                    if (sl.busy) return false;
                return true;
            });
        }
        CUDA_TRY(c, cudaStreamSynchronize(c->copy_stream));
        if (d->dev) cudaFree(d->dev);
        d->dev = nullptr;
        for (auto &sl : d->slots) {
            if (sl.host) cudaFreeHost(sl.host);
            sl.host = nullptr;
        }
        d->cap = c->n_cap;
        CUDA_TRY(c, cudaMalloc(&d->dev, dump_bytes(d->cap)));
        for (auto &sl : d->slots) CUDA_TRY(c, cudaMallocHost(&sl.host, dump_bytes(d->cap)));
    }
    CUDA_TRY(c, cudaStreamWaitEvent(st, d->staged_free, 0));
    const int b = c->cur;
    const float hk = c->primed ? 0.0f : (float)(0.5 * c->dt);
    const IntegP ip = integ(c, 0.0f, 0.0f);
    const float3 org = make_float3(c->origin[0], c->origin[1], c->origin[2]);
    const int64_t cap = d->cap;
    long long *hdr = reinterpret_cast<long long *>(d->dev);
    float *p3 = reinterpret_cast<float *>(d->dev + 16);
    float *v3 = p3 + 3 * cap;
    int32_t *ids = reinterpret_cast<int32_t *>(v3 + 3 * cap);
    const int nb = (int)std::min<int64_t>(nblk(std::max<int64_t>(cap, 1), 256), 148 * 8);
    return launch(c, KID_GATHER, [&] {
        k_snapshot<<<nb, 256, 0, st>>>(c->pos[b].p, c->vel[b].p, c->frc[b].p, count_ptr(c), (int)cap, hk, ip, org, hdr,
                                       p3, v3, ids);
    });
}

// Copy-out of the staging block into a free pinned slot (copy stream) and hand-off to the
// I/O worker, which waits for the copy and writes the file.  Blocks only when every slot is
// still owned by the writer (backpressure, nothing dropped).
int dump_copyout(dpd_ctx *c, cudaStream_t st)
{
    DumpState *d = c->dump;
    int k = -1;
    {
        std::unique_lock<std::mutex> lk(d->m);
        d->cv.wait(lk, [d, &k] {
            for (int i = 0; i < (int)d->slots.size(); ++i) {
                const int j = (d->last_slot + 1 + i) % (int)d->slots.size();
                if (!d->slots[j].busy) {
                    k = j;
                    return true;
                }
            }
            return false;
        });
        d->slots[k].busy = true;
        d->last_slot = k;
    }
    DumpSlot &sl = d->slots[k];
    CUDA_TRY(c, cudaMemcpyAsync(sl.host, d->dev, dump_bytes(d->cap), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaEventRecord(sl.copied, st));
    CUDA_TRY(c, cudaEventRecord(d->staged_free, st));
    char path[4096];
    snprintf(path, sizeof path, "%s_r%d_s%010lld.dpd", d->prefix.c_str(), c->rank, (long long)c->step);
    const std::string fpath = path;
    const int64_t step = c->step, cap = d->cap;
    const int rank = c->rank;
    double box[3], org[3];
    for (int q = 0; q < 3; ++q) {
        box[q] = c->box[q];
        org[q] = c->origin[q];
    }
    auto job = [d, k, fpath, step, cap, rank, box, org](std::string &err) -> int {
        DumpSlot &s2 = d->slots[k];
        int rc = 0;
        cudaSetDevice(d->device);
        if (cudaEventSynchronize(s2.copied) != cudaSuccess) {
            err = "snapshot copy failed";
            rc = -1;
        }
        if (rc == 0 && d->delay_us > 0) std::this_thread::sleep_for(std::chrono::microseconds(d->delay_us));
        if (rc == 0) {
            const long long n = *reinterpret_cast<const long long *>(s2.host);
            FILE *f = fopen(fpath.c_str(), "wb");
            if (!f) {
                err = "cannot open " + fpath;
                rc = -1;
            } else {
                // header: magic, n, step, rank, box[3], origin of the subdomain[3]
                const char magic[8] = {'D', 'P', 'D', 'S', 'N', 'A', 'P', '1'};
                const int64_t hdr[3] = {(int64_t)n, step, (int64_t)rank};
                const char *p3 = s2.host + 16;
                const char *v3 = p3 + 12 * cap;
                const char *id = v3 + 12 * cap;
                bool ok = fwrite(magic, 1, 8, f) == 8 && fwrite(hdr, 8, 3, f) == 3 && fwrite(box, 8, 3, f) == 3 &&
                          fwrite(org, 8, 3, f) == 3;
                ok = ok && fwrite(p3, 12, (size_t)n, f) == (size_t)n && fwrite(v3, 12, (size_t)n, f) == (size_t)n &&
                     fwrite(id, 4, (size_t)n, f) == (size_t)n;
                ok = (fclose(f) == 0) && ok;
                if (!ok) {
                    err = "short write to " + fpath;
                    rc = -1;
                }
            }
        }
        {
            std::lock_guard<std::mutex> lk(d->m);
            s2.busy = false;
        }
        d->cv.notify_all();
        return rc;
    };
    std::string err;
    if (d->q->submit(job, err) != 0) return fail(c, DPD_ERR_IO, "dump: %s", err.c_str());
    ++d->submitted;
    return DPD_OK;
}

// ---- one step of one context as a task graph (NCCL or single) ----------------------------
// Tasks (stream slot): kick_drift_bin (0) -> [migrate_exchange (0)] -> scan_scatter (0) ->
// [ghost_pack -> ghost_exchange -> ghost_sort -> halo_force (all 1, comm stream)] ; force_local
// (0) -> [join (0), after force_local and halo_force] -> [snapshot (0) -> snapshot_d2h (2, copy
// stream)].  Kahn's order
// issues ghost_exchange before force_local, so the exchange overlaps the interior forces
// (P:244-247); cross-stream edges become CUDA events.
dpd::TaskGraph *build_step_graph(dpd_ctx *c, bool with_dump)
{
    auto *g = new dpd::TaskGraph();
    const int t_bin = g->add("kick_drift_bin", 0, [c](cudaStream_t) {
        const float kick = c->primed ? (float)(0.5 * c->dt) : (float)c->dt;
        c->ip_step = integ(c, (float)c->dt, kick);
        return phase_bin(c, c->ip_step);
    });
    int last = t_bin;
    if (c->dist) {
        const int t = g->add("migrate_exchange", 0, [c](cudaStream_t s) { return exchange_nccl(c, c->mig, s); });
        g->edge(last, t);
        last = t;
    }
    const int t_sort = g->add("scan_scatter", 0, [c](cudaStream_t) -> int {
        TRY(phase_sort(c, c->ip_step));
        c->step += 1;
        return DPD_OK;
    });
    g->edge(last, t_sort);
    int t_gx = -1;
    if (c->dist) {
        const int t_gp = g->add("ghost_pack", 1, [c](cudaStream_t s) { return phase_ghost_pack(c, s); });
        g->edge(t_sort, t_gp);
        t_gx = g->add("ghost_exchange", 1, [c](cudaStream_t s) { return exchange_nccl(c, c->gh, s); });
        g->edge(t_gp, t_gx);
        const int t_gs = g->add("ghost_sort", 1, [c](cudaStream_t s) { return phase_ghost_sort(c, s); });
        g->edge(t_gx, t_gs);
        t_gx = t_gs; // the halo forces wait for the sorted ghosts
    }
    const int t_force = g->add("force_local", 0, [c](cudaStream_t) {
        return force_pass(c, c->step, c->frc[c->cur].p, PairRec{nullptr, nullptr, 0}, false);
    });
    g->edge(t_sort, t_force);
    last = t_force;
    if (c->dist) {
        // the halo forces run on the communication stream right after the ghost sort,
        // concurrent with the interior force pass: both add into the step's force array with
        // vector reductions; the step ends when both are done (join on the compute stream)
        const int t_h = g->add("halo_force", 1, [c](cudaStream_t s) { return phase_halo_force(c, c->step, s); });
        g->edge(t_gx, t_h);
        const int t_j = g->add("join", 0, nullptr);
        g->edge(t_force, t_j);
        g->edge(t_h, t_j);
        last = t_j;
    }
    if (with_dump) {
        const int t_s = g->add("snapshot", 0, [c](cudaStream_t s) { return dump_snapshot(c, s); });
        g->edge(last, t_s);
        const int t_c = g->add("snapshot_d2h", 2, [c](cudaStream_t s) { return dump_copyout(c, s); });
        g->edge(t_s, t_c);
    }
    if (g->build() != 0) {
        delete g;
        return nullptr;
    }
    return g;
}

int run_graph(dpd_ctx *c, dpd::TaskGraph *g)
{
    const cudaStream_t streams[3] = {c->stream, c->comm_stream ? c->comm_stream : c->stream,
                                     c->copy_stream ? c->copy_stream : c->stream};
    const int rc = g->run(streams);
    if (rc == -1) return fail(c, DPD_ERR_CONFIG, "step task graph has a cycle");
    if (rc == -2) return fail(c, DPD_ERR_CUDA, "task graph: %s", cudaGetErrorString(cudaGetLastError()));
    return rc;
}

int step_one(dpd_ctx *c, bool with_dump = false)
{
    const int k = with_dump ? 1 : 0;
    if (!c->step_graph[k]) {
        c->step_graph[k] = build_step_graph(c, with_dump);
        if (!c->step_graph[k]) return fail(c, DPD_ERR_CONFIG, "step task graph has a cycle");
    }
    TRY(run_graph(c, c->step_graph[k]));
    c->primed = false;
    return DPD_OK;
}

// Forces of the freshly set state at s = step (prime, C-2 item 2), NCCL or single.
int prime_one(dpd_ctx *c)
{
    if (c->dist) {
        TRY(phase_ghost_pack(c));
        TRY(exchange_nccl(c, c->gh, c->stream));
    }
    TRY(force_pass(c, c->step, c->frc[c->cur].p, PairRec{nullptr, nullptr, 0}, false));
    if (c->dist) TRY(phase_halo(c, c->step));
    return DPD_OK;
}

// In-process group: every phase for every member, then the device-copy exchange.
int group_prime(dpd_ctx **g, int n)
{
    // identical message layouts on every member, sized from the global density
    int64_t nglob = 0;
    for (int r = 0; r < n; ++r) nglob += g[r]->n;
    const double rho = (double)nglob / (g[0]->box[0] * g[0]->box[1] * g[0]->box[2]);
    for (int r = 0; r < n; ++r)
        if (!g[r]->msgs_ready) TRY(setup_messages(g[r], rho));
    for (int r = 0; r < n; ++r) TRY(phase_ghost_pack(g[r]));
    TRY(exchange_group(g, n, true));
    for (int r = 0; r < n; ++r) {
        TRY(force_pass(g[r], g[r]->step, g[r]->frc[g[r]->cur].p, PairRec{nullptr, nullptr, 0}, false));
        TRY(phase_halo(g[r], g[r]->step));
        g[r]->need_prime = false;
    }
    return DPD_OK;
}

// The in-process group's step as one task graph: the production step of build_step_graph for
// every member -- kick_drift_bin -> migrate_exchange -> scan_scatter -> [ghost_pack ->
// ghost_exchange -> ghost_sort] on the member's communication stream, concurrent with
// force_local on the compute stream -> halo_force -- with the NCCL send/recv tasks swapped
// for one device copy of every member's capacity-padded messages (the bytes NCCL sends).
// Slot 0 = the group's compute stream, slot 1 + r = member r's communication stream;
// cross-slot edges are CUDA events (TaskGraph::run).
dpd::TaskGraph *build_group_graph(dpd_ctx **g, int n)
{
    auto *G = new dpd::TaskGraph();
    std::vector<int> bin(n), sort(n), pack(n), gsort(n), force(n);
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        bin[r] = G->add("kick_drift_bin", 0, [c](cudaStream_t) {
            const float kick = c->primed ? (float)(0.5 * c->dt) : (float)c->dt;
            c->ip_step = integ(c, (float)c->dt, kick);
            return phase_bin(c, c->ip_step);
        });
    }
    const int mx = G->add("migrate_exchange", 0, [g, n](cudaStream_t s) { return exchange_group(g, n, false, s, true); });
    for (int r = 0; r < n; ++r) G->edge(bin[r], mx);
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        sort[r] = G->add("scan_scatter", 0, [c](cudaStream_t) -> int {
            TRY(phase_sort(c, c->ip_step));
            c->step += 1;
            return DPD_OK;
        });
        G->edge(mx, sort[r]);
    }
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        pack[r] = G->add("ghost_pack", 1 + r, [c](cudaStream_t s) { return phase_ghost_pack(c, s); });
        G->edge(sort[r], pack[r]);
    }
    const int gx = G->add("ghost_exchange", 1, [g, n](cudaStream_t s) { return exchange_group(g, n, true, s, true); });
    for (int r = 0; r < n; ++r) G->edge(pack[r], gx);
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        gsort[r] = G->add("ghost_sort", 1 + r, [c](cudaStream_t s) { return phase_ghost_sort(c, s); });
        G->edge(gx, gsort[r]);
    }
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        force[r] = G->add("force_local", 0, [c](cudaStream_t) {
            return force_pass(c, c->step, c->frc[c->cur].p, PairRec{nullptr, nullptr, 0}, false);
        });
        G->edge(sort[r], force[r]);
    }
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        const int h = G->add("halo_force", 0, [c](cudaStream_t) {
            const int rc = phase_halo_force(c, c->step);
            c->primed = false;
            return rc;
        });
        G->edge(force[r], h);
        G->edge(gsort[r], h);
    }
    if (G->build() != 0) {
        delete G;
        return nullptr;
    }
    return G;
}

int group_step_graph(dpd_ctx **g, int n)
{
    dpd_ctx *c0 = g[0];
    if (!c0->group_graph) {
        c0->group_graph = build_group_graph(g, n);
        if (!c0->group_graph) return fail(c0, DPD_ERR_CONFIG, "group task graph has a cycle");
    }
    std::vector<cudaStream_t> streams(1 + n);
    streams[0] = c0->stream;
    for (int r = 0; r < n; ++r) streams[1 + r] = g[r]->comm_stream ? g[r]->comm_stream : c0->stream;
    const int rc = c0->group_graph->run(streams.data());
    if (rc == -1) return fail(c0, DPD_ERR_CONFIG, "group task graph has a cycle");
    if (rc == -2) return fail(c0, DPD_ERR_CUDA, "group task graph: %s", cudaGetErrorString(cudaGetLastError()));
    return rc;
}

int group_step(dpd_ctx **g, int n)
{
    if (g[0]->group_graph_mode) return group_step_graph(g, n);
    IntegP ip[64];
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        ip[r] = integ(c, (float)c->dt, c->primed ? (float)(0.5 * c->dt) : (float)c->dt);
        TRY(phase_bin(c, ip[r]));
    }
    TRY(exchange_group(g, n, false));
    for (int r = 0; r < n; ++r) {
        TRY(phase_sort(g[r], ip[r]));
        g[r]->step += 1;
        TRY(phase_ghost_pack(g[r]));
    }
    TRY(exchange_group(g, n, true));
    for (int r = 0; r < n; ++r) {
        dpd_ctx *c = g[r];
        TRY(force_pass(c, c->step, c->frc[c->cur].p, PairRec{nullptr, nullptr, 0}, false));
        TRY(phase_halo(c, c->step));
        c->primed = false;
    }
    return DPD_OK;
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

// Geometry of a (sub)domain of extent len with the given split flags.
int setup_geometry(dpd_ctx *c, const double len[3], const int split[3])
{
    Geom g{};
    int64_t ncell = 1;
    for (int k = 0; k < 3; ++k) {
        const int nd = (int)std::floor(len[k] / c->rc);
        if (nd < 3) return fail(c, DPD_ERR_CONFIG, "subdomain needs >= 3 cells per dimension (dim %d: %d)", k, nd);
        if ((split[0] || split[1] || split[2]) && nd >= 1024) // boundary-cell list: 10-bit coordinates
            return fail(c, DPD_ERR_CONFIG, "a decomposed subdomain needs < 1024 cells per dimension (dim %d: %d)", k, nd);
        g.n[k] = nd;
        g.split[k] = split[k];
        g.off[k] = split[k] ? 1 : 0;
        g.ext[k] = nd + 2 * g.off[k];
        g.L[k] = (float)len[k];
        volatile float nf = (float)nd, lf = (float)len[k];
        g.inv_h[k] = nf / lf;
        ncell *= g.ext[k];
        c->sub[k] = len[k];
    }
    if (ncell > (int64_t)1 << 30) return fail(c, DPD_ERR_CONFIG, "too many cells (%lld)", (long long)ncell);
    g.ncell = (int)ncell;
    c->geom = g;
    return DPD_OK;
}

// Fixed-point scale of the tiled kernel for the largest pair amplitudes a and
// gamma in use: bound a single pair's force magnitude by a + 6.7 sigma/sqrt(dt) (|xi| <= 6.66
// with 32-bit u1) + 20 gamma max(1, sqrt(kT)) (relative speed), keep |f scale| < 2^21;
// larger magnitudes are detected on the device and reported as DPD_ERR_NUMERIC.
// sqrt(2 ln 2): the device pair paths use box_muller_s = xi / sqrt(2 ln 2) and fold the
// constant into sigma/sqrt(dt) here (PairP::sig_dt, PairP::ss)
constexpr double kBMd = 1.1774100225154747;

void set_fixed_scale(dpd_ctx *c, double amax, double gmax)
{
    const double sig_dt = std::sqrt(2.0 * gmax * c->kT) / std::sqrt(c->dt);
    const double bound = amax + 6.7 * sig_dt + 20.0 * gmax * std::max(1.0, std::sqrt(c->kT)) + 1e-30;
    int k = (int)std::floor(std::log2(std::ldexp(1.0, 21) / bound));
    k = std::min(20, std::max(-20, k));
    c->fix.scale = (float)std::ldexp(1.0, k);
    c->fix.inv_scale = (float)std::ldexp(1.0, -k);
    c->fix.mag_lim = (float)std::ldexp(1.0, 21 - k);
    // row-end pruning slack: far above the cell-binning rounding of
    // coordinates up to the box extent, far below any cell size
    const double lmax = std::max(c->box[0], std::max(c->box[1], c->box[2]));
    c->fix.slack = (float)(1e-4 + lmax * std::ldexp(1.0, -20));
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
    for (int d = 0; d < 27; ++d) c->peer_to[d] = c->peer_from[d] = -1;
    PairP pp{};
    pp.a = (float)a;
    pp.gamma = (float)gamma;
    pp.sig_dt = (float)(std::sqrt(2.0 * gamma * kT) / std::sqrt(dt) * kBMd); // x sqrt(2 ln 2): box_muller_s
    pp.sa[0] = pp.a; // one species until dpd_set_species
    pp.sg[0] = pp.gamma;
    pp.ss[0] = pp.sig_dt;
    pp.inv_rc = (float)(1.0 / rc);
    pp.rc2 = (float)(rc * rc);
    pp.power = (float)power;
    pp.seed_lo = (uint32_t)seed;
    pp.seed_hi = (uint32_t)(seed >> 32);
    c->pp = pp;
    set_fixed_scale(c, a, gamma);
    {
        // three tiles per SM need the maximum shared-memory carveout (3 x (smem + 1 KB) <= 228 KB)
        const int smem = (int)sizeof(ForceTileSmem);
        const void *fns[8] = {(const void *)k_force_tile<false, 0>, (const void *)k_force_tile<false, 1>,
                              (const void *)k_force_tile<false, 2>, (const void *)k_force_tile<false, 3>,
                              (const void *)k_force_tile<true, 0>,  (const void *)k_force_tile<true, 1>,
                              (const void *)k_force_tile<true, 2>,  (const void *)k_force_tile<true, 3>};
        int dev = 0;
        CUDA_TRY(c, cudaGetDevice(&dev));
        CUDA_TRY(c, cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev));
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
    CUDA_TRY(c, cudaMallocHost(&c->h_err, 16 * sizeof(int)));
    CUDA_TRY(c, c->scan_epoch.reserve(2));
    CUDA_TRY(c, cudaMemset(c->scan_epoch.p, 0, 2 * sizeof(unsigned)));
    return DPD_OK;
}

int alloc_grid(dpd_ctx *c)
{
    const int ncell = c->geom.ncell;
    CUDA_TRY(c, c->count.reserve((size_t)ncell + 16));
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(c, c->start[b].reserve((size_t)ncell + 16));
        CUDA_TRY(c, cudaMemset(c->start[b].p, 0, sizeof(int) * c->start[b].cap));
    }
    const int ntile = (ncell + kScanTile - 1) / kScanTile;
    CUDA_TRY(c, c->scan_state.reserve((size_t)ntile));
    CUDA_TRY(c, cudaMemset(c->count.p, 0, sizeof(int) * c->count.cap));
    CUDA_TRY(c, cudaMemset(c->scan_state.p, 0, sizeof(unsigned long long) * c->scan_state.cap));
    if (c->dist) {
        CUDA_TRY(c, c->gcount.reserve((size_t)ncell + 16));
        CUDA_TRY(c, c->gstart.reserve((size_t)ncell + 16));
        CUDA_TRY(c, c->gscan_state.reserve((size_t)ntile));
        CUDA_TRY(c, cudaMemset(c->gcount.p, 0, sizeof(int) * c->gcount.cap));
        CUDA_TRY(c, cudaMemset(c->gstart.p, 0, sizeof(int) * c->gstart.cap));
        CUDA_TRY(c, cudaMemset(c->gscan_state.p, 0, sizeof(unsigned long long) * c->gscan_state.cap));
    }
    return DPD_OK;
}

// Rank grid bookkeeping: coordinates and the peers of every direction.
void setup_ranks(dpd_ctx *c, int rank, const int32_t grid[3])
{
    c->rank = rank;
    for (int k = 0; k < 3; ++k) c->grid[k] = grid[k];
    c->world = grid[0] * grid[1] * grid[2];
    c->coord[0] = rank % grid[0];
    c->coord[1] = (rank / grid[0]) % grid[1];
    c->coord[2] = rank / (grid[0] * grid[1]);
    for (int d = 0; d < 27; ++d) {
        const int D[3] = {d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1};
        int to[3], from[3];
        for (int k = 0; k < 3; ++k) {
            to[k] = (c->coord[k] + D[k] + grid[k]) % grid[k];
            from[k] = (c->coord[k] - D[k] + grid[k]) % grid[k];
        }
        c->peer_to[d] = to[0] + grid[0] * (to[1] + grid[1] * to[2]);
        c->peer_from[d] = from[0] + grid[0] * (from[1] + grid[1] * from[2]);
    }
    for (int k = 0; k < 3; ++k) c->origin[k] = (float)(c->coord[k] * c->sub[k]);
}

// loop[k] (may be null): dimension k is split although grid[k] == 1 -- its periodic halo and
// migrants travel through the exchange to the rank itself (dpd_create_loopback).
int create_common(const double box[3], double rc, double a, double gamma, double kT, double power, double dt,
                  uint64_t seed, int rank, const int32_t grid[3], dpd_ctx **out, dpd_ctx *c,
                  const int32_t *loop = nullptr)
{
    int r = init_ctx(c, box, rc, a, gamma, kT, power, dt, seed);
    if (r != DPD_OK) return r;
    double sub[3];
    int split[3];
    for (int k = 0; k < 3; ++k) {
        if (grid[k] < 1) return fail(c, DPD_ERR_CONFIG, "grid[%d] = %d must be >= 1", k, grid[k]);
        sub[k] = box[k] / grid[k];
        split[k] = grid[k] > 1 || (loop && loop[k] != 0);
    }
    c->dist = split[0] || split[1] || split[2];
    TRY(setup_geometry(c, sub, split));
    setup_ranks(c, rank, grid);
    TRY(alloc_grid(c));
    if (c->dist) {
        // the communication stream at the highest priority: its ghost pack / exchange / sort
        // become ready when the interior force kernel already fills every SM, and take the
        // slots its CTAs free first, instead of queueing behind the whole force pass
        int prio_lo = 0, prio_hi = 0;
        CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        CUDA_TRY(c, cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, prio_hi));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_ghost, cudaEventDisableTiming));
    }
    *out = c;
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
    const int32_t grid[3] = {1, 1, 1};
    int r = create_common(box, rc, a, gamma, kT, power, dt, seed, 0, grid, out, c);
    if (r != DPD_OK) {
        fprintf(stderr, "dpd_create: %s\n", c->last_error.c_str());
        *out = nullptr;
        dpd_destroy(c);
    }
    return r;
}

void dpd_destroy(dpd_ctx *c)
{
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    if (c->dump) dpd_dump_close(c, nullptr);
    for (auto *g : c->step_graph) delete g;
    delete c->group_graph;
    for (int b = 0; b < 2; ++b) {
        c->pos[b].release();
        c->vel[b].release();
        c->frc[b].release();
        c->start[b].release();
    }
    c->rank_buf.release();
    c->count.release();
    c->scan_state.release();
    c->scan_epoch.release();
    c->err.release();
    c->stage.release();
    c->mig.send.release();
    c->mig.recv.release();
    c->gh.send.release();
    c->gh.recv.release();
    c->rank_in.release();
    c->gcount.release();
    c->blist.release();
    c->gstart.release();
    c->grank.release();
    c->gpos.release();
    c->gvel.release();
    c->gscan_state.release();
    for (auto &p : c->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    if (c->ev_pack) cudaEventDestroy(c->ev_pack);
    if (c->ev_ghost) cudaEventDestroy(c->ev_ghost);
#ifdef DPD_HAVE_NCCL
    if (c->nccl) ncclCommDestroy(c->nccl);
#endif
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->h_err) cudaFreeHost(c->h_err);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (c->group) {
        // the group array and stream are shared: the last member to go frees them
        int alive = 0;
        for (int r = 0; r < c->group_n; ++r)
            if (c->group[r] && c->group[r] != c) ++alive;
        for (int r = 0; r < c->group_n; ++r)
            if (c->group[r] == c) c->group[r] = nullptr;
        if (alive == 0) {
            delete[] c->group;
            if (c->stream) cudaStreamDestroy(c->stream);
        }
    }
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
        if (value != 0 && c->dist) return fail(c, DPD_ERR_ARG, "force_kernel %d is single-domain only", (int)value);
        c->force_impl = (int)value;
        return DPD_OK;
    }
    if (strcmp(name, "group_task_graph") == 0) {
        if (value < 0 || value > 1) return fail(c, DPD_ERR_ARG, "group_task_graph must be 0 or 1");
        if (!c->group || c->group[0] != c) return fail(c, DPD_ERR_ARG, "group_task_graph is set on member 0 of a group");
        c->group_graph_mode = (int)value;
        return DPD_OK;
    }
    if (strcmp(name, "body_force_mode") == 0) {
        if (value < 0 || value > 1) return fail(c, DPD_ERR_ARG, "body_force_mode must be 0 or 1");
        c->body_mode = (int)value;
        return DPD_OK;
    }
    if (strcmp(name, "dump_delay_us") == 0) {
        if (!c->dump) return fail(c, DPD_ERR_ARG, "dpd_dump_open first");
        if (value < 0 || value > 60000000) return fail(c, DPD_ERR_ARG, "dump_delay_us out of range");
        c->dump->delay_us = value;
        return DPD_OK;
    }
    if (strcmp(name, "message_capacity_percent") == 0) {
        if (value < 10 || value > 100000) return fail(c, DPD_ERR_ARG, "message_capacity_percent out of range");
        c->cap_factor = value / 100.0;
        c->msgs_ready = false; // re-sized at the next set_particles
        return DPD_OK;
    }
    return fail(c, DPD_ERR_ARG, "unknown option '%s'", name);
}

int dpd_get_stat(dpd_ctx *c, const char *name, int64_t *value)
{
    if (!c || !name || !value) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (strcmp(name, "fallback_tiles") == 0) {
        *value = c->fallback[0] + c->fallback[1];
        return DPD_OK;
    }
    if (strcmp(name, "fallback_staged") == 0) { *value = c->fallback[0]; return DPD_OK; }
    if (strcmp(name, "fallback_home") == 0) { *value = c->fallback[1]; return DPD_OK; }
    if (strcmp(name, "full_list_particles") == 0) { *value = c->fallback[2]; return DPD_OK; }
    return fail(c, DPD_ERR_ARG, "unknown statistic '%s'", name);
}

int dpd_set_species(dpd_ctx *c, int nspecies, const double *a, const double *gamma)
{
    if (!c) return DPD_ERR_ARG;
    if (nspecies < 1 || nspecies > DPD_MAX_SPECIES)
        return fail(c, DPD_ERR_ARG, "nspecies must be in [1, %d]", DPD_MAX_SPECIES);
    if (!a || !gamma) return fail(c, DPD_ERR_ARG, "null species matrix");
    if (c->primed) return fail(c, DPD_ERR_ARG, "dpd_set_species must precede dpd_set_particles*");
    const int ns = nspecies;
    double amax = 0.0, gmax = 0.0;
    for (int i = 0; i < ns; ++i)
        for (int j = 0; j < ns; ++j) {
            const double av = a[i * ns + j], gv = gamma[i * ns + j];
            if (!std::isfinite(av) || !std::isfinite(gv) || av < 0.0 || gv < 0.0)
                return fail(c, DPD_ERR_CONFIG, "species matrix entries must be finite and >= 0");
            if (av != a[j * ns + i] || gv != gamma[j * ns + i])
                return fail(c, DPD_ERR_CONFIG, "species matrices must be symmetric (Newton-3 pairs)");
            amax = std::max(amax, av);
            gmax = std::max(gmax, gv);
        }
    PairP &pp = c->pp;
    for (int t = 0; t < DPD_MAX_SPECIES * DPD_MAX_SPECIES; ++t) pp.sa[t] = pp.sg[t] = pp.ss[t] = 0.0f;
    for (int i = 0; i < ns; ++i)
        for (int j = 0; j < ns; ++j) {
            const int t = i * DPD_MAX_SPECIES + j;
            const double gv = gamma[i * ns + j];
            pp.sa[t] = (float)a[i * ns + j];
            pp.sg[t] = (float)gv;
            pp.ss[t] = (float)(std::sqrt(2.0 * gv * c->kT) / std::sqrt(c->dt) * kBMd); // FDT per pair
        }
    if (ns == 1) {
        c->a = a[0];
        c->gamma = gamma[0];
        pp.a = (float)a[0];
        pp.gamma = (float)gamma[0];
        pp.sig_dt = pp.ss[0];
    }
    c->nspecies = ns;
    c->kmode = (ns > 1) ? 3 : ((c->power == 0.5) ? 0 : (c->power == 1.0 ? 1 : 2));
    set_fixed_scale(c, amax, gmax);
    return DPD_OK;
}

int dpd_set_walls(dpd_ctx *c, int nprim, const int32_t *type, const double *prm, const double *uw)
{
    if (!c) return DPD_ERR_ARG;
    if (nprim < 0 || nprim > DPD_MAX_WALLS) return fail(c, DPD_ERR_ARG, "nprim must be in [0, %d]", DPD_MAX_WALLS);
    if (nprim > 0 && (!type || !prm || !uw)) return fail(c, DPD_ERR_ARG, "null wall arrays");
    for (int k = 0; k < nprim; ++k) {
        const double *q = prm + 4 * k;
        for (int t = 0; t < 4; ++t)
            if (!std::isfinite(q[t])) return fail(c, DPD_ERR_CONFIG, "wall %d: non-finite parameter", k);
        for (int t = 0; t < 3; ++t)
            if (!std::isfinite(uw[3 * k + t])) return fail(c, DPD_ERR_CONFIG, "wall %d: non-finite velocity", k);
        if (type[k] == 1) {
            const double nn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
            if (std::fabs(nn - 1.0) > 1e-6) return fail(c, DPD_ERR_CONFIG, "wall %d: plane normal must be unit", k);
        } else if (type[k] >= 2 && type[k] <= 4) {
            if (!(q[2] > 0.0) || std::fabs(std::fabs(q[3]) - 1.0) != 0.0)
                return fail(c, DPD_ERR_CONFIG, "wall %d: cylinder needs R > 0 and sign +-1", k);
        } else {
            return fail(c, DPD_ERR_CONFIG, "wall %d: unknown type %d", k, (int)type[k]);
        }
    }
    c->nwall = nprim;
    for (int k = 0; k < DPD_MAX_WALLS; ++k) {
        c->wtype[k] = k < nprim ? type[k] : 0;
        for (int t = 0; t < 4; ++t) c->wprm[k][t] = k < nprim ? (float)prm[4 * k + t] : 0.0f;
        for (int t = 0; t < 3; ++t) c->wvel[k][t] = k < nprim ? (float)uw[3 * k + t] : 0.0f;
    }
    return DPD_OK;
}

int dpd_set_frozen_species(dpd_ctx *c, int32_t mask)
{
    if (!c) return DPD_ERR_ARG;
    if (mask < 0) return fail(c, DPD_ERR_ARG, "mask must be >= 0");
    c->frozen_mask = mask;
    return DPD_OK;
}

int dpd_wall_sdf(dpd_ctx *c, int64_t n, const float *x, float *sdf)
{
    if (!c) return DPD_ERR_ARG;
    if (n < 0 || (n > 0 && (!x || !sdf))) return fail(c, DPD_ERR_ARG, "bad arguments");
    if (n == 0) return DPD_OK;
    TRY(sync_check(c));
    CUDA_TRY(c, c->stage.reserve((size_t)n * 4));
    float *dx = c->stage.p, *ds = c->stage.p + 3 * n;
    CUDA_TRY(c, cudaMemcpyAsync(dx, x, sizeof(float) * 3 * n, cudaMemcpyDefault, c->stream));
    IntegP ip = integ(c, 0.0f, 0.0f);
    ip.origin[0] = ip.origin[1] = ip.origin[2] = 0.0f; // x is global
    TRY(launch(c, KID_DEBUG, [&] { k_wall_sdf_eval<<<nblk(n, 256), 256, 0, c->stream>>>(dx, (int)n, ip, ds); }));
    CUDA_TRY(c, cudaMemcpyAsync(sdf, ds, sizeof(float) * n, cudaMemcpyDefault, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return DPD_OK;
}

int dpd_wall_carve(dpd_ctx *c, int32_t wall_species, int64_t *n_frozen, int64_t *n_removed)
{
    if (!c) return DPD_ERR_ARG;
    if (wall_species < 0 || wall_species > 30 || (c->nspecies > 1 && wall_species >= c->nspecies))
        return fail(c, DPD_ERR_ARG, "wall species %d out of range", (int)wall_species);
    TRY(sync_check(c));
    if (c->need_prime) return fail(c, DPD_ERR_ARG, "group members must be primed (dpd_group_step(.., 0)) first");
    const int n = (int)c->n;
    const int b = c->cur, o = 1 - c->cur;
    ScopedBuf<int> keep, cnt, kbid, nid, epoch; // freed on every return path
    ScopedBuf<unsigned long long> tstate;
    CUDA_TRY(c, keep.reserve((size_t)std::max(n, 1)));
    CUDA_TRY(c, cnt.reserve(2));
    CUDA_TRY(c, cudaMemsetAsync(cnt.p, 0, 2 * sizeof(int), c->stream));
    const bool renumber = c->dense_ids && !c->dist && n > 0;
    if (renumber) {
        CUDA_TRY(c, kbid.reserve((size_t)n));
        CUDA_TRY(c, nid.reserve((size_t)n + 1));
        const size_t tiles = (size_t)(n + kScanTile - 1) / kScanTile;
        CUDA_TRY(c, tstate.reserve(tiles));
        CUDA_TRY(c, epoch.reserve(1));
        CUDA_TRY(c, cudaMemsetAsync(tstate.p, 0, tiles * sizeof(unsigned long long), c->stream));
        CUDA_TRY(c, cudaMemsetAsync(epoch.p, 0, sizeof(int), c->stream));
    }
    const IntegP ip = integ(c, 0.0f, 0.0f);
    const float hk = c->primed ? 0.0f : (float)(0.5 * c->dt); // stored u -> full-step v
    int hc[2] = {0, 0};
    if (n > 0) {
        TRY(launch(c, KID_GATHER, [&] {
            k_wall_classify<<<nblk(n, 256), 256, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, c->frc[b].p, n, ip, hk,
                                                                 (float)c->rc, wall_species, keep.p, cnt.p);
        }));
        CUDA_TRY(c, cudaMemsetAsync(count_ptr(c), 0, sizeof(int), c->stream));
        TRY(launch(c, KID_GATHER, [&] {
            k_wall_compact<<<nblk(n, 256), 256, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, n, keep.p, c->pos[o].p,
                                                                c->vel[o].p, c->frc[o].p, count_ptr(c),
                                                                renumber ? kbid.p : nullptr);
        }));
        CUDA_TRY(c, cudaMemcpyAsync(hc, cnt.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        c->cur = o;
        TRY(sync_check(c));
        if (renumber && hc[1] > 0) {
            const unsigned tiles = (unsigned)((n + kScanTile - 1) / kScanTile);
            TRY(launch(c, KID_GATHER, [&] {
                k_scan<<<tiles, kScanThreads, 0, c->stream>>>(kbid.p, nid.p, n, tstate.p,
                                                              reinterpret_cast<unsigned *>(epoch.p));
            }));
            TRY(launch(c, KID_GATHER, [&] {
                k_renumber<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->pos[c->cur].p, (int)c->n, nid.p);
            }));
        }
    }
    c->frozen_mask |= 1 << wall_species;
    // re-sort the survivors into cells (dt = 0) and prime F at the current step (C-2 item 2)
    const IntegP ip0 = integ(c, 0.0f, 0.0f);
    TRY(phase_bin(c, ip0, false));
    TRY(phase_sort(c, ip0, false, true));
    c->primed = true;
    if (c->group) {
        c->need_prime = true;
    } else {
        TRY(prime_one(c));
    }
    TRY(sync_check(c));
    if (n_frozen) *n_frozen = hc[0];
    if (n_removed) *n_removed = hc[1];
    return DPD_OK;
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
    return dpd_set_particles_typed(c, n, pos, vel, ids, nullptr, step0);
}

int dpd_set_particles_typed(dpd_ctx *c, int64_t n, const float *pos, const float *vel, const int32_t *ids,
                            const int32_t *species, int64_t step0)
{
    if (!c) return DPD_ERR_ARG;
    if (n < 0 || n > (int64_t)INT32_MAX / 2) return fail(c, DPD_ERR_ARG, "bad particle count %lld", (long long)n);
    if (n > 0 && (!pos || !vel)) return fail(c, DPD_ERR_ARG, "null pos/vel");
    if (step0 < 0) return fail(c, DPD_ERR_ARG, "step0 must be >= 0");
    TRY(sync_check(c));
    // dense-id check (host): ids must be a permutation of 0..n-1 for id-order getters
    bool dense = !c->dist;
    if (ids && dense) {
        std::vector<char> seen((size_t)n, 0);
        for (int64_t i = 0; i < n; ++i) {
            const int32_t id = ids[i];
            if (id < 0) return fail(c, DPD_ERR_ARG, "negative id at %lld", (long long)i);
            if (id >= n || seen[(size_t)id]) { dense = false; continue; }
            seen[(size_t)id] = 1;
        }
    }
    c->dense_ids = dense;
    c->step = step0;
    c->cur = 0;
    c->scur = 0;
    // 8 words per particle for this upload; 10 covers every getter (gather 9, forces 10), so a
    // first get does not re-allocate (cudaFree + cudaMalloc synchronise the device)
    const size_t words = (size_t)std::max<int64_t>(n, 1) * 10;
    CUDA_TRY(c, c->stage.reserve(words));
    float *d_pos = c->stage.p, *d_vel = c->stage.p + 3 * (size_t)n;
    int32_t *d_ids = ids ? reinterpret_cast<int32_t *>(c->stage.p + 6 * (size_t)n) : nullptr;
    int32_t *d_species = species ? reinterpret_cast<int32_t *>(c->stage.p + 7 * (size_t)n) : nullptr;
    int *n_out = count_ptr(c);
    const float3 gbox = make_float3((float)c->box[0], (float)c->box[1], (float)c->box[2]);
    const float3 org = make_float3(c->origin[0], c->origin[1], c->origin[2]);
    CUDA_TRY(c, cudaMemsetAsync(n_out, 0, sizeof(int), c->stream));
    if (n > 0) {
        CUDA_TRY(c, cudaMemcpyAsync(d_pos, pos, sizeof(float) * 3 * n, cudaMemcpyDefault, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(d_vel, vel, sizeof(float) * 3 * n, cudaMemcpyDefault, c->stream));
        if (ids) CUDA_TRY(c, cudaMemcpyAsync(d_ids, ids, sizeof(int32_t) * n, cudaMemcpyDefault, c->stream));
        if (species)
            CUDA_TRY(c, cudaMemcpyAsync(d_species, species, sizeof(int32_t) * n, cudaMemcpyDefault, c->stream));
    }
    // particle arrays: exactly n on one domain; decomposed runs count the particles inside the
    // subdomain first and leave room for migration fluctuations
    int64_t want = n;
    if (c->dist && n > 0) {
        const float3 sub = make_float3((float)c->sub[0], (float)c->sub[1], (float)c->sub[2]);
        TRY(launch(c, KID_PACK, [&] {
            k_count_inside<<<nblk(n, 256), 256, 0, c->stream>>>(d_pos, n, gbox, org, sub, n_out);
        }));
        int inside = 0;
        CUDA_TRY(c, cudaMemcpyAsync(&inside, n_out, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        want = (int64_t)(1.1 * inside + 12.0 * std::sqrt((double)inside + 1.0) + 4096.0);
        CUDA_TRY(c, cudaMemsetAsync(n_out, 0, sizeof(int), c->stream));
    }
    TRY(ensure_capacity(c, want));
    if (n > 0) {
        const Geom g = c->geom;
        const int cap = (int)c->n_cap;
        TRY(launch(c, KID_PACK, [&] {
            k_pack_input<<<nblk(n, 256), 256, 0, c->stream>>>(d_pos, d_vel, d_ids, d_species, c->nspecies, n, g,
                                                              gbox, org, c->pos[0].p, c->vel[0].p, c->frc[0].p,
                                                              n_out, cap, c->err.p);
        }));
    }
    TRY(sync_check(c)); // local count (capacity errors surface here)
    if (c->dist) {
        int64_t nglob = c->n;
#ifdef DPD_HAVE_NCCL
        if (c->nccl) {
            // global count -> density for the message capacities (collective on all ranks)
            DevBuf<long long> t;
            CUDA_TRY(c, t.reserve(1));
            long long v = c->n;
            CUDA_TRY(c, cudaMemcpy(t.p, &v, sizeof v, cudaMemcpyHostToDevice));
            NCCL_TRY(c, ncclAllReduce(t.p, t.p, 1, ncclInt64, ncclSum, c->nccl, c->stream));
            CUDA_TRY(c, cudaMemcpyAsync(&v, t.p, sizeof v, cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(c, cudaStreamSynchronize(c->stream));
            t.release();
            nglob = v;
        }
#endif
        // in-process groups size their messages once every member is set (dpd_group_step)
        if (!c->group && !c->msgs_ready)
            TRY(setup_messages(c, (double)nglob / (c->box[0] * c->box[1] * c->box[2])));
    }
    // sort into cells without moving (dt = 0, kick = 0), then prime F_0 at s = step0
    const IntegP ip0 = integ(c, 0.0f, 0.0f);
    TRY(phase_bin(c, ip0, false));
    TRY(phase_sort(c, ip0, false, true));
    c->primed = true;
    if (c->group) {
        c->need_prime = true; // forces need every member's ghosts: dpd_group_step(..., 0)
    } else {
        TRY(prime_one(c));
    }
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
    if (c->group) return fail(c, DPD_ERR_ARG, "group members are stepped with dpd_group_step");
    for (int64_t it = 0; it < nsteps; ++it) {
        const bool due = c->dump && c->dump->every > 0 && (c->step + 1) % c->dump->every == 0;
        TRY(step_one(c, due));
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

static int gather(dpd_ctx *c, float *pos, float *vel, float *f, int by_id)
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
    const IntegP ip = integ(c, 0.0f, 0.0f);
    const float3 org = make_float3(c->origin[0], c->origin[1], c->origin[2]);
    TRY(launch(c, KID_GATHER, [&] {
        k_gather_id<<<nblk(cnt, 256), 256, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, c->frc[b].p, (int)cnt, hk, ip,
                                                           org, d_pos, d_vel, d_f, by_id);
    }));
    if (pos) CUDA_TRY(c, cudaMemcpyAsync(pos, d_pos, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    if (vel) CUDA_TRY(c, cudaMemcpyAsync(vel, d_vel, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    if (f) CUDA_TRY(c, cudaMemcpyAsync(f, d_f, sizeof(float) * 3 * cnt, cudaMemcpyDefault, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return DPD_OK;
}

static int copy_ids(dpd_ctx *c, int32_t *ids)
{
    if (!ids || c->n == 0) return DPD_OK;
    CUDA_TRY(c, c->stage.reserve((size_t)c->n));
    int32_t *d = reinterpret_cast<int32_t *>(c->stage.p);
    const int b = c->cur;
    const Geom g = c->geom;
    TRY(launch(c, KID_GATHER, [&] {
        k_ids_cells<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->pos[b].p, (int)c->n, g, d, nullptr);
    }));
    CUDA_TRY(c, cudaMemcpyAsync(ids, d, sizeof(int32_t) * c->n, cudaMemcpyDefault, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return DPD_OK;
}

int dpd_get_particles(dpd_ctx *c, int64_t n, float *pos, float *vel)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n != c->n) return fail(c, DPD_ERR_ARG, "n = %lld but the context holds %lld", (long long)n, (long long)c->n);
    if (!c->dense_ids) return fail(c, DPD_ERR_ARG, "ids are not dense 0..n-1; use dpd_get_particles_ex");
    return gather(c, pos, vel, nullptr, 1);
}

int dpd_get_forces(dpd_ctx *c, int64_t n, float *f)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n != c->n) return fail(c, DPD_ERR_ARG, "n = %lld but the context holds %lld", (long long)n, (long long)c->n);
    if (!c->dense_ids) return fail(c, DPD_ERR_ARG, "ids are not dense 0..n-1; use dpd_get_forces_ex");
    return gather(c, nullptr, nullptr, f, 1);
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
    const float3 org = make_float3(c->origin[0], c->origin[1], c->origin[2]);
    TRY(launch(c, KID_GATHER, [&] {
        k_state<<<nblk(cnt, 256), 256, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, c->frc[b].p, (int)cnt, org, dp, du,
                                                      df, di);
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
    if (c->dist) return fail(c, DPD_ERR_ARG, "dpd_debug_cells is single-domain only");
    TRY(sync_check(c));
    const int ncell = c->geom.ncell;
    const int64_t cnt = c->n;
    if (cell_of_id && !c->dense_ids) return fail(c, DPD_ERR_ARG, "cell_of_id needs dense ids");
    std::vector<int32_t> st((size_t)ncell + 1);
    CUDA_TRY(c, cudaMemcpy(st.data(), c->start[c->scur].p, sizeof(int32_t) * (ncell + 1), cudaMemcpyDeviceToHost));
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
    if (c->dist) return fail(c, DPD_ERR_ARG, "dpd_debug_pairs is single-domain only");
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
    k_pair_words<<<nblk(n, 128), 128>>>(din, (uint32_t)seed, (uint32_t)(seed >> 32), dxi, dw, (int)n);
    cudaMemcpy(words, dw, sizeof(uint2) * n, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaMemcpy(xi, dxi, sizeof(float) * n, cudaMemcpyDeviceToHost);
    cudaFree(din);
    cudaFree(dw);
    cudaFree(dxi);
    return e == cudaSuccess ? DPD_OK : DPD_ERR_CUDA;
}

// ---- multi-GPU -------------------------------------------------------------------------------
int dpd_plan_peers(const int32_t grid[3], int rank, int32_t peer_to[27], int32_t peer_from[27], int32_t used[27])
{
    if (!grid || grid[0] < 1 || grid[1] < 1 || grid[2] < 1) return DPD_ERR_ARG;
    const int world = grid[0] * grid[1] * grid[2];
    if (rank < 0 || rank >= world) return DPD_ERR_ARG;
    dpd_ctx tmp; // host-only bookkeeping, no device state touched
    for (int k = 0; k < 3; ++k) tmp.sub[k] = 1.0;
    setup_ranks(&tmp, rank, grid);
    for (int d = 0; d < 27; ++d) {
        const int D[3] = {d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1};
        bool u = d != 13;
        for (int k = 0; k < 3; ++k)
            if (D[k] != 0 && grid[k] < 2) u = false;
        if (peer_to) peer_to[d] = tmp.peer_to[d];
        if (peer_from) peer_from[d] = tmp.peer_from[d];
        if (used) used[d] = u;
    }
    return DPD_OK;
}

int dpd_nccl_unique_id(uint8_t id[128])
{
#ifdef DPD_HAVE_NCCL
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return DPD_ERR_COMM;
    memcpy(id, &u, 128);
    return DPD_OK;
#else
    (void)id;
    return DPD_ERR_COMM;
#endif
}

int dpd_create_dist(const double box[3], double rc, double a, double gamma, double kT, double power, double dt,
                    uint64_t seed, int rank, int world, const int32_t grid[3], const uint8_t nccl_id[128],
                    dpd_ctx **out)
{
    if (!out || !box || !grid || !nccl_id) return DPD_ERR_ARG;
    *out = nullptr;
    if (world != grid[0] * grid[1] * grid[2] || rank < 0 || rank >= world) return DPD_ERR_ARG;
    dpd_ctx *c = new dpd_ctx();
    int r = create_common(box, rc, a, gamma, kT, power, dt, seed, rank, grid, out, c);
#ifdef DPD_HAVE_NCCL
    if (r == DPD_OK && world > 1) {
        ncclUniqueId u;
        memcpy(&u, nccl_id, 128);
        ncclResult_t nr = ncclCommInitRank(&c->nccl, world, u, rank);
        if (nr != ncclSuccess) r = fail(c, DPD_ERR_COMM, "ncclCommInitRank: %s", ncclGetErrorString(nr));
    }
#else
    if (r == DPD_OK && world > 1) r = fail(c, DPD_ERR_COMM, "libdpd was built without NCCL");
#endif
    if (r != DPD_OK) {
        fprintf(stderr, "dpd_create_dist: %s\n", c->last_error.c_str());
        *out = nullptr;
        dpd_destroy(c);
    }
    return r;
}

int dpd_create_loopback(const double box[3], double rc, double a, double gamma, double kT, double power, double dt,
                        uint64_t seed, const int32_t split[3], const uint8_t nccl_id[128], dpd_ctx **out)
{
    if (!out || !box || !split || !nccl_id) return DPD_ERR_ARG;
    *out = nullptr;
    if (!(split[0] || split[1] || split[2])) return DPD_ERR_ARG;
    dpd_ctx *c = new dpd_ctx();
    const int32_t grid[3] = {1, 1, 1};
    int r = create_common(box, rc, a, gamma, kT, power, dt, seed, 0, grid, out, c, split);
#ifdef DPD_HAVE_NCCL
    if (r == DPD_OK) {
        ncclUniqueId u;
        memcpy(&u, nccl_id, 128);
        ncclResult_t nr = ncclCommInitRank(&c->nccl, 1, u, 0);
        if (nr != ncclSuccess) r = fail(c, DPD_ERR_COMM, "ncclCommInitRank: %s", ncclGetErrorString(nr));
    }
#else
    if (r == DPD_OK) r = fail(c, DPD_ERR_COMM, "libdpd was built without NCCL");
#endif
    if (r != DPD_OK) {
        fprintf(stderr, "dpd_create_loopback: %s\n", c->last_error.c_str());
        *out = nullptr;
        dpd_destroy(c);
    }
    return r;
}

int dpd_create_group(const double box[3], double rc, double a, double gamma, double kT, double power, double dt,
                     uint64_t seed, const int32_t grid[3], dpd_ctx **out)
{
    if (!out || !box || !grid) return DPD_ERR_ARG;
    const int world = grid[0] * grid[1] * grid[2];
    if (world < 1 || world > 64) return DPD_ERR_ARG;
    dpd_ctx **members = new dpd_ctx *[world]();
    cudaStream_t shared = nullptr;
    for (int r = 0; r < world; ++r) {
        dpd_ctx *c = new dpd_ctx();
        dpd_ctx *o = nullptr;
        int rc_ = create_common(box, rc, a, gamma, kT, power, dt, seed, r, grid, &o, c);
        if (rc_ == DPD_OK && r == 0) {
            shared = c->stream;
            c->own_stream = false; // owned by the group (freed with its last member)
        }
        if (rc_ == DPD_OK && r > 0) {
            // all members run on member 0's stream so the phases order themselves
            cudaStreamDestroy(c->stream);
            c->stream = shared;
            c->own_stream = false;
        }
        if (rc_ != DPD_OK) {
            fprintf(stderr, "dpd_create_group: %s\n", c->last_error.c_str());
            dpd_destroy(c);
            for (int k = 0; k < r; ++k) {
                members[k]->group = nullptr;
                dpd_destroy(members[k]);
            }
            delete[] members;
            return rc_;
        }
        members[r] = c;
    }
    for (int r = 0; r < world; ++r) {
        members[r]->group = members;
        members[r]->group_n = world;
        out[r] = members[r];
    }
    return DPD_OK;
}

int dpd_group_step(dpd_ctx **ctxs, int nctx, int64_t nsteps)
{
    if (!ctxs || nctx < 1 || nsteps < 0) return DPD_ERR_ARG;
    dpd_ctx **g = ctxs[0]->group;
    if (!g || ctxs[0]->group_n != nctx) return fail(ctxs[0], DPD_ERR_ARG, "not the full group of a dpd_create_group");
    for (int r = 0; r < nctx; ++r)
        if (ctxs[r] != g[r]) return fail(ctxs[0], DPD_ERR_ARG, "contexts must be passed in rank order");
    bool prime = false;
    for (int r = 0; r < nctx; ++r) prime |= g[r]->need_prime;
    if (prime) TRY(group_prime(g, nctx));
    for (int64_t it = 0; it < nsteps; ++it) TRY(group_step(g, nctx));
    for (int r = 0; r < nctx; ++r) TRY(sync_check(g[r]));
    return DPD_OK;
}

int dpd_get_particles_ex(dpd_ctx *c, int64_t cap, float *pos, float *vel, int32_t *ids, int64_t *n)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n) *n = c->n;
    if (cap < c->n) return fail(c, DPD_ERR_ARG, "cap %lld < count %lld", (long long)cap, (long long)c->n);
    TRY(gather(c, pos, vel, nullptr, 0));
    return copy_ids(c, ids);
}

static int species_out(dpd_ctx *c, int32_t *species, int by_id)
{
    if (!species || c->n == 0) return DPD_OK;
    CUDA_TRY(c, c->stage.reserve((size_t)c->n));
    int32_t *d = reinterpret_cast<int32_t *>(c->stage.p);
    const int b = c->cur;
    TRY(launch(c, KID_GATHER, [&] {
        k_species_out<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->pos[b].p, c->vel[b].p, (int)c->n, d, by_id);
    }));
    CUDA_TRY(c, cudaMemcpyAsync(species, d, sizeof(int32_t) * c->n, cudaMemcpyDefault, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return DPD_OK;
}

int dpd_get_species(dpd_ctx *c, int64_t n, int32_t *species)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n != c->n) return fail(c, DPD_ERR_ARG, "n = %lld but the context holds %lld", (long long)n, (long long)c->n);
    if (!c->dense_ids) return fail(c, DPD_ERR_ARG, "ids are not dense 0..n-1; use dpd_get_species_ex");
    return species_out(c, species, 1);
}

int dpd_get_species_ex(dpd_ctx *c, int64_t cap, int32_t *species, int32_t *ids, int64_t *n)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n) *n = c->n;
    if (cap < c->n) return fail(c, DPD_ERR_ARG, "cap %lld < count %lld", (long long)cap, (long long)c->n);
    TRY(species_out(c, species, 0));
    return copy_ids(c, ids);
}

int dpd_get_forces_ex(dpd_ctx *c, int64_t cap, float *f, int32_t *ids, int64_t *n)
{
    if (!c) return DPD_ERR_ARG;
    TRY(sync_check(c));
    if (n) *n = c->n;
    if (cap < c->n) return fail(c, DPD_ERR_ARG, "cap %lld < count %lld", (long long)cap, (long long)c->n);
    TRY(gather(c, nullptr, nullptr, f, 0));
    return copy_ids(c, ids);
}

// ---- NEXT-4: asynchronous dumps, step schedule, task graph and I/O queue (host) ----------
// Device / pinned resources of a dump state (its writer already closed).
static void dump_free(DumpState *d)
{
    for (auto &sl : d->slots) {
        if (sl.host) cudaFreeHost(sl.host);
        if (sl.copied) cudaEventDestroy(sl.copied);
    }
    if (d->staged_free) cudaEventDestroy(d->staged_free);
    if (d->dev) cudaFree(d->dev);
    delete d->q;
    delete d;
}

static int dump_setup(dpd_ctx *c, DumpState *d)
{
    for (auto &sl : d->slots) CUDA_TRY(c, cudaEventCreateWithFlags(&sl.copied, cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventCreateWithFlags(&d->staged_free, cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventRecord(d->staged_free, c->stream));
    if (!c->copy_stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    if (c->n_cap > 0) {
        // staging block and pinned slots for the current capacity now, not inside the first
        // dumping step (pinned allocations take tens of ms); dump_snapshot re-sizes on growth
        d->cap = c->n_cap;
        CUDA_TRY(c, cudaMalloc(&d->dev, dump_bytes(d->cap)));
        for (auto &sl : d->slots) CUDA_TRY(c, cudaMallocHost(&sl.host, dump_bytes(d->cap)));
    }
    return DPD_OK;
}

int dpd_dump_open(dpd_ctx *c, const char *path_prefix, int queue_depth)
{
    if (!c || !path_prefix) return DPD_ERR_ARG;
    if (queue_depth < 0 || queue_depth > 64) return fail(c, DPD_ERR_ARG, "queue_depth must be in [0, 64]");
    if (c->dump) return fail(c, DPD_ERR_ARG, "dumps already open; dpd_dump_close first");
    auto *d = new DumpState();
    d->prefix = path_prefix;
    d->depth = queue_depth;
    cudaGetDevice(&d->device);
    d->slots.resize(queue_depth + 1);
    const int rc = dump_setup(c, d);
    if (rc != DPD_OK) {
        dump_free(d); // nothing was queued: no writer yet
        return rc;
    }
    d->q = new dpd::IoQueue(queue_depth);
    c->dump = d;
    return DPD_OK;
}

int dpd_dump_every(dpd_ctx *c, int64_t every)
{
    if (!c) return DPD_ERR_ARG;
    if (!c->dump) return fail(c, DPD_ERR_ARG, "dpd_dump_open first");
    if (every < 0) return fail(c, DPD_ERR_ARG, "every must be >= 0");
    if (c->group) return fail(c, DPD_ERR_ARG, "dumps are per NCCL / single context");
    c->dump->every = every;
    return DPD_OK;
}

int dpd_dump_now(dpd_ctx *c)
{
    if (!c) return DPD_ERR_ARG;
    if (!c->dump) return fail(c, DPD_ERR_ARG, "dpd_dump_open first");
    TRY(dump_snapshot(c, c->stream));
    CUDA_TRY(c, cudaEventRecord(c->dump->staged_free, c->stream)); // orders the copy-out after the snapshot
    CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->dump->staged_free, 0));
    return dump_copyout(c, c->copy_stream);
}

int dpd_dump_close(dpd_ctx *c, int64_t *written)
{
    if (!c) return DPD_ERR_ARG;
    DumpState *d = c->dump;
    if (!d) return fail(c, DPD_ERR_ARG, "dumps are not open");
    std::string err;
    const int rc = d->q->close(&err);
    if (written) *written = d->q->completed();
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    dump_free(d);
    c->dump = nullptr;
    delete c->step_graph[1]; // the snapshot tasks refer to the closed state
    c->step_graph[1] = nullptr;
    if (rc != 0) return fail(c, DPD_ERR_IO, "dump: %s", err.c_str());
    return DPD_OK;
}

int dpd_step_schedule(dpd_ctx *c, int with_dump, char *buf, int64_t cap)
{
    if (!c || !buf || cap <= 0) return DPD_ERR_ARG;
    dpd::TaskGraph *g = build_step_graph(c, with_dump != 0);
    if (!g) return fail(c, DPD_ERR_CONFIG, "step task graph has a cycle");
    std::string out;
    for (int u : g->order) {
        const auto &t = g->tasks[u];
        out += std::to_string(t.slot) + " " + t.name;
        for (size_t k = 0; k < t.pred.size(); ++k) out += (k ? "," : " <- ") + g->tasks[t.pred[k]].name;
        out += "\n";
    }
    delete g;
    if ((int64_t)out.size() + 1 > cap) return fail(c, DPD_ERR_ARG, "buffer too small (%zu bytes needed)", out.size() + 1);
    memcpy(buf, out.c_str(), out.size() + 1);
    return DPD_OK;
}

} // extern "C"

struct dpd_taskgraph {
    dpd::TaskGraph g;
};

struct dpd_ioq {
    dpd::IoQueue *q = nullptr;
    std::string last_error;
};

extern "C" {

int dpd_tg_create(dpd_taskgraph **out)
{
    if (!out) return DPD_ERR_ARG;
    *out = new dpd_taskgraph();
    return DPD_OK;
}

int dpd_tg_add(dpd_taskgraph *g, const char *name, int slot, int32_t *id)
{
    if (!g || !name || !id || slot < 0) return DPD_ERR_ARG;
    *id = g->g.add(name, slot);
    return DPD_OK;
}

int dpd_tg_edge(dpd_taskgraph *g, int32_t before, int32_t after)
{
    if (!g) return DPD_ERR_ARG;
    return g->g.edge(before, after) == 0 ? DPD_OK : DPD_ERR_ARG;
}

int dpd_tg_order(dpd_taskgraph *g, int64_t cap, int32_t *order, int64_t *n)
{
    if (!g || !n) return DPD_ERR_ARG;
    if (g->g.build() != 0) {
        *n = 0;
        return DPD_ERR_CONFIG;
    }
    *n = (int64_t)g->g.order.size();
    if (cap < *n || (*n > 0 && !order)) return DPD_ERR_ARG;
    for (int64_t k = 0; k < *n; ++k) order[k] = g->g.order[k];
    return DPD_OK;
}

void dpd_tg_destroy(dpd_taskgraph *g) { delete g; }

int dpd_ioq_create(int depth, dpd_ioq **out)
{
    if (!out || depth < 0 || depth > 64) return DPD_ERR_ARG;
    *out = new dpd_ioq();
    (*out)->q = new dpd::IoQueue(depth);
    return DPD_OK;
}

int dpd_ioq_write(dpd_ioq *q, const char *path, const void *data, int64_t bytes, int64_t delay_us)
{
    if (!q || !path || bytes < 0 || (bytes > 0 && !data) || delay_us < 0) return DPD_ERR_ARG;
    auto buf = std::make_shared<std::vector<char>>((const char *)data, (const char *)data + bytes);
    const std::string p = path;
    auto job = [buf, p, delay_us](std::string &err) -> int {
        if (delay_us > 0) std::this_thread::sleep_for(std::chrono::microseconds(delay_us));
        FILE *f = fopen(p.c_str(), "wb");
        if (!f) {
            err = "cannot open " + p;
            return -1;
        }
        const bool ok = fwrite(buf->data(), 1, buf->size(), f) == buf->size();
        if (fclose(f) != 0 || !ok) {
            err = "short write to " + p;
            return -1;
        }
        return 0;
    };
    std::string err;
    if (q->q->submit(job, err) != 0) {
        q->last_error = err;
        return DPD_ERR_IO;
    }
    return DPD_OK;
}

int dpd_ioq_pending(dpd_ioq *q, int64_t *n)
{
    if (!q || !n) return DPD_ERR_ARG;
    *n = q->q->pending();
    return DPD_OK;
}

int dpd_ioq_close(dpd_ioq *q, int64_t *completed)
{
    if (!q) return DPD_ERR_ARG;
    std::string err;
    const int rc = q->q->close(&err);
    if (completed) *completed = q->q->completed();
    delete q->q;
    delete q;
    return rc == 0 ? DPD_OK : DPD_ERR_IO;
}

const char *dpd_ioq_last_error(const dpd_ioq *q) { return q ? q->last_error.c_str() : "null queue"; }

} // extern "C"

