// dpd_dist.cuh -- kernels of the 3D domain decomposition (
// equal rectangular subdomains, halo exchange overlapped with the local
// forces, forces due to the received particles, redistribution of leaving particles).
//
// Frames: each rank works in local coordinates x - origin in [0, L_sub).  A particle sent
// in direction D (migrant or ghost) is shifted by -D L_sub, i.e. written directly in the
// receiver's frame.  Split dimensions carry a one-cell halo ring in the extended cell grid
// (index 0 and n + 1); ghosts are binned there, local particles never are.
#pragma once

#include "dpd_kernels.cuh"

namespace dpd {

__global__ void k_zero_headers(Msgs m)
{
    const int d = threadIdx.x;
    if (d < 27 && m.cap[d] > 0) *msg_count(m, d) = 0;
}

__device__ __forceinline__ int msg_received(const Msgs &m, int d, int *err)
{
    const int c = *msg_count(m, d);
    if (c > m.cap[d]) {
        raise_err(err, ERR_CAPACITY, c);
        return m.cap[d];
    }
    return c;
}

// Cell coordinate of a received ghost along one dimension: halo layers map to -1 / n in
// split dimensions (x in [-h, 0) / [L, L + h)), interior otherwise (C-8 formula).
__device__ __forceinline__ int ghost_coord(float x, float inv_h, int n, int split)
{
    if (!split) return cell_coord(x, inv_h, n);
    const int q = (int)floorf(__fmul_rn(x, inv_h));
    return min(max(q, -1), n);
}

__device__ __forceinline__ int ghost_cell(const Geom &g, float x, float y, float z)
{
    const int ix = ghost_coord(x, g.inv_h[0], g.n[0], g.split[0]) + g.off[0];
    const int iy = ghost_coord(y, g.inv_h[1], g.n[1], g.split[1]) + g.off[1];
    const int iz = ghost_coord(z, g.inv_h[2], g.n[2], g.split[2]) + g.off[2];
    return ix + g.ext[0] * (iy + g.ext[1] * iz);
}

// ---- row a10: received migrants -> local cell histogram ---------------------------------
// grid = (ceil(maxcap / 256), 27): block row d handles direction d's message.
__global__ void __launch_bounds__(256) k_bin_recv(Msgs rec, Geom g, int maxcap, int *__restrict__ count,
                                                  int *__restrict__ rank_in, int *err)
{
    const int d = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (rec.cap[d] == 0 || blockIdx.x * blockDim.x >= rec.cap[d]) return; // block-uniform
    const int cnt = msg_received(rec, d, err);
    int c = -1;
    if (k < cnt) {
        const float4 p = msg_data(rec, d)[2 * k];
        const float3 x = make_float3(p.x, p.y, p.z);
        if (!in_local_box(g, x)) raise_err(err, ERR_RANGE, __float_as_int(p.w));
        else c = cell_index(g, p.x, p.y, p.z);
    }
    const int r = warp_rank_in_cell(count, c);
    if (k < cnt) rank_in[d * maxcap + k] = (c >= 0) ? r : -1;
}

__global__ void __launch_bounds__(256) k_scatter_recv(Msgs rec, Geom g, int maxcap, const int *__restrict__ start,
                                                      const int *__restrict__ rank_in, float4 *__restrict__ pos_o,
                                                      float4 *__restrict__ vel_o, float4 *__restrict__ frc_o)
{
    const int d = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (rec.cap[d] == 0) return;
    const int cnt = min(*msg_count(rec, d), rec.cap[d]);
    if (k >= cnt) return;
    const int r = rank_in[d * maxcap + k];
    if (r < 0) return;
    const float4 p = msg_data(rec, d)[2 * k], v = msg_data(rec, d)[2 * k + 1];
    const int dst = start[cell_index(g, p.x, p.y, p.z)] + r;
    pos_o[dst] = p;
    vel_o[dst] = v;
    frc_o[dst] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
}

// ---- row a7: ghost identify + pack ------------------------------------------------------
// A particle in the first (last) interior cell layer of a split dimension goes to the
// neighbour below (above); edge and corner cells go to every combination (up to 7 messages).
__global__ void __launch_bounds__(256) k_ghost_pack(const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                                                    const int *__restrict__ n_ptr, Geom g, Msgs gs, int *err)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = *n_ptr;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f), v = p;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    if (i < n) {
        p = pos[i];
        v = vel[i];
        const float xs[3] = {p.x, p.y, p.z};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (!g.split[k]) continue;
            const int ic = cell_coord(xs[k], g.inv_h[k], g.n[k]);
            lo[k] = ic == 0;
            hi[k] = ic == g.n[k] - 1;
        }
    }
    const int lane = threadIdx.x & 31;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int d = dir_index(dx, dy, dz);
                if (d == 13 || gs.cap[d] == 0) continue; // uniform
                const bool want = i < n && (dx == 0 || (dx < 0 ? lo[0] : hi[0])) &&
                                  (dy == 0 || (dy < 0 ? lo[1] : hi[1])) && (dz == 0 || (dz < 0 ? lo[2] : hi[2]));
                const unsigned m = __ballot_sync(0xffffffffu, want);
                if (!m) continue;
                int base = 0;
                const int leader = __ffs(m) - 1;
                if (lane == leader) base = atomicAdd(msg_count(gs, d), __popc(m));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (want) {
                    const int slot = base + __popc(m & lanemask_lt());
                    if (slot < gs.cap[d]) {
                        float4 *q = msg_data(gs, d) + 2 * slot;
                        q[0] = make_float4(p.x - dx * g.L[0], p.y - dy * g.L[1], p.z - dz * g.L[2], p.w);
                        q[1] = v;
                    } else {
                        raise_err(err, ERR_CAPACITY, __float_as_int(p.w));
                    }
                }
            }
}

// ---- rows a8/a9: received ghosts -> halo cells (count, scan, scatter) ------------------
__global__ void __launch_bounds__(256) k_ghost_bin(Msgs rec, Geom g, int maxcap, int *__restrict__ gcount,
                                                   int *__restrict__ grank, int *err)
{
    const int d = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (rec.cap[d] == 0 || blockIdx.x * blockDim.x >= rec.cap[d]) return;
    const int cnt = msg_received(rec, d, err);
    int c = -1;
    if (k < cnt) {
        const float4 p = msg_data(rec, d)[2 * k];
        c = ghost_cell(g, p.x, p.y, p.z);
    }
    const int r = warp_rank_in_cell(gcount, c);
    if (k < cnt) grank[d * maxcap + k] = r;
}

__global__ void __launch_bounds__(256) k_ghost_scatter(Msgs rec, Geom g, int maxcap, const int *__restrict__ gstart,
                                                       const int *__restrict__ grank, float4 *__restrict__ gpos,
                                                       float4 *__restrict__ gvel)
{
    const int d = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (rec.cap[d] == 0) return;
    const int cnt = min(*msg_count(rec, d), rec.cap[d]);
    if (k >= cnt) return;
    const float4 p = msg_data(rec, d)[2 * k];
    const int dst = gstart[ghost_cell(g, p.x, p.y, p.z)] + grank[d * maxcap + k];
    gpos[dst] = p;
    gvel[dst] = msg_data(rec, d)[2 * k + 1];
}

// ---- row a7 (cell-driven): one thread per interior cell; only the cells of the boundary
// layers of split dimensions do work.  A boundary cell's particles (contiguous in the sorted
// arrays) are written to every direction its position calls for (face / edge / corner) with
// one warp-aggregated slot reservation per direction, and appended to the boundary list
// blist[1..blist[0]] that drives the halo force (row a9).  Same messages as k_ghost_pack
// (a multiset: the order inside a message is irrelevant to the receiver's binning), ~5 % of
// the work at 128^3 per rank.
__global__ void __launch_bounds__(256) k_ghost_pack_cells(const float4 *__restrict__ pos,
                                                          const float4 *__restrict__ vel,
                                                          const int *__restrict__ start, Geom g, Msgs gs,
                                                          int *__restrict__ blist, int *err)
{
    const int ncell = g.n[0] * g.n[1] * g.n[2];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    unsigned dmask = 0;
    int s0 = 0, cnt = 0;
    bool border = false;
    if (t < ncell) {
        const int ic[3] = {t % g.n[0], (t / g.n[0]) % g.n[1], t / (g.n[0] * g.n[1])};
        int lo[3], hi[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            lo[k] = g.split[k] && ic[k] == 0;
            hi[k] = g.split[k] && ic[k] == g.n[k] - 1;
            border = border || lo[k] || hi[k];
        }
        if (border) {
            const int gc = (ic[0] + g.off[0]) + g.ext[0] * ((ic[1] + g.off[1]) + g.ext[1] * (ic[2] + g.off[2]));
            s0 = start[gc];
            cnt = start[gc + 1] - s0;
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int d = dir_index(dx, dy, dz);
                        if (d == 13 || gs.cap[d] == 0) continue;
                        if ((dx == 0 || (dx < 0 ? lo[0] : hi[0])) && (dy == 0 || (dy < 0 ? lo[1] : hi[1])) &&
                            (dz == 0 || (dz < 0 ? lo[2] : hi[2])))
                            dmask |= 1u << d;
                    }
        }
    }
    // boundary list
    {
        const int v = border ? cnt : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot) {
            int base = 0;
            if (lane == 31) base = atomicAdd(&blist[0], tot);
            base = __shfl_sync(0xffffffffu, base, 31);
            for (int k = 0; k < v; ++k) blist[1 + base + incl - v + k] = s0 + k;
        }
    }
    // ghost messages, one direction at a time over the directions any lane needs
    unsigned wm = __reduce_or_sync(0xffffffffu, cnt ? dmask : 0u);
    while (wm) {
        const int d = __ffs(wm) - 1;
        wm &= wm - 1;
        const int v = ((dmask >> d) & 1u) ? cnt : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int base = 0;
        if (lane == 31) base = atomicAdd(msg_count(gs, d), tot);
        base = __shfl_sync(0xffffffffu, base, 31);
        if (v) {
            const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
            const float shx = dx * g.L[0], shy = dy * g.L[1], shz = dz * g.L[2];
            float4 *q = msg_data(gs, d);
            for (int k = 0; k < v; ++k) {
                const int slot = base + incl - v + k;
                const float4 p = pos[s0 + k];
                if (slot < gs.cap[d]) {
                    q[2 * slot] = make_float4(p.x - shx, p.y - shy, p.z - shz, p.w);
                    q[2 * slot + 1] = vel[s0 + k];
                } else {
                    raise_err(err, ERR_CAPACITY, __float_as_int(p.w));
                }
            }
        }
    }
}

// ---- row a9: one-sided local-ghost forces ------------------------------------------------
// Local particle i in a boundary cell sums f_ij over the ghosts j of its halo neighbour
// cells; the peer rank computes the exact negation for its own copy (global ids key the
// RNG, C-19).  Runs after the interior pass on the same stream: plain read-modify-write.
// Halo neighbour cell d (0..26 = dir_index) of interior cell ci: extended-grid index and the
// periodic shift of its ghosts; -1 if the cell is not in the halo ring.
__device__ __forceinline__ int halo_cell(const Geom &g, const int ci[3], int d, float sh[3])
{
    const int dd[3] = {d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1};
    int e[3];
    bool halo = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        int jc = ci[k] + dd[k];
        sh[k] = 0.0f;
        if (g.split[k]) {
            halo |= (jc < 0 || jc >= g.n[k]);
            e[k] = jc + 1;
        } else {
            if (jc < 0) {
                jc += g.n[k];
                sh[k] = -g.L[k];
            } else if (jc >= g.n[k]) {
                jc -= g.n[k];
                sh[k] = g.L[k];
            }
            e[k] = jc;
        }
    }
    return halo ? e[0] + g.ext[0] * (e[1] + g.ext[1] * e[2]) : -1;
}

// One local-ghost pair (one-sided: the force on local i only).
template <int KMODE>
__device__ __forceinline__ void halo_pair(const float4 &pi, const float4 &vi, const float4 &pj, const float4 &vj,
                                          const float sh[3], const PairP &pp, uint32_t ks, float &Fx, float &Fy,
                                          float &Fz)
{
    const float rx = pi.x - (pj.x + sh[0]), ry = pi.y - (pj.y + sh[1]), rz = pi.z - (pj.z + sh[2]);
    const float r2 = rx * rx + ry * ry + rz * rz;
    const float dv = rx * (vi.x - vj.x) + ry * (vi.y - vj.y) + rz * (vi.z - vj.z);
    const float s = pair_scalar<KMODE>(pp, r2, dv, (uint32_t)__float_as_int(pi.w), (uint32_t)__float_as_int(pj.w), ks,
                                       vi.w, vj.w);
    Fx += s * rx;
    Fy += s * ry;
    Fz += s * rz;
}

constexpr int kHaloThreads = 128;
constexpr int kHaloCap = 24; // hits kept per boundary particle before evaluating in place (mean ~6-12)

// Halo forces of local particle i: all ghosts j of its halo neighbour cells (one-sided).
// Two passes: the distance sweep collects the hits (ghost index | neighbour code << 27) in
// the thread's shared-memory list, then the pair bodies run back to back -- the heavy pair
// body is not executed for every candidate a neighbour lane hits.
template <int KMODE>
__device__ __forceinline__ void halo_particle(int i, const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                                              float4 *__restrict__ frc, const float4 *__restrict__ gpos,
                                              const float4 *__restrict__ gvel, const int *__restrict__ gstart,
                                              const Geom &g, const PairP &pp, uint32_t ks, unsigned *hl)
{
    const float4 pi = pos[i];
    const int ci[3] = {cell_coord(pi.x, g.inv_h[0], g.n[0]), cell_coord(pi.y, g.inv_h[1], g.n[1]),
                       cell_coord(pi.z, g.inv_h[2], g.n[2])};
    const float4 vi = vel[i];
    float Fx = 0.f, Fy = 0.f, Fz = 0.f;
    int nh = 0;
    for (int d = 0; d < 27; ++d) {
        float sh[3];
        const int c = halo_cell(g, ci, d, sh);
        if (c < 0) continue;
        for (int j = gstart[c]; j < gstart[c + 1]; ++j) {
            const float4 pj = gpos[j];
            const float rx = pi.x - (pj.x + sh[0]), ry = pi.y - (pj.y + sh[1]), rz = pi.z - (pj.z + sh[2]);
            const float r2 = rx * rx + ry * ry + rz * rz;
            if (r2 < pp.rc2 && r2 > 0.0f) {
                if (nh < kHaloCap) {
                    hl[nh * kHaloThreads] = (unsigned)j | ((unsigned)d << 27);
                    ++nh;
                } else {
                    halo_pair<KMODE>(pi, vi, pj, gvel[j], sh, pp, ks, Fx, Fy, Fz);
                }
            }
        }
    }
    for (int k = 0; k < nh; ++k) {
        const unsigned e = hl[k * kHaloThreads];
        const int j = (int)(e & 0x07FFFFFFu);
        float sh[3];
        halo_cell(g, ci, (int)(e >> 27), sh);
        halo_pair<KMODE>(pi, vi, gpos[j], gvel[j], sh, pp, ks, Fx, Fy, Fz);
    }
    float4 f = frc[i];
    f.x += Fx;
    f.y += Fy;
    f.z += Fz;
    frc[i] = f;
}

template <int KMODE>
__global__ void __launch_bounds__(kHaloThreads) k_force_halo(const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                                                    float4 *__restrict__ frc, const int *__restrict__ n_ptr,
                                                    const float4 *__restrict__ gpos, const float4 *__restrict__ gvel,
                                                    const int *__restrict__ gstart, Geom g, PairP pp,
                                                    uint32_t s_lo, uint32_t s_hi)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= *n_ptr) return;
    const float4 pi = pos[i];
    const int ci[3] = {cell_coord(pi.x, g.inv_h[0], g.n[0]), cell_coord(pi.y, g.inv_h[1], g.n[1]),
                       cell_coord(pi.z, g.inv_h[2], g.n[2])};
    bool boundary = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) boundary |= g.split[k] && (ci[k] == 0 || ci[k] == g.n[k] - 1);
    __shared__ unsigned hl[kHaloThreads * kHaloCap];
    if (!boundary) return;
    halo_particle<KMODE>(i, pos, vel, frc, gpos, gvel, gstart, g, pp, step_key(s_lo, s_hi, pp.seed_fold),
                         hl + threadIdx.x);
}

// The same over the boundary list of k_ghost_pack_cells (blist[0] entries): every thread
// busy, no pass over the interior particles.
template <int KMODE>
__global__ void __launch_bounds__(kHaloThreads) k_force_halo_list(const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                                                         float4 *__restrict__ frc, const int *__restrict__ blist,
                                                         const float4 *__restrict__ gpos,
                                                         const float4 *__restrict__ gvel,
                                                         const int *__restrict__ gstart, Geom g, PairP pp,
                                                         uint32_t s_lo, uint32_t s_hi)
{
    __shared__ unsigned hl[kHaloThreads * kHaloCap];
    const int nb = blist[0];
    const uint32_t ks = step_key(s_lo, s_hi, pp.seed_fold);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += gridDim.x * blockDim.x)
        halo_particle<KMODE>(blist[1 + t], pos, vel, frc, gpos, gvel, gstart, g, pp, ks, hl + threadIdx.x);
}

} // namespace dpd
