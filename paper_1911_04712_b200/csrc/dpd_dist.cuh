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

// In-process group transport: every (sender, direction) message of one exchange in one
// launch (blockIdx.y = job).  Copies the int4 count header and the min(count, cap) particles
// actually packed (two int4 each) -- or, with full set, the whole capacity-padded slot, the
// bytes the NCCL transport sends; an overflowing count is copied as is so the receiver
// raises ERR_CAPACITY (msg_received).
constexpr int kCopyJobs = 512;
struct CopyJob {
    const int4 *src;
    int4 *dst;
    int cap;
    int full;
};
struct CopyJobs {
    CopyJob j[kCopyJobs];
};

__global__ void __launch_bounds__(256) k_group_copy(const __grid_constant__ CopyJobs jobs)
{
    const CopyJob &J = jobs.j[blockIdx.y];
    const int cnt = J.full ? J.cap : min(max(J.src[0].x, 0), J.cap);
    const int total = 1 + 2 * cnt;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) J.dst[k] = J.src[k];
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

// Cell coordinate of a received ghost along one dimension: in split dimensions a ghost
// below 0 / at or above L lies in the halo layer -1 / n (decided by the sign test, not by
// floor(x n / L), whose fp32 product can round L + tiny into interior cell n - 1); interior
// positions use the C-8 formula.
__device__ __forceinline__ int ghost_coord(float x, float inv_h, int n, int split, float L)
{
    if (split) {
        if (x < 0.0f) return -1;
        if (x >= L) return n;
    }
    return cell_coord(x, inv_h, n);
}

__device__ __forceinline__ int ghost_cell(const Geom &g, float x, float y, float z)
{
    const int ix = ghost_coord(x, g.inv_h[0], g.n[0], g.split[0], g.L[0]) + g.off[0];
    const int iy = ghost_coord(y, g.inv_h[1], g.n[1], g.split[1], g.L[1]) + g.off[1];
    const int iz = ghost_coord(z, g.inv_h[2], g.n[2], g.split[2], g.L[2]) + g.off[2];
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
                                                      float4 *__restrict__ vel_o, int cap, int *err)
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
    if (dst >= cap) { // more particles than the member's arrays hold: DPD_ERR_CAPACITY
        raise_err(err, ERR_CAPACITY, __float_as_int(p.w));
        return;
    }
    pos_o[dst] = p;
    vel_o[dst] = v; // the force slot is already zero (k_force_tile zeroes the buffer a step ahead)
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

// ---- row a7: ghost identify + pack, one thread per interior cell (3D grid) -----------------
// Only the cells of the boundary layers of split dimensions do work (~5 % at 128^3 per
// rank).  A boundary cell's particles (contiguous in the sorted arrays) are written to every
// direction its position calls for (face / edge / corner: a corner cell's particles go to 7
// messages), shifted by -D L_sub into the receiver's frame, with one warp-aggregated slot
// reservation per direction; the cell itself is appended to the boundary-cell list
// blist[1..blist[0]] (packed interior coordinates) that drives the halo force (row a9).  The order inside a message is
// irrelevant: the receiver bins the ghosts into its halo ring.
constexpr int kGpThreads = 128; // 1D grid over the boundary cells (GpPlan)
#ifndef GP_SUB
#define GP_SUB 1
#endif
constexpr int kGpSub = GP_SUB;  // threads per boundary cell (a power of two <= 32); 2x2x2 group
                                // overhead at 128^3 per subdomain: 1 -> 6.9 %, 4 -> 7.5 %, 8 -> 8.7 %

// The boundary cells of a subdomain (a split dimension's first or last interior layer) as
// disjoint boxes, one per split dimension k: coordinate k on {0, n_k - 1}, the split
// dimensions before k restricted to their inner range [1, n - 2], the others full.  A
// thread's linear index b walks the boxes in order, x fastest, so every lane of a warp has a
// boundary cell (the round-1/2 kernel ran one thread per interior cell and left ~half of
// the lanes of the x-face warps idle).
struct GpPlan {
    int nbox;        // number of boxes (split dimensions)
    int end[3];      // exclusive prefix end of each box's cell count
    int lo[3][3];    // per box: lower coordinate per dimension
    int ext[3][3];   // per box: extent per dimension (dimension k of box k: 2, stride n_k - 1)
    int dimk[3];     // per box: its split dimension
};

__global__ void __launch_bounds__(kGpThreads) k_ghost_pack_cells(const float4 *__restrict__ pos,
                                                                 const float4 *__restrict__ vel,
                                                                 const int *__restrict__ start, Geom g, Msgs gs,
                                                                 int *__restrict__ blist, int *err, GpPlan pl)
{
    const int lane = threadIdx.x & 31;
    // kGpSub consecutive lanes share a boundary cell and split its copies (more loads in
    // flight per cell); the cell's lane 0 (sub == 0) does the list entry and reservations
    const int sub = lane & (kGpSub - 1);
    const int b = (blockIdx.x * kGpThreads + threadIdx.x) / kGpSub;
    int ic[3] = {g.n[0], 0, 0}; // past the grid: no work
    if (b < pl.end[pl.nbox - 1]) {
        int x = 0;
        while (x + 1 < pl.nbox && b >= pl.end[x]) ++x;
        int r = b - (x > 0 ? pl.end[x - 1] : 0);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int e = pl.ext[x][k];
            const int v = r % e;
            r /= e;
            ic[k] = pl.lo[x][k] + (k == pl.dimk[x] ? v * (g.n[k] - 1) : v);
        }
    }
    unsigned dmask = 0;
    int s0 = 0, cnt = 0, gc = 0;
    bool border = false;
    if (ic[0] < g.n[0]) {
        int sd[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            sd[k] = !g.split[k] ? 0 : (ic[k] == 0 ? -1 : (ic[k] == g.n[k] - 1 ? 1 : 0));
            border = border || sd[k] != 0;
        }
        if (border) {
            gc = (ic[0] + g.off[0]) + g.ext[0] * ((ic[1] + g.off[1]) + g.ext[1] * (ic[2] + g.off[2]));
            s0 = start[gc];
            cnt = start[gc + 1] - s0;
            // directions: every non-empty combination of this cell's face offsets (a face
            // cell 1, an edge cell 3, a corner cell 7); all of them are used (split) directions
#pragma unroll
            for (int m = 1; m < 8; ++m) {
                const int dx = (m & 1) ? sd[0] : 0, dy = (m & 2) ? sd[1] : 0, dz = (m & 4) ? sd[2] : 0;
                const bool ok = ((m & 1) == 0 || dx) && ((m & 2) == 0 || dy) && ((m & 4) == 0 || dz);
                if (ok) dmask |= 1u << dir_index(dx, dy, dz);
            }
        }
    }
    // boundary-cell list (extended-grid index of every non-empty boundary cell)
    {
        const bool has = border && cnt > 0 && sub == 0;
        const unsigned bm = __ballot_sync(0xffffffffu, has);
        if (bm) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&blist[0], __popc(bm));
            base = __shfl_sync(0xffffffffu, base, 0);
            // packed interior coordinates (10 bits each; setup_geometry keeps n < 1024 in
            // decomposed contexts): the halo kernel needs them and the extended index, and
            // rebuilding the index is cheaper than dividing it back into coordinates
            if (has) blist[1 + base + __popc(bm & lanemask_lt())] = ic[0] | (ic[1] << 10) | (ic[2] << 20);
        }
    }
    // ghost messages, one direction at a time over the directions any lane needs
    unsigned wm = __reduce_or_sync(0xffffffffu, cnt ? dmask : 0u);
    while (wm) {
        const int d = __ffs(wm) - 1;
        wm &= wm - 1;
        const int v = ((dmask >> d) & 1u) ? cnt : 0;
        const int vs = sub == 0 ? v : 0; // each cell counted once
        int incl = vs;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int base = 0;
        if (lane == 31) base = atomicAdd(msg_count(gs, d), tot);
        base = __shfl_sync(0xffffffffu, base, 31);
        const int slot0 = __shfl_sync(0xffffffffu, base + incl - vs, lane & ~(kGpSub - 1));
        if (v) {
            const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
            const float shx = dx * g.L[0], shy = dy * g.L[1], shz = dz * g.L[2];
            float4 *q = msg_data(gs, d);
            const int vfit = max(0, min(v, gs.cap[d] - slot0)); // overflow: counted, not written
            // no branch in the copy loop: the loads of several particles are in flight
#pragma unroll 2
            for (int k = sub; k < vfit; k += kGpSub) {
                const float4 p = pos[s0 + k], u = vel[s0 + k];
                q[2 * (slot0 + k)] = make_float4(p.x - shx, p.y - shy, p.z - shz, p.w);
                q[2 * (slot0 + k) + 1] = u;
            }
            if (vfit < v && sub == 0) raise_err(err, ERR_CAPACITY, __float_as_int(pos[s0 + vfit].w));
        }
    }
}

// ---- row a9: one-sided local-ghost forces ------------------------------------------------
// Local particle i in a boundary cell sums f_ij over the ghosts j of its halo neighbour
// cells; the peer rank computes the exact negation for its own copy (global ids key the
// RNG, C-19).  Runs after the interior pass on the same stream.
//
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

// ---- row a9, warp per boundary cell ------------------------------------------------------
// One warp per boundary cell of the list above.  The ghosts of its halo neighbour cells are
// staged once per chunk of kHcG into the warp's shared buffer -- shifted into the local frame,
// velocity and id alongside -- with coalesced loads whose latencies overlap (round 1 gathered
// them from global memory per candidate chunk and again per evaluated pair: the kernel was
// bound by those load latencies).  Its local particles (<= 32 per pass, in shared memory for
// broadcast reads) are tested against the staged ghosts one ghost per lane, kHcI locals per
// round; in-cutoff combinations are compacted into a per-warp queue and evaluated 32 at a time
// with both sides read from shared memory.  One-sided (C-19): the i-side sums go to
// fixed-point shared accumulators, then once to frc.
constexpr int kHcWarps = 4;
#ifndef HC_I
#define HC_I 4
#endif
constexpr int kHcI = HC_I;   // local particles tested per candidate round (2 / 4 / 8: halo 184 / 177 / 200 us
                             // per 128^3 loopback step)
#ifndef KHC_G
#define KHC_G 128
#endif
constexpr int kHcG = KHC_G; // ghosts staged per chunk (a face cell has ~72, an edge ~120 at rho = 8)

template <int KMODE>
__global__ void __launch_bounds__(32 * kHcWarps, 9) // 56 registers: 36 warps per SM
    k_force_halo_cells(const float4 *__restrict__ pos, const float4 *__restrict__ vel, float4 *__restrict__ frc,
                       const int *__restrict__ bcells, const int *__restrict__ start,
                       const float4 *__restrict__ gpos, const float4 *__restrict__ gvel,
                       const int *__restrict__ gstart, Geom g, PairP pp, float scale, float inv_scale,
                       float mag_lim, uint32_t s_lo, uint32_t s_hi, int *err)
{
    __shared__ unsigned qbuf[kHcWarps][32 + 32 * kHcI]; // < 32 pending + kHcI x 32 new
    __shared__ float4 spi[kHcWarps][32 + kHcI];         // the cell's local positions (broadcast reads);
                                                        // slots >= ni hold a far-away point
    __shared__ float4 svi[kHcWarps][32];                // ... and velocities
    __shared__ float4 sgp[kHcWarps][kHcG];              // staged ghosts: local-frame position, id bits
    __shared__ float4 sgv[kHcWarps][kHcG];              // ... velocity, species
    __shared__ int acc[kHcWarps][3][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned *q = qbuf[warp];
    const uint32_t ks = step_key(s_lo, s_hi, pp.seed_lo, pp.seed_hi);
    const int nbc = bcells[0];
    float amax = 0.0f; // largest pair force magnitude: the fixed-point range check
    for (int w = blockIdx.x * kHcWarps + warp; w < nbc; w += gridDim.x * kHcWarps) {
        const int pc = bcells[1 + w]; // packed interior coordinates (k_ghost_pack_cells)
        const int ci[3] = {pc & 1023, (pc >> 10) & 1023, pc >> 20};
        const int gc = (ci[0] + g.off[0]) + g.ext[0] * ((ci[1] + g.off[1]) + g.ext[1] * (ci[2] + g.off[2]));
        const int s0 = start[gc], ntot = start[gc + 1] - s0;
        // halo neighbour d of this cell on lane d: ghost range and periodic shift
        int ha = 0, hn = 0;
        float hsh[3] = {0.0f, 0.0f, 0.0f};
        if (lane < 27) {
            const int c = halo_cell(g, ci, lane, hsh);
            if (c >= 0) {
                ha = gstart[c];
                hn = gstart[c + 1] - ha;
            }
        }
        // exclusive prefix of the halo cells' ghost counts over lanes 0..26
        int hex = hn;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, hex, o);
            if (lane >= o) hex += y;
        }
        const int G = __shfl_sync(0xffffffffu, hex, 31);
        hex -= hn;
        for (int ib = 0; ib < ntot; ib += 32) {
            const int ni = min(32, ntot - ib);
            float4 pi = make_float4(0.f, 0.f, 0.f, 0.f), vi = pi;
            if (lane < ni) {
                pi = pos[s0 + ib + lane];
                vi = vel[s0 + ib + lane];
            }
            acc[warp][0][lane] = acc[warp][1][lane] = acc[warp][2][lane] = 0;
            // slots past the cell's particles (and the kHcI overhang of the last round) are
            // far away: they fail r^2 < r_c^2, so the candidate test needs no index predicate
            spi[warp][lane] = lane < ni ? pi : make_float4(1.0e18f, 1.0e18f, 1.0e18f, 0.0f);
            if (lane < kHcI) spi[warp][32 + lane] = make_float4(1.0e18f, 1.0e18f, 1.0e18f, 0.0f);
            svi[warp][lane] = vi;
            for (int gb = 0; gb < G; gb += kHcG) {
                const int gn = min(kHcG, G - gb);
                __syncwarp(); // the previous chunk's evaluations are done with the buffer
                // stage ghosts [gb, gb + gn): halo cell of each by a search over the prefix
                for (int k = lane; k < ((gn + 31) & ~31); k += 32) {
                    const int gi = gb + k;
                    int d = 0; // largest halo lane with prefix <= gi (the prefix is non-decreasing)
#pragma unroll
                    for (int stp = 16; stp > 0; stp >>= 1) {
                        const int t = d + stp;
                        const int off_t = __shfl_sync(0xffffffffu, hex, t & 31);
                        if (t < 27 && off_t <= gi) d = t;
                    }
                    const int a = __shfl_sync(0xffffffffu, ha, d), off = __shfl_sync(0xffffffffu, hex, d);
                    const float shx = __shfl_sync(0xffffffffu, hsh[0], d), shy = __shfl_sync(0xffffffffu, hsh[1], d),
                                shz = __shfl_sync(0xffffffffu, hsh[2], d);
                    if (k < gn) {
                        const int jidx = a + gi - off;
                        const float4 pj = gpos[jidx];
                        sgp[warp][k] = make_float4(pj.x + shx, pj.y + shy, pj.z + shz, pj.w);
                        sgv[warp][k] = gvel[jidx];
                    }
                }
                __syncwarp();
                int qn = 0;
                // evaluate queue entries [0, cnt): lane k takes entry k (both sides from shared memory)
                auto evaluate = [&](int cnt) {
                    if (lane < cnt) {
                        const unsigned e = q[lane];
                        const int k = (int)(e & 0xFFFFu), ii = (int)(e >> 16);
                        const float4 pj = sgp[warp][k], vj = sgv[warp][k];
                        const float4 p = spi[warp][ii], u = svi[warp][ii];
                        const float rx = p.x - pj.x, ry = p.y - pj.y, rz = p.z - pj.z;
                        const float r2 = rx * rx + ry * ry + rz * rz;
                        const float dv = rx * (u.x - vj.x) + ry * (u.y - vj.y) + rz * (u.z - vj.z);
                        float mag;
                        const float sc = pair_mag<KMODE>(pp, fmaxf(r2, 1e-30f), dv, (uint32_t)__float_as_int(p.w),
                                                         (uint32_t)__float_as_int(pj.w), ks, __float_as_int(u.w),
                                                         __float_as_int(vj.w), mag);
                        amax = fmaxf(amax, fabsf(mag));
                        atomicAdd(&acc[warp][0][ii], __float_as_int(__fmaf_rn(sc * rx, scale, 12582912.0f)) - 0x4B400000);
                        atomicAdd(&acc[warp][1][ii], __float_as_int(__fmaf_rn(sc * ry, scale, 12582912.0f)) - 0x4B400000);
                        atomicAdd(&acc[warp][2][ii], __float_as_int(__fmaf_rn(sc * rz, scale, 12582912.0f)) - 0x4B400000);
                    }
                };
                // the staged ghosts, 32 per chunk with one ghost per lane, tested against the
                // cell's local particles kHcI at a time (broadcast LDS.128)
                for (int cb = 0; cb < gn; cb += 32) {
                    const int k = cb + lane;
                    float px = 3.0e30f, py = 0.0f, pz = 0.0f; // beyond the chunk: never within r_c
                    if (k < gn) {
                        const float4 pj = sgp[warp][k];
                        px = pj.x;
                        py = pj.y;
                        pz = pj.z;
                    }
                    for (int ii = 0; ii < ni; ii += kHcI) { // kHcI local particles per round
                        unsigned m[kHcI];
                        bool h[kHcI];
#pragma unroll
                        for (int u = 0; u < kHcI; ++u) {
                            const float4 p = spi[warp][ii + u]; // LDS.128 broadcast
                            const float rx = p.x - px, ry = p.y - py, rz = p.z - pz;
                            const float r2 = rx * rx + ry * ry + rz * rz;
                            // one predicate: padded slots are far away, and a coincident pair
                            // (r^2 = 0) evaluates to zero force (clamped r^2, d = 0; C-11)
                            h[u] = r2 < pp.rc2;
                            m[u] = __ballot_sync(0xffffffffu, h[u]);
                        }
                        const unsigned lt = lanemask_lt();
#pragma unroll
                        for (int u = 0; u < kHcI; ++u) {
                            if (h[u]) q[qn + __popc(m[u] & lt)] = (unsigned)k | ((unsigned)(ii + u) << 16);
                            qn += __popc(m[u]);
                        }
                        __syncwarp();
                        while (qn >= 32) {
                            evaluate(32);
                            __syncwarp();
                            for (int t = lane; t < qn - 32; t += 32) q[t] = q[t + 32];
                            qn -= 32;
                            __syncwarp();
                        }
                    }
                }
                if (qn > 0) evaluate(qn);
            }
            __syncwarp();
            if (lane < ni) { // a vector reduction: the interior force kernel may still be adding
                const int ax = acc[warp][0][lane], ay = acc[warp][1][lane], az = acc[warp][2][lane];
                if (ax | ay | az)
                    atomicAdd(&frc[s0 + ib + lane],
                              make_float4((float)ax * inv_scale, (float)ay * inv_scale, (float)az * inv_scale, 0.0f));
            }
            __syncwarp();
        }
    }
    if (amax > mag_lim) raise_err(err, ERR_RANGE, 0); // |f scale| >= 2^21: DPD_ERR_NUMERIC
}

} // namespace dpd
