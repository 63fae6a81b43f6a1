// dpd_kernels.cuh -- the kernels of one DPD time step on sm_100a (single-GPU path).
//
// Step, all on one stream:
//   k_bin      a1+a2  kick-drift-wrap in registers, cell index, warp-aggregated atomic
//                     histogram -> rank within cell
//   k_scan     a3     single-pass exclusive scan of the counts (decoupled look-back)
//   k_scatter  a4     recompute a1 bit-identically, write the cell-sorted copy
//   k_force    a5     half-stencil pair sweep, Newton-3 via atomics
//   (a6, the second half-kick, is folded into the next step's kick and into the getters)
#pragma once

#include "dpd_device.cuh"

namespace dpd {

// Error word bits (device int err[4]: [0] flags, [1] offending id, [2] overflow amount)
enum : int { ERR_NONFINITE = 1, ERR_CAPACITY = 2, ERR_RANGE = 4, ERR_SPECIES = 8, ERR_IDRANGE = 16 };

__device__ __forceinline__ void raise_err(int *err, int bit, int id)
{
    if ((atomicOr(&err[0], bit) & bit) == 0) err[1] = id;
}

__device__ __forceinline__ bool finite3(float a, float b, float c)
{
    return isfinite(a) && isfinite(b) && isfinite(c);
}

// Wrap into [0, L) (C-10): x<0 -> x+L; x>=L -> x-L; then x>=L -> 0.
__device__ __forceinline__ float wrap_coord(float x, float L)
{
    if (x < 0.0f) x = __fadd_rn(x, L);
    else if (x >= L) x = __fsub_rn(x, L);
    if (x >= L) x = 0.0f;
    return x;
}

// Linear index of the cell holding local position (x, y, z) (C-8), extended grid.
__device__ __forceinline__ int cell_index(const Geom &g, float x, float y, float z)
{
    const int ix = cell_coord(x, g.inv_h[0], g.n[0]) + g.off[0];
    const int iy = cell_coord(y, g.inv_h[1], g.n[1]) + g.off[1];
    const int iz = cell_coord(z, g.inv_h[2], g.n[2]) + g.off[2];
    return ix + g.ext[0] * (iy + g.ext[1] * iz);
}

// Body force along z: periodic Poiseuille, or uniform (wall-bounded flows).
__device__ __forceinline__ float body_fz(const IntegP &ip, float x_local)
{
    if (ip.body_mode == 1) return ip.body_f;
    return (x_local <= ip.x_half) ? -ip.body_f : ip.body_f;
}

__device__ __forceinline__ bool is_frozen(const IntegP &ip, const float4 v)
{
    return (ip.frozen_mask >> (__float_as_int(v.w) & 31)) & 1;
}

// Wall SDF at a local-frame point (C-23): s = max over primitives of the signed distance
// (global frame), *arg = the maximising primitive.  Fixed _rn arithmetic: k_bin and
// k_scatter must take the same bounce decisions.
__device__ __forceinline__ float wall_sdf(const IntegP &ip, float x, float y, float z, int &arg)
{
    const float g[3] = {__fadd_rn(x, ip.origin[0]), __fadd_rn(y, ip.origin[1]), __fadd_rn(z, ip.origin[2])};
    float best = -3.0e38f;
    arg = 0;
    for (int k = 0; k < ip.nwall; ++k) {
        const float *q = ip.wprm[k];
        float sk;
        if (ip.wtype[k] == 1) {
            sk = __fsub_rn(__fmaf_rn(q[2], g[2], __fmaf_rn(q[1], g[1], __fmul_rn(q[0], g[0]))), q[3]);
        } else {
            const int ax = ip.wtype[k] - 2, a = (ax + 1) % 3, b = (ax + 2) % 3;
            const float da = __fsub_rn(g[a], q[0]), db = __fsub_rn(g[b], q[1]);
            sk = __fmul_rn(q[3], __fsub_rn(q[2], __fsqrt_rn(__fmaf_rn(da, da, __fmul_rn(db, db)))));
        }
        if (sk > best) {
            best = sk;
            arg = k;
        }
    }
    return best;
}

// First half of GW-VV fused with the previous step's second half (C-6):
//   u' = u + kick (F + f_body(x));  x' = wrap(x + dt u')
// with bounce-back off SDF walls (C-23): if x' is inside the solid, bisection
// (32 halvings) finds the last point x + t u with s <= 0, the particle is placed there and
// u' <- 2 u_w - u'.  Frozen species do not move.  Explicit _rn intrinsics pin the rounding
// so k_bin and k_scatter agree bit-for-bit.
template <bool LEAN>
__device__ __forceinline__ void advance(const Geom &g, const IntegP &ip, const float4 p, const float4 v,
                                        const float4 f, float3 &xn, float3 &un)
{
    // LEAN: no frozen species, no walls (k_bin / k_scatter instantiate both forms identically)
    if (!LEAN && ip.frozen_mask && is_frozen(ip, v)) {
        un = make_float3(v.x, v.y, v.z);
        xn = make_float3(p.x, p.y, p.z);
        return;
    }
    const float fb = body_fz(ip, p.x);
    un.x = __fmaf_rn(ip.kick, f.x, v.x);
    un.y = __fmaf_rn(ip.kick, f.y, v.y);
    un.z = __fmaf_rn(ip.kick, __fadd_rn(f.z, fb), v.z);
    xn.x = __fmaf_rn(ip.dt, un.x, p.x);
    xn.y = __fmaf_rn(ip.dt, un.y, p.y);
    xn.z = __fmaf_rn(ip.dt, un.z, p.z);
    if (!LEAN && ip.nwall > 0) {
        int arg;
        if (wall_sdf(ip, xn.x, xn.y, xn.z, arg) > 0.0f) {
            float lo = 0.0f, hi = ip.dt;
            if (wall_sdf(ip, p.x, p.y, p.z, arg) > 0.0f) hi = 0.0f; // already inside: stay, reverse
            for (int it = 0; it < 32 && hi > 0.0f; ++it) {
                const float mid = __fmul_rn(0.5f, __fadd_rn(lo, hi));
                if (wall_sdf(ip, __fmaf_rn(mid, un.x, p.x), __fmaf_rn(mid, un.y, p.y), __fmaf_rn(mid, un.z, p.z),
                             arg) > 0.0f)
                    hi = mid;
                else
                    lo = mid;
            }
            xn.x = __fmaf_rn(lo, un.x, p.x);
            xn.y = __fmaf_rn(lo, un.y, p.y);
            xn.z = __fmaf_rn(lo, un.z, p.z);
            wall_sdf(ip, xn.x, xn.y, xn.z, arg);
            un.x = __fsub_rn(2.0f * ip.wvel[arg][0], un.x);
            un.y = __fsub_rn(2.0f * ip.wvel[arg][1], un.y);
            un.z = __fsub_rn(2.0f * ip.wvel[arg][2], un.z);
        }
    }
    if (!g.split[0]) xn.x = wrap_coord(xn.x, g.L[0]);
    if (!g.split[1]) xn.y = wrap_coord(xn.y, g.L[1]);
    if (!g.split[2]) xn.z = wrap_coord(xn.z, g.L[2]);
}

__device__ __forceinline__ bool in_local_box(const Geom &g, const float3 &x)
{
    return x.x >= 0.0f && x.x < g.L[0] && x.y >= 0.0f && x.y < g.L[1] && x.z >= 0.0f && x.z < g.L[2];
}

__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp-aggregated atomic histogram: returns this lane's rank within cell c (c < 0: none).
__device__ __forceinline__ int warp_rank_in_cell(int *count, int c)
{
    const unsigned mask = __match_any_sync(0xffffffffu, c);
    const int leader = __ffs(mask) - 1;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == leader && c >= 0) base = atomicAdd(&count[c], __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + __popc(mask & lanemask_lt());
}

// ---------------------------------------------------------------------------------------
// Per-direction message buffers of the decomposition (ghosts and migrants).  Direction
// D = (dx, dy, dz) in {-1,0,1}^3 has index d = (dx+1) + 3 (dy+1) + 9 (dz+1) (13 = none).
// Message d starts at base + off[d] bytes: an int4 header {count, 0, 0, 0} followed by cap[d]
// particles of two float4 each (x, y, z, id bits) and (u_x, u_y, u_z, 0).  cap[d] = 0 marks an
// unused direction.  base == nullptr: single domain, no messages.
// ---------------------------------------------------------------------------------------
struct Msgs {
    char *base;
    int off[27];
    int cap[27];
};

__device__ __forceinline__ int *msg_count(const Msgs &m, int d) { return reinterpret_cast<int *>(m.base + m.off[d]); }
__device__ __forceinline__ float4 *msg_data(const Msgs &m, int d)
{
    return reinterpret_cast<float4 *>(m.base + m.off[d] + 16);
}

// ---------------------------------------------------------------------------------------
// Input packing (set_particles): AoS xyz -> pos4 (x, y, z, id bits), vel4; periodic wrap
// into the global box (C-10), then (decomposed runs) keep only the particles inside this
// rank's subdomain, in local coordinates.  *n_out counts the kept particles.
// ---------------------------------------------------------------------------------------
__global__ void k_pack_input(const float *__restrict__ pos3, const float *__restrict__ vel3,
                             const int32_t *__restrict__ ids, const int32_t *__restrict__ species, int nspecies,
                             int64_t n, Geom g, float3 gbox, float3 origin, float4 *__restrict__ pos4,
                             float4 *__restrict__ vel4, float4 *__restrict__ frc4, int *n_out, int cap, int *err)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool keep = false;
    float4 p4, v4;
    if (i < n) {
        float x = pos3[3 * i + 0], y = pos3[3 * i + 1], z = pos3[3 * i + 2];
        const float vx = vel3[3 * i + 0], vy = vel3[3 * i + 1], vz = vel3[3 * i + 2];
        const int id = ids ? ids[i] : (int)i;
        if (!finite3(x, y, z) || !finite3(vx, vy, vz)) {
            raise_err(err, ERR_NONFINITE, id);
            x = y = z = 0.0f;
        }
        // periodic wrap by whole multiples of the global box (input may lie several boxes away)
        x = wrap_coord(x - gbox.x * floorf(x / gbox.x), gbox.x);
        y = wrap_coord(y - gbox.y * floorf(y / gbox.y), gbox.y);
        z = wrap_coord(z - gbox.z * floorf(z / gbox.z), gbox.z);
        x -= origin.x;
        y -= origin.y;
        z -= origin.z;
        keep = x >= 0.0f && x < g.L[0] && y >= 0.0f && y < g.L[1] && z >= 0.0f && z < g.L[2];
        int sp = species ? species[i] : 0;
        if (sp < 0 || sp >= nspecies) {
            raise_err(err, ERR_SPECIES, id);
            sp = 0;
        }
        // the tiled force kernel carries the species in bits 30-31 of the staged id word
        if (id < 0 || (nspecies > 1 && id >= (1 << 30))) raise_err(err, ERR_IDRANGE, id);
        p4 = make_float4(x, y, z, __int_as_float(id));
        v4 = make_float4(vx, vy, vz, __int_as_float(sp)); // w: species index (NEXT-2)
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(n_out, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) {
        const int slot = base + __popc(m & lanemask_lt());
        if (slot < cap) {
            pos4[slot] = p4;
            vel4[slot] = v4;
            frc4[slot] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        } else {
            raise_err(err, ERR_CAPACITY, __float_as_int(p4.w));
        }
    }
}

// Number of input particles that fall inside this rank's subdomain (sizes the arrays).
__global__ void k_count_inside(const float *__restrict__ pos3, int64_t n, float3 gbox, float3 origin, float3 sub,
                               int *out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool in = false;
    if (i < n) {
        float x = pos3[3 * i + 0], y = pos3[3 * i + 1], z = pos3[3 * i + 2];
        if (isfinite(x) && isfinite(y) && isfinite(z)) {
            x = wrap_coord(x - gbox.x * floorf(x / gbox.x), gbox.x) - origin.x;
            y = wrap_coord(y - gbox.y * floorf(y / gbox.y), gbox.y) - origin.y;
            z = wrap_coord(z - gbox.z * floorf(z / gbox.z), gbox.z) - origin.z;
            in = x >= 0.0f && x < sub.x && y >= 0.0f && y < sub.y && z >= 0.0f && z < sub.z;
        } else {
            in = origin.x == 0.0f && origin.y == 0.0f && origin.z == 0.0f; // reported by the pack kernel
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, __popc(m));
}

__device__ __forceinline__ int dir_index(int dx, int dy, int dz) { return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1); }

// ---------------------------------------------------------------------------------------
// a1 + a2: kick, drift, wrap (periodic-local dimensions), cell index, atomic histogram.
// In decomposed runs a particle that crossed a split face is a migrant (row a10): it is
// shifted into the neighbour's frame and appended to the message of its exit direction;
// rank = -1 drops it from the local sort.  The particle count comes from the device
// (start_old[ncell]) so no host synchronisation is needed between steps.
// ---------------------------------------------------------------------------------------
// 8 resident blocks (full occupancy, 32 registers) hide the load + histogram-atomic latency:
// measured 29.1 -> 27.0 us at 2.1 M particles
template <bool LEAN> // LEAN: single domain, no walls, no frozen species (the bench / eq64 path)
__global__ void __launch_bounds__(256, 8) k_bin(const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                                             const float4 *__restrict__ frc, const int *__restrict__ n_ptr, Geom g,
                                             IntegP ip, int *__restrict__ count, int *__restrict__ rank, Msgs mig,
                                             int *err)
{
#ifndef KBIN_REVERSE
#define KBIN_REVERSE 1
#endif
    // blocks walk the particles from the high end: the force kernel just touched the high
    // addresses last (tiles in increasing z), so they are still in L2; k_scatter then walks
    // forward from the low end that this kernel touched last
    const int blk = KBIN_REVERSE ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
    const int i = blk * blockDim.x + threadIdx.x;
    const int n = *n_ptr;
    int c = -1;
    if (i < n) {
        const float4 p = pos[i], v = vel[i], f = frc[i];
        float3 xn, un;
        advance<LEAN>(g, ip, p, v, f, xn, un);
        int dx = 0, dy = 0, dz = 0;
        if (!LEAN && g.split[0]) dx = xn.x < 0.0f ? -1 : (xn.x >= g.L[0] ? 1 : 0);
        if (!LEAN && g.split[1]) dy = xn.y < 0.0f ? -1 : (xn.y >= g.L[1] ? 1 : 0);
        if (!LEAN && g.split[2]) dz = xn.z < 0.0f ? -1 : (xn.z >= g.L[2] ? 1 : 0);
        if (dx | dy | dz) {
            // migrant: into the destination frame.  x - (-L) = x + L can round up to L for
            // x within an ulp below 0; keep it inside [0, L) (the C-10 rule for wrapped axes)
            xn.x -= dx * g.L[0];
            xn.y -= dy * g.L[1];
            xn.z -= dz * g.L[2];
            if (dx < 0 && xn.x >= g.L[0]) xn.x = __int_as_float(__float_as_int(g.L[0]) - 1);
            if (dy < 0 && xn.y >= g.L[1]) xn.y = __int_as_float(__float_as_int(g.L[1]) - 1);
            if (dz < 0 && xn.z >= g.L[2]) xn.z = __int_as_float(__float_as_int(g.L[2]) - 1);
            const int d = dir_index(dx, dy, dz);
            if (!finite3(xn.x, xn.y, xn.z) || !in_local_box(g, xn)) {
                raise_err(err, ERR_RANGE, __float_as_int(p.w));
            } else {
                const int slot = atomicAdd(msg_count(mig, d), 1);
                if (slot < mig.cap[d]) {
                    float4 *q = msg_data(mig, d) + 2 * slot;
                    q[0] = make_float4(xn.x, xn.y, xn.z, p.w);
                    q[1] = make_float4(un.x, un.y, un.z, v.w); // w: species
                } else {
                    raise_err(err, ERR_CAPACITY, __float_as_int(p.w));
                }
            }
        } else {
            if (!finite3(xn.x, xn.y, xn.z) || !finite3(un.x, un.y, un.z) || !in_local_box(g, xn)) {
                raise_err(err, finite3(un.x, un.y, un.z) ? ERR_RANGE : ERR_NONFINITE, __float_as_int(p.w));
                xn = make_float3(0.0f, 0.0f, 0.0f);
            }
            c = cell_index(g, xn.x, xn.y, xn.z);
        }
    }
    const int r = warp_rank_in_cell(count, c);
    if (i < n) rank[i] = (c >= 0) ? r : -1;
}

// ---------------------------------------------------------------------------------------
// a3: exclusive scan start[c] = sum_{c'<c} count[c'], start[ncell] = total; count := 0
// for the next step.  Single pass, decoupled look-back over 4096-cell tiles; the tile
// status words carry a launch epoch kept on the device (graph-replay safe).
// ---------------------------------------------------------------------------------------
constexpr int kScanThreads = 256;
#ifndef KSCAN_ITEMS
#define KSCAN_ITEMS 16
#endif
constexpr int kScanItems = KSCAN_ITEMS;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned long long scan_pack(unsigned epoch, int flag, int value)
{
    return ((unsigned long long)((epoch << 2) | (unsigned)flag) << 32) | (unsigned)value;
}

__global__ void __launch_bounds__(kScanThreads) k_scan(int *__restrict__ count, int *__restrict__ start,
                                                       int ncell, unsigned long long *tstate,
                                                       unsigned *epoch_ptr)
{
    __shared__ int warp_sums[kScanThreads / 32];
    __shared__ int tile_prefix;
    __shared__ unsigned s_epoch;
    const int tile = blockIdx.x;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) s_epoch = *((volatile unsigned *)epoch_ptr) + 1u;
    const int base = tile * kScanTile + t * kScanItems;
    int v[kScanItems];
    if (base + kScanItems <= ncell) {
        const int4 *src = reinterpret_cast<const int4 *>(count + base);
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            const int4 a = src[q];
            v[4 * q + 0] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = (base + k < ncell) ? count[base + k] : 0;
    }
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) sum += v[k];
    // block exclusive scan of the per-thread sums
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    const unsigned epoch = s_epoch;
    int warp_off = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
        const int s = warp_sums[w];
        if (w < warp) warp_off += s;
        total += s;
    }
    int excl = warp_off + incl - sum;
    // publish and look back
    if (warp == 0) {
        volatile unsigned long long *vs = tstate;
        if (tile == 0) {
            if (lane == 0) {
                vs[0] = scan_pack(epoch, 2, total);
                tile_prefix = 0;
            }
        } else {
            if (lane == 0) vs[tile] = scan_pack(epoch, 1, total);
            int prefix = 0;
            int pred = tile - 1;
            while (true) {
                const int idx = pred - lane;
                unsigned long long st = idx >= 0 ? vs[idx] : scan_pack(epoch, 2, 0);
                unsigned hi = (unsigned)(st >> 32);
                int flag = ((hi >> 2) == epoch) ? (int)(hi & 3u) : 0;
                if (__any_sync(0xffffffffu, flag == 0)) continue; // a predecessor not yet published
                const unsigned incl_mask = __ballot_sync(0xffffffffu, flag == 2);
                const int val = (int)(unsigned)st;
                if (incl_mask) {
                    const int first = __ffs(incl_mask) - 1; // nearest inclusive predecessor
                    int s = lane <= first ? val : 0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    prefix += s;
                    break;
                }
                int s = val;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                prefix += s;
                pred -= 32;
            }
            if (lane == 0) {
                vs[tile] = scan_pack(epoch, 2, prefix + total);
                tile_prefix = prefix;
            }
        }
    }
    __syncthreads();
    excl += tile_prefix;
    if (base + kScanItems <= ncell) {
        int4 *dst = reinterpret_cast<int4 *>(start + base);
        int4 *cz = reinterpret_cast<int4 *>(count + base);
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            int4 o;
            o.x = excl; excl += v[4 * q + 0];
            o.y = excl; excl += v[4 * q + 1];
            o.z = excl; excl += v[4 * q + 2];
            o.w = excl; excl += v[4 * q + 3];
            dst[q] = o;
            cz[q] = make_int4(0, 0, 0, 0);
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (base + k < ncell) {
                start[base + k] = excl;
                count[base + k] = 0;
            }
            excl += v[k];
        }
    }
    if (tile == gridDim.x - 1) {
        if (t == kScanThreads - 1) start[ncell] = tile_prefix + total;
        if (t == 0) *((volatile unsigned *)epoch_ptr) = epoch; // every tile has read it by now
    }
}

// ---------------------------------------------------------------------------------------
// a4: scatter into cell order; recomputes a1 in registers (bit-identical to k_bin).  The
// sorted force array it pairs with is already zero (k_force_tile zeroes it one step ahead).
// ---------------------------------------------------------------------------------------
template <bool LEAN>
__global__ void __launch_bounds__(256) k_scatter(const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                                                 const float4 *__restrict__ frc, const int *__restrict__ n_ptr, Geom g,
                                                 IntegP ip, const int *__restrict__ start,
                                                 const int *__restrict__ rank, float4 *__restrict__ pos_o,
                                                 float4 *__restrict__ vel_o, int cap, int *err)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= *n_ptr || rank[i] < 0) return; // rank < 0: migrant, sent away
    const float4 p = pos[i], v = vel[i], f = frc[i];
    float3 xn, un;
    advance<LEAN>(g, ip, p, v, f, xn, un);
    if (!finite3(xn.x, xn.y, xn.z) || !finite3(un.x, un.y, un.z) || !in_local_box(g, xn))
        xn = make_float3(0.0f, 0.0f, 0.0f);
    const int c = cell_index(g, xn.x, xn.y, xn.z);
    const int dst = start[c] + rank[i];
    if (dst >= cap) { // a decomposed member gained more particles than its arrays hold
        raise_err(err, ERR_CAPACITY, __float_as_int(p.w));
        return;
    }
    pos_o[dst] = make_float4(xn.x, xn.y, xn.z, p.w);
    vel_o[dst] = make_float4(un.x, un.y, un.z, v.w); // w: species
    // no force write: the target force buffer was zeroed by the previous force pass
}

// ---------------------------------------------------------------------------------------
// a5 (reference kernel, v1): one thread per particle i of the sorted arrays; j over the
// own cell (j > i) and the 13 forward neighbour cells; F_i in registers, F_j -= f via
// vector atomics.  RECORD dumps (lo id, hi id, w0, w1) of every pair.
// ---------------------------------------------------------------------------------------
struct PairRec {
    uint4 *quad;
    unsigned long long *count;
    long long cap;
};

__constant__ int c_fwd[14][3] = {{0, 0, 0},  {1, 0, 0},  {-1, 1, 0}, {0, 1, 0},  {1, 1, 0},
                                 {-1, -1, 1}, {0, -1, 1}, {1, -1, 1}, {-1, 0, 1}, {0, 0, 1},
                                 {1, 0, 1},  {-1, 1, 1}, {0, 1, 1},  {1, 1, 1}};

__device__ __forceinline__ void atomic_add_f3(float4 *p, float x, float y, float z)
{
    atomicAdd(p, make_float4(x, y, z, 0.0f));
}

template <bool RECORD, int KMODE>
__global__ void __launch_bounds__(128) k_force_ref(const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                                                   float4 *frc, const int *__restrict__ start, int n, Geom g,
                                                   PairP pp, uint32_t s_lo, uint32_t s_hi, PairRec rec)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t ks = step_key(s_lo, s_hi, pp.seed_lo, pp.seed_hi);
    const float4 pi = pos[i], vi = vel[i];
    const uint32_t idi = (uint32_t)__float_as_int(pi.w);
    const int cx = cell_coord(pi.x, g.inv_h[0], g.n[0]);
    const int cy = cell_coord(pi.y, g.inv_h[1], g.n[1]);
    const int cz = cell_coord(pi.z, g.inv_h[2], g.n[2]);
    float Fx = 0.0f, Fy = 0.0f, Fz = 0.0f;
    for (int o = 0; o < 14; ++o) {
        int jx = cx + c_fwd[o][0], jy = cy + c_fwd[o][1], jz = cz + c_fwd[o][2];
        float sx = 0.0f, sy = 0.0f, sz = 0.0f;
        if (jx < 0) { jx += g.n[0]; sx = -g.L[0]; } else if (jx >= g.n[0]) { jx -= g.n[0]; sx = g.L[0]; }
        if (jy < 0) { jy += g.n[1]; sy = -g.L[1]; } else if (jy >= g.n[1]) { jy -= g.n[1]; sy = g.L[1]; }
        if (jz < 0) { jz += g.n[2]; sz = -g.L[2]; } else if (jz >= g.n[2]) { jz -= g.n[2]; sz = g.L[2]; }
        const int c = jx + g.ext[0] * (jy + g.ext[1] * jz);
        int j0 = start[c];
        const int j1 = start[c + 1];
        if (o == 0) j0 = i + 1;
        for (int j = j0; j < j1; ++j) {
            const float4 pj = pos[j];
            const float dx = pi.x - (pj.x + sx);
            const float dy = pi.y - (pj.y + sy);
            const float dz = pi.z - (pj.z + sz);
            const float r2 = dx * dx + dy * dy + dz * dz;
            if (r2 < pp.rc2 && r2 > 0.0f) {
                const float4 vj = vel[j];
                const float dvdot = dx * (vi.x - vj.x) + dy * (vi.y - vj.y) + dz * (vi.z - vj.z);
                const uint32_t idj = (uint32_t)__float_as_int(pj.w);
                const float s = pair_scalar<KMODE>(pp, r2, dvdot, idi, idj, ks, vi.w, vj.w);
                Fx += s * dx;
                Fy += s * dy;
                Fz += s * dz;
                atomic_add_f3(&frc[j], -s * dx, -s * dy, -s * dz);
                if constexpr (RECORD) {
                    const unsigned long long k = atomicAdd(rec.count, 1ull);
                    if ((long long)k < rec.cap) {
                        const uint2 wd = pair_words(idi, idj, ks);
                        rec.quad[k] = make_uint4(min(idi, idj), max(idi, idj), wd.x, wd.y);
                    }
                }
            }
        }
    }
    atomic_add_f3(&frc[i], Fx, Fy, Fz);
}

// ---------------------------------------------------------------------------------------
// Output helpers.
// ---------------------------------------------------------------------------------------
// Full-step velocity v = u + hk (F + f_body(x)), hk = kick_next - dt/2 (0 right after set).
__global__ void k_gather_id(const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                            const float4 *__restrict__ frc, int n, float hk, IntegP ip,
                            float3 origin, float *__restrict__ pos3, float *__restrict__ vel3,
                            float *__restrict__ f3, int by_id)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = pos[i], v = vel[i], f = frc[i];
    const int row = by_id ? __float_as_int(p.w) : i;
    if (pos3) {
        pos3[3 * row + 0] = p.x + origin.x;
        pos3[3 * row + 1] = p.y + origin.y;
        pos3[3 * row + 2] = p.z + origin.z;
    }
    if (vel3) {
        const float fb = body_fz(ip, p.x);
        const float h = (ip.frozen_mask && is_frozen(ip, v)) ? 0.0f : hk; // frozen: the wall velocity
        vel3[3 * row + 0] = __fmaf_rn(h, f.x, v.x);
        vel3[3 * row + 1] = __fmaf_rn(h, f.y, v.y);
        vel3[3 * row + 2] = __fmaf_rn(h, __fadd_rn(f.z, fb), v.z);
    }
    if (f3) {
        f3[3 * row + 0] = f.x;
        f3[3 * row + 1] = f.y;
        f3[3 * row + 2] = f.z;
    }
}

// Snapshot of the asynchronous dump: the first *count
// particles (device-resident count) in cell order -- positions in the global frame,
// full-step velocities (row a6, as k_gather_id) and ids -- into a staging block
// [int64 count | pad][pos n x 3][vel n x 3][ids n] laid out for `cap` particles.
__global__ void k_snapshot(const float4 *__restrict__ pos, const float4 *__restrict__ vel,
                           const float4 *__restrict__ frc, const int *__restrict__ count, int cap, float hk,
                           IntegP ip, float3 origin, long long *__restrict__ hdr, float *__restrict__ pos3,
                           float *__restrict__ vel3, int32_t *__restrict__ ids)
{
    const int n = min(*count, cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        hdr[0] = n;
        hdr[1] = 0;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 p = pos[i], v = vel[i], f = frc[i];
        pos3[3 * i + 0] = p.x + origin.x;
        pos3[3 * i + 1] = p.y + origin.y;
        pos3[3 * i + 2] = p.z + origin.z;
        const float fb = body_fz(ip, p.x);
        const float h = (ip.frozen_mask && is_frozen(ip, v)) ? 0.0f : hk;
        vel3[3 * i + 0] = __fmaf_rn(h, f.x, v.x);
        vel3[3 * i + 1] = __fmaf_rn(h, f.y, v.y);
        vel3[3 * i + 2] = __fmaf_rn(h, __fadd_rn(f.z, fb), v.z);
        ids[i] = __float_as_int(p.w);
    }
}

__global__ void k_ids_cells(const float4 *__restrict__ pos, int n, Geom g, int32_t *__restrict__ ids,
                            int32_t *__restrict__ cell_of_id)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = pos[i];
    const int id = __float_as_int(p.w);
    if (ids) ids[i] = id;
    if (cell_of_id) cell_of_id[id] = cell_index(g, p.x, p.y, p.z);
}

// ---------------------------------------------------------------------------------------
// NEXT-3 walls: frozen-layer carve (C-23).  s > r_c: removed; 0 < s <= r_c:
// frozen wall particle of species wall_species with the wall velocity; else fluid, whose
// stored half-step velocity is first completed to the full-step v = u + hk (F + f_body).
// ---------------------------------------------------------------------------------------
__global__ void k_wall_classify(float4 *__restrict__ pos, float4 *__restrict__ vel, const float4 *__restrict__ frc,
                                int n, IntegP ip, float hk, float rc, int wall_species, int *__restrict__ keep,
                                int *counters)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = pos[i];
    float4 v = vel[i];
    int arg;
    const float sd = wall_sdf(ip, p.x, p.y, p.z, arg);
    int k = 1;
    if (ip.frozen_mask && is_frozen(ip, v)) {
        // an existing wall particle stays as it is
    } else if (sd > rc) {
        k = 0;
        atomicAdd(&counters[1], 1);
    } else if (sd > 0.0f) {
        v = make_float4(ip.wvel[arg][0], ip.wvel[arg][1], ip.wvel[arg][2], __int_as_float(wall_species));
        atomicAdd(&counters[0], 1);
    } else {
        const float4 f = frc[i];
        v.x = __fmaf_rn(hk, f.x, v.x);
        v.y = __fmaf_rn(hk, f.y, v.y);
        v.z = __fmaf_rn(hk, __fadd_rn(f.z, body_fz(ip, p.x)), v.z);
    }
    vel[i] = v;
    keep[i] = k;
}

// Compaction of the kept particles (order is irrelevant: they are re-sorted into cells).
__global__ void k_wall_compact(const float4 *__restrict__ pos, const float4 *__restrict__ vel, int n,
                               const int *__restrict__ keep, float4 *__restrict__ pos_o, float4 *__restrict__ vel_o,
                               float4 *__restrict__ frc_o, int *n_out, int *__restrict__ keep_by_id)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool k = i < n && keep[i];
    if (i < n && keep_by_id) keep_by_id[__float_as_int(pos[i].w)] = k ? 1 : 0;
    const unsigned m = __ballot_sync(0xffffffffu, k);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(n_out, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (k) {
        const int slot = base + __popc(m & lanemask_lt());
        pos_o[slot] = pos[i];
        vel_o[slot] = vel[i];
        frc_o[slot] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
}

// Dense renumbering after a carve (single domain): id <- rank of id among the kept ids.
__global__ void k_renumber(float4 *__restrict__ pos, int n, const int *__restrict__ new_id)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    pos[i].w = __int_as_float(new_id[__float_as_int(pos[i].w)]);
}

// Wall SDF at global points (test hook for the device SDF).
__global__ void k_wall_sdf_eval(const float *__restrict__ x3, int n, IntegP ip, float *__restrict__ s)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int arg;
    s[i] = wall_sdf(ip, x3[3 * i], x3[3 * i + 1], x3[3 * i + 2], arg);
}

// Species index (vel.w, NEXT-2) per particle, in id order (by_id) or storage order.
__global__ void k_species_out(const float4 *__restrict__ pos, const float4 *__restrict__ vel, int n,
                              int32_t *__restrict__ out, int by_id)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[by_id ? __float_as_int(pos[i].w) : i] = __float_as_int(vel[i].w);
}

// Raw-state copy in storage order (x in global coordinates, u, F as float3 rows).
__global__ void k_state(const float4 *__restrict__ pos, const float4 *__restrict__ vel, const float4 *__restrict__ frc,
                        int n, float3 origin, float *__restrict__ pos3, float *__restrict__ u3,
                        float *__restrict__ f3, int32_t *__restrict__ ids)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = pos[i], v = vel[i], f = frc[i];
    if (pos3) { pos3[3 * i] = p.x + origin.x; pos3[3 * i + 1] = p.y + origin.y; pos3[3 * i + 2] = p.z + origin.z; }
    if (u3) { u3[3 * i] = v.x; u3[3 * i + 1] = v.y; u3[3 * i + 2] = v.z; }
    if (f3) { f3[3 * i] = f.x; f3[3 * i + 1] = f.y; f3[3 * i + 2] = f.z; }
    if (ids) ids[i] = __float_as_int(p.w);
}

// Philox cross-check kernels (T0 on the device).
__global__ void k_philox2(const uint2 *__restrict__ ctr, const uint32_t *__restrict__ key, uint2 *__restrict__ out,
                          int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = philox2x32_10(ctr[i].x, ctr[i].y, key[i]);
}

__global__ void k_pair_words(const uint4 *__restrict__ in, uint32_t seed_lo, uint32_t seed_hi, float *__restrict__ xi,
                             uint2 *__restrict__ w, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 q = in[i]; // ida, idb, s_lo, s_hi
    const uint2 wd = pair_words(q.x, q.y, step_key(q.z, q.w, seed_lo, seed_hi));
    w[i] = wd;
    xi[i] = box_muller(wd.x, wd.y);
}

} // namespace dpd
