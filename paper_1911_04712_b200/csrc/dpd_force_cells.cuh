// dpd_force_cells.cuh -- pair-force sweep with one WARP per home CELL.
//
// Same tile staging, fixed-point shared accumulation and flush as k_force_tile
// (dpd_force_tile.cuh), but the candidate sweep and the pair evaluation are organised per
// home cell so that a warp's lanes share their candidate segments:
//   * a warp takes home cells from a per-CTA queue; the cell's n_c particles get
//     Q = floor(32 / n_c) lanes each, which split every candidate segment (packed pairs of
//     consecutive candidates at stride 2 Q) -- all lanes of the warp sweep segments of the
//     same length (the 27-cell neighbourhood is shared by the cell), so the sweep runs at
//     near-full SIMT efficiency instead of the max-over-lanes of a particle-per-lane sweep;
//   * own-cell pairs are split circularly (slot a takes a+1 .. a+hh mod n_c), so every
//     particle owns about half of its cell mates;
//   * hits go to short per-lane lists (owner = the lane's particle) that the same warp then
//     evaluates 32 pairs at a time in contiguous per-lane chunks (warp-local: no CTA barrier
//     between sweep and pairs).
// The smaller lists make the tile fit 3 CTAs per SM (24 warps).
#pragma once

#include "dpd_force_tile.cuh"

namespace dpd {

constexpr int FC_NTHR = 256;
constexpr int FC_NWARP = FC_NTHR / 32;
constexpr int FC_SCAP = 1152;                // staged particles (mean 864, sd 29 at rho = 8)
constexpr int FC_LCAP = 24;                  // hits per lane (mean 16.8 / Q)
constexpr int FC_LSTRIDE = FC_LCAP + 2;      // 13 words (odd): conflict-free appends
constexpr int FC_NHC = FT_BX * FT_BY * FT_BZ; // home cells per tile (32)

struct ForceCellSmem {
    float4 sv[FC_SCAP];                          // staged velocities
    float sx[FC_SCAP], sy[FC_SCAP], sz[FC_SCAP]; // staged positions (tile frame)
    int sid[FC_SCAP];                            // staged global ids
    int acc[3][FC_SCAP];                         // fixed-point force sums
    unsigned short lst[FC_NTHR * FC_LSTRIDE];    // per-lane pair lists
    int wexcl[FC_NWARP][33];                     // per-warp compacted owners: list prefix (+ total)
    int wsi[FC_NWARP][32];                       //   owner particle
    int wrow[FC_NWARP][32];                      //   list base minus prefix
    int soff[FT_NSC + 1];                        // staged cell -> smem start
    int cgs[FT_NSC];                             // staged cell -> global start
    int total;
    int next_task;
};

__device__ __forceinline__ float4 ldp_c(const ForceCellSmem &S, int j)
{
    return make_float4(S.sx[j], S.sy[j], S.sz[j], __int_as_float(S.sid[j]));
}

// Pair force in the global-memory convention (pi.w = id bits, vi.w = species bits):
// f_ij = s (dx, dy, dz), s = 0 for coincident particles (C-11).
template <int KMODE>
__device__ __forceinline__ float pair_core_c(const PairP &pp, float4 pi, float4 vi, float4 pj, float4 vj,
                                             uint32_t ks, float &dx, float &dy, float &dz)
{
    dx = pi.x - pj.x;
    dy = pi.y - pj.y;
    dz = pi.z - pj.z;
    const float r2 = dx * dx + dy * dy + dz * dz;
    const float dvdot = dx * (vi.x - vj.x) + dy * (vi.y - vj.y) + dz * (vi.z - vj.z);
    const float s = pair_scalar<KMODE>(pp, fmaxf(r2, 1e-30f), dvdot, (uint32_t)__float_as_int(pi.w),
                                       (uint32_t)__float_as_int(pj.w), ks, vi.w, vj.w);
    return r2 > 0.0f ? s : 0.0f;
}

// Range check of the fixed-point conversion and (debug) pair recording.
template <bool RECORD>
__device__ __forceinline__ void pair_checks_c(const PairP &pp, const FixP &fx, float4 pi, float4 pj, float s,
                                              float dx, float dy, float dz, uint32_t ks, PairRec &rec, int *err)
{
    const float r2 = dx * dx + dy * dy + dz * dz;
    if (fabsf(s) * (r2 * rsqrtf(fmaxf(r2, 1e-30f))) > fx.mag_lim) raise_err(err, ERR_RANGE, __float_as_int(pi.w));
    if constexpr (RECORD) {
        if (r2 > 0.0f) {
            const uint32_t idi = (uint32_t)__float_as_int(pi.w), idj = (uint32_t)__float_as_int(pj.w);
            const unsigned long long k = atomicAdd(rec.count, 1ull);
            if ((long long)k < rec.cap) {
                const uint2 wd = pair_words(idi, idj, ks);
                rec.quad[k] = make_uint4(min(idi, idj), max(idi, idj), wd.x, wd.y);
            }
        }
    }
}

// Strided sweep of [lo, hi): this lane takes the aligned candidate pairs (2m, 2m + 1) with
// m = m0 + q, m0 + q + Q, ... (m0 = lo / 2), appending at most `room` hits.  Returns the
// first candidate index it did not examine (hi if done) -- only relevant when the list
// filled up.
__device__ __forceinline__ void sweep_strided(const ForceCellSmem &S, unsigned &lptr, int lo, int hi, int q, int Q,
                                              float px, float py, float pz, float rc2)
{
    const unsigned long long PX = f2dup(px), PY = f2dup(py), PZ = f2dup(pz);
    for (int j = (lo & ~1) + 2 * q; j < hi; j += 2 * Q) {
        float ra, rb;
        r2_pair(ld_f2(&S.sx[j]), ld_f2(&S.sy[j]), ld_f2(&S.sz[j]), PX, PY, PZ, ra, rb);
        if (j < lo) ra = 3.0e38f;      // the pair straddles the segment start
        if (j + 1 >= hi) rb = 3.0e38f; // ... or its end
        append_if(lptr, ra, rc2, (unsigned)j);
        append_if(lptr, rb, rc2, (unsigned)(j + 1));
    }
}

// Warp-local evaluation of the 32 lanes' lists (owner of lane k's list = s_i of lane k).
template <bool RECORD, int KMODE>
__device__ __forceinline__ void warp_pairs(ForceCellSmem &S, int lane, int warp, int tid, int cnt, int s_i,
                                           const PairP &pp, const FixP &fx, uint32_t ks, PairRec &rec, int *err)
{
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    const int excl = incl - cnt;
    const unsigned nz = __ballot_sync(0xffffffffu, cnt > 0);
    const int nown = __popc(nz);
    if (cnt > 0) {
        const int rk = __popc(nz & lanemask_lt());
        S.wexcl[warp][rk] = excl;
        S.wsi[warp][rk] = s_i;
        S.wrow[warp][rk] = tid * FC_LSTRIDE - excl;
    }
    if (lane == 0) S.wexcl[warp][nown] = total;
    __syncwarp();
    const int C = (total + 31) >> 5;
    const int t0 = min(lane * C, total), t1 = min(t0 + C, total);
    if (t0 < t1) {
        int o = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
            if (o + step < nown && S.wexcl[warp][o + step] <= t0) o += step;
        int enext = S.wexcl[warp][o + 1];
        int si = S.wsi[warp][o];
        int lrow = S.wrow[warp][o];
        float4 pi = ldp_c(S, si), vi = S.sv[si];
        int fxi = 0, fyi = 0, fzi = 0;
        for (int t = t0; t < t1; ++t) {
            if (t >= enext) { // next owner (never empty): flush the i-side sum
                atomicAdd(&S.acc[0][si], fxi);
                atomicAdd(&S.acc[1][si], fyi);
                atomicAdd(&S.acc[2][si], fzi);
                fxi = fyi = fzi = 0;
                ++o;
                enext = S.wexcl[warp][o + 1];
                si = S.wsi[warp][o];
                lrow = S.wrow[warp][o];
                pi = ldp_c(S, si);
                vi = S.sv[si];
            }
            const int j = S.lst[lrow + t];
            const float4 pj = ldp_c(S, j);
            float dx, dy, dz;
            const float s = pair_core_c<KMODE>(pp, pi, vi, pj, S.sv[j], ks, dx, dy, dz);
            pair_checks_c<RECORD>(pp, fx, pi, pj, s, dx, dy, dz, ks, rec, err);
            const int qx = to_fixed(s * dx, fx.scale), qy = to_fixed(s * dy, fx.scale),
                      qz = to_fixed(s * dz, fx.scale);
            fxi += qx;
            fyi += qy;
            fzi += qz;
            atomicAdd(&S.acc[0][j], -qx);
            atomicAdd(&S.acc[1][j], -qy);
            atomicAdd(&S.acc[2][j], -qz);
        }
        atomicAdd(&S.acc[0][si], fxi);
        atomicAdd(&S.acc[1][si], fyi);
        atomicAdd(&S.acc[2][si], fzi);
    }
    __syncwarp();
}

template <bool RECORD, int KMODE>
__global__ void __launch_bounds__(FC_NTHR, 3)
    k_force_cells(const float4 *__restrict__ pos, const float4 *__restrict__ vel, float4 *__restrict__ frc,
                  const int *__restrict__ start, Geom g, PairP pp, FixP fx, uint32_t s_lo, uint32_t s_hi,
                  PairRec rec, int *err)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ForceCellSmem &S = *reinterpret_cast<ForceCellSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ks = step_key(s_lo, s_hi, pp.seed_lo, pp.seed_hi);

    // ---- tile geometry: every thread decodes blockIdx ----------------------------------
    const int ntx = (g.n[0] + FT_BX - 1) / FT_BX, nty = (g.n[1] + FT_BY - 1) / FT_BY;
    const int x0 = (blockIdx.x % ntx) * FT_BX, y0 = ((blockIdx.x / ntx) % nty) * FT_BY,
              z0 = (blockIdx.x / (ntx * nty)) * FT_BZ;
    if (tid == 0) S.next_task = 0; // read only after the barriers below
    const int bx = min(FT_BX, g.n[0] - x0), by = min(FT_BY, g.n[1] - y0), bz = min(FT_BZ, g.n[2] - z0);
    const int sxa = bx + 2, sya = by + 2, sza = bz + 1;
    const int nsc = sxa * sya * sza;

    // ---- 1a. staged cell table --------------------------------------------------------
    for (int row = warp; row < sya * sza; row += FC_NWARP) {
        const int lz = row >= 2 * sya ? 2 : (row >= sya ? 1 : 0);
        const int ly = row - lz * sya;
        const int gy = ext_coord(y0 - 1 + ly, g.n[1], g.split[1]);
        const int gz = ext_coord(z0 + lz, g.n[2], g.split[2]);
        if (lane < sxa) {
            const int gx = ext_coord(x0 - 1 + lane, g.n[0], g.split[0]);
            const int gc = gx + g.ext[0] * (gy + g.ext[1] * gz);
            const int a = start[gc];
            const int c = row * sxa + lane;
            S.cgs[c] = a;
            S.soff[c] = start[gc + 1] - a;
        }
    }
    __syncthreads();
    if (warp == 0) {
        constexpr int PER = (FT_NSC + 31) / 32;
        int v[PER], sum = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int c = lane * PER + k;
            v[k] = c < nsc ? S.soff[c] : 0;
            sum += v[k];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int run = incl - sum;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int c = lane * PER + k;
            if (c < nsc) S.soff[c] = run;
            run += v[k];
        }
        if (lane == 31) {
            S.soff[nsc] = incl;
            S.total = incl;
        }
    }
    __syncthreads();
    const int total = S.total;
    if (total > FC_SCAP) {
        if (tid == 0) atomicAdd(&err[4], 1); // fallback statistics
        tile_fallback<RECORD, KMODE>(pos, vel, frc, start, g, pp, fx, round_keys(ks), rec, err, x0, y0, z0, bx, by, bz, 1.0f);
        return;
    }

    // ---- 1b. stage rows (<= 3 contiguous global segments each) -------------------------
    for (int row = warp; row < sya * sza; row += FC_NWARP) {
        const int lz = row >= 2 * sya ? 2 : (row >= sya ? 1 : 0);
        const int ly = row - lz * sya;
        const int gy = y0 - 1 + ly, gz = z0 + lz;
        const float sy = g.split[1] ? 0.0f : (gy < 0 ? -g.L[1] : (gy >= g.n[1] ? g.L[1] : 0.0f));
        const float sz = g.split[2] ? 0.0f : (gz >= g.n[2] ? g.L[2] : 0.0f);
        const int c0 = sxa * row;
        const bool wrap_lo = !g.split[0] && x0 == 0, wrap_hi = !g.split[0] && x0 + bx == g.n[0];
        const float sxl = wrap_lo ? -g.L[0] : 0.0f, sxh = wrap_hi ? g.L[0] : 0.0f;
        const int a0 = S.soff[c0], b0 = S.soff[c0 + 1], c0s = S.soff[c0 + bx + 1], e0 = S.soff[c0 + bx + 2];
        const int mlo = wrap_lo ? b0 : a0, mhi = wrap_hi ? c0s : e0;
        const int gm = wrap_lo ? S.cgs[c0 + 1] : S.cgs[c0];
        for (int s = a0 + lane; s < e0; s += 32) {
            int gi;
            float sx = 0.0f;
            if (s < mlo) {
                gi = S.cgs[c0] + (s - a0);
                sx = sxl;
            } else if (s < mhi) {
                gi = gm + (s - mlo);
            } else {
                gi = S.cgs[c0 + bx + 1] + (s - c0s);
                sx = sxh;
            }
            const float4 p = pos[gi];
            S.sx[s] = p.x + sx;
            S.sy[s] = p.y + sy;
            S.sz[s] = p.z + sz;
            S.sid[s] = __float_as_int(p.w);
            S.sv[s] = vel[gi];
            S.acc[0][s] = 0;
            S.acc[1][s] = 0;
            S.acc[2][s] = 0;
        }
    }
    __syncthreads();

    // ---- 2 + 3. warp per home cell: strided sweep into short lists, then warp-local pairs --
    const int nhc = bx * by * bz;
    const int rowz = sxa * sya;
    const unsigned lbase = (unsigned)__cvta_generic_to_shared(&S.lst[tid * FC_LSTRIDE]);
    while (true) {
        int task = 0;
        if (lane == 0) task = atomicAdd(&S.next_task, 1);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task >= nhc) break;
        const int lx = 1 + task % bx, ly = 1 + (task / bx) % by, lz = task / (bx * by);
        const int c = lx + sxa * (ly + sya * lz);
        const int cs0 = S.soff[c], ce0 = S.soff[c + 1];
        const int nc = ce0 - cs0;
        if (nc == 0) continue;
        const int Q = nc <= 32 ? 32 / nc : 1; // lanes per particle
        const int ppw = 32 / Q;               // particles per pass
        const int c1 = c - 1 + sxa;           // (lx - 1, ly + 1, lz)
        for (int pbase = 0; pbase < nc; pbase += ppw) {
            const int pl = lane / Q, q = lane % Q;
            const bool act = pl < ppw && pbase + pl < nc;
            const int al = pbase + pl; // slot within the cell
            const int s_i = act ? cs0 + al : cs0;
            const float px = S.sx[s_i], py = S.sy[s_i], pz = S.sz[s_i];
            // own-cell circular forward half: slot al takes al+1 .. al+hh (mod nc)
            const int hh = (nc & 1) ? (nc - 1) >> 1 : ((al < (nc >> 1)) ? (nc >> 1) : (nc >> 1) - 1);
            const int own_end = s_i + 1 + hh;
            unsigned lptr = lbase;
            bool full = false;
#pragma unroll 1
            for (int k = 0; k < 7; ++k) {
                int a, b;
                if (k == 0) {
                    a = s_i + 1;
                    b = min(own_end, ce0);
                } else if (k == 1) {
                    a = cs0;
                    b = cs0 + max(0, own_end - ce0);
                } else if (k == 2) {
                    a = ce0;
                    b = S.soff[c + 2];
                } else {
                    const int cs = (k == 3) ? c1 : c1 - 2 * sxa + rowz + (k - 4) * sxa;
                    a = S.soff[cs];
                    b = S.soff[cs + 3];
                }
                if (!act) b = a;
                // this lane examines at most ceil((b - a) / Q) + 2 candidates of the segment
                const int worst = (b - a + Q - 1) / Q + 2;
                if ((int)((lptr - lbase) >> 1) + worst > FC_LCAP) full = true;
                if (!full) {
                    sweep_strided(S, lptr, a, b, q, Q, px, py, pz, pp.rc2);
                } else if (a < b) {
                    // list could overflow (crowded cell, rare): evaluate this lane's share in place
                    const float4 pi = ldp_c(S, s_i), vi = S.sv[s_i];
                    for (int j = (a & ~1) + 2 * q; j < b; j += 2 * Q) {
#pragma unroll
                        for (int h2 = 0; h2 < 2; ++h2) {
                            const int jj = j + h2;
                            if (jj < a || jj >= b) continue;
                            const float ddx = px - S.sx[jj], ddy = py - S.sy[jj], ddz = pz - S.sz[jj];
                            if (!(ddx * ddx + ddy * ddy + ddz * ddz < pp.rc2)) continue;
                            const float4 pj = ldp_c(S, jj);
                            float dx, dy, dz;
                            const float s = pair_core_c<KMODE>(pp, pi, vi, pj, S.sv[jj], ks, dx, dy, dz);
                            pair_checks_c<RECORD>(pp, fx, pi, pj, s, dx, dy, dz, ks, rec, err);
                            const int qx = to_fixed(s * dx, fx.scale), qy = to_fixed(s * dy, fx.scale),
                                      qz = to_fixed(s * dz, fx.scale);
                            atomicAdd(&S.acc[0][s_i], qx);
                            atomicAdd(&S.acc[1][s_i], qy);
                            atomicAdd(&S.acc[2][s_i], qz);
                            atomicAdd(&S.acc[0][jj], -qx);
                            atomicAdd(&S.acc[1][jj], -qy);
                            atomicAdd(&S.acc[2][jj], -qz);
                        }
                    }
                }
            }
            if (full && act) atomicAdd(&err[6], 1); // statistics: in-place evaluations
            const int cnt = (int)((lptr - lbase) >> 1);
            __syncwarp();
            warp_pairs<RECORD, KMODE>(S, lane, warp, tid, cnt, s_i, pp, fx, ks, rec, err);
        }
    }
    __syncthreads();

    // ---- 5. flush (rows map back to <= 3 contiguous global segments) ----------------------
    for (int row = warp; row < sya * sza; row += FC_NWARP) {
        const int c0 = sxa * row;
        const int a0 = S.soff[c0], b0 = S.soff[c0 + 1], c0s = S.soff[c0 + bx + 1], e0 = S.soff[c0 + bx + 2];
        const bool wrap_lo = !g.split[0] && x0 == 0, wrap_hi = !g.split[0] && x0 + bx == g.n[0];
        const int mlo = wrap_lo ? b0 : a0, mhi = wrap_hi ? c0s : e0;
        const int gm = wrap_lo ? S.cgs[c0 + 1] : S.cgs[c0];
        for (int s = a0 + lane; s < e0; s += 32) {
            const int gi = (s < mlo) ? S.cgs[c0] + (s - a0)
                                     : (s < mhi ? gm + (s - mlo) : S.cgs[c0 + bx + 1] + (s - c0s));
            const int qx = S.acc[0][s], qy = S.acc[1][s], qz = S.acc[2][s];
            if (qx | qy | qz)
                atomicAdd(&frc[gi], make_float4((float)qx * fx.inv_scale, (float)qy * fx.inv_scale,
                                                (float)qz * fx.inv_scale, 0.0f));
        }
    }
}

} // namespace dpd
