// dpd_force_tile.cuh -- production pair-force sweep for sm_100a.
//
// One CTA per tile of BX x BY x BZ home cells (cell lists, symmetric forces):
//   1. stage   : the tile's forward half-stencil region, (BX+2) x (BY+2) x (BZ+1) cells,
//                is copied row by row (contiguous global ranges) into shared memory, with
//                periodic images pre-shifted into the tile frame;
//   2. scan    : each lane owns one home particle i and sweeps its 5 contiguous smem
//                segments (own cell after i + next cell, the y+1 row, three z+1 rows),
//                appending in-cutoff j to a private list -- 2 predicated instructions per
//                candidate, no divergent pair body;
//   3. pairs   : the warp evaluates the concatenated lists 32 pairs at a time (full SIMT
//                efficiency), the owner lane found by a shuffle binary search over the
//                list prefix sums;
//   4. accumulate: f is quantised once to 32-bit fixed point and added with native
//                shared-memory integer atomics (+q on i, -q on j): exact Newton-3,
//                order-independent sums;
//   5. flush   : every staged particle's sum is converted back to fp32 and added to the
//                global force array with one vector reduction (REDG.F32x4).
#pragma once

#include "dpd_kernels.cuh"

namespace dpd {

constexpr int FT_BX = 4, FT_BY = 4, FT_BZ = 2;
constexpr int FT_SX = FT_BX + 2, FT_SY = FT_BY + 2, FT_SZ = FT_BZ + 1;
constexpr int FT_NSC = FT_SX * FT_SY * FT_SZ; // staged cells (108)
constexpr int FT_NROW = FT_SY * FT_SZ;        // staged rows (18)
constexpr int FT_NHROW = FT_BY * FT_BZ;       // home rows (8)
constexpr int FT_NTHR = 288;                 // > mean home count (256): no straggler rounds
constexpr int FT_SCAP = 1280;                 // staged particles (mean 864 at rho = 8)
constexpr int FT_LCAP = 48;                   // per-lane pair-list capacity
constexpr int FT_LSTRIDE = FT_LCAP + 2;       // 25 words per lane (odd): conflict-free appends
constexpr int FT_NWARP = FT_NTHR / 32;

// Fixed-point force quantisation: q = rint(f * scale), |f * scale| < 2^21 enforced.
struct FixP {
    float scale;     // 2^k
    float inv_scale; // 2^-k
    float mag_lim;   // 2^21 / scale: larger pair magnitudes raise ERR_RANGE
};

struct ForceTileSmem {
    float4 sp[FT_SCAP];                        // staged positions (tile frame), w = id bits
    float4 sv[FT_SCAP];                        // staged velocities
    float sx[FT_SCAP], sy[FT_SCAP], sz[FT_SCAP]; // SoA copy of the positions for the f32x2 sweep
    int acc[3][FT_SCAP];                       // fixed-point force sums
    int gidx[FT_SCAP];                         // slot in the global sorted arrays
    unsigned short lst[FT_NTHR * FT_LSTRIDE];  // per-lane pair lists (lane-major, padded)
    int soff[FT_NSC + 1];                      // staged cell -> smem start (exclusive scan)
    int cgs[FT_NSC];                           // staged cell -> global start
    int hoff[FT_NHROW + 1];                    // home row -> first home index (prefix)
    int wexcl[FT_NWARP][33];                   // per-warp list prefix sums (+ total)
    int wsi[FT_NWARP][32];                     // per-warp owner smem indices
    int total;
};

__device__ __forceinline__ int to_fixed(float f, float scale)
{
    // round-to-nearest via the 1.5 * 2^23 magic constant; valid for |f * scale| < 2^22
    return __float_as_int(__fmaf_rn(f, scale, 12582912.0f)) - 0x4B400000;
}

// Pair-list evaluation for one warp.  Lanes hold (cnt, s_i) of their own home particle; the
// 32 lists form one flat sequence of `total` pairs, cut into 32 contiguous chunks of
// C = ceil(total / 32): lane k evaluates entries [k C, (k+1) C).  A chunk spans one or two
// owners, so the i-side sum stays in registers and is flushed with one atomic per owner
// change, and in any iteration the 32 lanes touch 32 different owners (no same-address
// atomics).  The j side is one fixed-point shared atomic per component.
template <bool RECORD, int KMODE>
__device__ __forceinline__ void tile_pairs(ForceTileSmem &S, int lane, int tid, int cnt, int s_i, const PairP &pp,
                                           const FixP &fx, uint32_t ks, PairRec &rec, int *err)
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
    const int wbase = tid - lane;
    const int warp = tid >> 5;
    S.wexcl[warp][lane] = excl;
    S.wsi[warp][lane] = s_i;
    if (lane == 0) S.wexcl[warp][32] = total;
    const int C = (total + 31) >> 5;
    const int t0 = lane * C;
    const int t1 = min(t0 + C, total);
    // owner of t0: largest lane o with excl_o <= t0
    int o = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
        const int e = __shfl_sync(0xffffffffu, excl, o + step);
        if (e <= t0) o += step;
    }
    __syncwarp();
    int eo = S.wexcl[warp][o], enext = S.wexcl[warp][o + 1];
    int si = S.wsi[warp][o];
    float4 pi = S.sp[si], vi = S.sv[si];
    int fx_i = 0, fy_i = 0, fz_i = 0;
    for (int r = 0; r < C; ++r) {
        const int t = t0 + r;
        if (t >= t1) break;
        if (t >= enext) { // next owner: flush the i-side sum
            atomicAdd(&S.acc[0][si], fx_i);
            atomicAdd(&S.acc[1][si], fy_i);
            atomicAdd(&S.acc[2][si], fz_i);
            fx_i = fy_i = fz_i = 0;
            eo = enext;
            ++o;
            enext = S.wexcl[warp][o + 1];
            while (enext <= t) { // skip owners with empty lists (rare)
                ++o;
                enext = S.wexcl[warp][o + 1];
            }
            si = S.wsi[warp][o];
            pi = S.sp[si];
            vi = S.sv[si];
        }
        const int j = S.lst[(wbase + o) * FT_LSTRIDE + (t - eo)];
        const float4 pj = S.sp[j], vj = S.sv[j];
        const float dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
        const float r2 = dx * dx + dy * dy + dz * dz;
        const float dvdot = dx * (vi.x - vj.x) + dy * (vi.y - vj.y) + dz * (vi.z - vj.z);
        const uint32_t idi = (uint32_t)__float_as_int(pi.w), idj = (uint32_t)__float_as_int(pj.w);
        float s = 0.0f;
        if (r2 > 0.0f) {
            s = pair_scalar<KMODE>(pp, r2, dvdot, idi, idj, ks);
            if (fabsf(s) * (r2 * rsqrtf(r2)) > fx.mag_lim) raise_err(err, ERR_RANGE, (int)idi);
            if constexpr (RECORD) {
                const unsigned long long k = atomicAdd(rec.count, 1ull);
                if ((long long)k < rec.cap) {
                    const uint2 wd = pair_words(idi, idj, ks);
                    rec.quad[k] = make_uint4(min(idi, idj), max(idi, idj), wd.x, wd.y);
                }
            }
        }
        const int qx = to_fixed(s * dx, fx.scale);
        const int qy = to_fixed(s * dy, fx.scale);
        const int qz = to_fixed(s * dz, fx.scale);
        fx_i += qx;
        fy_i += qy;
        fz_i += qz;
        atomicAdd(&S.acc[0][j], -qx); // native ATOMS.ADD (the fp32 variant is a CAS loop)
        atomicAdd(&S.acc[1][j], -qy);
        atomicAdd(&S.acc[2][j], -qz);
    }
    if (t0 < t1) {
        atomicAdd(&S.acc[0][si], fx_i);
        atomicAdd(&S.acc[1][si], fy_i);
        atomicAdd(&S.acc[2][si], fz_i);
    }
    __syncwarp();
}

// Candidate sweep helpers.  The list pointer `lptr` is a shared-memory byte address; an
// in-cutoff candidate j costs one predicated 16-bit store and one predicated add.
__device__ __forceinline__ void append_if(unsigned &lptr, float r2, float rc2, unsigned j)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, %2;\n\t@p st.shared.u16 [%0], %3;\n\t"
                 "@p add.u32 %0, %0, 2;\n\t}"
                 : "+r"(lptr)
                 : "f"(r2), "f"(rc2), "r"(j)
                 : "memory");
}

__device__ __forceinline__ unsigned long long f2dup(float a)
{
    const unsigned long long u = __float_as_uint(a);
    return (u << 32) | u;
}

__device__ __forceinline__ unsigned long long ld_f2(const float *p)
{
    return *reinterpret_cast<const unsigned long long *>(p);
}

// r2 of two candidates at once with packed fp32x2 arithmetic (FADD2/FMUL2/FFMA2).
__device__ __forceinline__ void r2_pair(unsigned long long X, unsigned long long Y, unsigned long long Z,
                                        unsigned long long PX, unsigned long long PY, unsigned long long PZ,
                                        float &ra, float &rb)
{
    unsigned long long dx, dy, dz, r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(PX), "l"(X));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(PY), "l"(Y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(PZ), "l"(Z));
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r) : "l"(dx));
    asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r) : "l"(dy));
    asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(r) : "l"(dz));
    ra = __uint_as_float((unsigned)r);
    rb = __uint_as_float((unsigned)(r >> 32));
}

__device__ __forceinline__ float r2_one(const ForceTileSmem &S, int j, float px, float py, float pz)
{
    const float dx = px - S.sx[j], dy = py - S.sy[j], dz = pz - S.sz[j];
    return dx * dx + dy * dy + dz * dz;
}

// Sweep of one contiguous smem segment [lo, hi): append every in-cutoff j.
__device__ __forceinline__ void sweep(const ForceTileSmem &S, unsigned &lptr, int lo, int hi, float px, float py,
                                      float pz, float rc2)
{
    int j = lo;
    if ((j & 1) && j < hi) {
        append_if(lptr, r2_one(S, j, px, py, pz), rc2, (unsigned)j);
        ++j;
    }
    const unsigned long long PX = f2dup(px), PY = f2dup(py), PZ = f2dup(pz);
    for (; j + 1 < hi; j += 2) {
        float ra, rb;
        r2_pair(ld_f2(&S.sx[j]), ld_f2(&S.sy[j]), ld_f2(&S.sz[j]), PX, PY, PZ, ra, rb);
        append_if(lptr, ra, rc2, (unsigned)j);
        append_if(lptr, rb, rc2, (unsigned)(j + 1));
    }
    if (j < hi) append_if(lptr, r2_one(S, j, px, py, pz), rc2, (unsigned)j);
}

// Contiguous copy of global particles [g0, g0 + len) to smem [s0, s0 + len) with a shift.
__device__ __forceinline__ void stage_segment(ForceTileSmem &S, const float4 *__restrict__ pos,
                                              const float4 *__restrict__ vel, int g0, int s0, int len, float sx,
                                              float sy, float sz, int lane)
{
    for (int k = lane; k < len; k += 32) {
        const float4 p = pos[g0 + k];
        const int s = s0 + k;
        const float px = p.x + sx, py = p.y + sy, pz = p.z + sz;
        S.sp[s] = make_float4(px, py, pz, p.w);
        S.sx[s] = px;
        S.sy[s] = py;
        S.sz[s] = pz;
        S.sv[s] = vel[g0 + k];
        S.gidx[s] = g0 + k;
        S.acc[0][s] = 0;
        S.acc[1][s] = 0;
        S.acc[2][s] = 0;
    }
}

template <bool RECORD, int KMODE>
__global__ void __launch_bounds__(FT_NTHR, 2)
    k_force_tile(const float4 *__restrict__ pos, const float4 *__restrict__ vel, float4 *__restrict__ frc,
                 const int *__restrict__ start, Geom g, PairP pp, FixP fx, uint32_t s_lo, uint32_t s_hi,
                 PairRec rec, int *err)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ForceTileSmem &S = *reinterpret_cast<ForceTileSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // ---- tile geometry ---------------------------------------------------------------
    const int ntx = (g.n[0] + FT_BX - 1) / FT_BX, nty = (g.n[1] + FT_BY - 1) / FT_BY;
    const int tx = blockIdx.x % ntx, ty = (blockIdx.x / ntx) % nty, tz = blockIdx.x / (ntx * nty);
    const int x0 = tx * FT_BX, y0 = ty * FT_BY, z0 = tz * FT_BZ;
    const int bx = min(FT_BX, g.n[0] - x0), by = min(FT_BY, g.n[1] - y0), bz = min(FT_BZ, g.n[2] - z0);
    const int sxa = bx + 2, sya = by + 2, sza = bz + 1;
    const int nsc = sxa * sya * sza;

    // ---- 1a. staged cell table (counts, then one-warp exclusive scan) -----------------
    for (int c = tid; c < nsc; c += FT_NTHR) {
        const int lx = c % sxa, ly = (c / sxa) % sya, lz = c / (sxa * sya);
        int gx = x0 - 1 + lx, gy = y0 - 1 + ly, gz = z0 + lz;
        gx += (gx < 0) ? g.n[0] : (gx >= g.n[0] ? -g.n[0] : 0);
        gy += (gy < 0) ? g.n[1] : (gy >= g.n[1] ? -g.n[1] : 0);
        gz += (gz >= g.n[2]) ? -g.n[2] : 0;
        const int gc = gx + g.ext[0] * (gy + g.ext[1] * gz);
        const int a = start[gc];
        S.cgs[c] = a;
        S.soff[c] = start[gc + 1] - a;
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
    if (total > FT_SCAP) {
        if (tid == 0) raise_err(err, ERR_CAPACITY, total);
        return;
    }
    if (warp == 1 && lane == 0) {
        // home rows (ly = 1..by, lz = 0..bz-1), cells lx = 1..bx: prefix of their sizes
        int run = 0;
        for (int r = 0; r < by * bz; ++r) {
            const int ly = 1 + r % by, lz = r / by;
            const int c = 1 + sxa * (ly + sya * lz);
            S.hoff[r] = run;
            run += S.soff[c + bx] - S.soff[c];
        }
        S.hoff[by * bz] = run;
    }

    // ---- 1b. stage rows: each row is <= 3 contiguous global segments -----------------
    for (int row = warp; row < sya * sza; row += FT_NWARP) {
        const int ly = row % sya, lz = row / sya;
        const int gy = y0 - 1 + ly, gz = z0 + lz;
        const float sy = gy < 0 ? -g.L[1] : (gy >= g.n[1] ? g.L[1] : 0.0f);
        const float sz = gz >= g.n[2] ? g.L[2] : 0.0f;
        const int c0 = sxa * row; // lx = 0
        const bool wrap_lo = (x0 == 0), wrap_hi = (x0 + bx == g.n[0]);
        const float sxl = wrap_lo ? -g.L[0] : 0.0f, sxh = wrap_hi ? g.L[0] : 0.0f;
        // segment A: lx = 0; B: lx = 1..bx; C: lx = bx + 1 (merged when not wrapped)
        const int a0 = S.soff[c0], b0 = S.soff[c0 + 1], c0s = S.soff[c0 + bx + 1], e0 = S.soff[c0 + bx + 2];
        if (wrap_lo) stage_segment(S, pos, vel, S.cgs[c0], a0, b0 - a0, sxl, sy, sz, lane);
        const int mlo = wrap_lo ? b0 : a0;
        const int mhi = wrap_hi ? c0s : e0;
        const int gm = wrap_lo ? S.cgs[c0 + 1] : S.cgs[c0];
        stage_segment(S, pos, vel, gm, mlo, mhi - mlo, 0.0f, sy, sz, lane);
        if (wrap_hi) stage_segment(S, pos, vel, S.cgs[c0 + bx + 1], c0s, e0 - c0s, sxh, sy, sz, lane);
    }
    __syncthreads();

    // ---- 2 + 3. per-lane candidate sweep, then warp-balanced pair evaluation ----------
    const uint32_t ks = step_key(s_lo, s_hi, pp.seed_fold);
    const int nhome = S.hoff[by * bz];
    const unsigned lbase = (unsigned)__cvta_generic_to_shared(&S.lst[tid * FT_LSTRIDE]);
    const int rowz = sxa * sya;
    for (int h0 = warp * 32; h0 < nhome; h0 += FT_NTHR) {
        const int h = h0 + lane;
        int s_i = 0, cnt = 0;
        int lo[5], hi[5];
        float4 pi = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 5; ++k) lo[k] = hi[k] = 0;
        if (h < nhome) {
            int r = 0;
            while (r + 1 < by * bz && S.hoff[r + 1] <= h) ++r;
            const int ly = 1 + r % by, lz = r / by;
            const int crow = sxa * (ly + sya * lz);
            s_i = S.soff[crow + 1] + (h - S.hoff[r]);
            int lx = 1;
            while (lx < bx && S.soff[crow + lx + 1] <= s_i) ++lx;
            const int c = crow + lx;
            pi = S.sp[s_i];
            lo[0] = s_i + 1;
            hi[0] = S.soff[c + 2];
            const int c1 = (lx - 1) + sxa * (ly + 1) + rowz * lz;
            lo[1] = S.soff[c1];
            hi[1] = S.soff[c1 + 3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int c2 = (lx - 1) + sxa * (ly - 1 + d) + rowz * (lz + 1);
                lo[2 + d] = S.soff[c2];
                hi[2 + d] = S.soff[c2 + 3];
            }
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            int a = lo[k];
            const int b = hi[k];
            // chunks of at most FT_LCAP candidates; evaluate the lists early if they could
            // overflow (rare at rho = 8: a segment holds ~24 candidates)
            while (__any_sync(0xffffffffu, a < b)) {
                const int e = min(b, a + FT_LCAP);
                if (__any_sync(0xffffffffu, cnt + (e - a) > FT_LCAP)) {
                    __syncwarp();
                    tile_pairs<RECORD, KMODE>(S, lane, tid, cnt, s_i, pp, fx, ks, rec, err);
                    cnt = 0;
                    __syncwarp();
                }
                unsigned lptr = lbase + 2u * (unsigned)cnt;
                sweep(S, lptr, a, e, pi.x, pi.y, pi.z, pp.rc2);
                cnt = (int)(lptr - lbase) >> 1;
                a = e;
            }
        }
        __syncwarp();
        tile_pairs<RECORD, KMODE>(S, lane, tid, cnt, s_i, pp, fx, ks, rec, err);
        __syncwarp();
    }
    __syncthreads();

    // ---- 5. flush: fixed point -> fp32, one vector reduction per staged particle -------
    for (int s = tid; s < total; s += FT_NTHR) {
        const int qx = S.acc[0][s], qy = S.acc[1][s], qz = S.acc[2][s];
        if (qx | qy | qz)
            atomicAdd(&frc[S.gidx[s]], make_float4((float)qx * fx.inv_scale, (float)qy * fx.inv_scale,
                                                   (float)qz * fx.inv_scale, 0.0f));
    }
}

} // namespace dpd
