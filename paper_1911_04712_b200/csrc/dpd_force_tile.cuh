// dpd_force_tile.cuh -- production pair-force sweep for sm_100a.
//
// One CTA of 9 warps per tile of BX x BY x BZ home cells (cell lists, symmetric
// forces), 3 tiles resident per SM (74 KB shared memory, 72 registers); launched on a 3D grid,
// one CTA per tile:
//   1. table   : one warp loads the staged cell table of the forward half-stencil region,
//                (BX+2) x (BY+2) x (BZ+1) cells, straight from the cell starts and scans it
//                (one extra entry per row: the row's end); another warp scans the home rows;
//   2. stage   : every staged row (<= 3 contiguous global ranges) is copied with cp.async.cg,
//                then shifted to the periodic image in the tile frame and split into SoA
//                x, y, z; the particle id rides in the staged velocity's w word; every row is
//                followed by FT_GAP far-away sentinels;
//   3. sweep   : one home particle per lane; its first own-cell block (masked, j > i) is
//                peeled, then one loop walks a queue of its segments -- the y+1 row and the
//                three z+1 rows first (lanes of one cell in lockstep: their candidate quads
//                are the same shared-memory addresses), the rest of the own cell last -- in
//                unmasked 4-aligned blocks: a block running past a segment meets cells two
//                away or sentinels, both beyond r_c.  One LDS.128 per coordinate, packed
//                fp32x2 distance math (FADD2/FFMA2), one predicated 16-bit store + add per hit;
//   4. pairs   : phase A -- every lane walks the first FT_PHASEA entries of its own list
//                (owner = its home particle, no owner switches); phase B -- the leftovers of
//                the warp's lists are concatenated and cut into 32 contiguous lane chunks,
//                each walked by one cursor; the i-side sum stays in registers until the
//                owner changes;
//   5. accumulate: a, gamma, sigma are pre-scaled by the power-of-two fixed-point scale, so
//                one FFMA quantises each force component; native shared-memory integer
//                atomics (+q on i, -q on j): exact Newton-3, order-independent sums;
//   6. flush   : every staged particle's sum is converted back to fp32 and added to the
//                global force array with one vector reduction (REDG.F32x4).
// Tiles whose particle counts exceed the shared-memory capacities (never seen at rho = 8,
// > 9 sigma) are evaluated by a direct global-memory fallback with the same pair function.
// DESIGN.md §6 records the measured history of every choice.
#pragma once

#include "dpd_kernels.cuh"

namespace dpd {

constexpr int FT_BX = 4, FT_BY = 4, FT_BZ = 2;
constexpr int FT_SX = FT_BX + 2, FT_SY = FT_BY + 2, FT_SZ = FT_BZ + 1;
constexpr int FT_NSC = FT_SX * FT_SY * FT_SZ; // staged cells (108)

constexpr int FT_NHROW = FT_BY * FT_BZ;       // home rows (8)
#ifndef FT_NTHR_DEF
#define FT_NTHR_DEF 288
#endif
constexpr int FT_NTHR = FT_NTHR_DEF;          // 9 warps: ~28 home particles each (balanced ranges)
constexpr int FT_NWARP = FT_NTHR / 32;
constexpr int FT_GAP = 3;                     // far-away sentinel slots after every staged row
constexpr int FT_ROWPAD = 1;                  // one extra table entry per staged row: the row's end
constexpr int FT_SCAP = 1088;                 // staged particles + 18 row gaps (mean 864 + 54, sd 29)
constexpr int FT_HCAP = 352;                  // home particles (mean 256, sd 16)
#ifndef FT_LCAP_DEF
#define FT_LCAP_DEF 40
#endif
constexpr int FT_LCAP = FT_LCAP_DEF;                 // hits per home particle (mean 16.8, sd 4.1)
constexpr int FT_LSTRIDE = FT_LCAP + 2;       // 21 words per list (odd): conflict-free appends
#ifndef FT_NCUR_DEF
#define FT_NCUR_DEF 1
#endif
constexpr int FT_NCUR = FT_NCUR_DEF;          // independent pair chains per lane (ILP)
#ifndef FT_MINB
#define FT_MINB 3                             // resident tiles per SM (register budget)
#endif
constexpr float FT_FAR = 1.0e18f;             // sentinel coordinate (its r^2 ~ 3e36 stays finite)
constexpr int FT_WSTRIDE = 34;                // per-warp owner-table stride (32 owners + sentinel)
#ifndef FT_PA_UNROLL
#define FT_PA_UNROLL 1
#endif
#ifndef FT_SW_UNROLL
#define FT_SW_UNROLL 1
#endif
#ifndef FT_PA2
#define FT_PA2 1
#endif
#ifndef FT_PAW
#define FT_PAW 2 // phase-A entries per iteration (FT_PA2)
#endif
constexpr int kFtPaUnroll = FT_PA_UNROLL;     // unroll of the phase-A pair loop (1: none)
constexpr int kFtSwUnroll = FT_SW_UNROLL;     // unroll of the sweep loop (1: none)

// Fixed-point force quantisation: q = rint(f * scale), |f * scale| < 2^21 enforced.
struct FixP {
    float scale;     // 2^k
    float inv_scale; // 2^-k
    float mag_lim;   // 2^21 / scale: larger pair magnitudes raise ERR_RANGE
    float slack;     // row-end pruning: distance bounds are lowered by this much
};

// Cell table of one tile (SURVEY §8a row a5 staging): staged cell -> smem / global start,
// home rows -> first home index, staged particle count.
struct TileTab {
    int soff[(FT_SX + FT_ROWPAD) * FT_SY * FT_SZ + 1]; // staged cell -> smem start; with FT_ROWPAD the
                                                       // entry after a row's last cell is the row's end
    int cgs[(FT_SX + FT_ROWPAD) * FT_SY * FT_SZ];      // staged cell -> global start
    int hoff[FT_NHROW + 1]; // home row -> first home index (prefix)
    int rend[FT_SY * FT_SZ]; // staged row -> end of its particles (the sentinel gap follows)
    int total;            // staged particles
};

struct ForceTileSmem {
    float4 sv[FT_SCAP];                       // staged velocities; w: id bits | species << 30 (stage_fix)
    unsigned short lst[FT_NTHR * FT_LSTRIDE]; // per-thread pair lists (one home particle each);
                                              // during staging: the AoS landing buffer of the positions
    float sx[FT_SCAP], sy[FT_SCAP], sz[FT_SCAP]; // staged positions (tile frame), SoA
    int acc[3][FT_SCAP];                         // fixed-point force sums
    int4 wrec[FT_NWARP * FT_WSTRIDE];            // per warp, compacted owners: {list prefix, prefix + count,
                                                 //   list base minus prefix, staged index} (one LDS.128)
    TileTab tab[1];                              // the tile's cell table
    int nown;                                    // owners with a non-empty list
};

// Extended-grid coordinate of interior cell coordinate c in [-1, n]: split dimensions
// address their halo ring (index 0 / n + 1), periodic-local dimensions wrap.
__device__ __forceinline__ int ext_coord(int c, int n, int split)
{
    if (split) return c + 1;
    return c < 0 ? c + n : (c >= n ? c - n : c);
}

static_assert(sizeof(unsigned short) * FT_NTHR * FT_LSTRIDE >= sizeof(float4) * FT_SCAP,
              "the list area doubles as the position landing buffer");
static_assert(offsetof(ForceTileSmem, sx) % 16 == 0 && offsetof(ForceTileSmem, sy) % 16 == 0 &&
                  offsetof(ForceTileSmem, sz) % 16 == 0,
              "LDS.128 candidate quads");
static_assert(offsetof(ForceTileSmem, lst) % 16 == 0 && offsetof(ForceTileSmem, sx) % 8 == 0 &&
                  offsetof(ForceTileSmem, sy) % 8 == 0 && offsetof(ForceTileSmem, sz) % 8 == 0,
              "cp.async / packed-pair alignment");

// The staged velocity word w carries the particle's id (and, for the species matrix, its
// species in bits 30-31; ids stay below 2^30), so one LDS.128 fetches velocity and id.
template <int KMODE>
__device__ __forceinline__ uint32_t w_id(float w)
{
    return KMODE == 3 ? (__float_as_uint(w) & 0x3FFFFFFFu) : __float_as_uint(w);
}

__device__ __forceinline__ int w_species(float w)
{
    return (int)(__float_as_uint(w) >> 30);
}

// Staged particle j in the global-memory convention: position (x, y, z, id bits) and
// velocity (u_x, u_y, u_z, species bits) -- cold paths (record, in-place, fallback).
template <int KMODE>
__device__ __forceinline__ float4 ldp(const ForceTileSmem &S, int j)
{
    return make_float4(S.sx[j], S.sy[j], S.sz[j], __uint_as_float(w_id<KMODE>(S.sv[j].w)));
}

template <int KMODE>
__device__ __forceinline__ float4 ldv(const ForceTileSmem &S, int j)
{
    const float4 v = S.sv[j];
    return make_float4(v.x, v.y, v.z, __int_as_float(KMODE == 3 ? w_species(v.w) : 0));
}

// The tiled kernel's PairP is pre-scaled by FixP::scale (capi scaled_pair), so a pair scalar
// s is already in fixed-point units and q = rint(d * s) is one FFMA per component.
__device__ __forceinline__ int fix_q(float d, float s)
{
    return __float_as_int(__fmaf_rn(d, s, 12582912.0f)) - 0x4B400000;
}

// Pair-force accumulation: 32-bit fixed point in shared memory (exact Newton-3, order-
// independent tile sums, flushed once per staged particle; DESIGN §6.1 measures the fp32
// global-reduction alternative).
using AccT = int;
__device__ __forceinline__ AccT acc_q(float d, float s) { return fix_q(d, s); }

__device__ __forceinline__ int to_fixed(float f, float scale)
{
    // round-to-nearest via the 1.5 * 2^23 magic constant; valid for |f * scale| < 2^22
    return __float_as_int(__fmaf_rn(f, scale, 12582912.0f)) - 0x4B400000;
}

// ---------------------------------------------------------------------------------------
// Sweep helpers.  `lptr` is a shared-memory byte address into the particle's list; an
// in-cutoff candidate j costs one predicated 16-bit store and one predicated add.
// ---------------------------------------------------------------------------------------
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

// Append j if r2 < rc2 and lo <= j < hi (the masked end blocks of the aligned sweep).
__device__ __forceinline__ void append_if_in(unsigned &lptr, float r2, float rc2, unsigned j, int lo, int hi)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, %2;\n\tsetp.ge.and.s32 p, %3, %4, p;\n\t"
                 "setp.lt.and.s32 p, %3, %5, p;\n\t@p st.shared.u16 [%0], %3;\n\t@p add.u32 %0, %0, 2;\n\t}"
                 : "+r"(lptr)
                 : "f"(r2), "f"(rc2), "r"(j), "r"(lo), "r"(hi)
                 : "memory");
}

// Four candidates j..j+3 (j % 4 == 0): one LDS.128 per coordinate, packed r2.
__device__ __forceinline__ void r2_quad(const ForceTileSmem &S, int j, unsigned long long PX, unsigned long long PY,
                                        unsigned long long PZ, float &ra, float &rb, float &rc, float &rd)
{
    const ulonglong2 X = *reinterpret_cast<const ulonglong2 *>(&S.sx[j]);
    const ulonglong2 Y = *reinterpret_cast<const ulonglong2 *>(&S.sy[j]);
    const ulonglong2 Z = *reinterpret_cast<const ulonglong2 *>(&S.sz[j]);
    r2_pair(X.x, Y.x, Z.x, PX, PY, PZ, ra, rb);
    r2_pair(X.y, Y.y, Z.y, PX, PY, PZ, rc, rd);
}

// Asynchronous copy (LDGSTS, no register round trip) of global particles [g0, g0 + len)
// to smem [s0, s0 + len): every load of the tile is in flight before any is waited for.
__device__ __forceinline__ void cp_async16(void *dst, const void *src)
{
    // .cg: the staged rows bypass L1 (measured .ca 457 vs .cg 452 us)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}

template <class SM>
__device__ __forceinline__ void stage_copy(SM &S, const float4 *__restrict__ pos,
                                           const float4 *__restrict__ vel, int g0, int s0, int len, int lane)
{
    for (int k = lane; k < len; k += 32) {
        cp_async16(reinterpret_cast<float4 *>(S.lst) + s0 + k, &pos[g0 + k]);
        cp_async16(&S.sv[s0 + k], &vel[g0 + k]);
    }
}

// Second pass over a staged range: periodic-image shift, SoA copy, id (| species << 30) into
// the velocity word, zeroed accumulators.
template <int KMODE, class SM>
__device__ __forceinline__ void stage_fix(SM &S, int s0, int len, float sx, float sy, float sz, int lane)
{
    for (int k = lane; k < len; k += 32) {
        const int s = s0 + k;
        const float4 p = reinterpret_cast<const float4 *>(S.lst)[s];
        S.sx[s] = p.x + sx;
        S.sy[s] = p.y + sy;
        S.sz[s] = p.z + sz;
        uint32_t word = __float_as_uint(p.w);
        if constexpr (KMODE == 3) word |= (uint32_t)__float_as_int(S.sv[s].w) << 30;
        S.sv[s].w = __uint_as_float(word);
        S.acc[0][s] = 0;
        S.acc[1][s] = 0;
        S.acc[2][s] = 0;
    }
}

// Warp-wide inclusive scan of one int per lane.
__device__ __forceinline__ int warp_incl_scan(int v, int lane)
{
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// Pair evaluation shared by the fast path (smem operands) and the record path.
template <bool RECORD, int KMODE>
__device__ __forceinline__ float pair_eval(const PairP &pp, const FixP &fx, float4 pi, float4 vi, float4 pj,
                                           float4 vj, const RoundKeys &ks, PairRec &rec, int *err, float &dx, float &dy,
                                           float &dz)
{
    dx = pi.x - pj.x;
    dy = pi.y - pj.y;
    dz = pi.z - pj.z;
    const float r2 = dx * dx + dy * dy + dz * dz;
    const float dvdot = dx * (vi.x - vj.x) + dy * (vi.y - vj.y) + dz * (vi.z - vj.z);
    const uint32_t idi = (uint32_t)__float_as_int(pi.w), idj = (uint32_t)__float_as_int(pj.w);
    float s = 0.0f;
    if (r2 > 0.0f) {
        s = pair_scalar<KMODE>(pp, r2, dvdot, idi, idj, ks, vi.w, vj.w);
        if (fabsf(s) * (r2 * rsqrtf(r2)) > fx.mag_lim * fx.scale) raise_err(err, ERR_RANGE, (int)idi);
        if constexpr (RECORD) {
            const unsigned long long k = atomicAdd(rec.count, 1ull);
            if ((long long)k < rec.cap) {
                const uint2 wd = pair_words(idi, idj, ks);
                rec.quad[k] = make_uint4(min(idi, idj), max(idi, idj), wd.x, wd.y);
            }
        }
    }
    return s;
}

// Branch-free pair force of the hot loop: f_ij = s (dx, dy, dz) for staged i (position p*,
// velocity word vi) and staged j.  A coincident pair (r2 = 0: the idle second cursor's self
// pair, or two particles at the same point) gets d = 0 and a finite s, hence f = 0 (C-11).
// The largest |mag| seen is kept in amax and range-checked once per walk.
template <int KMODE>
__device__ __forceinline__ float pair_core(const PairP &pp, float pix, float piy, float piz, float4 vi, float pjx,
                                           float pjy, float pjz, float4 vj, const RoundKeys &ks, float &dx, float &dy,
                                           float &dz, float &amax)
{
    dx = pix - pjx;
    dy = piy - pjy;
    dz = piz - pjz;
    const float r2 = dx * dx + dy * dy + dz * dz;
    const float dvdot = dx * (vi.x - vj.x) + dy * (vi.y - vj.y) + dz * (vi.z - vj.z);
    float mag;
    const float s = pair_mag<KMODE>(pp, fmaxf(r2, 1e-30f), dvdot, w_id<KMODE>(vi.w), w_id<KMODE>(vj.w), ks,
                                    w_species(vi.w), w_species(vj.w), mag);
    amax = fmaxf(amax, fabsf(mag));
    return s;
}

// Debug pair recording (RECORD instantiation only).
template <int KMODE>
__device__ __forceinline__ void pair_record(float4 vi, float4 vj, float dx, float dy, float dz, const RoundKeys &ks,
                                            PairRec &rec)
{
    if (dx * dx + dy * dy + dz * dz > 0.0f) {
        const uint32_t idi = w_id<KMODE>(vi.w), idj = w_id<KMODE>(vj.w);
        const unsigned long long k = atomicAdd(rec.count, 1ull);
        if ((long long)k < rec.cap) {
            const uint2 wd = pair_words(idi, idj, ks);
            rec.quad[k] = make_uint4(min(idi, idj), max(idi, idj), wd.x, wd.y);
        }
    }
}

// Walk over a contiguous range [t, t1) of one warp's concatenated pair lists.  Owners (home
// particles with a non-empty list) change at most a few times per range; the i-side
// fixed-point sum is kept in registers and flushed on each owner change.  `o` indexes the
// warp's owner table (wrec at stride FT_WSTRIDE).
struct PairCursor {
    int t, t1, o, enext, si, lrow;
    float px, py, pz;
    float4 vi;
    AccT fx, fy, fz;
};

// Add (x, y, z) to staged particle s's force.
__device__ __forceinline__ void acc_add(ForceTileSmem &S, float4 *frc, int s, AccT x, AccT y, AccT z)
{
    (void)frc;
    atomicAdd(&S.acc[0][s], x); // native ATOMS.ADD (the fp32 variant is a CAS loop)
    atomicAdd(&S.acc[1][s], y);
    atomicAdd(&S.acc[2][s], z);
}

__device__ __forceinline__ void cursor_load(PairCursor &c, const ForceTileSmem &S)
{
    const int4 r = S.wrec[c.o];
    c.enext = r.y;
    c.lrow = r.z;
    c.si = r.w;
    c.px = S.sx[c.si];
    c.py = S.sy[c.si];
    c.pz = S.sz[c.si];
    c.vi = S.sv[c.si];
}

__device__ __forceinline__ void cursor_init(PairCursor &c, const ForceTileSmem &S, int t0, int t1, int base, int nown)
{
    c.t = t0;
    c.t1 = t1;
    c.fx = c.fy = c.fz = 0;
    int o = 0; // largest owner slot whose list prefix is <= t0
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
        if (o + step < nown && S.wrec[base + o + step].x <= t0) o += step;
    c.o = base + o;
    cursor_load(c, S);
}

__device__ __forceinline__ void cursor_flush(PairCursor &c, ForceTileSmem &S, float4 *frc)
{
    if (c.fx != 0 || c.fy != 0 || c.fz != 0) acc_add(S, frc, c.si, c.fx, c.fy, c.fz);
    c.fx = c.fy = c.fz = 0;
}

// Entry t of the list (the partner j); moves to the next owner first when t crosses it.
__device__ __forceinline__ int cursor_next(PairCursor &c, ForceTileSmem &S, float4 *frc)
{
    if (c.t >= c.enext) { // next owner (never empty)
        cursor_flush(c, S, frc);
        ++c.o;
        cursor_load(c, S);
    }
    return S.lst[c.lrow + c.t];
}

__device__ __forceinline__ void cursor_accumulate(PairCursor &c, ForceTileSmem &S, float4 *frc, int j, float s,
                                                  float dx, float dy, float dz)
{
    const AccT qx = acc_q(dx, s), qy = acc_q(dy, s), qz = acc_q(dz, s);
    c.fx += qx;
    c.fy += qy;
    c.fz += qz;
    acc_add(S, frc, j, -qx, -qy, -qz);
    ++c.t;
}

// Direct global-memory evaluation of one tile's home cells (capacity overflow only).
template <bool RECORD, int KMODE>
__device__ void tile_fallback(const float4 *__restrict__ pos, const float4 *__restrict__ vel, float4 *frc,
                              const int *__restrict__ start, const Geom &g, const PairP &pp, const FixP &fx,
                              const RoundKeys &ks, PairRec &rec, int *err, int x0, int y0, int z0, int bx, int by, int bz,
                              float to_force)
{
    // home particle h of the tile -> (home cell, slot) by a scan over the <= 32 home cells
    int nh = 0;
    for (int hc = 0; hc < bx * by * bz; ++hc) {
        const int cx = x0 + hc % bx, cy = y0 + (hc / bx) % by, cz = z0 + hc / (bx * by);
        const int c0 = (cx + g.off[0]) + g.ext[0] * ((cy + g.off[1]) + g.ext[1] * (cz + g.off[2]));
        nh += start[c0 + 1] - start[c0];
    }
    for (int h = threadIdx.x; h < nh; h += blockDim.x) {
        int hc = 0, base = 0, cx = 0, cy = 0, cz = 0, c0 = 0;
        for (;; ++hc) {
            cx = x0 + hc % bx;
            cy = y0 + (hc / bx) % by;
            cz = z0 + hc / (bx * by);
            c0 = (cx + g.off[0]) + g.ext[0] * ((cy + g.off[1]) + g.ext[1] * (cz + g.off[2]));
            const int cnt = start[c0 + 1] - start[c0];
            if (h < base + cnt) break;
            base += cnt;
        }
        const int i = start[c0] + (h - base);
        {
            const float4 pi = pos[i], vi = vel[i];
            float Fx = 0.f, Fy = 0.f, Fz = 0.f;
            for (int o = 0; o < 14; ++o) {
                const int jxi = cx + c_fwd[o][0], jyi = cy + c_fwd[o][1], jzi = cz + c_fwd[o][2];
                float sx = 0.f, sy = 0.f, sz = 0.f;
                if (!g.split[0]) sx = jxi < 0 ? -g.L[0] : (jxi >= g.n[0] ? g.L[0] : 0.f);
                if (!g.split[1]) sy = jyi < 0 ? -g.L[1] : (jyi >= g.n[1] ? g.L[1] : 0.f);
                if (!g.split[2]) sz = jzi >= g.n[2] ? g.L[2] : 0.f;
                const int c = ext_coord(jxi, g.n[0], g.split[0]) +
                              g.ext[0] * (ext_coord(jyi, g.n[1], g.split[1]) +
                                          g.ext[1] * ext_coord(jzi, g.n[2], g.split[2]));
                for (int j = (o == 0 ? i + 1 : start[c]); j < start[c + 1]; ++j) {
                    float4 pj = pos[j];
                    pj.x += sx;
                    pj.y += sy;
                    pj.z += sz;
                    float dx, dy, dz;
                    const float r2 = (pi.x - pj.x) * (pi.x - pj.x) + (pi.y - pj.y) * (pi.y - pj.y) +
                                     (pi.z - pj.z) * (pi.z - pj.z);
                    if (!(r2 < pp.rc2)) continue;
                    // to_force: 1 / scale when pp is in fixed-point units (tiled kernel), else 1
                    const float s = to_force *
                                    pair_eval<RECORD, KMODE>(pp, fx, pi, vi, pj, vel[j], ks, rec, err, dx, dy, dz);
                    Fx += s * dx;
                    Fy += s * dy;
                    Fz += s * dz;
                    atomicAdd(&frc[j], make_float4(-s * dx, -s * dy, -s * dz, 0.0f));
                }
            }
            atomicAdd(&frc[i], make_float4(Fx, Fy, Fz, 0.0f));
        }
    }
}

// ---------------------------------------------------------------------------------------
// Tile phases.
// ---------------------------------------------------------------------------------------
struct TileGeo {
    int x0, y0, z0, bx, by, bz;
};

// 1a. staged cell table straight from global memory.  role 0 (one warp): one staged row per
// lane -- its cells' starts and counts, a warp scan of the row sums, the in-row prefix;
// role 1 (another warp): one home row per lane (two loads: the home cells of a row are
// contiguous in the extended grid) and their scan.
__device__ __forceinline__ void tile_table(TileTab &T, const TileGeo &G, const Geom &g,
                                           const int *__restrict__ start, int role, int lane)
{
    const int x0 = G.x0, y0 = G.y0, z0 = G.z0, bx = G.bx, by = G.by, bz = G.bz;
    const int sxa = bx + 2, sya = by + 2, sza = bz + 1;
    (void)x0; (void)y0; (void)z0; (void)sza;
    const int nsc = (sxa + FT_ROWPAD) * sya * sza;
    static_assert(FT_SY * FT_SZ <= 32 && FT_NHROW <= 32, "one lane per row");
    if (role == 0) {
        const int nrows = sya * sza;
        int cnt[FT_SX], gst[FT_SX], rsum = 0;
        if (lane < nrows) {
            const int lz = lane >= 2 * sya ? 2 : (lane >= sya ? 1 : 0); // sza <= 3
            const int ly = lane - lz * sya;
            // extended-grid coordinates: split dimensions index the halo ring (empty in the
            // local lists) without wrapping; periodic-local dimensions wrap
            const int gy = ext_coord(y0 - 1 + ly, g.n[1], g.split[1]);
            const int gz = ext_coord(z0 + lz, g.n[2], g.split[2]);
            const int base = g.ext[0] * (gy + g.ext[1] * gz);
#pragma unroll
            for (int x = 0; x < FT_SX; ++x) {
                cnt[x] = gst[x] = 0;
                if (x < sxa) {
                    const int gc = ext_coord(x0 - 1 + x, g.n[0], g.split[0]) + base;
                    gst[x] = start[gc];
                    cnt[x] = start[gc + 1] - gst[x];
                    rsum += cnt[x];
                }
            }
        }
        const int incl = warp_incl_scan(rsum, lane);
        if (lane < nrows) {
            int run = incl - rsum + FT_GAP * lane; // rows separated by FT_GAP sentinel slots
            const int c0 = lane * (sxa + FT_ROWPAD);
#pragma unroll
            for (int x = 0; x < FT_SX; ++x) {
                if (x < sxa) {
                    T.soff[c0 + x] = run;
                    T.cgs[c0 + x] = gst[x];
                    run += cnt[x];
                }
            }
            T.rend[lane] = run;
            if (FT_ROWPAD) T.soff[c0 + sxa] = run; // segment ends never include the sentinel gap
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31) + FT_GAP * nrows;
        if (lane == 0) {
            T.soff[nsc] = tot;
            T.total = tot;
        }
    } else {
        const int nr = by * bz;
        int sz = 0;
        if (lane < nr) {
            const int lz = lane >= by ? 1 : 0;
            const int ly = 1 + lane - lz * by;
            const int base = g.ext[0] * (ext_coord(y0 - 1 + ly, g.n[1], g.split[1]) +
                                         g.ext[1] * ext_coord(z0 + lz, g.n[2], g.split[2]));
            const int ga = ext_coord(x0, g.n[0], g.split[0]) + base; // x0 .. x0 + bx - 1: no wrap
            sz = start[ga + bx] - start[ga];
        }
        const int incl = warp_incl_scan(sz, lane);
        if (lane < nr) T.hoff[lane] = incl - sz;
        if (lane == nr - 1) T.hoff[nr] = incl;
    }
}

// 1b. issue the staging copies of this warp's rows (cp.async, not waited for).
template <class SM>
__device__ __forceinline__ void tile_stage_issue(SM &S, const TileTab &T, const TileGeo &G,
                                                 const Geom &g, const float4 *__restrict__ pos,
                                                 const float4 *__restrict__ vel, int warp, int lane)
{
    const int x0 = G.x0, y0 = G.y0, z0 = G.z0, bx = G.bx, by = G.by, bz = G.bz;
    const int sxa = bx + 2, sya = by + 2, sza = bz + 1;
    (void)x0; (void)y0; (void)z0; (void)sza;
    const bool wrap_lo = !g.split[0] && x0 == 0, wrap_hi = !g.split[0] && x0 + bx == g.n[0];
    for (int row = warp; row < sya * sza; row += FT_NWARP) {
        const int c0 = (sxa + FT_ROWPAD) * row; // lx = 0
        // segment A: lx = 0; B: lx = 1..bx; C: lx = bx + 1 (merged when not wrapped)
        const int a0 = T.soff[c0], b0 = T.soff[c0 + 1], c0s = T.soff[c0 + bx + 1], e0 = T.rend[row];
        const int mlo = wrap_lo ? b0 : a0, mhi = wrap_hi ? c0s : e0;
        if (wrap_lo) stage_copy(S, pos, vel, T.cgs[c0], a0, b0 - a0, lane);
        stage_copy(S, pos, vel, wrap_lo ? T.cgs[c0 + 1] : T.cgs[c0], mlo, mhi - mlo, lane);
        if (wrap_hi) stage_copy(S, pos, vel, T.cgs[c0 + bx + 1], c0s, e0 - c0s, lane);
    }
}

// 1b (second half, after cp.async.wait_all): periodic shift, SoA copy, ids, zeroed sums.
template <int KMODE, class SM>
__device__ __forceinline__ void tile_stage_fix(SM &S, const TileTab &T, const TileGeo &G, const Geom &g,
                                               int warp, int lane)
{
    const int x0 = G.x0, y0 = G.y0, z0 = G.z0, bx = G.bx, by = G.by, bz = G.bz;
    const int sxa = bx + 2, sya = by + 2, sza = bz + 1;
    (void)x0; (void)y0; (void)z0; (void)sza;
    const bool wrap_lo = !g.split[0] && x0 == 0, wrap_hi = !g.split[0] && x0 + bx == g.n[0];
    for (int row = warp; row < sya * sza; row += FT_NWARP) {
        const int lz = row >= 2 * sya ? 2 : (row >= sya ? 1 : 0);
        const int ly = row - lz * sya;
        const int gy = y0 - 1 + ly, gz = z0 + lz;
        const float sy = g.split[1] ? 0.0f : (gy < 0 ? -g.L[1] : (gy >= g.n[1] ? g.L[1] : 0.0f));
        const float sz = g.split[2] ? 0.0f : (gz >= g.n[2] ? g.L[2] : 0.0f);
        const int c0 = (sxa + FT_ROWPAD) * row;
        const int a0 = T.soff[c0], b0 = T.soff[c0 + 1], c0s = T.soff[c0 + bx + 1], e0 = T.rend[row];
        const int mlo = wrap_lo ? b0 : a0, mhi = wrap_hi ? c0s : e0;
        if (wrap_lo) stage_fix<KMODE>(S, a0, b0 - a0, -g.L[0], sy, sz, lane);
        stage_fix<KMODE>(S, mlo, mhi - mlo, 0.0f, sy, sz, lane);
        if (wrap_hi) stage_fix<KMODE>(S, c0s, e0 - c0s, g.L[0], sy, sz, lane);
        if (lane < FT_GAP) { // sentinels: a sweep block running past a row end fails the cutoff test
            S.sx[e0 + lane] = FT_FAR;
            S.sy[e0 + lane] = FT_FAR;
            S.sz[e0 + lane] = FT_FAR;
        }
    }
}

// 2-4. sweep + pairs of this warp's home particles.
template <bool RECORD, int KMODE>
__device__ __forceinline__ void tile_pairs(ForceTileSmem &S, const TileTab &T, const TileGeo &G, const Geom &g,
                                           const PairP &pp, const FixP &fx, const RoundKeys &ks, PairRec &rec,
                                           int *err, float4 *frc, int tid, int warp, int lane)
{
    const int x0 = G.x0, y0 = G.y0, z0 = G.z0, bx = G.bx, by = G.by, bz = G.bz;
    const int sxa = bx + 2, sya = by + 2, sza = bz + 1;
    (void)x0; (void)y0; (void)z0; (void)sza;
    const int nhome = T.hoff[by * bz];
    // ---- 2-4. per warp, one home particle per lane (a second round only past FT_NTHR):
    //           sweep the lane's 5 segments into its list, then evaluate the warp's pairs
    //           with a warp-balanced split -- no CTA barrier between sweep and pairs
    const int rs = sxa + FT_ROWPAD; // table row stride
    const int rowz = rs * sya;
    const float hx = g.L[0] / (float)g.n[0], hy = g.L[1] / (float)g.n[1], hz = g.L[2] / (float)g.n[2];
    const int wb = warp * FT_WSTRIDE;
    const unsigned lbase = (unsigned)__cvta_generic_to_shared(&S.lst[tid * FT_LSTRIDE]);
#ifndef FT_CHUNK32
#define FT_CHUNK32 1
#endif
#if FT_CHUNK32
    // warp w owns the full 32-particle chunks w, w + NWARP, ...: every sweep lane busy but in
    // the last chunk -- an idle warp costs no issue slots, an idle lane does (round 2: 396.5 ->
    // 390.6 us against equal counts per warp, [w nhome / NWARP, (w + 1) nhome / NWARP), which
    // left ~11 % of the sweep's lanes idle; profiles/r02d_ab_chunk32.jsonl)
    const int hend = nhome;
    for (int hb = warp * 32; hb < hend; hb += 32 * FT_NWARP) {
#else
    const int hend = ((warp + 1) * nhome) / FT_NWARP;
    for (int hb = (warp * nhome) / FT_NWARP; hb < hend; hb += 32) {
#endif
        const int h = hb + lane;
        int cnt = 0, s_i = 0;
        if (h < hend) {
            int r = 0;
            while (r + 1 < by * bz && T.hoff[r + 1] <= h) ++r;
            const int lz = r >= by ? 1 : 0;
            const int ly = 1 + r - lz * by;
            const int crow = rs * (ly + sya * lz);
            s_i = T.soff[crow + 1] + (h - T.hoff[r]);
            int lx = 1;
            while (lx < bx && T.soff[crow + lx + 1] <= s_i) ++lx;
            const int c = crow + lx;
            const int c1 = c - 1 + rs; // (lx - 1, ly + 1, lz): the y+1 row
            const float px = S.sx[s_i], py = S.sy[s_i], pz = S.sz[s_i];
            // row-end pruning: lower bounds (minus a rounding slack) on the distance from i
            // to its cell's faces; a row / end cell farther than r_c holds no partner
            const float ox = px - (float)(x0 + lx - 1) * hx, oy = py - (float)(y0 + ly - 1) * hy,
                        oz = pz - (float)(z0 + lz) * hz;
            const float dxl = fmaxf(ox - fx.slack, 0.0f), dxr = fmaxf(hx - ox - fx.slack, 0.0f);
            const float dyl = fmaxf(oy - fx.slack, 0.0f), dyr = fmaxf(hy - oy - fx.slack, 0.0f);
            const float dzr = fmaxf(hz - oz - fx.slack, 0.0f);
            unsigned lptr = lbase;
            bool full = false;
#ifndef PROBE_NOPAIR
#define PROBE_NOPAIR 0
#endif
#define PROBE_NOPAIR_A PROBE_NOPAIR
#ifndef PROBE_NOSWEEP // timing probes: compile the sweep / pair walk out; wrong forces
#define PROBE_NOSWEEP 0
#endif
            // Fused sweep.  The first aligned block of segment 0 (own cell after i, next cell)
            // is the only masked one (j > i) and is peeled: every lane runs exactly one.  All
            // later blocks are unmasked: a block running past a segment end meets a cell two
            // away (distance > h >= r_c) or the row's sentinels, which fail the cutoff test.
            // The lane's remaining segments (rest of 0, then the pruned rows) are one queue,
            // walked by one loop, so a lane's trip count is its total block count.
            const unsigned long long PX = f2dup(px), PY = f2dup(py), PZ = f2dup(pz);
            const int a0s = s_i + 1, b0s = T.soff[c + 2];
            const int j0 = a0s & ~3;
            if (!PROBE_NOSWEEP && j0 < b0s) {
                float ra, rb, rc, rd;
                r2_quad(S, j0, PX, PY, PZ, ra, rb, rc, rd);
                append_if_in(lptr, ra, pp.rc2, (unsigned)j0, a0s, b0s);
                append_if_in(lptr, rb, pp.rc2, (unsigned)(j0 + 1), a0s, b0s);
                append_if_in(lptr, rc, pp.rc2, (unsigned)(j0 + 2), a0s, b0s);
                append_if_in(lptr, rd, pp.rc2, (unsigned)(j0 + 3), a0s, b0s);
            }
            // queue of non-empty segments, packed (end << 16) | aligned start, in sweep order
            unsigned q0 = 0, q1 = 0, q2 = 0, q3 = 0, q4 = 0;
#ifndef FT_LOCKSTEP
#define FT_LOCKSTEP 1
#endif
#pragma unroll
            for (int kk = 0; kk < 5; ++kk) {
                // push-front order: FT_LOCKSTEP walks the four rows first, unpruned, so lanes
                // of one cell read the same candidate quads together (shared-memory broadcast),
                // and their own-cell rest last; else own-cell rest first, rows pruned
                const int k = FT_LOCKSTEP ? (kk == 0 ? 0 : 5 - kk) : 4 - kk;
                int a, b;
                bool ne;
                if (k == 0) {
                    a = j0 + 4;
                    b = b0s;
                    ne = a < b;
                } else {
                    const int cs = (k == 1) ? c1 : c1 - 2 * rs + rowz + (k - 2) * rs;
                    const float qy = (k == 2) ? dyl : (k == 3 ? 0.0f : dyr);
                    const float qz = (k == 1) ? 0.0f : dzr;
                    const float q = qy * qy + qz * qz;
                    a = (FT_LOCKSTEP || dxl * dxl + q < pp.rc2) ? T.soff[cs] : T.soff[cs + 1];
                    b = (FT_LOCKSTEP || dxr * dxr + q < pp.rc2) ? T.soff[cs + 3] : T.soff[cs + 2];
                    ne = (FT_LOCKSTEP || q < pp.rc2) && a < b;
                }
                if (PROBE_NOSWEEP) ne = false;
                if (ne) {
                    q4 = q3;
                    q3 = q2;
                    q2 = q1;
                    q1 = q0;
                    q0 = ((unsigned)b << 16) | (unsigned)(a & ~3);
                }
            }
            int j = (int)(q0 & 0xFFFFu), hi = (int)(q0 >> 16);
            q0 = q1;
            q1 = q2;
            q2 = q3;
            q3 = q4;
            q4 = 0;
#pragma unroll kFtSwUnroll
            while (j < hi) {
                if ((int)(lptr - lbase) > 2 * (FT_LCAP - 4)) { // list full (~4 sigma): the rest in place
                    full = true;
                    break;
                }
                float ra, rb, rc, rd;
                r2_quad(S, j, PX, PY, PZ, ra, rb, rc, rd);
                append_if(lptr, ra, pp.rc2, (unsigned)j);
                append_if(lptr, rb, pp.rc2, (unsigned)(j + 1));
                append_if(lptr, rc, pp.rc2, (unsigned)(j + 2));
                append_if(lptr, rd, pp.rc2, (unsigned)(j + 3));
                j += 4;
                if (j >= hi) { // next segment (predicated pop)
                    j = (int)(q0 & 0xFFFFu);
                    hi = (int)(q0 >> 16);
                    q0 = q1;
                    q1 = q2;
                    q2 = q3;
                    q3 = q4;
                    q4 = 0;
                }
            }
            if (full) {
                const float4 pi = ldp<KMODE>(S, s_i), vi = ldv<KMODE>(S, s_i);
                for (;;) {
                    for (; j < hi; ++j) { // candidates before a segment's start fail the cutoff test
                        if (!(r2_one(S, j, px, py, pz) < pp.rc2)) continue;
                        float dx, dy, dz;
                        const float s =
                            pair_eval<RECORD, KMODE>(pp, fx, pi, vi, ldp<KMODE>(S, j), ldv<KMODE>(S, j), ks, rec, err, dx, dy, dz);
                        const AccT qx = acc_q(dx, s), qy = acc_q(dy, s), qz = acc_q(dz, s);
                        acc_add(S, frc, s_i, qx, qy, qz);
                        acc_add(S, frc, j, -qx, -qy, -qz);
                    }
                    if (q0 == 0) break;
                    j = (int)(q0 & 0xFFFFu);
                    hi = (int)(q0 >> 16);
                    q0 = q1;
                    q1 = q2;
                    q2 = q3;
                    q3 = q4;
                    q4 = 0;
                }
            }
            if (full) atomicAdd(&err[6], 1); // statistics: in-place evaluations
            cnt = (int)(lptr - lbase) >> 1;
        }

#ifndef FT_PHASEA
#define FT_PHASEA 10
#endif
        // ---- 3a. phase A: every lane walks the first FT_PHASEA entries of its OWN list (the
        //          owner is the lane's home particle: no owner switches, i-side sums in
        //          registers); the ~ (cnt - FT_PHASEA)+ leftovers are balanced in phase B.
        //          Round 2 (profiles/r02e_ab_phasea.jsonl): 390.6 us without phase A, 388.2 /
        //          387.5 / 386.9 / 387.5 / 389.6 us with 6 / 8 / 10 / 12 / 14, 389.8 with the
        //          warp's shortest list -- the owner-switch blocks of the balanced walk ran at
        //          ~2 lanes in 78 % of its iterations
        // FT_PHASEA < 0: phase A takes the warp's shortest list length (every lane busy)
        const int pa = FT_PHASEA >= 0 ? FT_PHASEA : (int)__reduce_min_sync(0xffffffffu, (unsigned)(h < hend ? cnt : 1 << 20));
        if (FT_PHASEA != 0 && !PROBE_NOPAIR_A) {
            const int na = min(cnt, pa);
            const int namax = __reduce_max_sync(0xffffffffu, na);
            if (namax > 0) {
                const int lrow = tid * FT_LSTRIDE;
                const float px = S.sx[s_i], py = S.sy[s_i], pz = S.sz[s_i];
                const float4 vi = S.sv[s_i];
                AccT ax = 0, ay = 0, az = 0;
                float amax = 0.0f;
#if FT_PA2
                // two entries per iteration, predicated (an inactive slot evaluates the self pair:
                // r2 = 0 -> f = 0, and skips its j-side atomics): two independent Philox /
                // Box-Muller chains in flight (v65: 386.9 -> 381.6 us, 56 -> 64 registers; a
                // loop unrolled by the compiler gave 386.2, the sweep unrolled 387.3, two
                // cursors in phase B again 389.8; three / four entries per iteration 381.3 /
                // 383.0 us at 68 / 69 registers; profiles/r02f_ab_phasea2.jsonl)
                for (int t = 0; t < namax; t += FT_PAW) {
                    bool a[FT_PAW];
                    int jj[FT_PAW];
                    float4 vv[FT_PAW];
                    float sv[FT_PAW], dx[FT_PAW], dy[FT_PAW], dz[FT_PAW];
#pragma unroll
                    for (int k = 0; k < FT_PAW; ++k) {
                        a[k] = t + k < na;
                        jj[k] = a[k] ? (int)S.lst[lrow + t + k] : s_i;
                    }
#pragma unroll
                    for (int k = 0; k < FT_PAW; ++k) vv[k] = S.sv[jj[k]];
#pragma unroll
                    for (int k = 0; k < FT_PAW; ++k)
                        sv[k] = pair_core<KMODE>(pp, px, py, pz, vi, S.sx[jj[k]], S.sy[jj[k]], S.sz[jj[k]], vv[k], ks,
                                                 dx[k], dy[k], dz[k], amax);
                    if constexpr (RECORD) {
#pragma unroll
                        for (int k = 0; k < FT_PAW; ++k)
                            if (a[k]) pair_record<KMODE>(vi, vv[k], dx[k], dy[k], dz[k], ks, rec);
                    }
#pragma unroll
                    for (int k = 0; k < FT_PAW; ++k) {
                        const AccT qx = acc_q(dx[k], sv[k]), qy = acc_q(dy[k], sv[k]), qz = acc_q(dz[k], sv[k]);
                        ax += qx;
                        ay += qy;
                        az += qz;
                        if (a[k]) acc_add(S, frc, jj[k], -qx, -qy, -qz);
                    }
                }
#else
#pragma unroll kFtPaUnroll
                for (int t = 0; t < namax; ++t) {
                    if (t < na) {
                        const int j = S.lst[lrow + t];
                        const float4 vj = S.sv[j];
                        float dx, dy, dz;
                        const float sv = pair_core<KMODE>(pp, px, py, pz, vi, S.sx[j], S.sy[j], S.sz[j], vj, ks, dx, dy,
                                                          dz, amax);
                        if constexpr (RECORD) pair_record<KMODE>(vi, vj, dx, dy, dz, ks, rec);
                        const AccT qx = acc_q(dx, sv), qy = acc_q(dy, sv), qz = acc_q(dz, sv);
                        ax += qx;
                        ay += qy;
                        az += qz;
                        acc_add(S, frc, j, -qx, -qy, -qz);
                    }
                }
#endif
                if (na > 0 && (ax != 0 || ay != 0 || az != 0)) acc_add(S, frc, s_i, ax, ay, az);
                if (amax > fx.mag_lim * fx.scale) raise_err(err, ERR_RANGE, (int)w_id<KMODE>(vi.w));
            }
        }
        const int cnt_b = max(cnt - pa, 0);
        // ---- 3. the warp's compacted owner table of the phase-B leftovers: one packed scan
        //         (owners | entries << 8)
        const int v = (cnt_b > 0 ? 1 : 0) | (cnt_b << 8);
        const int incl = warp_incl_scan(v, lane);
        const int tp = __shfl_sync(0xffffffffu, incl, 31);
        const int nown = tp & 0xFF, tot = tp >> 8;
        if (cnt_b > 0) {
            const int o = (incl - v) & 0xFF, e = (incl - v) >> 8;
            S.wrec[wb + o] = make_int4(e, e + cnt_b, tid * FT_LSTRIDE + pa - e, s_i);
        }
        __syncwarp();

        // ---- 4. pair evaluation: contiguous chunk of the warp's lists per lane, walked by two
        //         independent cursors (halves of the chunk) so two Philox/Box-Muller chains
        //         are in flight per thread (instruction-level parallelism)
        if (tot > 0 && !PROBE_NOPAIR) {
            const int C = (tot + 31) >> 5;
            const int t0 = min(lane * C, tot);
            const int t1 = min(t0 + C, tot);
            const int q = (t1 - t0 + FT_NCUR - 1) / FT_NCUR;
            PairCursor cu[FT_NCUR];
#pragma unroll
            for (int k = 0; k < FT_NCUR; ++k) cursor_init(cu[k], S, min(t0 + k * q, t1), min(t0 + (k + 1) * q, t1), wb, nown);
            float amax = 0.0f;
            while (cu[0].t < cu[0].t1) { // later cursors are never longer than the first
                int j[FT_NCUR];
                bool act[FT_NCUR];
#pragma unroll
                for (int k = 0; k < FT_NCUR; ++k) {
                    act[k] = (k == 0) || cu[k].t < cu[k].t1;
                    j[k] = act[k] ? cursor_next(cu[k], S, frc) : cu[k].si; // idle: self pair, r2 = 0 -> f = 0
                }
                float4 vj[FT_NCUR];
                float sv_[FT_NCUR], dx[FT_NCUR], dy[FT_NCUR], dz[FT_NCUR];
#pragma unroll
                for (int k = 0; k < FT_NCUR; ++k) vj[k] = S.sv[j[k]];
#pragma unroll
                for (int k = 0; k < FT_NCUR; ++k)
                    sv_[k] = pair_core<KMODE>(pp, cu[k].px, cu[k].py, cu[k].pz, cu[k].vi, S.sx[j[k]], S.sy[j[k]],
                                              S.sz[j[k]], vj[k], ks, dx[k], dy[k], dz[k], amax);
                if constexpr (RECORD) {
#pragma unroll
                    for (int k = 0; k < FT_NCUR; ++k)
                        if (act[k]) pair_record<KMODE>(cu[k].vi, vj[k], dx[k], dy[k], dz[k], ks, rec);
                }
#pragma unroll
                for (int k = 0; k < FT_NCUR; ++k)
                    cursor_accumulate(cu[k], S, frc, j[k], sv_[k], dx[k], dy[k], dz[k]); // idle: adds zeros
            }
#pragma unroll
            for (int k = 0; k < FT_NCUR; ++k) cursor_flush(cu[k], S, frc);
            if (amax > fx.mag_lim * fx.scale) // one pair must stay below 2^21 fixed-point units
                raise_err(err, ERR_RANGE, (int)w_id<KMODE>(cu[0].vi.w));
        }
        __syncwarp(); // the lists and the owner table are rewritten by the next round
    }
}

// 5. flush: fixed point -> fp32, one vector reduction per staged particle; rows map back
// to <= 3 contiguous global segments, exactly as they were staged.
template <class SM>
__device__ __forceinline__ void tile_flush(const SM &S, const TileTab &T, const TileGeo &G,
                                           const Geom &g, const FixP &fx, float4 *frc, int warp, int lane)
{
    const int x0 = G.x0, y0 = G.y0, z0 = G.z0, bx = G.bx, by = G.by, bz = G.bz;
    const int sxa = bx + 2, sya = by + 2, sza = bz + 1;
    (void)x0; (void)y0; (void)z0; (void)sza;
    const bool wrap_lo = !g.split[0] && x0 == 0, wrap_hi = !g.split[0] && x0 + bx == g.n[0];
    for (int row = warp; row < sya * sza; row += FT_NWARP) {
        const int c0 = (sxa + FT_ROWPAD) * row;
        const int a0 = T.soff[c0], b0 = T.soff[c0 + 1], c0s = T.soff[c0 + bx + 1], e0 = T.rend[row];
        const int mlo = wrap_lo ? b0 : a0, mhi = wrap_hi ? c0s : e0;
        const int gm = wrap_lo ? T.cgs[c0 + 1] : T.cgs[c0];
        for (int s = a0 + lane; s < e0; s += 32) {
            const int gi = (s < mlo) ? T.cgs[c0] + (s - a0)
                                     : (s < mhi ? gm + (s - mlo) : T.cgs[c0 + bx + 1] + (s - c0s));
            const int qx = S.acc[0][s], qy = S.acc[1][s], qz = S.acc[2][s];
            if (qx | qy | qz)
                atomicAdd(&frc[gi], make_float4((float)qx * fx.inv_scale, (float)qy * fx.inv_scale,
                                                (float)qz * fx.inv_scale, 0.0f));
        }
    }
}

__device__ __forceinline__ bool tile_overflows(const TileTab &T, const TileGeo &G)
{
    return T.total > FT_SCAP || T.hoff[G.by * G.bz] > FT_HCAP;
}

template <bool RECORD, int KMODE>
__global__ void __launch_bounds__(FT_NTHR, FT_MINB)
    k_force_tile(const float4 *__restrict__ pos, const float4 *__restrict__ vel, float4 *__restrict__ frc,
                 const int *__restrict__ start, Geom g, PairP pp, FixP fx, const __grid_constant__ RoundKeys rk,
                 PairRec rec, int *err, float4 *__restrict__ fzero, int nzero)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ForceTileSmem &S = *reinterpret_cast<ForceTileSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // the step's other force buffer (read by this step's bin/scatter, accumulated into by the
    // next step's force pass) is zeroed here, a slice per CTA: this kernel leaves HBM idle, so
    // k_scatter no longer writes a zeroed force array
#ifndef FZERO_CTAS
#define FZERO_CTAS 888 // the first two waves (2 x 3 tiles x 148 SMs): the zeroed lines age out of L2 before
                        // k_bin (v65: 296 / 444 / 888 / all CTAs: 0.4309 / 0.4309 / 0.4297 / 0.4327 ms per step)
#endif
    if (fzero) {
        const int nb = min((int)(gridDim.x * gridDim.y * gridDim.z), FZERO_CTAS);
        const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        if (b < nb)
            for (int k = b * FT_NTHR + tid; k < nzero; k += nb * FT_NTHR) fzero[k] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
    const RoundKeys &ks = rk; // host-computed round keys of this step (constant bank)
    static_assert(FT_BZ <= 2, "home-row decoding assumes at most two home layers");
    // 3D grid: one CTA per tile, no integer division
    TileGeo G;
    G.x0 = blockIdx.x * FT_BX;
    G.y0 = blockIdx.y * FT_BY;
    G.z0 = blockIdx.z * FT_BZ;
    G.bx = min(FT_BX, g.n[0] - G.x0);
    G.by = min(FT_BY, g.n[1] - G.y0);
    G.bz = min(FT_BZ, g.n[2] - G.z0);
    TileTab &T = S.tab[0];
    if (warp < 2) tile_table(T, G, g, start, warp, lane);
    __syncthreads();
    if (tile_overflows(T, G)) {
        if (tid == 0) atomicAdd(&err[T.total > FT_SCAP ? 4 : 5], 1); // fallback statistics
        tile_fallback<RECORD, KMODE>(pos, vel, frc, start, g, pp, fx, ks, rec, err, G.x0, G.y0, G.z0, G.bx, G.by,
                                     G.bz, fx.inv_scale);
        return;
    }
    tile_stage_issue(S, T, G, g, pos, vel, warp, lane);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    tile_stage_fix<KMODE>(S, T, G, g, warp, lane);
    __syncthreads();
    tile_pairs<RECORD, KMODE>(S, T, G, g, pp, fx, ks, rec, err, frc, tid, warp, lane);
    __syncthreads();
    tile_flush(S, T, G, g, fx, frc, warp, lane);
}

} // namespace dpd
