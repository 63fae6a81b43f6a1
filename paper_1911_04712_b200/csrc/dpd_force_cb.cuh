// dpd_force_cb.cuh -- production pair-force sweep, cell-block form.
//
// Same tile, staging, fixed-point accumulation and flush as dpd_force_tile.cuh (one CTA of 9
// warps per 4 x 4 x 2 home cells), but the candidate sweep is lane-uniform:
//   sweep : per home cell A the warp spreads the forward half-stencil candidate set
//           J(A) = A, A+x, the y+1 row and the three z+1 rows (<= 5 contiguous staged ranges,
//           ~112 particles at rho = 8) over its lanes, 32 per slot, positions in registers;
//           A's particles i are broadcast one after the other, every lane tests its slots
//           (packed fp32x2 distances), and each slot's hits become one ballot word.  The
//           pair list of i is its slot words (a bit per lane) -- no per-lane segment loops,
//           no divergence, no list appends;
//   pairs : the warp's bit lists are concatenated and cut into 32 balanced lane chunks, each
//           walked by two cursors (two Philox chains in flight) that decode the next set bit
//           into a J index and, through the cell's J map, into a staged particle; the i-side
//           sum stays in registers until the owner changes (as dpd_force_tile.cuh).
// A warp owns an equal share of the tile's home particles (cells split between two warps
// are set up by both).  Cells with more than 32 particles or |J| > 192 (rho-8 tails beyond
// 7 sigma) send the tile to the global-memory fallback.  DESIGN.md §6 records the measured
// effect of this form.
#pragma once

#include "dpd_force_tile.cuh"

namespace dpd {

constexpr int CB_NSW = 6;                              // slot words per home particle (|J| <= 192)
constexpr int CB_NHC = FT_BX * FT_BY * FT_BZ;         // home cells per tile (32)
constexpr int CB_JCAP = CB_NHC * CB_NSW * 32;         // J-map entries of a tile
constexpr int CB_OVL = FT_HCAP * 16 + FT_HCAP * 8 + FT_HCAP * 16 + CB_JCAP * 2;
constexpr float CB_FAR = 1.0e18f;                     // position of an empty slot lane

// Per home cell: J index -> staged index is jj + D_s on range s (jj >= P_s), five ranges;
// A's first home index and particle count; its J-map base and slot count.
struct CBCell {
    int4 a;  // D0 (= A's first staged particle), D1, D2, D3
    int4 b;  // D4, P1, P2, P3
    int4 c;  // P4, |J|, first home index, n_A
    int4 d;  // J-map base, slots, 0, 0
};

struct ForceCBSmem {
    float4 sv[FT_SCAP];                          // staged velocities; w: id bits | species << 30
    // overlay: the AoS landing buffer of the staged positions (cp.async), then the slot words,
    // owner records and J maps of the sweep
    unsigned short lst[CB_OVL / 2];
    float sx[FT_SCAP], sy[FT_SCAP], sz[FT_SCAP]; // staged positions (tile frame), SoA
    int acc[3][FT_SCAP];                         // fixed-point force sums
    CBCell cell[CB_NHC];
    TileTab tab[1];
    int flag;                                    // a cell outside the bit-list limits
};

static_assert(CB_OVL >= (int)sizeof(float4) * FT_SCAP, "the overlay doubles as the position landing buffer");
static_assert(offsetof(ForceCBSmem, lst) % 16 == 0 && offsetof(ForceCBSmem, sx) % 16 == 0 &&
                  offsetof(ForceCBSmem, acc) % 16 == 0 && offsetof(ForceCBSmem, cell) % 16 == 0,
              "vector shared accesses");

__device__ __forceinline__ uint4 *cb_bits4(ForceCBSmem &S) { return reinterpret_cast<uint4 *>(S.lst); }
__device__ __forceinline__ uint2 *cb_bits2(ForceCBSmem &S)
{
    return reinterpret_cast<uint2 *>(reinterpret_cast<char *>(S.lst) + FT_HCAP * 16);
}
__device__ __forceinline__ int4 *cb_hrec(ForceCBSmem &S)
{
    return reinterpret_cast<int4 *>(reinterpret_cast<char *>(S.lst) + FT_HCAP * 24);
}
__device__ __forceinline__ unsigned short *cb_jmap(ForceCBSmem &S)
{
    return reinterpret_cast<unsigned short *>(reinterpret_cast<char *>(S.lst) + FT_HCAP * 40);
}

// Slot word k of home particle h (k < 4: the uint4 record, else the uint2 one).
__device__ __forceinline__ unsigned cb_word(ForceCBSmem &S, int h, int k)
{
    const unsigned *p = (k < 4) ? reinterpret_cast<const unsigned *>(cb_bits4(S) + h) + k
                                : reinterpret_cast<const unsigned *>(cb_bits2(S) + h) + (k - 4);
    return *p;
}

// Per-home-cell table (one lane per home cell, one warp): J(A) ranges as (D_s, P_s), home
// prefix, J-map prefix; flags cells beyond the bit-list limits.
__device__ __forceinline__ void cb_cells(ForceCBSmem &S, const TileGeo &G, int lane)
{
    const TileTab &T = S.tab[0];
    const int bx = G.bx, by = G.by, bz = G.bz;
    const int sxa = bx + 2, sya = by + 2, rowz = sxa * sya;
    const int nhc = bx * by * bz;
    int nA = 0, nsl = 0;
    bool bad = false;
    int4 ca = make_int4(0, 0, 0, 0), cbv = ca, cc = ca;
    if (lane < nhc) {
        const int hx = lane % bx, hy = (lane / bx) % by, hz = lane / (bx * by);
        const int c = (hx + 1) + sxa * ((hy + 1) + sya * hz);
        const int a0 = T.soff[c];
        nA = T.soff[c + 1] - a0;
        const int c1 = c + sxa - 1;        // (x-1 .. x+1, y+1, z)
        const int c2 = c + rowz - sxa - 1; // (x-1 .. x+1, y-1 .. y+1, z+1)
        const int a1 = T.soff[c1], a2 = T.soff[c2], a3 = T.soff[c2 + sxa], a4 = T.soff[c2 + 2 * sxa];
        const int P1 = T.soff[c + 2] - a0;                 // A and A + x
        const int P2 = P1 + T.soff[c1 + 3] - a1;
        const int P3 = P2 + T.soff[c2 + 3] - a2;
        const int P4 = P3 + T.soff[c2 + sxa + 3] - a3;
        const int J = P4 + T.soff[c2 + 2 * sxa + 3] - a4;
        ca = make_int4(a0, a1 - P1, a2 - P2, a3 - P3);
        cbv = make_int4(a4 - P4, P1, P2, P3);
        cc = make_int4(P4, J, 0, nA);
        nsl = J <= 128 ? 4 : CB_NSW;
        bad = nA > 32 || J > 32 * CB_NSW;
    }
    cc.z = warp_incl_scan(nA, lane) - nA;
    const int js = warp_incl_scan(nsl * 32, lane) - nsl * 32;
    if (lane < nhc) {
        S.cell[lane].a = ca;
        S.cell[lane].b = cbv;
        S.cell[lane].c = cc;
        S.cell[lane].d = make_int4(js, nsl, 0, 0);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) S.flag = 1;
}

// J index jj of a cell -> staged particle (branch-free; -1 beyond |J|).
__device__ __forceinline__ int cb_staged(const CBCell &C, int jj)
{
    int d = C.a.x;
    d = jj >= C.b.y ? C.a.y : d;
    d = jj >= C.b.z ? C.a.z : d;
    d = jj >= C.b.w ? C.a.w : d;
    d = jj >= C.c.x ? C.b.x : d;
    return jj < C.c.y ? jj + d : -1;
}

// Sweep of home particles [ii0, ii1) of one cell with NS slots: slot words into the bit
// lists, owner records {cumulative end, staged i, J-map base} into hrec.
template <int NS>
__device__ __forceinline__ void cb_sweep_cell(ForceCBSmem &S, const CBCell &C, int ii0, int ii1, float rc2, int lane,
                                              int &cum)
{
    float jx[NS], jy[NS], jz[NS];
    unsigned short *jm = cb_jmap(S) + C.d.x;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const int t = cb_staged(C, 32 * k + lane);
        const int sj = max(t, 0);
        jm[32 * k + lane] = (unsigned short)sj;
        jx[k] = t >= 0 ? S.sx[sj] : CB_FAR;
        jy[k] = t >= 0 ? S.sy[sj] : CB_FAR;
        jz[k] = t >= 0 ? S.sz[sj] : CB_FAR;
    }
    unsigned long long X[NS / 2], Y[NS / 2], Z[NS / 2];
#pragma unroll
    for (int k = 0; k < NS / 2; ++k) {
        X[k] = ((unsigned long long)__float_as_uint(jx[2 * k + 1]) << 32) | __float_as_uint(jx[2 * k]);
        Y[k] = ((unsigned long long)__float_as_uint(jy[2 * k + 1]) << 32) | __float_as_uint(jy[2 * k]);
        Z[k] = ((unsigned long long)__float_as_uint(jz[2 * k + 1]) << 32) | __float_as_uint(jz[2 * k]);
    }
    uint4 *b4 = cb_bits4(S);
    uint2 *b2 = cb_bits2(S);
    int4 *hr = cb_hrec(S);
    const int h0 = C.c.z;
#pragma unroll 1
    for (int ii = ii0; ii < ii1; ++ii) {
        const int si = C.a.x + ii;
        const unsigned long long PX = f2dup(S.sx[si]), PY = f2dup(S.sy[si]), PZ = f2dup(S.sz[si]);
        unsigned B[NS];
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < NS / 2; ++k) {
            float ra, rb;
            r2_pair(X[k], Y[k], Z[k], PX, PY, PZ, ra, rb);
            // J index of slot 0 lanes: A's own particles first, so j > i <=> lane > ii there
            const bool h_a = ra < rc2 && (k > 0 || lane > ii);
            const bool h_b = rb < rc2;
            B[2 * k] = __ballot_sync(0xffffffffu, h_a);
            B[2 * k + 1] = __ballot_sync(0xffffffffu, h_b);
            cnt += __popc(B[2 * k]) + __popc(B[2 * k + 1]);
        }
        cum += cnt;
        if (lane == 0) {
            const int h = h0 + ii;
            b4[h] = make_uint4(B[0], B[1], B[2], B[3]);
            if constexpr (NS > 4) b2[h] = make_uint2(B[4], B[5]);
            hr[h] = make_int4(cum, si, C.d.x, 0);
        }
    }
}

// Pair cursor over the warp's bit lists (owners = home particles [h_lo, h_hi)).
struct CBCursor {
    int t, t1, o, enext, si, jb, k;
    unsigned w;
    float px, py, pz;
    float4 vi;
    int fx, fy, fz;
};

__device__ __forceinline__ void cb_load_owner(CBCursor &c, ForceCBSmem &S)
{
    const int4 r = cb_hrec(S)[c.o];
    c.enext = r.x;
    c.si = r.y;
    c.jb = r.z;
    c.k = 0;
    c.w = cb_bits4(S)[c.o].x;
    c.px = S.sx[c.si];
    c.py = S.sy[c.si];
    c.pz = S.sz[c.si];
    c.vi = S.sv[c.si];
}

// Index of the n-th (0-based) set bit of w (n < popc(w)): binary search on the halves.
__device__ __forceinline__ int nth_bit(unsigned w, int n)
{
    int pos = 0;
#pragma unroll
    for (int half = 16; half > 0; half >>= 1) {
        const int lo = __popc(w & ((1u << half) - 1u));
        if (n >= lo) {
            n -= lo;
            w >>= half;
            pos += half;
        } else {
            w &= (1u << half) - 1u;
        }
    }
    return pos;
}

__device__ __forceinline__ void cb_cursor_init(CBCursor &c, ForceCBSmem &S, int t0, int t1, int h_lo, int h_hi)
{
    c.t = t0;
    c.t1 = t1;
    c.fx = c.fy = c.fz = 0;
    // first owner whose cumulative end exceeds t0 (owners with empty lists are skipped)
    const int4 *hr = cb_hrec(S);
    int lo = h_lo, n = h_hi - h_lo;
    while (n > 0) {
        const int half = n >> 1;
        if (hr[lo + half].x <= t0) {
            lo += half + 1;
            n -= half + 1;
        } else {
            n = half;
        }
    }
    c.o = min(lo, h_hi - 1);
    cb_load_owner(c, S);
    if (t0 < t1) { // skip the entries of this owner that precede t0
        int r = t0 - (c.o > h_lo ? hr[c.o - 1].x : 0);
        int pc = __popc(c.w);
        while (r >= pc) {
            r -= pc;
            ++c.k;
            c.w = cb_word(S, c.o, c.k);
            pc = __popc(c.w);
        }
        // drop the r lowest set bits
        const int b = nth_bit(c.w, r);
        c.w &= ~((1u << b) - 1u);
    }
}

__device__ __forceinline__ void cb_cursor_flush(CBCursor &c, ForceCBSmem &S)
{
    if (c.fx | c.fy | c.fz) {
        atomicAdd(&S.acc[0][c.si], c.fx);
        atomicAdd(&S.acc[1][c.si], c.fy);
        atomicAdd(&S.acc[2][c.si], c.fz);
    }
    c.fx = c.fy = c.fz = 0;
}

// Staged index of entry t (the partner j); moves to the next owner first when t crosses it.
// The slot word is refilled right after its last bit (predicated load, no loop in the
// common case); an all-zero slot word is skipped by the loop.
__device__ __forceinline__ int cb_cursor_next(CBCursor &c, ForceCBSmem &S)
{
    if (c.t >= c.enext) {
        cb_cursor_flush(c, S);
        const int4 *hr = cb_hrec(S);
        do {
            ++c.o;
        } while (hr[c.o].x <= c.t);
        cb_load_owner(c, S);
    }
    while (c.w == 0) {
        ++c.k;
        c.w = cb_word(S, c.o, c.k);
    }
    const int b = __ffs(c.w) - 1;
    const int j = cb_jmap(S)[c.jb + 32 * c.k + b];
    c.w &= c.w - 1;
    const int kn = c.k + 1;
    const unsigned wn = cb_word(S, c.o, min(kn, CB_NSW - 1));
    if (c.w == 0) {
        c.k = kn;
        c.w = wn;
    }
    return j;
}

__device__ __forceinline__ void cb_cursor_accumulate(CBCursor &c, ForceCBSmem &S, int j, float s, float dx, float dy,
                                                     float dz)
{
    const int qx = fix_q(dx, s), qy = fix_q(dy, s), qz = fix_q(dz, s);
    c.fx += qx;
    c.fy += qy;
    c.fz += qz;
    atomicAdd(&S.acc[0][j], -qx); // native ATOMS.ADD (the fp32 variant is a CAS loop)
    atomicAdd(&S.acc[1][j], -qy);
    atomicAdd(&S.acc[2][j], -qz);
    ++c.t;
}

// 2-4. sweep + pairs of this warp's share of the home particles.
template <bool RECORD, int KMODE>
__device__ __forceinline__ void cb_pairs(ForceCBSmem &S, const TileGeo &G, const PairP &pp, const FixP &fx,
                                         const RoundKeys &ks, PairRec &rec, int *err, int warp, int lane)
{
    const int nhc = G.bx * G.by * G.bz;
    const int nh = S.tab[0].hoff[G.by * G.bz];
    const int h_lo = (warp * nh) / FT_NWARP, h_hi = ((warp + 1) * nh) / FT_NWARP;
    if (h_lo >= h_hi) return;
    // the cell holding h_lo: the last cell whose first home index is <= h_lo
    int hc = __popc(__ballot_sync(0xffffffffu, lane < nhc && S.cell[lane].c.z <= h_lo)) - 1;
    int cum = 0;
    for (int h = h_lo; h < h_hi; ++hc) {
        const CBCell C = S.cell[hc];
        const int ii0 = h - C.c.z, ii1 = min(C.c.w, h_hi - C.c.z);
        if (ii0 >= ii1) continue; // empty cell
        if (C.d.y == 4) cb_sweep_cell<4>(S, C, ii0, ii1, pp.rc2, lane, cum);
        else cb_sweep_cell<CB_NSW>(S, C, ii0, ii1, pp.rc2, lane, cum);
        h = C.c.z + ii1;
    }
    __syncwarp();
    const int tot = cum;
#ifndef PROBE_NOPAIR
#define PROBE_NOPAIR 0
#endif
    if (tot == 0 || PROBE_NOPAIR) return;
    const int Cn = (tot + 31) >> 5;
    const int t0 = min(lane * Cn, tot);
    const int t1 = min(t0 + Cn, tot);
    const int q = (t1 - t0 + FT_NCUR - 1) / FT_NCUR;
    CBCursor cu[FT_NCUR];
#pragma unroll
    for (int k = 0; k < FT_NCUR; ++k) cb_cursor_init(cu[k], S, min(t0 + k * q, t1), min(t0 + (k + 1) * q, t1), h_lo, h_hi);
    float amax = 0.0f;
    while (cu[0].t < cu[0].t1) { // later cursors are never longer than the first
        int j[FT_NCUR];
        bool act[FT_NCUR];
#pragma unroll
        for (int k = 0; k < FT_NCUR; ++k) {
            act[k] = (k == 0) || cu[k].t < cu[k].t1;
            j[k] = act[k] ? cb_cursor_next(cu[k], S) : cu[k].si; // idle: self pair, r2 = 0 -> f = 0
        }
        float4 vj[FT_NCUR];
        float sv_[FT_NCUR], dx[FT_NCUR], dy[FT_NCUR], dz[FT_NCUR];
#pragma unroll
        for (int k = 0; k < FT_NCUR; ++k) vj[k] = S.sv[j[k]];
#pragma unroll
        for (int k = 0; k < FT_NCUR; ++k)
            sv_[k] = pair_core<KMODE>(pp, cu[k].px, cu[k].py, cu[k].pz, cu[k].vi, S.sx[j[k]], S.sy[j[k]], S.sz[j[k]],
                                      vj[k], ks, dx[k], dy[k], dz[k], amax);
        if constexpr (RECORD) {
#pragma unroll
            for (int k = 0; k < FT_NCUR; ++k)
                if (act[k]) pair_record<KMODE>(cu[k].vi, vj[k], dx[k], dy[k], dz[k], ks, rec);
        }
#pragma unroll
        for (int k = 0; k < FT_NCUR; ++k) cb_cursor_accumulate(cu[k], S, j[k], sv_[k], dx[k], dy[k], dz[k]);
    }
#pragma unroll
    for (int k = 0; k < FT_NCUR; ++k) cb_cursor_flush(cu[k], S);
    if (amax > fx.mag_lim * fx.scale) raise_err(err, ERR_RANGE, (int)w_id<KMODE>(cu[0].vi.w));
}

template <bool RECORD, int KMODE>
__global__ void __launch_bounds__(FT_NTHR, FT_MINB)
    k_force_cb(const float4 *__restrict__ pos, const float4 *__restrict__ vel, float4 *__restrict__ frc,
               const int *__restrict__ start, Geom g, PairP pp, FixP fx, const __grid_constant__ RoundKeys rk,
               PairRec rec, int *err)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ForceCBSmem &S = *reinterpret_cast<ForceCBSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const RoundKeys &ks = rk;
    TileGeo G;
    G.x0 = blockIdx.x * FT_BX;
    G.y0 = blockIdx.y * FT_BY;
    G.z0 = blockIdx.z * FT_BZ;
    G.bx = min(FT_BX, g.n[0] - G.x0);
    G.by = min(FT_BY, g.n[1] - G.y0);
    G.bz = min(FT_BZ, g.n[2] - G.z0);
    TileTab &T = S.tab[0];
    if (warp < 2) tile_table(T, G, g, start, warp, lane);
    if (tid == 0) S.flag = 0;
    __syncthreads();
    if (tile_overflows(T, G)) {
        if (tid == 0) atomicAdd(&err[T.total > FT_SCAP ? 4 : 5], 1); // fallback statistics
        tile_fallback<RECORD, KMODE>(pos, vel, frc, start, g, pp, fx, ks, rec, err, G.x0, G.y0, G.z0, G.bx, G.by,
                                     G.bz, fx.inv_scale);
        return;
    }
    tile_stage_issue(S, T, G, g, pos, vel, warp, lane);
    if (warp == FT_NWARP - 1) cb_cells(S, G, lane); // while this warp's copies are in flight
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    tile_stage_fix<KMODE>(S, T, G, g, warp, lane);
    __syncthreads();
    if (S.flag) { // a cell beyond the bit-list limits (dense clusters only)
        if (tid == 0) atomicAdd(&err[5], 1);
        tile_fallback<RECORD, KMODE>(pos, vel, frc, start, g, pp, fx, ks, rec, err, G.x0, G.y0, G.z0, G.bx, G.by,
                                     G.bz, fx.inv_scale);
        return;
    }
    cb_pairs<RECORD, KMODE>(S, G, pp, fx, ks, rec, err, warp, lane);
    __syncthreads();
    tile_flush(S, T, G, g, fx, frc, warp, lane);
}

} // namespace dpd
