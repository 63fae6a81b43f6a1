// dpd_device.cuh -- device-side building blocks of the DPD step (sm_100a).
//
// Independent of oracle/ (no shared code): the pair RNG and pair force below are written
// from PAPER.md P:109-136 and the readings C-3..C-11 in DESIGN.md §3.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dpd {

// ---------------------------------------------------------------------------------------
// Parameter blocks passed by value to kernels.
// ---------------------------------------------------------------------------------------

// Geometry of one (sub)domain's cell grid (C-8).  Local coordinates x in [0, L).
// Dimensions that are split across ranks carry a one-cell halo ring (ext = n + 2, off = 1);
// periodic-local dimensions wrap inside the grid (ext = n, off = 0).
struct Geom {
    int n[3];       // interior cells per dimension, n_d = floor(L_d / r_c) >= 3
    int ext[3];     // extended cells per dimension (n + 2 if split else n)
    int off[3];     // 1 if split else 0
    int split[3];   // 1 if the dimension is split across ranks
    float L[3];     // local (sub)domain extent
    float inv_h[3]; // (float)n_d / (float)L_d, evaluated in fp32 on the host (C-8)
    int ncell;      // ext_x * ext_y * ext_z
};

constexpr int DPD_MAX_SPECIES = 4;

// Pair-force parameters.
struct PairP {
    float a;        // conservative amplitude
    float gamma;    // dissipative coefficient
    float sig_dt;   // sigma / sqrt(dt) * kBM, sigma = sqrt(2 gamma kT)      (C-3; kBM below)
    float inv_rc;   // 1 / r_c
    float rc2;      // r_c^2
    float power;    // k (w_R = w^k)                                         (C-4)
    uint32_t seed_lo, seed_hi; // the 64-bit seed, unfolded: per-step key       (C-7)
    // NEXT-2 species matrix (KMODE == 3 only): entry ti * DPD_MAX_SPECIES + tj holds the
    // pair's a, gamma and sigma/sqrt(dt); ti, tj travel in vel.w
    float sa[DPD_MAX_SPECIES * DPD_MAX_SPECIES];
    float sg[DPD_MAX_SPECIES * DPD_MAX_SPECIES];
    float ss[DPD_MAX_SPECIES * DPD_MAX_SPECIES]; // x kBM like sig_dt
};

// Integrator parameters (C-2 item 3 / C-6).
constexpr int DPD_MAX_WALLS = 4;

struct IntegP {
    float dt;       // drift time step (0 when only re-binning at set time)
    float kick;     // velocity kick factor: dt/2 on the first step after set, dt after
    float body_f;   // body-force magnitude f
    float x_half;   // global L_x / 2 expressed in local coordinates
    int body_mode;  // 0: periodic Poiseuille (sign flips at L_x/2), 1: uniform +f along z
    int frozen_mask; // species s never moves iff bit s (NEXT-3 frozen wall layer)
    // SDF walls (NEXT-3, C-23): solid = union of primitives, s = max_k s_k > 0 inside
    int nwall;
    int wtype[DPD_MAX_WALLS];      // 1 plane s = n.x - c; 2/3/4 cylinder along x/y/z
    float wprm[DPD_MAX_WALLS][4];  // plane (nx, ny, nz, c); cylinder (c1, c2, R, sign)
    float wvel[DPD_MAX_WALLS][3];  // translational wall velocity
    float origin[3];               // local -> global coordinates (walls are global)
};

// ---------------------------------------------------------------------------------------
// Pair RNG (C-7): Philox2x32-10 (Random123).  Round: (hi, lo) = M * c0;
// c' = (hi ^ k ^ c1, lo); k += W.  Per-step key k_s = fmix32(s_lo ^ seed_lo ^ fmix32(s_hi))
// ^ seed_hi (a bijection of s_lo: no two steps below 2^32 share a key); pair words
// (w0, w1) = Philox2x32-10({min id, max id}, k_s).
// ---------------------------------------------------------------------------------------
constexpr uint32_t kPhilox2M = 0xD256D193u;
constexpr uint32_t kPhilox2W = 0x9E3779B9u;

__device__ __forceinline__ uint2 philox2x32_10(uint32_t c0, uint32_t c1, uint32_t k)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi = __umulhi(kPhilox2M, c0), lo = kPhilox2M * c0;
        c0 = hi ^ k ^ c1;
        c1 = lo;
        k += kPhilox2W;
    }
    return make_uint2(c0, c1);
}

// MurmurHash3's 32-bit finalizer: five bijective steps (xor-shifts, odd multipliers).
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h)
{
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

__host__ __device__ __forceinline__ uint32_t step_key(uint32_t s_lo, uint32_t s_hi, uint32_t seed_lo,
                                                      uint32_t seed_hi)
{
    return fmix32(s_lo ^ seed_lo ^ fmix32(s_hi)) ^ seed_hi;
}

// Words (w0, w1) of the pair (ida, idb) under the per-step key ks.
__device__ __forceinline__ uint2 pair_words(uint32_t ida, uint32_t idb, uint32_t ks)
{
    return philox2x32_10(min(ida, idb), max(ida, idb), ks);
}

// The ten round keys k_s + r W of one step, computed once on the host: as a kernel
// parameter they sit in the constant bank and feed the round's LOP3 directly (no per-pair
// key schedule).
struct RoundKeys {
    uint32_t k[10];
};

__device__ __forceinline__ uint2 pair_words(uint32_t ida, uint32_t idb, const RoundKeys &K)
{
    uint32_t c0 = min(ida, idb), c1 = max(ida, idb);
#ifndef PROBE_ROUNDS // timing probe only (tools/build_variants.sh): other values break C-7 parity
#define PROBE_ROUNDS 10
#endif
#pragma unroll
    for (int r = 0; r < PROBE_ROUNDS; ++r) {
        const uint32_t hi = __umulhi(kPhilox2M, c0), lo = kPhilox2M * c0;
        c0 = hi ^ K.k[r] ^ c1;
        c1 = lo;
    }
    return make_uint2(c0, c1);
}

__device__ __forceinline__ RoundKeys round_keys(uint32_t ks)
{
    RoundKeys K;
#pragma unroll
    for (int r = 0; r < 10; ++r) K.k[r] = ks + (uint32_t)r * kPhilox2W;
    return K;
}

__device__ __forceinline__ float sqrt_approx(float x)
{
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Box-Muller (C-7): u1 = (w0 + 1) 2^-32 in (0, 1], u2 = w1 2^-32;
// xi = sqrt(-2 ln u1) cos(2 pi u2).  cos is evaluated on the signed image of u2 in
// [-1/2, 1/2) so the fast cosine sees |arg| <= pi.
// box_muller_s returns xi / kBM with kBM = sqrt(2 ln 2): -2 ln u1 = 2 ln 2 (-log2 u1), so the
// constant leaves the per-pair path and is folded into sigma/sqrt(dt) on the host (PairP).
constexpr float kBM = 1.1774100225154747f; // sqrt(2 ln 2)

__device__ __forceinline__ float box_muller_s(uint32_t w0, uint32_t w1)
{
    const float two_m32 = 2.3283064365386963e-10f; // 2^-32
    const float u1 = __fmaf_rn(__uint2float_rn(w0), two_m32, two_m32);
    const float rad = sqrt_approx(fmaxf(-__log2f(u1), 0.0f));
    return rad * __cosf(__int2float_rn((int)w1) * (6.283185307179586f * two_m32));
}

__device__ __forceinline__ float box_muller(uint32_t w0, uint32_t w1)
{
    return kBM * box_muller_s(w0, w1);
}

// w_R for the kernel exponent k (C-4): k = 1/2 -> sqrt(w); k = 1 -> w; else w^k.
template <int KMODE>
__device__ __forceinline__ float weight_R(float w, float k)
{
    if constexpr (KMODE == 0) return sqrt_approx(w);
    else if constexpr (KMODE == 1) return w;
    else return w > 0.0f ? exp2f(k * __log2f(w)) : 0.0f; // 2 (generic k) and 3 (species matrix)
}

// Scalar pair force along d = r_i - r_j: returns s such that f_ij = s * d, and
// the force magnitude mag (for the fixed-point range check of the tiled kernel).
//   mag = a w - gamma w_D (e . v_ij) + sigma/sqrt(dt) w_R xi ;  s = mag / r
// r2 in (0, rc2) assumed.  KMODE 0: k = 1/2, 1: k = 1, 2: generic k, 3: generic k with the
// species matrix (a, gamma, sigma of the pair looked up from the species ti, tj).
// pp.sig_dt / pp.ss hold sigma/sqrt(dt) * kBM (box_muller_s convention).
template <int KMODE, class KeyT>
__device__ __forceinline__ float pair_mag(const PairP &pp, float r2, float dvdot, uint32_t idi, uint32_t idj,
                                          const KeyT &ks, int ti, int tj, float &mag)
{
    float a = pp.a, gamma = pp.gamma, sig_dt = pp.sig_dt;
    if constexpr (KMODE == 3) {
        const int t = ti * DPD_MAX_SPECIES + tj;
        a = pp.sa[t];
        gamma = pp.sg[t];
        sig_dt = pp.ss[t];
    }
    const float rinv = rsqrtf(r2);
    const float r = r2 * rinv;
    const float w = fmaxf(__fmaf_rn(-r, pp.inv_rc, 1.0f), 0.0f);
    const float wR = weight_R<KMODE>(w, pp.power);
    const uint2 wd = pair_words(idi, idj, ks);
    const float xr = box_muller_s(wd.x, wd.y) * wR;
    float cons;
    if constexpr (KMODE == 0) cons = w * __fmaf_rn(-gamma, dvdot * rinv, a); // w_D = w_R^2 = w
    else cons = __fmaf_rn(a, w, -gamma * (wR * wR) * (dvdot * rinv));
    mag = __fmaf_rn(xr, sig_dt, cons);
    return mag * rinv;
}

template <int KMODE, class KeyT>
__device__ __forceinline__ float pair_scalar(const PairP &pp, float r2, float dvdot, uint32_t idi, uint32_t idj,
                                             const KeyT &ks, float vwi, float vwj)
{
    float mag;
    return pair_mag<KMODE>(pp, r2, dvdot, idi, idj, ks, __float_as_int(vwi), __float_as_int(vwj), mag);
}

// Cell coordinate along one dimension (C-8): min((int)(x * inv_h), n - 1), fp32 product.
__device__ __forceinline__ int cell_coord(float x, float inv_h, int n)
{
    const int q = __float2int_rz(__fmul_rn(x, inv_h));
    return min(max(q, 0), n - 1);
}

} // namespace dpd
