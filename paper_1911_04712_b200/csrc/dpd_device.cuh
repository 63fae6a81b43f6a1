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

// Pair-force parameters.
struct PairP {
    float a;        // conservative amplitude
    float gamma;    // dissipative coefficient
    float sig_dt;   // sigma / sqrt(dt), sigma = sqrt(2 gamma kT)            (C-3)
    float inv_rc;   // 1 / r_c
    float rc2;      // r_c^2
    float power;    // k (w_R = w^k)                                         (C-4)
    uint32_t k0;    // Philox key words = seed lo, seed hi                   (C-7)
    uint32_t k1;
};

// Integrator parameters (C-2 item 3 / C-6).
struct IntegP {
    float dt;       // drift time step (0 when only re-binning at set time)
    float kick;     // velocity kick factor: dt/2 on the first step after set, dt after
    float body_f;   // periodic-Poiseuille magnitude f
    float x_half;   // global L_x / 2 expressed in local coordinates
};

// ---------------------------------------------------------------------------------------
// Philox4x32-10 (C-7).  ctr = {lo id, hi id, step lo, step hi}, key = {k0, k1}.
// Only output words 0 and 1 are needed, so the 10th round skips the M0 product.
// ---------------------------------------------------------------------------------------
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(kPhiloxM0, c.x), lo0 = kPhiloxM0 * c.x;
        const uint32_t hi1 = __umulhi(kPhiloxM1, c.z), lo1 = kPhiloxM1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return c;
}

// Words (w0, w1) of the pair (ida, idb) at step s.
__device__ __forceinline__ uint2 pair_words(uint32_t ida, uint32_t idb, uint32_t s_lo, uint32_t s_hi,
                                            uint32_t k0, uint32_t k1)
{
    const uint32_t lo = min(ida, idb), hi = max(ida, idb);
    uint32_t c0 = lo, c1 = hi, c2 = s_lo, c3 = s_hi;
#pragma unroll
    for (int r = 0; r < 9; ++r) {
        const uint32_t hi0 = __umulhi(kPhiloxM0, c0), lo0 = kPhiloxM0 * c0;
        const uint32_t hi1 = __umulhi(kPhiloxM1, c2), lo1 = kPhiloxM1 * c2;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    // round 10: outputs 0 and 1 only depend on the M1 product
    const uint32_t hi1 = __umulhi(kPhiloxM1, c2), lo1 = kPhiloxM1 * c2;
    return make_uint2(hi1 ^ c1 ^ k0, lo1);
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
__device__ __forceinline__ float box_muller(uint32_t w0, uint32_t w1)
{
    const float two_m32 = 2.3283064365386963e-10f; // 2^-32
    const float u1 = __fmaf_rn(__uint2float_rn(w0), two_m32, two_m32);
    const float m2ln = -2.0f * __logf(u1);
    const float rad = sqrt_approx(fmaxf(m2ln, 0.0f));
    const float u2s = __int2float_rn((int)w1) * two_m32;
    return rad * __cosf(6.283185307179586f * u2s);
}

// w_R for the kernel exponent k (C-4): k = 1/2 -> sqrt(w); k = 1 -> w; else w^k.
template <int KMODE>
__device__ __forceinline__ float weight_R(float w, float k)
{
    if constexpr (KMODE == 0) return sqrt_approx(w);
    else if constexpr (KMODE == 1) return w;
    else return w > 0.0f ? exp2f(k * __log2f(w)) : 0.0f;
}

// Scalar pair force along d = r_i - r_j: returns s such that f_ij = s * d.
//   mag = a w - gamma w_D (e . v_ij) + sigma/sqrt(dt) w_R xi ;  s = mag / r
// r2 in (0, rc2) assumed.
template <int KMODE>
__device__ __forceinline__ float pair_scalar(const PairP &pp, float r2, float dvdot, uint32_t idi, uint32_t idj,
                                             uint32_t s_lo, uint32_t s_hi)
{
    const float rinv = rsqrtf(r2);
    const float r = r2 * rinv;
    const float w = fmaxf(__fmaf_rn(-r, pp.inv_rc, 1.0f), 0.0f);
    const float wR = weight_R<KMODE>(w, pp.power);
    const float wD = (KMODE == 0) ? w : wR * wR;
    const uint2 wd = pair_words(idi, idj, s_lo, s_hi, pp.k0, pp.k1);
    const float xi = box_muller(wd.x, wd.y);
    const float mag = pp.a * w - pp.gamma * wD * (dvdot * rinv) + pp.sig_dt * wR * xi;
    return mag * rinv;
}

// Cell coordinate along one dimension (C-8): min((int)(x * inv_h), n - 1), fp32 product.
__device__ __forceinline__ int cell_coord(float x, float inv_h, int n)
{
    const int q = __float2int_rz(__fmul_rn(x, inv_h));
    return min(max(q, 0), n - 1);
}

} // namespace dpd
