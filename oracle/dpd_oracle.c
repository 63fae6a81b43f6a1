/*
 * dpd_oracle.c -- plain, slow, double-precision CPU oracle for the DPD solvent step
 * of Mirheo (Alexeev et al., arXiv:1911.04712).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_1911_04712_b200/csrc)
 * and neither side includes or links the other.
 *
 * Citation convention: "P:n" = /root/reference/PAPER.md line n (section named),
 * "S:n" = SPEC.md line n, "C-n" = the reading adopted in DESIGN.md §3.
 *
 * What it computes (all in fp64 unless stated):
 *   - Philox2x32-10 / Philox4x32-10 (Random123) counter-based generators  (C-7)
 *   - per-pair Gaussian xi by Box-Muller on words w0,w1                  (C-7)
 *   - DPD pair force F^C + F^D + F^R                      (eqs. 2-5; C-3..C-5)
 *   - all-pairs O(N^2) minimum-image force sum (the plain definition)    (C-1)
 *   - cell index / counts / starts, in fp32 arithmetic                   (C-8)
 *   - Groot-Warren velocity Verlet, lambda = 1/2 ("fused VV")            (C-6)
 *   - observables: kinetic T (full-step v), conservative virial p       (C-14, C-15)
 *   - an fp64 cell-list sweep (CPU timing mode, never used as truth)    (C-2 item 7)
 *   - per-pair (a, gamma) from a species matrix
 *   - SDF walls: frozen layer, bounce-back
 *
 * Parity pins: see tests/test_oracle_*.py (Random123 KATs, hand examples S:194/S:196,
 * closed forms, invariants, brute force vs cell list, T = kT, Groot-Warren EOS).
 * Nothing in this file is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    double box[3];  /* periodic box edge lengths L_x, L_y, L_z   */
    double rc;      /* cutoff radius r_c */
    double a;       /* conservative amplitude alpha     */
    double gamma;   /* dissipative coefficient     */
    double kT;      /* k_B T; sigma = sqrt(2 gamma kT)     */
    double power;   /* k: w_R = w^k, w_D = w_R^2                             (C-4)*/
    double dt;      /* time step                                             (C-3)       */
    uint64_t seed;  /* Philox key                                            (C-7)       */
    double body_f;  /* periodic-Poiseuille body force magnitude f */
    /* Species interaction matrix: with nspecies > 1 and a
     * species array, the pair (i, j) uses a = amat[s_i][s_j], gamma = gmat[s_i][s_j] and
     * sigma = sqrt(2 gamma kT) (per pair) in place of a, gamma above.            */
    int32_t nspecies;        /* 0 or 1: single species                                */
    double amat[16];         /* nspecies x nspecies, row-major (nspecies <= 4)        */
    double gmat[16];
    const int32_t *species;  /* species of particle index i (NULL: all 0)             */
    /* SDF walls, reading C-23: the solid is the
     * union of up to 4 primitives, s(x) = max_k s_k(x) > 0 inside the solid; particles of
     * a frozen species (bit s of frozen_mask) never move and keep the wall velocity.     */
    int32_t nwall;           /* number of primitives (0: no walls)                     */
    int32_t wtype[4];        /* 1 plane: s = n.x - c, prm (nx, ny, nz, c), |n| = 1;
                                2/3/4 cylinder along x/y/z: prm (c1, c2, R, sign),
                                s = sign (R - dist to the axis) (+1 post, -1 pipe)     */
    double wprm[16];
    double wvel[12];         /* translational wall velocity of each primitive           */
    int32_t frozen_mask;
    int32_t body_mode;       /* 0: periodic Poiseuille; 1: uniform +f along z */
} oracle_params;

/* Signed distance of one primitive (C-23). */
static double wall_prim(const oracle_params *p, int k, const double x[3])
{
    const double *q = &p->wprm[4 * k];
    if (p->wtype[k] == 1) return q[0] * x[0] + q[1] * x[1] + q[2] * x[2] - q[3];
    const int ax = p->wtype[k] - 2, a = (ax + 1) % 3, b = (ax + 2) % 3;
    const double da = x[a] - q[0], db = x[b] - q[1];
    return q[3] * (q[2] - sqrt(da * da + db * db));
}

/* s(x) = max_k s_k(x) (union of solids); uw (may be NULL) = velocity of the maximising
 * primitive.  Without walls s = -inf. */
double oracle_wall_sdf(const oracle_params *p, const double x[3], double uw[3])
{
    double best = -INFINITY;
    int arg = -1;
    for (int k = 0; k < p->nwall; ++k) {
        double sk = wall_prim(p, k, x);
        if (sk > best) { best = sk; arg = k; }
    }
    if (uw) {
        for (int c = 0; c < 3; ++c) uw[c] = arg >= 0 ? p->wvel[3 * arg + c] : 0.0;
    }
    return best;
}

static int is_frozen(const oracle_params *p, int64_t i)
{
    const int32_t sp = p->species ? p->species[i] : 0;
    return (p->frozen_mask >> sp) & 1;
}

/* The parameters of pair (i, j): p itself, or a copy with the pair's (a, gamma). */
static const oracle_params *pair_params(const oracle_params *p, int64_t i, int64_t j, oracle_params *q)
{
    if (p->nspecies <= 1 || !p->species) return p;
    *q = *p;
    const int32_t ns = p->nspecies, si = p->species[i], sj = p->species[j];
    q->a = p->amat[si * ns + sj];
    q->gamma = p->gmat[si * ns + sj];
    return q;
}

/* ------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11 "Random123"), as fixed by reading C-7.
 * Round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2;
 *        c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key bump k += (W0, W1).
 * Ten rounds, key bumped between rounds.
 * ---------------------------------------------------------------------------------- */
static const uint32_t PHILOX_M0 = 0xD2511F53u, PHILOX_M1 = 0xCD9E8D57u;
static const uint32_t PHILOX_W0 = 0x9E3779B9u, PHILOX_W1 = 0xBB67AE85u;

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
        uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Philox2x32-10 (Random123): round (hi, lo) = M * c0; c' = (hi ^ k ^ c1, lo); k += W. */
static const uint32_t PHILOX2_M = 0xD256D193u, PHILOX2_W = 0x9E3779B9u;

void oracle_philox2x32_10(const uint32_t ctr[2], uint32_t key, uint32_t out[2])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], k = key;
    for (int round = 0; round < 10; ++round) {
        if (round > 0) k += PHILOX2_W;
        uint64_t p = (uint64_t)PHILOX2_M * (uint64_t)c0;
        uint32_t hi = (uint32_t)(p >> 32), lo = (uint32_t)p;
        uint32_t n0 = hi ^ k ^ c1;
        c0 = n0;
        c1 = lo;
    }
    out[0] = c0;
    out[1] = c1;
}

/* MurmurHash3's 32-bit finalizer fmix32 (A. Appleby, public domain): xor-shift by 16,
 * multiply by 0x85ebca6b, xor-shift by 13, multiply by 0xc2b2ae35, xor-shift by 16.  Each
 * of the five steps is a bijection of the 32-bit words (odd multipliers are invertible mod
 * 2^32), so fmix32 is a permutation with fmix32(0) = 0. */
uint32_t oracle_fmix32(uint32_t h)
{
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}

/* Per-step key (C-7, revised in round 2 so that <xi(t) xi(t')> = delta(t - t'), holds
 * over a whole run):  k_s = fmix32(s_lo ^ seed_lo ^ fmix32(s_hi)) ^ seed_hi.
 * For a fixed seed and s_hi the map s_lo -> k_s is a composition of bijections, so no two
 * steps 0 <= s < 2^32 share a key; the 64-bit seed enters as (seed_lo, seed_hi) without
 * folding, so two seeds give the same key sequence only if they are equal. */
uint32_t oracle_step_key(uint64_t seed, int64_t step)
{
    uint64_t s = (uint64_t)step;
    uint32_t s_lo = (uint32_t)s, s_hi = (uint32_t)(s >> 32);
    uint32_t seed_lo = (uint32_t)seed, seed_hi = (uint32_t)(seed >> 32);
    return oracle_fmix32(s_lo ^ seed_lo ^ oracle_fmix32(s_hi)) ^ seed_hi;
}

/* Step keys of n consecutive steps s0, s0 + 1, ... (test helper for the injectivity pin). */
void oracle_step_keys(uint64_t seed, int64_t s0, int64_t n, uint32_t *out)
{
    for (int64_t k = 0; k < n; ++k) out[k] = oracle_step_key(seed, s0 + k);
}

/* Pair words (C-7): (w0, w1) = Philox2x32-10(ctr = {min id, max id}, key = k_s).
 * Symmetric in (ida, idb) by construction: xi_ij = xi_ji; a fresh key per step
 * makes xi delta-correlated in time. */
void oracle_pair_words(uint64_t seed, int64_t step, uint32_t ida, uint32_t idb, uint32_t w[2])
{
    uint32_t ctr[2];
    ctr[0] = ida < idb ? ida : idb;
    ctr[1] = ida < idb ? idb : ida;
    oracle_philox2x32_10(ctr, oracle_step_key(seed, step), w);
}

/* Box-Muller (C-7): u1 = (w0+1) 2^-32 in (0,1], u2 = w1 2^-32 in [0,1),
 * xi = sqrt(-2 ln u1) cos(2 pi u2): zero-mean, unit-variance Gaussian. */
double oracle_xi(uint32_t w0, uint32_t w1)
{
    const double two_m32 = 1.0 / 4294967296.0;
    double u1 = ((double)w0 + 1.0) * two_m32;
    double u2 = (double)w1 * two_m32;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* Minimum-image separation d = x_i - x_j, d_k -= L_k rint(d_k / L_k)  (C-1). */
void oracle_min_image(const oracle_params *p, const double xi[3], const double xj[3], double d[3])
{
    for (int k = 0; k < 3; ++k) {
        double dk = xi[k] - xj[k];
        dk -= p->box[k] * rint(dk / p->box[k]);
        d[k] = dk;
    }
}

/* DPD pair force on i due to j:
 *   F^C = a w(r) e,  w = 1 - r/r_c  for r < r_c                       (eqs. 3-4)
 *   F^D = -gamma w_D(r) (v_ij . e) e                                    (eq. 5)
 *   F^R = sigma xi_ij w_R(r) e / sqrt(dt)                               (eq. 5, C-3)
 *   w_R = w^k, w_D = w_R^2, sigma^2 = 2 gamma kT                        (C-4)
 * d = r_i - r_j (minimum image), vij = v_i - v_j (C-5).
 * Interacts iff 0 < r^2 < r_c^2 (C-11).  Returns 1 and writes f if interacting, else
 * writes zero and returns 0.  xi_out (may be NULL) receives xi. */
int oracle_pair_force(const oracle_params *p, const double d[3], const double vij[3],
                      uint32_t ida, uint32_t idb, int64_t step, double f[3], double *xi_out)
{
    f[0] = f[1] = f[2] = 0.0;
    double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    if (!(r2 > 0.0 && r2 < p->rc * p->rc))
        return 0;
    double r = sqrt(r2);
    double e[3] = {d[0] / r, d[1] / r, d[2] / r};
    double w = 1.0 - r / p->rc;
    double wR = pow(w, p->power);
    double wD = wR * wR;
    double sigma = sqrt(2.0 * p->gamma * p->kT);
    uint32_t wds[2];
    oracle_pair_words(p->seed, step, ida, idb, wds);
    double xi = oracle_xi(wds[0], wds[1]);
    double ev = e[0] * vij[0] + e[1] * vij[1] + e[2] * vij[2];
    double mag = p->a * w - p->gamma * wD * ev + sigma * wR * xi / sqrt(p->dt);
    f[0] = mag * e[0];
    f[1] = mag * e[1];
    f[2] = mag * e[2];
    if (xi_out) *xi_out = xi;
    return 1;
}

/* Upper bound on |f| for a pair whose r lies within eps of r_c (reading C-12):
 * evaluates each term's magnitude at w = 2 eps / r_c, the largest w such a pair can
 * have under either precision's rounding of r. */
static double boundary_bound(const oracle_params *p, double eps, const double vij[3], double xi)
{
    double w = 2.0 * eps / p->rc;
    double wR = pow(w, p->power);
    double sigma = sqrt(2.0 * p->gamma * p->kT);
    double vabs = sqrt(vij[0] * vij[0] + vij[1] * vij[1] + vij[2] * vij[2]);
    return p->a * w + p->gamma * wR * wR * vabs + sigma * wR * fabs(xi) / sqrt(p->dt);
}

/* Boundary window of one pair (C-12): eps for pairs whose minimum image is the plain
 * difference, eps_image for pairs that reach across a periodic edge (some d_k needed a
 * shift by L_k): the fp32 path forms x_j + L_k there, which rounds at ulp(L_k). */
static double pair_window(const oracle_params *p, const double xi[3], const double xj[3], double eps,
                          double eps_image)
{
    for (int k = 0; k < 3; ++k)
        if (rint((xi[k] - xj[k]) / p->box[k]) != 0.0) return eps_image;
    return eps;
}

/* PairForces(x, v, s) -- the plain definition (C-1, C-2 item 4): for every particle i,
 * F_i = sum over all j != i of the pair force, minimum image, O(N^2).
 * x, v: n x 3 row-major; ids: global particle ids (C-7).
 * allow (may be NULL): per-particle sum of boundary_bound over pairs with |r - r_c| below the
 *   pair's window (eps, or eps_image across a periodic edge: pair_window, C-12);
 *   npairs (may be NULL): number of unordered interacting pairs. */
int oracle_forces(const oracle_params *p, int64_t n, const double *x, const double *v,
                  const uint32_t *ids, int64_t step, double eps, double eps_image, double *F, double *allow,
                  int64_t *npairs)
{
    int64_t count = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : count)
    for (int64_t i = 0; i < n; ++i) {
        double Fi[3] = {0.0, 0.0, 0.0};
        double al = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double d[3], vij[3], f[3], xi = 0.0;
            oracle_params q;
            const oracle_params *pp = pair_params(p, i, j, &q);
            oracle_min_image(p, &x[3 * i], &x[3 * j], d);
            for (int k = 0; k < 3; ++k) vij[k] = v[3 * i + k] - v[3 * j + k];
            int hit = oracle_pair_force(pp, d, vij, ids[i], ids[j], step, f, &xi);
            if (hit) {
                Fi[0] += f[0]; Fi[1] += f[1]; Fi[2] += f[2];
                if (j > i) count += 1;
            }
            if (allow) {
                double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                double w = pair_window(p, &x[3 * i], &x[3 * j], eps, eps_image);
                if (fabs(r - p->rc) < w) {
                    if (!hit) {
                        uint32_t wds[2];
                        oracle_pair_words(p->seed, step, ids[i], ids[j], wds);
                        xi = oracle_xi(wds[0], wds[1]);
                    }
                    al += boundary_bound(pp, w, vij, xi);
                }
            }
        }
        F[3 * i + 0] = Fi[0];
        F[3 * i + 1] = Fi[1];
        F[3 * i + 2] = Fi[2];
        if (allow) allow[i] = al;
    }
    if (npairs) *npairs = count;
    return 0;
}

/* PairForces restricted to the particles listed in sel[0..m): the same all-j sum as
 * oracle_forces for each selected i (sampled parity at full size, where the O(N^2) sweep
 * over every i is out of reach).  F and allow are m x 3 / m. */
int oracle_forces_subset(const oracle_params *p, int64_t n, const double *x, const double *v,
                         const uint32_t *ids, int64_t step, double eps, double eps_image, int64_t m,
                         const int64_t *sel, double *F, double *allow)
{
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < m; ++k) {
        const int64_t i = sel[k];
        double Fi[3] = {0.0, 0.0, 0.0};
        double al = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double d[3], vij[3], f[3], xi = 0.0;
            oracle_min_image(p, &x[3 * i], &x[3 * j], d);
            double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
            double wmax = eps > eps_image ? eps : eps_image;
            if (r2 >= (p->rc + wmax) * (p->rc + wmax)) continue; /* no force, not a boundary pair */
            for (int c = 0; c < 3; ++c) vij[c] = v[3 * i + c] - v[3 * j + c];
            oracle_params q;
            const oracle_params *pp = pair_params(p, i, j, &q);
            int hit = oracle_pair_force(pp, d, vij, ids[i], ids[j], step, f, &xi);
            if (hit) { Fi[0] += f[0]; Fi[1] += f[1]; Fi[2] += f[2]; }
            double r = sqrt(r2);
            double w = pair_window(p, &x[3 * i], &x[3 * j], eps, eps_image);
            if (fabs(r - p->rc) < w) {
                if (!hit) {
                    uint32_t wds[2];
                    oracle_pair_words(p->seed, step, ids[i], ids[j], wds);
                    xi = oracle_xi(wds[0], wds[1]);
                }
                al += boundary_bound(pp, w, vij, xi);
            }
        }
        F[3 * k + 0] = Fi[0];
        F[3 * k + 1] = Fi[1];
        F[3 * k + 2] = Fi[2];
        allow[k] = al;
    }
    return 0;
}

/* Enumerate unordered pairs (brute force), for pair-set / RNG-word parity (T3).
 * Every pair i<j that interacts (0 < r^2 < r_c^2) or lies within its window of the cutoff
 * (|r - r_c| < eps, or eps_image across a periodic edge: a boundary pair, C-12) is written as (min id, max id, w0, w1) into
 * quad[4*k..] with flag[k] = (interacts ? 1 : 0) | (boundary ? 2 : 0).  Returns the
 * total number of such pairs (may exceed cap; only the first cap are written). */
int64_t oracle_pairs(const oracle_params *p, int64_t n, const double *x, const uint32_t *ids,
                     int64_t step, double eps, double eps_image, int64_t cap, uint32_t *quad, uint8_t *flag)
{
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = i + 1; j < n; ++j) {
            double d[3];
            oracle_min_image(p, &x[3 * i], &x[3 * j], d);
            double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
            double r = sqrt(r2);
            int hit = (r2 > 0.0 && r2 < p->rc * p->rc);
            int near = fabs(r - p->rc) < pair_window(p, &x[3 * i], &x[3 * j], eps, eps_image);
            if (!hit && !near) continue;
            if (k < cap) {
                uint32_t wds[2];
                uint32_t lo = ids[i] < ids[j] ? ids[i] : ids[j];
                uint32_t hi = ids[i] < ids[j] ? ids[j] : ids[i];
                oracle_pair_words(p->seed, step, lo, hi, wds);
                quad[4 * k + 0] = lo;
                quad[4 * k + 1] = hi;
                quad[4 * k + 2] = wds[0];
                quad[4 * k + 3] = wds[1];
                flag[k] = (uint8_t)(hit | (near << 1));
            }
            ++k;
        }
    }
    return k;
}

/* Cell grid (C-8): n_d = floor(L_d / r_c); cell coordinate evaluated in fp32
 * arithmetic i_d = min((int)(x_d * ((float)n_d / (float)L_d)), n_d - 1);
 * linear index c = i_x + n_x (i_y + n_y i_z); counts and exclusive starts
 * (start[c] = sum_{c'<c} count[c'], start[Ncell] = N).  pos: n x 3 fp32 in [0, L). */
void oracle_grid_dims(const oracle_params *p, int32_t dims[3])
{
    for (int k = 0; k < 3; ++k) dims[k] = (int32_t)floor(p->box[k] / p->rc);
}

int oracle_cells(const oracle_params *p, int64_t n, const float *pos, int32_t *cell,
                 int32_t *count, int32_t *start)
{
    int32_t nd[3];
    oracle_grid_dims(p, nd);
    int64_t ncell = (int64_t)nd[0] * nd[1] * nd[2];
    float inv[3];
    for (int k = 0; k < 3; ++k) {
        volatile float nf = (float)nd[k];
        volatile float lf = (float)p->box[k];
        inv[k] = nf / lf;
    }
    for (int64_t c = 0; c < ncell; ++c) count[c] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t ic[3];
        for (int k = 0; k < 3; ++k) {
            volatile float prod = pos[3 * i + k] * inv[k]; /* one fp32 rounding */
            int32_t q = (int32_t)prod;
            ic[k] = q < nd[k] - 1 ? q : nd[k] - 1;
        }
        int32_t c = ic[0] + nd[0] * (ic[1] + nd[1] * ic[2]);
        cell[i] = c;
        count[c] += 1;
    }
    int32_t acc = 0;
    for (int64_t c = 0; c < ncell; ++c) {
        start[c] = acc;
        acc += count[c];
    }
    start[ncell] = acc;
    return 0;
}

/* Wrap into [0, L) (C-10): x<0 -> x+L; x>=L -> x-L; then x>=L -> 0. */
static double wrap1(double x, double L)
{
    if (x < 0.0) x += L;
    else if (x >= L) x -= L;
    if (x >= L) x = 0.0;
    return x;
}

/* Body force along z: periodic Poiseuille: (0,0,-f) for r_x <= L/2, else
 * (0,0,+f); body_mode 1: uniform (0,0,+f) (wall-bounded Poiseuille, NEXT-3). */
static double body_fz(const oracle_params *p, double rx)
{
    if (p->body_mode == 1) return p->body_f;
    return rx <= 0.5 * p->box[0] ? -p->body_f : p->body_f;
}

/* Kick-drift of one particle with wall bounce-back (C-6, C-23): u = v + kick
 * (F + f_body); x' = x + dt u.  If x' is inside the solid (s > 0) the collision time
 * t* in [0, dt] with s(x + t u) = 0 is found by bisection (80 halvings in fp64), the
 * particle is placed at x + t_lo u (the last point with s <= 0) and its velocity is
 * reversed in the wall frame, u <- 2 u_w - u.  Frozen particles do not move.  x' is then
 * wrapped (C-10).  Returns 1 if the particle bounced. */
static int kick_drift_one(const oracle_params *p, int64_t i, double *x, double *v, const double *F,
                          double kick)
{
    if (is_frozen(p, i)) return 0;
    double fz = body_fz(p, x[0]);
    double u[3] = {v[0] + kick * F[0], v[1] + kick * F[1], v[2] + kick * (F[2] + fz)};
    double xn[3] = {x[0] + p->dt * u[0], x[1] + p->dt * u[1], x[2] + p->dt * u[2]};
    int bounced = 0;
    if (p->nwall > 0 && oracle_wall_sdf(p, xn, NULL) > 0.0) {
        double lo = 0.0, hi = p->dt;
        if (oracle_wall_sdf(p, x, NULL) > 0.0) {
            hi = 0.0; /* already inside (never for a valid state): stay, reverse */
        } else {
            for (int it = 0; it < 80; ++it) {
                double mid = 0.5 * (lo + hi), xm[3];
                for (int c = 0; c < 3; ++c) xm[c] = x[c] + mid * u[c];
                if (oracle_wall_sdf(p, xm, NULL) > 0.0) hi = mid; else lo = mid;
            }
        }
        double uw[3];
        for (int c = 0; c < 3; ++c) xn[c] = x[c] + lo * u[c];
        oracle_wall_sdf(p, xn, uw);
        for (int c = 0; c < 3; ++c) u[c] = 2.0 * uw[c] - u[c];
        bounced = 1;
    }
    for (int c = 0; c < 3; ++c) {
        x[c] = wrap1(xn[c], p->box[c]);
        v[c] = u[c];
    }
    return bounced;
}

/* One kick-drift (+ bounce-back) of every particle in place: v <- u, x <- x'.  Returns the
 * number of bounces.  The per-step parity test predicts the GPU's x_s, u_s with it. */
int64_t oracle_kick_drift(const oracle_params *p, int64_t n, double *x, double *v, const double *F, double kick)
{
    int64_t nb = 0;
    for (int64_t i = 0; i < n; ++i) nb += kick_drift_one(p, i, &x[3 * i], &v[3 * i], &F[3 * i], kick);
    return nb;
}

/* Carve a fluid configuration with the walls (C-23): particles with s > r_c are
 * removed (keep[i] = 0), those with 0 < s <= r_c become the frozen layer (species :=
 * wall_species, v := u_w(x)), the rest is untouched.  Returns the number of frozen. */
int64_t oracle_wall_carve(const oracle_params *p, int64_t n, const double *x, double *v, int32_t *species,
                          int32_t wall_species, uint8_t *keep)
{
    int64_t nf = 0;
    for (int64_t i = 0; i < n; ++i) {
        double uw[3];
        double sd = oracle_wall_sdf(p, &x[3 * i], uw);
        keep[i] = sd <= p->rc;
        if (sd > 0.0 && sd <= p->rc) {
            species[i] = wall_species;
            for (int c = 0; c < 3; ++c) v[3 * i + c] = uw[c];
            ++nf;
        }
    }
    return nf;
}

/* Prime (C-2 item 2): F = PairForces(x, v, s). */
int oracle_prime(const oracle_params *p, int64_t n, const double *x, const double *v,
                 const uint32_t *ids, int64_t step, double *F)
{
    return oracle_forces(p, n, x, v, ids, step, 0.0, 0.0, F, NULL, NULL);
}

/* Groot-Warren velocity Verlet with lambda = 1/2, one force evaluation per step
 * (C-2 item 3, C-6).  State on entry: x_s, v_s (full-step), F_s.
 * Each step:  u  = v + dt/2 (F + f_body(x))
 *             x  = wrap(x + dt u)
 *             s  = s + 1
 *             F  = PairForces(x, u, s)
 *             v  = u + dt/2 (F + f_body(x))
 * u (n x 3, may be NULL) receives the last half-step velocity used for F. */
int oracle_step(const oracle_params *p, int64_t n, double *x, double *v, double *F,
                const uint32_t *ids, int64_t *step, int64_t nsteps, double *u_out)
{
    double *u = (double *)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    if (!u) return 1;
    for (int64_t it = 0; it < nsteps; ++it) {
        memcpy(u, v, sizeof(double) * 3 * (size_t)n);
        oracle_kick_drift(p, n, x, u, F, 0.5 * p->dt);
        *step += 1;
        oracle_forces(p, n, x, u, ids, *step, 0.0, 0.0, F, NULL, NULL);
        for (int64_t i = 0; i < n; ++i) {
            if (is_frozen(p, i)) { /* the wall velocity, unchanged */
                for (int k = 0; k < 3; ++k) v[3 * i + k] = u[3 * i + k];
                continue;
            }
            double fz = body_fz(p, x[3 * i + 0]);
            v[3 * i + 0] = u[3 * i + 0] + 0.5 * p->dt * F[3 * i + 0];
            v[3 * i + 1] = u[3 * i + 1] + 0.5 * p->dt * F[3 * i + 1];
            v[3 * i + 2] = u[3 * i + 2] + 0.5 * p->dt * (F[3 * i + 2] + fz);
        }
    }
    if (u_out) memcpy(u_out, u, sizeof(double) * 3 * (size_t)n);
    free(u);
    return 0;
}

/* Kinetic temperature from full-step velocities (C-14):
 * T = sum |v_i - vbar|^2 / (3 (N - 1)), m = 1 (C-18). */
double oracle_temperature(int64_t n, const double *v)
{
    if (n < 2) return 0.0;
    double m[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) m[k] += v[3 * i + k];
    for (int k = 0; k < 3; ++k) m[k] /= (double)n;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            double d = v[3 * i + k] - m[k];
            s += d * d;
        }
    return s / (3.0 * (double)(n - 1));
}

/* Conservative virial sum W = sum_{i<j} a w(r) r (C-2 item 6), so that
 * p = rho T + W / (3 V).  Brute force, minimum image; single species (uses p->a). */
double oracle_virial(const oracle_params *p, int64_t n, const double *x)
{
    double W = 0.0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : W)
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = i + 1; j < n; ++j) {
            double d[3];
            oracle_min_image(p, &x[3 * i], &x[3 * j], d);
            double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
            if (r2 > 0.0 && r2 < p->rc * p->rc) {
                double r = sqrt(r2);
                W += p->a * (1.0 - r / p->rc) * r;
            }
        }
    }
    return W;
}

/* ------------------------------------------------------------------------------------
 * CPU-timing mode (C-2 item 7): the same per-pair arithmetic (oracle_min_image +
 * oracle_pair_force) restricted to the 27 cells around each particle's cell, fp64 cells
 * of edge >= r_c.  Every pair within r_c lies in adjacent cells, so the pair set equals
 * the brute-force set (pinned by tests/test_oracle_celllist.py); only the order of
 * summation differs.  Requires n_d >= 3.
 * ---------------------------------------------------------------------------------- */
int oracle_forces_celllist(const oracle_params *p, int64_t n, const double *x, const double *v,
                           const uint32_t *ids, int64_t step, double *F, int64_t *npairs)
{
    int32_t nd[3];
    oracle_grid_dims(p, nd);
    if (nd[0] < 3 || nd[1] < 3 || nd[2] < 3) return 2;
    int64_t ncell = (int64_t)nd[0] * nd[1] * nd[2];
    int64_t *start = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
    int64_t *fill = (int64_t *)calloc((size_t)ncell, sizeof(int64_t));
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int32_t *cellof = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!start || !fill || !order || !cellof) return 1;
    for (int64_t i = 0; i < n; ++i) {
        int32_t ic[3];
        for (int k = 0; k < 3; ++k) {
            int32_t q = (int32_t)(x[3 * i + k] * nd[k] / p->box[k]);
            if (q < 0) q = 0;
            ic[k] = q < nd[k] - 1 ? q : nd[k] - 1;
        }
        cellof[i] = ic[0] + nd[0] * (ic[1] + nd[1] * ic[2]);
        start[cellof[i] + 1] += 1;
    }
    for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
    for (int64_t i = 0; i < n; ++i) {
        int32_t c = cellof[i];
        order[start[c] + fill[c]] = i;
        fill[c] += 1;
    }
    int64_t count = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : count)
    for (int64_t i = 0; i < n; ++i) {
        int32_t c = cellof[i];
        int32_t cx = c % nd[0], cy = (c / nd[0]) % nd[1], cz = c / (nd[0] * nd[1]);
        double Fi[3] = {0.0, 0.0, 0.0};
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int32_t jx = (cx + dx + nd[0]) % nd[0];
                    int32_t jy = (cy + dy + nd[1]) % nd[1];
                    int32_t jz = (cz + dz + nd[2]) % nd[2];
                    int32_t cj = jx + nd[0] * (jy + nd[1] * jz);
                    for (int64_t t = start[cj]; t < start[cj + 1]; ++t) {
                        int64_t j = order[t];
                        if (j == i) continue;
                        double d[3], vij[3], f[3];
                        oracle_min_image(p, &x[3 * i], &x[3 * j], d);
                        for (int k = 0; k < 3; ++k) vij[k] = v[3 * i + k] - v[3 * j + k];
                        oracle_params q;
                        if (oracle_pair_force(pair_params(p, i, j, &q), d, vij, ids[i], ids[j], step, f, NULL)) {
                            Fi[0] += f[0]; Fi[1] += f[1]; Fi[2] += f[2];
                            if (j > i) count += 1;
                        }
                    }
                }
        F[3 * i + 0] = Fi[0];
        F[3 * i + 1] = Fi[1];
        F[3 * i + 2] = Fi[2];
    }
    if (npairs) *npairs = count;
    free(start); free(fill); free(order); free(cellof);
    return 0;
}

/* Same GW-VV step as oracle_step but with the cell-list force sweep (timing mode). */
int oracle_step_celllist(const oracle_params *p, int64_t n, double *x, double *v, double *F,
                         const uint32_t *ids, int64_t *step, int64_t nsteps)
{
    double *u = (double *)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    if (!u) return 1;
    int rc = 0;
    for (int64_t it = 0; it < nsteps && rc == 0; ++it) {
        memcpy(u, v, sizeof(double) * 3 * (size_t)n);
        oracle_kick_drift(p, n, x, u, F, 0.5 * p->dt);
        *step += 1;
        rc = oracle_forces_celllist(p, n, x, u, ids, *step, F, NULL);
        for (int64_t i = 0; i < n; ++i) {
            if (is_frozen(p, i)) {
                for (int k = 0; k < 3; ++k) v[3 * i + k] = u[3 * i + k];
                continue;
            }
            double fz = body_fz(p, x[3 * i + 0]);
            v[3 * i + 0] = u[3 * i + 0] + 0.5 * p->dt * F[3 * i + 0];
            v[3 * i + 1] = u[3 * i + 1] + 0.5 * p->dt * F[3 * i + 1];
            v[3 * i + 2] = u[3 * i + 2] + 0.5 * p->dt * (F[3 * i + 2] + fz);
        }
    }
    free(u);
    return rc;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the OpenMP loops (CPU-timing legs of bench.py: 1 thread and all). */
void oracle_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
