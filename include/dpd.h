/*
 * dpd.h -- C-ABI of the B200-native DPD solvent step (Mirheo, arXiv:1911.04712).
 *
 * One library (libdpd.so, sources in paper_1911_04712_b200/csrc/) owns all device state.
 * Every entry point is extern "C", takes plain pointers and sizes, and returns one of the
 * DPD_* status codes below (never throws, never aborts).  On failure the context keeps a
 * message readable with dpd_last_error().  A context is NOT thread-safe: calls on one
 * context must be serialised by the caller.
 *
 * Citation convention: P:n = PAPER.md line n (section named), C-n = reading adopted in
 * DESIGN.md §3.  The method:
 *   - particles evolve by Newton's law dr/dt = v, dv/dt = F/m, m = 1      (C-18)
 *   - F_i = sum_j (F^C + F^D + F^R) over j within r_c                     (eq. 2)
 *     F^C = a w e, w = 1 - r/r_c;  F^D = -gamma w_D (v_ij.e) e;
 *     F^R = sigma xi_ij w_R e / sqrt(dt);  w_R = w^k, w_D = w_R^2,
 *     sigma^2 = 2 gamma kT                                               (C-3, C-4)
 *   - xi_ij by Box-Muller on (w0, w1) = Philox2x32-10(ctr = {min id, max id}, key = k_s),
 *     k_s = fmix32(step_lo ^ seed_lo ^ fmix32(step_hi)) ^ seed_hi, a bijection of step_lo
 *     (no two steps below 2^32 share a key; fmix32 = MurmurHash3's finalizer) (C-7)
 *   - cell lists of edge >= r_c rebuilt every step
 *   - "fused Velocity-Verlet" = Groot-Warren VV, lambda = 1/2             (C-6)
 *   - 3D domain decomposition with ghost exchange and redistribution
 *
 * Host-side layouts: positions / velocities / forces are n x 3 row-major float32 (AoS
 * xyz).  Pointers passed to set/get may be host (pageable or pinned) or device memory
 * (copies use cudaMemcpyDefault under unified addressing).  Positions outside [0, L) are
 * wrapped on input (C-10).
 */
#ifndef DPD_H
#define DPD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dpd_ctx dpd_ctx; /* opaque; owns all device memory of one (sub)domain */

enum {
    DPD_OK = 0,
    DPD_ERR_ARG = 1,      /* bad argument (null pointer, n mismatch, ids not dense, ...)   */
    DPD_ERR_CONFIG = 2,   /* invalid parameters: rc<=0, box < 3 rc, power not in (0,1] ... */
    DPD_ERR_CUDA = 3,     /* CUDA runtime error (message in dpd_last_error)               */
    DPD_ERR_NUMERIC = 4,  /* non-finite position/velocity/force (input or during a step)  */
    DPD_ERR_CAPACITY = 5, /* a device buffer (cell, ghost, migration) overflowed          */
    DPD_ERR_COMM = 6,     /* NCCL error (multi-GPU)                                       */
    DPD_ERR_IO = 7        /* file I/O error of the asynchronous writer (dumps, dpd_ioq)   */
};

/* Create a single-GPU context on the current CUDA device for a periodic box.
 *   box[3]  : box edge lengths L_x, L_y, L_z (> 0; each >= 3 rc so the 27-cell stencil
 *             has distinct cells)
 *   rc      : cutoff radius (> 0)
 *   a       : conservative amplitude (>= 0)
 *   gamma   : dissipative coefficient (>= 0)
 *   kT      : temperature (>= 0); sigma = sqrt(2 gamma kT) is derived
 *   power   : kernel exponent k in (0, 1]; w_R = w^k                          P:136, C-4
 *   dt      : time step (> 0)
 *   seed    : 64-bit seed of the pair RNG (enters the per-step key unfolded)   C-7
 *   out     : receives the new context (NULL on failure)
 * Returns DPD_OK, DPD_ERR_ARG (out == NULL), DPD_ERR_CONFIG or DPD_ERR_CUDA. */
int dpd_create(const double box[3], double rc, double a, double gamma, double kT,
               double power, double dt, uint64_t seed, dpd_ctx **out);

/* Destroy a context and free its device memory.  NULL is a no-op. */
void dpd_destroy(dpd_ctx *ctx);

/* Message for the last failed call on ctx ("" if none).  Owned by ctx. */
const char *dpd_last_error(const dpd_ctx *ctx);

/* Launch all work on this CUDA stream (a cudaStream_t; NULL = the context's own
 * non-blocking stream, the default).  The caller keeps ownership of the stream. */
int dpd_set_stream(dpd_ctx *ctx, void *cuda_stream);

/* Engine options (name, value):
 *   "force_kernel" 0 = tiled shared-memory kernel with fixed-point accumulation (default,
 *                  DESIGN.md §6), 1 = reference thread-per-particle kernel with fp32
 *                  global atomics (P:276-278 mapping; kept as a cross-check), 2 = cell-warp
 *                  variant of the tiled kernel (one warp per home cell; same results up
 *                  to fp32 summation order).  1 and 2 are single-domain only.
 *   "message_capacity_percent" (distributed contexts) scales the per-direction message
 *                  capacities (default 100; >= 10).  Capacities follow the set's global mean
 *                  density; a strongly non-uniform set (a dense block in an empty box) needs
 *                  head-room here, else the step returns DPD_ERR_CAPACITY (nothing is written
 *                  past a slot).
 *   "tile_persistent" 1 = run the tiled kernel as resident CTAs walking the tiles (the next
 *                  tile's cell table and staging overlap the current tile's pairs / flush);
 *                  0 = one CTA per tile (default, measured faster: DESIGN.md §6).
 *   "body_force_mode" 0 = periodic Poiseuille (default), 1 = uniform +f along z.
 *   "dump_delay_us" (after dpd_dump_open) sleep this long before each snapshot write: a
 *                  simulated slow disk for overlap tests (default 0).
 *   "row_pruning"  1 = prune stencil rows / end cells farther than r_c (default), 0 = off.
 * Out-of-range values -> DPD_ERR_ARG; unknown names -> DPD_ERR_ARG. */
int dpd_set_option(dpd_ctx *ctx, const char *name, int64_t value);

/* Engine statistics (cumulative since creation), name -> *value:
 *   "fallback_tiles"      tiles of the tiled force kernel that exceeded a shared-memory
 *                         capacity and were evaluated by its global-memory fallback;
 *   "fallback_staged", "fallback_home"  the same split by cause (staged / home capacity);
 *   "full_list_particles" home particles whose pair list filled up, so that the rest of
 *                         their candidates were evaluated in place (still exact).
 * Unknown names -> DPD_ERR_ARG. */
int dpd_get_stat(dpd_ctx *ctx, const char *name, int64_t *value);

/* Species interaction matrix (fluids of different
 * viscosity, conservative-only or viscous-only cross interactions are per-pair choices of
 * a and gamma).  a and gamma are nspecies x nspecies row-major, symmetric, finite, >= 0;
 * the pair of species (s_i, s_j) interacts with a_{s_i s_j}, gamma_{s_i s_j} and
 * sigma_{s_i s_j} = sqrt(2 gamma_{s_i s_j} kT) (fluctuation-dissipation per pair);
 * r_c, kT and k stay global.  1 <= nspecies <= 4.  Must precede dpd_set_particles*
 * (DPD_ERR_ARG otherwise).  nspecies = 1 replaces (a, gamma) of dpd_create.  Species of
 * each particle are given to dpd_set_particles_typed (default 0) and travel with it
 * through migration and ghost exchange.  Errors: DPD_ERR_ARG, DPD_ERR_CONFIG (negative,
 * non-finite or asymmetric entries). */
int dpd_set_species(dpd_ctx *ctx, int nspecies, const double *a, const double *gamma);

/* SDF walls (reading C-23).  The solid is the
 * union of nprim <= 4 primitives, s(x) = max_k s_k(x) > 0 inside the solid, in GLOBAL
 * coordinates:
 *   type 1 plane:      prm = (nx, ny, nz, c), |n| = 1, s = n.x - c
 *   type 2/3/4 cylinder along x/y/z: prm = (c1, c2, R, sign) with (c1, c2) the axis in the
 *                      two other coordinates (cyclic order), s = sign (R - distance to the
 *                      axis): sign +1 a solid post, -1 a pipe (solid outside)
 *   uw[3k..3k+2]       translational velocity of primitive k (moving walls, Couette)
 * Every step, a fluid particle whose drift ends inside the solid is put back at its
 * collision point (bisection on t in [0, dt]) and its velocity is reversed in the wall
 * frame, u <- 2 u_w - u, where u_w is that of the primitive with the largest s there.
 * nprim = 0 removes the walls.  Errors: DPD_ERR_ARG (nprim > 4, NULL arrays),
 * DPD_ERR_CONFIG (unknown type, non-unit normal, R <= 0, sign not +-1, non-finite). */
int dpd_set_walls(dpd_ctx *ctx, int nprim, const int32_t *type, const double *prm, const double *uw);

/* Species whose particles never move (bit s of mask set): the frozen wall layer.  Their
 * velocity stays the wall velocity; they still interact with the fluid. */
int dpd_set_frozen_species(dpd_ctx *ctx, int32_t mask);

/* Carve the current configuration with the walls: particles with s > r_c are
 * removed, those with 0 < s <= r_c become frozen particles of species wall_species with
 * the wall velocity (wall_species is added to the frozen mask), fluid velocities are
 * completed to full-step values, the survivors are re-sorted and the forces re-primed at
 * the current step.  On one domain with dense ids the ids are renumbered densely (kept
 * particles keep their id order).  *n_frozen / *n_removed (may be NULL) receive this
 * rank's counts.  Collective in distributed contexts; group members must have been primed.
 * wall_species < nspecies when a species matrix is set, else <= 30. */
int dpd_wall_carve(dpd_ctx *ctx, int32_t wall_species, int64_t *n_frozen, int64_t *n_removed);

/* Device SDF s(x) of the current walls at n global points x (n x 3 float32) -> sdf[n]
 * (test hook; -3e38 without walls). */
int dpd_wall_sdf(dpd_ctx *ctx, int64_t n, const float *x, float *sdf);

/* Periodic-Poiseuille body force: f_body = (0,0,-f) for r_x <= L_x/2 and
 * (0,0,+f) otherwise (global coordinates); with the engine option "body_force_mode" = 1
 * it is the uniform (0,0,+f) of a wall-bounded channel.  f = 0 (default) disables it.
 * The body force acts on non-frozen particles and enters the integrator, not
 * dpd_get_forces. */
int dpd_set_body_force(dpd_ctx *ctx, double f);

/* Load n particles (copied; the caller keeps its buffers), assign ids 0..n-1, set the
 * step counter s = 0, build the cell list and prime F_0 = F(x_0, v_0, s=0) (C-2 item 2).
 *   pos, vel : n x 3 float32; pos is wrapped into [0, L) (C-10)
 * n = 0 is legal.  Non-finite input -> DPD_ERR_NUMERIC. */
int dpd_set_particles(dpd_ctx *ctx, int64_t n, const float *pos, const float *vel);

/* As dpd_set_particles, with caller-chosen global ids (each < 2^31, unique) and the
 * starting step index step0 (checkpoint resume, C-20).  In a distributed context every
 * rank may pass any superset of its particles: each rank keeps those inside its
 * subdomain.  ids may be NULL (ids := 0..n-1). */
int dpd_set_particles_ex(dpd_ctx *ctx, int64_t n, const float *pos, const float *vel,
                         const int32_t *ids, int64_t step0);

/* As dpd_set_particles_ex with a species index per particle (species may be NULL: all
 * 0).  An index outside [0, nspecies) is reported as DPD_ERR_ARG by this call, and so is a
 * particle id >= 2^30 while a species matrix (nspecies > 1) is set: the tiled force kernel
 * carries the species in the top two bits of the staged id word. */
int dpd_set_particles_typed(dpd_ctx *ctx, int64_t n, const float *pos, const float *vel,
                            const int32_t *ids, const int32_t *species, int64_t step0);

/* Advance nsteps >= 0 steps of Groot-Warren VV (C-2 item 3):
 *   u = v + dt/2 (F + f_body);  x = wrap(x + dt u);  s += 1;  rebuild cells;
 *   F = F(x, u, s);  v = u + dt/2 (F + f_body)
 * implemented fused (kick-drift on the half-step velocity u).
 * Synchronises the context's stream before returning and reports the first device-side
 * error (DPD_ERR_NUMERIC / DPD_ERR_CAPACITY / DPD_ERR_COMM).  DPD_ERR_NUMERIC also covers a
 * single pair force too large for the tiled kernel's fixed-point sums: |F_ij| above
 * a + 6.7 sigma/sqrt(dt) + 20 gamma max(1, sqrt(kT)) rounded up to a power of two (a pair
 * approaching at > ~20 sqrt(kT)), i.e. a diverged state; the step's results are then not
 * to be used (the reference kernel, option "force_kernel" 1, has no such bound). */
int dpd_step(dpd_ctx *ctx, int64_t nsteps);

/* As dpd_step but does not synchronise; a device-side error is reported by the next
 * synchronising call (dpd_step, dpd_get_*, dpd_sync). */
int dpd_step_async(dpd_ctx *ctx, int64_t nsteps);

/* Wait for the context's stream and report any pending device-side error. */
int dpd_sync(dpd_ctx *ctx);

/* Number of particles currently owned by this context (local particles when distributed). */
int dpd_get_count(const dpd_ctx *ctx, int64_t *n);

/* Step counter s (completed steps since set_particles, plus step0). */
int dpd_get_step(const dpd_ctx *ctx, int64_t *step);

/* Positions x_s and FULL-STEP velocities v_s = u_s + dt/2 (F_s + f_body) (C-6, C-14),
 * written in id order: row id of pos/vel.  Requires the owned ids to be exactly 0..n-1
 * (true after dpd_set_particles on one GPU), else DPD_ERR_ARG.  n must equal the count. */
int dpd_get_particles(dpd_ctx *ctx, int64_t n, float *pos, float *vel);

/* DPD pair forces F_s = F(x_s, u_s, s) (body force excluded), id order as above. */
int dpd_get_forces(dpd_ctx *ctx, int64_t n, float *f);

/* Raw state in storage (cell-sorted) order: x_s, the half-step velocity u_s used for F_s
 * (v_0 right after set_particles), F_s and ids.  Any pointer may be NULL.  cap is the
 * row capacity of the buffers; *n receives the count (DPD_ERR_ARG if cap < count). */
int dpd_get_state(dpd_ctx *ctx, int64_t cap, float *pos, float *uhalf, float *f,
                  int32_t *ids, int64_t *n);

/* Cell list of the current positions (C-8): cell_of_id[id] (ids must be dense 0..n-1; may
 * be NULL), count[ncell] and start[ncell + 1] (exclusive scan; may be NULL).  ncell is the
 * product of dpd_get_grid's dims.  Single-GPU contexts only. */
int dpd_debug_cells(dpd_ctx *ctx, int32_t *cell_of_id, int32_t *count, int32_t *start);

/* Grid dims n_d = floor(L_d / rc) (C-8) of this context's (sub)domain. */
int dpd_get_grid(const dpd_ctx *ctx, int32_t dims[3]);

/* Re-run the force pass on the current state in recording mode and dump every interacting
 * pair as (min id, max id, w0, w1) (T3 parity).  quad: cap x 4 uint32; *npairs receives the
 * total (may exceed cap; only cap rows are written).  Forces are recomputed identically. */
int dpd_debug_pairs(dpd_ctx *ctx, int64_t cap, uint32_t *quad, int64_t *npairs);

/* Per-kernel timing with CUDA events on the launch stream (disables CUDA-graph replay
 * while on).  Kernel ids: see dpd_kernel_name.  total_ms: summed event time since the
 * last reset; launches: number of timed launches. */
int dpd_set_timing(dpd_ctx *ctx, int enable);
int dpd_get_timing(dpd_ctx *ctx, int kernel_id, double *total_ms, int64_t *launches);
const char *dpd_kernel_name(int kernel_id); /* NULL past the last id */

/* Number of kernel launches issued by this context since creation (all kinds). */
int dpd_get_launch_count(const dpd_ctx *ctx, int64_t *launches);

/* ---- multi-GPU (3D domain decomposition) ---------------------------------- */

/* Communication plan of one rank (host only, no GPU needed): for each direction index
 * d = (dx+1) + 3 (dy+1) + 9 (dz+1), the rank its message goes to (coord + D, periodic),
 * the rank it receives direction-d messages from (coord - D), and whether d is used (every
 * nonzero component lies in a split dimension, grid > 1).  Messages are posted in
 * increasing d on every rank, which makes point-to-point matching order-consistent. */
int dpd_plan_peers(const int32_t grid[3], int rank, int32_t peer_to[27], int32_t peer_from[27],
                   int32_t used[27]);

/* Write a fresh NCCL unique id (128 bytes) for rank 0 to broadcast to the others. */
int dpd_nccl_unique_id(uint8_t id[128]);

/* Create the context of one rank of a world of size prod(grid) over NCCL.
 * box/rc/.../seed as dpd_create (the GLOBAL box); rank in [0, world);
 * grid[3] = ranks per dimension (rank = gx + grid_x (gy + grid_y gz));
 * nccl_id = the 128-byte id from dpd_nccl_unique_id on rank 0.
 * Each subdomain must be >= 3 rc wide in every dimension. */
int dpd_create_dist(const double box[3], double rc, double a, double gamma, double kT,
                    double power, double dt, uint64_t seed, int rank, int world,
                    const int32_t grid[3], const uint8_t nccl_id[128], dpd_ctx **out);

/* Create a one-rank NCCL context whose dimensions with split[k] != 0 are decomposed into
 * one subdomain that is its own neighbour: the periodic halo and the leavers of those
 * dimensions are packed into the 26-direction messages, sent with ncclSend / ncclRecv to the
 * rank itself (a self-peer; NCCL matches them in posting order, increasing d) and received
 * as ghosts / migrants -- P:234-247's exchange, P:243-247's overlap of the transfer with the
 * local forces, run end to end on one GPU.  Results equal those of dpd_create's periodic
 * context up to fp32 summation order.  nccl_id: a fresh id from dpd_nccl_unique_id.
 * Errors: DPD_ERR_ARG (no split dimension, null pointers), DPD_ERR_CONFIG (< 3 cells per
 * dimension), DPD_ERR_COMM (library built without NCCL, communicator init failed). */
int dpd_create_loopback(const double box[3], double rc, double a, double gamma, double kT,
                        double power, double dt, uint64_t seed, const int32_t split[3],
                        const uint8_t nccl_id[128], dpd_ctx **out);

/* Create an in-process group of prod(grid) subdomain contexts on the current device that
 * exchange ghosts / migrants by device copies instead of NCCL (same kernels, transport
 * swapped; used to test the decomposition on one GPU).  out receives grid-many contexts
 * in rank order.  Step them together with dpd_group_step. */
int dpd_create_group(const double box[3], double rc, double a, double gamma, double kT,
                     double power, double dt, uint64_t seed, const int32_t grid[3],
                     dpd_ctx **out);
int dpd_group_step(dpd_ctx **ctxs, int nctx, int64_t nsteps);

/* Local particles of a distributed context in storage order, with global ids, positions
 * in GLOBAL coordinates and full-step velocities.  *n receives the local count. */
int dpd_get_particles_ex(dpd_ctx *ctx, int64_t cap, float *pos, float *vel, int32_t *ids,
                         int64_t *n);

/* Forces of the local particles in storage order (same order as dpd_get_particles_ex). */
int dpd_get_forces_ex(dpd_ctx *ctx, int64_t cap, float *f, int32_t *ids, int64_t *n);

/* Species index of every particle (NEXT-2), row id of species[n] (dense ids required, as
 * dpd_get_particles). */
int dpd_get_species(dpd_ctx *ctx, int64_t n, int32_t *species);

/* Species of the local particles in storage order (same order as dpd_get_particles_ex);
 * ids (may be NULL) receives the matching ids, *n the count; cap < count -> DPD_ERR_ARG. */
int dpd_get_species_ex(dpd_ctx *ctx, int64_t cap, int32_t *species, int32_t *ids, int64_t *n);

/* ---- debug / parity hooks (T0: device RNG against the Random123 known answers) ------- */

/* Run the device Philox2x32-10 (C-7) on n counters: ctr n x 2, key n, out n x 2 (uint32). */
int dpd_debug_philox(int64_t n, const uint32_t *ctr, const uint32_t *key, uint32_t *out);

/* Device pair words and Box-Muller xi for n (ida, idb, step lo, step hi) quads under seed:
 * words n x 2 (w0, w1), xi n floats.  Host pointers. */
int dpd_debug_pair_words(int64_t n, const uint32_t *quad_in, uint64_t seed, uint32_t *words, float *xi);

/* ---- NEXT-4: compute / I/O overlap and the task-scheduled step -----------
 * PAPER.md §3.4: a "compute task" time-steps on the GPU while a "postprocess
 * task" does all heavy I/O; a "GPU-aware task scheduler based on the Kahn's
 * topological sorting algorithm, that supports task execution on concurrent CUDA streams"
 * orders the ~30 fine-grained tasks of a step.  Here the postprocess task is a
 * host worker thread per context behind a bounded queue, fed by
 * device-to-host copies on a separate copy stream into pinned slots.
 *
 * dpd_dump_open: start the writer.  path_prefix: files are written as
 *   <path_prefix>_r<rank>_s<step, 10 digits>.dpd ; queue_depth in [0, 64] (default of the
 *   Python binding 4): at most that many snapshots wait for the disk; a full queue blocks the
 *   submitting call (never drops); 0 = synchronous (each dump is written before the call
 *   returns).  Errors: DPD_ERR_ARG (already open, bad depth), DPD_ERR_CUDA.
 * dpd_dump_every: inside dpd_step / dpd_step_async, snapshot after every `every`-th step
 *   (global step index divisible by every; 0 = off).  The snapshot kernel runs on the compute
 *   stream after the step's forces; the copy-out on the copy stream; the next steps proceed
 *   without waiting for either.
 * dpd_dump_now: snapshot of the current state (same path).
 * dpd_dump_close: drain every pending snapshot, join the writer, free the slots; *written
 *   (may be NULL) receives the number of snapshots written.  A failed write surfaces as
 *   DPD_ERR_IO at the next dump submission or here.
 * File layout (little endian): char magic[8] = "DPDSNAP1"; int64 n, step, rank;
 *   float64 box[3] (global), origin[3] (this rank's subdomain corner); float32 pos[n][3]
 *   (global frame); float32 vel[n][3] (full-step velocity, C-6); int32 id[n].  Particles are
 *   in the rank's cell order (sort by id to compare with dpd_get_particles). */
int dpd_dump_open(dpd_ctx *ctx, const char *path_prefix, int queue_depth);
int dpd_dump_every(dpd_ctx *ctx, int64_t every);
int dpd_dump_now(dpd_ctx *ctx);
int dpd_dump_close(dpd_ctx *ctx, int64_t *written);

/* The step pipeline as scheduled: one line per task in issue (Kahn) order,
 *   "<stream slot> <task name>[ <- <predecessor>,...]\n"
 * slot 0 = compute stream, 1 = communication stream, 2 = copy stream.  with_dump selects
 * the variant with the snapshot tasks.  buf receives a NUL-terminated string of at most
 * cap bytes (DPD_ERR_ARG if too small). */
int dpd_step_schedule(dpd_ctx *ctx, int with_dump, char *buf, int64_t cap);

/* Host-side task graph (the scheduler of dpd_step_schedule, exposed for inspection and
 * tests; no device work): named tasks on stream slots, edges before -> after, Kahn order.
 * dpd_tg_order: DPD_ERR_CONFIG (and *n = 0) if the edges contain a cycle; among ready tasks
 * the earliest added is emitted first.  dpd_tg_edge: DPD_ERR_ARG on unknown ids / self
 * edges. */
typedef struct dpd_taskgraph dpd_taskgraph;
int dpd_tg_create(dpd_taskgraph **out);
int dpd_tg_add(dpd_taskgraph *g, const char *name, int stream_slot, int32_t *id);
int dpd_tg_edge(dpd_taskgraph *g, int32_t before, int32_t after);
int dpd_tg_order(dpd_taskgraph *g, int64_t cap, int32_t *order, int64_t *n);
void dpd_tg_destroy(dpd_taskgraph *g);

/* Host-side bounded I/O queue (the writer behind the dumps; no GPU needed).  depth as in
 * dpd_dump_open.  dpd_ioq_write copies `bytes` from data and writes them to path on the
 * worker after delay_us microseconds (a simulated slow disk for tests; 0 normally); it
 * blocks while depth writes are pending and returns DPD_ERR_IO (message in
 * dpd_ioq_last_error) if an EARLIER write failed.  dpd_ioq_close drains every pending write,
 * joins the worker, frees the queue, stores the number of completed writes and returns
 * DPD_ERR_IO if a write failed and was not yet reported. */
typedef struct dpd_ioq dpd_ioq;
int dpd_ioq_create(int depth, dpd_ioq **out);
int dpd_ioq_write(dpd_ioq *q, const char *path, const void *data, int64_t bytes, int64_t delay_us);
int dpd_ioq_pending(dpd_ioq *q, int64_t *n);
int dpd_ioq_close(dpd_ioq *q, int64_t *completed);
const char *dpd_ioq_last_error(const dpd_ioq *q);

#ifdef __cplusplus
}
#endif
#endif /* DPD_H */
