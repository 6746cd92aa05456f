/*
 * bdm.h -- C ABI of the B200-native BioDynaMo mechanical-interaction step (libbdm.so).
 *
 * One mechanical step over N spherical agents (BASELINE.json north_star):
 *   (a) uniform-grid rebuild, box edge = largest diameter      PAPER.md:313-322 (§2.1, Environment)
 *   (b) 27-box neighbour search                                  PAPER.md:318-320 (§2.1)
 *   (c) sphere-sphere force  f = k*delta - gamma*sqrt(r*delta)   north_star
 *   (d) displacement with adherence threshold and max-displacement clamp, then position update
 *                                                                north_star
 * The arithmetic reading (O1-O8, every ambiguity) is DESIGN.md §3.
 *
 * Conventions (all functions):
 *   - Return int status: BDM_OK (0) or a negative BDM_E* code.  Functions never abort or throw.
 *     The message for the last failure is returned by bdm_last_error(h) (thread-local when h is NULL
 *     or the handle could not be created).
 *   - Positions are n x 3 row-major fp64 (x0,y0,z0,x1,...) in micrometres; diameters n fp64.
 *   - Agent id = input index (0..n-1).  Every per-agent output is in id order.
 *   - Pointers are HOST pointers unless params.flags has BDM_DEVICE_PTRS, in which case every
 *     array argument of bdm_init and of the bdm_get_* array getters is a CUDA device pointer on the
 *     handle's device, used on the handle's stream (bdm_set_stream).
 *   - Input arrays are caller-owned and only read during the call (the library copies them).
 *     Outputs go to caller-allocated buffers of the documented size.  The handle owns all device
 *     state until bdm_destroy.  A handle is not thread-safe: one controlling caller.
 *   - All work is issued on the handle's stream.  Host-pointer getters synchronise that stream;
 *     device-pointer getters and bdm_mech_step return once the work is enqueued (call bdm_sync to
 *     wait and to collect asynchronous errors such as BDM_ENONFINITE / BDM_ERANGE).
 */
#ifndef BDM_H
#define BDM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BDM_ABI_VERSION 1

/* status codes */
#define BDM_OK 0
#define BDM_EINVAL (-1)     /* bad argument: n<0, NULL with n>0, D<=0 or non-finite, non-finite
                               position, bad params (eta<=0, max_disp<=0, negative or
                               non-finite k/gamma/adherence/dt/box_edge_min) */
#define BDM_ESTATE (-2)     /* call out of order (e.g. displacements before any step, handle poisoned
                               by an earlier asynchronous error) */
#define BDM_ENOMEM (-3)     /* device or host allocation failed */
#define BDM_ECUDA (-4)      /* CUDA runtime error (no device, launch failure, ...) */
#define BDM_ENCCL (-5)      /* NCCL error, or libnccl.so.2 could not be loaded (distributed handles) */
#define BDM_ENONFINITE (-6) /* a summed force or displacement was not finite; the message
                               names the agent and the offending pair (id, partner id): the first
                               partner, in O5's canonical order, whose term or partial sum is not
                               finite */
#define BDM_ERANGE (-7)     /* n >= 2^32, n_boxes >= 2^32, or |p * inv| >= 2^20 boxes (R9) */
#define BDM_ETRUNC (-8)     /* output buffer too small; the required size was written back */

/* params.flags */
#define BDM_DEVICE_PTRS 0x1u /* array arguments are CUDA device pointers */
#define BDM_RECORD 0x2u      /* force kernel also records per-agent neighbour / contact statistics */
#define BDM_SKIP_STATIONARY 0x4u /* NEXT-1: skip the neighbourhood search of agents no moving agent
                                    could affect ("detect stationary regions ... and
                                    skip the expensive collision detection"); bit-identical results */

/* bdm_get_pairs kind */
#define BDM_NEIGHBOR 0 /* unordered pairs with d2 <= L2 (O3) */
#define BDM_CONTACT 1  /* unordered pairs with delta > 0  (O4) */

typedef struct bdm_ctx* bdm_handle;

typedef struct {
  double k_rep;        /* repulsion coefficient k          default 10.0          */
  double gamma_att;    /* attraction coefficient gamma     default 4.0   (R3)          */
  double adherence;    /* |F| threshold; |F| <= it -> no motion, default 0.1 (R4)      */
  double dt;           /* time step                        default 1.0          */
  double eta;          /* viscosity                        default 1.0          */
  double max_disp;     /* clamp on |Delta p| per step, um  default 3.0          */
  double box_edge_min; /* box edge = max(max D, this), um  default 0.0          */
  uint32_t flags;      /* BDM_DEVICE_PTRS | BDM_RECORD                                          */
  int32_t device;      /* CUDA device ordinal; -1 = current device                              */
} bdm_params;

typedef struct {
  double L;         /* box edge (O1) */
  double L2;        /* L*L, the neighbour threshold on d2 (O3) */
  double inv;       /* 1/(L*(1+2^-30)), binning factor (O1, R9) */
  int32_t lo[3];    /* min integer box coordinate per axis (O2) */
  int32_t hi[3];    /* max integer box coordinate per axis */
  int64_t n_boxes;  /* (hi-lo+1) product */
  int64_t n_agents; /* N */
} bdm_grid_info;

/* Per-agent statistics (only with BDM_RECORD; arrays of n, id order; any pointer may be NULL). */
typedef struct {
  int32_t* n_cand;   /* candidates visited in the 27 boxes, self excluded */
  int32_t* n_nb;     /* neighbours, d2 <= L2 */
  int32_t* n_ct;     /* contacts, delta > 0 */
  int8_t* branch;    /* 0 = below adherence, 1 = clamped, 2 = free (O6) */
  uint64_t* nb_hash; /* sum over neighbours j of mix64(j) mod 2^64 (order-free digest) */
  uint64_t* ct_hash; /* sum over contacts j of mix64(j) mod 2^64 */
} bdm_agent_stats;

/* Fill *p with the defaults listed above.  EINVAL if p is NULL. */
int bdm_params_default(bdm_params* p);

/* Create a handle holding n agents.  pos: n x 3 fp64, diam: n fp64 (host, or device with
 * BDM_DEVICE_PTRS).  Validates every input (EINVAL, message names the first bad index).  n = 0 is
 * valid: steps are no-ops.  The state is "no grid" until bdm_grid_build or the
 * first step.  On failure *h is set to NULL. */
int bdm_init(bdm_handle* h, int64_t n, const double* pos, const double* diam, const bdm_params* p);

/* Rebuild the uniform grid from the current positions (O1-O2 + counting sort, ascending id inside
 * each box, box start table).  Marks the grid fresh so the next step does not rebuild again. */
int bdm_grid_build(bdm_handle h);

/* Run n_steps mechanical steps (n_steps >= 0; 0 is a no-op).  Each step: rebuild the
 * grid unless fresh, compute every force from the step-start snapshot, displacements (O6), then
 * update all positions (O7, Jacobi).  Asynchronous; errors detected on the device are reported by
 * the next synchronising call.  Inside one call, the rebuilds of steps 0..n_steps-2 may skip their
 * host round trip (deferred builds; at most bdm_set_defer's count in a row, default
 * 8): a range or frame error of such a step is then reported by the next
 * synchronised rebuild (at the latest the last step of the same call) as BDM_ERANGE, and the handle
 * is poisoned; the results of the steps in between are not to be used.  Displacements are stored
 * for the last step of the call only (bdm_get_displacements). */
int bdm_mech_step(bdm_handle h, int32_t n_steps);

/* At most max_deferred consecutive deferred builds inside one bdm_mech_step call (see above; 0 = a
 * host round trip every build; default 8, or the environment's BDM_DEFER).  EINVAL if
 * max_deferred < 0. */
int bdm_set_defer(bdm_handle h, int max_deferred);

/* Displacements Delta p of the last step, n x 3 fp64, id order.  ESTATE before the first step. */
int bdm_get_displacements(bdm_handle h, double* out);

/* Current positions, n x 3 fp64, id order. */
int bdm_get_positions(bdm_handle h, double* out);

/* Current diameters, n fp64, id order (they change under bdm_set_growth). */
int bdm_get_diameters(bdm_handle h, double* out);

/* Integer box coordinates floor(p * inv) of the current positions under the current grid,
 * n x 3 int32, id order.  Builds the grid if it is not fresh. */
int bdm_get_box_coords(bdm_handle h, int32_t* out);

/* Grid of the last build (host struct).  ESTATE if no grid was built yet. */
int bdm_get_grid_info(bdm_handle h, bdm_grid_info* out);

/* Per-agent statistics of the last step (requires BDM_RECORD at init; ESTATE otherwise).  Output
 * arrays are host or device according to BDM_DEVICE_PTRS. */
int bdm_get_agent_stats(bdm_handle h, const bdm_agent_stats* out);

/* Unordered pair set of the current positions (kind BDM_NEIGHBOR or BDM_CONTACT): pairs (min id,
 * max id) sorted lexicographically into out[2*cap] (HOST memory always).  *n_pairs receives the
 * count; ETRUNC (and nothing written) if it exceeds cap.  Builds the grid if not fresh. */
int bdm_get_pairs(bdm_handle h, int kind, int64_t* n_pairs, int64_t* out, int64_t cap);

/* NEXT-2, cell growth and division ("cell growth and
 * division" benchmark; SPEC.md:82-91 volume-conserving division).  After the mechanics of every
 * later step: D <- D + growth; agents with D >= div_diam divide into two spheres of diameter
 * D * 2^(-1/3) touching along a counter-hash direction (seed, step, id); the k-th divider in id
 * order creates agent id N + k.  growth = 0 and div_diam = +inf switch it off.  The population
 * grows (capacity doubles as needed); displacements refer to the agents of the last mechanics. */
int bdm_set_growth(bdm_handle h, double growth, double div_diam, uint64_t seed);

/* NEXT-3, soma clustering ("soma clustering" benchmark;
 * SPEC.md:260-329 diffusion-field).  Two substances on a lattice of dims nodes at spacing h from
 * origin (node (i,j,k) at origin + h*(i,j,k)), closed boundary.  Every later step, before the
 * mechanics: agents of type t add `secretion` to their nearest node of field t; both fields take one
 * explicit-Euler step c += dt*(diff*lap(c) - decay*c) (7-point stencil; needs diff*dt/h^2 <= 1/6,
 * else EINVAL); every agent moves `speed` along the normalised gradient of its own field. */
typedef struct {
  double h;         /* lattice spacing, um */
  double origin[3]; /* position of node (0,0,0), um */
  int32_t dims[3];  /* nodes per axis */
  double diff;      /* diffusion coefficient, um^2/step */
  double decay;     /* decay rate, 1/step */
  double dt;        /* time step of the diffusion update */
  double secretion; /* amount added per agent per step */
  double speed;     /* chemotaxis displacement per step, um */
} bdm_field_params;

/* Enable the soma-clustering operations; types: n int8 (0 or 1) in id order (host or device per
 * BDM_DEVICE_PTRS).  Both fields start at 0. */
int bdm_set_fields(bdm_handle h, const bdm_field_params* fp, const int8_t* types);

/* Field `which` (0 or 1), dims[0]*dims[1]*dims[2] fp64 with z fastest. */
int bdm_get_field(bdm_handle h, int which, double* out);

/* NEXT-4, neurite elements (PAPER.md:402-415 springs with a distal point mass,
 * PAPER.md:768-769; SPEC.md:230-238 sphere-cylinder force, SPEC.md:377-386 spring chains).
 * n_el cylinders (HOST arrays, element id = index): distal point (n_el x 3), diameter, resting length,
 * anchor (n_el x 3, the proximal point of roots), mother (-1 for roots), daughters (n_el x 2, -1 =
 * none).  Every later step moves spheres and distal points together: sphere-sphere and
 * sphere-cylinder contacts, axial springs k_spring*(len - rest)/rest, one box edge for both grids.
 * n_el = 0 removes them. */
int bdm_set_neurites(bdm_handle h, int64_t n_el, const double* distal, const double* diam, const double* rest_len,
                     const double* anchor, const int64_t* mother, const int64_t* daughters, double k_spring);

/* Distal points (n_el x 3) and their displacements of the last step (n_el x 3), HOST arrays; either
 * pointer may be NULL. */
int bdm_get_neurites(bdm_handle h, double* distal, double* ddistal);

/* Make room for `capacity` agents (dynamic populations).  Never shrinks. */
int bdm_reserve(bdm_handle h, int64_t capacity);

/* out2[0] = current number of agents, out2[1] = agents of the last mechanics step (rows of
 * bdm_get_displacements / bdm_get_agent_stats). */
int bdm_get_count(bdm_handle h, int64_t* out2);

/* Stationary-region skip statistics of the last step (BDM_SKIP_STATIONARY): out3[0] agents that
 * moved (dp != 0), out3[1] agents whose neighbourhood was searched, out3[2] N.  -1 entries when not
 * available (no step yet, or the flag is off). */
int bdm_get_skip_stats(bdm_handle h, int64_t* out3);

/* Force path of the last step: out2[0] = 1 if it ran the half-shell pair path
 * (k_half_search + k_half_sum: each candidate pair tested once, Newton's third law), 2 if it ran it
 * band by band over a ring of pair rows (populations whose rows do not fit beside the state, e.g.
 * 10^9 agents on one GPU), 0 if the single-pass k_force (BDM_RECORD, BDM_SKIP_STATIONARY,
 * bdm_set_force_path(BDM_PATH_SINGLE), or no pair rows / a grid whose two-layer span exceeds the
 * ring); out2[1] = agents of that step whose pair rows overflowed and took the exact full-search path
 * (results are identical either way).  -1 entries before the first step. */
int bdm_get_path_stats(bdm_handle h, int64_t* out2);

/* Force-path selection for plain steps of this handle: BDM_PATH_AUTO (default)
 * runs the half-shell passes (band by band over a ring of pair rows when rows for every agent, 72 B
 * each, do not fit) and falls back to the single-pass k_force otherwise; BDM_PATH_SINGLE always runs
 * k_force.  Both compute O3-O7 in the canonical order: results are bit-identical.  EINVAL for any
 * other value. */
#define BDM_PATH_AUTO 0
#define BDM_PATH_SINGLE 1
int bdm_set_force_path(bdm_handle h, int path);

/* Issue all later work on this CUDA stream (cudaStream_t; NULL = legacy default stream). */
int bdm_set_stream(bdm_handle h, void* cuda_stream);

/* Wait for the handle's stream; returns any pending asynchronous error. */
int bdm_sync(bdm_handle h);

/* Replace the population of h (same n) with new positions / diameters (host or device per
 * BDM_DEVICE_PTRS), re-validated as in bdm_init; ids stay 0..n-1.  Reuses every device buffer, so
 * repeated batches pay only the copy.  Clears an earlier asynchronous data error. */
int bdm_set_agents(bdm_handle h, const double* pos, const double* diam);

/* Per-step device timing with CUDA events on the handle's stream (bdm_set_timing(h, 1) enables
 * it).  bdm_get_timing synchronises and writes, summed over the steps since the previous call:
 * out4[0] grid-build ms, out4[1] force-kernel ms, out4[2] steps, out4[3] kernels of this library
 * launched (counted whether or not timing is enabled); then resets the sums. */
int bdm_set_timing(bdm_handle h, int enabled);
int bdm_get_timing(bdm_handle h, double* out4);
/* As bdm_get_timing, plus the force phase split of the half-shell path:
 * out6[4] ms of the search pass (row-counter and fused-column resets + k_half_search), out6[5] ms of
 * the sum pass (k_half_sum); both 0 for steps that ran k_force or the banded ring phase (whose
 * passes interleave).  Resets the sums. */
int bdm_get_timing_ex(bdm_handle h, double* out6);

/* Counter-based uniform population on the device (kernel K0; bdm_inputs/__init__.py holds the
 * NumPy twin): for ids [id0, id0+n): pos[i][a] = lo[a] + (hi[a]-lo[a])*u(seed, id, a),
 * diam[i] = dlo + (dhi-dlo)*u(seed, id, 3), u = (splitmix64(seed*0x9E3779B97F4A7C15 + 4*id + s) >> 11)
 * * 2^-53.  pos (n x 3) and diam (n) are DEVICE pointers; issued on the given stream. */
int bdm_generate_uniform(uint64_t seed, int64_t id0, int64_t n, const double* lo3, const double* hi3, double dlo,
                         double dhi, double* pos, double* diam, void* cuda_stream);

/* ---------------------------------------------------------------------------------------------
 * x-slab mode (multi-GPU; north_star "the domain is split into x-slabs. Each step does
 * a halo exchange of boundary-box agents and migrates agents that cross slab boundaries").  One
 * handle per rank owns the agents whose box-x lies in [x_begin, x_end) (rank 0: x_begin = INT32_MIN,
 * last rank: x_end = INT32_MAX).  The exchange itself (counts, payloads, allreduce of L and the
 * extents) is done by the caller -- paper_2006_06775_b200/dist.py over torch.distributed.  Every
 * array is a DEVICE pointer (BDM_DEVICE_PTRS required).  Exchange records are 5 fp64 per agent
 * (x, y, z, D, id).  Per step: local_extents -> allreduce -> pack(HALO) -> exchange -> step ->
 * pack(MIGRANTS) -> exchange -> add.  Owned sums use ghosts with global ids in canonical order, so
 * results are bit-identical to the single-handle path.
 * --------------------------------------------------------------------------------------------- */
#define BDM_HALO 0
#define BDM_MIGRANTS 1
#define BDM_OWNED_POSITIONS 0
#define BDM_LAST_DISPLACEMENTS 1

/* Create a slab handle with n_local owned agents (global ids < 2^32, positions n x 3, diameters n)
 * and room for `capacity` owned + ghost agents.  EINVAL without BDM_DEVICE_PTRS. */
int bdm_slab_init(bdm_handle* h, int64_t n_local, int64_t capacity, const uint32_t* ids, const double* pos,
                  const double* diam, const bdm_params* p);

/* Replace the owned agents with a new batch (device arrays; same rules as bdm_slab_init), keeping
 * every allocation.  The global box edge stays as set (call bdm_slab_set_box_edge if diameters grew). */
int bdm_slab_load(bdm_handle h, int64_t n_local, const uint32_t* ids, const double* pos, const double* diam);

/* Largest diameter among the owned agents (0 if none); the caller allreduces it (O1). */
int bdm_slab_local_maxd(bdm_handle h, double* maxd);

/* Set the global box edge (max over ranks of the local max D; box_edge_min still applies). */
int bdm_slab_set_box_edge(bdm_handle h, double L);

/* Integer box extents (lo[3], hi[3]) of the owned agents' current positions (after a step: of the
 * positions the step produced, before migration).  INT32_MAX / INT32_MIN if none.  ERANGE as O2. */
int bdm_slab_local_extents(bdm_handle h, int32_t* lohi6);

/* Pack records to send to the lower (box-x below) and upper neighbour.  what = BDM_HALO: owned
 * agents in the first / last box-x layer of the slab.  what = BDM_MIGRANTS: owned agents whose box-x
 * left [x_begin, x_end); they are removed from the handle.  send_lo / send_hi hold cap records
 * each; ETRUNC (state unchanged) if either count exceeds cap, with the counts written back. */
int bdm_slab_pack(bdm_handle h, int what, int32_t x_begin, int32_t x_end, double* send_lo, double* send_hi,
                  int64_t cap, int64_t* n_lo, int64_t* n_hi);

/* Single-sync protocol, after a step: split the owned agents without a host round
 * trip.  Emigrants (box-x left [x_begin, x_end)) go to the FRONT of send_lo / send_hi, the agents
 * that stay are compacted (committed by bdm_slab_commit), and the stayers of the first / last box-x
 * layer -- the neighbours' ghosts of the next step -- go to the BACK of send_lo / send_hi (record
 * cap-1-k).  info (DEVICE int64[12], asynchronous): [0] emigrants lo, [1] halo lo, [2] emigrants hi,
 * [3] halo hi, [4] stayers, [5..7] box extents lo of the owned agents' positions, [8..10] hi,
 * [11] 1 if a buffer's cap records did not hold emigrants + halo (then resend with larger buffers
 * through bdm_slab_pack).  ESTATE if a split is pending. */
int bdm_slab_split(bdm_handle h, int32_t x_begin, int32_t x_end, double* send_lo, double* send_hi, int64_t cap,
                   int64_t* info);

/* Commit the pending split: the owned agents become the n_stay stayers (info[4] of the split);
 * n_stay < 0 cancels it (owned agents unchanged, e.g. to split again with larger buffers). */
int bdm_slab_commit(bdm_handle h, int64_t n_stay);

/* Append received records (immigrants) to the owned agents.  ERANGE past the capacity. */
int bdm_slab_add(bdm_handle h, const double* recv_lo, int64_t n_lo, const double* recv_hi, int64_t n_hi);

/* One mechanical step of the owned agents: ghosts = the records received from the lower
 * (box-x = x_begin - 1) and upper (box-x = x_end) neighbours; slab-local grid over box-x
 * [x_begin-1, x_end] with the global y/z extents glo3/ghi3 (allreduced local extents); force,
 * displacement and update of the owned agents only.  want_dp != 0 keeps the displacements. */
int bdm_slab_step(bdm_handle h, const int32_t* glo3, const int32_t* ghi3, int32_t x_begin, int32_t x_end,
                  const double* recv_lo, int64_t n_lo, const double* recv_hi, int64_t n_hi, int want_dp);

/* Owned agents (what = BDM_OWNED_POSITIONS: ids + n x 3 positions) or the displacements of the last
 * step with want_dp (BDM_LAST_DISPLACEMENTS: ids + n x 3), in the handle's internal order; *n gets
 * the count.  ids / vals may be NULL to query the count. */
int bdm_slab_get(bdm_handle h, int what, int64_t* n, uint32_t* ids, double* vals);

/* ---------------------------------------------------------------------------------------------
 * Distributed handles (multi-GPU).  north_star: "Across the 8
 * GPUs of one box the domain is split into x-slabs.  Each step does a halo exchange of boundary-box
 * agents and migrates agents that cross slab boundaries, using NCCL send/recv over NVLink."
 * PAPER.md:436-453 (§2.3 (i)-(iii): the parallel runtime this replaces); SPEC.md:118 (one
 * controlling caller per instance: here one per rank).
 *
 * One process (rank) per GPU.  The library owns the exchange's data plane: an NCCL communicator
 * (libnccl.so.2 loaded at the first distributed call), the partition, the halo exchange and the
 * migration.  A rank owns the agents whose integer box-x lies in its slab [cut[r], cut[r+1]);
 * the cuts are chosen at init from a global per-layer histogram and then from each rank's own
 * per-layer work (sum n_b + sum n_b^2 / mean), all on the device.  bdm_mech_step runs
 * chunks of up to 16 steps with no host synchronisation inside a chunk (device-resident counts,
 * fixed-capacity messages whose headers carry the counts, a fixed grid frame per chunk); a chunk
 * in which a message overflowed is re-run from a device checkpoint with larger buffers.  Results
 * are bit-identical to a single handle (ghosts keep their global ids and canonical order).
 * Errors: NCCL failures -> BDM_ENCCL; the others as for bdm_init / bdm_mech_step.
 * --------------------------------------------------------------------------------------------- */

/* Rank 0 creates the communicator id (128 bytes into out128) and broadcasts it to the other ranks
 * (e.g. over torch.distributed); ENCCL if NCCL cannot be loaded. */
int bdm_nccl_unique_id(void* out128);

/* Collective over the `world` ranks (every rank calls it with the same uid).  This rank contributes
 * n_local agents with global ids (int64, unique over all ranks, 0 <= id < 2^32 - 1), positions
 * (n x 3) and diameters (n); any initial distribution is allowed (agents are redistributed to
 * their owners).  Arrays are host pointers, or device pointers with p->flags & BDM_DEVICE_PTRS.
 * device: CUDA ordinal of this rank; cuda_stream: the stream all work of the handle runs on (also
 * NCCL's).  Validates as bdm_init (EINVAL names the first bad agent).  The returned handle accepts
 * bdm_mech_step, bdm_set_timing / bdm_get_timing(_ex), bdm_get_stats, bdm_get_local,
 * bdm_get_cuts, bdm_sync and bdm_destroy. */
int bdm_init_dist(bdm_handle* h, int64_t n_local, const int64_t* ids, const double* pos, const double* diam,
                  const bdm_params* p, int rank, int world, const void* nccl_uid, int device, void* cuda_stream);

/* A new batch for a distributed handle (collective, same rules as bdm_init_dist): the agents are
 * validated, the cuts recomputed and every agent sent to its owner; the communicator and the device
 * buffers are reused (bdm_set_agents for distributed handles). */
int bdm_set_agents_dist(bdm_handle h, int64_t n_local, const int64_t* ids, const double* pos, const double* diam);

/* Virtual ranks (tests of the data plane on one GPU): all `world` ranks live in this process on
 * p->device over a 1-rank NCCL communicator (every message a self send/recv); counts[r] agents
 * start on rank r, the arrays hold them concatenated in rank order.  Same protocol and kernels as
 * bdm_init_dist; getters return all ranks' owned agents. */
int bdm_init_dist_local(bdm_handle* h, int world, const int64_t* counts, const int64_t* ids, const double* pos,
                        const double* diam, const bdm_params* p, void* cuda_stream);

/* Owned agents of a distributed handle (all local ranks): what = BDM_OWNED_POSITIONS (ids + n x 3
 * positions) or BDM_LAST_DISPLACEMENTS (ids + n x 3 displacements of the last step; ESTATE before
 * one).  *n receives the count; ids / vals may be NULL (count only).  Host or device pointers per
 * BDM_DEVICE_PTRS at init.  Synchronises. */
int bdm_get_local(bdm_handle h, int what, int64_t* n, int64_t* ids, double* vals);

/* The partition of a distributed handle: world + 1 box-x cuts (cut[0] = INT32_MIN, cut[world] =
 * INT32_MAX) into out[cap]; ETRUNC if cap is too small. */
int bdm_get_cuts(bdm_handle h, int32_t* out, int32_t cap);

/* Order-free pair digest of the current positions (SURVEY §8(c) outputs, used for large configs):
 * for every agent (id order) the number of partners of kind BDM_NEIGHBOR (d2 <= L2, O3) or
 * BDM_CONTACT (delta > 0, O4) and the sum over them of mix64(partner id) mod 2^64 (mix64 = the
 * SplitMix64 finaliser).  Builds the grid if needed.  count: n uint32, hash: n uint64, host or
 * device per BDM_DEVICE_PTRS.  Single handles only (ESTATE otherwise). */
int bdm_get_pair_digest(bdm_handle h, int kind, uint32_t* count, uint64_t* hash);

/* Counters of a handle since init (SURVEY §8(b) bdm_get_stats). */
typedef struct {
  int64_t n_agents;       /* agents (distributed: owned by this process's ranks) */
  int64_t steps;          /* mechanical steps run */
  int64_t launches;       /* kernels of this library launched */
  int64_t host_syncs;     /* host synchronisations with the device (distributed: set-up, one per chunk
                             of up to 16 steps, getters) */
  int64_t half_path;      /* 1: the last step ran the half-shell passes, 2: the same band by band over a
                             ring of pair rows, 0: k_force, -1: no step */
  int64_t migrated;       /* distributed: agents that changed owner during steps */
  int64_t ghosts;         /* distributed: ghost agents of the last step (all local ranks) */
  int64_t exchange_bytes; /* distributed: bytes sent by this process's ranks */
  int64_t chunks;         /* distributed: synchronised chunks of steps */
  int64_t redo_chunks;    /* distributed: chunks re-run after a message overflow */
  int64_t world;          /* ranks (1 for single handles) */
  int64_t local_ranks;    /* ranks in this process */
} bdm_stats;
int bdm_get_stats(bdm_handle h, bdm_stats* out);

/* Human-readable message of the last failure on h (or of the calling thread when h is NULL). */
const char* bdm_last_error(bdm_handle h);

/* Release every resource of h.  NULL is a no-op. */
void bdm_destroy(bdm_handle h);

/* ABI version (BDM_ABI_VERSION). */
int bdm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BDM_H */
