/*
 * zpic.h — C ABI of the B200-native 2D3V EM-PIC hot path (ZPIC em2d, arxiv 2106.12485).
 *
 * The step this library runs is the paper's main loop (Fig. 1):
 *   (1) bilinear field interpolation at each particle "with the field values from the
 *       previous iteration",
 *   (2) leapfrog + relativistic Boris particle advance,
 *   (3) "exact charge conserving" current deposition (Villasenor-Buneman
 *       trajectory split at cell crossings per BASELINE.json north_star), the ghost-cell
 *       current reduction and the optional digital filter,
 *   (4) Yee-mesh FDTD field advance and the ghost-field update,
 * plus particle boundaries (periodic / open / moving window) and the per-tile
 * particle re-sort.  Readings of everything the paper leaves open: SURVEY.md §8(c) R1-R25,
 * repeated in DESIGN.md.  All arithmetic is fp32 on the device; energies are fp64.
 *
 * Conventions (normalised units, c = 1):
 *   - grid quantities are returned as [component][y][x] fp32, interior cells only;
 *     Yee staggering Ex(i+1/2,j) Ey(i,j+1/2) Ez(i,j) Bx(i,j+1/2) By(i+1/2,j) Bz(i+1/2,j+1/2);
 *   - a particle is (ix, iy) cell index + (x, y) in-cell offset in [0,1) + proper momentum
 *     (ux, uy, uz) = gamma v;
 *   - per-particle charge q_s = sign(m_q) * n_s / (ppc_x * ppc_y) (R8).
 *
 * Errors: every function returns a zpic_status; nothing throws across the ABI.  Device
 * errors (capacity overflow, |displacement| >= 1 cell) are sticky: they are raised on the
 * device, and reported by the next synchronising call (get_*, zpic_energy, zpic_sync).
 * zpic_last_error() gives a one-line message.  A ctx is not thread-safe.
 *
 * Ownership: the library owns every device buffer (allocated through the optional allocator
 * hooks in zpic_options — the Python binding passes PyTorch's caching allocator — else
 * cudaMalloc).  The caller owns every host buffer; get_* fill them by copy.  Work is enqueued
 * on options->stream (a cudaStream_t; NULL = a stream the library creates).
 */
#ifndef ZPIC_H
#define ZPIC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ZPIC_OK = 0,
  ZPIC_E_INVALID = -1,    /* bad argument / config (message in zpic_last_error) */
  ZPIC_E_CFL = -2,        /* dt >= 1/sqrt(dx^-2 + dy^-2) */
  ZPIC_E_EMPTY_GRID = -3, /* nx or ny < 1 */
  ZPIC_E_DECOMP = -4,     /* slab rows < 2 or ny % world != 0 */
  ZPIC_E_LASER = -5,
  ZPIC_E_OOM = -6,
  ZPIC_E_CUDA = -7,
  ZPIC_E_NCCL = -8,
  ZPIC_E_OVERFLOW = -9,   /* mover buffer capacity exceeded (particles would be lost) */
  ZPIC_E_MIGRATION = -10, /* a particle moved >= 1 cell in one step (CFL / logic bug) */
  ZPIC_E_BUFSIZE = -11,   /* caller buffer too small */
  ZPIC_E_STATE = -12      /* call not valid in the current state */
} zpic_status;

typedef struct {
  int32_t nx, ny; /* cells (global) */
  double dx, dy;  /* cell size, c/omega_p */
} zpic_grid;

typedef enum {
  ZPIC_BC_PERIODIC = 0,
  ZPIC_BC_OPEN = 1,          /* particles removed at the edge; Mur-1 on tangential E (R13) */
  ZPIC_BC_MOVING_WINDOW = 2  /* x only: window moves at c; fresh plasma injected (R14, R15): the
                                entering column gets the profile's density beyond the box, so a
                                species must be uniform or a ramp ending inside the box (x1 <= nx dx);
                                a slab profile is rejected at zpic_init (ZPIC_E_INVALID) */
} zpic_bc;

typedef struct {
  zpic_bc x, y;
} zpic_boundaries;

typedef enum {
  ZPIC_DENS_UNIFORM = 0, /* n everywhere */
  ZPIC_DENS_SLAB = 1,    /* n for cell-centre x in [x0, x1), 0 elsewhere */
  ZPIC_DENS_NONE = 2,    /* no particles from zpic_init: load them with zpic_set_particles */
  ZPIC_DENS_RAMP = 3     /* 0 for x < x0, linear 0 -> n over [x0, x1), n beyond:
                            along x every y sub-row places its particles by inverting the
                            cumulative density, X_k = x0 + sqrt(2 L (k + 1/2) dx / ppc_x) in the
                            ramp (L = x1 - x0), the regular sub-lattice from x1 on; ids follow the
                            sub-row-major order of that list */
} zpic_dens;

/* One species.  The device injector (zpic_init) fills the ppc_x x ppc_y regular sub-lattice
 * x = (k+1/2)/ppc_x, y = (l+1/2)/ppc_y of every filled cell, u = ufl + uth * N(0,1) with the
 * counter-based generator of DESIGN.md "RNG" keyed by (seed, species index, particle id). */
typedef struct {
  double m_q;         /* mass / charge (-1 electrons) */
  int32_t ppc[2];     /* particles per cell along x, y */
  double n;           /* density (sets q_s) */
  zpic_dens profile;
  double x0, x1;      /* slab limits (physical x) */
  double ufl[3], uth[3];
} zpic_species;

typedef void* (*zpic_alloc_fn)(size_t bytes, void* user);
typedef void (*zpic_free_fn)(void* ptr, void* user);

/* Optional settings; pass NULL for defaults. */
typedef struct {
  int32_t filter_passes;      /* 0 = no filter; n passes of (1/4,1/2,1/4) along x */
  int32_t filter_compensated; /* 1 = add the (-n/4, 1+n/2, -n/4) compensator pass (R12) */
  int32_t track_ids;          /* 1 = carry a uint32 id per particle (validation runs) */
  int32_t tile[2];            /* tile size in cells: 8, 16 or 32 (square); 0 = auto (default):
                                 16 x 16 unless that gives fewer than 2 tiles per SM, then 8 x 8 */
  double capacity_slack;      /* per-tile capacity = slack * initial count (default 1.5) */
  double mover_fraction;      /* mover buffer capacity as a fraction of particles (default 0.05) */
  int32_t profile;            /* 1 = record per-kernel CUDA-event times (zpic_kernel_times) */
  void* stream;               /* cudaStream_t to enqueue on (NULL: library-owned stream) */
  zpic_alloc_fn alloc;        /* device allocator hook (NULL: cudaMalloc) */
  zpic_free_fn free;
  void* alloc_user;
  int32_t current_mode;       /* ghost-current combination of the tiles (the paper's
                                 Table 1 second axis):
                                 0 = "reduction" (default): every tile stores its private current block
                                     and K4 sums the overlapping guard nodes (no atomics);
                                 1 = "commutative": every tile adds its block into the global J with
                                     fp32 global atomics (J zeroed first each step, no K4); on the
                                     PEER transports the slab-edge tiles and loose particles also add
                                     their ghost rows (-1, 0 / ny, ny+1) straight into the neighbour
                                     slab's J over peer memory, so round 1 carries particles only
                                     (each J zeroed and flagged before any neighbour's K1 adds). */
  int32_t laser;              /* 1 = initialise E, B with a laser pulse: linearly
                                 polarised along y, travelling along +x, E_y = a0 w0 env(x)
                                 exp(-(y - Ly/2)^2 / W0^2) cos(w0 (x - xc)), B_z = E_y at B_z's points;
                                 env = sin^2 rise and fall of length fwhm each ending at x = start,
                                 xc = start - fwhm (no divergence cleaning); ZPIC_E_LASER if fwhm or
                                 W0 <= 0 or the pulse misses the box */
  double laser_a0, laser_omega0, laser_fwhm, laser_W0, laser_start;
  int32_t no_graphs;          /* 0 (default): zpic_step replays a captured CUDA graph of two steps
                                 when it can (single domain, no moving window, profile = 0), which
                                 removes the per-launch host cost of small grids; 1 = plain launches */
  int32_t current_precision;  /* accumulation of the tile current, both order-independent:
                                 0 = auto (default): one int32 fixed-point atomic per node at the
                                     tile's scale 2^S, the largest S that the tile's bound |J_node| <=
                                     (particles in any 4 x 4 cell window) * max|q| keeps below 2^31
                                     (rounding <= 2^-(S+1) per contribution, ~2^-27 at 16 ppc);
                                     tiles with S < 22 take the exact form;
                                 1 = exact: every tile accumulates contributions scaled by 2^32 as
                                     int64 split into two int32 atomics (error <= 2^-33 each). */
  int32_t halo_particles;     /* y-slabs: particle records per halo message and direction (0 = auto:
                                 a quarter of a boundary row at the nominal density, >= 4096); more
                                 crossers in one step stop the run with ZPIC_E_OVERFLOW */
} zpic_options;

/* y-slab decomposition (the paper's row-band regions).
 * Rank r owns rows [r*ny/world, (r+1)*ny/world) with all nx columns; ny % world == 0 and at
 * least 2 rows per slab.  Every step exchanges, with the y neighbours only: (1) raw current
 * guard rows + migrating particles, (2) E/B ghost rows.  Transports:
 *   ZPIC_TRANSPORT_NCCL: one process per GPU; nccl_comm is an ncclComm_t (e.g. torch's
 *     ProcessGroupNCCL._comm_ptr()), or NULL with nccl_id = the 128-byte ncclUniqueId from
 *     zpic_nccl_unique_id() on rank 0, broadcast by the caller (the library then owns a comm);
 *   ZPIC_TRANSPORT_LOOPBACK: `world` contexts in one process on one device and one stream,
 *     stepped together with zpic_step_group (validation of the slab logic on one GPU);
 *   ZPIC_TRANSPORT_PEER: one process per GPU of one node; no NCCL send / recv in the step: the
 *     library's own kernels write the halo straight into the neighbours' memory over NVLink (the
 *     particles leaving the slab appended by the kernels that route them, the E / B rows of
 *     round 2 by the Yee kernel's slab-edge tiles into the neighbours' guard rows, the raw J rows
 *     by a put kernel or, with current_mode = 1, added by the push kernel into the neighbours' J;
 *     CUDA IPC pointers exchanged once at zpic_init with an all-gather on the NCCL communicator
 *     given as for ZPIC_TRANSPORT_NCCL) and signal each round with a system-scope epoch flag that
 *     the receiver acquires (a wait kernel, or the slab-edge CTAs of the next push for round 2; a
 *     wait that never completes stops the run with ZPIC_E_OVERFLOW after ~20 s instead of
 *     hanging); world = 1 is a ring on the context's own buffers;
 *   ZPIC_TRANSPORT_LOOPBACK_PEER: the PEER kernels in a loopback group (zpic_step_group; every
 *     signal is enqueued before the wait that reads it, so no kernel ever waits on another).
 * The PEER transports allocate the receive block and the E / B field buffers (and, with
 * current_mode = 1, J) with cudaMalloc, independent of zpic_options.alloc: the neighbours write
 * into them (CUDA IPC across processes).
 * Pass NULL for the unsplit single-GPU domain. */
typedef enum { ZPIC_TRANSPORT_NCCL = 0, ZPIC_TRANSPORT_LOOPBACK = 1, ZPIC_TRANSPORT_PEER = 2,
               ZPIC_TRANSPORT_LOOPBACK_PEER = 3 } zpic_transport;
typedef struct {
  int32_t rank, world;
  void* nccl_comm;
  int32_t device;
  const void* nccl_id;      /* 128 bytes, used when nccl_comm == NULL */
  zpic_transport transport;
} zpic_dist;

typedef struct zpic_ctx zpic_ctx;

/* Validate, allocate, inject every species (UNIFORM / SLAB lattices with the seeded momenta, RAMP
 * by cumulative inversion), zero the fields and, with options->laser, write the laser pulse.
 * nx, ny in [2, 32767]; dt below the Courant limit 1/sqrt(dx^-2 + dy^-2).
 * Errors: ZPIC_E_INVALID, ZPIC_E_CFL, ZPIC_E_EMPTY_GRID, ZPIC_E_DECOMP, ZPIC_E_LASER, ZPIC_E_OOM,
 * ZPIC_E_CUDA, ZPIC_E_NCCL. On error *out is NULL and zpic_last_error(NULL) says why. */
zpic_status zpic_init(zpic_ctx** out, const zpic_grid* grid, double dt, const zpic_species* species,
                      int32_t n_species, const zpic_boundaries* bc, uint64_t seed,
                      const zpic_options* options, const zpic_dist* dist);

/* Replace the particles of one species by n host particles (global ix, iy; x, y in [0, 1)).
 * id may be NULL (then ids are 0..n-1 if track_ids).  The arrays are copied (pinned host memory
 * uploads at the PCIe rate; large uploads stream in chunks, overlapped with the binning on the
 * device).  A particle outside the local slab or with an offset outside [0, 1) is an error
 * (ZPIC_E_INVALID; the species is left empty).  Tiles without room send particles to the loose
 * list, which is re-packed when it grows.  Synchronous.  Drops the captured step graphs. */
zpic_status zpic_set_particles(zpic_ctx* ctx, int32_t species, int64_t n, const int32_t* ix,
                               const int32_t* iy, const float* x, const float* y, const float* ux,
                               const float* uy, const float* uz, const uint32_t* id);

/* Overwrite E (which=0) or B (which=1) interior values from host [comp][y][x] (laser init). */
zpic_status zpic_set_fields(zpic_ctx* ctx, int32_t which, const float* in, size_t in_len);

/* Enqueue n time steps (asynchronous w.r.t. the host, on the context's stream).  Without slabs
 * and with profile = 0 the steps are replayed as captured CUDA graphs (two-step graphs, or one-step
 * graphs keyed by the window shift).  Every 16 steps the host reads the loose-list count (one
 * stream synchronisation) and re-packs the tile stores if it grew.  With NCCL slabs every rank must
 * call it with the same n (the halo exchanges are collective between neighbours); the exchanges run
 * on a second stream overlapped with interior tiles, and the context's stream has waited for them
 * when zpic_step returns.  Errors raised on the device are reported by the next synchronising
 * call. */
zpic_status zpic_step(zpic_ctx* ctx, int32_t n);

/* Step `count` loopback slab contexts (ranks 0..count-1 of one decomposition, same device and
 * stream) together for n steps.  ZPIC_E_STATE if they are not one complete loopback group. */
zpic_status zpic_step_group(zpic_ctx** ctxs, int32_t count, int32_t n);

/* Write a fresh ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128 bytes) to out (out_len >= 128). */
zpic_status zpic_nccl_unique_id(void* out, size_t out_len);

/* Self-test of the PEER halo protocol (the ZPIC_TRANSPORT_PEER rounds): `ranks`
 * emulated slabs of nx x ny cells (a ring if periodic, else a chain), one CTA each in one
 * cooperative launch on the current device, run `epochs` steps of round 1 (raw J rows -1, 0 /
 * ny, ny+1 and particle messages of up to pcap records), signal, wait, verify, round 2 (E/B rows),
 * signal, wait, verify, with the transport's own put / signal / wait code and receive-block
 * layout; the waits spin on flags the other CTAs store concurrently.  commutative = 1 replaces
 * the J rows of round 1 by the cross-slab commutative current (J zeroed, "zeroed" signalled and
 * awaited, the shared rows added into the neighbours' J with peer atomics; after round 1 each
 * shared row must hold its own plus the neighbour's contribution).  Every value is a hash of
 * (sender, epoch, place), so a record that arrives late, twice, from the wrong neighbour or into
 * the wrong area is counted.  *errors_out = mismatched values + 2^40 per wait that exceeded
 * budget_cycles (GPU clocks).  fault: 0 none; 1 rank 0 corrupts one J value it sent at epoch 2;
 * 2 rank 0 skips its round-1 signal at epoch 2 (both must make *errors_out non-zero).  Allocates
 * and frees its own device memory.  ZPIC_E_INVALID for ranks outside [1, 64], epochs < 1, nx < 1,
 * ny < 4, pcap outside [32, 4096] or a null errors_out; ZPIC_E_CUDA if allocation or the launch
 * fails.  The particle records are appended into the neighbours' areas the way K3 / K1L append the
 * slab exits (a slot from the receiver's count, any order) and checked as a set. */
zpic_status zpic_peer_selftest(int32_t ranks, int32_t epochs, int32_t nx, int32_t ny, int32_t pcap, int32_t periodic,
                               int32_t commutative, int64_t budget_cycles, int32_t fault, int64_t* errors_out);

/* Block until all enqueued work is done; surface sticky device errors. */
zpic_status zpic_sync(zpic_ctx* ctx);

/* which: 0 = E, 1 = B, 2 = J used by the last field advance (after reduction and filter),
 * 3 = J of the last step before the filter.  out: 3*nx*ny_local floats [comp][y][x]. */
zpic_status zpic_get_fields(zpic_ctx* ctx, int32_t which, float* out, size_t out_len);

/* Diagnostics (validation only): the charge density at the nodes from the
 * current particle positions, summed over species, rho(i, j) = sum_p q_s * W, with the bilinear
 * area weights W = (1-x)(1-y), x(1-y), (1-x)y, xy to nodes (ix, iy), (ix+1, iy), (ix, iy+1),
 * (ix+1, iy+1), node indices wrapped periodically in x and (one domain) y.
 * With a slab decomposition, nodes beyond the slab's rows are dropped.  out: nx*ny_local floats
 * [y][x].  Errors: ZPIC_E_INVALID, ZPIC_E_BUFSIZE, ZPIC_E_CUDA. */
zpic_status zpic_get_charge(zpic_ctx* ctx, float* out, size_t out_len);

/* Size query when ix == NULL (count_inout <- count).  Otherwise fills up to *count_inout
 * particles (order unspecified) with global ix, iy; id requires track_ids (may be NULL). */
zpic_status zpic_get_particles(zpic_ctx* ctx, int32_t species, int64_t* count_inout, int32_t* ix,
                               int32_t* iy, float* x, float* y, float* ux, float* uy, float* uz,
                               uint32_t* id);

/* Energies of the input state of the last step taken (time level iter = steps-1):
 * field = 1/2 dx dy sum(E^2 + B^2), kinetic[s] = q_s m_q,s dx dy sum(gamma - 1) (R8).
 * Before any step: iter = -1 and zeros.  NCCL slabs: summed over all ranks (collective: every
 * rank must call it); loopback slabs: this slab only. */
zpic_status zpic_energy(zpic_ctx* ctx, int64_t* iter, double* field, double* kinetic);

/* Local slab rows [y0, y0 + ny_local). */
zpic_status zpic_layout(zpic_ctx* ctx, int32_t* y0, int32_t* ny_local);

/* Counters: out[0] particles (all species), out[1] movers of the last step, out[2] max
 * tile occupancy / capacity in per-mille, out[3] re-packs done, out[4] steps taken,
 * out[5] number of tiles, out[6] kernels launched by zpic_step so far, out[7] tile size T,
 * out[8] / out[9] tiles the periodic in-tile re-sort (K2s, ZPIC_SORT_EVERY) sorted / left unsorted
 * (a tile holding more particles than its shared-memory stage) so far, out[10] particles in the
 * loose list now (no room in their tile; pushed from global memory).  n <= 11 entries are written. */
zpic_status zpic_counters(zpic_ctx* ctx, int64_t* out, int32_t n);

/* Per-kernel device time (ms) summed over the steps since the last call, when
 * options->profile: names of the kernels in order, up to n entries; returns count. */
zpic_status zpic_kernel_times(zpic_ctx* ctx, const char** names, double* ms, int32_t* launches,
                              int32_t* n_inout);

void zpic_free(zpic_ctx* ctx);

/* Message of the last failure on ctx (NULL ctx: the last failed zpic_init on this thread). */
const char* zpic_last_error(const zpic_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* ZPIC_H */
