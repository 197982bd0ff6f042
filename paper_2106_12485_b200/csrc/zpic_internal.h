// zpic_internal.h — device data layout and kernel parameter blocks of the B200 EM-PIC path.
// Not part of the ABI (include/zpic.h is).  Layouts are documented in DESIGN.md "Data layout".
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/zpic.h"

namespace zpic {

constexpr int kMaxSpecies = 4;
constexpr int kXOff = 4;          // interior column 0 sits at column 4 of a padded row (16 B aligned)
constexpr int kEnergySlots = 256; // fp64 partial-sum slots (spread the atomics), per quantity
constexpr int kBlock = 256;       // threads per CTA of the particle kernels
constexpr int kSMin = 22;         // smallest tile scale exponent of the one-word int32 current
// K5 tile: 128 x 8 (same-box sweep at C5, profiles/r2_ab_yee_tiles.log: 0.70 ms vs 0.72 for 64 x 16,
// 0.79 for 32 x 32 and 128 x 4, 0.87 for 128 x 16: wide rows make long TMA rows and coalesced
// stores; 8 rows keep 4 CTAs / SM in 48 KB of staged boxes)
#ifndef ZPIC_YEE_TX
#define ZPIC_YEE_TX 128
#endif
#ifndef ZPIC_YEE_TY
#define ZPIC_YEE_TY 8
#endif
constexpr int kYeeTX = ZPIC_YEE_TX;   // K5 tile: columns
constexpr int kYeeTY = ZPIC_YEE_TY;   // K5 tile: rows

// A guard-extended field grid: 3 planes of `rows` x `pitch` floats; interior cell (i, j) of a
// plane is at (j + 1) * pitch + (i + kXOff), valid for -1 <= i <= nx + 1, -1 <= j <= ny + 1
// (guards 1 low / 2 high per axis).
struct GridDesc {
  int nx, ny;      // local interior cells
  int pitch;       // floats per row (multiple of 32)
  int rows;        // ny + 3
  long plane;      // rows * pitch
  __host__ __device__ long at(int i, int j) const { return (long)(j + 1) * pitch + (i + kXOff); }
};

// One species' tile-sorted particle store, AoSoA with 32-particle blocks: slot k lives in block
// k / 32 at lane k % 32, and field f of the block is the contiguous run of 32 words at f * 32,
// so a warp reading 32 consecutive slots gets one 128 B line per field and a thread needs one
// address per particle (fields are immediate offsets).  Fields: 0 cell (ix | iy << 16), 1 x,
// 2 y, 3 ux, 4 uy, 5 uz, 6 id (only with track_ids).  Tile t owns slots
// [t * cap, t * cap + cnt[t]); cap is a multiple of 32.
enum PField { F_CELL = 0, F_X, F_Y, F_UX, F_UY, F_UZ, F_ID };
struct PStore {
  uint32_t* data;  // ntiles * cap / 32 blocks of 32 * nf words
  int nf;          // 6, or 7 with ids
  int32_t* cnt;    // [ntiles]
  int cap;         // slots per tile (multiple of 32)
  __host__ __device__ uint32_t* slot(long k) const { return data + (k >> 5) * (32L * nf) + (k & 31); }
};

// Per-tile mailboxes of one species (K1 -> K3m): a particle leaving tile t across an edge or a
// corner goes to slot k of box (t, d), d = the direction of travel (mail_dir); the destination
// tile's warp in K3m reads the 8 boxes addressed to it and appends them to its segment with
// coalesced stores.  Boxes have fixed capacities (edges cap_edge, corners cap_corner); a
// particle that finds its box full goes through the flat mover list instead.  Fields as in
// PStore, one record per slot (nf consecutive words: a box is one contiguous run): field f of
// slot q at data[q * nf + f], q = t * per_tile + offset(d) + k.
struct MailBox {
  uint32_t* data;
  int32_t* cnt;    // [ntiles][8] entries of each box this step
  int cap_edge, cap_corner, per_tile;
  long stride;     // ntiles * per_tile (slots)
  int nf;
};

// Particles that left their tile (or could not be inserted): a flat SoA list.
struct PList {
  int32_t* cell;
  float *x, *y, *ux, *uy, *uz;
  uint32_t* id;
  int32_t* species;
  int32_t* count;  // device counter
  int cap;
};

struct SpeciesConst {
  float q;      // per-particle charge q_s = sign(m_q) n / ppc (R8)
  float h;      // dt / (2 m_q)  (Boris half-kick factor)
  float jx, jy; // q dx/dt, q dy/dt (deposit flux scales)
  double ke_scale;  // q m_q dx dy
};

// Everything the particle kernels need, passed by value (K1 takes it as a __grid_constant__
// parameter: the TMA descriptors are read from parameter space).
struct PushParams {
  CUtensorMap tmE, tmB;   // 3D TMA maps of the current E and B buffers: (pitch, rows, 3) floats,
                          // box (T + 4 rounded to 4, T + 2, 3); zero fill outside (K1 staging)
  GridDesc g;
  const float* E;   // current E (3 planes)
  const float* B;
  float* J;         // assembled J grid (loose-particle deposits)
  float* Jt;        // per-tile J blocks [ntiles][3][(T+3)^2]
  int T, ntx, nty;
  int nspecies;
  SpeciesConst sc[kMaxSpecies];
  PStore ps[kMaxSpecies];
  PList movers;     // written by the tile kernel this step
  PList spill_in;   // loose particles to push this step
  PList spill_out;  // loose particles for the next step
  float dtdx, dtdy; // dt/dx, dt/dy
  int bcx, bcy;
  int shift;        // 1 when the moving window shifts at the end of this step (ix -= 1)
  // y-slab decomposition (§8(e)): slab = 1 when the y neighbours are other slabs; has_lo /
  // has_hi = a neighbour exists below / above (else a domain edge).  Particles leaving the
  // slab go to send[0] (down, iy += ny) or send[1] (up, iy -= ny).
  int slab, has_lo, has_hi;
  PList send[2];
  int peer_send;        // 1: send[] are the neighbours' receive areas (PEER transport): the kernels
                        // that append to them (K3, K1L) end with a system-scope fence
  int skip_cell_store;  // tuning switch: write the cell word only when it changed
  int commutative;      // 1: K1 adds its current block into J with global atomics (no Jt, no K4)
  int use_mail;         // 1: tile leavers go through the per-tile mailboxes (K3m), else the mover list
  MailBox mail[kMaxSpecies];
  int fx_smin;          // a tile uses the one-word int32 current when its scale exponent S >= fx_smin
  // Per-tile occupancy bound (DESIGN.md §2 "fixed-point current"): occ[t] >= the number of particles
  // (all species) in any 4 x 4 cell window of tile t at the start of K1 — K1 writes the window
  // maximum of its stayers' end cells, every insertion into the tile (K3m, K3, loose re-insertion,
  // halo receive, window injection) adds to it; -1 = unknown (the tile count bounds it).
  int32_t* occ;
  int32_t* tscale;      // [ntiles] the scale exponent S of each tile's current this step (K1s)
  int32_t* hist;        // [ntiles][T * T] particles per cell of each tile (all species), exact at the
                        // start of every K1: K1 moves its crossing particles, insertions add
  int check_occ;        // 1: K1s verifies hist against a recount (ZPIC_CHECK_OCC; tests)
  float qmax;           // max_s |q_s|
  int tile0;            // K1 launches over tiles [tile0, tile0 + grid) (the slab overlap splits it)
  // PEER round 2 fused into K1 (NEXT-1, per tile row): boundary_last = 1 runs the interior tile rows
  // first and the slab-edge rows last in one grid (2: the slab-edge rows only, in one grid: the
  // NCCL path after its round-2 event); a slab-edge CTA first acquire-waits until
  // r2_flags[2] (from the lower) / [3] (from the upper) reach r2_epoch: the neighbours' E/B rows of
  // this step are then in this slab's guard rows (null: no wait)
  int boundary_last;
  const unsigned long long* r2_flags;
  unsigned long long r2_epoch;
  // Cross-slab "commutative" current (PEER transport + current_mode 1): deposits on
  // this slab's rows -1, 0 are also added into the lower neighbour's J rows ny_lo - 1, ny_lo, those on
  // rows ny, ny + 1 into the upper neighbour's rows 0, 1 (peer pointers; null = not this mode / edge)
  float* Jlo;
  float* Jhi;
  long lo_plane, hi_plane;
  int lo_ny;
  double* ke_slots; // [kMaxSpecies][kEnergySlots]
  int* err;         // sticky device error flags (bit 0 overflow, bit 1 migration)
};

struct YeeParams {
  CUtensorMap tmE, tmB, tmJ;   // TMA maps of E0, B0 (box 40 x (T+3|T+2) x 3) and J (36 x (T+1) x 3)
  GridDesc g;
  const float* E0; const float* B0; const float* J;
  float* E1; float* B1;
  float dt, dtdx, dtdy, hdx, hdy;   // dt, dt/dx, dt/dy, (dt/2)/dx, (dt/2)/dy
  float murx, mury;                 // Mur-1 coefficients (dt - dx)/(dt + dx), (dt - dy)/(dt + dy)
  int bcx, bcy;
  int shift;                        // 1: store the result one column toward -x (window shift)
  int y_images;                     // write periodic y guard images (1 GPU, periodic y)
  int ylo_edge, yhi_edge;           // the slab's low / high y boundary is a domain edge
  double* fe_slots;
  double fe_scale;  // dx dy / 2
  int row0;         // first tile row of this launch (the slab overlap splits the grid)
  // PEER round 2 fused into K5: the slab-edge tiles also write their output rows 0, 1 into the lower
  // neighbour's guard rows ny_lo, ny_lo + 1 and row ny - 1 into the upper neighbour's guard row -1
  // of the buffers of the same parity (null: not this mode / no neighbour)
  float* peer_lo_E;
  float* peer_lo_B;
  long peer_lo_plane;
  int peer_lo_ny;
  float* peer_hi_E;
  float* peer_hi_B;
  long peer_hi_plane;
};

struct InjectParams {
  PStore ps;
  int T, ntx, nx_global, y0, ny;
  int px, py;
  int col_lo, col_hi;   // filled global columns [col_lo, col_hi)
  uint64_t key;         // mix64(mix64(seed) + species)
  double ufl[3], uth[3];
};

struct LaserParams {
  double a0, omega0, fwhm, W0, start, yc;
};

// A neighbour's receive area of the PEER transports (zpic_peer.cu): its own pointers in a loopback
// group, CUDA IPC pointers across processes, this context's block in a one-rank ring.
struct PeerView {
  float* jrup;       // [3][2][pitch] the upper neighbour's raw J rows -1, 0 (round 1)
  float* jrdn;       // [3][2][pitch] the lower neighbour's raw J rows ny, ny+1 (round 1)
  char* pmsg[2];     // particle messages from the lower [0] / upper [1] neighbour (round 1)
  // round 2 writes straight into the owner's field buffers (their guard rows -1, ny, ny + 1):
  float* E[2];       // the owner's E / B buffers (both parities), each [3][ny + 3][pitch]
  float* B[2];
  long plane;        // (ny + 3) * pitch of the owner
  int ny;            // the owner's interior rows
  unsigned long long* flags;   // [6] epochs: round 1 from lower / upper, round 2 from lower / upper,
                               // J zeroed by the lower / upper neighbour (cross-slab commutative current)
};

enum ErrBits { ERR_OVERFLOW = 1, ERR_MIGRATION = 2, ERR_HALO = 8, ERR_HIST = 16 };   // 4: k_count's out-of-slab upload

}  // namespace zpic

// The opaque ABI handle.
struct zpic_ctx {
  zpic::GridDesc g;
  int nx_global, ny_global, y0;
  double dx, dy, dt;
  int bcx, bcy;
  int nspecies;
  zpic_species species[zpic::kMaxSpecies];
  zpic::SpeciesConst sc[zpic::kMaxSpecies];
  uint64_t seed;
  zpic_options opt;
  zpic_dist dist;
  int T, ntx, nty, ntiles;
  cudaStream_t stream;
  bool own_stream;
  CUtensorMap tm[2][2];   // [E / B][buffer] TMA maps for K1's field staging
  CUtensorMap ytm[2][2];  // [E / B][buffer] TMA maps for K5's staging (boxes of YeeBox)
  CUtensorMap ytmJ[2];    // [J / Jf] for K5
  // device buffers
  float* E[2];
  float* B[2];
  float* J;        // assembled (and folded, filtered) current used by the field advance
  float* Jf;       // filtered current (only with a filter; J keeps the pre-filter values)
  float* Jt;       // per-tile blocks
  zpic::PStore ps[zpic::kMaxSpecies];
  zpic::MailBox mail[zpic::kMaxSpecies];
  zpic::PList movers, spill[2];
  double* ke_slots;
  double* fe_slots;
  double* energy;  // [1 + kMaxSpecies] last finished step: FE, KE_s
  int* err;
  int* stats;      // [0] movers of last step, [1] spill count
  int32_t* occ = nullptr;   // [ntiles] occupancy bound of the fixed-point current (PushParams::occ)
  int32_t* tscale = nullptr;   // [ntiles] per-tile scale exponent, from occ before every K1 (K1s)
  int32_t* hist = nullptr;     // [ntiles][T * T] per-tile cell histogram (PushParams::hist)
  int check_occ = 0;           // ZPIC_CHECK_OCC=1: verify hist every step (ERR_HIST)
  bool occ_stale = true;    // the particles were (re)loaded: recompute occ before the next step
  int cur;         // index of the current E/B buffer
  int64_t steps;
  int64_t repacks;
  int since_check = 0;   // steps since the last loose-list check (re-pack, zpic_api.cu)
  bool repacking = false;
  int64_t population = 0;  // particles at the last (re)load
  int64_t launches;  // kernels enqueued by zpic_step so far
  int64_t n_move;    // moving-window shifts so far
  // y-slab decomposition (§8(e)); slab == false: the whole domain, no exchanges
  bool slab;
  int rank, world, lower, upper, has_lo, has_hi;
  int transport;
  void* comm;        // ncclComm_t
  cudaStream_t comm_stream = nullptr;   // NCCL halo rounds, overlapped with interior kernels
  cudaStream_t copy_stream = nullptr;   // chunked host uploads (zpic_set_particles)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};   // phase-A end, round 1, Yee end, round 2
  bool r2_pending = false;              // round 2 of the last step is in flight on comm_stream
  bool own_comm;
  float* jrup;       // [3][2][pitch]: the upper neighbour's raw J rows -1, 0
  float* jrdn;       // [3][2][pitch]: the lower neighbour's raw J rows ny, ny+1
  void* pmsg_send[2];  // particle messages to the lower [0] / upper [1] neighbour
  void* pmsg_recv[2];  // from the lower [0] / upper [1] neighbour
  int pcap;
  bool halo_dirty;
  // PEER transports: this context's receive block (cudaMalloc: exportable), the neighbours' views
  bool peer = false;
  void* peer_block = nullptr;
  zpic::PeerView peer_self{}, peer_lo{}, peer_hi{};
  unsigned long long peer_e1 = 0, peer_e2 = 0;   // rounds 1 / 2 done (the next epoch to signal is +1)
  // cross-slab commutative current (PEER + current_mode 1): J in its own cudaMalloc (exportable),
  // the neighbours' J, their planes and the lower's ny; e0 counts the "J zeroed" signals
  bool peer_j = false, j_zeroed = false;
  void* j_block = nullptr;
  void* eb_block = nullptr;   // PEER: E[0], E[1], B[0], B[1] in one cudaMalloc (exported by CUDA IPC)
  float* jlo = nullptr;
  float* jhi = nullptr;
  long lo_plane = 0, hi_plane = 0;
  int lo_ny = 0;
  unsigned long long peer_e0 = 0;
  std::vector<void*> ipc_open;                   // neighbour blocks opened with cudaIpcOpenMemHandle   // E/B guard rows of the current buffer must be exchanged before the next step
  std::vector<void*> allocations;
  std::string last_error;
  // CUDA graphs of two steps, by step parity (the state a two-step replay returns to)
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  int graph_launches = 0;  // kernels in one two-step graph
  cudaGraphExec_t graph1[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // one step, [parity][shift]
  int graph1_launches[2][2] = {{0, 0}, {0, 0}};
  int64_t* d_nmove = nullptr;   // the window shift count on the device (column injection ids)
  // periodic in-tile re-sort (K2s, in place) every sort_every steps
  int sort_every = 0;
  int64_t last_sort = 0;
  int64_t sorts = 0;
  // profiling
  bool prof;
  std::vector<std::string> prof_names;
  std::vector<cudaEvent_t> prof_ev;  // pairs
  std::vector<double> prof_ms;
  std::vector<int> prof_count;
  std::vector<std::pair<int, int>> prof_pending;  // (kernel id, event pair index)
};
