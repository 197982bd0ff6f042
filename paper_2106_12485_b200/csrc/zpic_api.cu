// zpic_api.cu — host runtime behind include/zpic.h: validation, device memory, the step
// sequence, exports, energies, profiling.  No compute happens on the host:
// every stage of the step is one of the kernels in zpic_kernels.cu.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "zpic_internal.h"

namespace zpic {
void launch_push_tiles(const PushParams& p, int tile_begin, int tile_end, cudaStream_t st);
void launch_insert(const PushParams& p, int grid, cudaStream_t st);
void launch_mail_gather(const PushParams& p, cudaStream_t st);
void launch_charge(const PushParams& p, double* rho, int wrap_y, cudaStream_t st);
void launch_to_float(const double* a, float* b, long n, cudaStream_t st);
void launch_ramp_rows(long n, int n_row, int py, int y0, const int32_t* ixr, const float* xr, uint64_t key,
                      const double* ufl, const double* uth, int32_t* ix, int32_t* iy, float* x, float* y, float* ux,
                      float* uy, float* uz, uint32_t* id, cudaStream_t st);
void launch_laser(float* E, float* B, const GridDesc& g, int y0, double dx, double dy, const LaserParams& L,
                  cudaStream_t st);
void launch_loose_extract(const PList& L, int s, int y0, int64_t out0, int32_t* ix, int32_t* iy, float* x, float* y,
                          float* ux, float* uy, float* uz, uint32_t* id, int* counter, cudaStream_t st);
void launch_loose(const PushParams& p, int grid, cudaStream_t st);
void launch_assemble(float* J, const float* Jt, const GridDesc& g, int T, int ntx, int nty, cudaStream_t st);
void launch_guard_x(float* F, const GridDesc& g, int mode, int keep, cudaStream_t st);
void launch_guard_y(float* F, const GridDesc& g, int mode, int keep, cudaStream_t st);
void launch_yee(const YeeParams& p, cudaStream_t st, int row_begin = 0, int row_end = -1);
int yee_tile_rows(const GridDesc& g);
void launch_epilogue(double* ke_slots, double* fe_slots, double* energy, int nspecies, const double* ke_scale4, int* mc,
                     int* sic, int* soc, int* stats, int64_t* d_nmove, int shifted, cudaStream_t st);
void launch_inject(const InjectParams& q, int ntiles, cudaStream_t st);
void launch_bin(const PStore& ps, int T, int ntx, int y0, long n, const int32_t* ix, const int32_t* iy, const float* x,
                const float* y, const float* ux, const float* uy, const float* uz, const uint32_t* id, int* err,
                const PList& loose, int s, cudaStream_t st, int nx = 0, int ny = 0, int* bad = nullptr, long id0 = 0);
void launch_export(const PStore& ps, int ntiles, const int64_t* prefix, int y0, int32_t* ix, int32_t* iy, float* x,
                   float* y, float* ux, float* uy, float* uz, uint32_t* id, cudaStream_t st);
void launch_count(int T, int ntx, int nx, int ny, int y0, long n, const int32_t* ix, const int32_t* iy, const float* x,
                  const float* y, int* counts, int* err, cudaStream_t st);
void launch_inject_column(const PushParams& p, int s, int px, int py, const int64_t* n_move, int ny_global, int y0, uint64_t key,
                          const double* ufl, const double* uth, cudaStream_t st);
void launch_filter_x(const float* Jin, float* Jout, const GridDesc& g, int npass, int compensated, int periodic,
                     cudaStream_t st);
void launch_apply_j_halo(float* J, const GridDesc& g, const float* rup, const float* rdn, int has_lo, int has_hi,
                         cudaStream_t st);
size_t particle_msg_bytes(int cap);
PeerView peer_view(void* block, int pitch, int pcap);
size_t peer_block_bytes(int pitch, int pcap);
void launch_peer_put1(const float* J, const GridDesc& g, const PeerView& lo, const PeerView& up, int has_lo,
                      int has_hi, cudaStream_t st);
void launch_peer_put2(const float* E, const float* B, const GridDesc& g, const PeerView& lo, const PeerView& up,
                      int has_lo, int has_hi, int b, cudaStream_t st);
void launch_peer_signal(unsigned long long* fa, unsigned long long* fb, unsigned long long e, cudaStream_t st);
void launch_peer_wait(const unsigned long long* flags, int ia, int ib, unsigned long long e, int* err, cudaStream_t st);
PList particle_msg_list(void* buf, int cap);
void launch_recv_insert(const PushParams& p, const PList& lo, const PList& hi, cudaStream_t st);
void launch_sort_tiles(const PStore& ps, int T, int ntx, int ntiles, int* stats, cudaStream_t st);
void launch_occupancy(const PushParams& p, cudaStream_t st, int mode = 0);
void launch_loose_drop_species(const PList& L, int s, const PList& out, cudaStream_t st);
void launch_tile_scale(const PushParams& p, cudaStream_t st);
}  // namespace zpic

using namespace zpic;

namespace {
thread_local std::string g_init_error;

uint64_t host_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Fail {
  zpic_status st;
  std::string msg;
};

#define CUDA_OR_THROW(x)                                                                          \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) throw Fail{ZPIC_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

void* dev_alloc(zpic_ctx* c, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* p = nullptr;
  if (c->opt.alloc) {
    p = c->opt.alloc(bytes, c->opt.alloc_user);
    if (!p) throw Fail{ZPIC_E_OOM, "allocator hook returned NULL for " + std::to_string(bytes) + " bytes"};
  } else {
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) throw Fail{ZPIC_E_OOM, "cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e)};
  }
  c->allocations.push_back(p);
  return p;
}

void dev_free(zpic_ctx* c, void* p) {
  if (!p) return;
  auto it = std::find(c->allocations.begin(), c->allocations.end(), p);
  if (it == c->allocations.end()) return;
  c->allocations.erase(it);
  if (c->opt.free) c->opt.free(p, c->opt.alloc_user);
  else cudaFree(p);
}

// A temporary device buffer released when the scope ends (also when a Fail unwinds it).
struct TmpBuf {
  zpic_ctx* c;
  void* p;
  TmpBuf(zpic_ctx* c_, size_t bytes) : c(c_), p(dev_alloc(c_, bytes)) {}
  ~TmpBuf() { dev_free(c, p); }
  TmpBuf(const TmpBuf&) = delete;
  TmpBuf& operator=(const TmpBuf&) = delete;
};

template <class T>
T* alloc_n(zpic_ctx* c, size_t n) {
  T* p = (T*)dev_alloc(c, n * sizeof(T));
  CUDA_OR_THROW(cudaMemsetAsync(p, 0, n * sizeof(T), c->stream));
  return p;
}

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// A 3D TMA map of one guard-extended field buffer: dims (pitch, rows, 3 components) floats, box
// (BX, T + 2, 3) with BX = T + 5 rounded up to 4 floats (the box starts at a 16-byte aligned column
// 4 cells left of the tile: TMA faults on an unaligned start column), zero fill outside.
// cuTensorMapEncodeTiled is taken from the driver through the runtime (no -lcuda).
void make_tmap(CUtensorMap* map, float* F, const GridDesc& g, int bx, int by) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      throw Fail{ZPIC_E_CUDA, "cuTensorMapEncodeTiled is not available"};
  }
  const cuuint64_t dims[3] = {(cuuint64_t)g.pitch, (cuuint64_t)g.rows, 3};
  const cuuint64_t strides[2] = {(cuuint64_t)g.pitch * 4, (cuuint64_t)g.plane * 4};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 3};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, F, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Fail{ZPIC_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
}
void make_field_tmap(CUtensorMap* map, float* F, const GridDesc& g, int T) {
  make_tmap(map, F, g, (T + 5 + 3) & ~3, T + 2);
}

void alloc_store(zpic_ctx* c, int s, int cap) {
  PStore& ps = c->ps[s];
  size_t n = (size_t)cap * c->ntiles;
  ps.cap = cap;
  ps.nf = c->opt.track_ids ? 7 : 6;
  ps.data = (uint32_t*)dev_alloc(c, n * ps.nf * sizeof(uint32_t));   // contents defined by cnt, no memset
  ps.cnt = alloc_n<int32_t>(c, c->ntiles);
  // mailboxes: an edge box holds half a tile column of the species' lattice, a corner box 32;
  // with a moving window 1.5 columns (every shift moves each tile's first column into the -x box)
  MailBox& M = c->mail[s];
  const int ppc = c->species[s].ppc[0] * c->species[s].ppc[1];
  const int edge = c->bcx == ZPIC_BC_MOVING_WINDOW ? c->T * ppc * 3 / 2 : c->T * ppc / 2;
  M.cap_edge = round_up(std::max(32, std::min(edge, cap)), 32);
  M.cap_corner = 32;
  M.per_tile = 4 * M.cap_edge + 4 * M.cap_corner;
  M.stride = (long)c->ntiles * M.per_tile;
  M.nf = ps.nf;
  M.data = (uint32_t*)dev_alloc(c, (size_t)M.stride * M.nf * sizeof(uint32_t));
  M.cnt = alloc_n<int32_t>(c, (size_t)c->ntiles * 8);
}

// The tile current is accumulated as fixed point with a per-tile scale 2^S chosen from the
// tile's particle count (zpic_kernels.cuh fx_scale_exponent), which needs 2 * (particles per
// tile) well below 2^31; 2^24 particles per tile is the sanity limit.
void check_tile_capacity(zpic_ctx* c) {
  long total = 0;
  for (int s = 0; s < c->nspecies; ++s) total += c->ps[s].cap;
  if (total > (1L << 24))
    throw Fail{ZPIC_E_INVALID, "tile capacity " + std::to_string(total) +
                                   " > 2^24 particles (fixed-point current range): use a smaller tile"};
}

void free_store(zpic_ctx* c, int s) {
  PStore& ps = c->ps[s];
  dev_free(c, ps.data); dev_free(c, ps.cnt);
  ps = PStore{};
  dev_free(c, c->mail[s].data); dev_free(c, c->mail[s].cnt);
  c->mail[s] = MailBox{};
}

PList alloc_list(zpic_ctx* c, int cap) {
  PList L{};
  L.cap = cap;
  L.cell = alloc_n<int32_t>(c, cap);
  L.x = alloc_n<float>(c, cap);
  L.y = alloc_n<float>(c, cap);
  L.ux = alloc_n<float>(c, cap);
  L.uy = alloc_n<float>(c, cap);
  L.uz = alloc_n<float>(c, cap);
  L.id = c->opt.track_ids ? alloc_n<uint32_t>(c, cap) : nullptr;
  L.species = alloc_n<int32_t>(c, cap);
  L.count = alloc_n<int32_t>(c, 1);
  return L;
}

// Mover / loose list capacity: mover_fraction of the largest population the run can reach (with a
// moving window the injected plasma fills the box: nx * ny * ppc per species); on window-shift
// steps every particle of a tile's first column changes tile, so add 1.5 / T of it.
int mover_capacity(zpic_ctx* c, int64_t total) {
  int64_t pop = total;
  double frac = c->opt.mover_fraction;
  if (c->bcx == ZPIC_BC_MOVING_WINDOW) {
    int64_t full = 0;
    for (int s = 0; s < c->nspecies; ++s)
      if (c->species[s].n > 0) full += (int64_t)c->g.nx * c->g.ny * c->species[s].ppc[0] * c->species[s].ppc[1];
    pop = std::max(pop, full);
    frac += 1.5 / c->T;
  }
  const int64_t cap = std::max<int64_t>(65536, (int64_t)std::ceil(pop * frac));
  if (cap > 2000000000) throw Fail{ZPIC_E_INVALID, "mover list capacity exceeds 2^31"};
  return (int)cap;
}

// Guard mode of an axis for a field (E, B) or the current.
int field_guard_mode(int bc) { return bc == ZPIC_BC_PERIODIC ? 1 : 2; }

void refresh_field_guards(zpic_ctx* c, float* F, bool is_E) {
  const int kx = (is_E && c->bcx == ZPIC_BC_OPEN) ? 0b110 : 0;  // Ey, Ez keep node nx
  const int ky = (is_E && c->bcy == ZPIC_BC_OPEN) ? 0b101 : 0;  // Ex, Ez keep node ny
  launch_guard_x(F, c->g, kx ? 3 : field_guard_mode(c->bcx), kx, c->stream);
  if (c->slab) {
    // slab interfaces get their guard rows from the neighbours before the next step
    if (c->bcy != ZPIC_BC_PERIODIC) launch_guard_y(F, c->g, ky ? 3 : 2, ky, c->stream);
    c->halo_dirty = true;
  } else {
    launch_guard_y(F, c->g, ky ? 3 : field_guard_mode(c->bcy), ky, c->stream);
  }
}

// ---- profiling ---------------------------------------------------------------------------
constexpr int kSortEveryDefault = 0;   // steps between K2s re-sorts (ZPIC_SORT_EVERY overrides; 0 = off)
enum KId { K_PUSH = 0, K_INSERT, K_ASSEMBLE, K_LOOSE, K_FOLD, K_HALO, K_FILTER, K_YEE, K_WINDOW, K_EPI, K_EXCHANGE,
           K_MAIL, K_SORT, K_SCALE, K_COUNT };
const char* kNames[K_COUNT] = {"k_push_tiles", "k_insert",        "k_assemble_j", "k_push_loose",
                               "k_guard_fold", "k_apply_halo",    "k_filter_x",   "k_yee",
                               "k_inject_column", "k_epilogue",   "halo_exchange", "k_mail_gather",
                               "k_sort_tiles", "k_tile_scale"};

struct ProfScope {
  zpic_ctx* c;
  int id;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(zpic_ctx* c_, int id_) : c(c_), id(id_) {
    if (!c->prof) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, c->stream);
  }
  ~ProfScope() {
    if (!c->prof) return;
    cudaEventRecord(b, c->stream);
    c->prof_ev.push_back(a);
    c->prof_ev.push_back(b);
    c->prof_pending.push_back({id, (int)c->prof_ev.size() - 2});
  }
};

void drain_profile(zpic_ctx* c) {
  for (auto& pr : c->prof_pending) {
    float ms = 0.f;
    cudaEventSynchronize(c->prof_ev[pr.second + 1]);
    cudaEventElapsedTime(&ms, c->prof_ev[pr.second], c->prof_ev[pr.second + 1]);
    c->prof_ms[pr.first] += ms;
    c->prof_count[pr.first] += 1;
  }
  for (auto e : c->prof_ev) cudaEventDestroy(e);
  c->prof_ev.clear();
  c->prof_pending.clear();
}

// Smallest per-tile fixed-point exponent for the one-word int32 current (kSMin; the environment
// variable ZPIC_FX_SMIN overrides it for precision experiments: 99 forces the exact two-word form).
int fx_smin() {
  static int v = [] {
    const char* e = getenv("ZPIC_FX_SMIN");
    return e ? atoi(e) : kSMin;
  }();
  return v;
}

PushParams push_params(zpic_ctx* c) {
  PushParams p{};
  p.tmE = c->tm[0][c->cur];
  p.tmB = c->tm[1][c->cur];
  p.g = c->g;
  p.E = c->E[c->cur];
  p.B = c->B[c->cur];
  p.J = c->J;
  p.Jt = c->Jt;
  p.commutative = c->opt.current_mode == 1;
  static const int mail = [] { const char* e = getenv("ZPIC_MAIL"); return e ? atoi(e) : 1; }();
  p.use_mail = mail;
  for (int s = 0; s < c->nspecies; ++s) p.mail[s] = c->mail[s];
  p.fx_smin = c->opt.current_precision == 1 ? 99 : fx_smin();
  p.occ = c->occ;
  p.tscale = c->tscale;
  p.hist = c->hist;
  p.check_occ = c->check_occ;
  p.qmax = 0.f;
  for (int s = 0; s < c->nspecies; ++s) p.qmax = std::max(p.qmax, std::fabs(c->sc[s].q));
  p.T = c->T; p.ntx = c->ntx; p.nty = c->nty;
  p.nspecies = c->nspecies;
  for (int s = 0; s < c->nspecies; ++s) { p.sc[s] = c->sc[s]; p.ps[s] = c->ps[s]; }
  p.movers = c->movers;
  p.spill_in = c->spill[c->steps & 1];
  p.spill_out = c->spill[(c->steps + 1) & 1];
  p.dtdx = (float)(c->dt / c->dx);
  p.dtdy = (float)(c->dt / c->dy);
  p.bcx = c->bcx; p.bcy = c->bcy;
  p.ke_slots = c->ke_slots;
  p.err = c->err;
  p.slab = c->slab;
  p.has_lo = c->has_lo;
  p.has_hi = c->has_hi;
  static const int skip = [] { const char* e = getenv("ZPIC_SKIP_CELL_STORE"); return e ? atoi(e) : 0; }();
  p.skip_cell_store = skip;
  if (c->slab) {
    p.send[0] = particle_msg_list(c->pmsg_send[0], c->pcap);
    p.send[1] = particle_msg_list(c->pmsg_send[1], c->pcap);
    if (c->peer) {   // PEER: the slab exits go straight into the neighbours' receive areas (K3, K1L)
      if (c->has_lo) p.send[0] = particle_msg_list(c->peer_lo.pmsg[1], c->pcap);
      if (c->has_hi) p.send[1] = particle_msg_list(c->peer_hi.pmsg[0], c->pcap);
      p.peer_send = 1;
    }
  }
  if (c->peer_j) {   // cross-slab commutative current: the neighbours' J
    p.Jlo = c->has_lo ? c->jlo : nullptr;
    p.Jhi = c->has_hi ? c->jhi : nullptr;
    p.lo_plane = c->lo_plane;
    p.hi_plane = c->hi_plane;
    p.lo_ny = c->lo_ny;
  }
  return p;
}

// ---- y-slab halo exchange (§8(e)) ----------------------------------------------------------
// Message order per neighbour pair is fixed so that ring sizes 1 and 2 (where the lower and
// the upper neighbour are the same rank) match sends with receives: first everything that
// travels up (+y), then everything that travels down (-y).
float* jrow(zpic_ctx* c, int comp, int row) { return c->J + comp * c->g.plane + (long)(row + 1) * c->g.pitch; }
float* frow(float* F, const GridDesc& g, int comp, int row) { return F + comp * g.plane + (long)(row + 1) * g.pitch; }

ncclResult_t nccl_exchange_round1(zpic_ctx* c, cudaStream_t st) {
  ncclComm_t comm = (ncclComm_t)c->comm;
  const size_t rows2 = 2 * (size_t)c->g.pitch;
  const size_t mb = particle_msg_bytes(c->pcap);
  ncclResult_t r = ncclGroupStart();
  if (c->has_hi) {   // up: my raw J rows ny, ny+1 and my up-going particles
    for (int k = 0; k < 3 && r == ncclSuccess; ++k) r = ncclSend(jrow(c, k, c->g.ny), rows2, ncclFloat, c->upper, comm, st);
    if (r == ncclSuccess) r = ncclSend(c->pmsg_send[1], mb, ncclChar, c->upper, comm, st);
  }
  if (c->has_lo && r == ncclSuccess) {   // from below: the lower's rows ny, ny+1 and its up-going particles
    for (int k = 0; k < 3 && r == ncclSuccess; ++k) r = ncclRecv(c->jrdn + k * rows2, rows2, ncclFloat, c->lower, comm, st);
    if (r == ncclSuccess) r = ncclRecv(c->pmsg_recv[0], mb, ncclChar, c->lower, comm, st);
  }
  if (c->has_lo && r == ncclSuccess) {   // down: my raw J rows -1, 0 and my down-going particles
    for (int k = 0; k < 3 && r == ncclSuccess; ++k) r = ncclSend(jrow(c, k, -1), rows2, ncclFloat, c->lower, comm, st);
    if (r == ncclSuccess) r = ncclSend(c->pmsg_send[0], mb, ncclChar, c->lower, comm, st);
  }
  if (c->has_hi && r == ncclSuccess) {   // from above: the upper's rows -1, 0 and its down-going particles
    for (int k = 0; k < 3 && r == ncclSuccess; ++k) r = ncclRecv(c->jrup + k * rows2, rows2, ncclFloat, c->upper, comm, st);
    if (r == ncclSuccess) r = ncclRecv(c->pmsg_recv[1], mb, ncclChar, c->upper, comm, st);
  }
  ncclResult_t e = ncclGroupEnd();
  return r != ncclSuccess ? r : e;
}

// Round 2: E, B ghost rows of buffer `b`: my row ny-1 -> the upper's guard row -1 (up); my rows
// 0, 1 -> the lower's guard rows ny, ny+1 (down).
ncclResult_t nccl_exchange_round2(zpic_ctx* c, int b, cudaStream_t st) {
  ncclComm_t comm = (ncclComm_t)c->comm;
  const GridDesc& g = c->g;
  const size_t row = g.pitch;
  float* F[2] = {c->E[b], c->B[b]};
  ncclResult_t r = ncclGroupStart();
  for (int f = 0; f < 2 && c->has_hi && r == ncclSuccess; ++f)
    for (int k = 0; k < 3 && r == ncclSuccess; ++k) r = ncclSend(frow(F[f], g, k, g.ny - 1), row, ncclFloat, c->upper, comm, st);
  for (int f = 0; f < 2 && c->has_lo && r == ncclSuccess; ++f)
    for (int k = 0; k < 3 && r == ncclSuccess; ++k) r = ncclRecv(frow(F[f], g, k, -1), row, ncclFloat, c->lower, comm, st);
  for (int f = 0; f < 2 && c->has_lo && r == ncclSuccess; ++f)
    for (int k = 0; k < 3 && r == ncclSuccess; ++k) r = ncclSend(frow(F[f], g, k, 0), 2 * row, ncclFloat, c->lower, comm, st);
  for (int f = 0; f < 2 && c->has_hi && r == ncclSuccess; ++f)
    for (int k = 0; k < 3 && r == ncclSuccess; ++k) r = ncclRecv(frow(F[f], g, k, g.ny), 2 * row, ncclFloat, c->upper, comm, st);
  ncclResult_t e = ncclGroupEnd();
  return r != ncclSuccess ? r : e;
}

// Loopback versions (all contexts of a group share one device and one stream).
void loop_exchange_round1(zpic_ctx** cs, int n) {
  for (int r = 0; r < n; ++r) {
    zpic_ctx* c = cs[r];
    const size_t rows2b = 2 * (size_t)c->g.pitch * sizeof(float);
    const size_t mb = particle_msg_bytes(c->pcap);
    if (c->has_lo) {
      zpic_ctx* lo = cs[c->lower];
      CUDA_OR_THROW(cudaMemcpy2DAsync(c->jrdn, rows2b, jrow(lo, 0, lo->g.ny), lo->g.plane * sizeof(float), rows2b, 3,
                                      cudaMemcpyDeviceToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(c->pmsg_recv[0], lo->pmsg_send[1], mb, cudaMemcpyDeviceToDevice, c->stream));
    }
    if (c->has_hi) {
      zpic_ctx* up = cs[c->upper];
      CUDA_OR_THROW(cudaMemcpy2DAsync(c->jrup, rows2b, jrow(up, 0, -1), up->g.plane * sizeof(float), rows2b, 3,
                                      cudaMemcpyDeviceToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(c->pmsg_recv[1], up->pmsg_send[0], mb, cudaMemcpyDeviceToDevice, c->stream));
    }
  }
}

void loop_exchange_round2(zpic_ctx** cs, int n, int b) {
  for (int r = 0; r < n; ++r) {
    zpic_ctx* c = cs[r];
    const GridDesc& g = c->g;
    const size_t rowb = (size_t)g.pitch * sizeof(float);
    for (int f = 0; f < 2; ++f) {
      if (c->has_lo) {
        zpic_ctx* lo = cs[c->lower];
        float* src = f ? lo->B[b] : lo->E[b];
        float* dst = f ? c->B[b] : c->E[b];
        CUDA_OR_THROW(cudaMemcpy2DAsync(frow(dst, g, 0, -1), g.plane * sizeof(float), frow(src, g, 0, g.ny - 1),
                                        g.plane * sizeof(float), rowb, 3, cudaMemcpyDeviceToDevice, c->stream));
      }
      if (c->has_hi) {
        zpic_ctx* up = cs[c->upper];
        float* src = f ? up->B[b] : up->E[b];
        float* dst = f ? c->B[b] : c->E[b];
        CUDA_OR_THROW(cudaMemcpy2DAsync(frow(dst, g, 0, g.ny), g.plane * sizeof(float), frow(src, g, 0, 0),
                                        g.plane * sizeof(float), 2 * rowb, 3, cudaMemcpyDeviceToDevice, c->stream));
      }
    }
  }
}

zpic_status check_sticky(zpic_ctx* c) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) { c->last_error = std::string("CUDA: ") + cudaGetErrorString(e); return ZPIC_E_CUDA; }
  int err = 0;
  cudaMemcpy(&err, c->err, sizeof(int), cudaMemcpyDeviceToHost);
  if (err & ERR_OVERFLOW) {
    int counts[3] = {0, 0, 0};
    cudaMemcpy(&counts[0], c->movers.count, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&counts[1], c->spill[0].count, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&counts[2], c->spill[1].count, 4, cudaMemcpyDeviceToHost);
    c->last_error = "particle capacity overflow (mover / loose / send list full): movers " + std::to_string(counts[0]) +
                    " loose " + std::to_string(counts[1]) + "/" + std::to_string(counts[2]) + " cap " +
                    std::to_string(c->movers.cap) + " err " + std::to_string(err) + " steps " + std::to_string(c->steps);
    return ZPIC_E_OVERFLOW;
  }
  if (err & ERR_HALO) {
    c->last_error = "slab halo particle message full: more than " + std::to_string(c->pcap) +
                    " particles crossed a slab edge in one step (raise zpic_options.halo_particles)";
    return ZPIC_E_OVERFLOW;
  }
  if (err & ERR_MIGRATION) { c->last_error = "a particle moved >= 1 cell in one step"; return ZPIC_E_MIGRATION; }
  if (err & ERR_HIST) { c->last_error = "tile cell histogram / occupancy bound inconsistent (ZPIC_CHECK_OCC)"; return ZPIC_E_STATE; }
  return ZPIC_OK;
}

}  // namespace

// =============================================================================================
extern "C" {

const char* zpic_last_error(const zpic_ctx* ctx) { return ctx ? ctx->last_error.c_str() : g_init_error.c_str(); }

static void load_species(zpic_ctx* c, int s, int64_t n, char* tmp, bool has_id);
static void size_lists(zpic_ctx* c, int64_t extra = 0);

// PEER across processes: the CUDA IPC handles of every rank's receive block, all-gathered once on
// the NCCL communicator; the y neighbours' blocks opened (peer access over NVLink).
struct PeerRecord {
  cudaIpcMemHandle_t block, j, eb;   // the receive block; J (cross-slab commutative current only); E/B
  int32_t ny;
  int32_t pad[15];
};
static void open_peer_blocks(zpic_ctx* c) {
  PeerRecord mine{};
  CUDA_OR_THROW(cudaIpcGetMemHandle(&mine.block, c->peer_block));
  if (c->peer_j) CUDA_OR_THROW(cudaIpcGetMemHandle(&mine.j, c->j_block));
  CUDA_OR_THROW(cudaIpcGetMemHandle(&mine.eb, c->eb_block));
  mine.ny = c->g.ny;
  const size_t hb = sizeof(PeerRecord);
  char* dbuf = alloc_n<char>(c, hb * (c->world + 1));
  CUDA_OR_THROW(cudaMemcpyAsync(dbuf + hb * c->world, &mine, hb, cudaMemcpyHostToDevice, c->stream));
  ncclResult_t r = ncclAllGather(dbuf + hb * c->world, dbuf, hb, ncclChar, (ncclComm_t)c->comm, c->stream);
  if (r != ncclSuccess) throw Fail{ZPIC_E_NCCL, std::string("PEER handle all-gather: ") + ncclGetErrorString(r)};
  std::vector<PeerRecord> all(c->world);
  CUDA_OR_THROW(cudaMemcpyAsync(all.data(), dbuf, hb * c->world, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  dev_free(c, dbuf);
  std::vector<void*> opened(3 * c->world, nullptr);   // each peer allocation opened once per process
  auto open_ptr = [&](int rank, int which) -> void* {   // 0 receive block, 1 J, 2 E/B
    if (rank == c->rank) return which == 2 ? c->eb_block : which ? c->j_block : c->peer_block;
    void*& p = opened[3 * rank + which];
    if (!p) {
      const cudaIpcMemHandle_t& h = which == 2 ? all[rank].eb : which ? all[rank].j : all[rank].block;
      CUDA_OR_THROW(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      c->ipc_open.push_back(p);
    }
    return p;
  };
  const long row_floats = c->g.pitch;
  auto view_of = [&](int rank) {
    PeerView v = peer_view(open_ptr(rank, 0), c->g.pitch, c->pcap);
    float* eb = (float*)open_ptr(rank, 2);
    v.ny = all[rank].ny;
    v.plane = (long)(all[rank].ny + 3) * row_floats;
    for (int b = 0; b < 2; ++b) { v.E[b] = eb + (size_t)b * 3 * v.plane; v.B[b] = eb + (size_t)(2 + b) * 3 * v.plane; }
    return v;
  };
  if (c->has_lo) {
    c->peer_lo = view_of(c->lower);
    if (c->peer_j) {
      c->jlo = (float*)open_ptr(c->lower, 1);
      c->lo_ny = all[c->lower].ny;
      c->lo_plane = (long)(all[c->lower].ny + 3) * row_floats;
    }
  }
  if (c->has_hi) {
    c->peer_hi = view_of(c->upper);
    if (c->peer_j) {
      c->jhi = (float*)open_ptr(c->upper, 1);
      c->hi_plane = (long)(all[c->upper].ny + 3) * row_floats;
    }
  }
}

// The one x sub-row of a ramp species (R16), in the oracle-independent arithmetic of the library:
// ramp positions by cumulative inversion, then the regular sub-lattice from x1 on; cell index and
// fp32 offset with the R6 rule.
static void ramp_row(const zpic_species& sp, int nx, double dx, std::vector<int32_t>& ix, std::vector<float>& x) {
  const int px = sp.ppc[0];
  const double x0 = sp.x0, x1 = sp.x1, L = x1 - x0;
  std::vector<double> X;
  const long nramp = (long)std::nearbyint(px * L / (2.0 * dx));
  for (long k = 0; k < nramp; ++k) X.push_back(x0 + std::sqrt(2.0 * L * ((double)k + 0.5) * dx / px));
  const int first = (int)std::ceil(x1 / dx - 1e-9);
  for (int col = std::max(first, 0); col < nx; ++col)
    for (int k = 0; k < px; ++k) X.push_back(((double)col + ((double)k + 0.5) / px) * dx);
  ix.clear(); x.clear();
  for (double Xv : X) {
    const double gx = Xv / dx;
    int i = (int)std::floor(gx);
    float f = (float)(gx - i);
    if (f >= 1.0f) { i += 1; f = 0.0f; }
    if (i < 0 || i >= nx) continue;
    ix.push_back(i);
    x.push_back(f);
  }
}

zpic_status zpic_init(zpic_ctx** out, const zpic_grid* grid, double dt, const zpic_species* species, int32_t n_species,
                      const zpic_boundaries* bc, uint64_t seed, const zpic_options* options, const zpic_dist* dist) {
  if (!out || !grid || !species || !bc) { g_init_error = "NULL argument"; return ZPIC_E_INVALID; }
  *out = nullptr;
  if (grid->nx < 1 || grid->ny < 1) { g_init_error = "nx, ny must be >= 1"; return ZPIC_E_EMPTY_GRID; }
  if (grid->nx < 2 || grid->ny < 2 || grid->nx > 32767 || grid->ny > 32767) {
    g_init_error = "nx, ny must be in [2, 32767]"; return ZPIC_E_INVALID;
  }
  if (!(grid->dx > 0) || !(grid->dy > 0) || !(dt > 0)) { g_init_error = "dx, dy, dt must be > 0"; return ZPIC_E_INVALID; }
  const double cfl = 1.0 / std::sqrt(1.0 / (grid->dx * grid->dx) + 1.0 / (grid->dy * grid->dy));
  if (dt >= cfl) { g_init_error = "CFL: dt >= " + std::to_string(cfl); return ZPIC_E_CFL; }
  if (n_species < 0 || n_species > kMaxSpecies) { g_init_error = "n_species must be in [0, 4]"; return ZPIC_E_INVALID; }
  for (int s = 0; s < n_species; ++s) {
    const zpic_species& sp = species[s];
    if (sp.ppc[0] < 1 || sp.ppc[1] < 1 || sp.m_q == 0.0 || !(sp.n >= 0))
      { g_init_error = "species " + std::to_string(s) + ": ppc >= 1, m_q != 0, n >= 0"; return ZPIC_E_INVALID; }
    for (int k = 0; k < 3; ++k)
      if (sp.uth[k] < 0) { g_init_error = "species " + std::to_string(s) + ": uth >= 0"; return ZPIC_E_INVALID; }
  }
  if (bc->y == ZPIC_BC_MOVING_WINDOW) { g_init_error = "moving window is x only"; return ZPIC_E_INVALID; }
  if (bc->x == ZPIC_BC_MOVING_WINDOW)   // R15: the injected column takes the profile beyond its end
    for (int s = 0; s < n_species; ++s)
      if (species[s].profile == ZPIC_DENS_SLAB ||
          (species[s].profile == ZPIC_DENS_RAMP && species[s].x1 > grid->nx * grid->dx)) {
        g_init_error = "species " + std::to_string(s) +
                       ": a moving window needs a uniform profile or a ramp that ends inside the box (R15)";
        return ZPIC_E_INVALID;
      }
  if (dist) {
    if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world) { g_init_error = "bad rank / world"; return ZPIC_E_DECOMP; }
    if (grid->ny % dist->world != 0 || grid->ny / dist->world < 2) {
      g_init_error = "ny must be a multiple of world with >= 2 rows per slab"; return ZPIC_E_DECOMP;
    }
    if ((dist->transport == ZPIC_TRANSPORT_NCCL || (dist->transport == ZPIC_TRANSPORT_PEER && dist->world > 1)) &&
        !dist->nccl_comm && !dist->nccl_id) {
      g_init_error = "NCCL / PEER transport needs nccl_comm or nccl_id"; return ZPIC_E_DECOMP;
    }
    if (dist->transport < ZPIC_TRANSPORT_NCCL || dist->transport > ZPIC_TRANSPORT_LOOPBACK_PEER) {
      g_init_error = "unknown transport"; return ZPIC_E_DECOMP;
    }
  }

  zpic_ctx* c = new zpic_ctx();
  try {
    c->opt = zpic_options{};
    c->opt.tile[0] = c->opt.tile[1] = 0;   // auto (below)
    c->opt.capacity_slack = 1.25;
    c->opt.mover_fraction = 0.05;
    if (options) {
      c->opt = *options;
      if (c->opt.capacity_slack <= 0) c->opt.capacity_slack = 1.25;
      if (c->opt.mover_fraction <= 0) c->opt.mover_fraction = 0.05;
    }
    if (c->opt.tile[0] != c->opt.tile[1] ||
        (c->opt.tile[0] != 0 && c->opt.tile[0] != 8 && c->opt.tile[0] != 16 && c->opt.tile[0] != 32))
      throw Fail{ZPIC_E_INVALID, "tile must be 8x8, 16x16 or 32x32"};
    if (c->opt.stream) { c->stream = (cudaStream_t)c->opt.stream; c->own_stream = false; }
    else { CUDA_OR_THROW(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)); c->own_stream = true; }
    c->prof = c->opt.profile != 0;
    {
      const char* e = getenv("ZPIC_SORT_EVERY");   // read per context
      c->sort_every = e ? atoi(e) : kSortEveryDefault;
    }
    c->prof_ms.assign(K_COUNT, 0.0);
    c->prof_count.assign(K_COUNT, 0);
    if (dist) c->dist = *dist; else c->dist = zpic_dist{0, 1, nullptr, 0, nullptr, ZPIC_TRANSPORT_NCCL};
    c->nx_global = grid->nx; c->ny_global = grid->ny;
    c->slab = dist != nullptr;
    c->rank = c->dist.rank; c->world = c->dist.world;
    c->transport = c->dist.transport;
    c->lower = (c->rank + c->world - 1) % c->world;
    c->upper = (c->rank + 1) % c->world;
    c->has_lo = bc->y == ZPIC_BC_PERIODIC || c->rank > 0;
    c->has_hi = bc->y == ZPIC_BC_PERIODIC || c->rank < c->world - 1;
    const int ny_local = grid->ny / c->world;
    c->y0 = c->rank * ny_local;
    c->dx = grid->dx; c->dy = grid->dy; c->dt = dt;
    c->bcx = bc->x; c->bcy = bc->y;
    c->nspecies = n_species;
    c->seed = seed;
    for (int s = 0; s < n_species; ++s) c->species[s] = species[s];
    GridDesc& g = c->g;
    g.nx = grid->nx; g.ny = ny_local;
    g.pitch = round_up(g.nx + kXOff + 2, 32);
    g.rows = g.ny + 3;
    g.plane = (long)g.rows * g.pitch;
    // tile 0 = auto: 16 x 16 (the C5-tuned K1 shape) unless that leaves fewer than 2 tiles per SM,
    // then 8 x 8 (small grids such as C1, C2 are otherwise latency-bound on a few CTAs)
    c->T = c->opt.tile[0] ? c->opt.tile[0]
                          : (((g.nx + 15) / 16) * ((g.ny + 15) / 16) >= 2 * 148 ? 16 : 8);
    c->ntx = (g.nx + c->T - 1) / c->T;
    c->nty = (g.ny + c->T - 1) / c->T;
    c->ntiles = c->ntx * c->nty;
    for (int s = 0; s < n_species; ++s) {
      const zpic_species& sp = species[s];
      const int ppc = sp.ppc[0] * sp.ppc[1];
      SpeciesConst& k = c->sc[s];
      const double q = (sp.m_q > 0 ? 1.0 : -1.0) * sp.n / ppc;   // R8
      k.q = (float)q;
      k.h = (float)(0.5 * dt / sp.m_q);
      k.jx = (float)(q * grid->dx / dt);
      k.jy = (float)(q * grid->dy / dt);
      k.ke_scale = q * sp.m_q * grid->dx * grid->dy;
    }
    // fields
    const bool peer_tr = c->slab && (c->transport == ZPIC_TRANSPORT_PEER || c->transport == ZPIC_TRANSPORT_LOOPBACK_PEER);
    if (peer_tr) {   // PEER: the neighbours write their round-2 rows into these buffers (CUDA IPC export)
      CUDA_OR_THROW(cudaMalloc(&c->eb_block, sizeof(float) * 12 * g.plane));
      CUDA_OR_THROW(cudaMemsetAsync(c->eb_block, 0, sizeof(float) * 12 * g.plane, c->stream));
      for (int b = 0; b < 2; ++b) {
        c->E[b] = (float*)c->eb_block + (size_t)b * 3 * g.plane;
        c->B[b] = (float*)c->eb_block + (size_t)(2 + b) * 3 * g.plane;
      }
    } else {
      for (int b = 0; b < 2; ++b) { c->E[b] = alloc_n<float>(c, 3 * g.plane); c->B[b] = alloc_n<float>(c, 3 * g.plane); }
    }
    for (int b = 0; b < 2; ++b) {   // TMA maps for K1's staging of a tile's fields (+1 cell halo)
      make_field_tmap(&c->tm[0][b], c->E[b], g, c->T);
      make_field_tmap(&c->tm[1][b], c->B[b], g, c->T);
    }
    c->peer_j = c->slab && c->opt.current_mode == 1 &&
                (c->transport == ZPIC_TRANSPORT_PEER || c->transport == ZPIC_TRANSPORT_LOOPBACK_PEER);
    if (c->peer_j) {   // its own cudaMalloc: the neighbours open it with CUDA IPC
      CUDA_OR_THROW(cudaMalloc(&c->j_block, sizeof(float) * 3 * g.plane));
      c->J = (float*)c->j_block;
      c->jlo = c->jhi = c->J;   // a one-rank ring adds into itself; groups / IPC rebind them
      c->lo_plane = c->hi_plane = g.plane;
      c->lo_ny = g.ny;
    } else {
      c->J = alloc_n<float>(c, 3 * g.plane);
    }
    c->Jf = c->opt.filter_passes > 0 ? alloc_n<float>(c, 3 * g.plane) : nullptr;
    // K5's TMA maps (boxes: zpic_kernels.cu YeeBox)
    for (int b = 0; b < 2; ++b) {
      make_tmap(&c->ytm[0][b], c->E[b], g, kYeeTX + 8, kYeeTY + 3);
      make_tmap(&c->ytm[1][b], c->B[b], g, kYeeTX + 8, kYeeTY + 2);
    }
    make_tmap(&c->ytmJ[0], c->J, g, kYeeTX + 4, kYeeTY + 1);
    if (c->Jf) make_tmap(&c->ytmJ[1], c->Jf, g, kYeeTX + 4, kYeeTY + 1);
    if (c->opt.filter_passes < 0 || c->opt.filter_passes > 64) throw Fail{ZPIC_E_INVALID, "filter_passes must be in [0, 64]"};
    if (c->opt.current_mode != 0 && c->opt.current_mode != 1) throw Fail{ZPIC_E_INVALID, "current_mode must be 0 or 1"};
    const int WJ = c->T + 3;
    c->Jt = c->opt.current_mode == 1 ? nullptr : alloc_n<float>(c, (size_t)c->ntiles * 3 * WJ * WJ);
    c->ke_slots = alloc_n<double>(c, kMaxSpecies * kEnergySlots);
    c->fe_slots = alloc_n<double>(c, kEnergySlots);
    c->energy = alloc_n<double>(c, 1 + 2 * kMaxSpecies);
    c->err = alloc_n<int>(c, 1);
    c->stats = alloc_n<int>(c, 4);
    c->occ = alloc_n<int32_t>(c, (size_t)c->ntiles);
    c->tscale = alloc_n<int32_t>(c, (size_t)c->ntiles);
    c->hist = alloc_n<int32_t>(c, (size_t)c->ntiles * c->T * c->T);
    {
      const char* e = getenv("ZPIC_CHECK_OCC");   // read per context (tests)
      c->check_occ = e ? atoi(e) : 0;
    }
    if (c->opt.current_precision != 0 && c->opt.current_precision != 1)
      throw Fail{ZPIC_E_INVALID, "current_precision must be 0 or 1"};
    {
      double kes[kMaxSpecies] = {0, 0, 0, 0};
      for (int s = 0; s < n_species; ++s) kes[s] = c->sc[s].ke_scale;
      CUDA_OR_THROW(cudaMemcpyAsync(c->energy + 1 + kMaxSpecies, kes, sizeof(kes), cudaMemcpyHostToDevice, c->stream));
    }
    // particles: per-tile capacity from the largest initial tile count
    int64_t total = 0;
    for (int s = 0; s < n_species; ++s) {
      const zpic_species& sp = species[s];
      const int ppc = sp.ppc[0] * sp.ppc[1];
      int col_lo = 0, col_hi = g.nx;
      if (sp.profile == ZPIC_DENS_SLAB) {
        col_lo = (int)std::ceil(sp.x0 / grid->dx - 0.5);
        col_hi = (int)std::ceil(sp.x1 / grid->dx - 0.5);
        col_lo = std::max(0, std::min(g.nx, col_lo));
        col_hi = std::max(col_lo, std::min(g.nx, col_hi));
      }
      int maxcount = c->T * c->T * ppc;
      if (sp.profile == ZPIC_DENS_NONE || sp.profile == ZPIC_DENS_RAMP || sp.n == 0.0) { col_lo = col_hi = 0; }
      // the device injector writes every lattice particle into its tile: no less than a full tile
      // (also for NONE, which zpic_set_particles then usually fills without reallocating); a ramp
      // species is sized when it is loaded below
      const bool later = sp.profile == ZPIC_DENS_RAMP;
      const int cap = later ? 32
                            : std::max(32, round_up((int)std::ceil(maxcount * (sp.profile == ZPIC_DENS_NONE
                                                                                    ? c->opt.capacity_slack
                                                                                    : std::max(1.0, c->opt.capacity_slack))),
                                                    32));
      if ((double)cap * c->ntiles > 2.0e9) throw Fail{ZPIC_E_INVALID, "particle store exceeds 2^31 slots"};
      alloc_store(c, s, cap);
      check_tile_capacity(c);
      if (col_hi > col_lo) {
        InjectParams q{};
        q.ps = c->ps[s];
        q.T = c->T; q.ntx = c->ntx; q.nx_global = g.nx; q.y0 = c->y0; q.ny = g.ny;
        q.px = sp.ppc[0]; q.py = sp.ppc[1];
        q.col_lo = col_lo; q.col_hi = col_hi;
        q.key = host_mix64(host_mix64(seed) + (uint64_t)s);
        for (int k = 0; k < 3; ++k) { q.ufl[k] = sp.ufl[k]; q.uth[k] = sp.uth[k]; }
        launch_inject(q, c->ntiles, c->stream);
        total += (int64_t)(col_hi - col_lo) * g.ny * ppc;
      }
    }
    c->population = total;
    c->d_nmove = alloc_n<int64_t>(c, 1);
    const int mcap = mover_capacity(c, total);
    c->movers = alloc_list(c, (int)mcap);
    c->spill[0] = alloc_list(c, (int)mcap);
    c->spill[1] = alloc_list(c, (int)mcap);
    c->cur = 0;
    c->steps = 0;
    // ramp species (R16): generated on the device from one host-computed x sub-row, then binned
    bool ramped = false;
    for (int s = 0; s < n_species; ++s) {
      const zpic_species& sp = species[s];
      if (sp.profile != ZPIC_DENS_RAMP || !(sp.n > 0)) continue;
      std::vector<int32_t> ixr;
      std::vector<float> xr;
      ramp_row(sp, g.nx, grid->dx, ixr, xr);
      const int n_row = (int)ixr.size();
      const int64_t n = (int64_t)n_row * g.ny * sp.ppc[1];
      int32_t* dixr = alloc_n<int32_t>(c, std::max(n_row, 1));
      float* dxr = alloc_n<float>(c, std::max(n_row, 1));
      CUDA_OR_THROW(cudaMemcpyAsync(dixr, ixr.data(), n_row * 4, cudaMemcpyHostToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(dxr, xr.data(), n_row * 4, cudaMemcpyHostToDevice, c->stream));
      char* tmp = (char*)dev_alloc(c, (size_t)std::max<int64_t>(n, 1) * 32);
      int32_t* dix = (int32_t*)tmp;
      int32_t* diy = dix + n;
      float* dxx = (float*)(diy + n);
      float* dyy = dxx + n;
      float* dux = dyy + n;
      float* duy = dux + n;
      float* duz = duy + n;
      uint32_t* did = (uint32_t*)(duz + n);
      launch_ramp_rows((long)n, n_row, sp.ppc[1], c->y0, dixr, dxr, host_mix64(host_mix64(seed) + (uint64_t)s), sp.ufl,
                       sp.uth, dix, diy, dxx, dyy, dux, duy, duz, c->opt.track_ids ? did : nullptr, c->stream);
      CUDA_OR_THROW(cudaGetLastError());
      load_species(c, s, n, tmp, c->opt.track_ids != 0);
      dev_free(c, dixr);
      dev_free(c, dxr);
      ramped = true;
    }
    if (ramped) size_lists(c);
    // laser initial fields (R17)
    if (c->opt.laser) {
      const LaserParams L{c->opt.laser_a0, c->opt.laser_omega0, c->opt.laser_fwhm, c->opt.laser_W0, c->opt.laser_start,
                          0.5 * grid->ny * grid->dy};
      if (!(L.fwhm > 0) || !(L.W0 > 0)) throw Fail{ZPIC_E_LASER, "laser: fwhm and W0 must be > 0"};
      if (L.start <= 0.0 || L.start - 2.0 * L.fwhm >= grid->nx * grid->dx)
        throw Fail{ZPIC_E_LASER, "laser: the pulse [start - 2 fwhm, start] misses the box"};
      launch_laser(c->E[0], c->B[0], g, c->y0, grid->dx, grid->dy, L, c->stream);
      CUDA_OR_THROW(cudaGetLastError());
      refresh_field_guards(c, c->E[0], true);
      refresh_field_guards(c, c->B[0], false);
    }
    if (c->slab) {
      // halo buffers: raw J rows from both neighbours; particle messages (a count header and
      // `pcap` records, all sent every step) sized to the traffic: only particles of the boundary
      // row can cross, and a quarter of that row at the nominal density is ~9x
      // the thermal crossing rate of C5 (u_th = 0.1: 2.8 % per step and direction) — 1 MB per
      // direction at C5 instead of a whole-row bound; more crossers than that stop the run with
      // ZPIC_E_OVERFLOW (ERR_HALO; zpic_options.halo_particles raises the capacity)
      int ppc_sum = 0;
      for (int s = 0; s < n_species; ++s) ppc_sum += species[s].ppc[0] * species[s].ppc[1];
      c->pcap = c->opt.halo_particles > 0 ? round_up(c->opt.halo_particles, 32)
                                          : std::max(4096, round_up(g.nx * std::max(ppc_sum, 1) / 4, 32));
      for (int d = 0; d < 2; ++d) c->pmsg_send[d] = alloc_n<char>(c, particle_msg_bytes(c->pcap));
      c->peer = c->transport == ZPIC_TRANSPORT_PEER || c->transport == ZPIC_TRANSPORT_LOOPBACK_PEER;
      if (c->peer) {   // the receive areas in one cudaMalloc'd block (exportable with CUDA IPC)
        const size_t pb = peer_block_bytes(g.pitch, c->pcap);
        CUDA_OR_THROW(cudaMalloc(&c->peer_block, pb));
        CUDA_OR_THROW(cudaMemsetAsync(c->peer_block, 0, pb, c->stream));
        c->peer_self = peer_view(c->peer_block, g.pitch, c->pcap);
        for (int b = 0; b < 2; ++b) { c->peer_self.E[b] = c->E[b]; c->peer_self.B[b] = c->B[b]; }
        c->peer_self.plane = g.plane;
        c->peer_self.ny = g.ny;
        c->peer_lo = c->peer_hi = c->peer_self;   // a one-rank ring; loopback groups bind at zpic_step_group
        c->jrup = c->peer_self.jrup;
        c->jrdn = c->peer_self.jrdn;
        c->pmsg_recv[0] = c->peer_self.pmsg[0];
        c->pmsg_recv[1] = c->peer_self.pmsg[1];
      } else {
        c->jrup = alloc_n<float>(c, (size_t)3 * 2 * g.pitch);
        c->jrdn = alloc_n<float>(c, (size_t)3 * 2 * g.pitch);
        for (int d = 0; d < 2; ++d) c->pmsg_recv[d] = alloc_n<char>(c, particle_msg_bytes(c->pcap));
      }
      if (c->transport == ZPIC_TRANSPORT_NCCL || (c->transport == ZPIC_TRANSPORT_PEER && c->world > 1)) {
        if (c->dist.nccl_comm) {
          c->comm = c->dist.nccl_comm;
          c->own_comm = false;
        } else {
          ncclUniqueId id;
          std::memcpy(&id, c->dist.nccl_id, sizeof(id));
          ncclComm_t comm;
          ncclResult_t r = ncclCommInitRank(&comm, c->world, id, c->rank);
          if (r != ncclSuccess) throw Fail{ZPIC_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)};
          c->comm = comm;
          c->own_comm = true;
        }
        if (c->transport == ZPIC_TRANSPORT_NCCL) {
          CUDA_OR_THROW(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
          for (auto& e : c->ev) CUDA_OR_THROW(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        } else {
          open_peer_blocks(c);   // PEER across processes: every rank's block by CUDA IPC
        }
      }
    }
    CUDA_OR_THROW(cudaGetLastError());
    CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  } catch (const Fail& f) {
    g_init_error = f.msg;
    zpic_free(c);
    return f.st;
  }
  *out = c;
  return ZPIC_OK;
}

static void drop_graphs(zpic_ctx* c);

// Bin n particles held on the device (SoA block `tmp`: ix, iy (global), x, y, ux, uy, uz, id, n
// entries each) into species s's tile store, sized anew for the largest tile; frees `tmp`.
static void load_species(zpic_ctx* c, int s, int64_t n, char* tmp, bool has_id) {
  c->occ_stale = true;   // the occupancy bound of the fixed-point current is recomputed before the next step
  int32_t* dix = (int32_t*)tmp;
  int32_t* diy = dix + n;
  float* dx_ = (float*)(diy + n);
  float* dy_ = dx_ + n;
  float* dux = dy_ + n;
  float* duy = dux + n;
  float* duz = duy + n;
  uint32_t* did = (uint32_t*)(duz + n);
  int* dcounts = alloc_n<int>(c, c->ntiles + 1);
  if (n > 0) {
    launch_count(c->T, c->ntx, c->g.nx, c->g.ny, c->y0, (long)n, dix, diy, dx_, dy_, dcounts, dcounts + c->ntiles,
                 c->stream);
    CUDA_OR_THROW(cudaGetLastError());
  }
  std::vector<int> counts(c->ntiles + 1, 0);
  CUDA_OR_THROW(cudaMemcpyAsync(counts.data(), dcounts, (c->ntiles + 1) * 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  dev_free(c, dcounts);
  if (counts[c->ntiles]) {
    dev_free(c, tmp);
    throw Fail{ZPIC_E_INVALID, "set_particles: a particle is outside the local slab or its offset is not in [0,1)"};
  }
  int maxc = 0;
  for (int t = 0; t < c->ntiles; ++t) maxc = std::max(maxc, counts[t]);
  const int ppc = c->species[s].ppc[0] * c->species[s].ppc[1];
  const double slack = c->repacking ? std::max(1.1, c->opt.capacity_slack) : c->opt.capacity_slack;
  const int cap = std::max({32, round_up((int)std::ceil(maxc * slack), 32),
                            round_up((int)std::ceil(c->T * c->T * ppc * slack), 32)});
  if (cap > c->ps[s].cap || cap < c->ps[s].cap / 2 || c->repacking) {   // else keep the store
    free_store(c, s);
    alloc_store(c, s, cap);
    check_tile_capacity(c);
  } else {
    CUDA_OR_THROW(cudaMemsetAsync(c->ps[s].cnt, 0, (size_t)c->ntiles * 4, c->stream));
  }
  if (n > 0) {
    launch_bin(c->ps[s], c->T, c->ntx, c->y0, (long)n, dix, diy, dx_, dy_, dux, duy, duz, has_id ? did : nullptr, c->err,
               c->spill[c->steps & 1], s, c->stream);
    CUDA_OR_THROW(cudaGetLastError());
  }
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  dev_free(c, tmp);
}

// Movers / loose lists sized for the current population (the live loose list keeps its
// contents when it grows); `extra` particles about to be loaded are counted in.
static void size_lists(zpic_ctx* c, int64_t extra) {
  int64_t total = extra;
  for (int q = 0; q < c->nspecies; ++q) {
    std::vector<int> cnt(c->ntiles);
    CUDA_OR_THROW(cudaMemcpy(cnt.data(), c->ps[q].cnt, c->ntiles * 4, cudaMemcpyDeviceToHost));
    for (int v : cnt) total += v;
  }
  int nl = 0;
  PList& live = c->spill[c->steps & 1];
  CUDA_OR_THROW(cudaMemcpy(&nl, live.count, 4, cudaMemcpyDeviceToHost));
  nl = std::min(nl, live.cap);
  c->population = total + nl;
  const int need = mover_capacity(c, c->population);
  if (need > c->movers.cap) {
    for (PList* L : {&c->movers, &c->spill[0], &c->spill[1]}) {
      PList N = alloc_list(c, need);
      if (L == &live && nl > 0) {
        const size_t b = (size_t)nl * 4;
        CUDA_OR_THROW(cudaMemcpyAsync(N.cell, L->cell, b, cudaMemcpyDeviceToDevice, c->stream));
        CUDA_OR_THROW(cudaMemcpyAsync(N.x, L->x, b, cudaMemcpyDeviceToDevice, c->stream));
        CUDA_OR_THROW(cudaMemcpyAsync(N.y, L->y, b, cudaMemcpyDeviceToDevice, c->stream));
        CUDA_OR_THROW(cudaMemcpyAsync(N.ux, L->ux, b, cudaMemcpyDeviceToDevice, c->stream));
        CUDA_OR_THROW(cudaMemcpyAsync(N.uy, L->uy, b, cudaMemcpyDeviceToDevice, c->stream));
        CUDA_OR_THROW(cudaMemcpyAsync(N.uz, L->uz, b, cudaMemcpyDeviceToDevice, c->stream));
        if (N.id && L->id) CUDA_OR_THROW(cudaMemcpyAsync(N.id, L->id, b, cudaMemcpyDeviceToDevice, c->stream));
        CUDA_OR_THROW(cudaMemcpyAsync(N.species, L->species, b, cudaMemcpyDeviceToDevice, c->stream));
        CUDA_OR_THROW(cudaMemcpyAsync(N.count, &nl, 4, cudaMemcpyHostToDevice, c->stream));
        CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
      }
      dev_free(c, L->cell); dev_free(c, L->x); dev_free(c, L->y); dev_free(c, L->ux); dev_free(c, L->uy);
      dev_free(c, L->uz); dev_free(c, L->id); dev_free(c, L->species); dev_free(c, L->count);
      *L = N;
    }
  }
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
}

// Re-pack (SURVEY.md §8(d) "slack plus an overflow -> global re-pack path"): when the loose list
// (particles that found no slack in their tile) grows, every species is exported from its tiles
// and the loose list to a flat device buffer and binned again into tiles sized for the current
// largest tile.  Host-driven and rare: zpic_step checks the loose count every kRepackCheck steps.
constexpr int kRepackCheck = 16;
static void repack(zpic_ctx* c) {
  c->repacking = true;
  const PList L = c->spill[c->steps & 1];   // the loose particles of the next step
  int nl = 0;
  CUDA_OR_THROW(cudaMemcpy(&nl, L.count, 4, cudaMemcpyDeviceToHost));
  nl = std::min(nl, L.cap);
  // 1. every species out to a flat device block (tiles, then its loose particles)
  std::vector<char*> tmps(c->nspecies, nullptr);
  std::vector<int64_t> ms(c->nspecies, 0);
  for (int s = 0; s < c->nspecies; ++s) {
    std::vector<int> cnt(c->ntiles);
    CUDA_OR_THROW(cudaMemcpy(cnt.data(), c->ps[s].cnt, c->ntiles * 4, cudaMemcpyDeviceToHost));
    std::vector<int64_t> prefix(c->ntiles + 1, 0);
    for (int t = 0; t < c->ntiles; ++t) prefix[t + 1] = prefix[t] + std::min(cnt[t], c->ps[s].cap);
    const int64_t nt = prefix[c->ntiles], n = nt + nl;   // upper bound (the loose list mixes species)
    char* tmp = (char*)dev_alloc(c, (size_t)std::max<int64_t>(n, 1) * 32);
    int32_t* dix = (int32_t*)tmp;
    int32_t* diy = dix + n;
    float* dxx = (float*)(diy + n);
    float* dyy = dxx + n;
    float* dux = dyy + n;
    float* duy = dux + n;
    float* duz = duy + n;
    uint32_t* did = (uint32_t*)(duz + n);
    const bool ids = c->ps[s].nf > F_ID;
    int64_t* dprefix = (int64_t*)dev_alloc(c, (c->ntiles + 1) * 8);
    int* dn = alloc_n<int>(c, 1);
    CUDA_OR_THROW(cudaMemcpyAsync(dprefix, prefix.data(), (c->ntiles + 1) * 8, cudaMemcpyHostToDevice, c->stream));
    launch_export(c->ps[s], c->ntiles, dprefix, c->y0, dix, diy, dxx, dyy, dux, duy, duz, ids ? did : nullptr, c->stream);
    launch_loose_extract(L, s, c->y0, nt, dix, diy, dxx, dyy, dux, duy, duz, ids ? did : nullptr, dn, c->stream);
    CUDA_OR_THROW(cudaGetLastError());
    int ns = 0;
    CUDA_OR_THROW(cudaMemcpyAsync(&ns, dn, 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
    dev_free(c, dprefix);
    dev_free(c, dn);
    // compact the SoA block to m = nt + ns entries per field (load_species expects that layout)
    const int64_t m = nt + ns;
    if (m < n) {
      char* t2 = (char*)dev_alloc(c, (size_t)std::max<int64_t>(m, 1) * 32);
      for (int f = 0; f < 8; ++f)
        CUDA_OR_THROW(cudaMemcpyAsync(t2 + (size_t)f * m * 4, tmp + (size_t)f * n * 4, (size_t)m * 4,
                                      cudaMemcpyDeviceToDevice, c->stream));
      CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
      dev_free(c, tmp);
      tmp = t2;
    }
    tmps[s] = tmp;
    ms[s] = m;
  }
  // 2. empty loose list; every species back into tiles sized for its largest tile (+10 %)
  CUDA_OR_THROW(cudaMemsetAsync(L.count, 0, 4, c->stream));
  for (int s = 0; s < c->nspecies; ++s) load_species(c, s, ms[s], tmps[s], c->ps[s].nf > F_ID);
  c->repacking = false;
  size_lists(c);
  drop_graphs(c);
  c->repacks += 1;
}

// Called between steps: re-pack when the loose list holds more than a quarter of its capacity
// (or 4096 particles, whichever is larger).
static void maybe_repack_now(zpic_ctx* c) {
  int nl = 0;
  CUDA_OR_THROW(cudaMemcpyAsync(&nl, c->spill[c->steps & 1].count, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  if (nl > std::max<int64_t>(4096, std::min<int64_t>(c->spill[0].cap / 4, c->population / 64))) repack(c);
}
static void maybe_repack(zpic_ctx* c) {
  if (c->since_check < kRepackCheck) return;
  c->since_check = 0;
  int nl = 0;
  CUDA_OR_THROW(cudaMemcpyAsync(&nl, c->spill[c->steps & 1].count, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  if (nl > std::max<int64_t>(4096, std::min<int64_t>(c->spill[0].cap / 4, c->population / 64))) repack(c);
}

static void maybe_repack_now(zpic_ctx* c);

// K2s every sort_every steps (ZPIC_SORT_EVERY; 0 = never): each species' tiles re-sorted in
// place (the store pointer does not change: the captured graphs stay valid).
static void maybe_sort(zpic_ctx* c) {
  if (c->occ_stale) {   // particles (re)loaded: the fixed-point current's occupancy bound, from scratch
    launch_occupancy(push_params(c), c->stream);
    CUDA_OR_THROW(cudaGetLastError());
    c->launches += 1;
    c->occ_stale = false;
  }
  if (c->sort_every <= 0 || c->steps - c->last_sort < c->sort_every) return;
  c->last_sort = c->steps;
  for (int s = 0; s < c->nspecies; ++s) {
    if (!c->ps[s].data) continue;
    ProfScope pr(c, K_SORT);
    launch_sort_tiles(c->ps[s], c->T, c->ntx, c->ntiles, c->stats, c->stream);
    CUDA_OR_THROW(cudaGetLastError());
    c->launches += 1;
  }
  c->sorts += 1;
}

// Chunked direct load: when the species' tile store already has room for n particles on average
// (it was sized for the species' lattice at zpic_init), the host arrays are copied in chunks into
// two device staging buffers on a copy stream while the compute stream bins the previous chunk
// (validation inside the binning; a full tile sends the rest to the loose list, re-packed after if
// it grew).  No full-size device copy of the input, and the upload overlaps the binning.
constexpr int64_t kLoadChunk = 1 << 23;
static bool load_chunked(zpic_ctx* c, int s, int64_t n, const int32_t* ix, const int32_t* iy, const float* x,
                         const float* y, const float* ux, const float* uy, const float* uz, const uint32_t* id) {
  PStore& ps = c->ps[s];
  if (!ps.data || n <= kLoadChunk || (double)n > 0.9 * (double)ps.cap * c->ntiles) return false;
  c->occ_stale = true;
  CUDA_OR_THROW(cudaMemsetAsync(ps.cnt, 0, (size_t)c->ntiles * 4, c->stream));
  size_lists(c, n);   // loose list room for what may not fit
  if (!c->copy_stream) CUDA_OR_THROW(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  cudaEvent_t copied[2], binned[2];
  for (int b = 0; b < 2; ++b) {
    CUDA_OR_THROW(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
    CUDA_OR_THROW(cudaEventCreateWithFlags(&binned[b], cudaEventDisableTiming));
  }
  TmpBuf stage_buf(c, (size_t)2 * kLoadChunk * 32), bad_buf(c, 4);
  char* stage = (char*)stage_buf.p;
  int* bad = (int*)bad_buf.p;
  CUDA_OR_THROW(cudaMemsetAsync(bad, 0, 4, c->stream));
  const int64_t nchunks = (n + kLoadChunk - 1) / kLoadChunk;
  for (int64_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k & 1);
    const int64_t o = k * kLoadChunk, m = std::min(kLoadChunk, n - o);
    char* buf = stage + (size_t)b * kLoadChunk * 32;
    int32_t* dix = (int32_t*)buf;
    int32_t* diy = dix + kLoadChunk;
    float* dx_ = (float*)(diy + kLoadChunk);
    float* dy_ = dx_ + kLoadChunk;
    float* dux = dy_ + kLoadChunk;
    float* duy = dux + kLoadChunk;
    float* duz = duy + kLoadChunk;
    uint32_t* did = (uint32_t*)(duz + kLoadChunk);
    if (k >= 2) CUDA_OR_THROW(cudaStreamWaitEvent(c->copy_stream, binned[b], 0));
    const size_t mb = (size_t)m * 4;
    CUDA_OR_THROW(cudaMemcpyAsync(dix, ix + o, mb, cudaMemcpyHostToDevice, c->copy_stream));
    CUDA_OR_THROW(cudaMemcpyAsync(diy, iy + o, mb, cudaMemcpyHostToDevice, c->copy_stream));
    CUDA_OR_THROW(cudaMemcpyAsync(dx_, x + o, mb, cudaMemcpyHostToDevice, c->copy_stream));
    CUDA_OR_THROW(cudaMemcpyAsync(dy_, y + o, mb, cudaMemcpyHostToDevice, c->copy_stream));
    CUDA_OR_THROW(cudaMemcpyAsync(dux, ux + o, mb, cudaMemcpyHostToDevice, c->copy_stream));
    CUDA_OR_THROW(cudaMemcpyAsync(duy, uy + o, mb, cudaMemcpyHostToDevice, c->copy_stream));
    CUDA_OR_THROW(cudaMemcpyAsync(duz, uz + o, mb, cudaMemcpyHostToDevice, c->copy_stream));
    if (id) CUDA_OR_THROW(cudaMemcpyAsync(did, id + o, mb, cudaMemcpyHostToDevice, c->copy_stream));
    CUDA_OR_THROW(cudaEventRecord(copied[b], c->copy_stream));
    CUDA_OR_THROW(cudaStreamWaitEvent(c->stream, copied[b], 0));
    launch_bin(ps, c->T, c->ntx, c->y0, (long)m, dix, diy, dx_, dy_, dux, duy, duz, id ? did : nullptr, c->err,
               c->spill[c->steps & 1], s, c->stream, c->g.nx, c->g.ny, bad, (long)o);
    CUDA_OR_THROW(cudaGetLastError());
    CUDA_OR_THROW(cudaEventRecord(binned[b], c->stream));
  }
  int nbad = 0;
  CUDA_OR_THROW(cudaMemcpyAsync(&nbad, bad, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  for (int b = 0; b < 2; ++b) { cudaEventDestroy(copied[b]); cudaEventDestroy(binned[b]); }
  if (nbad) {
    CUDA_OR_THROW(cudaMemsetAsync(ps.cnt, 0, (size_t)c->ntiles * 4, c->stream));
    throw Fail{ZPIC_E_INVALID, "set_particles: a particle is outside the local slab or its offset is not in [0,1)"};
  }
  maybe_repack_now(c);
  return true;
}

// Species s emptied: its tiles (counts 0) and its loose-list entries (the live loose list is
// compacted through the other, idle spill list).  zpic_set_particles starts from here and comes back
// here on any error, so a failed upload leaves the species empty (include/zpic.h).
static void clear_species(zpic_ctx* c, int s) {
  c->occ_stale = true;
  if (c->ps[s].data) CUDA_OR_THROW(cudaMemsetAsync(c->ps[s].cnt, 0, (size_t)c->ntiles * 4, c->stream));
  PList& live = c->spill[c->steps & 1];
  PList& idle = c->spill[(c->steps & 1) ^ 1];
  if (!live.count || !idle.count) return;
  int nl = 0;
  CUDA_OR_THROW(cudaMemcpyAsync(&nl, live.count, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  if (nl == 0) return;
  CUDA_OR_THROW(cudaMemsetAsync(idle.count, 0, 4, c->stream));
  launch_loose_drop_species(live, s, idle, c->stream);
  CUDA_OR_THROW(cudaGetLastError());
  int m = 0;
  CUDA_OR_THROW(cudaMemcpyAsync(&m, idle.count, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
  m = std::min(m, idle.cap);
  const size_t b = (size_t)m * 4;
  if (m > 0) {
    for (auto f : {std::make_pair((void*)live.cell, (void*)idle.cell), std::make_pair((void*)live.x, (void*)idle.x),
                   std::make_pair((void*)live.y, (void*)idle.y), std::make_pair((void*)live.ux, (void*)idle.ux),
                   std::make_pair((void*)live.uy, (void*)idle.uy), std::make_pair((void*)live.uz, (void*)idle.uz),
                   std::make_pair((void*)live.species, (void*)idle.species)})
      CUDA_OR_THROW(cudaMemcpyAsync(f.first, f.second, b, cudaMemcpyDeviceToDevice, c->stream));
    if (live.id && idle.id) CUDA_OR_THROW(cudaMemcpyAsync(live.id, idle.id, b, cudaMemcpyDeviceToDevice, c->stream));
  }
  CUDA_OR_THROW(cudaMemcpyAsync(live.count, &m, 4, cudaMemcpyHostToDevice, c->stream));
  CUDA_OR_THROW(cudaMemsetAsync(idle.count, 0, 4, c->stream));
  CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
}

zpic_status zpic_set_particles(zpic_ctx* c, int32_t s, int64_t n, const int32_t* ix, const int32_t* iy, const float* x,
                               const float* y, const float* ux, const float* uy, const float* uz, const uint32_t* id) {
  if (!c) return ZPIC_E_INVALID;
  if (s < 0 || s >= c->nspecies || n < 0 || (n > 0 && (!ix || !iy || !x || !y || !ux || !uy || !uz))) {
    c->last_error = "set_particles: bad arguments"; return ZPIC_E_INVALID;
  }
  drop_graphs(c);
  try {
    clear_species(c, s);   // the old particles of species s go (tiles and loose list)
    if (load_chunked(c, s, n, ix, iy, x, y, ux, uy, uz, id)) {
      size_lists(c);
      return check_sticky(c);
    }
    // upload, then validate + count per tile and bin on the device
    char* tmp = (char*)dev_alloc(c, (size_t)std::max<int64_t>(n, 1) * (7 * 4 + 4));
    int32_t* dix = (int32_t*)tmp;
    int32_t* diy = dix + n;
    float* dx_ = (float*)(diy + n);
    float* dy_ = dx_ + n;
    float* dux = dy_ + n;
    float* duy = dux + n;
    float* duz = duy + n;
    uint32_t* did = (uint32_t*)(duz + n);
    if (n > 0) {
      CUDA_OR_THROW(cudaMemcpyAsync(dix, ix, n * 4, cudaMemcpyHostToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(diy, iy, n * 4, cudaMemcpyHostToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(dx_, x, n * 4, cudaMemcpyHostToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(dy_, y, n * 4, cudaMemcpyHostToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(dux, ux, n * 4, cudaMemcpyHostToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(duy, uy, n * 4, cudaMemcpyHostToDevice, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(duz, uz, n * 4, cudaMemcpyHostToDevice, c->stream));
      if (id) CUDA_OR_THROW(cudaMemcpyAsync(did, id, n * 4, cudaMemcpyHostToDevice, c->stream));
    }
    load_species(c, s, n, tmp, id != nullptr);
    size_lists(c);
  } catch (const Fail& f) {
    c->last_error = f.msg;
    try { clear_species(c, s); } catch (const Fail&) {}   // a failed upload leaves the species empty
    return f.st;
  }
  return check_sticky(c);
}

zpic_status zpic_set_fields(zpic_ctx* c, int32_t which, const float* in, size_t in_len) {
  if (!c || !in || (which != 0 && which != 1)) return ZPIC_E_INVALID;
  const GridDesc& g = c->g;
  if (in_len < (size_t)3 * g.nx * g.ny) { c->last_error = "set_fields: buffer too small"; return ZPIC_E_BUFSIZE; }
  float* F = which == 0 ? c->E[c->cur] : c->B[c->cur];
  for (int k = 0; k < 3; ++k) {
    cudaError_t e = cudaMemcpy2DAsync(F + k * g.plane + g.at(0, 0), g.pitch * 4, in + (size_t)k * g.nx * g.ny, g.nx * 4,
                                      g.nx * 4, g.ny, cudaMemcpyHostToDevice, c->stream);
    if (e != cudaSuccess) { c->last_error = cudaGetErrorString(e); return ZPIC_E_CUDA; }
  }
  refresh_field_guards(c, F, which == 0);
  return check_sticky(c);
}

// ---- the step, in phases --------------------------------------------------
// phase A: particles (K1, K3, K4, K1L) and the x ghost-current fold (+ the y fold on one slab)
// [exchange round 1: raw J rows + migrating particles]
// phase B: slab J halo + received particles, filter, Yee
// [exchange round 2: E, B ghost rows]
// phase C: window injection, energies, bookkeeping
struct StepState {
  PushParams p;
  int shift;
  int launches;
  bool r1_async;   // exchange round 1 runs on the comm stream while interior Yee tiles run
};

// Overlap of the NCCL halo rounds with interior work (SURVEY.md §8(e) "Overlap"): round 2 (E/B
// ghost rows) with the next step's K1 on tile rows 1 .. nty-2 (they read no ghost row); round 1
// (raw J rows + particles) with the Yee tile rows whose J rows avoid 0, 1, ny-1, ny (the rows
// the halo changes).  Round 1 stays in order when a filter needs every J row first.
bool overlap_round1(const zpic_ctx* c) {
  return c->slab && c->transport == ZPIC_TRANSPORT_NCCL && c->comm_stream && c->opt.filter_passes == 0;
}

// PEER transports (zpic_peer.cu): round 1 = raw J rows + particle messages into the neighbours'
// receive areas, round 2 = E/B rows of buffer b into their guard-row areas; epochs count the rounds
// (every rank of a chain steps in lockstep, so the epochs agree).
void peer_round1_send(zpic_ctx* c) {
  c->peer_e1 += 1;
  // the particles are already in the neighbours' areas (K3 / K1L wrote them there); the raw J rows
  // too with the cross-slab commutative current (K1 / K1L added them): then only the signal
  if (!c->peer_j)
    launch_peer_put1(c->J, c->g, c->peer_lo, c->peer_hi, c->has_lo, c->has_hi, c->stream);
  launch_peer_signal(c->has_hi ? c->peer_hi.flags + 0 : nullptr, c->has_lo ? c->peer_lo.flags + 1 : nullptr, c->peer_e1,
                     c->stream);
}
void peer_round1_wait(zpic_ctx* c) {
  launch_peer_wait(c->peer_self.flags, c->has_lo ? 0 : -1, c->has_hi ? 1 : -1, c->peer_e1, c->err, c->stream);
}
// PEER: the per-step round 2 is written by K5's slab-edge tiles (ZPIC_PEER_PUT2=1: by the separate
// put kernel, for A/B); only the signal follows K5.
static bool peer_fused_r2() {
  static const bool put = [] { const char* e = getenv("ZPIC_PEER_PUT2"); return e && atoi(e); }();
  return !put;
}
void peer_round2_signal(zpic_ctx* c) {
  c->peer_e2 += 1;
  launch_peer_signal(c->has_hi ? c->peer_hi.flags + 2 : nullptr, c->has_lo ? c->peer_lo.flags + 3 : nullptr, c->peer_e2,
                     c->stream);
}
void peer_round2_send(zpic_ctx* c, int b) {
  c->peer_e2 += 1;
  launch_peer_put2(c->E[b], c->B[b], c->g, c->peer_lo, c->peer_hi, c->has_lo, c->has_hi, b, c->stream);
  launch_peer_signal(c->has_hi ? c->peer_hi.flags + 2 : nullptr, c->has_lo ? c->peer_lo.flags + 3 : nullptr, c->peer_e2,
                     c->stream);
}
// Cross-slab commutative current: J zeroed, then "zeroed" signalled to both neighbours (whose K1
// adds into this J only after they waited for it, before their first K1 launch of the step).
void peer_zero_j(zpic_ctx* c) {
  CUDA_OR_THROW(cudaMemsetAsync(c->J, 0, (size_t)3 * c->g.plane * sizeof(float), c->stream));
  c->peer_e0 += 1;
  launch_peer_signal(c->has_hi ? c->peer_hi.flags + 4 : nullptr, c->has_lo ? c->peer_lo.flags + 5 : nullptr, c->peer_e0,
                     c->stream);
  c->j_zeroed = true;
}
void peer_zero_wait(zpic_ctx* c) {
  launch_peer_wait(c->peer_self.flags, c->has_lo ? 4 : -1, c->has_hi ? 5 : -1, c->peer_e0, c->err, c->stream);
  c->j_zeroed = false;
}
// (the rows are already in this slab's guard rows: waiting is all there is to receive)
void peer_round2_wait(zpic_ctx* c) {
  launch_peer_wait(c->peer_self.flags, c->has_lo ? 2 : -1, c->has_hi ? 3 : -1, c->peer_e2, c->err, c->stream);
}

StepState step_phase_a(zpic_ctx* c) {
  StepState s{};
  s.p = push_params(c);
  // moving window: the host knows in advance that the window shifts at the end of
  // this step, when (n+1) dt > dx (n_move + 1) — the oracle's test, in the same fp64 arithmetic
  s.shift = (c->bcx == ZPIC_BC_MOVING_WINDOW && (double)(c->steps + 1) * c->dt > c->dx * (double)(c->n_move + 1)) ? 1 : 0;
  s.p.shift = s.shift;
  const int grid_small = 148 * 4;
  const PushParams& p = s.p;
  if (p.commutative) {   // the tiles add into J: start from zero (guards included)
    ProfScope ps(c, K_ASSEMBLE);
    if (c->peer_j) {   // and the neighbours add into it too: zeroed on both sides before any K1
      if (!c->j_zeroed) peer_zero_j(c);
      peer_zero_wait(c);
      s.launches += 2;
    } else {
      CUDA_OR_THROW(cudaMemsetAsync(c->J, 0, (size_t)3 * c->g.plane * sizeof(float), c->stream));
    }
  }
  {
    ProfScope ps(c, K_SCALE);
    if (c->check_occ) { launch_occupancy(p, c->stream, 1); ++s.launches; }   // verify hist / occ (tests)
    launch_tile_scale(p, c->stream);   // K1s: the tiles' current scales from the occupancy bounds
    ++s.launches;
  }
  {
    ProfScope ps(c, K_PUSH);
    if (c->r2_pending && c->peer) {   // one grid: interior tile rows first, the slab-edge CTAs wait
      PushParams q = p;                 // for the neighbours' rows themselves (NEXT-1 per tile row)
      q.boundary_last = 1;
      q.r2_flags = c->peer_self.flags;
      q.r2_epoch = c->peer_e2;
      launch_push_tiles(q, 0, c->ntiles, c->stream);
      c->r2_pending = false;
      ++s.launches;
    } else if (c->r2_pending) {   // NCCL: the E/B ghost rows of this step are still in flight
      const int tb = c->ntx, te = std::max(c->ntx, (c->nty - 1) * c->ntx);
      launch_push_tiles(p, tb, te, c->stream);
      CUDA_OR_THROW(cudaStreamWaitEvent(c->stream, c->ev[3], 0));   // round 2 landed (comm stream)
      c->r2_pending = false;
      PushParams q = p;   // both slab-edge tile rows in one grid (one wave tail instead of two)
      q.boundary_last = 2;
      launch_push_tiles(q, 0, c->nty >= 2 ? 2 * c->ntx : c->ntx, c->stream);
      s.launches += 2;
    } else {
      launch_push_tiles(p, 0, c->ntiles, c->stream);
      ++s.launches;
    }
  }
  if (p.use_mail) { ProfScope ps(c, K_MAIL); launch_mail_gather(p, c->stream); ++s.launches; }
  { ProfScope ps(c, K_INSERT); launch_insert(p, grid_small, c->stream); ++s.launches; }
  if (!p.commutative) {
    ProfScope ps(c, K_ASSEMBLE);
    launch_assemble(c->J, c->Jt, c->g, c->T, c->ntx, c->nty, c->stream);
    ++s.launches;
  }
  { ProfScope ps(c, K_LOOSE); launch_loose(p, grid_small, c->stream); ++s.launches; }
  if (!c->peer_j) {   // (cross-slab commutative current: after the neighbours' adds, phase b)
    ProfScope ps(c, K_FOLD);
    launch_guard_x(c->J, c->g, c->bcx == ZPIC_BC_PERIODIC ? 0 : 2, 0, c->stream);
    ++s.launches;
    if (!c->slab) {
      launch_guard_y(c->J, c->g, c->bcy == ZPIC_BC_PERIODIC ? 0 : 2, 0, c->stream);
      ++s.launches;
    }
  }
  return s;
}

void step_phase_b(zpic_ctx* c, StepState& s) {
  YeeParams y{};
  y.tmE = c->ytm[0][c->cur];
  y.tmB = c->ytm[1][c->cur];
  y.tmJ = c->ytmJ[0];
  y.g = c->g;
  y.E0 = c->E[c->cur]; y.B0 = c->B[c->cur]; y.J = c->J;
  y.E1 = c->E[c->cur ^ 1]; y.B1 = c->B[c->cur ^ 1];
  y.dt = (float)c->dt;
  y.dtdx = (float)(c->dt / c->dx); y.dtdy = (float)(c->dt / c->dy);
  y.hdx = (float)(0.5 * c->dt / c->dx); y.hdy = (float)(0.5 * c->dt / c->dy);
  y.murx = (float)((c->dt - c->dx) / (c->dt + c->dx));
  y.mury = (float)((c->dt - c->dy) / (c->dt + c->dy));
  y.bcx = c->bcx; y.bcy = c->bcy;
  y.shift = s.shift;
  y.y_images = !c->slab && c->bcy == ZPIC_BC_PERIODIC;
  y.ylo_edge = !c->slab || !c->has_lo;
  y.yhi_edge = !c->slab || !c->has_hi;
  y.fe_slots = c->fe_slots;
  y.fe_scale = 0.5 * c->dx * c->dy;
  if (c->slab && c->peer && peer_fused_r2()) {   // round 2 written by the slab-edge Yee tiles
    const int b = c->cur ^ 1;
    if (c->has_lo) {
      y.peer_lo_E = c->peer_lo.E[b]; y.peer_lo_B = c->peer_lo.B[b];
      y.peer_lo_plane = c->peer_lo.plane; y.peer_lo_ny = c->peer_lo.ny;
    }
    if (c->has_hi) {
      y.peer_hi_E = c->peer_hi.E[b]; y.peer_hi_B = c->peer_hi.B[b];
      y.peer_hi_plane = c->peer_hi.plane;
    }
  }
  int yee_done_to = 0;   // tile rows [1, yee_done_to) already advanced (round 1 overlap)
  if (s.r1_async) {
    const int hi = (c->g.ny - 2) / kYeeTY;   // tile rows r < hi: J rows [TY r, TY r + TY] avoid ny - 1, ny
    if (hi > 1) {
      ProfScope ps(c, K_YEE);
      launch_yee(y, c->stream, 1, hi);
      ++s.launches;
      yee_done_to = hi;
    }
    if (!c->peer) CUDA_OR_THROW(cudaStreamWaitEvent(c->stream, c->ev[1], 0));
  }
  if (c->slab) {
    ProfScope ps(c, K_HALO);
    if (c->peer) peer_round1_wait(c);
    if (c->peer_j) {   // every add into this J is in: the x-guard fold now
      launch_guard_x(c->J, c->g, c->bcx == ZPIC_BC_PERIODIC ? 0 : 2, 0, c->stream);
      ++s.launches;
    }
    launch_apply_j_halo(c->J, c->g, c->peer_j ? nullptr : c->jrup, c->peer_j ? nullptr : c->jrdn, c->has_lo, c->has_hi,
                        c->stream);
    launch_recv_insert(s.p, particle_msg_list(c->pmsg_recv[0], c->pcap), particle_msg_list(c->pmsg_recv[1], c->pcap),
                       c->stream);
    s.launches += 2;
    if (c->peer)   // consumed: the senders append the next step's exits from zero (after round 2)
      for (int d = 0; d < 2; ++d) CUDA_OR_THROW(cudaMemsetAsync(c->pmsg_recv[d], 0, 4, c->stream));
  }
  const float* Jyee = c->J;
  if (c->opt.filter_passes > 0) {
    ProfScope ps(c, K_FILTER);
    GridDesc gf = c->g;
    if (c->slab) gf.ny += 1;   // also the guard row ny (the neighbour's final row 0), used by the Yee kernel
    launch_filter_x(c->J, c->Jf, gf, c->opt.filter_passes, c->opt.filter_compensated, c->bcx == ZPIC_BC_PERIODIC,
                    c->stream);
    ++s.launches;
    if (!c->slab) {
      launch_guard_y(c->Jf, c->g, c->bcy == ZPIC_BC_PERIODIC ? 1 : 2, 0, c->stream);
      ++s.launches;
    }
    Jyee = c->Jf;
  }
  {
    ProfScope ps(c, K_YEE);
    y.J = Jyee;
    y.tmJ = c->ytmJ[Jyee == c->Jf ? 1 : 0];
    if (yee_done_to > 1) {
      launch_yee(y, c->stream, 0, 1);
      launch_yee(y, c->stream, yee_done_to, -1);
      s.launches += 2;
    } else {
      launch_yee(y, c->stream);
      ++s.launches;
    }
  }
}

void step_phase_c(zpic_ctx* c, StepState& s) {
  if (s.shift) {
    ProfScope ps(c, K_WINDOW);
    for (int q = 0; q < c->nspecies; ++q) {
      const zpic_species& sp = c->species[q];
      if (!(sp.n > 0)) continue;
      const uint64_t key = host_mix64(host_mix64(c->seed) + (uint64_t)q);
      launch_inject_column(s.p, q, sp.ppc[0], sp.ppc[1], c->d_nmove, c->ny_global, c->y0, key, sp.ufl, sp.uth,
                           c->stream);
      ++s.launches;
    }
    c->n_move += 1;
  }
  {
    ProfScope ps(c, K_EPI);
    launch_epilogue(c->ke_slots, c->fe_slots, c->energy, c->nspecies, c->energy + 1 + kMaxSpecies, c->movers.count,
                    s.p.spill_in.count, s.p.spill_out.count, c->stats, c->d_nmove, s.shift, c->stream);
    ++s.launches;
    if (c->slab) {
      for (int d = 0; d < 2; ++d) CUDA_OR_THROW(cudaMemsetAsync(c->pmsg_send[d], 0, 4, c->stream));
    }
  }
  c->cur ^= 1;
  c->steps += 1;
  c->since_check += 1;
  c->launches += s.launches;
}

zpic_status step_error(zpic_ctx* c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { c->last_error = std::string("launch: ") + cudaGetErrorString(e); return ZPIC_E_CUDA; }
  return ZPIC_OK;
}

// ---- CUDA graphs ---------------------------------------------------------
// Without a slab decomposition or a moving window, the launches of a step depend on the host
// state only through the E/B buffer index and the loose-list parity, which both flip every step:
// a two-step graph replayed from the same parity repeats exactly.  A graph bakes in the buffer
// pointers, so anything that reallocates (zpic_set_particles) drops the graphs.
static bool graphs_eligible(const zpic_ctx* c) { return !c->opt.no_graphs && !c->prof && !c->slab; }
static void drop_graphs(zpic_ctx* c) {
  for (auto& g : c->graph)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  for (auto& row : c->graph1)
    for (auto& g : row)
      if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}
// With a moving window the launches of a step also depend on whether the window shifts at its
// end (a host decision, step_phase_a): one-step graphs keyed by (step parity, shift).  The column
// injection reads n_move from the device, so the graphs stay valid as the window advances.
static bool window_shifts(const zpic_ctx* c) {
  return c->bcx == ZPIC_BC_MOVING_WINDOW && (double)(c->steps + 1) * c->dt > c->dx * (double)(c->n_move + 1);
}
static void run_step(zpic_ctx* c) {
  StepState s = step_phase_a(c);
  step_phase_b(c, s);
  step_phase_c(c, s);
}
static cudaGraphExec_t one_step_graph(zpic_ctx* c, int shift) {
  const int par = (int)(c->steps & 1);
  cudaGraphExec_t& ge = c->graph1[par][shift];
  if (ge) return ge;
  const int cur = c->cur, since = c->since_check;
  const int64_t steps = c->steps, launches = c->launches, n_move = c->n_move;
  cudaGraph_t g = nullptr;
  CUDA_OR_THROW(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    run_step(c);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CUDA_OR_THROW(cudaStreamEndCapture(c->stream, &g));
  c->graph1_launches[par][shift] = (int)(c->launches - launches);
  c->cur = cur; c->steps = steps; c->launches = launches; c->n_move = n_move; c->since_check = since;
  const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) { ge = nullptr; throw Fail{ZPIC_E_CUDA, std::string("graph: ") + cudaGetErrorString(e)}; }
  return ge;
}

static cudaGraphExec_t two_step_graph(zpic_ctx* c) {
  cudaGraphExec_t& ge = c->graph[c->steps & 1];
  if (ge) return ge;
  const int cur = c->cur;
  const int64_t steps = c->steps, launches = c->launches;
  cudaGraph_t g = nullptr;
  CUDA_OR_THROW(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    run_step(c);
    run_step(c);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CUDA_OR_THROW(cudaStreamEndCapture(c->stream, &g));
  c->graph_launches = (int)(c->launches - launches);
  c->cur = cur; c->steps = steps; c->launches = launches;   // capture only recorded the work
  const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) { ge = nullptr; throw Fail{ZPIC_E_CUDA, std::string("graph: ") + cudaGetErrorString(e)}; }
  return ge;
}

// One step of a context on the NCCL transport (or the unsplit domain): the halo rounds run on the
// comm stream, overlapped with interior work; round 2 stays pending into the
// next step's K1 (r2_pending) until slab_join.
static void run_step_nccl(zpic_ctx* c) {
  StepState s = step_phase_a(c);
  if (c->slab && c->peer) {   // round 1 by the peer-put kernels; interior Yee rows before the wait
    peer_round1_send(c);
    // interior Yee rows before the wait need a folded J: not with the cross-slab commutative
    // current, whose x-guard fold waits for the neighbours' adds
    s.r1_async = c->opt.filter_passes == 0 && !c->peer_j;
  } else if (c->slab) {
    ncclResult_t r;
    if (overlap_round1(c)) {   // round 1 on the comm stream, interior Yee rows meanwhile
      CUDA_OR_THROW(cudaEventRecord(c->ev[0], c->stream));
      CUDA_OR_THROW(cudaStreamWaitEvent(c->comm_stream, c->ev[0], 0));
      r = nccl_exchange_round1(c, c->comm_stream);
      CUDA_OR_THROW(cudaEventRecord(c->ev[1], c->comm_stream));
      s.r1_async = true;
    } else {
      ProfScope ps(c, K_EXCHANGE);
      r = nccl_exchange_round1(c, c->stream);
    }
    if (r != ncclSuccess) throw Fail{ZPIC_E_NCCL, std::string("NCCL round 1: ") + ncclGetErrorString(r)};
  }
  step_phase_b(c, s);
  if (c->slab && c->peer) {   // round 2 (K5 wrote the rows, or the put kernel); received in the next K1
    if (peer_fused_r2()) peer_round2_signal(c);
    else peer_round2_send(c, c->cur ^ 1);
    static const bool no_overlap = [] { const char* e = getenv("ZPIC_NO_R2_OVERLAP"); return e && atoi(e); }();
    if (no_overlap) peer_round2_wait(c);
    else c->r2_pending = true;
  } else if (c->slab) {
    ncclResult_t r;
    if (c->comm_stream) {   // round 2 on the comm stream, the next step's interior K1 meanwhile
      CUDA_OR_THROW(cudaEventRecord(c->ev[2], c->stream));
      CUDA_OR_THROW(cudaStreamWaitEvent(c->comm_stream, c->ev[2], 0));
      r = nccl_exchange_round2(c, c->cur ^ 1, c->comm_stream);
      CUDA_OR_THROW(cudaEventRecord(c->ev[3], c->comm_stream));
      c->r2_pending = true;
    } else {
      ProfScope ps(c, K_EXCHANGE);
      r = nccl_exchange_round2(c, c->cur ^ 1, c->stream);
    }
    if (r != ncclSuccess) throw Fail{ZPIC_E_NCCL, std::string("NCCL round 2: ") + ncclGetErrorString(r)};
  }
  step_phase_c(c, s);
}
static void slab_join(zpic_ctx* c) {
  if (c->r2_pending) {
    if (c->peer) peer_round2_wait(c);
    else CUDA_OR_THROW(cudaStreamWaitEvent(c->stream, c->ev[3], 0));
    c->r2_pending = false;
  }
}
// NEXT-1 on the y-slab path: two NCCL steps captured as one CUDA graph (NCCL send / recv are
// capturable; the comm stream forks from and joins the compute stream through the captured event
// edges, so inside the graph round 2 of the first step still overlaps the second step's interior
// K1, and the two halo rounds overlap interior kernels as in plain launches).  The graph starts and
// ends joined (no pending round), so the host state after a replay is that of two plain steps.
static bool graphs_eligible_slab(const zpic_ctx* c) {
  return !c->opt.no_graphs && !c->prof && c->slab && c->transport == ZPIC_TRANSPORT_NCCL &&
         c->bcx != ZPIC_BC_MOVING_WINDOW && !c->r2_pending;
}
static cudaGraphExec_t slab_two_step_graph(zpic_ctx* c) {
  cudaGraphExec_t& ge = c->graph[c->steps & 1];
  if (ge) return ge;
  const int cur = c->cur, since = c->since_check;
  const int64_t steps = c->steps, launches = c->launches;
  cudaGraph_t g = nullptr;
  CUDA_OR_THROW(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    run_step_nccl(c);
    run_step_nccl(c);
    slab_join(c);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    c->r2_pending = false;
    throw;
  }
  CUDA_OR_THROW(cudaStreamEndCapture(c->stream, &g));
  c->graph_launches = (int)(c->launches - launches);
  c->cur = cur; c->steps = steps; c->launches = launches; c->since_check = since;   // capture only recorded the work
  const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) { ge = nullptr; throw Fail{ZPIC_E_CUDA, std::string("graph: ") + cudaGetErrorString(e)}; }
  return ge;
}

zpic_status zpic_step(zpic_ctx* c, int32_t n) {
  if (!c || n < 0) return ZPIC_E_INVALID;
  if (graphs_eligible(c) && n >= 2 && c->bcx == ZPIC_BC_MOVING_WINDOW) {
    try {
      for (int k = 0; k < n; ++k) {
        maybe_repack(c);
        maybe_sort(c);
        const int shift = window_shifts(c) ? 1 : 0;
        const int par = c->steps & 1;
        CUDA_OR_THROW(cudaGraphLaunch(one_step_graph(c, shift), c->stream));
        c->cur ^= 1;
        c->steps += 1;
        c->since_check += 1;
        c->launches += c->graph1_launches[par][shift];
        if (shift) c->n_move += 1;
      }
    } catch (const Fail& f) {
      c->last_error = f.msg;
      return f.st;
    }
    return step_error(c);
  }
  if (graphs_eligible(c) && n >= 2) {
    try {
      int k = 0;
      for (; k + 2 <= n; k += 2) {
        maybe_repack(c);
        maybe_sort(c);
        CUDA_OR_THROW(cudaGraphLaunch(two_step_graph(c), c->stream));
        c->steps += 2;
        c->since_check += 2;
        c->launches += c->graph_launches;
      }
      if (k < n) { maybe_repack(c); maybe_sort(c); run_step(c); }
    } catch (const Fail& f) {
      c->last_error = f.msg;
      return f.st;
    }
    return step_error(c);
  }
  if (c->slab && (c->transport == ZPIC_TRANSPORT_LOOPBACK || c->transport == ZPIC_TRANSPORT_LOOPBACK_PEER)) {
    c->last_error = "loopback slabs are stepped with zpic_step_group";
    return ZPIC_E_STATE;
  }
  try {
    if (c->slab && c->halo_dirty) {
      if (c->peer) {
        peer_round2_send(c, c->cur);
        peer_round2_wait(c);
      } else {
        ncclResult_t r = nccl_exchange_round2(c, c->cur, c->stream);
        if (r != ncclSuccess) throw Fail{ZPIC_E_NCCL, std::string("NCCL halo: ") + ncclGetErrorString(r)};
      }
      c->halo_dirty = false;
    }
    int k = 0;
    if (c->slab && graphs_eligible_slab(c)) {   // two steps per replayed graph (NEXT-1)
      for (; k + 2 <= n; k += 2) {
        maybe_repack(c);
        maybe_sort(c);
        CUDA_OR_THROW(cudaGraphLaunch(slab_two_step_graph(c), c->stream));
        c->steps += 2;
        c->since_check += 2;
        c->launches += c->graph_launches;
      }
    }
    for (; k < n; ++k) {
      maybe_repack(c);
      maybe_sort(c);
      run_step_nccl(c);
    }
    slab_join(c);   // the caller's stream sees complete ghost rows after zpic_step
  } catch (const Fail& f) {
    c->last_error = f.msg;
    return f.st;
  }
  return step_error(c);
}

zpic_status zpic_step_group(zpic_ctx** cs, int32_t count, int32_t n) {
  if (!cs || count < 1 || n < 0) return ZPIC_E_INVALID;
  for (int r = 0; r < count; ++r) {
    zpic_ctx* c = cs[r];
    if (!c || !c->slab || c->transport != cs[0]->transport ||
        (c->transport != ZPIC_TRANSPORT_LOOPBACK && c->transport != ZPIC_TRANSPORT_LOOPBACK_PEER) ||
        c->world != count || c->rank != r || c->stream != cs[0]->stream) {
      if (c) c->last_error = "zpic_step_group: not one complete loopback group on one stream (ranks in order)";
      return ZPIC_E_STATE;
    }
  }
  const bool peer = cs[0]->transport == ZPIC_TRANSPORT_LOOPBACK_PEER;
  try {
    if (peer)   // the group's views of each other's receive areas (one address space)
      for (int r = 0; r < count; ++r) {
        zpic_ctx* lo = cs[cs[r]->lower];
        zpic_ctx* hi = cs[cs[r]->upper];
        cs[r]->peer_lo = lo->peer_self;
        cs[r]->peer_hi = hi->peer_self;
        if (cs[r]->peer_j) {
          cs[r]->jlo = lo->J; cs[r]->lo_plane = lo->g.plane; cs[r]->lo_ny = lo->g.ny;
          cs[r]->jhi = hi->J; cs[r]->hi_plane = hi->g.plane;
        }
      }
    if (cs[0]->halo_dirty) {
      if (peer) {   // every signal is enqueued before the wait that reads it
        for (int r = 0; r < count; ++r) peer_round2_send(cs[r], cs[r]->cur);
        for (int r = 0; r < count; ++r) peer_round2_wait(cs[r]);
      } else {
        loop_exchange_round2(cs, count, cs[0]->cur);
      }
      for (int r = 0; r < count; ++r) cs[r]->halo_dirty = false;
    }
    for (int k = 0; k < n; ++k) {
      for (int r = 0; r < count; ++r) maybe_sort(cs[r]);
      for (int r = 0; r < count; ++r)   // every "zeroed" signal before the first wait for one
        if (cs[r]->peer_j) peer_zero_j(cs[r]);
      std::vector<StepState> st(count);
      for (int r = 0; r < count; ++r) st[r] = step_phase_a(cs[r]);
      if (peer) for (int r = 0; r < count; ++r) peer_round1_send(cs[r]);
      else loop_exchange_round1(cs, count);
      for (int r = 0; r < count; ++r) step_phase_b(cs[r], st[r]);
      if (peer) {
        for (int r = 0; r < count; ++r) {
          if (peer_fused_r2()) peer_round2_signal(cs[r]);
          else peer_round2_send(cs[r], cs[r]->cur ^ 1);
        }
        for (int r = 0; r < count; ++r) peer_round2_wait(cs[r]);
      } else {
        loop_exchange_round2(cs, count, cs[0]->cur ^ 1);
      }
      for (int r = 0; r < count; ++r) step_phase_c(cs[r], st[r]);
    }
  } catch (const Fail& f) {
    cs[0]->last_error = f.msg;
    return f.st;
  }
  return step_error(cs[0]);
}

zpic_status zpic_nccl_unique_id(void* out, size_t out_len) {
  if (!out || out_len < sizeof(ncclUniqueId)) return ZPIC_E_BUFSIZE;
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) { g_init_error = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r); return ZPIC_E_NCCL; }
  std::memcpy(out, &id, sizeof(id));
  return ZPIC_OK;
}

zpic_status zpic_sync(zpic_ctx* c) {
  if (!c) return ZPIC_E_INVALID;
  return check_sticky(c);
}

zpic_status zpic_get_fields(zpic_ctx* c, int32_t which, float* out, size_t out_len) {
  if (!c || !out || which < 0 || which > 3) return ZPIC_E_INVALID;
  zpic_status st = check_sticky(c);
  if (st != ZPIC_OK) return st;
  const GridDesc& g = c->g;
  if (out_len < (size_t)3 * g.nx * g.ny) { c->last_error = "get_fields: buffer too small"; return ZPIC_E_BUFSIZE; }
  const float* F = which == 0 ? c->E[c->cur] : which == 1 ? c->B[c->cur] : (which == 2 && c->Jf) ? c->Jf : c->J;
  for (int k = 0; k < 3; ++k) {
    cudaError_t e = cudaMemcpy2DAsync(out + (size_t)k * g.nx * g.ny, g.nx * 4, F + k * g.plane + g.at(0, 0), g.pitch * 4,
                                      g.nx * 4, g.ny, cudaMemcpyDeviceToHost, c->stream);
    if (e != cudaSuccess) { c->last_error = cudaGetErrorString(e); return ZPIC_E_CUDA; }
  }
  return check_sticky(c);
}

zpic_status zpic_get_particles(zpic_ctx* c, int32_t s, int64_t* count_inout, int32_t* ix, int32_t* iy, float* x,
                               float* y, float* ux, float* uy, float* uz, uint32_t* id) {
  if (!c || !count_inout || s < 0 || s >= c->nspecies) return ZPIC_E_INVALID;
  zpic_status st = check_sticky(c);
  if (st != ZPIC_OK) return st;
  if (id && !c->opt.track_ids) { c->last_error = "get_particles: ids requested without track_ids"; return ZPIC_E_STATE; }
  try {
    std::vector<int> cnt(c->ntiles);
    CUDA_OR_THROW(cudaMemcpy(cnt.data(), c->ps[s].cnt, c->ntiles * 4, cudaMemcpyDeviceToHost));
    std::vector<int64_t> prefix(c->ntiles + 1, 0);
    for (int t = 0; t < c->ntiles; ++t) prefix[t + 1] = prefix[t] + std::min(cnt[t], c->ps[s].cap);
    // loose particles of this species
    const PList& L = c->spill[c->steps & 1];
    int nl = 0;
    CUDA_OR_THROW(cudaMemcpy(&nl, L.count, 4, cudaMemcpyDeviceToHost));
    nl = std::min(nl, L.cap);
    std::vector<int32_t> lsp(nl), lcell(nl);
    std::vector<float> lf[5];
    std::vector<uint32_t> lid(nl);
    int nls = 0;
    if (nl > 0) {
      CUDA_OR_THROW(cudaMemcpy(lsp.data(), L.species, nl * 4, cudaMemcpyDeviceToHost));
      for (int k = 0; k < nl; ++k) nls += lsp[k] == s;
    }
    const int64_t total = prefix[c->ntiles] + nls;
    if (!ix) { *count_inout = total; return ZPIC_OK; }
    if (*count_inout < total) { c->last_error = "get_particles: buffer too small"; *count_inout = total; return ZPIC_E_BUFSIZE; }
    const int64_t nt = prefix[c->ntiles];
    if (nt > 0) {
      int64_t* dprefix = (int64_t*)dev_alloc(c, (c->ntiles + 1) * 8);
      char* tmp = (char*)dev_alloc(c, (size_t)nt * 32);
      int32_t* dix = (int32_t*)tmp;
      int32_t* diy = dix + nt;
      float* dxx = (float*)(diy + nt);
      float* dyy = dxx + nt;
      float* dux = dyy + nt;
      float* duy = dux + nt;
      float* duz = duy + nt;
      uint32_t* did = (uint32_t*)(duz + nt);
      CUDA_OR_THROW(cudaMemcpyAsync(dprefix, prefix.data(), (c->ntiles + 1) * 8, cudaMemcpyHostToDevice, c->stream));
      launch_export(c->ps[s], c->ntiles, dprefix, c->y0, dix, diy, dxx, dyy, dux, duy, duz, id ? did : nullptr, c->stream);
      CUDA_OR_THROW(cudaGetLastError());
      CUDA_OR_THROW(cudaMemcpyAsync(ix, dix, nt * 4, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(iy, diy, nt * 4, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(x, dxx, nt * 4, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(y, dyy, nt * 4, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(ux, dux, nt * 4, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(uy, duy, nt * 4, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OR_THROW(cudaMemcpyAsync(uz, duz, nt * 4, cudaMemcpyDeviceToHost, c->stream));
      if (id) CUDA_OR_THROW(cudaMemcpyAsync(id, did, nt * 4, cudaMemcpyDeviceToHost, c->stream));
      CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
      dev_free(c, tmp);
      dev_free(c, dprefix);
    }
    if (nls > 0) {
      for (auto& v : lf) v.resize(nl);
      CUDA_OR_THROW(cudaMemcpy(lcell.data(), L.cell, nl * 4, cudaMemcpyDeviceToHost));
      CUDA_OR_THROW(cudaMemcpy(lf[0].data(), L.x, nl * 4, cudaMemcpyDeviceToHost));
      CUDA_OR_THROW(cudaMemcpy(lf[1].data(), L.y, nl * 4, cudaMemcpyDeviceToHost));
      CUDA_OR_THROW(cudaMemcpy(lf[2].data(), L.ux, nl * 4, cudaMemcpyDeviceToHost));
      CUDA_OR_THROW(cudaMemcpy(lf[3].data(), L.uy, nl * 4, cudaMemcpyDeviceToHost));
      CUDA_OR_THROW(cudaMemcpy(lf[4].data(), L.uz, nl * 4, cudaMemcpyDeviceToHost));
      if (L.id) CUDA_OR_THROW(cudaMemcpy(lid.data(), L.id, nl * 4, cudaMemcpyDeviceToHost));
      int64_t o = nt;
      for (int k = 0; k < nl; ++k) {
        if (lsp[k] != s) continue;
        ix[o] = lcell[k] & 0xffff;
        iy[o] = (lcell[k] >> 16) + c->y0;
        x[o] = lf[0][k]; y[o] = lf[1][k]; ux[o] = lf[2][k]; uy[o] = lf[3][k]; uz[o] = lf[4][k];
        if (id) id[o] = lid[k];
        ++o;
      }
    }
    *count_inout = total;
  } catch (const Fail& f) {
    c->last_error = f.msg;
    return f.st;
  }
  return ZPIC_OK;
}

zpic_status zpic_energy(zpic_ctx* c, int64_t* iter, double* field, double* kinetic) {
  if (!c) return ZPIC_E_INVALID;
  zpic_status st = check_sticky(c);
  if (st != ZPIC_OK) return st;
  double e[1 + kMaxSpecies] = {0, 0, 0, 0, 0};
  if (c->slab && c->transport == ZPIC_TRANSPORT_NCCL) {
    // global sums over the slabs (collective over all ranks)
    double* red = nullptr;
    try { red = alloc_n<double>(c, 1 + kMaxSpecies); } catch (const Fail& f) { c->last_error = f.msg; return f.st; }
    ncclResult_t r = ncclAllReduce(c->energy, red, 1 + kMaxSpecies, ncclDouble, ncclSum, (ncclComm_t)c->comm, c->stream);
    if (r != ncclSuccess) { c->last_error = ncclGetErrorString(r); dev_free(c, red); return ZPIC_E_NCCL; }
    cudaMemcpyAsync(e, red, sizeof(e), cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    dev_free(c, red);
    if (c->steps == 0) for (double& v : e) v = 0.0;
  } else if (c->steps > 0) {
    cudaMemcpy(e, c->energy, sizeof(e), cudaMemcpyDeviceToHost);
  }
  if (iter) *iter = c->steps - 1;
  if (field) *field = e[0];
  if (kinetic)
    for (int s = 0; s < c->nspecies; ++s) kinetic[s] = e[1 + s];
  return ZPIC_OK;
}

zpic_status zpic_get_charge(zpic_ctx* c, float* out, size_t out_len) {
  if (!c || !out) return ZPIC_E_INVALID;
  zpic_status st = check_sticky(c);
  if (st != ZPIC_OK) return st;
  const GridDesc& g = c->g;
  if (out_len < (size_t)g.nx * g.ny) { c->last_error = "get_charge: buffer too small"; return ZPIC_E_BUFSIZE; }
  try {
    double* rho = alloc_n<double>(c, (size_t)g.nx * g.ny);   // zeroed
    float* rhof = alloc_n<float>(c, (size_t)g.nx * g.ny);
    const PushParams p = push_params(c);                      // spill_in = the live loose list
    launch_charge(p, rho, !c->slab && c->bcy == ZPIC_BC_PERIODIC ? 1 : 0, c->stream);
    launch_to_float(rho, rhof, (long)g.nx * g.ny, c->stream);
    CUDA_OR_THROW(cudaGetLastError());
    CUDA_OR_THROW(cudaMemcpyAsync(out, rhof, (size_t)g.nx * g.ny * 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OR_THROW(cudaStreamSynchronize(c->stream));
    dev_free(c, rho);
    dev_free(c, rhof);
  } catch (const Fail& f) {
    c->last_error = f.msg;
    return f.st;
  }
  return ZPIC_OK;
}

zpic_status zpic_layout(zpic_ctx* c, int32_t* y0, int32_t* ny_local) {
  if (!c) return ZPIC_E_INVALID;
  if (y0) *y0 = c->y0;
  if (ny_local) *ny_local = c->g.ny;
  return ZPIC_OK;
}

zpic_status zpic_counters(zpic_ctx* c, int64_t* out, int32_t n) {
  if (!c || !out) return ZPIC_E_INVALID;
  zpic_status st = check_sticky(c);
  if (st != ZPIC_OK) return st;
  int stats[4] = {0, 0, 0, 0};   // [0] movers of the last step, [1] loose, [2] / [3] tiles K2s sorted / left
  cudaMemcpy(stats, c->stats, sizeof(stats), cudaMemcpyDeviceToHost);
  int64_t total = 0;
  int maxfill = 0;
  for (int s = 0; s < c->nspecies; ++s) {
    std::vector<int> cnt(c->ntiles);
    cudaMemcpy(cnt.data(), c->ps[s].cnt, c->ntiles * 4, cudaMemcpyDeviceToHost);
    for (int v : cnt) { total += v; maxfill = std::max(maxfill, (int)(1000.0 * v / c->ps[s].cap)); }
  }
  int nl = 0;
  cudaMemcpy(&nl, c->spill[c->steps & 1].count, 4, cudaMemcpyDeviceToHost);
  const int64_t v[11] = {total + nl, stats[0], maxfill, c->repacks, c->steps, c->ntiles, c->launches, c->T,
                          stats[2], stats[3], nl};
  for (int k = 0; k < n && k < 11; ++k) out[k] = v[k];
  return ZPIC_OK;
}

zpic_status zpic_kernel_times(zpic_ctx* c, const char** names, double* ms, int32_t* launches, int32_t* n_inout) {
  if (!c || !n_inout) return ZPIC_E_INVALID;
  cudaStreamSynchronize(c->stream);
  drain_profile(c);
  const int n = std::min<int>(*n_inout, K_COUNT);
  for (int k = 0; k < n; ++k) {
    if (names) names[k] = kNames[k];
    if (ms) ms[k] = c->prof_ms[k];
    if (launches) launches[k] = c->prof_count[k];
    c->prof_ms[k] = 0.0;
    c->prof_count[k] = 0;
  }
  *n_inout = K_COUNT;
  return ZPIC_OK;
}

void zpic_free(zpic_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graphs(c);
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  if (c->own_comm && c->comm) ncclCommDestroy((ncclComm_t)c->comm);
  for (auto e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
  if (c->peer_block) cudaFree(c->peer_block);
  if (c->j_block) cudaFree(c->j_block);
  if (c->eb_block) cudaFree(c->eb_block);
  for (auto e : c->prof_ev) cudaEventDestroy(e);
  for (void* p : c->allocations) {
    if (c->opt.free) c->opt.free(p, c->opt.alloc_user);
    else cudaFree(p);
  }
  c->allocations.clear();
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // extern "C"
