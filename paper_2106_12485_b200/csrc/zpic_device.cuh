// zpic_device.cuh — small device helpers shared by the particle kernels (warp-aggregated
// reservations, block reductions, cell packing, particle boundary conditions, tile insertion).
#pragma once
#include "zpic_kernels.cuh"

namespace zpic {


__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// warp-aggregated slot reservation on a global counter
__device__ __forceinline__ int warp_reserve(int* counter, bool want) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  return want ? base + __popc(m & lanemask_lt()) : -1;
}

__device__ __forceinline__ void block_add_double(double v, double* slot) {
  __shared__ double s_red[kBlock / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) s_red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kBlock / 32; ++k) t += s_red[k];
    if (t != 0.0) atomicAdd(slot, t);
  }
  __syncthreads();
}

// Mailbox direction of travel (dx, dy) in {-1, 0, 1}^2 \ {0}: d = 3 (dy + 1) + (dx + 1), the
// centre skipped.  Corners are d = 0, 2, 5, 7; edges 1, 3, 4, 6.
__host__ __device__ __forceinline__ int mail_dir(int dx, int dy) {
  const int k = 3 * (dy + 1) + (dx + 1);
  return k < 4 ? k : k - 1;
}
__host__ __device__ __forceinline__ void mail_delta(int d, int& dx, int& dy) {
  const int k = d < 4 ? d : d + 1;
  dx = k % 3 - 1;
  dy = k / 3 - 1;
}
__host__ __device__ __forceinline__ bool mail_corner(int d) { return (0xA5u >> d) & 1u; }
__host__ __device__ __forceinline__ int mail_cap(const MailBox& M, int d) {
  return mail_corner(d) ? M.cap_corner : M.cap_edge;
}
__host__ __device__ __forceinline__ int mail_offset(const MailBox& M, int d) {
  const int corners = (0x33222110u >> (4 * d)) & 0xFu;   // corner boxes before d
  return corners * M.cap_corner + (d - corners) * M.cap_edge;
}

__device__ __forceinline__ int pack_cell(int ix, int iy) { return (ix & 0xffff) | (iy << 16); }
__device__ __forceinline__ int cell_ix(int c) { return c & 0xffff; }
__device__ __forceinline__ int cell_iy(int c) { return c >> 16; }

// Apply the particle boundary conditions to a new cell (a5).  Returns false if the particle
// leaves the domain through an open / window edge (removed).  x: periodic wrap or removal.
// y, one slab: periodic wrap or removal; y, slab decomposition: a particle crossing to an
// existing neighbour keeps its out-of-slab iy (-1 or ny) and is routed by insert_particle.
__device__ __forceinline__ bool domain_bc(int& ix, int& iy, const PushParams& p) {
  const GridDesc& g = p.g;
  if (ix < 0 || ix >= g.nx) {
    if (p.bcx != ZPIC_BC_PERIODIC) return false;
    ix += ix < 0 ? g.nx : -g.nx;
  }
  if (iy < 0 || iy >= g.ny) {
    if (p.slab) return iy < 0 ? p.has_lo : p.has_hi;
    if (p.bcy != ZPIC_BC_PERIODIC) return false;
    iy += iy < 0 ? g.ny : -g.ny;
  }
  return true;
}

__device__ __forceinline__ void list_put(const PList& L, int k, int cell, float x, float y, float ux, float uy, float uz,
                                         uint32_t id, int s) {
  L.cell[k] = cell; L.x[k] = x; L.y[k] = y; L.ux[k] = ux; L.uy[k] = uy; L.uz[k] = uz;
  if (L.id) L.id[k] = id;
  L.species[k] = s;
}

__device__ __forceinline__ void list_append(const PList& L, int* err, int cell, float x, float y, float ux, float uy,
                                            float uz, uint32_t id, int s, int err_bit = ERR_OVERFLOW) {
  const int k = atomicAdd(L.count, 1);
  if (k < L.cap) list_put(L, k, cell, x, y, ux, uy, uz, id, s);
  else atomicOr(err, err_bit);
}

// Insert one particle into its tile's slack, else into the loose list; a particle outside the
// slab (iy = -1 or ny, slab decomposition only) goes to the send list of that neighbour with iy
// already in the neighbour's local rows (equal slabs).
__device__ __forceinline__ void insert_particle(const PushParams& p, int s, int ix, int iy, float x, float y, float ux,
                                                float uy, float uz, uint32_t id) {
  if (iy < 0) { list_append(p.send[0], p.err, pack_cell(ix, iy + p.g.ny), x, y, ux, uy, uz, id, s, ERR_HALO); return; }
  if (iy >= p.g.ny) { list_append(p.send[1], p.err, pack_cell(ix, iy - p.g.ny), x, y, ux, uy, uz, id, s, ERR_HALO); return; }
  const int t = (iy / p.T) * p.ntx + (ix / p.T);
  const PStore& ps = p.ps[s];
  const int slot = atomicAdd(ps.cnt + t, 1);
  const int cell = pack_cell(ix, iy);
  if (slot < ps.cap) {
    atomicAdd(p.occ + t, 1);   // the tile's occupancy bound grows with every arrival
    atomicAdd(p.hist + (long)t * p.T * p.T + (iy - (iy / p.T) * p.T) * p.T + (ix - (ix / p.T) * p.T), 1);
    uint32_t* q = ps.slot((long)t * ps.cap + slot);
    q[F_CELL * 32] = (uint32_t)cell;
    q[F_X * 32] = __float_as_uint(x); q[F_Y * 32] = __float_as_uint(y);
    q[F_UX * 32] = __float_as_uint(ux); q[F_UY * 32] = __float_as_uint(uy); q[F_UZ * 32] = __float_as_uint(uz);
    if (ps.nf > F_ID) q[F_ID * 32] = id;
  } else {
    atomicSub(ps.cnt + t, 1);
    list_append(p.spill_out, p.err, cell, x, y, ux, uy, uz, id, s);
  }
}

// Largest particle count of a 4 x 4 cell window of a tile (h: T x T per-cell counts, row width T;
// tw x th: the tile's cells; windows clipped to a smaller tile).  Node (i, k) of a tile's current
// block only receives from particles that start in cells [i-2, i+1] x [k-2, k+1] (a path moves less
// than a cell and its pieces touch the two nodes of their cell per axis), so this bounds the
// number of particles adding into any node.  Per-thread partial maximum over a block-stride.
__device__ __forceinline__ int window_max_4x4(const int* h, int T, int tw, int th) {
  const int wx = min(4, tw), wy = min(4, th), na = tw - wx + 1, nb = th - wy + 1;
  int m = 0;
  for (int k = threadIdx.x; k < na * nb; k += blockDim.x) {
    const int a = k % na, b = k / na;
    int sum = 0;
    for (int y = b; y < b + wy; ++y)
      for (int x = a; x < a + wx; ++x) sum += h[y * T + x];
    m = max(m, sum);
  }
  return m;
}
// The same for a full T x T tile with T known at compile time: lane a < T - 3 of the calling warp
// slides a 4-row window down column strip [a, a + 4) (4 loads per row, running sums in registers);
// returns the warp maximum (every lane), so one warp does the whole tile.
template <int T>
__device__ __forceinline__ int window_max_4x4_full_warp(const int* h) {
  const int a = threadIdx.x & 31;
  int m = 0;
  if (a < T - 3) {
    int r0 = 0, r1 = 0, r2 = 0;
#pragma unroll
    for (int y = 0; y < T; ++y) {
      const int r = h[y * T + a] + h[y * T + a + 1] + h[y * T + a + 2] + h[y * T + a + 3];
      if (y >= 3) m = max(m, r0 + r1 + r2 + r);
      r0 = r1; r1 = r2; r2 = r;
    }
  }
  return __reduce_max_sync(0xffffffffu, m);
}
// Particle message: [count, pad x3][cell][x][y][ux][uy][uz][id][species], each `cap` long.
__host__ __device__ inline size_t msg_bytes(int cap) { return 16 + (size_t)cap * 32; }
__host__ __device__ inline PList msg_list(void* buf, int cap) {
  char* b = (char*)buf;
  PList L;
  L.count = (int32_t*)b;
  L.cell = (int32_t*)(b + 16);
  L.x = (float*)(L.cell + cap);
  L.y = L.x + cap;
  L.ux = L.y + cap;
  L.uy = L.ux + cap;
  L.uz = L.uy + cap;
  L.id = (uint32_t*)(L.uz + cap);
  L.species = (int32_t*)(L.id + cap);
  L.cap = cap;
  return L;
}

// Cross-slab commutative current ("adjacent regions ... in any order"): a deposit
// at node offset o (component c) on this slab's row y <= 0 is also added into the lower neighbour's
// J at its row y + ny_lo, one on row y >= ny into the upper neighbour's row y - ny (same pitch).
__device__ __forceinline__ void peer_add_j(float* Jlo, float* Jhi, long lo_plane, long hi_plane, int lo_ny,
                                           const GridDesc& g, int c, int y, long o, float v) {
  if (Jlo && y <= 0) atomicAdd(Jlo + c * lo_plane + o + (long)lo_ny * g.pitch, v);
  if (Jhi && y >= g.ny) atomicAdd(Jhi + c * hi_plane + o - (long)g.ny * g.pitch, v);
}
__device__ __forceinline__ void peer_add_j(const PushParams& p, int c, int y, long o, float v) {
  peer_add_j(p.Jlo, p.Jhi, p.lo_plane, p.hi_plane, p.lo_ny, p.g, c, y, o, v);
}
// K1L's accumulator in that mode: the slab's own J plus the neighbour's copy of the shared rows
struct PeerGlobalCurrent {
  const PushParams* p;
  __device__ __forceinline__ long index(int i, int k) const { return p->g.at(i, k); }
  __device__ __forceinline__ long row() const { return p->g.pitch; }
  __device__ __forceinline__ void add(int c, long o, float v) const {
    atomicAdd(p->J + c * p->g.plane + o, v);
    peer_add_j(*p, c, (int)(o / p->g.pitch) - 1, o, v);
  }
};

// ---- PEER transport epoch flags (zpic_peer.cu; also K1's fused round-2 wait) -------------------
// Release-store the epoch into a receiver's flag (system scope: NVLink peers).
__device__ __forceinline__ void signal_flag(unsigned long long* f, unsigned long long e) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
}
// Acquire-spin until flags[ia] (and flags[ib]) reach the epoch (-1: not waited for); false when
// `budget` GPU clock cycles pass first.
__device__ __forceinline__ bool wait_flags(const unsigned long long* flags, int ia, int ib, unsigned long long e,
                                           long long budget) {
  const long long t0 = clock64();
  for (int q = 0; q < 2; ++q) {
    const int i = q ? ib : ia;
    if (i < 0) continue;
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + i) : "memory");
      if (v >= e) break;
      if (clock64() - t0 > budget) return false;
      __nanosleep(256);
    }
  }
  return true;
}

}  // namespace zpic
