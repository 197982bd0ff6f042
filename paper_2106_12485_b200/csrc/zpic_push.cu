// zpic_push.cu — K1, the fused particle kernel of the B200 EM-PIC step.
//
// One CTA per tile of T x T cells.  It stages the tile's E and B (+1 guard cell each side) in
// shared memory, pushes every particle of every species of the tile — interpolation
// (PAPER.md:144), relativistic Boris, charge-conserving deposit
// — and accumulates the tile's current in shared memory as fixed point with
// native integer atomics (one int32 per node at a per-tile scale, or the exact two-word form;
// DESIGN.md §2).  Then it stores the (T+3)^2 current block for K4 (or adds it into J:
// current_mode 1) and fixes up the tile's particle segment.
//
// Divergence control: a path inside its start cell (most of them) is deposited as one piece in
// the main loop; a path that crosses a cell edge is queued (start point, displacement, z weight)
// in a per-warp ring buffer in shared memory, and the queue is drained 32 paths at a time with
// all lanes active: each lane splits its path at the crossings and deposits all 2-3 pieces.
// Re-sort: particles that stay in the tile are written back in place; leavers leave a hole
// (cell = -1) and go to this tile's mailbox for their direction of travel (K3m appends them to
// the destination tile), or to the flat mover list when the box is full or they leave the slab
// (K3).  Once per tile and species, the holes below the new count are filled from the tail — no
// block barrier per chunk, and only O(#leavers) particle moves.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "zpic_device.cuh"

namespace zpic {

constexpr int kQRing = 64;  // per-warp ring of queued crossing paths (<= 31 left + 32 new)
constexpr int kHCap = 256;  // holes recorded per tile and species (else the sentinel fallback)
constexpr int kHole = -1;   // cell value of a vacated slot

// Per-warp ring of crossing paths in shared memory: one 16-byte (x0, y0, dx, dy) and one 8-byte
// (cells, q vz) record per entry (two vector stores per put, two vector loads per drain; the
// entries of a put / drain are consecutive: conflict-free quarter-warps).  The cells word packs
// bytes: start cell lx + 8, ly + 8; end cell (this tile, after the window shift) ex + 8, ey + 8,
// or ey + 8 = 255 when the particle leaves the tile.
struct PathRing {
  float4* p4;
  float2* p2;
  __device__ __forceinline__ void put(int k, int lx, int ly, int ex, int ey, float x0, float y0, float dxp, float dyp,
                                      float q) const {
    p4[k] = make_float4(x0, y0, dxp, dyp);
    p2[k] = make_float2(__int_as_float((lx + 8) | ((ly + 8) << 8) | ((ex + 8) << 16) | ((ey + 8) << 24)), q);
  }
};
constexpr int kRingLeaves = 255 - 8;   // ey of a path whose particle leaves the tile

// Deposit every piece of queued crossing path k (the split of PAPER.md:197).
// The tile's cell histogram follows the particle: -1 at its start cell (in the frame after the
// window shift; a start cell shifted out of the tile was dropped with its column), +1 at its end
// cell if it stays in the tile (occupancy bound).
template <int T, class A>
__device__ __forceinline__ void drain_path(const A& acc, const PathRing& Q, int k, float jxs, float jys, int* err,
                                           int* hist, int shift) {
  const float4 a = Q.p4[k];
  const float2 b = Q.p2[k];
  const int v = __float_as_int(b.x);
  const int lx = (v & 0xff) - 8, ly = ((v >> 8) & 0xff) - 8;
  const int ex = ((v >> 16) & 0xff) - 8, ey = ((v >> 24) & 0xff) - 8;
  if (lx - shift >= 0) atomicAdd(&hist[ly * T + lx - shift], -1);
  if (ey != kRingLeaves) atomicAdd(&hist[ey * T + ex], 1);
  const float x = a.x, y = a.y, dxp = a.z, dyp = a.w, qvz = b.y;
  // a path that stays in its cell moved less than a cell: only a queued path can move >= 1
  if (fabsf(dxp) >= 1.0f || fabsf(dyp) >= 1.0f) atomicOr(err, ERR_MIGRATION);
  const float x1 = __fadd_rn(x, dxp), y1 = __fadd_rn(y, dyp);
  const Crossing c = path_crossings(x, y, dxp, dyp, x1, y1);
  deposit_seg(acc, Seg{lx, ly, x, y, c.xa, c.ya, qvz * c.t1}, jxs, jys);
  Seg s1, s2;
  later_pieces(lx, ly, x1, y1, qvz, c, s1, s2);
  deposit_seg(acc, s1, jxs, jys);
  if (c.di && c.dj) deposit_seg(acc, s2, jxs, jys);
}

// Shared-memory layout of K1 (bytes): the current accumulators (128 B aligned), the per-warp path
// rings, then the repacked fields.  Before the current is zeroed and the rings are used, the
// accumulator + ring bytes receive the TMA boxes of E and B.  A box starts 4 cells left of the
// tile (TMA needs a 16-byte aligned start column: interior column 0 sits at padded column 4) and
// is T + 5 cells rounded up to 4 wide, W = T + 2 rows (local cells -1 .. T).
template <int T>
struct K1Smem {
  static constexpr int W = T + 2, WJ = T + 3;
  static constexpr int BX = (T + 5 + 3) & ~3;                  // TMA box row (16 B multiple)
  static constexpr int BOX = 3 * W * BX * 4;                   // one field's box: 3 components
  static constexpr int BOFF = (BOX + 127) & ~127;              // B's box offset
  static constexpr int JWORDS = (3 * WJ * WJ + 3) & ~3;        // int4-aligned
  static constexpr int JBYTES = (2 * JWORDS * 4 + 127) & ~127;
  static constexpr int QBYTES(int blk) { return 6 * (blk / 32) * kQRing * 4; }
  static constexpr int FBYTES = W * W * (16 + 8 + 2 * 4);   // (Ex, By) node pairs, (Ey, Bx), Ez, Bz
  static constexpr size_t bytes(int blk) { return (size_t)JBYTES + QBYTES(blk) + FBYTES; }
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// NSPEC > 0: the species count is a compile-time constant (species constants become immediate
// constant-bank operands instead of indexed reloads); 0: p.nspecies.
template <int T, int BLK, int MINB, int NSPEC>
__global__ void __launch_bounds__(BLK, MINB) k_push_tiles(const __grid_constant__ PushParams p) {
  const int nspec = NSPEC > 0 ? NSPEC : p.nspecies;
  using L = K1Smem<T>;
  constexpr int W = T + 2, WJ = T + 3, NW = BLK / 32;
  constexpr int JWORDS = L::JWORDS;
  static_assert(2 * kHCap * 4 <= L::QBYTES(BLK), "hole lists exceed the path rings");
  static_assert(L::BOFF + L::BOX <= L::JBYTES + L::QBYTES(BLK), "TMA landing exceeds the current + ring bytes");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  int* s_j = reinterpret_cast<int*>(smem_raw);         // int32 current, or the high words (exact form)
  int* s_jlo = s_j + JWORDS;                           // low words (exact form only)
  int* s_q = reinterpret_cast<int*>(smem_raw + L::JBYTES);   // path rings: NW x kQRing float4, then float2
  float4* s_eb1 = reinterpret_cast<float4*>(smem_raw + L::JBYTES + L::QBYTES(BLK));
  float2* s_eb2 = reinterpret_cast<float2*>(s_eb1 + W * W);
  float* s_ez = reinterpret_cast<float*>(s_eb2 + W * W);
  float* s_bz = s_ez + W * W;
  __shared__ __align__(8) unsigned long long s_bar;
  __shared__ int s_holes[kHCap];
  // the hole fill's lists live in the path rings: it runs after every warp drained its ring and
  // before the next species' loop (a barrier), so the static shared memory stays at 8 CTAs / SM
  int* s_hb = reinterpret_cast<int*>(smem_raw + L::JBYTES);
  int* s_sa = s_hb + kHCap;
  __shared__ unsigned s_bits[kHCap / 32];
  __shared__ int s_cnt[4];  // holes, holes below, stayers above, hole-list overflow
  __shared__ int s_mbc[8];  // mailbox fill per direction (this species)
  __shared__ int s_wsum[2][NW];
  __shared__ double s_ke[kMaxSpecies];
  __shared__ int s_hist[T * T];   // the tile's particles per cell (all species)
  __shared__ int s_occ;            // the tile current's scale exponent S
  if (threadIdx.x < kMaxSpecies) s_ke[threadIdx.x] = 0.0;

  // tile of this CTA; with boundary_last = 1 the interior tile rows come first, the slab-edge rows
  // last; 2: the slab-edge rows only (row 0, then row nty - 1)
#ifndef ZPIC_AB_NO_FUSED_R2
  const int t = p.boundary_last ? [&] {
    const int nint = (p.boundary_last == 1 && p.nty > 2) ? (p.nty - 2) * p.ntx : 0, b = (int)blockIdx.x;
    return b < nint ? p.ntx + b : (b - nint < p.ntx ? b - nint : (p.nty - 1) * p.ntx + (b - nint - p.ntx));
  }() : (int)blockIdx.x + p.tile0;
#else
  const int t = (int)blockIdx.x + p.tile0;
#endif
  const int tx = t % p.ntx, ty = t / p.ntx;
  const int i0 = tx * T, j0 = ty * T;
  const int tw = min(T, p.g.nx - i0), th = min(T, p.g.ny - j0);
  const long pl = p.g.plane;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned ltmask = lanemask_lt();

  // Stage E, B on local cells [-1, T+1)^2 with two TMA box loads (cp.async.bulk.tensor, one
  // elected thread, completion on an mbarrier), then repack into the gather's pair layout.
  // Cells beyond the guard-extended grid come back zero (TMA out-of-bounds fill; the padding
  // columns of a row are zero).
  {
    const float* landE = reinterpret_cast<const float*>(smem_raw);
    const float* landB = reinterpret_cast<const float*>(smem_raw + L::BOFF);
    const unsigned bar = smem_u32(&s_bar);
    if (threadIdx.x == 0) {
      // PEER round 2 fused (boundary_last): a slab-edge tile waits for its neighbour's E/B rows in
      // its guard rows (acquire), then orders them before its TMA (async proxy) reads
#ifndef ZPIC_AB_NO_FUSED_R2
      if (p.r2_flags) {
        const int ia = (ty == 0 && p.has_lo) ? 2 : -1, ib = (ty == p.nty - 1 && p.has_hi) ? 3 : -1;
        if ((ia >= 0 || ib >= 0) && !wait_flags(p.r2_flags, ia, ib, p.r2_epoch, 40000000000LL))
          atomicOr(p.err, ERR_HALO);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
#endif
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * L::BOX) : "memory");
      const int cx = i0 - 4 + kXOff, cy = j0;   // padded column of local cell -4 (16 B aligned), row of -1
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(smem_u32(landE)), "l"(reinterpret_cast<uint64_t>(&p.tmE)), "r"(cx), "r"(cy), "r"(0), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(smem_u32(landB)), "l"(reinterpret_cast<uint64_t>(&p.tmB)), "r"(cx), "r"(cy), "r"(0), "r"(bar)
          : "memory");
    }
    // the tile's cell histogram (p.hist, exact at every step start); with a window shift at the
    // end of this step every cell moves one column left and column 0 leaves the tile
    {
      const int* h = p.hist + (long)t * T * T;
      for (int k = threadIdx.x; k < T * T; k += BLK) {
        const int cx = k % T;
        s_hist[k] = (cx + p.shift < T) ? __ldcg(h + k + p.shift) : 0;
      }
    }
    // the tile current's scale exponent S, computed by K1s from this tile's occupancy bound
    // before this kernel (a plain load: nothing of it stays live in the particle loop)
    if (threadIdx.x == 32) s_occ = p.tscale[t];
    __syncthreads();   // the barrier is initialised before anyone waits on it
    asm volatile(
        "{\n .reg .pred done;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n"
        " @!done bra WAIT_%=;\n}" ::"r"(bar)
        : "memory");
    constexpr int C = W * L::BX;   // one component of a box
    for (int k = threadIdx.x; k < W * W; k += BLK) {
      const int q = (k / W) * L::BX + k % W + 3;   // local cell k % W - 1 sits at box column k % W + 3
      // (Ex, By) of nodes k and k + 1 (the last column's partner is never read)
      s_eb1[k] = make_float4(landE[q], landB[C + q], landE[q + 1], landB[C + q + 1]);
      s_eb2[k] = make_float2(landE[C + q], landB[q]);         // (Ey, Bx)
      s_ez[k] = landE[2 * C + q];
      s_bz[k] = landB[2 * C + q];
    }
    __syncthreads();   // the boxes are consumed before the current is zeroed and the rings are used
  }
  const int S = s_occ;   // (the tile's scale exponent, see above)
  // CTA-uniform choice: one int32 atomic per node at scale 2^S, else (S below the floor: a tile so
  // dense that 2^-S would be coarse, or current_precision = exact) the exact two-word form
  const bool fast = S >= p.fx_smin;
  for (int k = threadIdx.x; k < (fast ? 1 : 2) * JWORDS / 4; k += BLK)
    reinterpret_cast<int4*>(s_j)[k] = make_int4(0, 0, 0, 0);

  const SmemFields<W> F{s_eb1, s_eb2, s_ez, s_bz};
  const int qo = warp * kQRing;
  const PathRing Q{reinterpret_cast<float4*>(s_q) + qo, reinterpret_cast<float2*>(s_q + 4 * NW * kQRing) + qo};

  auto push_all = [&](const auto& A, const float fscale) {
  for (int s = 0; s < nspec; ++s) {
    const PStore ps = p.ps[s];
    const SpeciesConst sc = p.sc[s];
    const float jxs = sc.jx * fscale, jys = sc.jy * fscale, qs = sc.q * fscale;
    const int n = ps.cnt[t];
    const long base = (long)t * ps.cap;
    const bool has_id = ps.nf > F_ID;
    const int chunk_words = BLK * ps.nf;   // a chunk is BLK / 32 whole AoSoA blocks
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
    if (threadIdx.x < 8) s_mbc[threadIdx.x] = 0;
    __syncthreads();
    float ke = 0.f;
    int qn = 0, qh = 0;  // warp-uniform ring fill and head
    // this thread's slot of the current chunk (segments and chunks start on 32-slot blocks)
    uint32_t* pp = ps.slot(base + threadIdx.x);
    // software pipeline: the next chunk's particle is loaded while this one is pushed
    int ncell = 0;
    float nxo = 0.f, nyo = 0.f, nux = 0.f, nuy = 0.f, nuz = 0.f;
    uint32_t nid = 0;
    if ((int)threadIdx.x < n) {
      ncell = (int)__ldcs(pp + F_CELL * 32);
      nxo = __uint_as_float(__ldcs(pp + F_X * 32)); nyo = __uint_as_float(__ldcs(pp + F_Y * 32));
      nux = __uint_as_float(__ldcs(pp + F_UX * 32)); nuy = __uint_as_float(__ldcs(pp + F_UY * 32));
      nuz = __uint_as_float(__ldcs(pp + F_UZ * 32));
      if (has_id) nid = __ldcs(pp + F_ID * 32);
    }
    for (int c0 = 0; c0 < n; c0 += BLK, pp += chunk_words) {
      const int i = c0 + threadIdx.x;
      const bool valid = i < n;
      const int cell = ncell;
      float x = nxo, y = nyo, ux = nux, uy = nuy, uz = nuz;
      const uint32_t id = nid;
      if (i + BLK < n) {
        const uint32_t* qn_ = pp + chunk_words;
        ncell = (int)__ldcs(qn_ + F_CELL * 32);
        nxo = __uint_as_float(__ldcs(qn_ + F_X * 32)); nyo = __uint_as_float(__ldcs(qn_ + F_Y * 32));
        nux = __uint_as_float(__ldcs(qn_ + F_UX * 32)); nuy = __uint_as_float(__ldcs(qn_ + F_UY * 32));
        nuz = __uint_as_float(__ldcs(qn_ + F_UZ * 32));
        if (has_id) nid = __ldcs(qn_ + F_ID * 32);
      }
      bool cross = false, stay = false, move = false;
      int mdir = -1;
      // set on valid lanes only; read only under cross / stay / move, which are false elsewhere
      // (no initialisers: no per-chunk register zeroing)
      int ix, iy, lx, ly;
      float x0 = 0.f, y0 = 0.f, dxp = 0.f, dyp = 0.f, qvz = 0.f;
      if (valid) {
        ix = cell_ix(cell); iy = cell_iy(cell);
        lx = ix - i0; ly = iy - j0;
        float ex, ey, ez, bx, by, bz;
        interpolate(F, lx, ly, x, y, ex, ey, ez, bx, by, bz);
        ke += boris(ux, uy, uz, ex, ey, ez, bx, by, bz, sc.h);
        const float rg = rsqrtf(1.0f + fmaf(ux, ux, fmaf(uy, uy, uz * uz)));
        // __fmul_rn: no contraction into x + dxp, so the drain recomputes the same end point
        dxp = __fmul_rn(ux * rg, p.dtdx);
        dyp = __fmul_rn(uy * rg, p.dtdy);
        qvz = qs * uz * rg;
        x0 = x; y0 = y;
        const float x1 = __fadd_rn(x, dxp), y1 = __fadd_rn(y, dyp);
        const float fx1 = floorf(x1), fy1 = floorf(y1);
        int di = (int)fx1, dj = (int)fy1;
        cross = (di | dj) != 0;
        // a path inside its start cell is one piece, deposited now; a crossing path is queued
        // and split in the drain (the same pieces path_crossings gives, t1 = 1: fma(1, d, x) = x1)
        if (!cross) deposit_seg(A, Seg{lx, ly, x, y, x1, y1, qvz}, jxs, jys);
        {   // x1 - floor(x1) equals x1 - di exactly; the R6 rule as in renormalise
          float xn = x1 - fx1, yn = y1 - fy1;
          if (xn >= 1.0f) { xn = 0.0f; di += 1; }
          if (yn >= 1.0f) { yn = 0.0f; dj += 1; }
          x = xn;
          y = yn;
        }
        di -= p.shift;   // moving window: the cell index follows the shift at the end of the step
        ix += di; iy += dj;
        if ((unsigned)(lx + di) < (unsigned)tw && (unsigned)(ly + dj) < (unsigned)th) stay = true;
        else move = domain_bc(ix, iy, p);
        // direction of travel out of the tile (a slab exit in y goes through the mover list)
        if (move && p.use_mail && !(p.slab && (iy < 0 || iy >= p.g.ny))) {
          const int ex = lx + di, ey = ly + dj;
          mdir = mail_dir(ex < 0 ? -1 : (ex >= tw ? 1 : 0), ey < 0 ? -1 : (ey >= th ? 1 : 0));
        }
      }
      // crossing paths -> this warp's ring; drain full batches of 32 with every lane active
      const unsigned bal = __ballot_sync(0xffffffffu, cross);
      if (bal) {   // warp-uniform
        if (cross)
          Q.put((qh + qn + __popc(bal & ltmask)) & (kQRing - 1), lx, ly, stay ? ix - i0 : 0, stay ? iy - j0 : kRingLeaves,
                x0, y0, dxp, dyp, qvz);
        qn += __popc(bal);
        __syncwarp();
        if (qn >= 32) {
          drain_path<T>(A, Q, (qh + lane) & (kQRing - 1), jxs, jys, p.err, s_hist, p.shift);
          qh = (qh + 32) & (kQRing - 1);
          qn -= 32;
          __syncwarp();   // the drained entries are read before the next put overwrites them
        }
      }
      if (valid && stay) {
        const int ncell_ = pack_cell(ix, iy);
        if (!p.skip_cell_store || ncell_ != cell) __stcs(pp + F_CELL * 32, (uint32_t)ncell_);
        __stcs(pp + F_X * 32, __float_as_uint(x)); __stcs(pp + F_Y * 32, __float_as_uint(y));
        __stcs(pp + F_UX * 32, __float_as_uint(ux)); __stcs(pp + F_UY * 32, __float_as_uint(uy));
        __stcs(pp + F_UZ * 32, __float_as_uint(uz));
      }
      // leavers (~20 % of the warp-chunks at C5): one warp-uniform branch for the hole record, the
      // mailbox and the mover list
      const bool leave = valid && !stay;
      if (__any_sync(0xffffffffu, leave)) {
        if (leave) {
          pp[F_CELL * 32] = (uint32_t)kHole;
          const int h = atomicAdd(&s_cnt[0], 1);
          if (h < kHCap) s_holes[h] = i;
          else s_cnt[3] = 1;
        }
        // this tile's mailbox for the direction of travel, else (box full, slab exit) the list
        int mslot = -1;
        if (mdir >= 0) {
          const int k = atomicAdd(&s_mbc[mdir], 1);
          if (k < mail_cap(p.mail[s], mdir)) mslot = k;
        }
        const bool glob = move && mslot < 0;
        const int m = warp_reserve(p.movers.count, glob);
        if (mslot >= 0) {
          const MailBox& M = p.mail[s];
          uint32_t* q = M.data + ((long)t * M.per_tile + mail_offset(M, mdir) + mslot) * M.nf;
          q[F_CELL] = (uint32_t)pack_cell(ix, iy);
          q[F_X] = __float_as_uint(x); q[F_Y] = __float_as_uint(y);
          q[F_UX] = __float_as_uint(ux); q[F_UY] = __float_as_uint(uy);
          q[F_UZ] = __float_as_uint(uz);
          if (M.nf > F_ID) q[F_ID] = id;
        }
        if (glob) {
          if (m < p.movers.cap) list_put(p.movers, m, pack_cell(ix, iy), x, y, ux, uy, uz, id, s);
          else atomicOr(p.err, ERR_OVERFLOW);
        }
      }
    }
    if (lane < qn) drain_path<T>(A, Q, (qh + lane) & (kQRing - 1), jxs, jys, p.err, s_hist, p.shift);
    // kinetic energy: warp reduction, one shared fp64 add per warp, one global add per CTA
    for (int o = 16; o > 0; o >>= 1) ke += __shfl_xor_sync(0xffffffffu, ke, o);
    if (lane == 0) atomicAdd(&s_ke[s], (double)ke);
    __syncthreads();   // all deposits, hole records and in-place writes of this species are done
    if (p.use_mail && threadIdx.x < 8)
      p.mail[s].cnt[t * 8 + threadIdx.x] = min(s_mbc[threadIdx.x], mail_cap(p.mail[s], threadIdx.x));

    // ---- re-sort: fill the holes below the new count from the tail --------------------------
    const int nh = s_cnt[0], n2 = n - nh;
    if (nh > 0 && s_cnt[3] == 0) {
      if (warp == 0) {   // one warp, warp-synchronous: the other warps go on (J flush / next species)
        for (int k = lane; k < (nh + 31) / 32; k += 32) s_bits[k] = 0u;
        __syncwarp();
        for (int k = lane; k < nh; k += 32) {
          const int pos = s_holes[k];
          if (pos >= n2) atomicOr(&s_bits[(pos - n2) >> 5], 1u << ((pos - n2) & 31));
        }
        __syncwarp();
        int nhb = 0, nsa = 0;
        for (int k0 = 0; k0 < nh; k0 += 32) {
          const int k = k0 + lane;
          const int pos = k < nh ? s_holes[k] : n2;
          const bool hb = k < nh && pos < n2;                                   // hole below the new count
          const bool sa = k < nh && !((s_bits[k >> 5] >> (k & 31)) & 1u);      // tail slot n2 + k holds a stayer
          const unsigned mb = __ballot_sync(0xffffffffu, hb), ms = __ballot_sync(0xffffffffu, sa);
          if (hb) s_hb[nhb + __popc(mb & ltmask)] = pos;
          if (sa) s_sa[nsa + __popc(ms & ltmask)] = n2 + k;
          nhb += __popc(mb);
          nsa += __popc(ms);
        }
        __syncwarp();
        for (int k = lane; k < nhb; k += 32) {
          uint32_t* d = ps.slot(base + s_hb[k]);
          const uint32_t* src = ps.slot(base + s_sa[k]);
          for (int f = 0; f < ps.nf; ++f) d[f * 32] = src[f * 32];
        }
      }
    } else if (nh > 0) {
      // more holes than the list holds: stable compaction of the whole segment by the sentinel
      __syncthreads();
      int out = 0, buf = 0;
      for (int c0 = 0; c0 < n; c0 += BLK) {
        const int i = c0 + threadIdx.x;
        uint32_t v[7] = {(uint32_t)kHole, 0u, 0u, 0u, 0u, 0u, 0u};
        if (i < n) {
          const uint32_t* src = ps.slot(base + i);
#pragma unroll
          for (int f = 0; f < 7; ++f)
            if (f < ps.nf) v[f] = src[f * 32];
        }
        const bool keep = (int)v[F_CELL] != kHole;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_wsum[buf][warp] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
        for (int w = 0; w < NW; ++w) {
          const int v = s_wsum[buf][w];
          before += (w < warp) ? v : 0;
          tot += v;
        }
        buf ^= 1;
        __syncthreads();   // every thread has read its slot before any slot of this chunk is rewritten
        if (keep) {
          uint32_t* d = ps.slot(base + out + before + __popc(bal & ltmask));
#pragma unroll
          for (int f = 0; f < 7; ++f)
            if (f < ps.nf) d[f * 32] = v[f];
        }
        out += tot;
      }
    }
    if (threadIdx.x == 0) ps.cnt[t] = n2;
    if (s + 1 < nspec) __syncthreads();   // the hole lists / counters are reused by the next species
  }
  };
  if (fast) push_all(SmemCurrentI32<WJ>{s_j}, ldexpf(1.0f, S));
  else push_all(SmemCurrentFx<WJ>{s_j, s_jlo}, kFxScale);
  const bool fast2 = s_occ >= p.fx_smin;   // re-derived after the loop (no register kept live)
  if (p.commutative) {
    // "commutative" ghost current: add the block into J with global atomics;
    // nodes a tile cannot reach stay zero and are skipped (they may lie outside the guards)
    for (int k = threadIdx.x; k < 3 * WJ * WJ; k += BLK) {
      const float v = fast2 ? (float)s_j[k] * ldexpf(1.0f, -s_occ)
                           : (float)(fma((double)s_j[k], 32768.0, (double)s_jlo[k]) * kFxInv);
      const int c = k / (WJ * WJ), r = k % (WJ * WJ);
      if (v != 0.0f) {
        const long o = p.g.at(i0 - 1 + r % WJ, j0 - 1 + r / WJ);
        atomicAdd(p.J + c * pl + o, v);
        if (p.Jlo || p.Jhi) peer_add_j(p, c, j0 - 1 + r / WJ, o, v);   // a slab-edge tile row
      }
    }
    if (p.Jlo || p.Jhi) __threadfence_system();   // the neighbours' round-1 wait follows this kernel
  } else if (fast2) {
    float* jt = p.Jt + (long)t * 3 * WJ * WJ;
    const float finv = ldexpf(1.0f, -s_occ);
    for (int k = threadIdx.x; k < 3 * WJ * WJ; k += BLK) __stcg(jt + k, (float)s_j[k] * finv);
  } else {
    float* jt = p.Jt + (long)t * 3 * WJ * WJ;
    for (int k = threadIdx.x; k < 3 * WJ * WJ; k += BLK)
      __stcg(jt + k, (float)(fma((double)s_j[k], 32768.0, (double)s_jlo[k]) * kFxInv));
  }
  if ((int)threadIdx.x < nspec && s_ke[threadIdx.x] != 0.0)
    atomicAdd(p.ke_slots + threadIdx.x * kEnergySlots + (t & (kEnergySlots - 1)), s_ke[threadIdx.x]);
  // the next step's occupancy bound: the largest 4 x 4 window of this tile's stayers (the histogram
  // is complete: every species' loop ended at a barrier); arrivals add to it after this kernel, to
  // the bound and to their cell of the stored histogram
  if (tw == T && th == T) {   // full tile: one warp slides the windows (T known at compile time)
    if (warp == NW - 1) {
      const int m = window_max_4x4_full_warp<T>(s_hist);
      if (lane == 0 && m > 0) atomicMax(p.occ + t, m);
    }
  } else {
    const int m = __reduce_max_sync(0xffffffffu, window_max_4x4(s_hist, T, tw, th));
    if (lane == 0 && m > 0) atomicMax(p.occ + t, m);
  }
  {
    int* h = p.hist + (long)t * T * T;
    for (int k = threadIdx.x; k < T * T; k += BLK) __stcg(h + k, s_hist[k]);
  }
}

template <int T, int BLK, int MINB, int NSPEC>
static void launch_push_N(const PushParams& p, int ntiles, cudaStream_t st) {
  constexpr size_t smem = K1Smem<T>::bytes(BLK);
  // the attribute is per device: set it once for every device this process launches on
  static unsigned attr_set = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 32 || !((attr_set >> dev) & 1u)) {
    cudaFuncSetAttribute(k_push_tiles<T, BLK, MINB, NSPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev < 32) attr_set |= 1u << dev;
  }
  k_push_tiles<T, BLK, MINB, NSPEC><<<ntiles, BLK, smem, st>>>(p);
}
template <int T, int BLK, int MINB>
static void launch_push_T(const PushParams& p, int ntiles, cudaStream_t st) {
  switch (p.nspecies) {
    case 1: launch_push_N<T, BLK, MINB, 1>(p, ntiles, st); break;
    case 2: launch_push_N<T, BLK, MINB, 2>(p, ntiles, st); break;
    default: launch_push_N<T, BLK, MINB, 0>(p, ntiles, st); break;
  }
}

// K1 launch shape for 16x16 tiles (threads per CTA, CTAs per SM the register budget is sized
// for).  ZPIC_K1_SHAPE selects it for tuning experiments: 0 = 256 x 3 (80 registers),
// 1 = 256 x 4 (64 registers), 2 = 128 x 6 (80 registers), 4 = 128 x 7 (72 registers), 3 = 128 x 8 (64 registers, the
// default: 63.4 % vs 60.5 % of HBM for shape 2 at C5).
static int k1_shape() {
  static int v = [] {
    const char* e = getenv("ZPIC_K1_SHAPE");
    return e ? atoi(e) : 3;
  }();
  return v;
}

void launch_push_tiles(const PushParams& p_in, int tile_begin, int tile_end, cudaStream_t st) {
  if (tile_end <= tile_begin) return;
  PushParams p = p_in;
  p.tile0 = tile_begin;
  const int ntiles = tile_end - tile_begin;
  switch (p.T) {
    case 8:   // a grid of at most two tiles per SM (C1): 256 threads per tile halve each CTA's path
      if (p.ntx * p.nty <= 2 * 148) launch_push_T<8, 256, 4>(p, ntiles, st);
      else launch_push_T<8, 128, 8>(p, ntiles, st);
      break;
    case 16:
      switch (k1_shape()) {
        case 0: launch_push_T<16, 256, 3>(p, ntiles, st); break;
        case 1: launch_push_T<16, 256, 4>(p, ntiles, st); break;
        case 2: launch_push_T<16, 128, 6>(p, ntiles, st); break;
        case 4: launch_push_T<16, 128, 7>(p, ntiles, st); break;
        default: launch_push_T<16, 128, 8>(p, ntiles, st); break;
      }
      break;
    case 32: launch_push_T<32, 256, 2>(p, ntiles, st); break;
  }
}

}  // namespace zpic
