// zpic_kernels.cu — the sm_100a kernels of the B200 EM-PIC step.
//   K1 k_push_tiles   fused gather + Boris + charge-conserving deposit + cell update + tile
//                     compaction, one CTA per tile, fields and current in shared memory
//   K3m k_mail_gather per-tile mailboxes -> destination tile segments (one warp per tile)
//   K3 k_insert       flat mover list (full boxes, slab exits) -> destination tile slack (or the loose list)
//   K4 k_assemble_j   per-tile current blocks -> guard-extended J grid (plain stores, no atomics)
//   K1L k_push_loose  the loose list: same physics, global-memory fields / current
//   K4b k_guard_x/y   ghost-current reduction and guard refresh
//   K5 k_yee          fused B half step, E step, B half step on a 128x8 tile
//   K0 k_inject       counter-based lattice injection; k_ramp_rows, k_laser:
//                     the C4 density ramp (R16) and laser fields (R17) at zpic_init
//   k_inject_column   moving-window injection (R15); k_filter_x the compensated filter (R12)
//   k_apply_j_halo, k_recv_insert   y-slab halo rounds (§8(e))
//   k_charge, k_export, k_count, k_bin, k_loose_extract   diagnostics, loading and re-packing
//   k_epilogue        energies, counters
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "zpic_device.cuh"

namespace zpic {

// =============================================================================================
// K3: movers -> destination tiles (grid-stride over the device-side count).  Latency-bound by
// the returning slot atomics, so each thread takes kInsU movers at once: all loads, then all
// slot reservations, then all stores (kInsU independent chains in flight).  A warp's movers come
// from a few source tiles (K1 appends them warp by warp) and go to a few destination tiles: lanes
// with the same destination reserve their slots with one atomic (match_any), so their stores
// land on consecutive slots (coalesced in the AoSoA blocks).
constexpr int kInsU = 4;
__global__ void __launch_bounds__(kBlock) k_insert(PushParams p) {
  const int n = min(*p.movers.count, p.movers.cap);
  const int stride = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  // warp-uniform trip count: every lane takes part in the warp collectives
  const int wbase = (blockIdx.x * blockDim.x + (threadIdx.x & ~31));
  for (int k0w = wbase; k0w < n; k0w += kInsU * stride) {
    const int k0 = k0w + lane;
    int cell[kInsU], sp[kInsU], slot[kInsU], t[kInsU];
    float x[kInsU], y[kInsU], ux[kInsU], uy[kInsU], uz[kInsU];
    uint32_t id[kInsU];
#pragma unroll
    for (int u = 0; u < kInsU; ++u) {
      const int k = k0 + u * stride;
      t[u] = -2;   // no mover
      if (k < n) {
        cell[u] = p.movers.cell[k]; sp[u] = p.movers.species[k];
        x[u] = p.movers.x[k]; y[u] = p.movers.y[k];
        ux[u] = p.movers.ux[k]; uy[u] = p.movers.uy[k]; uz[u] = p.movers.uz[k];
        id[u] = p.movers.id ? p.movers.id[k] : 0u;
        const int iy = cell_iy(cell[u]);
        t[u] = (iy < 0 || iy >= p.g.ny) ? -1 : (iy / p.T) * p.ntx + cell_ix(cell[u]) / p.T;
      }
    }
#pragma unroll
    for (int u = 0; u < kInsU; ++u) {
      const int key = t[u] >= 0 ? (sp[u] << 27) | t[u] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(peers) - 1;
      int base = 0;
      if (key >= 0 && lane == leader) base = atomicAdd(p.ps[sp[u]].cnt + t[u], __popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      slot[u] = base + __popc(peers & lt);
    }
#pragma unroll
    for (int u = 0; u < kInsU; ++u) {
      if (t[u] == -2) continue;
      if (t[u] < 0) {   // slab exchange (insert_particle routes it to the neighbour's send list)
        insert_particle(p, sp[u], cell_ix(cell[u]), cell_iy(cell[u]), x[u], y[u], ux[u], uy[u], uz[u], id[u]);
        continue;
      }
      const PStore& ps = p.ps[sp[u]];
      if (slot[u] < ps.cap) {
        atomicAdd(p.occ + t[u], 1);   // occupancy bound and cell histogram of the destination tile
        atomicAdd(p.hist + (long)t[u] * p.T * p.T + (cell_iy(cell[u]) % p.T) * p.T + cell_ix(cell[u]) % p.T, 1);
        uint32_t* q = ps.slot((long)t[u] * ps.cap + slot[u]);
        q[F_CELL * 32] = (uint32_t)cell[u];
        q[F_X * 32] = __float_as_uint(x[u]); q[F_Y * 32] = __float_as_uint(y[u]);
        q[F_UX * 32] = __float_as_uint(ux[u]); q[F_UY * 32] = __float_as_uint(uy[u]); q[F_UZ * 32] = __float_as_uint(uz[u]);
        if (ps.nf > F_ID) q[F_ID * 32] = id[u];
      } else {
        atomicSub(ps.cnt + t[u], 1);
        list_append(p.spill_out, p.err, cell[u], x[u], y[u], ux[u], uy[u], uz[u], id[u], sp[u]);
      }
    }
  }
  if (p.peer_send) __threadfence_system();   // slab exits written into a neighbour's memory
}

// =============================================================================================
// K3m: one warp per (destination tile, species) appends the particles of the 8 mailboxes
// addressed to its tile (the migration to the adjacent region of PAPER.md:197): box (n, d) of
// the neighbour n = tile - delta(d), read and written with consecutive lanes (coalesced loads
// from the box, coalesced stores into the AoSoA segment).  The warp owns the tile's count in
// this kernel; a full segment sends the rest to the loose list.
// 8 CTAs / SM (32 registers, a 16-byte spill): K3m is latency-bound, the extra warps in flight
// take it from 0.30 to 0.26 ms at C5 (same-box A/B, profiles/r2_ab_k3m.log)
#ifndef K3M_MINB
#define K3M_MINB 8
#endif
__global__ void __launch_bounds__(kBlock, K3M_MINB) k_mail_gather(PushParams p) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int ntiles = p.ntx * p.nty;
  if (w >= ntiles * p.nspecies) return;
  const int s = w / ntiles, t = w - s * ntiles;
  const MailBox& M = p.mail[s];
  const PStore& ps = p.ps[s];
  // lane d < 8: the sender of box direction d and its fill (one round trip for all 8 boxes)
  int n = -1, c = 0;
  if (lane < 8) {
    const int tx = t % p.ntx, ty = t / p.ntx;
    int dx, dy;
    mail_delta(lane, dx, dy);
    int sx = tx - dx, sy = ty - dy;
    bool ok = true;
    if (sx < 0 || sx >= p.ntx) {
      ok = p.bcx == ZPIC_BC_PERIODIC;
      sx = sx < 0 ? sx + p.ntx : sx - p.ntx;
    }
    if (sy < 0 || sy >= p.nty) {
      ok = ok && p.bcy == ZPIC_BC_PERIODIC && !p.slab;
      sy = sy < 0 ? sy + p.nty : sy - p.nty;
    }
    if (ok) {
      n = sy * p.ntx + sx;
      c = M.cnt[n * 8 + lane];
    }
  }
  const int pos = ps.cnt[t];
  // exclusive prefix of the 8 fills, then every lane takes entries e = lane, lane + 32, ...
  int off = c;
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, off, o);
    if (lane >= o) off += v;
  }
  const int total = __shfl_sync(0xffffffffu, off, 7);
  off -= c;
  int offs[8], ns[8];
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    offs[d] = __shfl_sync(0xffffffffu, off, d);
    ns[d] = __shfl_sync(0xffffffffu, n, d);
  }
  for (int e = lane; e < total; e += 32) {
    int d = 0;
#pragma unroll
    for (int q = 1; q < 8; ++q) d = e >= offs[q] ? q : d;   // offsets are non-decreasing
    int nd = ns[0], od = offs[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) {
      if (q == d) { nd = ns[q]; od = offs[q]; }
    }
    const uint32_t* src = M.data + ((long)nd * M.per_tile + mail_offset(M, d) + (e - od)) * M.nf;
    const uint32_t cell = src[F_CELL];
    const uint32_t x = src[F_X], y = src[F_Y];
    const uint32_t ux = src[F_UX], uy = src[F_UY], uz = src[F_UZ];
    const uint32_t id = M.nf > F_ID ? src[F_ID] : 0u;
    const int slot = pos + e;
    if (slot < ps.cap) {
#ifndef K3M_NOHIST
      atomicAdd(p.hist + (long)t * p.T * p.T + (cell_iy((int)cell) % p.T) * p.T + cell_ix((int)cell) % p.T, 1);
#endif
      uint32_t* q = ps.slot((long)t * ps.cap + slot);
      q[F_CELL * 32] = cell; q[F_X * 32] = x; q[F_Y * 32] = y;
      q[F_UX * 32] = ux; q[F_UY * 32] = uy; q[F_UZ * 32] = uz;
      if (ps.nf > F_ID) q[F_ID * 32] = id;
    } else {
      list_append(p.spill_out, p.err, (int)cell, __uint_as_float(x), __uint_as_float(y), __uint_as_float(ux),
                  __uint_as_float(uy), __uint_as_float(uz), id, s);
    }
  }
  if (lane == 0) {
    ps.cnt[t] = min(pos + total, ps.cap);
    if (total > 0) atomicAdd(p.occ + t, min(total, max(ps.cap - pos, 0)));   // arrivals: occupancy bound
  }
}

// =============================================================================================
// K4: J grid node (i, j), -1 <= i <= nx+1, -1 <= j <= ny+1, = sum of the (at most 2 x 2) tile
// blocks covering it.  No periodic wrap here: blocks at the domain edge land in the guards and
// K4b folds them ("the reduction is only required for ghost cells").
// Each thread assembles K4R nodes of one column (rows j, j + 1, ...): all their block loads are
// issued before the sums (more bytes in flight per thread; K4 is latency-bound otherwise).
#ifndef ZPIC_K4R   // rows per thread (tools/gpu/k4_ab.sh)
#define ZPIC_K4R 4
#endif
constexpr int K4R = ZPIC_K4R;
template <int T>
__global__ void __launch_bounds__(kBlock) k_assemble_j(float* __restrict__ J, const float* __restrict__ Jt, GridDesc g,
                                                       int ntx, int nty) {
  constexpr int WJ = T + 3;
  const int i = blockIdx.x * blockDim.x + threadIdx.x - 1;
  if (i > g.nx + 1) return;
  // column i's entry in the (at most 2) x-overlapping tile blocks of tile row 0
  const int thx = (i + 1) / T, lhx = i - thx * T;
  const bool xa = thx < ntx, xb = lhx <= 1 && thx >= 1;
  const float* bxa = Jt + (long)thx * 3 * WJ * WJ + (lhx + 1);
  const float* bxb = Jt + (long)(thx - 1) * 3 * WJ * WJ + (lhx + T + 1);
  float v[K4R][3];
#pragma unroll
  for (int r = 0; r < K4R; ++r) {
    const int j = blockIdx.y * K4R + r - 1;
    const int th = (j + 1) / T, lh = j - th * T;
    const bool in = j <= g.ny + 1;
    const bool ya = in && th < nty, yb = in && lh <= 1 && th >= 1;
    const long oa = (long)th * ntx * 3 * WJ * WJ + (lh + 1) * WJ;
    const long ob = (long)(th - 1) * ntx * 3 * WJ * WJ + (lh + T + 1) * WJ;
    v[r][0] = v[r][1] = v[r][2] = 0.f;
    auto add = [&](bool ok, const float* blk) {
      if (ok) {
        v[r][0] += __ldcg(blk);
        v[r][1] += __ldcg(blk + WJ * WJ);
        v[r][2] += __ldcg(blk + 2 * WJ * WJ);
      }
    };
    add(ya && xa, bxa + oa);
    add(ya && xb, bxb + oa);
    add(yb && xa, bxa + ob);
    add(yb && xb, bxb + ob);
  }
#pragma unroll
  for (int r = 0; r < K4R; ++r) {
    const int j = blockIdx.y * K4R + r - 1;
    if (j > g.ny + 1) break;
    const long o = g.at(i, j);
    J[o] = v[r][0];
    J[g.plane + o] = v[r][1];
    J[2 * g.plane + o] = v[r][2];
  }
}

// =============================================================================================
// K2s: periodic in-tile particle re-sort, in place.  K1 writes a particle back into its own slot,
// so a warp's 32 slots, which the injection fills with 32 consecutive cells, drift towards random
// cells as particles cross edges and holes are refilled: the shared-memory gather and current
// atomics of K1 then hit ~2.5x more bank conflicts ("order decay").  The re-sort
// restores the injection order: rank-major, cell-minor (the first particle of every cell in cell
// order, then the second, ...), i.e. the rank of the unique key rank_in_cell * T^2 + cell in a
// shared-memory bitmap (ranks past the bitmap go to the end in arbitrary order).  One CTA per
// tile stages the tile's particles in shared memory (all loads in flight at once), then stores
// them back in sorted order (coalesced).  The cell word is rebuilt from the local cell, so only
// the other fields are staged; a tile with more than `nstage` particles is left as it is.
constexpr int kSortBlock = 512;
constexpr int kSortK = 9;   // particles per thread: nstage <= kSortBlock * kSortK
// key bitmap bits: ranks below kSortBits / T^2 are placed exactly (64 per cell at T = 16)
template <int T>
constexpr int kSortBits = T == 16 ? 16384 : 32768;
template <int T>
__global__ void __launch_bounds__(kSortBlock, 2) k_sort_tiles(PStore ps, int ntx, int nstage, int* stats) {
  constexpr int NC = T * T, RMAX = kSortBits<T> / NC, NW = kSortBits<T> / 32, PER = NW / kSortBlock > 0 ? NW / kSortBlock : 1;
  extern __shared__ __align__(16) uint32_t sort_smem[];
  __shared__ int s_cnt[NC];
  __shared__ unsigned s_bits[NW];
  __shared__ int s_pre[NW];
  __shared__ int s_wsum[kSortBlock / 32];
  __shared__ int s_ovf;
  const int t = blockIdx.x;
  const int n = min(ps.cnt[t], ps.cap);
  if (n > nstage) {   // CTA-uniform: this tile stays unsorted (counted: zpic_counters "unsorted_tiles")
    if (threadIdx.x == 0) atomicAdd(stats + 3, 1);
    return;
  }
  if (threadIdx.x == 0 && n > 0) atomicAdd(stats + 2, 1);
  const int nf = ps.nf;
  uint32_t* stage = sort_smem;                                                        // [nf - 1][nstage]
  unsigned short* sidx = reinterpret_cast<unsigned short*>(sort_smem + (nf - 1) * nstage);   // [nstage]
  unsigned short* lcs = sidx + nstage;                                                // [nstage]
  const int i0 = (t % ntx) * T, j0 = (t / ntx) * T;
  uint32_t* seg = ps.data + ((long)t * ps.cap >> 5) * (32L * nf);   // the tile's segment (cap is a multiple of 32)
  const int wstep = kSortBlock * nf;
  const int off0 = (threadIdx.x >> 5) * 32 * nf + (threadIdx.x & 31);   // slot tid, field 0
  for (int k = threadIdx.x; k < NC; k += kSortBlock) s_cnt[k] = 0;
  for (int k = threadIdx.x; k < NW; k += kSortBlock) s_bits[k] = 0u;
  if (threadIdx.x == 0) s_ovf = 0;
  __syncthreads();
  // 1. stage: the non-cell fields of this thread's slots go global -> shared with cp.async (no
  // registers, every copy in flight at once); the cell words come to registers for the keys
  int key[kSortK];
  uint32_t cellv[kSortK];
#pragma unroll
  for (int q = 0; q < kSortK; ++q) {
    const int i = threadIdx.x + q * kSortBlock;
    cellv[q] = 0u;
    if (i < n) {
      const uint32_t* src = seg + off0 + q * wstep;
      for (int f = 1; f < nf; ++f)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(stage + (f - 1) * nstage + i)), "l"(src + f * 32)
                     : "memory");
      cellv[q] = __ldcs(src + F_CELL * 32);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
  for (int q = 0; q < kSortK; ++q) {
    const int i = threadIdx.x + q * kSortBlock;
    key[q] = -2;
    if (i < n) {
      const int cell = (int)cellv[q];
      const int lc = (cell_ix(cell) - i0) + (cell_iy(cell) - j0) * T;
      lcs[i] = (unsigned short)lc;
      const int r = atomicAdd(&s_cnt[lc], 1);
      key[q] = r < RMAX ? r * NC + lc : -1;
      if (key[q] >= 0) atomicOr(&s_bits[key[q] >> 5], 1u << (key[q] & 31));
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");   // this thread's copies landed (the barrier publishes them)
  __syncthreads();
  // 2. exclusive prefix of the bitmap's popcounts
  int loc[PER], sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int w = threadIdx.x * PER + q;
    loc[q] = sum;
    sum += w < NW ? __popc(s_bits[w]) : 0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  int wbase = 0, nk = 0;
  for (int w = 0; w < kSortBlock / 32; ++w) {
    wbase += w < warp ? s_wsum[w] : 0;
    nk += s_wsum[w];
  }
  const int excl = wbase + incl - sum;
#pragma unroll
  for (int q = 0; q < PER; ++q)
    if (threadIdx.x * PER + q < NW) s_pre[threadIdx.x * PER + q] = excl + loc[q];
  __syncthreads();
  // 3. destination slot of every staged particle
#pragma unroll
  for (int q = 0; q < kSortK; ++q) {
    const int i = threadIdx.x + q * kSortBlock, k = key[q];
    if (k == -2) continue;
    const int slot = k >= 0 ? s_pre[k >> 5] + __popc(s_bits[k >> 5] & ((1u << (k & 31)) - 1u)) : nk + atomicAdd(&s_ovf, 1);
    sidx[slot] = (unsigned short)i;
  }
  __syncthreads();
  // 4. store back in sorted order (coalesced); the cell word from the local cell
#pragma unroll
  for (int q = 0; q < kSortK; ++q) {
    const int s = threadIdx.x + q * kSortBlock;
    if (s < n) {
      const int i = sidx[s], lc = lcs[i];
      uint32_t* d = seg + off0 + q * wstep;
      __stcs(d + F_CELL * 32, (uint32_t)pack_cell(i0 + lc % T, j0 + lc / T));
      for (int f = 1; f < nf; ++f) __stcs(d + f * 32, stage[(f - 1) * nstage + i]);
    }
  }
}

// particles of one tile the re-sort can stage (two CTAs per SM), 0 if it cannot run
int sort_stage_capacity(int nf) {
  const int per = 4 * (nf - 1) + 4;   // staged fields + slot index + local cell
  return std::min(kSortBlock * kSortK, (int)((104 * 1024) / per) / 32 * 32);   // 2 x (dyn + static + 1 KB) <= 228 KB
}
void launch_sort_tiles(const PStore& ps, int T, int ntx, int ntiles, int* stats, cudaStream_t st) {
  const int nstage = sort_stage_capacity(ps.nf);
  const size_t smem = (size_t)nstage * (4 * (ps.nf - 1) + 4);
  switch (T) {
    case 8:
      cudaFuncSetAttribute(k_sort_tiles<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_sort_tiles<8><<<ntiles, kSortBlock, smem, st>>>(ps, ntx, nstage, stats);
      break;
    case 16:
      cudaFuncSetAttribute(k_sort_tiles<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_sort_tiles<16><<<ntiles, kSortBlock, smem, st>>>(ps, ntx, nstage, stats);
      break;
    case 32:
      cudaFuncSetAttribute(k_sort_tiles<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_sort_tiles<32><<<ntiles, kSortBlock, smem, st>>>(ps, ntx, nstage, stats);
      break;
  }
}

// =============================================================================================
// K1L: loose particles (those that found no tile slack): global-memory gather, global atomics
// into the assembled J grid (guard-extended, folded afterwards), then re-insertion.
__global__ void __launch_bounds__(kBlock) k_push_loose(PushParams p) {
  const int n = min(*p.spill_in.count, p.spill_in.cap);
  const GlobalFields F{p.E, p.B, p.g};
  const GlobalCurrent A{p.J, p.g};
  float ke[kMaxSpecies] = {0.f, 0.f, 0.f, 0.f};
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int s = p.spill_in.species[k];
    const SpeciesConst sc = p.sc[s];
    const int cell = p.spill_in.cell[k];
    int ix = cell_ix(cell), iy = cell_iy(cell);
    float x = p.spill_in.x[k], y = p.spill_in.y[k];
    float ux = p.spill_in.ux[k], uy = p.spill_in.uy[k], uz = p.spill_in.uz[k];
    const uint32_t id = p.spill_in.id ? p.spill_in.id[k] : 0u;
    float ex, ey, ez, bx, by, bz;
    interpolate(F, ix, iy, x, y, ex, ey, ez, bx, by, bz);
    const float kk = boris(ux, uy, uz, ex, ey, ez, bx, by, bz, sc.h);
#pragma unroll
    for (int q = 0; q < kMaxSpecies; ++q) ke[q] += (q == s) ? kk : 0.f;
    const float rg = rsqrtf(1.0f + fmaf(ux, ux, fmaf(uy, uy, uz * uz)));
    const float dxp = ux * rg * p.dtdx, dyp = uy * rg * p.dtdy;
    if (fabsf(dxp) >= 1.0f || fabsf(dyp) >= 1.0f) atomicOr(p.err, ERR_MIGRATION);
    int di, dj;
    Seg seg[3];
    const int nseg = split_path(ix, iy, x, y, dxp, dyp, sc.q * uz * rg, seg, di, dj);
    if (p.Jlo || p.Jhi) for (int q = 0; q < nseg; ++q) deposit_seg(PeerGlobalCurrent{&p}, seg[q], sc.jx, sc.jy);
    else for (int q = 0; q < nseg; ++q) deposit_seg(A, seg[q], sc.jx, sc.jy);
    ix += di - p.shift; iy += dj;
    if (domain_bc(ix, iy, p)) insert_particle(p, s, ix, iy, x, y, ux, uy, uz, id);
  }
  for (int s = 0; s < p.nspecies; ++s) block_add_double((double)ke[s], p.ke_slots + s * kEnergySlots + (blockIdx.x & (kEnergySlots - 1)));
  if (p.Jlo || p.Jhi || p.peer_send) __threadfence_system();
}

// =============================================================================================
// K4b: guard handling of a 3-component grid along x (one thread per row and component) or y
// (one thread per column and component).
//   mode 0: ghost-current reduction + periodic refresh (periodic axis)
//   mode 1: periodic refresh (copies)
//   mode 2: zero the guards (open / window axis: guard deposits discarded, fields outside = 0)
//   mode 3: zero the guards but keep the first high guard node of components in keep_mask
//           (Mur-updated tangential E on an open edge, R13)
__global__ void k_guard_x(float* F, GridDesc g, int mode, int keep_mask) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = g.ny + 3;
  if (idx >= 3 * rows) return;
  const int c = idx / rows, j = idx % rows - 1;
  float* r = F + c * g.plane;
  const int nx = g.nx;
  if (mode == 0) {
    r[g.at(nx - 1, j)] += r[g.at(-1, j)];
    r[g.at(0, j)] += r[g.at(nx, j)];
    r[g.at(1, j)] += r[g.at(nx + 1, j)];
  }
  if (mode <= 1) {
    r[g.at(-1, j)] = r[g.at(nx - 1, j)];
    r[g.at(nx, j)] = r[g.at(0, j)];
    r[g.at(nx + 1, j)] = r[g.at(1, j)];
  } else {
    r[g.at(-1, j)] = 0.f;
    if (!(mode == 3 && ((keep_mask >> c) & 1))) r[g.at(nx, j)] = 0.f;
    r[g.at(nx + 1, j)] = 0.f;
  }
}

__global__ void k_guard_y(float* F, GridDesc g, int mode, int keep_mask) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cols = g.nx + 3;
  if (idx >= 3 * cols) return;
  const int c = idx / cols, i = idx % cols - 1;
  float* r = F + c * g.plane;
  const int ny = g.ny;
  if (mode == 0) {
    r[g.at(i, ny - 1)] += r[g.at(i, -1)];
    r[g.at(i, 0)] += r[g.at(i, ny)];
    r[g.at(i, 1)] += r[g.at(i, ny + 1)];
  }
  if (mode <= 1) {
    r[g.at(i, -1)] = r[g.at(i, ny - 1)];
    r[g.at(i, ny)] = r[g.at(i, 0)];
    r[g.at(i, ny + 1)] = r[g.at(i, 1)];
  } else {
    r[g.at(i, -1)] = 0.f;
    if (!(mode == 3 && ((keep_mask >> c) & 1))) r[g.at(i, ny)] = 0.f;
    r[g.at(i, ny + 1)] = 0.f;
  }
}

// =============================================================================================
// K5: Yee advance (R2) on a kYeeTX x kYeeTY (128 x 8) output tile.  E^n is staged on local
// [-1, T+2), B^n on [-1, T+1), J on [0, T+1).  B^{n+1/2} is computed on [-1, T], E^{n+1} on
// [0, T] (the row/column T redundantly, so no second exchange is needed), B^{n+1} on [0, T).
// Outputs go to the other buffer (E1, B1), interior plus periodic guard images, so no tile
// reads a value another tile writes.  FE(n) of the inputs is reduced on the way.
// 4-byte asynchronous global -> shared copy; valid = false zero-fills the destination.
__device__ __forceinline__ void cp_async4(float* sdst, const float* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gsrc), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// (row, column) of a block-strided walk k = tid, tid + kBlock, ... over a W-wide array, advanced
// without a division per step.
template <int W>
struct RowCol {
  int r, c;
  __device__ __forceinline__ explicit RowCol(int k) : r(k / W), c(k % W) {}
  __device__ __forceinline__ void next() {
    c += kBlock % W;
    r += kBlock / W;
    if (c >= W) { c -= W; ++r; }
  }
};

// K5 tile TX x TY.  Its staged boxes (TMA, one elected thread, mbarrier completion): E on local
// rows [-1, TY+2) and B on [-1, TY+1), both from column -4 (the 16-byte aligned padded column i0;
// TMA faults on an unaligned start) and TX + 8 wide; J on rows [0, TY+1) from column 0, TX + 4
// wide.  Outside the
// guard-extended grid the boxes read zero (out-of-bounds rows; the padding columns are zero).
struct YeeBox {
  static constexpr int TX = kYeeTX, TY = kYeeTY;
  static constexpr int XE = TX + 8, YE = TY + 3, XB = TX + 8, YB = TY + 2, XJ = TX + 4, YJ = TY + 1;
  static constexpr int E = 3 * YE * XE, B = 3 * YB * XB, J = 3 * YJ * XJ;   // floats
  static constexpr int OB = (E + 31) & ~31, OJ = OB + ((B + 31) & ~31);       // 128-byte aligned boxes
  static constexpr size_t bytes = (size_t)(OJ + J) * 4;
};
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, int x, int y, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(0), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(kBlock) k_yee(const __grid_constant__ YeeParams p) {
  constexpr int TX = kYeeTX, TY = kYeeTY, TM = (TX > TY ? TX : TY) + 1;
  constexpr int WE = YeeBox::XE, WB = YeeBox::XB, WJ = YeeBox::XJ;   // row widths of the staged boxes
  extern __shared__ __align__(128) float yee_smem[];
  float (*sE)[YeeBox::YE * YeeBox::XE] = reinterpret_cast<float (*)[YeeBox::YE * YeeBox::XE]>(yee_smem);
  float (*sB)[YeeBox::YB * YeeBox::XB] = reinterpret_cast<float (*)[YeeBox::YB * YeeBox::XB]>(yee_smem + YeeBox::OB);
  float (*sJ)[YeeBox::YJ * YeeBox::XJ] = reinterpret_cast<float (*)[YeeBox::YJ * YeeBox::XJ]>(yee_smem + YeeBox::OJ);
  __shared__ float s_mur[4][2][2][TM];  // E^n on Mur node lines: [edge][component][b, b'][index]
  __shared__ __align__(8) unsigned long long s_bar[2];   // [0] the E and B boxes, [1] the J box
  const GridDesc& g = p.g;
  const int i0 = blockIdx.x * TX, j0 = (blockIdx.y + p.row0) * TY;
  const int tw = min(TX, g.nx - i0), th = min(TY, g.ny - j0);
  const long pl = g.plane;
  // y edges of this slab that are domain edges (with a slab decomposition the others are
  // interfaces whose guards come from the neighbour)
  const bool ylo_dom = p.bcy != ZPIC_BC_PERIODIC && p.ylo_edge, yhi_dom = p.bcy != ZPIC_BC_PERIODIC && p.yhi_edge;

  const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar[0]);
  const unsigned barj = (unsigned)__cvta_generic_to_shared(&s_bar[1]);
  {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barj) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((YeeBox::E + YeeBox::B) * 4)
                   : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(barj), "r"(YeeBox::J * 4) : "memory");
      // padded column of local cell -4 is i0 (kXOff = 4); padded row of local row r is j0 + r + 1
      tma_load_3d((unsigned)__cvta_generic_to_shared(&sE[0][0]), &p.tmE, i0, j0, bar);
      tma_load_3d((unsigned)__cvta_generic_to_shared(&sB[0][0]), &p.tmB, i0, j0, bar);
      tma_load_3d((unsigned)__cvta_generic_to_shared(&sJ[0][0]), &p.tmJ, i0 + kXOff, j0 + 1, barj);
    }
    __syncthreads();
    asm volatile(
        "{\n .reg .pred done;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n"
        " @!done bra WAIT_%=;\n}" ::"r"(bar)
        : "memory");
  }

#define EI(lx, ly) (((ly) + 1) * WE + (lx) + 4)
#define BI(lx, ly) (((ly) + 1) * WB + (lx) + 4)
#define JI(lx, ly) ((ly) * WJ + (lx))
  // FE(n) = 1/2 dx dy sum(E^2 + B^2) over this tile's interior cells
  float fe = 0.f;
  for (int k = threadIdx.x; k < TX * TY; k += kBlock) {
    const int lx = k % TX, ly = k / TX;
    if (lx < tw && ly < th) {
      const int e = EI(lx, ly), b = BI(lx, ly);
#pragma unroll
      for (int c = 0; c < 3; ++c) fe += sE[c][e] * sE[c][e] + sB[c][b] * sB[c][b];
    }
  }
  // B^{n+1/2} on [-1, TX] x [-1, TY]
  RowCol<TX + 2> rcb(threadIdx.x);
  for (int k = threadIdx.x; k < (TX + 2) * (TY + 2); k += kBlock, rcb.next()) {
    const int lx = rcb.c - 1, ly = rcb.r - 1;
    const int bk = BI(lx, ly);
    const int gi = i0 + lx, gj = j0 + ly;
    if ((p.bcx != ZPIC_BC_PERIODIC && (gi < 0 || gi >= g.nx)) || (gj < 0 && ylo_dom) || (gj >= g.ny && yhi_dom))
      continue;   // B guards of a non-periodic axis stay 0 (only the interior is advanced)
    const float ez = sE[2][EI(lx, ly)];
    sB[0][bk] -= p.hdy * (sE[2][EI(lx, ly + 1)] - ez);
    sB[1][bk] += p.hdx * (sE[2][EI(lx + 1, ly)] - ez);
    sB[2][bk] += p.hdy * (sE[0][EI(lx, ly + 1)] - sE[0][EI(lx, ly)]) - p.hdx * (sE[1][EI(lx + 1, ly)] - sE[1][EI(lx, ly)]);
  }
  if (p.bcx == ZPIC_BC_OPEN || p.bcy == ZPIC_BC_OPEN) {   // save E^n on the Mur node lines
    for (int k = threadIdx.x; k < 4 * 2 * 2 * TM; k += kBlock) {
      const int idx = k % TM, node = (k / TM) % 2, comp = (k / (2 * TM)) % 2, edge = k / (4 * TM);
      float v = 0.f;
      if (edge < 2 && p.bcx == ZPIC_BC_OPEN && idx <= th) {
        const int bn = edge ? tw : 0, bp = edge ? tw - 1 : 1;
        v = sE[comp ? 2 : 1][EI(node ? bp : bn, idx)];
      } else if (edge >= 2 && p.bcy == ZPIC_BC_OPEN && idx <= tw) {
        const int bn = edge == 3 ? th : 0, bp = edge == 3 ? th - 1 : 1;
        v = sE[comp ? 2 : 0][EI(idx, node ? bp : bn)];
      }
      s_mur[edge][comp][node][idx] = v;
    }
  }
  __syncthreads();
  // the J box (its own barrier: its transfer overlaps the B half step)
  asm volatile(
      "{\n .reg .pred done;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n"
      " @!done bra WAIT_%=;\n}" ::"r"(barj)
      : "memory");
  // E^{n+1} on [0, TX] x [0, TY]
  RowCol<TX + 1> rcj(threadIdx.x);
  for (int k = threadIdx.x; k < (TX + 1) * (TY + 1); k += kBlock, rcj.next()) {
    const int lx = rcj.c, ly = rcj.r;
    const int jk = JI(lx, ly);
    const int e = EI(lx, ly), b = BI(lx, ly);
    sE[0][e] += p.dtdy * (sB[2][b] - sB[2][BI(lx, ly - 1)]) - p.dt * sJ[0][jk];
    sE[1][e] -= p.dtdx * (sB[2][b] - sB[2][BI(lx - 1, ly)]) + p.dt * sJ[1][jk];
    sE[2][e] += p.dtdx * (sB[1][b] - sB[1][BI(lx - 1, ly)]) - p.dtdy * (sB[0][b] - sB[0][BI(lx, ly - 1)]) - p.dt * sJ[2][jk];
  }
  __syncthreads();
  // Non-periodic edges (R13, R14).  The node line on a domain edge holds: Mur-1 values for the
  // tangential E on an open edge, E^{n+1}_b = E^n_b' + k (E^{n+1}_b' - E^n_b); zero (a guard) for
  // everything else outside the box.  x edges first, then y edges (the oracle's order).
  const bool xlo = i0 == 0, xhi = i0 + tw == g.nx, ylo = j0 == 0 && ylo_dom, yhi = j0 + th == g.ny && yhi_dom;
  if (p.bcx != ZPIC_BC_PERIODIC && (xlo || xhi)) {
    for (int k = threadIdx.x; k < 2 * (th + 1); k += kBlock) {
      const int ly = k % (th + 1), hiE = k / (th + 1);
      if (!(hiE ? xhi : xlo)) continue;
      const int gj = j0 + ly, bn = hiE ? tw : 0, bp = hiE ? tw - 1 : 1;
      const bool row_out = yhi && gj == g.ny;   // guard row of an open y axis
      if (p.bcx == ZPIC_BC_OPEN && !row_out) {
        sE[1][EI(bn, ly)] = s_mur[hiE][0][1][ly] + p.murx * (sE[1][EI(bp, ly)] - s_mur[hiE][0][0][ly]);
        // a corner node of two open edges (Ez at (0, 0), (nx, 0)) takes the y-edge Mur (R13 corner rule)
        if (!(ylo && p.bcy == ZPIC_BC_OPEN && gj == 0))
          sE[2][EI(bn, ly)] = s_mur[hiE][1][1][ly] + p.murx * (sE[2][EI(bp, ly)] - s_mur[hiE][1][0][ly]);
        if (hiE) sE[0][EI(bn, ly)] = 0.f;
      } else if (hiE) {
        sE[0][EI(bn, ly)] = 0.f; sE[1][EI(bn, ly)] = 0.f; sE[2][EI(bn, ly)] = 0.f;
      }
    }
  }
  __syncthreads();
  if (p.bcy != ZPIC_BC_PERIODIC && (ylo || yhi)) {
    for (int k = threadIdx.x; k < 2 * (tw + 1); k += kBlock) {
      const int lx = k % (tw + 1), hiE = k / (tw + 1);
      if (!(hiE ? yhi : ylo)) continue;
      const int gi = i0 + lx, bn = hiE ? th : 0, bp = hiE ? th - 1 : 1;
      // column nx of a non-periodic x axis: guards set by the x pass, except Ez on two open edges,
      // whose corner nodes (nx, 0) and (nx, ny) follow the y-edge Mur (R13 corner rule)
      const bool corner = p.bcx != ZPIC_BC_PERIODIC && gi == g.nx;
      if (corner && p.bcx != ZPIC_BC_OPEN) continue;
      if (p.bcy == ZPIC_BC_OPEN) {
        if (!corner)
          sE[0][EI(lx, bn)] = s_mur[2 + hiE][0][1][lx] + p.mury * (sE[0][EI(lx, bp)] - s_mur[2 + hiE][0][0][lx]);
        sE[2][EI(lx, bn)] = s_mur[2 + hiE][1][1][lx] + p.mury * (sE[2][EI(lx, bp)] - s_mur[2 + hiE][1][0][lx]);
        if (hiE && !corner) sE[1][EI(lx, bn)] = 0.f;
      }
    }
  }
  __syncthreads();
  // B^{n+1} on [0, TX) x [0, TY) and the stores
  for (int k = threadIdx.x; k < TX * TY; k += kBlock) {
    const int lx = k % TX, ly = k / TX;
    if (lx >= tw || ly >= th) continue;
    const int e = EI(lx, ly), b = BI(lx, ly);
    const float ez = sE[2][e];
    const float bx = sB[0][b] - p.hdy * (sE[2][EI(lx, ly + 1)] - ez);
    const float by = sB[1][b] + p.hdx * (sE[2][EI(lx + 1, ly)] - ez);
    const float bz = sB[2][b] + p.hdy * (sE[0][EI(lx, ly + 1)] - sE[0][e]) - p.hdx * (sE[1][EI(lx + 1, ly)] - sE[1][e]);
    const float ex = sE[0][e], ey = sE[1][e];
    const int gi = i0 + lx - p.shift, gj = j0 + ly;   // window shift: column i is stored at i - 1
    if (gi < 0) continue;
    auto put = [&](int xi, int yj) {
      const int o = (int)g.at(xi, yj), ipl = (int)pl;
      p.E1[o] = ex; p.E1[ipl + o] = ey; p.E1[2 * ipl + o] = ez;
      p.B1[o] = bx; p.B1[ipl + o] = by; p.B1[2 * ipl + o] = bz;
    };
    put(gi, gj);
    // periodic guard images (x: columns nx, nx + 1 <- 0, 1 and -1 <- nx - 1; y likewise)
    const bool px = p.bcx == ZPIC_BC_PERIODIC;
    const bool xa = px && gi <= 1, xb = px && gi == g.nx - 1;
    const bool ya = p.y_images && gj <= 1, yb = p.y_images && gj == g.ny - 1;
    if (xa | xb | ya | yb) {
      if (xa) put(gi + g.nx, gj);
      if (xb) put(-1, gj);
      if (ya) { put(gi, gj + g.ny); if (xa) put(gi + g.nx, gj + g.ny); if (xb) put(-1, gj + g.ny); }
      if (yb) { put(gi, -1); if (xa) put(gi + g.nx, -1); if (xb) put(-1, -1); }
    }
  }
  // Mur nodes on the high edges sit in the first high guard (node nx / ny)
  if (p.bcx == ZPIC_BC_OPEN && xhi) {
    for (int ly = threadIdx.x; ly < th; ly += kBlock) {
      const int gj = j0 + ly;
      int ys[3], nys = 1;
      ys[0] = gj;
      if (p.y_images) {
        if (gj <= 1) ys[nys++] = gj + g.ny;
        if (gj == g.ny - 1) ys[nys++] = -1;
      }
      for (int a = 0; a < nys; ++a) {
        const long o = g.at(g.nx, ys[a]);
        p.E1[pl + o] = sE[1][EI(tw, ly)];
        p.E1[2 * pl + o] = sE[2][EI(tw, ly)];
      }
    }
  }
  if (p.shift && xhi) {   // the column entering the window is empty (R14)
    for (int ly = threadIdx.x; ly <= th; ly += kBlock) {
      const int gj = j0 + ly;
      if (ly == th && !(p.bcy == ZPIC_BC_OPEN && yhi)) continue;   // row ny only holds Mur nodes
      int ys[3], nys = 1;
      ys[0] = gj;
      if (p.y_images) {
        if (gj <= 1) ys[nys++] = gj + g.ny;
        if (gj == g.ny - 1) ys[nys++] = -1;
      }
      for (int a = 0; a < nys; ++a) {
        const long o = g.at(g.nx - 1, ys[a]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          p.E1[c * pl + o] = 0.f;
          if (ly < th) p.B1[c * pl + o] = 0.f;
        }
      }
    }
  }
  if (p.bcy == ZPIC_BC_OPEN && yhi) {
    if (p.bcx == ZPIC_BC_OPEN && xhi && threadIdx.x == 0)   // corner node (nx, ny): Ez only
      p.E1[2 * pl + g.at(g.nx, g.ny)] = sE[2][EI(tw, th)];
    for (int lx = threadIdx.x; lx < tw; lx += kBlock) {
      const int gi = i0 + lx - p.shift;
      if (gi < 0 || (p.shift && gi == g.nx - 1)) continue;
      int xs[3], nxs = 1;
      xs[0] = gi;
      if (p.bcx == ZPIC_BC_PERIODIC) {
        if (gi <= 1) xs[nxs++] = gi + g.nx;
        if (gi == g.nx - 1) xs[nxs++] = -1;
      }
      for (int a = 0; a < nxs; ++a) {
        const long o = g.at(xs[a], g.ny);
        p.E1[o] = sE[0][EI(lx, th)];
        p.E1[2 * pl + o] = sE[2][EI(lx, th)];
      }
    }
  }
#undef EI
#undef BI
#undef JI
  // PEER round 2 (fused): the rows a slab-edge tile just stored, also into the neighbours' guard
  // rows, for the columns this CTA wrote (its output columns and the x guard columns it owns: the
  // periodic images of columns 0, 1 (first tile) and nx - 1 (last tile), the Mur node column nx of
  // an open x edge (last tile); the other guard columns are never written, zero on both sides)
  const bool lo_rows = p.peer_lo_E && j0 == 0, hi_rows = p.peer_hi_E && j0 + th == g.ny;
  if (lo_rows || hi_rows) {
    __syncthreads();   // this CTA's stores of the rows are visible to the whole CTA
    const bool xlo = i0 == 0, xhi = i0 + tw == g.nx, per = p.bcx == ZPIC_BC_PERIODIC;
    const int c0 = max(0, i0 - p.shift), c1 = xhi ? g.nx : i0 + tw - p.shift;
    const int nmain = c1 - c0;
    const int nguard = per ? (xlo ? 2 : 0) + (xhi ? 1 : 0) : (xhi && p.bcx == ZPIC_BC_OPEN ? 1 : 0);
    const int ncol = nmain + nguard;
    const int nrow = (lo_rows ? 2 : 0) + (hi_rows ? 1 : 0);
    const long P = g.pitch;
    for (int k = threadIdx.x; k < nrow * 6 * ncol; k += kBlock) {
      const int q = k % ncol, fc = (k / ncol) % 6, rr = k / (6 * ncol);
      int col;
      if (q < nmain) col = c0 + q;
      else if (per) col = (xlo && q - nmain < 2) ? g.nx + (q - nmain) : -1;
      else col = g.nx;
      const int f = fc / 3, c = fc % 3;
      const int row = (lo_rows && rr < 2) ? rr : g.ny - 1;
      const float v = (f ? p.B1 : p.E1)[c * pl + g.at(col, row)];
      if (lo_rows && rr < 2)
        (f ? p.peer_lo_B : p.peer_lo_E)[c * p.peer_lo_plane + (long)(p.peer_lo_ny + 1 + rr) * P + col + kXOff] = v;
      else
        (f ? p.peer_hi_B : p.peer_hi_E)[c * p.peer_hi_plane + col + kXOff] = v;
    }
    __threadfence_system();   // before the round's signal (the kernel after this one)
  }
  block_add_double((double)fe * p.fe_scale,
                   p.fe_slots + (((blockIdx.y + p.row0) * gridDim.x + blockIdx.x) & (kEnergySlots - 1)));
}

// =============================================================================================
// Epilogue (1 CTA): reduce the energy slots of the step just taken, reset per-step counters.
__global__ void k_epilogue(double* ke_slots, double* fe_slots, double* energy, int nspecies, const double* ke_scale4,
                           int* movers_count, int* spill_in_count, int* spill_out_count, int* stats,
                           int64_t* d_nmove, int shifted) {
  __shared__ double red[kBlock];
  for (int q = 0; q <= nspecies; ++q) {
    double* slots = q == 0 ? fe_slots : ke_slots + (q - 1) * kEnergySlots;
    double v = 0.0;
    for (int k = threadIdx.x; k < kEnergySlots; k += blockDim.x) { v += slots[k]; slots[k] = 0.0; }
    red[threadIdx.x] = v;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) energy[q] = q == 0 ? red[0] : red[0] * ke_scale4[q - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    stats[0] = *movers_count;
    *movers_count = 0;
    *spill_in_count = 0;
    stats[1] = *spill_out_count;
    if (shifted) *d_nmove += 1;
  }
}

// =============================================================================================
// K0: lattice injection with the counter-based generator (synth/generate.py
// documents the same definition for the host side).  One CTA per tile; the filled cells are the
// columns [c_lo, c_hi) of the tile; particle p of the tile goes to cell p % ncell (cell-strided,
// so consecutive threads deposit into different cells) and sub-lattice point p / ncell.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform01(uint64_t key, uint64_t id, int j) {
  const uint64_t r = mix64(key ^ mix64(id * 8ull + (uint64_t)j));
  return __dmul_rn(__dadd_rn((double)(r >> 11), 0.5), 1.1102230246251565e-16);  // 2^-53
}
__device__ __forceinline__ float thermal(uint64_t key, uint64_t id, int k, double ufl, double uth) {
  if (uth == 0.0) return (float)ufl;
  const double u1 = uniform01(key, id, 2 * k), u2 = uniform01(key, id, 2 * k + 1);
  const double nrm = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586, u2)));
  return (float)__dadd_rn(ufl, __dmul_rn(uth, nrm));
}

__global__ void __launch_bounds__(kBlock) k_inject(InjectParams q) {
  const int t = blockIdx.x;
  const int tx = t % q.ntx, ty = t / q.ntx;
  const int i0 = tx * q.T, j0 = ty * q.T;
  const int c_lo = max(i0, q.col_lo), c_hi = min(min(i0 + q.T, q.nx_global), q.col_hi);
  const int rows = min(q.T, q.ny - j0);
  const int wc = max(0, c_hi - c_lo);
  const int ncell = wc * rows;
  const int ppc = q.px * q.py;
  const int n = ncell * ppc;
  const long base = (long)t * q.ps.cap;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const int ck = p % ncell, sub = p / ncell;
    const int ix = c_lo + ck % wc, iy = j0 + ck / wc;
    const int k = sub % q.px, l = sub / q.px;
    const uint64_t id = (((uint64_t)(iy + q.y0) * q.nx_global + ix) * q.py + l) * q.px + k;
    uint32_t* o = q.ps.slot(base + p);
    o[F_CELL * 32] = (uint32_t)pack_cell(ix, iy);
    o[F_X * 32] = __float_as_uint((float)(((double)k + 0.5) / q.px));
    o[F_Y * 32] = __float_as_uint((float)(((double)l + 0.5) / q.py));
    o[F_UX * 32] = __float_as_uint(thermal(q.key, id, 0, q.ufl[0], q.uth[0]));
    o[F_UY * 32] = __float_as_uint(thermal(q.key, id, 1, q.ufl[1], q.uth[1]));
    o[F_UZ * 32] = __float_as_uint(thermal(q.key, id, 2, q.ufl[2], q.uth[2]));
    if (q.ps.nf > F_ID) o[F_ID * 32] = (uint32_t)id;
  }
  if (threadIdx.x == 0) q.ps.cnt[t] = n;
}

// Moving window (R15): fresh plasma in the column entering the window, ix = nx-1:
// the ppc sub-lattice at the species density, u = ufl + uth N with the counter-based generator,
// ids 2^31 + (n_move ny + iy) ppc + l ppc_x + k.  Inserted straight into the tiles.
// n_move is read from the device counter (advanced by the epilogue of every shift step), so a
// captured step graph injects the right column ids when it is replayed.
__global__ void k_inject_column(PushParams p, int s, int px, int py, const int64_t* d_nmove, int ny_global, int y0,
                                uint64_t key, double ufl0, double ufl1, double ufl2, double uth0, double uth1,
                                double uth2) {
  const int64_t n_move = *d_nmove;
  const int ppc = px * py;
  const int n = p.g.ny * ppc;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int iy = k / ppc, sub = k % ppc, l = sub / px, kk = sub % px;
    const uint64_t id = 2147483648ull + ((uint64_t)n_move * ny_global + (iy + y0)) * ppc + (uint64_t)l * px + kk;
    const float x = (float)(((double)kk + 0.5) / px), y = (float)(((double)l + 0.5) / py);
    insert_particle(p, s, p.g.nx - 1, iy, x, y, thermal(key, id, 0, ufl0, uth0), thermal(key, id, 1, ufl1, uth1),
                    thermal(key, id, 2, ufl2, uth2), (uint32_t)id);
  }
}

// Digital current filter along x (R12), all passes fused: one CTA per
// (interior row, component) keeps the row in shared memory, applies n passes of (1/4, 1/2, 1/4)
// and, if compensated, one pass of (-n/4, 1 + n/2, -n/4), refreshing the two guard values before
// every pass (periodic copy, or zero on a non-periodic x axis), and writes the row and its x
// guards once.
__global__ void k_filter_x(const float* __restrict__ Jin, float* __restrict__ Jout, GridDesc g, int npass,
                           int compensated, int periodic) {
  extern __shared__ float srow[];
  float* a = srow;
  float* b = srow + g.nx + 2;
  const int j = blockIdx.x % g.ny, c = blockIdx.x / g.ny;
  const float* in = Jin + c * g.plane;
  float* out = Jout + c * g.plane;
  for (int i = threadIdx.x; i < g.nx; i += blockDim.x) a[i + 1] = in[g.at(i, j)];
  const int total = npass + (compensated && npass > 0 ? 1 : 0);
  for (int pass = 0; pass < total; ++pass) {
    __syncthreads();
    if (threadIdx.x == 0) {
      a[0] = periodic ? a[g.nx] : 0.f;
      a[g.nx + 1] = periodic ? a[1] : 0.f;
    }
    __syncthreads();
    const bool comp = pass == npass;
    const float side = comp ? -0.25f * npass : 0.25f, centre = comp ? 1.0f + 0.5f * npass : 0.5f;
    for (int i = threadIdx.x; i < g.nx; i += blockDim.x) b[i + 1] = side * a[i] + centre * a[i + 1] + side * a[i + 2];
    float* t = a; a = b; b = t;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < g.nx; i += blockDim.x) out[g.at(i, j)] = a[i + 1];
  if (threadIdx.x == 0) {
    out[g.at(-1, j)] = periodic ? a[g.nx] : 0.f;
    out[g.at(g.nx, j)] = periodic ? a[1] : 0.f;
    out[g.at(g.nx + 1, j)] = periodic ? a[2] : 0.f;
  }
}

// The same filter with the passes in registers (total passes <= kFiltR): one thread per kFiltCW
// consecutive outputs of a row, reading the window of the kFiltCW + 2 R inputs around them
// straight from J (aligned 16-byte loads away from the row ends; the rows are L2-resident after
// K4) and applying the passes to the shrinking window without shared memory or barriers, so
// every SM keeps many rows' loads in flight (the row-per-CTA form above is latency-bound).
// Positions outside the row are the periodic images (the refresh before every pass makes the
// passes a circular convolution) or zero after every pass (the zero guards); the values and the
// order of operations per node are those of k_filter_x, so the result is the same bit for bit.
constexpr int kFiltCW = 8, kFiltR = 8;
template <int R>
__global__ void __launch_bounds__(256) k_filter_x_reg(const float* __restrict__ Jin, float* __restrict__ Jout, GridDesc g,
                                                       int npass, int compensated, int periodic) {
  static_assert(R <= 8, "the 16-byte window covers i0 - 8 .. i0 + 15");
  const int nx = g.nx;
  const int nch = (nx + kFiltCW - 1) / kFiltCW;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)nch * 3 * g.ny) return;
  const int row = (int)(idx / nch), i0 = (int)(idx - (long)row * nch) * kFiltCW;
  const int j = row % g.ny, c = row / g.ny;
  const float* in = Jin + c * g.plane + g.at(0, j);   // interior column 0 of the row
  float* out = Jout + c * g.plane + g.at(0, j);
  constexpr int W = kFiltCW + 2 * R;
  float a[W];
  if (i0 >= 8 && i0 + 16 <= nx) {   // (in + i0 is 16-byte aligned: kXOff = 4, pitch % 32 == 0)
    float f[24];
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(in + i0 - 8) + m);
      f[4 * m] = v.x; f[4 * m + 1] = v.y; f[4 * m + 2] = v.z; f[4 * m + 3] = v.w;
    }
#pragma unroll
    for (int k = 0; k < W; ++k) a[k] = f[k + 8 - R];
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      int i = i0 - R + k;
      const bool inside = i >= 0 && i < nx;
      if (periodic) i = ((i % nx) + nx) % nx;
      a[k] = (inside || periodic) ? in[i] : 0.f;
    }
  }
  const int total = npass + (compensated && npass > 0 ? 1 : 0);
#pragma unroll
  for (int pass = 0; pass < R; ++pass) {
    if (pass < total) {
      const bool comp = pass == npass;
      const float side = comp ? -0.25f * npass : 0.25f, centre = comp ? 1.0f + 0.5f * npass : 0.5f;
      float prev = a[pass];   // the old value left of k (updated in place, left to right)
#pragma unroll
      for (int k = pass + 1; k < W - pass - 1; ++k) {
        const float v = side * prev + centre * a[k] + side * a[k + 1];
        prev = a[k];
        const int i = i0 - R + k;
        a[k] = (periodic || (i >= 0 && i < nx)) ? v : 0.f;
      }
    }
  }
  // a[R + q] is output i0 + q (the window shrank by one per pass from each side: R >= passes)
  if (i0 + kFiltCW <= nx) {
    reinterpret_cast<float4*>(out + i0)[0] = make_float4(a[R], a[R + 1], a[R + 2], a[R + 3]);
    reinterpret_cast<float4*>(out + i0)[1] = make_float4(a[R + 4], a[R + 5], a[R + 6], a[R + 7]);
  } else {
#pragma unroll
    for (int q = 0; q < kFiltCW; ++q)
      if (i0 + q < nx) out[i0 + q] = a[R + q];
  }
  // the x guards of the row: the periodic images of the filtered row (the threads that computed
  // them write them), or zero
  if (i0 == 0) {
    out[nx] = periodic ? a[R] : 0.f;
    out[nx + 1] = periodic ? a[R + 1] : 0.f;
  }
  if (i0 + kFiltCW >= nx) {
    float last = 0.f;
#pragma unroll
    for (int q = 0; q < kFiltCW; ++q) last = i0 + q == nx - 1 ? a[R + q] : last;   // (registers only)
    out[-1] = periodic ? last : 0.f;
  }
}

// ---- y-slab decomposition (§8(e)) -----------------------------------------------------------
// Round 1, current: the rows arrive raw (x-folded, not y-folded).  From the upper neighbour:
// its raw rows -1, 0 (rup[c][0..1]); from the lower neighbour: its raw rows ny, ny+1
// (rdn[c][0..1]).  Then ("the reduction is only required for ghost cells"):
//   row ny-1 += upper's row -1;   guard row ny = upper's row 0 + my guard row ny  (= the upper's
//   final row 0, which the redundant E^{n+1} row of the Yee kernel needs);
//   row 0 += lower's row ny;      row 1 += lower's row ny+1.
// At a domain edge (no neighbour) the guard deposits are discarded.  One thread per column of
// the padded row and component (guard columns included: the rows are already x-refreshed).
__global__ void k_apply_j_halo(float* J, GridDesc g, const float* rup, const float* rdn, int has_lo, int has_hi) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 3 * g.pitch) return;
  const int c = idx / g.pitch, col = idx % g.pitch;
  float* F = J + c * g.plane + col;
  const long P = g.pitch;
  if (has_hi) {
    if (rup) {   // (null: the cross-slab commutative current added these rows already)
      F[(long)g.ny * P] += rup[(2 * c) * P + col];                     // row ny-1
      F[(long)(g.ny + 1) * P] += rup[(2 * c + 1) * P + col];           // guard row ny
    }
  } else {
    F[(long)(g.ny + 1) * P] = 0.f;
    F[(long)(g.ny + 2) * P] = 0.f;
  }
  if (has_lo) {
    if (rdn) {
      F[1 * P] += rdn[(2 * c) * P + col];                              // row 0
      F[2 * P] += rdn[(2 * c + 1) * P + col];                          // row 1
    }
  } else {
    F[0] = 0.f;                                                        // guard row -1
  }
}

// Round 1, particles: insert the particles received from both neighbours (already pushed this
// step; iy already in this slab's rows).
__global__ void k_recv_insert(PushParams p, PList from_lo, PList from_hi) {
  const int n_lo = min(*from_lo.count, from_lo.cap), n_hi = min(*from_hi.count, from_hi.cap);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_lo + n_hi; k += gridDim.x * blockDim.x) {
    const PList& L = k < n_lo ? from_lo : from_hi;
    const int q = k < n_lo ? k : k - n_lo;
    const int cell = L.cell[q];
    insert_particle(p, L.species[q], cell_ix(cell), cell_iy(cell), L.x[q], L.y[q], L.ux[q], L.uy[q], L.uz[q], L.id[q]);
  }
}

// Validate host-uploaded particles and count them per tile (err bit 4 = out of the slab).
__global__ void k_count(int T, int ntx, int nx, int ny, int y0, long n, const int32_t* ix, const int32_t* iy,
                        const float* x, const float* y, int* counts, int* err) {
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const int cx = ix[k], cy = iy[k] - y0;
    const float px = x[k], py = y[k];
    if (cx < 0 || cx >= nx || cy < 0 || cy >= ny || !(px >= 0.f && px < 1.f) || !(py >= 0.f && py < 1.f)) {
      atomicOr(err, 4);
      continue;
    }
    atomicAdd(counts + (cy / T) * ntx + cx / T, 1);
  }
}

// Bin host-uploaded particles (global iy -> slab-local) into tiles.
// bad != nullptr: also validate (a particle outside the slab or with an offset outside [0, 1) is
// skipped and counted in *bad); id0: the id of entry 0 when no ids are given.
__global__ void k_bin(PStore ps, int T, int ntx, int y0, long n, const int32_t* ix, const int32_t* iy, const float* x,
                      const float* y, const float* ux, const float* uy, const float* uz, const uint32_t* id, int* err,
                      PList loose, int s, int nx, int ny, int* bad, long id0) {
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const int cx = ix[k], cy = iy[k] - y0;
    if (bad && (cx < 0 || cx >= nx || cy < 0 || cy >= ny || !(x[k] >= 0.f && x[k] < 1.f) || !(y[k] >= 0.f && y[k] < 1.f))) {
      atomicAdd(bad, 1);
      continue;
    }
    const int t = (cy / T) * ntx + cx / T;
    const int slot = atomicAdd(ps.cnt + t, 1);
    if (slot >= ps.cap) {   // tile full (capacity slack < 1): the loose list takes it
      atomicSub(ps.cnt + t, 1);
      list_append(loose, err, pack_cell(cx, cy), x[k], y[k], ux[k], uy[k], uz[k], id ? id[k] : (uint32_t)(id0 + k), s);
      continue;
    }
    uint32_t* o = ps.slot((long)t * ps.cap + slot);
    o[F_CELL * 32] = (uint32_t)pack_cell(cx, cy);
    o[F_X * 32] = __float_as_uint(x[k]); o[F_Y * 32] = __float_as_uint(y[k]);
    o[F_UX * 32] = __float_as_uint(ux[k]); o[F_UY * 32] = __float_as_uint(uy[k]); o[F_UZ * 32] = __float_as_uint(uz[k]);
    if (ps.nf > F_ID) o[F_ID * 32] = id ? id[k] : (uint32_t)(id0 + k);
  }
}

// Ramp species (ZPIC_DENS_RAMP, R16): the host gives one x sub-row (cell ix_r[c], offset x_r[c],
// c < n_row); every y sub-row r of the slab repeats it at y = ((r mod py) + 1/2) / py, with
// id = r_global n_row + c and the seeded momenta.  Output: the flat SoA block of load_species.
__global__ void k_ramp_rows(long n, int n_row, int py, int y0, const int32_t* ixr, const float* xr, uint64_t key,
                            double ufl0, double ufl1, double ufl2, double uth0, double uth1, double uth2, int32_t* ix,
                            int32_t* iy, float* x, float* y, float* ux, float* uy, float* uz, uint32_t* id) {
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const long r = (long)y0 * py + k / n_row;   // global sub-row
    const int c = (int)(k % n_row);
    const uint64_t gid = (uint64_t)r * n_row + c;
    ix[k] = ixr[c];
    iy[k] = (int)(r / py);
    x[k] = xr[c];
    y[k] = (float)(((double)(r % py) + 0.5) / py);
    ux[k] = thermal(key, gid, 0, ufl0, uth0);
    uy[k] = thermal(key, gid, 1, ufl1, uth1);
    uz[k] = thermal(key, gid, 2, ufl2, uth2);
    if (id) id[k] = (uint32_t)gid;
  }
}
void launch_ramp_rows(long n, int n_row, int py, int y0, const int32_t* ixr, const float* xr, uint64_t key,
                      const double* ufl, const double* uth, int32_t* ix, int32_t* iy, float* x, float* y, float* ux,
                      float* uy, float* uz, uint32_t* id, cudaStream_t st) {
  const int grid = (int)std::min<long>((n + kBlock - 1) / kBlock, 148L * 32);
  if (grid > 0)
    k_ramp_rows<<<grid, kBlock, 0, st>>>(n, n_row, py, y0, ixr, xr, key, ufl[0], ufl[1], ufl[2], uth[0], uth[1],
                                         uth[2], ix, iy, x, y, ux, uy, uz, id);
}

// Laser initial fields (zpic_options.laser, R17): E_y at (i, j + 1/2), B_z at (i + 1/2, j + 1/2)
// of the slab's interior (global row j = y0 + local), fp64 then rounded; other components 0.
__device__ __forceinline__ double laser_profile(const LaserParams& L, double xp, double yp) {
  const double lo = L.start - 2.0 * L.fwhm;
  if (!(xp >= lo && xp <= L.start)) return 0.0;
  const double s = sin(3.141592653589793 * (xp - lo) / (2.0 * L.fwhm));
  const double dy = yp - L.yc;
  return L.a0 * L.omega0 * (s * s) * exp(-(dy * dy) / (L.W0 * L.W0)) * cos(L.omega0 * (xp - (L.start - L.fwhm)));
}
__global__ void k_laser(float* E, float* B, GridDesc g, int y0, double dx, double dy, LaserParams L) {
  const long n = (long)g.nx * g.ny;
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const int i = (int)(k % g.nx), j = (int)(k / g.nx);
    const double yj = ((double)(y0 + j) + 0.5) * dy;
    E[g.plane + g.at(i, j)] = (float)laser_profile(L, (double)i * dx, yj);
    B[2 * g.plane + g.at(i, j)] = (float)laser_profile(L, ((double)i + 0.5) * dx, yj);
  }
}
void launch_laser(float* E, float* B, const GridDesc& g, int y0, double dx, double dy, const LaserParams& L,
                  cudaStream_t st) {
  const int grid = (int)std::min<long>(((long)g.nx * g.ny + kBlock - 1) / kBlock, 148L * 32);
  k_laser<<<grid, kBlock, 0, st>>>(E, B, g, y0, dx, dy, L);
}

// Diagnostic charge density (zpic_get_charge): one CTA per tile (and one grid-stride pass over
// the loose list), fp32 global atomics into an [ny][nx] node grid, indices wrapped (x, and y
// unless a slab), nodes outside dropped.
__device__ __forceinline__ void charge_add(double* rho, int nx, int ny, bool wrap_y, int i, int j, double v) {
  if (i >= nx) i -= nx;
  if (j >= ny) {
    if (!wrap_y) return;
    j -= ny;
  }
  atomicAdd(rho + (long)j * nx + i, v);
}
__device__ __forceinline__ void charge_particle(double* rho, int nx, int ny, bool wrap_y, int c, float x, float y, float q) {
  const int i = cell_ix(c), j = cell_iy(c);
  // fp64 weights and sums: the diagnostic resolves the fp32 state to ~1e-16 (its continuity
  // check is not limited by the summation of the node charge)
  const double X = x, Y = y, Q = q;
  charge_add(rho, nx, ny, wrap_y, i, j, Q * (1.0 - X) * (1.0 - Y));
  charge_add(rho, nx, ny, wrap_y, i + 1, j, Q * X * (1.0 - Y));
  charge_add(rho, nx, ny, wrap_y, i, j + 1, Q * (1.0 - X) * Y);
  charge_add(rho, nx, ny, wrap_y, i + 1, j + 1, Q * X * Y);
}
__global__ void k_charge(PushParams p, double* rho, int wrap_y) {
  const int t = blockIdx.x;
  if (t < p.ntx * p.nty) {
    for (int s = 0; s < p.nspecies; ++s) {
      const PStore& ps = p.ps[s];
      const int n = min(ps.cnt[t], ps.cap);
      for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const uint32_t* q = ps.slot((long)t * ps.cap + k);
        charge_particle(rho, p.g.nx, p.g.ny, wrap_y, (int)q[F_CELL * 32], __uint_as_float(q[F_X * 32]),
                        __uint_as_float(q[F_Y * 32]), p.sc[s].q);
      }
    }
  } else {
    const int n = min(*p.spill_in.count, p.spill_in.cap);
    for (int k = (t - p.ntx * p.nty) * blockDim.x + threadIdx.x; k < n; k += 148 * blockDim.x)
      charge_particle(rho, p.g.nx, p.g.ny, wrap_y, p.spill_in.cell[k], p.spill_in.x[k], p.spill_in.y[k],
                      p.sc[p.spill_in.species[k]].q);
  }
}
__global__ void k_to_float(const double* a, float* b, long n) {
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) b[k] = (float)a[k];
}
void launch_to_float(const double* a, float* b, long n, cudaStream_t st) {
  k_to_float<<<148 * 4, kBlock, 0, st>>>(a, b, n);
}
void launch_charge(const PushParams& p, double* rho, int wrap_y, cudaStream_t st) {
  k_charge<<<p.ntx * p.nty + 148, kBlock, 0, st>>>(p, rho, wrap_y);
}

// Copy every tile segment of one species to a contiguous buffer (prefix[t] = output offset);
// global ix, iy on the way out.
__global__ void k_export(PStore ps, const int64_t* prefix, int y0, int32_t* ix, int32_t* iy, float* x, float* y,
                         float* ux, float* uy, float* uz, uint32_t* id) {
  const int t = blockIdx.x;
  const int n = ps.cnt[t];
  const long src = (long)t * ps.cap;
  const int64_t dst = prefix[t];
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const uint32_t* q = ps.slot(src + k);
    const int c = (int)q[F_CELL * 32];
    ix[dst + k] = cell_ix(c);
    iy[dst + k] = cell_iy(c) + y0;
    x[dst + k] = __uint_as_float(q[F_X * 32]); y[dst + k] = __uint_as_float(q[F_Y * 32]);
    ux[dst + k] = __uint_as_float(q[F_UX * 32]); uy[dst + k] = __uint_as_float(q[F_UY * 32]);
    uz[dst + k] = __uint_as_float(q[F_UZ * 32]);
    if (id) id[dst + k] = ps.nf > F_ID ? q[F_ID * 32] : 0u;
  }
}

// ---- host-side launchers --------------------------------------------------------------------
// Re-pack: the loose particles of species s appended after out0 (global iy), in any order.
__global__ void k_loose_extract(PList L, int s, int y0, int32_t* ix, int32_t* iy, float* x, float* y, float* ux,
                                float* uy, float* uz, uint32_t* id, int* counter) {
  const int n = min(*L.count, L.cap);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    if (L.species[k] != s) continue;
    const int o = atomicAdd(counter, 1);
    const int c = L.cell[k];
    ix[o] = cell_ix(c); iy[o] = cell_iy(c) + y0;
    x[o] = L.x[k]; y[o] = L.y[k]; ux[o] = L.ux[k]; uy[o] = L.uy[k]; uz[o] = L.uz[k];
    if (id) id[o] = L.id ? L.id[k] : 0u;
  }
}
// The loose-list entries of every species but s, appended to `out` (zpic_set_particles replaces
// species s: its loose particles go with its old tile contents).
__global__ void k_loose_drop_species(PList L, int s, PList out) {
  const int n = min(*L.count, L.cap);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    if (L.species[k] == s) continue;
    const int o = atomicAdd(out.count, 1);
    list_put(out, o, L.cell[k], L.x[k], L.y[k], L.ux[k], L.uy[k], L.uz[k], L.id ? L.id[k] : 0u, L.species[k]);
  }
}
void launch_loose_drop_species(const PList& L, int s, const PList& out, cudaStream_t st) {
  k_loose_drop_species<<<148 * 2, kBlock, 0, st>>>(L, s, out);
}
void launch_loose_extract(const PList& L, int s, int y0, int64_t out0, int32_t* ix, int32_t* iy, float* x, float* y,
                          float* ux, float* uy, float* uz, uint32_t* id, int* counter, cudaStream_t st) {
  k_loose_extract<<<148 * 2, kBlock, 0, st>>>(L, s, y0, ix + out0, iy + out0, x + out0, y + out0, ux + out0, uy + out0,
                                              uz + out0, id ? id + out0 : nullptr, counter);
}

void launch_mail_gather(const PushParams& p, cudaStream_t st) {
  const long warps = (long)p.ntx * p.nty * p.nspecies;
  k_mail_gather<<<(int)((warps * 32 + kBlock - 1) / kBlock), kBlock, 0, st>>>(p);
}
void launch_insert(const PushParams& p, int grid, cudaStream_t st) { k_insert<<<grid * 2, kBlock, 0, st>>>(p); }
void launch_loose(const PushParams& p, int grid, cudaStream_t st) { k_push_loose<<<grid, kBlock, 0, st>>>(p); }
void launch_assemble(float* J, const float* Jt, const GridDesc& g, int T, int ntx, int nty, cudaStream_t st) {
  dim3 grid((g.nx + 3 + kBlock - 1) / kBlock, (g.ny + 3 + K4R - 1) / K4R);
  switch (T) {
    case 8: k_assemble_j<8><<<grid, kBlock, 0, st>>>(J, Jt, g, ntx, nty); break;
    case 16: k_assemble_j<16><<<grid, kBlock, 0, st>>>(J, Jt, g, ntx, nty); break;
    case 32: k_assemble_j<32><<<grid, kBlock, 0, st>>>(J, Jt, g, ntx, nty); break;
  }
}
void launch_guard_x(float* F, const GridDesc& g, int mode, int keep, cudaStream_t st) {
  const int n = 3 * (g.ny + 3);
  k_guard_x<<<(n + 255) / 256, 256, 0, st>>>(F, g, mode, keep);
}
void launch_guard_y(float* F, const GridDesc& g, int mode, int keep, cudaStream_t st) {
  const int n = 3 * (g.nx + 3);
  k_guard_y<<<(n + 255) / 256, 256, 0, st>>>(F, g, mode, keep);
}
// K5 over tile rows [row_begin, row_end) (row_end < 0: to the last)
void launch_yee(const YeeParams& p, cudaStream_t st, int row_begin, int row_end) {
  static unsigned attr_set = 0;   // per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 32 || !((attr_set >> dev) & 1u)) {
    cudaFuncSetAttribute(k_yee, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)YeeBox::bytes);
    if (dev < 32) attr_set |= 1u << dev;
  }
  const int nty = (p.g.ny + kYeeTY - 1) / kYeeTY;
  if (row_end < 0 || row_end > nty) row_end = nty;
  if (row_end <= row_begin) return;
  YeeParams q = p;
  q.row0 = row_begin;
  dim3 grid((p.g.nx + kYeeTX - 1) / kYeeTX, row_end - row_begin);
  k_yee<<<grid, kBlock, YeeBox::bytes, st>>>(q);
}
int yee_tile_rows(const GridDesc& g) { return (g.ny + kYeeTY - 1) / kYeeTY; }
void launch_epilogue(double* ke_slots, double* fe_slots, double* energy, int nspecies, const double* ke_scale4,
                     int* mc, int* sic, int* soc, int* stats, int64_t* d_nmove, int shifted, cudaStream_t st) {
  k_epilogue<<<1, kBlock, 0, st>>>(ke_slots, fe_slots, energy, nspecies, ke_scale4, mc, sic, soc, stats, d_nmove,
                                   shifted);
}
void launch_inject(const InjectParams& q, int ntiles, cudaStream_t st) { k_inject<<<ntiles, kBlock, 0, st>>>(q); }
void launch_bin(const PStore& ps, int T, int ntx, int y0, long n, const int32_t* ix, const int32_t* iy, const float* x,
                const float* y, const float* ux, const float* uy, const float* uz, const uint32_t* id, int* err,
                const PList& loose, int s, cudaStream_t st, int nx, int ny, int* bad, long id0) {
  const int grid = (int)std::min<long>((n + kBlock - 1) / kBlock, 148L * 32);
  if (grid > 0)
    k_bin<<<grid, kBlock, 0, st>>>(ps, T, ntx, y0, n, ix, iy, x, y, ux, uy, uz, id, err, loose, s, nx, ny, bad, id0);
}
void launch_inject_column(const PushParams& p, int s, int px, int py, const int64_t* n_move, int ny_global, int y0, uint64_t key,
                          const double* ufl, const double* uth, cudaStream_t st) {
  const int n = p.g.ny * px * py;
  k_inject_column<<<(n + kBlock - 1) / kBlock, kBlock, 0, st>>>(p, s, px, py, n_move, ny_global, y0, key, ufl[0], ufl[1],
                                                                ufl[2], uth[0], uth[1], uth[2]);
}
void launch_filter_x(const float* Jin, float* Jout, const GridDesc& g, int npass, int compensated, int periodic,
                     cudaStream_t st) {
  const size_t smem = 2 * (size_t)(g.nx + 2) * sizeof(float);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(k_filter_x, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  const int total = npass + (compensated && npass > 0 ? 1 : 0);
  static const bool v1 = [] { const char* e = getenv("ZPIC_FILTER_V1"); return e && atoi(e); }();
  if (total <= kFiltR && !v1) {   // the register form (same result bit for bit)
    const long n = (long)((g.nx + kFiltCW - 1) / kFiltCW) * 3 * g.ny;
    const int grid = (int)((n + 255) / 256);
    if (total <= 2) k_filter_x_reg<2><<<grid, 256, 0, st>>>(Jin, Jout, g, npass, compensated, periodic);
    else if (total <= 5) k_filter_x_reg<5><<<grid, 256, 0, st>>>(Jin, Jout, g, npass, compensated, periodic);
    else k_filter_x_reg<kFiltR><<<grid, 256, 0, st>>>(Jin, Jout, g, npass, compensated, periodic);
    return;
  }
  k_filter_x<<<3 * g.ny, kBlock, smem, st>>>(Jin, Jout, g, npass, compensated, periodic);
}
void launch_apply_j_halo(float* J, const GridDesc& g, const float* rup, const float* rdn, int has_lo, int has_hi,
                         cudaStream_t st) {
  const int n = 3 * g.pitch;
  k_apply_j_halo<<<(n + kBlock - 1) / kBlock, kBlock, 0, st>>>(J, g, rup, rdn, has_lo, has_hi);
}
size_t particle_msg_bytes(int cap) { return msg_bytes(cap); }
PList particle_msg_list(void* buf, int cap) { return msg_list(buf, cap); }
void launch_recv_insert(const PushParams& p, const PList& lo, const PList& hi, cudaStream_t st) {
  k_recv_insert<<<148 * 2, kBlock, 0, st>>>(p, lo, hi);
}
void launch_count(int T, int ntx, int nx, int ny, int y0, long n, const int32_t* ix, const int32_t* iy, const float* x,
                  const float* y, int* counts, int* err, cudaStream_t st) {
  const int grid = (int)std::min<long>((n + kBlock - 1) / kBlock, 148L * 32);
  if (grid > 0) k_count<<<grid, kBlock, 0, st>>>(T, ntx, nx, ny, y0, n, ix, iy, x, y, counts, err);
}
void launch_export(const PStore& ps, int ntiles, const int64_t* prefix, int y0, int32_t* ix, int32_t* iy, float* x,
                   float* y, float* ux, float* uy, float* uz, uint32_t* id, cudaStream_t st) {
  k_export<<<ntiles, kBlock, 0, st>>>(ps, prefix, y0, ix, iy, x, y, ux, uy, uz, id);
}

}  // namespace zpic

namespace zpic {
// =============================================================================================
// Occupancy bound of the fixed-point tile current after a (re)load (PushParams::occ): one CTA per
// tile histograms the cells of every species' particles and takes the largest 4 x 4 window sum.
// mode 0 (after a (re)load): store the histogram (p.hist) and the occupancy bound (p.occ).
// mode 1 (ZPIC_CHECK_OCC, before K1s): verify that p.hist equals the recount and that p.occ bounds
// the recount's largest window; a violation sets ERR_HIST (the step returns ZPIC_E_STATE).
__global__ void __launch_bounds__(kBlock) k_occupancy(PushParams p, int mode) {
  __shared__ int h[32 * 32];
  __shared__ int s_max;
  const int t = blockIdx.x, T = p.T;
  const int tx = t % p.ntx, ty = t / p.ntx, i0 = tx * T, j0 = ty * T;
  const int tw = min(T, p.g.nx - i0), th = min(T, p.g.ny - j0);
  for (int k = threadIdx.x; k < T * T; k += blockDim.x) h[k] = 0;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  for (int s = 0; s < p.nspecies; ++s) {
    const PStore& ps = p.ps[s];
    const int n = min(ps.cnt[t], ps.cap);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const int c = (int)*ps.slot((long)t * ps.cap + k);
      const int lx = cell_ix(c) - i0, ly = cell_iy(c) - j0;
      if ((unsigned)lx < (unsigned)tw && (unsigned)ly < (unsigned)th) atomicAdd(&h[ly * T + lx], 1);
    }
  }
  __syncthreads();
  const int m = window_max_4x4(h, T, tw, th);
  atomicMax(&s_max, m);
  int* H = p.hist + (long)t * T * T;
  if (mode == 0) {
    for (int k = threadIdx.x; k < T * T; k += blockDim.x) H[k] = h[k];
  } else {
    for (int k = threadIdx.x; k < T * T; k += blockDim.x)
      if (H[k] != h[k]) atomicOr(p.err, ERR_HIST);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode == 0) p.occ[t] = s_max;
    else if (p.occ[t] < s_max) atomicOr(p.err, ERR_HIST);
  }
}
void launch_occupancy(const PushParams& p, cudaStream_t st, int mode) {
  k_occupancy<<<p.ntx * p.nty, kBlock, 0, st>>>(p, mode);
}

// K1s: every tile's fixed-point scale exponent for the K1 that follows: 2^S from a
// bound on |J| at any node of the tile's block.  Every particle adds at most |q_s| to any node
// (|v| < 1, the weights of its pieces sum to 1), and only the particles of a 4 x 4 cell window reach
// a node: |J_node| <= occ * max_s |q_s|, occ the tile's occupancy bound (else the tile count:
// sum_s n_s |q_s|).  The occupancy slot is reset here; K1 (its stayers' window maximum) and every
// insertion after it (K3m, K3, loose re-insertion, halo receive, window injection) rebuild it.
__global__ void k_tile_scale(PushParams p) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= p.ntx * p.nty) return;
  const int occ = p.occ[t];
  p.occ[t] = 0;
  double bound = 0.0;
  int ntot = 0;
  for (int s = 0; s < p.nspecies; ++s) {
    const int n = p.ps[s].cnt[t];
    bound += (double)n * fabs((double)p.sc[s].q);
    ntot += n;
  }
  int npart = ntot;
  if (occ >= 0 && occ < ntot) {
    bound = fmin(bound, (double)occ * (double)p.qmax);
    npart = occ;
  }
  p.tscale[t] = fx_scale_exponent(bound, npart);
}
void launch_tile_scale(const PushParams& p, cudaStream_t st) {
  k_tile_scale<<<(p.ntx * p.nty + kBlock - 1) / kBlock, kBlock, 0, st>>>(p);
}
}  // namespace zpic
