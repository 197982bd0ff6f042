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

__device__ __forceinline__ int pack_cell(int ix, int iy) { return (ix & 0xffff) | (iy << 16); }
__device__ __forceinline__ int cell_ix(int c) { return c & 0xffff; }
__device__ __forceinline__ int cell_iy(int c) { return c >> 16; }

// Apply the particle boundary conditions to a new cell (a5).  Returns false if the particle
// leaves the domain through an open / window edge (removed).
__device__ __forceinline__ bool domain_bc(int& ix, int& iy, const GridDesc& g, int bcx, int bcy) {
  if (ix < 0 || ix >= g.nx) {
    if (bcx != ZPIC_BC_PERIODIC) return false;
    ix += ix < 0 ? g.nx : -g.nx;
  }
  if (iy < 0 || iy >= g.ny) {
    if (bcy != ZPIC_BC_PERIODIC) return false;
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

// Insert one particle into its tile's slack, else into the loose list.
__device__ __forceinline__ void insert_particle(const PushParams& p, int s, int ix, int iy, float x, float y, float ux,
                                                float uy, float uz, uint32_t id) {
  const int t = (iy / p.T) * p.ntx + (ix / p.T);
  const PStore& ps = p.ps[s];
  const int slot = atomicAdd(ps.cnt + t, 1);
  const int cell = pack_cell(ix, iy);
  if (slot < ps.cap) {
    const long k = (long)t * ps.cap + slot;
    ps.cell[k] = cell; ps.x[k] = x; ps.y[k] = y; ps.ux[k] = ux; ps.uy[k] = uy; ps.uz[k] = uz;
    if (ps.id) ps.id[k] = id;
  } else {
    atomicSub(ps.cnt + t, 1);
    const int k = atomicAdd(p.spill_out.count, 1);
    if (k < p.spill_out.cap) list_put(p.spill_out, k, cell, x, y, ux, uy, uz, id, s);
    else atomicOr(p.err, ERR_OVERFLOW);
  }
}

}  // namespace zpic
