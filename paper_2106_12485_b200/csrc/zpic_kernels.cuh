// zpic_kernels.cuh — per-particle physics of the ZPIC em2d step as device functions, shared by
// the tile kernel (shared-memory fields and current) and the loose-particle kernel (global
// memory).  Every function cites the passage it implements; the readings are SURVEY.md §8(c).
#pragma once
#include "zpic_internal.h"

namespace zpic {

// ---- field accessors -----------------------------------------------------------------------
// Tile-staged fields: (Ex, By) share the (1/2, 0) stagger, (Ey, Bx) share (0, 1/2); Ez (0, 0),
// Bz (1/2, 1/2).  Arrays cover local cells [-1, T+1) in both axes, row width W = T + 2.
// (Ex, By) is stored in pairs of nodes: entry o holds (Ex, By) of nodes o and o + 1 as one float4,
// so a stencil row is one LDS.128 instead of two LDS.64 (fewer shared-memory wavefronts when a
// warp's cells are scattered over the tile: -1.3 % K1 time in steady state, the same right after
// the injection).  Pairing (Ey, Bx) as well, or Ez / Bz, costs the 8th CTA per SM
// or gains nothing (profiles/r2_ab_pairs.log).
template <int W>   // row width (compile-time, so stencil offsets are immediates)
struct SmemFields {
  const float4* eb1;  // (Ex, By) of nodes o, o + 1
  const float2* eb2;  // (Ey, Bx)
  const float* ez;
  const float* bz;
  __device__ __forceinline__ int o(int lx, int ly) const { return (ly + 1) * W + (lx + 1); }
};

// Global-memory fields (loose particles): (i, j) are slab cell indices, guards valid.
struct GlobalFields {
  const float* E;
  const float* B;
  GridDesc g;
  __device__ __forceinline__ float one(const float* f, int i, int j, float wx, float wy) const {
    float a = __ldg(f + g.at(i, j)), b = __ldg(f + g.at(i + 1, j));
    float c = __ldg(f + g.at(i, j + 1)), d = __ldg(f + g.at(i + 1, j + 1));
    float l0 = fmaf(wx, b - a, a), l1 = fmaf(wx, d - c, c);
    return fmaf(wy, l1 - l0, l0);
  }
  __device__ __forceinline__ void hi(int i, int j, float wx, float wy, float& ex, float& by) const {
    ex = one(E, i, j, wx, wy);
    by = one(B + g.plane, i, j, wx, wy);
  }
  __device__ __forceinline__ void ih(int i, int j, float wx, float wy, float& ey, float& bx) const {
    ey = one(E + g.plane, i, j, wx, wy);
    bx = one(B, i, j, wx, wy);
  }
  __device__ __forceinline__ float fez(int i, int j, float wx, float wy) const { return one(E + 2 * g.plane, i, j, wx, wy); }
  __device__ __forceinline__ float fbz(int i, int j, float wx, float wy) const { return one(B + 2 * g.plane, i, j, wx, wy); }
};

// ---- current accumulators ----------------------------------------------------------------
// Shared-memory tile current as fixed point with one native 32-bit integer atomic per node
// (sm_100a has no native fp32 shared-memory atomic add: it compiles to a CAS loop).  Every
// contribution v is pre-scaled by the CTA's power of two 2^S (exact) and rounded once to an
// int32; the integer sums are exact and order-independent, so the tile current is
// bit-reproducible, and the only error is the rounding of each contribution to 2^-(S+1).
// S is chosen per CTA from a bound on |J| (fx_scale_exponent): every particle adds at most |q|
// in absolute value to any node of any component (|v| < 1 and the pieces' weights sum to 1), so
// |sum| <= sum_s n_s |q_s| over the tile's particles.  3 planes cover local nodes [-1, T+2),
// row width WJ = T + 3.
// Accumulator interface: index(i, k) = the linear index of node (i, k) in a component plane;
// row() = the index step to (i, k+1); add(c, idx + offset, v).  The deposit computes one index
// per path piece and reaches the other three nodes by constant offsets.
template <int WJ>   // row width (compile-time)
struct SmemCurrentI32 {
  int* j;
  __device__ __forceinline__ int index(int i, int k) const { return (k + 1) * WJ + (i + 1); }
  __device__ __forceinline__ int row() const { return WJ; }
  __device__ __forceinline__ void add(int c, int o, float v) const { atomicAdd(j + c * WJ * WJ + o, __float2int_rn(v)); }
};
// The exact two-word form, used for tiles whose bound would leave S < kSMin (dense tiles): every
// contribution is scaled by 2^32 and rounded once to an int64 V, split V = hi * 2^15 + lo with
// 0 <= lo < 2^15, and both halves are added with 32-bit atomics (|sum| < 2^14 per node, lo sums
// below 2^31 for < 21845 contributions per node).  Per contribution the error is <= 2^-33.
constexpr float kFxScale = 4294967296.0f;          // 2^32
constexpr double kFxInv = 2.3283064365386963e-10;  // 2^-32
template <int WJ>
struct SmemCurrentFx {
  int* hi;
  int* lo;
  __device__ __forceinline__ int index(int i, int k) const { return (k + 1) * WJ + (i + 1); }
  __device__ __forceinline__ int row() const { return WJ; }
  __device__ __forceinline__ void add(int c, int o, float v) const {
    const long long V = __float2ll_rn(v);
    atomicAdd(hi + c * WJ * WJ + o, (int)(V >> 15));
    atomicAdd(lo + c * WJ * WJ + o, (int)(V & 0x7fff));
  }
};
// Largest S such that bound * 2^S plus the rounding of up to 3 * npart contributions per node
// stays below 2^31 (bound = sum_s n_s |q_s|); 32 for an empty tile.
__device__ __forceinline__ int fx_scale_exponent(double bound, int npart) {
  if (!(bound > 0.0)) return 32;
  int e;
  frexp((2147483648.0 - 2.0 * npart - 1024.0) / bound, &e);   // ratio = m 2^e, m in [0.5, 1)
  return min(e - 1, 40);
}
struct GlobalCurrent {
  float* J;
  GridDesc g;
  __device__ __forceinline__ long index(int i, int k) const { return g.at(i, k); }
  __device__ __forceinline__ long row() const { return g.pitch; }
  __device__ __forceinline__ void add(int c, long o, float v) const { atomicAdd(J + c * g.plane + o, v); }
};

// ---- (1) interpolation, PAPER.md:144 -------------------------------------------------------
// Bilinear weights with the Yee staggering: for a half-staggered axis the stencil starts one
// cell lower when the offset is below 1/2.
template <class F>
__device__ __forceinline__ void interpolate(const F& f, int lx, int ly, float x, float y, float& ex, float& ey,
                                            float& ez, float& bx, float& by, float& bz) {
  const bool xl = x < 0.5f, yl = y < 0.5f;
  const int ih = xl ? lx - 1 : lx, jh = yl ? ly - 1 : ly;
  const float wxh = xl ? x + 0.5f : x - 0.5f, wyh = yl ? y + 0.5f : y - 0.5f;
  f.hi(ih, ly, wxh, y, ex, by);
  f.ih(lx, jh, x, wyh, ey, bx);
  ez = f.fez(lx, ly, x, y);
  bz = f.fbz(ih, jh, wxh, wyh);
}

// Packed fp32x2 form for the shared-memory tile (sm_100a FFMA2: two lanes of fp32 per
// instruction): the pairs (Ex, By), (Ey, Bx) share their stencil and weights, and (Ez, Bz) pair
// two stencils with per-lane weights.  Each lerp is fma(w, b - a, a) with b - a = fma(a, -1, b),
// the same roundings as the scalar form.
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 w) {
  const float2 d = __ffma2_rn(a, make_float2(-1.0f, -1.0f), b);
  return __ffma2_rn(w, d, a);
}
template <int W>
__device__ __forceinline__ void interpolate(const SmemFields<W>& f, int lx, int ly, float x, float y, float& ex,
                                            float& ey, float& ez, float& bx, float& by, float& bz) {
  const bool xl = x < 0.5f, yl = y < 0.5f;
  const int ih = xl ? lx - 1 : lx, jh = yl ? ly - 1 : ly;
  const float wxh = xl ? x + 0.5f : x - 0.5f, wyh = yl ? y + 0.5f : y - 0.5f;
  const int oa = f.o(ih, ly), ob = f.o(lx, jh), oz = f.o(lx, ly), oh = f.o(ih, jh);
  // (Ex, By) at (ih, ly) with weights (wxh, y)
  const float4 q0 = f.eb1[oa], q1 = f.eb1[oa + W];
  float2 l0 = lerp2(make_float2(q0.x, q0.y), make_float2(q0.z, q0.w), make_float2(wxh, wxh));
  float2 l1 = lerp2(make_float2(q1.x, q1.y), make_float2(q1.z, q1.w), make_float2(wxh, wxh));
  const float2 r1 = lerp2(l0, l1, make_float2(y, y));
  // (Ey, Bx) at (lx, jh) with weights (x, wyh)
  l0 = lerp2(f.eb2[ob], f.eb2[ob + 1], make_float2(x, x));
  l1 = lerp2(f.eb2[ob + W], f.eb2[ob + W + 1], make_float2(x, x));
  const float2 r2 = lerp2(l0, l1, make_float2(wyh, wyh));
  // (Ez at (lx, ly) weights (x, y), Bz at (ih, jh) weights (wxh, wyh))
  const float2 wx = make_float2(x, wxh), wy = make_float2(y, wyh);
  l0 = lerp2(make_float2(f.ez[oz], f.bz[oh]), make_float2(f.ez[oz + 1], f.bz[oh + 1]), wx);
  l1 = lerp2(make_float2(f.ez[oz + W], f.bz[oh + W]), make_float2(f.ez[oz + W + 1], f.bz[oh + W + 1]), wx);
  const float2 r3 = lerp2(l0, l1, wy);
  ex = r1.x; by = r1.y;
  ey = r2.x; bx = r2.y;
  ez = r3.x; bz = r3.y;
}

// ---- (2) relativistic Boris, PAPER.md:144-145 -------------------------------------------------
// Returns |u-|^2 / (1 + gamma-) for the kinetic energy at time n (R8).
__device__ __forceinline__ float boris(float& ux, float& uy, float& uz, float ex, float ey, float ez, float bx,
                                       float by, float bz, float h) {
  const float umx = fmaf(h, ex, ux), umy = fmaf(h, ey, uy), umz = fmaf(h, ez, uz);
  const float u2 = fmaf(umx, umx, fmaf(umy, umy, umz * umz));
  const float rg = rsqrtf(1.0f + u2);
  const float gm = (1.0f + u2) * rg;
  const float ke = __fdividef(u2, 1.0f + gm);
  const float tx = h * bx * rg, ty = h * by * rg, tz = h * bz * rg;
  const float upx = umx + (umy * tz - umz * ty);
  const float upy = umy + (umz * tx - umx * tz);
  const float upz = umz + (umx * ty - umy * tx);
  const float s = __fdividef(2.0f, 1.0f + fmaf(tx, tx, fmaf(ty, ty, tz * tz)));
  const float sx = s * tx, sy = s * ty, sz = s * tz;
  ux = fmaf(h, ex, umx + (upy * sz - upz * sy));
  uy = fmaf(h, ey, umy + (upz * sx - upx * sz));
  uz = fmaf(h, ez, umz + (upx * sy - upy * sx));
  return ke;
}

// ---- (3) charge-conserving deposit, PAPER.md:146 ---------------------------------------------
// One straight sub-segment of a particle path: local cell (cx, cy), offsets (a0,b0)->(a1,b1),
// and wz = q vz f (the z-current weight of the piece).
struct Seg {
  int cx, cy;
  float a0, b0, a1, b1, wz;
};

// Cell-edge crossings of the straight path (x, y) -> (x1, y1) = (x + dxp, y + dyp) from the
// start cell (at most one per axis, Villasenor-Buneman).  Branch-free: with the
// edge-crossing times tx, ty (2 = no crossing) sorted into t1 <= t2 (clamped to 1), the pieces
// are [0, t1] in the start cell, [t1, t2] in the cell across the first edge and [t2, 1] in the
// final cell; a crossed coordinate is pinned to the exact edge value (t = 1 gives exactly x1, y1
// since fma(1, d, x) = x + d).  The same inline arithmetic runs for the first piece in the main
// loop and for the later pieces in the queue drain, so the pieces chain bit-exactly.
struct Crossing {
  int di, dj;              // cell steps of the end point (before the R6 rule)
  bool xfirst;             // the x edge is crossed first (or together)
  float t1, t2;            // piece boundaries in path time
  float xa, ya, xc, yc;    // path points at t1, t2 (start-cell offsets)
};
__device__ __forceinline__ Crossing path_crossings(float x, float y, float dxp, float dyp, float x1, float y1) {
  Crossing c;
  c.di = (x1 >= 1.0f) - (x1 < 0.0f);
  c.dj = (y1 >= 1.0f) - (y1 < 0.0f);
  const float xb = c.di > 0 ? 1.0f : 0.0f, yb = c.dj > 0 ? 1.0f : 0.0f;
  const float tx = c.di ? __fdividef(xb - x, dxp) : 2.0f;
  const float ty = c.dj ? __fdividef(yb - y, dyp) : 2.0f;
  c.xfirst = tx <= ty;
  c.t1 = fminf(fminf(tx, ty), 1.0f);
  c.t2 = fminf(fmaxf(tx, ty), 1.0f);
  const bool both = c.di && c.dj;
  c.xa = (c.di && c.xfirst) ? xb : fmaf(c.t1, dxp, x);
  c.ya = (c.dj && !c.xfirst) ? yb : fmaf(c.t1, dyp, y);
  c.xc = (both && !c.xfirst) ? xb : fmaf(c.t2, dxp, x);
  c.yc = (both && c.xfirst) ? yb : fmaf(c.t2, dyp, y);
  return c;
}

// The pieces after the first (only for a path that crosses an edge): [t1, t2] in the cell across
// the first edge, and [t2, 1] in the final cell (zero length unless both edges are crossed).
__device__ __forceinline__ void later_pieces(int lx, int ly, float x1, float y1, float qvz, const Crossing& c, Seg& s1,
                                             Seg& s2) {
  const int c1x = c.xfirst ? c.di : 0, c1y = c.xfirst ? 0 : c.dj;   // cell across the first edge
  s1 = Seg{lx + c1x, ly + c1y, c.xa - c1x, c.ya - c1y, c.xc - c1x, c.yc - c1y, qvz * (c.t2 - c.t1)};
  s2 = Seg{lx + c.di, ly + c.dj, c.xc - c.di, c.yc - c.dj, x1 - c.di, y1 - c.dj, qvz * (1.0f - c.t2)};
}

// Renormalised end offset with the R6 rounding rule (an offset that renormalises to exactly 1
// becomes 0 in the next cell; only reachable when x1 < 0 rounds to 1).
__device__ __forceinline__ void renormalise(float x1, float y1, int& di, int& dj, float& x, float& y) {
  float xn = x1 - di, yn = y1 - dj;
  if (xn >= 1.0f) { xn = 0.0f; di += 1; }
  if (yn >= 1.0f) { yn = 0.0f; dj += 1; }
  x = xn;
  y = yn;
}

// The whole split (1-3 pieces in time order) for the loose-particle kernel.
__device__ __forceinline__ int split_path(int lx, int ly, float& x, float& y, float dxp, float dyp, float qvz, Seg* s,
                                          int& di, int& dj) {
  const float x1 = x + dxp, y1 = y + dyp;
  const Crossing c = path_crossings(x, y, dxp, dyp, x1, y1);
  s[0] = Seg{lx, ly, x, y, c.xa, c.ya, qvz * c.t1};
  later_pieces(lx, ly, x1, y1, qvz, c, s[1], s[2]);
  di = c.di;
  dj = c.dj;
  renormalise(x1, y1, di, dj, x, y);
  return 1 + (c.di != 0) + (c.dj != 0);
}

template <class A>
__device__ __forceinline__ void deposit_seg(const A& acc, const Seg& s, float jxs, float jys) {
  const float da = s.a1 - s.a0, db = s.b1 - s.b0;
  const float xm = 0.5f * (s.a0 + s.a1), ym = 0.5f * (s.b0 + s.b1);
  const float wx = jxs * da, wy = jys * db;
  const auto o = acc.index(s.cx, s.cy);
  const auto r = acc.row();
  acc.add(0, o, wx * (1.0f - ym));
  acc.add(0, o + r, wx * ym);
  acc.add(1, o, wy * (1.0f - xm));
  acc.add(1, o + 1, wy * xm);
  const float c = da * db * (1.0f / 12.0f);
  acc.add(2, o, s.wz * fmaf(1.0f - xm, 1.0f - ym, c));
  acc.add(2, o + 1, s.wz * fmaf(xm, 1.0f - ym, -c));
  acc.add(2, o + r, s.wz * fmaf(1.0f - xm, ym, -c));
  acc.add(2, o + r + 1, s.wz * fmaf(xm, ym, c));
}

}  // namespace zpic
