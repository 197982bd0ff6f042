// zpic_kernels.cuh — per-particle physics of the ZPIC em2d step as device functions, shared by
// the tile kernel (shared-memory fields and current) and the loose-particle kernel (global
// memory).  Every function cites the passage it implements; the readings are SURVEY.md §8(c).
#pragma once
#include "zpic_internal.h"

namespace zpic {

// ---- field accessors -----------------------------------------------------------------------
// Tile-staged fields: (Ex, By) share the (1/2, 0) stagger, (Ey, Bx) share (0, 1/2); Ez (0, 0),
// Bz (1/2, 1/2).  Arrays cover local cells [-1, T+1) in both axes, row width W = T + 2.
template <int W>   // row width (compile-time, so stencil offsets are immediates)
struct SmemFields {
  const float2* eb1;  // (Ex, By)
  const float2* eb2;  // (Ey, Bx)
  const float* ez;
  const float* bz;
  __device__ __forceinline__ int o(int lx, int ly) const { return (ly + 1) * W + (lx + 1); }
  __device__ __forceinline__ void hi(int i, int j, float wx, float wy, float& ex, float& by) const {
    float2 a = eb1[o(i, j)], b = eb1[o(i + 1, j)], c = eb1[o(i, j + 1)], d = eb1[o(i + 1, j + 1)];
    float l0 = fmaf(wx, b.x - a.x, a.x), l1 = fmaf(wx, d.x - c.x, c.x);
    ex = fmaf(wy, l1 - l0, l0);
    l0 = fmaf(wx, b.y - a.y, a.y); l1 = fmaf(wx, d.y - c.y, c.y);
    by = fmaf(wy, l1 - l0, l0);
  }
  __device__ __forceinline__ void ih(int i, int j, float wx, float wy, float& ey, float& bx) const {
    float2 a = eb2[o(i, j)], b = eb2[o(i + 1, j)], c = eb2[o(i, j + 1)], d = eb2[o(i + 1, j + 1)];
    float l0 = fmaf(wx, b.x - a.x, a.x), l1 = fmaf(wx, d.x - c.x, c.x);
    ey = fmaf(wy, l1 - l0, l0);
    l0 = fmaf(wx, b.y - a.y, a.y); l1 = fmaf(wx, d.y - c.y, c.y);
    bx = fmaf(wy, l1 - l0, l0);
  }
  __device__ __forceinline__ float one(const float* f, int i, int j, float wx, float wy) const {
    float a = f[o(i, j)], b = f[o(i + 1, j)], c = f[o(i, j + 1)], d = f[o(i + 1, j + 1)];
    float l0 = fmaf(wx, b - a, a), l1 = fmaf(wx, d - c, c);
    return fmaf(wy, l1 - l0, l0);
  }
  __device__ __forceinline__ float fez(int i, int j, float wx, float wy) const { return one(ez, i, j, wx, wy); }
  __device__ __forceinline__ float fbz(int i, int j, float wx, float wy) const { return one(bz, i, j, wx, wy); }
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
// Shared-memory tile current as exact fixed point: every contribution v (already scaled by
// kFxScale = 2^32, a power of two, so the scaling is exact) is rounded once to an int64
// V = rint(v), split V = hi * 2^15 + lo with 0 <= lo < 2^15, and both halves are added with
// native 32-bit shared-memory integer atomics (sm_100a has no native fp32 shared atomic add: it
// compiles to a CAS loop).  Integer sums are exact and order-independent, so the tile current
// is bit-reproducible; the only error is the 2^-33 rounding of each contribution.  Ranges:
// |sum v| < 2^14 per node; lo sums stay below 2^31 for < 21845 contributions per node (the tile
// capacity is capped accordingly, zpic_api.cu).  3 planes x 2 halves cover local nodes
// [-1, T+2), row width WJ = T + 3.
constexpr float kFxScale = 4294967296.0f;  // 2^32
constexpr double kFxInv = 2.3283064365386963e-10;  // 2^-32
// Accumulator interface: index(i, k) = the linear index of node (i, k) in a component plane;
// row() = the index step to (i, k+1); add(c, idx + offset, v).  The deposit computes one index
// per path piece and reaches the other three nodes by constant offsets.
template <int WJ>   // row width (compile-time)
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

// Villasenor-Buneman split of the path (x, y) -> (x + dxp, y + dyp) from local cell (lx, ly)
// into 1-3 straight pieces at the cell edges it crosses (at most one per axis),
// in time order; returns the piece count, the cell steps (di, dj) and the renormalised offset
// with the R6 rounding rule.  Branch-free: with the edge-crossing times tx, ty (2 = no
// crossing) sorted into t1 <= t2 (clamped to 1), the pieces are [0, t1] in the start cell,
// [t1, t2] in the cell across the first edge and [t2, 1] in the final cell; a crossed
// coordinate is pinned to the exact edge value.  Pieces beyond the count have zero length.
__device__ __forceinline__ int split_path(int lx, int ly, float& x, float& y, float dxp, float dyp, float qvz, Seg* s,
                                          int& di, int& dj) {
  const float x1 = x + dxp, y1 = y + dyp;
  di = (x1 >= 1.0f) - (x1 < 0.0f);
  dj = (y1 >= 1.0f) - (y1 < 0.0f);
  const float xb = di > 0 ? 1.0f : 0.0f, yb = dj > 0 ? 1.0f : 0.0f;
  const float tx = di ? __fdividef(xb - x, dxp) : 2.0f;
  const float ty = dj ? __fdividef(yb - y, dyp) : 2.0f;
  const bool xfirst = tx <= ty;
  const float t1 = fminf(fminf(tx, ty), 1.0f), t2 = fminf(fmaxf(tx, ty), 1.0f);
  // the path at t1 and t2 (start-cell offsets); the coordinate crossing an edge at that time is
  // pinned to the edge (t2 = 1 gives exactly x1, y1 since fma(1, d, x) = x + d)
  const bool both = di && dj;
  const float xa = (di && xfirst) ? xb : fmaf(t1, dxp, x);
  const float ya = (dj && !xfirst) ? yb : fmaf(t1, dyp, y);
  const float xc = (both && !xfirst) ? xb : fmaf(t2, dxp, x);
  const float yc = (both && xfirst) ? yb : fmaf(t2, dyp, y);
  const int c1x = xfirst ? di : 0, c1y = xfirst ? 0 : dj;   // cell across the first edge
  s[0] = Seg{lx, ly, x, y, xa, ya, qvz * t1};
  s[1] = Seg{lx + c1x, ly + c1y, xa - c1x, ya - c1y, xc - c1x, yc - c1y, qvz * (t2 - t1)};
  s[2] = Seg{lx + di, ly + dj, xc - di, yc - dj, x1 - di, y1 - dj, qvz * (1.0f - t2)};
  const int n = 1 + (di != 0) + (dj != 0);
  float xn = x1 - di, yn = y1 - dj;
  if (xn >= 1.0f) { xn = 0.0f; di += 1; }   // R6: only reachable when x1 < 0 rounds to 1
  if (yn >= 1.0f) { yn = 0.0f; dj += 1; }
  x = xn;
  y = yn;
  return n;
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
