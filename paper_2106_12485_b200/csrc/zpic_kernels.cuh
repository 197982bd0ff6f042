// zpic_kernels.cuh — per-particle physics of the ZPIC em2d step as device functions, shared by
// the tile kernel (shared-memory fields and current) and the loose-particle kernel (global
// memory).  Every function cites the passage it implements; the readings are SURVEY.md §8(c).
#pragma once
#include "zpic_internal.h"

namespace zpic {

// ---- field accessors -----------------------------------------------------------------------
// Tile-staged fields: (Ex, By) share the (1/2, 0) stagger, (Ey, Bx) share (0, 1/2); Ez (0, 0),
// Bz (1/2, 1/2).  Arrays cover local cells [-1, T+1) in both axes, row width W = T + 2.
struct SmemFields {
  const float2* eb1;  // (Ex, By)
  const float2* eb2;  // (Ey, Bx)
  const float* ez;
  const float* bz;
  int W;
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
// Shared-memory tile current: 3 planes covering local nodes [-1, T+2), row width WJ = T + 3.
struct SmemCurrent {
  float* j;
  int WJ;
  __device__ __forceinline__ void add(int c, int i, int k, float v) const {
    atomicAdd(j + c * WJ * WJ + (k + 1) * WJ + (i + 1), v);
  }
};
struct GlobalCurrent {
  float* J;
  GridDesc g;
  __device__ __forceinline__ void add(int c, int i, int k, float v) const { atomicAdd(J + c * g.plane + g.at(i, k), v); }
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

// ---- (3) charge-conserving deposit of one straight sub-segment, PAPER.md:146 ------------------
// Segment in local cell (cx, cy) from (a0, b0) to (a1, b1) (cell offsets), covering fraction f
// of the step.  Jx, Jy: the charge flux through the dual-cell faces (Villasenor-Buneman);
// Jz: q vz f times the exact path average of the bilinear weight,
//   W_ij = Sbar_x,i Sbar_y,j + dS_x,i dS_y,j / 12   (Sbar = mid-point weight, dS = +-(end-start)).
template <class A>
__device__ __forceinline__ void deposit_segment(const A& acc, int cx, int cy, float a0, float b0, float a1, float b1,
                                                float f, float jxs, float jys, float qvz) {
  const float da = a1 - a0, db = b1 - b0;
  const float xm = 0.5f * (a0 + a1), ym = 0.5f * (b0 + b1);
  const float wx = jxs * da, wy = jys * db;
  acc.add(0, cx, cy, wx * (1.0f - ym));
  acc.add(0, cx, cy + 1, wx * ym);
  acc.add(1, cx, cy, wy * (1.0f - xm));
  acc.add(1, cx + 1, cy, wy * xm);
  const float w = qvz * f, c = da * db * (1.0f / 12.0f);
  acc.add(2, cx, cy, w * fmaf(1.0f - xm, 1.0f - ym, c));
  acc.add(2, cx + 1, cy, w * fmaf(xm, 1.0f - ym, -c));
  acc.add(2, cx, cy + 1, w * fmaf(1.0f - xm, ym, -c));
  acc.add(2, cx + 1, cy + 1, w * fmaf(xm, ym, c));
}

// Position advance by (dxp, dyp) cells from local cell (lx, ly), offset (x, y): split the
// straight path at the cell edges it crosses (at most one per axis), deposit
// every piece, and return the new offset and the cell steps (di, dj) with the R6 rounding
// rule (an offset that rounds to 1 after renormalisation becomes 0 in the next cell).
template <class A>
__device__ __forceinline__ void advance_deposit(const A& acc, int lx, int ly, float& x, float& y, float dxp, float dyp,
                                                float jxs, float jys, float qvz, int& di, int& dj) {
  const float x1 = x + dxp, y1 = y + dyp;
  di = (x1 >= 1.0f) - (x1 < 0.0f);
  dj = (y1 >= 1.0f) - (y1 < 0.0f);
  if ((di | dj) == 0) {
    deposit_segment(acc, lx, ly, x, y, x1, y1, 1.0f, jxs, jys, qvz);
  } else if (dj == 0) {
    const float xb = di > 0 ? 1.0f : 0.0f;
    const float t = (xb - x) / dxp;
    const float yb = fmaf(t, dyp, y);
    deposit_segment(acc, lx, ly, x, y, xb, yb, t, jxs, jys, qvz);
    deposit_segment(acc, lx + di, ly, xb - di, yb, x1 - di, y1, 1.0f - t, jxs, jys, qvz);
  } else if (di == 0) {
    const float yb = dj > 0 ? 1.0f : 0.0f;
    const float t = (yb - y) / dyp;
    const float xb = fmaf(t, dxp, x);
    deposit_segment(acc, lx, ly, x, y, xb, yb, t, jxs, jys, qvz);
    deposit_segment(acc, lx, ly + dj, xb, yb - dj, x1, y1 - dj, 1.0f - t, jxs, jys, qvz);
  } else {
    const float xb = di > 0 ? 1.0f : 0.0f, yb = dj > 0 ? 1.0f : 0.0f;
    const float tx = (xb - x) / dxp, ty = (yb - y) / dyp;
    if (tx <= ty) {  // x edge first
      const float yx = fmaf(tx, dyp, y), xy = fmaf(ty, dxp, x);
      deposit_segment(acc, lx, ly, x, y, xb, yx, tx, jxs, jys, qvz);
      deposit_segment(acc, lx + di, ly, xb - di, yx, xy - di, yb, ty - tx, jxs, jys, qvz);
      deposit_segment(acc, lx + di, ly + dj, xy - di, yb - dj, x1 - di, y1 - dj, 1.0f - ty, jxs, jys, qvz);
    } else {         // y edge first
      const float xy = fmaf(ty, dxp, x), yx = fmaf(tx, dyp, y);
      deposit_segment(acc, lx, ly, x, y, xy, yb, ty, jxs, jys, qvz);
      deposit_segment(acc, lx, ly + dj, xy, yb - dj, xb, yx - dj, tx - ty, jxs, jys, qvz);
      deposit_segment(acc, lx + di, ly + dj, xb - di, yx - dj, x1 - di, y1 - dj, 1.0f - tx, jxs, jys, qvz);
    }
  }
  float xn = x1 - di, yn = y1 - dj;
  if (xn >= 1.0f) { xn = 0.0f; di += 1; }   // R6: only reachable when x1 < 0 rounds to 1
  if (yn >= 1.0f) { yn = 0.0f; dj += 1; }
  x = xn;
  y = yn;
}

}  // namespace zpic
