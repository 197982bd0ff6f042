/*
 * zpic_oracle.c — TEST INFRASTRUCTURE ONLY.  The plain, serial, fp64 CPU oracle of the
 * ZPIC em2d time step (arxiv 2106.12485).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code, header,
 * table or constant with the CUDA path in paper_2106_12485_b200/.
 *
 * What it computes (Fig. 1 "main stages"):
 *   (1) field interpolation "bi-linear interpolation with the field values from the
 *       previous iteration"               -> orc_interpolate
 *   (2) particle advance, leapfrog + Boris -> orc_boris
 *   (3) current deposition, "exact charge conserving method" [Villasenor-Buneman]
 *       (BASELINE.json north_star "trajectory split at cell crossings")
 *                                                        -> orc_advance_deposit
 *       plus the optional digital filter   -> orc_filter_x
 *   (4) FDTD field advance on a Yee mesh   -> orc_yee_advance
 *   ghost-current reduction / ghost-field update -> orc_fold_current,
 *   orc_refresh_guards.
 * Readings of what the paper leaves open are SURVEY.md §8(c) R1-R25, listed in DESIGN.md.
 *
 * Storage: every grid quantity is fp64, three components, each (ny+3) x (nx+3) with guard
 * cells 1 low / 2 high per axis (R7); interior cell (i,j) is at
 * [(j+1)*(nx+3) + (i+1)].  Yee staggering (D3): Ex(i+1/2,j) Ey(i,j+1/2) Ez(i,j)
 * Bx(i,j+1/2) By(i+1/2,j) Bz(i+1/2,j+1/2).  Lengths in cells for particle offsets; physical
 * lengths dx, dy; c = 1.
 *
 * Build: gcc -O2 -fPIC -shared -o liborc.so zpic_oracle.c -lm   (no -ffast-math: the oracle
 * must evaluate exactly the written expressions).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define BC_PERIODIC 0
#define BC_OPEN 1          /* particles removed + Mur-1 tangential E (R13) */
#define BC_WINDOW 2        /* moving window along x: zero guards (R14) */

/* flat index of component c, interior cell (i,j), guard-extended (-1 <= i <= nx+1) */
static inline long fidx(int nx, int ny, int c, int i, int j) {
  return (long)c * (ny + 3) * (nx + 3) + (long)(j + 1) * (nx + 3) + (i + 1);
}

/* ------------------------------------------------------------------------------------ */
/* (1) Field interpolation; SURVEY §8(c) step 2.1.
 * For a component with stagger (sx, sy) in {0, 1/2}: px = ix + x - sx, i0 = floor(px),
 * wx = px - i0 (same in y) and F_p = sum_{a,b} (a ? wx : 1-wx)(b ? wy : 1-wy) F[i0+a, j0+b]. */
static const double STAG_X[6] = {0.5, 0.0, 0.0, /* Ex Ey Ez */ 0.0, 0.5, 0.5 /* Bx By Bz */};
static const double STAG_Y[6] = {0.0, 0.5, 0.0, /* Ex Ey Ez */ 0.5, 0.0, 0.5 /* Bx By Bz */};

static double interp_one(const double* F, int nx, int ny, int c, double gx, double gy,
                         double sx, double sy) {
  double px = gx - sx, py = gy - sy;
  double fi = floor(px), fj = floor(py);
  int i0 = (int)fi, j0 = (int)fj;
  double wx = px - fi, wy = py - fj;
  return (1.0 - wx) * (1.0 - wy) * F[fidx(nx, ny, c, i0, j0)]
       + wx * (1.0 - wy) * F[fidx(nx, ny, c, i0 + 1, j0)]
       + (1.0 - wx) * wy * F[fidx(nx, ny, c, i0, j0 + 1)]
       + wx * wy * F[fidx(nx, ny, c, i0 + 1, j0 + 1)];
}

/* Ep, Bp: np x 3 outputs. */
void orc_interpolate(const double* E, const double* B, int nx, int ny, long np,
                     const int32_t* ix, const int32_t* iy, const double* x, const double* y,
                     double* Ep, double* Bp) {
  for (long p = 0; p < np; ++p) {
    double gx = (double)ix[p] + x[p], gy = (double)iy[p] + y[p];
    for (int c = 0; c < 3; ++c) {
      Ep[3 * p + c] = interp_one(E, nx, ny, c, gx, gy, STAG_X[c], STAG_Y[c]);
      Bp[3 * p + c] = interp_one(B, nx, ny, c, gx, gy, STAG_X[3 + c], STAG_Y[3 + c]);
    }
  }
}

/* ------------------------------------------------------------------------------------ */
/* (2) Particle advance, relativistic Boris.
 * h = dt/(2 m_q); u- = u + h E; g- = sqrt(1+|u-|^2); t = h B / g-; u' = u- + u- x t;
 * s = 2 t/(1+|t|^2); u+ = u- + u' x s; u(n+1/2) = u+ + h E.
 * ke_sum += |u-|^2/(1+g-)  (= g- - 1 without cancellation; R8). u updated in place. */
void orc_boris(long np, double* ux, double* uy, double* uz, const double* Ep, const double* Bp,
               double m_q, double dt, double* ke_sum) {
  double h = 0.5 * dt / m_q;
  double ke = 0.0;
  for (long p = 0; p < np; ++p) {
    double umx = ux[p] + h * Ep[3 * p + 0];
    double umy = uy[p] + h * Ep[3 * p + 1];
    double umz = uz[p] + h * Ep[3 * p + 2];
    double u2 = umx * umx + umy * umy + umz * umz;
    double gm = sqrt(1.0 + u2);
    ke += u2 / (1.0 + gm);
    double tx = h * Bp[3 * p + 0] / gm;
    double ty = h * Bp[3 * p + 1] / gm;
    double tz = h * Bp[3 * p + 2] / gm;
    double upx = umx + (umy * tz - umz * ty);
    double upy = umy + (umz * tx - umx * tz);
    double upz = umz + (umx * ty - umy * tx);
    double t2 = tx * tx + ty * ty + tz * tz;
    double sx = 2.0 * tx / (1.0 + t2), sy = 2.0 * ty / (1.0 + t2), sz = 2.0 * tz / (1.0 + t2);
    double uplx = umx + (upy * sz - upz * sy);
    double uply = umy + (upz * sx - upx * sz);
    double uplz = umz + (upx * sy - upy * sx);
    ux[p] = uplx + h * Ep[3 * p + 0];
    uy[p] = uply + h * Ep[3 * p + 1];
    uz[p] = uplz + h * Ep[3 * p + 2];
  }
  *ke_sum += ke;
}

/* ------------------------------------------------------------------------------------ */
/* (3) Charge-conserving deposit of one straight sub-segment lying in cell (cx, cy), from
 * local (a0,b0) to (a1,b1), covering fraction f of the time step (SURVEY §8(c) step 2.4,
 * R4, R5):
 *   Jx[cx,cy]   += q (a1-a0)(1-ym) dx/dt     Jx[cx,cy+1] += q (a1-a0) ym dx/dt
 *   Jy[cx,cy]   += q (b1-b0)(1-xm) dy/dt     Jy[cx+1,cy] += q (b1-b0) xm dy/dt
 *   Jz[cx+i,cy+j] += q vz f W_ij,
 *   W_ij = (S0x_i S0y_j + S1x_i S1y_j)/3 + (S0x_i S1y_j + S1x_i S0y_j)/6,
 * S0x = (1-a0, a0), S1x = (1-a1, a1), S0y = (1-b0, b0), S1y = (1-b1, b1).             */
static void deposit_segment(double* J, int nx, int ny, int cx, int cy, double a0, double b0,
                            double a1, double b1, double f, double q, double vz, double dx,
                            double dy, double dt) {
  double xm = 0.5 * (a0 + a1), ym = 0.5 * (b0 + b1);
  double jx = q * (a1 - a0) * dx / dt;
  double jy = q * (b1 - b0) * dy / dt;
  J[fidx(nx, ny, 0, cx, cy)] += jx * (1.0 - ym);
  J[fidx(nx, ny, 0, cx, cy + 1)] += jx * ym;
  J[fidx(nx, ny, 1, cx, cy)] += jy * (1.0 - xm);
  J[fidx(nx, ny, 1, cx + 1, cy)] += jy * xm;
  double S0x[2] = {1.0 - a0, a0}, S1x[2] = {1.0 - a1, a1};
  double S0y[2] = {1.0 - b0, b0}, S1y[2] = {1.0 - b1, b1};
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      double W = (S0x[i] * S0y[j] + S1x[i] * S1y[j]) / 3.0 + (S0x[i] * S1y[j] + S1x[i] * S0y[j]) / 6.0;
      J[fidx(nx, ny, 2, cx + i, cy + j)] += q * vz * f * W;
    }
}

/* Position advance + Villasenor-Buneman split + deposit + cell update, for one species
 * (SURVEY §8(c) steps 2.3-2.5).  u must already be u^{n+1/2}.  Displacement in cells:
 * Dx = (ux/g) dt/dx, Dy = (uy/g) dt/dy, vz = uz/g.  The straight path is split first at
 * the x cell edge, then each piece at the y edge (at most one crossing per axis, <= 3
 * sub-segments; "a particle can only move to a neighbor cell").
 * Cell update: x1 = x+Dx; di = [x1>=1]-[x1<0]; x1 -= di; if x1 == 1 then x1 = 0, di += 1
 * (R6); same in y.  Returns the number of particles with |D| >= 1 (MIGRATION error).
 * ix, iy are NOT wrapped here (boundary handling is a separate stage, a5). */
long orc_advance_deposit(long np, int32_t* ix, int32_t* iy, double* x, double* y,
                         const double* ux, const double* uy, const double* uz, double q,
                         double dt, double dx, double dy, double* J, int nx, int ny) {
  long bad = 0;
  for (long p = 0; p < np; ++p) {
    double g = sqrt(1.0 + ux[p] * ux[p] + uy[p] * uy[p] + uz[p] * uz[p]);
    double Dx = ux[p] / g * dt / dx;
    double Dy = uy[p] / g * dt / dy;
    double vz = uz[p] / g;
    if (fabs(Dx) >= 1.0 || fabs(Dy) >= 1.0) ++bad;
    double x0 = x[p], y0 = y[p];
    double x1 = x0 + Dx, y1 = y0 + Dy;
    int di = (x1 >= 1.0) - (x1 < 0.0);
    int dj = (y1 >= 1.0) - (y1 < 0.0);
    int cx0 = ix[p], cy0 = iy[p];

    /* split along x: pieces (cxo, a0,b0, a1,b1, ta,tb), b relative to the start row */
    double sa0[2], sb0[2], sa1[2], sb1[2], sta[2], stb[2];
    int scx[2], nxs;
    if (di == 0) {
      scx[0] = 0; sa0[0] = x0; sb0[0] = y0; sa1[0] = x1; sb1[0] = y1; sta[0] = 0.0; stb[0] = 1.0;
      nxs = 1;
    } else {
      double xb = (di > 0) ? 1.0 : 0.0;
      double t = (xb - x0) / Dx;
      double yb = y0 + t * Dy;
      scx[0] = 0;  sa0[0] = x0;      sb0[0] = y0; sa1[0] = xb;      sb1[0] = yb; sta[0] = 0.0; stb[0] = t;
      scx[1] = di; sa0[1] = xb - di; sb0[1] = yb; sa1[1] = x1 - di; sb1[1] = y1; sta[1] = t;   stb[1] = 1.0;
      nxs = 2;
    }
    /* split each x-piece along y */
    int cy = 0;
    for (int s = 0; s < nxs; ++s) {
      double b0r = sb0[s] - cy, b1r = sb1[s] - cy;
      if (cy == 0 && dj != 0 && (b1r >= 1.0 || b1r < 0.0)) {
        double yb = (dj > 0) ? 1.0 : 0.0;
        double tp = (yb - b0r) / (b1r - b0r);
        double am = sa0[s] + tp * (sa1[s] - sa0[s]);
        double tm = sta[s] + tp * (stb[s] - sta[s]);
        deposit_segment(J, nx, ny, cx0 + scx[s], cy0, sa0[s], b0r, am, yb, tm - sta[s], q, vz, dx, dy, dt);
        deposit_segment(J, nx, ny, cx0 + scx[s], cy0 + dj, am, yb - dj, sa1[s], b1r - dj, stb[s] - tm, q, vz, dx, dy, dt);
        cy = dj;
      } else {
        deposit_segment(J, nx, ny, cx0 + scx[s], cy0 + cy, sa0[s], b0r, sa1[s], b1r, stb[s] - sta[s], q, vz, dx, dy, dt);
      }
    }
    /* cell update (a3, R6) */
    x1 -= di;
    if (x1 == 1.0) { x1 = 0.0; di += 1; }
    y1 -= dj;
    if (y1 == 1.0) { y1 = 0.0; dj += 1; }
    x[p] = x1; y[p] = y1;
    ix[p] = cx0 + di; iy[p] = cy0 + dj;
  }
  return bad;
}

/* ------------------------------------------------------------------------------------ */
/* Guard refresh of a 3-component grid ("each region updates the values of the
 * EM fields in their ghost cells").  Periodic axis: guards are copies of the opposite
 * interior (-1 <- n-1, n <- 0, n+1 <- 1), x first over all rows, then y over all columns.
 * Non-periodic axis: guards are set to 0, except that for Mur (open) boundaries the caller
 * passes keep_hi_node = 1 to keep the first high guard node (the Mur-updated boundary node
 * of tangential E, R13) untouched. */
static void refresh_axis_x(double* F, int nx, int ny, int c, int bcx, int keep_hi_node) {
  for (int j = -1; j <= ny + 1; ++j) {
    if (bcx == BC_PERIODIC) {
      F[fidx(nx, ny, c, -1, j)] = F[fidx(nx, ny, c, nx - 1, j)];
      F[fidx(nx, ny, c, nx, j)] = F[fidx(nx, ny, c, 0, j)];
      F[fidx(nx, ny, c, nx + 1, j)] = F[fidx(nx, ny, c, 1, j)];
    } else {
      F[fidx(nx, ny, c, -1, j)] = 0.0;
      if (!keep_hi_node) F[fidx(nx, ny, c, nx, j)] = 0.0;
      F[fidx(nx, ny, c, nx + 1, j)] = 0.0;
    }
  }
}
static void refresh_axis_y(double* F, int nx, int ny, int c, int bcy, int keep_hi_node) {
  for (int i = -1; i <= nx + 1; ++i) {
    if (bcy == BC_PERIODIC) {
      F[fidx(nx, ny, c, i, -1)] = F[fidx(nx, ny, c, i, ny - 1)];
      F[fidx(nx, ny, c, i, ny)] = F[fidx(nx, ny, c, i, 0)];
      F[fidx(nx, ny, c, i, ny + 1)] = F[fidx(nx, ny, c, i, 1)];
    } else {
      F[fidx(nx, ny, c, i, -1)] = 0.0;
      if (!keep_hi_node) F[fidx(nx, ny, c, i, ny)] = 0.0;
      F[fidx(nx, ny, c, i, ny + 1)] = 0.0;
    }
  }
}
/* is_E selects which components are tangential E nodes on an open edge: on an x edge
 * (Ey, Ez), on a y edge (Ex, Ez) (R13). */
void orc_refresh_guards(double* F, int nx, int ny, int bcx, int bcy, int is_E) {
  for (int c = 0; c < 3; ++c) {
    int keepx = is_E && bcx == BC_OPEN && (c == 1 || c == 2);
    int keepy = is_E && bcy == BC_OPEN && (c == 0 || c == 2);
    refresh_axis_x(F, nx, ny, c, bcx, keepx);
    refresh_axis_y(F, nx, ny, c, bcy, keepy);
  }
}

/* ------------------------------------------------------------------------------------ */
/* Ghost-current reduction ("the reduction is only required for ghost cells";
 * SURVEY §8(c) step 4, a7).  Periodic axis: add the guard deposits into the opposite
 * interior cells (-1 -> n-1; n, n+1 -> 0, 1), x first over all rows, then y; then refresh
 * the guards as periodic copies.  Open / window axis: guard deposits are discarded (guards
 * zeroed). */
void orc_fold_current(double* J, int nx, int ny, int bcx, int bcy) {
  for (int c = 0; c < 3; ++c) {
    if (bcx == BC_PERIODIC) {
      for (int j = -1; j <= ny + 1; ++j) {
        J[fidx(nx, ny, c, nx - 1, j)] += J[fidx(nx, ny, c, -1, j)];
        J[fidx(nx, ny, c, 0, j)] += J[fidx(nx, ny, c, nx, j)];
        J[fidx(nx, ny, c, 1, j)] += J[fidx(nx, ny, c, nx + 1, j)];
      }
    }
    if (bcy == BC_PERIODIC) {
      for (int i = -1; i <= nx + 1; ++i) {
        J[fidx(nx, ny, c, i, ny - 1)] += J[fidx(nx, ny, c, i, -1)];
        J[fidx(nx, ny, c, i, 0)] += J[fidx(nx, ny, c, i, ny)];
        J[fidx(nx, ny, c, i, 1)] += J[fidx(nx, ny, c, i, ny + 1)];
      }
    }
    refresh_axis_x(J, nx, ny, c, bcx, 0);
    refresh_axis_y(J, nx, ny, c, bcy, 0);
  }
}

/* ------------------------------------------------------------------------------------ */
/* Digital current filter along x ("digital filter on the current density",
 * PAPER.md:327 "compensated binomial filter"; R12): n passes of (1/4, 1/2, 1/4), then, if
 * compensated, one pass of (-n/4, 1 + n/2, -n/4).  Guards refreshed before every pass
 * (periodic copy, or zeros on a non-periodic x axis).  Interior rows only. */
static void filter_pass(double* J, int nx, int ny, int bcx, int bcy, double side, double centre,
                        double* row) {
  for (int c = 0; c < 3; ++c) {
    refresh_axis_x(J, nx, ny, c, bcx, 0);
    for (int j = 0; j < ny; ++j) {
      for (int i = -1; i <= nx; ++i) row[i + 1] = J[fidx(nx, ny, c, i, j)];
      for (int i = 0; i < nx; ++i)
        J[fidx(nx, ny, c, i, j)] = side * row[i] + centre * row[i + 1] + side * row[i + 2];
    }
    refresh_axis_x(J, nx, ny, c, bcx, 0);
    refresh_axis_y(J, nx, ny, c, bcy, 0);
  }
}
/* row: scratch of nx+2 doubles */
void orc_filter_x(double* J, int nx, int ny, int bcx, int bcy, int n_pass, int compensated,
                  double* row) {
  for (int k = 0; k < n_pass; ++k) filter_pass(J, nx, ny, bcx, bcy, 0.25, 0.5, row);
  if (compensated && n_pass > 0)
    filter_pass(J, nx, ny, bcx, bcy, -0.25 * n_pass, 1.0 + 0.5 * n_pass, row);
}

/* ------------------------------------------------------------------------------------ */
/* (4) Yee FDTD advance: B half step, E full step,
 * B half step, each followed by a guard refresh.
 *   Bx -= h/dy (Ez[i,j+1]-Ez[i,j]);  By += h/dx (Ez[i+1,j]-Ez[i,j]);
 *   Bz += h/dy (Ex[i,j+1]-Ex[i,j]) - h/dx (Ey[i+1,j]-Ey[i,j]);          (h = dt/2)
 *   Ex += dt/dy (Bz[i,j]-Bz[i,j-1]) - dt Jx;  Ey -= dt/dx (Bz[i,j]-Bz[i-1,j]) + dt Jy;
 *   Ez += dt/dx (By[i,j]-By[i-1,j]) - dt/dy (Bx[i,j]-Bx[i,j-1]) - dt Jz.
 * Open edges (R13): first-order Mur on the tangential E of the boundary node line, applied
 * right after the interior E update with saved E^n values:
 *   E^{n+1}_b = E^n_{b'} + k (E^{n+1}_{b'} - E^n_b),  k = (dt - d)/(dt + d),
 *   low edge b = 0, b' = 1; high edge b = n (first high guard), b' = n-1.
 * x edges act on (Ey, Ez) (curl update skipped at node 0), y edges on (Ex, Ez).  A node on two
 * open edges (Ez at the four corners) takes the y-edge Mur, from its y neighbour (R13 corner rule).
 * save: scratch of 4*(max(nx,ny)+3) doubles per component pair (caller-provided). */
static void b_half(double* B, const double* E, int nx, int ny, double h, double dx, double dy) {
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      B[fidx(nx, ny, 0, i, j)] -= h / dy * (E[fidx(nx, ny, 2, i, j + 1)] - E[fidx(nx, ny, 2, i, j)]);
      B[fidx(nx, ny, 1, i, j)] += h / dx * (E[fidx(nx, ny, 2, i + 1, j)] - E[fidx(nx, ny, 2, i, j)]);
      B[fidx(nx, ny, 2, i, j)] += h / dy * (E[fidx(nx, ny, 0, i, j + 1)] - E[fidx(nx, ny, 0, i, j)])
                                - h / dx * (E[fidx(nx, ny, 1, i + 1, j)] - E[fidx(nx, ny, 1, i, j)]);
    }
}

void orc_yee_advance(double* E, double* B, const double* J, int nx, int ny, double dt, double dx,
                     double dy, int bcx, int bcy, double* save) {
  double h = 0.5 * dt;
  b_half(B, E, nx, ny, h, dx, dy);
  orc_refresh_guards(B, nx, ny, bcx, bcy, 0);

  /* save E^n on the Mur node lines: per edge 2 lines (b, b') x 2 components */
  int L = (nx > ny ? nx : ny) + 3;
  double* sxlo = save;            /* x edges: [comp(Ey,Ez)][line b/b'][j] */
  double* sxhi = save + 4 * L;
  double* sylo = save + 8 * L;    /* y edges: [comp(Ex,Ez)][line][i] */
  double* syhi = save + 12 * L;
  if (bcx == BC_OPEN)
    for (int k = 0; k < 2; ++k) {
      int c = (k == 0) ? 1 : 2;
      for (int j = 0; j <= ny; ++j) {
        sxlo[(2 * k + 0) * L + j] = E[fidx(nx, ny, c, 0, j)];
        sxlo[(2 * k + 1) * L + j] = E[fidx(nx, ny, c, 1, j)];
        sxhi[(2 * k + 0) * L + j] = E[fidx(nx, ny, c, nx, j)];
        sxhi[(2 * k + 1) * L + j] = E[fidx(nx, ny, c, nx - 1, j)];
      }
    }
  if (bcy == BC_OPEN)
    for (int k = 0; k < 2; ++k) {
      int c = (k == 0) ? 0 : 2;
      for (int i = 0; i <= nx; ++i) {
        sylo[(2 * k + 0) * L + i] = E[fidx(nx, ny, c, i, 0)];
        sylo[(2 * k + 1) * L + i] = E[fidx(nx, ny, c, i, 1)];
        syhi[(2 * k + 0) * L + i] = E[fidx(nx, ny, c, i, ny)];
        syhi[(2 * k + 1) * L + i] = E[fidx(nx, ny, c, i, ny - 1)];
      }
    }

  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      int mur_x = (bcx == BC_OPEN && i == 0);   /* node line x = 0 */
      int mur_y = (bcy == BC_OPEN && j == 0);   /* node line y = 0 */
      /* Mur nodes (tangential E on an open edge) are set after this loop */
      if (!mur_y)
        E[fidx(nx, ny, 0, i, j)] += dt / dy * (B[fidx(nx, ny, 2, i, j)] - B[fidx(nx, ny, 2, i, j - 1)]) - dt * J[fidx(nx, ny, 0, i, j)];
      if (!mur_x)
        E[fidx(nx, ny, 1, i, j)] += -dt / dx * (B[fidx(nx, ny, 2, i, j)] - B[fidx(nx, ny, 2, i - 1, j)]) - dt * J[fidx(nx, ny, 1, i, j)];
      if (!mur_x && !mur_y)
        E[fidx(nx, ny, 2, i, j)] += dt / dx * (B[fidx(nx, ny, 1, i, j)] - B[fidx(nx, ny, 1, i - 1, j)])
                                  - dt / dy * (B[fidx(nx, ny, 0, i, j)] - B[fidx(nx, ny, 0, i, j - 1)]) - dt * J[fidx(nx, ny, 2, i, j)];
    }

  if (bcx == BC_OPEN) {
    double kx = (dt - dx) / (dt + dx);
    for (int k = 0; k < 2; ++k) {
      int c = (k == 0) ? 1 : 2;
      for (int j = 0; j < ny; ++j) {
        if (c == 2 && bcy == BC_OPEN && j == 0) continue;  /* corner node: the y Mur below (R13) */
        E[fidx(nx, ny, c, 0, j)] = sxlo[(2 * k + 1) * L + j] + kx * (E[fidx(nx, ny, c, 1, j)] - sxlo[(2 * k + 0) * L + j]);
        E[fidx(nx, ny, c, nx, j)] = sxhi[(2 * k + 1) * L + j] + kx * (E[fidx(nx, ny, c, nx - 1, j)] - sxhi[(2 * k + 0) * L + j]);
      }
    }
  }
  if (bcy == BC_OPEN) {
    double ky = (dt - dy) / (dt + dy);
    for (int k = 0; k < 2; ++k) {
      int c = (k == 0) ? 0 : 2;
      /* corner rule (R13): a node on two open edges (Ez at (0,0), (nx,0), (0,ny),
       * (nx,ny)) follows the y-edge Mur, so the y node line of Ez runs over i = 0 .. nx when x is
       * open too (Ex node nx lies outside the box: held at 0) */
      int iend = (c == 2 && bcx == BC_OPEN) ? nx : nx - 1;
      for (int i = 0; i <= iend; ++i) {
        E[fidx(nx, ny, c, i, 0)] = sylo[(2 * k + 1) * L + i] + ky * (E[fidx(nx, ny, c, i, 1)] - sylo[(2 * k + 0) * L + i]);
        E[fidx(nx, ny, c, i, ny)] = syhi[(2 * k + 1) * L + i] + ky * (E[fidx(nx, ny, c, i, ny - 1)] - syhi[(2 * k + 0) * L + i]);
      }
    }
  }
  orc_refresh_guards(E, nx, ny, bcx, bcy, 1);

  b_half(B, E, nx, ny, h, dx, dy);
  orc_refresh_guards(B, nx, ny, bcx, bcy, 0);
}

/* ------------------------------------------------------------------------------------ */
/* FE(n) = 1/2 dx dy sum_interior (|E|^2 + |B|^2)  (R8). */
double orc_field_energy(const double* E, const double* B, int nx, int ny, double dx, double dy) {
  double s = 0.0;
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        double e = E[fidx(nx, ny, c, i, j)], b = B[fidx(nx, ny, c, i, j)];
        s += e * e + b * b;
      }
  return 0.5 * dx * dy * s;
}
