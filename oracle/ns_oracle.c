/*
 * ns_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU checker for the north-star HB Euler / laminar Navier-Stokes path
 * (SURVEY.md §8 row f2), a plain-C restatement of the specification in
 * paper_1304_7654_b200/nsflow.py's docstring, written independently of the
 * CUDA kernels (hb_ns.cu).  The reference (hbproxy) has no such physics
 * (hbcore.py:3-13), so this oracle is NOT pinned to any
 * reference output: parity for this row is "unpinned".
 * Compiled with -ffp-contract=off: every multiply / add / divide / sqrt is
 * separately rounded, in the order written.
 *
 * Layout (per block): states (P, 4, nj+4, ni+4), cell (i, j) -- i, j in
 * [-1, n+2] -- at [j+1][i+1]; node coordinates (Pg, nj+5, ni+5), node (I, J)
 * -- I, J in [-2, n+2] -- at [J+2][I+2]; geometry as nsflow.metrics.
 */
#include <math.h>
#include <stddef.h>
#include <string.h>

#define GAMMA 1.4
#define PR 0.72
#define K2 0.5
#define K4 (1.0 / 64.0)
#define NV 4

typedef struct {
    int ni, nj, P, Pg;
    const double *x, *y;         /* nodes (Pg, nj+5, ni+5) */
    const double *xt, *yt;       /* node velocities or NULL */
    int kinds[4];                /* south, north, west, east: 0 far, 1 no-slip, 2 slip, 3 cut */
    double *xc, *yc, *vol;       /* (Pg, nj+4, ni+4) */
    double *six, *siy, *gi;      /* (Pg, nj+4, ni+5) */
    double *sjx, *sjy, *gj;      /* (Pg, nj+5, ni+4) */
} nsblock_t;

/* ---- indexing ---------------------------------------------------------------- */

static inline size_t NX(const nsblock_t *b) { return (size_t)b->ni + 5; }
static inline size_t nd(const nsblock_t *b, int g, int J, int I) {   /* node */
    return ((size_t)g * (b->nj + 5) + (J + 2)) * NX(b) + (I + 2);
}
static inline size_t cc(const nsblock_t *b, int g, int j, int i) {   /* cell geometry */
    return ((size_t)g * (b->nj + 4) + (j + 1)) * (b->ni + 4) + (i + 1);
}
static inline size_t fi(const nsblock_t *b, int g, int j, int i) {   /* i-face east of cell i */
    return ((size_t)g * (b->nj + 4) + (j + 1)) * (b->ni + 5) + (i + 2);
}
static inline size_t fj(const nsblock_t *b, int g, int j, int i) {   /* j-face north of cell j */
    return ((size_t)g * (b->nj + 5) + (j + 2)) * (b->ni + 4) + (i + 1);
}
static inline size_t ws(const nsblock_t *b, int n, int k, int j, int i) {   /* state */
    return (((size_t)n * NV + k) * (b->nj + 4) + (j + 1)) * (b->ni + 4) + (i + 1);
}
static inline size_t rs(const nsblock_t *b, int n, int k, int j, int i) {   /* residual, interior */
    return (((size_t)n * NV + k) * b->nj + (j - 1)) * b->ni + (i - 1);
}

/* ---- geometry (nsflow.metrics) ---------------------------------------------------- */

void ns_geometry(nsblock_t *b) {
    for (int g = 0; g < b->Pg; ++g) {
        for (int j = -1; j <= b->nj + 2; ++j)
            for (int i = -1; i <= b->ni + 2; ++i) {
                /* cell (i, j): nodes (i-1, j-1) 00, (i, j-1) 10, (i, j) 11, (i-1, j) 01 */
                double x00 = b->x[nd(b, g, j - 1, i - 1)], x10 = b->x[nd(b, g, j - 1, i)];
                double x11 = b->x[nd(b, g, j, i)], x01 = b->x[nd(b, g, j, i - 1)];
                double y00 = b->y[nd(b, g, j - 1, i - 1)], y10 = b->y[nd(b, g, j - 1, i)];
                double y11 = b->y[nd(b, g, j, i)], y01 = b->y[nd(b, g, j, i - 1)];
                b->xc[cc(b, g, j, i)] = 0.25 * ((x00 + x10) + (x11 + x01));
                b->yc[cc(b, g, j, i)] = 0.25 * ((y00 + y10) + (y11 + y01));
                b->vol[cc(b, g, j, i)] = 0.5 * ((x11 - x00) * (y01 - y10) - (y11 - y00) * (x01 - x10));
            }
        /* i-face at node column I between nodes (I, J-1) and (I, J): cell row j = J */
        for (int j = -1; j <= b->nj + 2; ++j)
            for (int I = -2; I <= b->ni + 2; ++I) {
                size_t f = fi(b, g, j, I);
                double ya = b->y[nd(b, g, j - 1, I)], yb = b->y[nd(b, g, j, I)];
                double xa = b->x[nd(b, g, j - 1, I)], xb = b->x[nd(b, g, j, I)];
                b->six[f] = yb - ya;
                b->siy[f] = xa - xb;
                if (b->xt) {
                    double ut = 0.5 * (b->xt[nd(b, g, j, I)] + b->xt[nd(b, g, j - 1, I)]);
                    double vt = 0.5 * (b->yt[nd(b, g, j, I)] + b->yt[nd(b, g, j - 1, I)]);
                    b->gi[f] = ut * b->six[f] + vt * b->siy[f];
                }
            }
        /* j-face at node row J between nodes (I-1, J) and (I, J): cell column i = I */
        for (int J = -2; J <= b->nj + 2; ++J)
            for (int i = -1; i <= b->ni + 2; ++i) {
                size_t f = fj(b, g, J, i);
                double ya = b->y[nd(b, g, J, i - 1)], yb = b->y[nd(b, g, J, i)];
                double xa = b->x[nd(b, g, J, i - 1)], xb = b->x[nd(b, g, J, i)];
                b->sjx[f] = ya - yb;
                b->sjy[f] = xb - xa;
                if (b->xt) {
                    double ut = 0.5 * (b->xt[nd(b, g, J, i - 1)] + b->xt[nd(b, g, J, i)]);
                    double vt = 0.5 * (b->yt[nd(b, g, J, i - 1)] + b->yt[nd(b, g, J, i)]);
                    b->gj[f] = ut * b->sjx[f] + vt * b->sjy[f];
                }
            }
    }
}

/* ---- thermodynamics ------------------------------------------------------------------ */

typedef struct {
    double r, ru, rv, re, u, v, p, c, e;
} prim_t;

static inline prim_t prim(const double *w, size_t stride) {
    prim_t q;
    q.r = w[0];
    q.ru = w[stride];
    q.rv = w[2 * stride];
    q.re = w[3 * stride];
    q.u = q.ru / q.r;
    q.v = q.rv / q.r;
    q.p = (GAMMA - 1.0) * (q.re - 0.5 * (q.ru * q.u + q.rv * q.v));
    q.c = sqrt(GAMMA * q.p / q.r);
    q.e = q.p / ((GAMMA - 1.0) * q.r);
    return q;
}

/* ---- boundary halos -------------------------------------------------------------------- */

/* ghost state from interior state q for a side of kind `kind`, boundary face
 * normal (sx, sy) and grid flux g (slip wall), freestream winf */
static void ghost(int kind, const prim_t *q, double sx, double sy, double g, const double *winf, double *out) {
    if (kind == 0) {
        for (int k = 0; k < NV; ++k) out[k] = winf[k];
    } else if (kind == 1) {
        out[0] = q->r;
        out[1] = -q->ru;
        out[2] = -q->rv;
        out[3] = q->re;
    } else {
        double sa = sqrt(sx * sx + sy * sy);
        double nx = sx / sa, ny = sy / sa;
        double vn = (q->u * nx + q->v * ny) - g / sa;
        double ug = q->u - 2.0 * vn * nx;
        double vg = q->v - 2.0 * vn * ny;
        out[0] = q->r;
        out[1] = q->r * ug;
        out[2] = q->r * vg;
        out[3] = q->p / (GAMMA - 1.0) + (0.5 * q->r) * (ug * ug + vg * vg);
    }
}

/* non-cut sides: two halo layers; then the corner halos */
void ns_boundaries(const nsblock_t *b, double *w, const double *winf /* P x 4 */) {
    const size_t st = (size_t)(b->nj + 4) * (b->ni + 4);
    for (int n = 0; n < b->P; ++n) {
        const int g = b->Pg > 1 ? n : 0;
        double out[NV];
        for (int side = 0; side < 4; ++side) {
            const int kind = b->kinds[side];
            if (kind == 3) continue;
            for (int layer = 1; layer <= 2; ++layer) {
                const int len = side < 2 ? b->ni : b->nj;
                for (int e = 1; e <= len; ++e) {
                    int hi_, hj, ii, ij;
                    double sx, sy, gg = 0.0;
                    if (side == 0) {        /* south: halo (e, 1-layer) <- (e, layer); face j = 1/2 */
                        hi_ = e; hj = 1 - layer; ii = e; ij = layer;
                        sx = b->sjx[fj(b, g, 0, e)]; sy = b->sjy[fj(b, g, 0, e)];
                        if (b->xt) gg = b->gj[fj(b, g, 0, e)];
                    } else if (side == 1) { /* north */
                        hi_ = e; hj = b->nj + layer; ii = e; ij = b->nj + 1 - layer;
                        sx = b->sjx[fj(b, g, b->nj, e)]; sy = b->sjy[fj(b, g, b->nj, e)];
                        if (b->xt) gg = b->gj[fj(b, g, b->nj, e)];
                    } else if (side == 2) { /* west */
                        hi_ = 1 - layer; hj = e; ii = layer; ij = e;
                        sx = b->six[fi(b, g, e, 0)]; sy = b->siy[fi(b, g, e, 0)];
                        if (b->xt) gg = b->gi[fi(b, g, e, 0)];
                    } else {                /* east */
                        hi_ = b->ni + layer; hj = e; ii = b->ni + 1 - layer; ij = e;
                        sx = b->six[fi(b, g, e, b->ni)]; sy = b->siy[fi(b, g, e, b->ni)];
                        if (b->xt) gg = b->gi[fi(b, g, e, b->ni)];
                    }
                    prim_t q = prim(w + ws(b, n, 0, ij, ii), st);
                    ghost(kind, &q, sx, sy, gg, winf + NV * n, out);
                    for (int k = 0; k < NV; ++k) w[ws(b, n, k, hj, hi_)] = out[k];
                }
            }
        }
        /* corners: the i-halo cell of the nearest interior row */
        for (int k = 0; k < NV; ++k)
            for (int i = -1; i <= b->ni + 2; ++i) {
                if (i >= 1 && i <= b->ni) continue;
                for (int j = -1; j <= 0; ++j) w[ws(b, n, k, j, i)] = w[ws(b, n, k, 1, i)];
                for (int j = b->nj + 1; j <= b->nj + 2; ++j) w[ws(b, n, k, j, i)] = w[ws(b, n, k, b->nj, i)];
            }
    }
}

/* ---- fluxes --------------------------------------------------------------------------- */

typedef struct {
    const nsblock_t *b;
    const double *w;
    size_t st;
    int n, g;
    double mu;
} ctx_t;

static inline prim_t P_at(const ctx_t *c, int j, int i) { return prim(c->w + ws(c->b, c->n, 0, j, i), c->st); }
static inline double W_at(const ctx_t *c, int k, int j, int i) { return c->w[ws(c->b, c->n, k, j, i)]; }

/* face flux between L = (iL, jL) and R = (iL+di, jL+dj), normal (sx, sy), grid flux gf */
static void face_flux(const ctx_t *c, int jL, int iL, int dj, int di, double sx, double sy, double gf,
                      double *out) {
    const int jR = jL + dj, iR = iL + di;
    prim_t L = P_at(c, jL, iL), R = P_at(c, jR, iR);
    prim_t LL = P_at(c, jL - dj, iL - di), RR = P_at(c, jR + dj, iR + di);
    double unL = L.u * sx + L.v * sy, unR = R.u * sx + R.v * sy;
    double urL = unL - gf, urR = unR - gf;
    double FL[NV] = {L.r * urL, L.ru * urL + L.p * sx, L.rv * urL + L.p * sy, L.re * urL + L.p * unL};
    double FR[NV] = {R.r * urR, R.ru * urR + R.p * sx, R.rv * urR + R.p * sy, R.re * urR + R.p * unR};
    double sa = sqrt(sx * sx + sy * sy);
    double lamL = fabs(urL) + L.c * sa, lamR = fabs(urR) + R.c * sa;
    double lam = 0.5 * (lamL + lamR);
    double nuL = fabs((R.p - 2.0 * L.p) + LL.p) / ((R.p + 2.0 * L.p) + LL.p);
    double nuR = fabs((RR.p - 2.0 * R.p) + L.p) / ((RR.p + 2.0 * R.p) + L.p);
    double eps2 = (K2 * lam) * fmax(nuL, nuR);
    double eps4 = fmax(0.0, K4 * lam - eps2);
    double fv[NV] = {0.0, 0.0, 0.0, 0.0};
    if (c->mu > 0.0) {
        /* diamond: tangential neighbours across the face's other index */
        const int tj = di, ti = dj;   /* i-face: (j +- 1); j-face: (i +- 1) */
        prim_t Lp = P_at(c, jL + tj, iL + ti), Rp = P_at(c, jR + tj, iR + ti);
        prim_t Lm = P_at(c, jL - tj, iL - ti), Rm = P_at(c, jR - tj, iR - ti);
        const nsblock_t *b = c->b;
        const int g = c->g;
        double xL = b->xc[cc(b, g, jL, iL)], xR = b->xc[cc(b, g, jR, iR)];
        double yL = b->yc[cc(b, g, jL, iL)], yR = b->yc[cc(b, g, jR, iR)];
        double xLp = b->xc[cc(b, g, jL + tj, iL + ti)], xRp = b->xc[cc(b, g, jR + tj, iR + ti)];
        double xLm = b->xc[cc(b, g, jL - tj, iL - ti)], xRm = b->xc[cc(b, g, jR - tj, iR - ti)];
        double yLp = b->yc[cc(b, g, jL + tj, iL + ti)], yRp = b->yc[cc(b, g, jR + tj, iR + ti)];
        double yLm = b->yc[cc(b, g, jL - tj, iL - ti)], yRm = b->yc[cc(b, g, jR - tj, iR - ti)];
        double x_a = xR - xL, y_a = yR - yL;
        double x_b = 0.25 * ((xLp + xRp) - (xLm + xRm)), y_b = 0.25 * ((yLp + yRp) - (yLm + yRm));
        double jac = x_a * y_b - x_b * y_a;
        double ua = R.u - L.u, ub = 0.25 * ((Lp.u + Rp.u) - (Lm.u + Rm.u));
        double va = R.v - L.v, vb = 0.25 * ((Lp.v + Rp.v) - (Lm.v + Rm.v));
        double ea = R.e - L.e, eb = 0.25 * ((Lp.e + Rp.e) - (Lm.e + Rm.e));
        double ux = (ua * y_b - ub * y_a) / jac, uy = (ub * x_a - ua * x_b) / jac;
        double vx = (va * y_b - vb * y_a) / jac, vy = (vb * x_a - va * x_b) / jac;
        double ex = (ea * y_b - eb * y_a) / jac, ey = (eb * x_a - ea * x_b) / jac;
        double mu = c->mu;
        double div = ux + vy;
        double txx = mu * (2.0 * ux - (2.0 / 3.0) * div);
        double tyy = mu * (2.0 * vy - (2.0 / 3.0) * div);
        double txy = mu * (uy + vx);
        double kq = mu * GAMMA / PR;
        double qx = -(kq * ex), qy = -(kq * ey);
        double uf = 0.5 * (L.u + R.u), vf = 0.5 * (L.v + R.v);
        fv[1] = txx * sx + txy * sy;
        fv[2] = txy * sx + tyy * sy;
        fv[3] = ((uf * txx + vf * txy) - qx) * sx + ((uf * txy + vf * tyy) - qy) * sy;
    }
    for (int k = 0; k < NV; ++k) {
        double wl = W_at(c, k, jL, iL), wr = W_at(c, k, jR, iR);
        double wll = W_at(c, k, jL - dj, iL - di), wrr = W_at(c, k, jR + dj, iR + di);
        double fc = 0.5 * (FL[k] + FR[k]);
        double d = eps2 * (wr - wl) - eps4 * (((wrr - 3.0 * wr) + 3.0 * wl) - wll);
        out[k] = c->mu > 0.0 ? (fc - d) - fv[k] : fc - d;
    }
}

/* spatial residual of every interior cell and snapshot into r (P, 4, nj, ni) */
void ns_residual(const nsblock_t *b, const double *w, double *r, double mu) {
    ctx_t c = {b, w, (size_t)(b->nj + 4) * (b->ni + 4), 0, 0, mu};
    for (int n = 0; n < b->P; ++n) {
        c.n = n;
        c.g = b->Pg > 1 ? n : 0;
        const int g = c.g;
        for (int j = 1; j <= b->nj; ++j)
            for (int i = 1; i <= b->ni; ++i) {
                double fe[NV], fw[NV], fn[NV], fs[NV];
                face_flux(&c, j, i, 0, 1, b->six[fi(b, g, j, i)], b->siy[fi(b, g, j, i)],
                          b->xt ? b->gi[fi(b, g, j, i)] : 0.0, fe);
                face_flux(&c, j, i - 1, 0, 1, b->six[fi(b, g, j, i - 1)], b->siy[fi(b, g, j, i - 1)],
                          b->xt ? b->gi[fi(b, g, j, i - 1)] : 0.0, fw);
                face_flux(&c, j, i, 1, 0, b->sjx[fj(b, g, j, i)], b->sjy[fj(b, g, j, i)],
                          b->xt ? b->gj[fj(b, g, j, i)] : 0.0, fn);
                face_flux(&c, j - 1, i, 1, 0, b->sjx[fj(b, g, j - 1, i)], b->sjy[fj(b, g, j - 1, i)],
                          b->xt ? b->gj[fj(b, g, j - 1, i)] : 0.0, fs);
                for (int k = 0; k < NV; ++k) r[rs(b, n, k, j, i)] = ((fe[k] - fw[k]) + fn[k]) - fs[k];
            }
    }
}

/* local time step of every interior cell from the state w (all snapshots) */
void ns_timestep(const nsblock_t *b, const double *w, double *dt, double mu, double cfl, double omega_nh) {
    const size_t st = (size_t)(b->nj + 4) * (b->ni + 4);
    for (int j = 1; j <= b->nj; ++j)
        for (int i = 1; i <= b->ni; ++i) {
            double best = 0.0;
            for (int n = 0; n < b->P; ++n) {
                const int g = b->Pg > 1 ? n : 0;
                prim_t q = prim(w + ws(b, n, 0, j, i), st);
                double ax = b->six[fi(b, g, j, i - 1)], ay = b->siy[fi(b, g, j, i - 1)];
                double bx = b->six[fi(b, g, j, i)], by = b->siy[fi(b, g, j, i)];
                double cx = b->sjx[fj(b, g, j - 1, i)], cy = b->sjy[fj(b, g, j - 1, i)];
                double dx = b->sjx[fj(b, g, j, i)], dy = b->sjy[fj(b, g, j, i)];
                double ga = b->xt ? b->gi[fi(b, g, j, i - 1)] : 0.0, gb = b->xt ? b->gi[fi(b, g, j, i)] : 0.0;
                double gc = b->xt ? b->gj[fj(b, g, j - 1, i)] : 0.0, gd = b->xt ? b->gj[fj(b, g, j, i)] : 0.0;
                double la = fabs((q.u * ax + q.v * ay) - ga) + q.c * sqrt(ax * ax + ay * ay);
                double lb = fabs((q.u * bx + q.v * by) - gb) + q.c * sqrt(bx * bx + by * by);
                double lc = fabs((q.u * cx + q.v * cy) - gc) + q.c * sqrt(cx * cx + cy * cy);
                double ld = fabs((q.u * dx + q.v * dy) - gd) + q.c * sqrt(dx * dx + dy * dy);
                double V = b->vol[cc(b, g, j, i)];
                double den = 0.5 * (la + lb) + 0.5 * (lc + ld);
                if (mu > 0.0) {
                    double sxi = 0.5 * (ax + bx), syi = 0.5 * (ay + by);
                    double sxj = 0.5 * (cx + dx), syj = 0.5 * (cy + dy);
                    double lv = ((2.0 * GAMMA * mu) / (PR * q.r)) *
                                (((sxi * sxi + syi * syi) + (sxj * sxj + syj * syj)) / V);
                    den = den + lv;
                }
                den = den + omega_nh * V;
                double t = (cfl * V) / den;
                best = n == 0 ? t : fmin(best, t);
            }
            dt[(size_t)(j - 1) * b->ni + (i - 1)] = best;
        }
}

/* HB source + RK update: w_out = w0 - (coef dt / V) (R + V sum_m D[n][m] w_in[m]);
 * returns sum of (R_rho total)^2 when want_norm, into *sumsq (long double) */
int ns_update(const nsblock_t *b, const double *w_in, const double *w0, double *w_out, const double *r,
              const double *dt, const double *dmat, double coef, int want_norm, long double *sumsq) {
    int bad = 0;
    long double acc = 0.0L;
    for (int n = 0; n < b->P; ++n) {
        const int g = b->Pg > 1 ? n : 0;
        for (int k = 0; k < NV; ++k)
            for (int j = 1; j <= b->nj; ++j)
                for (int i = 1; i <= b->ni; ++i) {
                    double V = b->vol[cc(b, g, j, i)];
                    double s = dmat[n * b->P] * w_in[ws(b, 0, k, j, i)];
                    for (int m = 1; m < b->P; ++m) s = s + dmat[n * b->P + m] * w_in[ws(b, m, k, j, i)];
                    double R = r[rs(b, n, k, j, i)] + V * s;
                    if (want_norm && k == 0) acc += (long double)R * (long double)R;
                    double v = w0[ws(b, n, k, j, i)] - ((coef * dt[(size_t)(j - 1) * b->ni + (i - 1)]) / V) * R;
                    w_out[ws(b, n, k, j, i)] = v;
                    if (!isfinite(v)) bad = 1;
                }
    }
    if (want_norm) *sumsq += acc;
    return bad;
}

/* pressure forces on the wall sides, per snapshot: (fx, fy) folds in face
 * order, then rotated: cd = fx ca + fy sa, cl = fy ca - fx sa */
void ns_forces(const nsblock_t *b, const double *w, const double *ca, const double *sa, double *fxy /* P x 2 */) {
    const size_t st = (size_t)(b->nj + 4) * (b->ni + 4);
    for (int n = 0; n < b->P; ++n) {
        const int g = b->Pg > 1 ? n : 0;
        double fx = fxy[2 * n], fy = fxy[2 * n + 1];
        for (int side = 0; side < 4; ++side) {
            if (b->kinds[side] != 1 && b->kinds[side] != 2) continue;
            const int len = side < 2 ? b->ni : b->nj;
            for (int e = 1; e <= len; ++e) {
                int ci, cj;
                double sx, sy;
                if (side == 0) { ci = e; cj = 1; sx = b->sjx[fj(b, g, 0, e)]; sy = b->sjy[fj(b, g, 0, e)]; }
                else if (side == 1) { ci = e; cj = b->nj; sx = b->sjx[fj(b, g, b->nj, e)]; sy = b->sjy[fj(b, g, b->nj, e)]; }
                else if (side == 2) { ci = 1; cj = e; sx = b->six[fi(b, g, e, 0)]; sy = b->siy[fi(b, g, e, 0)]; }
                else { ci = b->ni; cj = e; sx = b->six[fi(b, g, e, b->ni)]; sy = b->siy[fi(b, g, e, b->ni)]; }
                prim_t q = prim(w + ws(b, n, 0, cj, ci), st);
                fx = fx + q.p * sx;
                fy = fy + q.p * sy;
            }
        }
        fxy[2 * n] = fx;
        fxy[2 * n + 1] = fy;
        (void)ca;
        (void)sa;
    }
}
